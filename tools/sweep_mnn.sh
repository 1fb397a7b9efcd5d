#!/usr/bin/env bash
# single-problem latency vs the multi-sample NN bound (PRRTC_MNN_NODES)
O=gpurun_out/mnn; mkdir -p $O
for rep in 1 2; do for v in 2048 1024 512 256 128; do
  echo -n "mnn $v: " >> $O/out.txt
  PRRTC_MNN_NODES=$v timeout 200 python tools/lat.py ${ROBOT:-panda} 300 2>/dev/null >> $O/out.txt
done; done
