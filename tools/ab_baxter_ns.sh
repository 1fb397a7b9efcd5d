#!/usr/bin/env bash
# Baxter batch with 32- vs 64-state chunks (256-thread CTAs)
O=gpurun_out/abns; mkdir -p $O
for rep in 1 2; do
  echo "ns32 $rep" >> $O/bax.txt; timeout 300 python tools/batch_work.py baxter 2>/dev/null | head -3 >> $O/bax.txt
  echo "ns64 $rep" >> $O/bax.txt; PRRTC_NS64=1 timeout 300 python tools/batch_work.py baxter 2>/dev/null | head -3 >> $O/bax.txt
done
