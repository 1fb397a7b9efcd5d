#!/usr/bin/env bash
# single-problem latency under each ab/lib<X>.so, alternating
O=gpurun_out/abl; mkdir -p $O
for rep in 1 2 3; do for X in "$@"; do
  echo -n "$X: " >> $O/out.txt
  PRRTC_B200_LIB=ab/lib$X.so timeout 200 python tools/lat.py ${ROBOT:-panda} 300 2>/dev/null >> $O/out.txt
done; done
