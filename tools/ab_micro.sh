#!/usr/bin/env bash
# microbenchmark kernels (tools/profile_micro.py) under each ab/lib<X>.so
O=gpurun_out/abm; mkdir -p $O
for rep in 1 2; do for X in "$@"; do
  echo "== $X rep $rep" >> $O/out.txt
  PRRTC_B200_LIB=ab/lib$X.so timeout 120 python tools/profile_micro.py ${ROBOT:-panda} >> $O/out.txt 2>&1
done; done
