#!/usr/bin/env bash
# A/B the planner libraries ab/lib<X>.so in one box session:
#   bash tools/ab.sh A B   -> gpurun_out/ab/<X>_<rep>.json (+ baxter batch)
O=gpurun_out/ab; mkdir -p $O
for rep in 1 2; do
  for X in "$@"; do
    PRRTC_B200_LIB=ab/lib$X.so timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-extras --latency-samples 60 > $O/${X}_$rep.json 2>/dev/null
    PRRTC_B200_LIB=ab/lib$X.so timeout 300 python tools/batch_work.py ${ROBOT:-baxter} > $O/${X}_${rep}_work.txt 2>&1
  done
done
