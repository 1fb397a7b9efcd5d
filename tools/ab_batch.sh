#!/usr/bin/env bash
# Batch kernel time (tools/batch_counters.py, 1000 problems, bench params) under
# each ab/lib<X>.so, alternating, REPS reps per robot:
#   bash tools/ab_batch.sh H N   -> gpurun_out/abb/out.txt
O=gpurun_out/abb; mkdir -p $O
for rep in $(seq ${REPS:-3}); do for r in ${ROBOTS:-panda fetch baxter}; do for X in "$@"; do
  echo -n "$X rep $rep: " >> $O/out.txt
  PRRTC_B200_LIB=ab/lib$X.so timeout 300 python tools/batch_counters.py $r 0 ${N:-1000} 2>&1 | head -1 | cut -c1-120 >> $O/out.txt
done; done; done
