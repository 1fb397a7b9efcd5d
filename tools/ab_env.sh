#!/usr/bin/env bash
# An environment knob's values alternated over batch kernel time
# (tools/batch_counters.py) per robot:
#   bash tools/ab_env.sh VAR "v1 v2 ..."  -> gpurun_out/env_VAR/out.txt
VAR=$1; O=gpurun_out/env_$VAR; mkdir -p $O
for rep in $(seq ${REPS:-2}); do for r in ${ROBOTS:-panda fetch baxter}; do for v in $2; do
  echo -n "$VAR=$v rep $rep: " >> $O/out.txt
  env $VAR=$v timeout 300 python tools/batch_counters.py $r 0 ${N:-1000} 2>&1 | head -1 | cut -c1-90 >> $O/out.txt
done; done; done
