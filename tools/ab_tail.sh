#!/usr/bin/env bash
# Ticket-block sizing near a problem's budget end (PRRTC_TAIL_MIN / _DIV),
# batch kernel time per robot:  bash tools/ab_tail.sh "4,2 1,2 ..."  -> gpurun_out/tail/out.txt
O=gpurun_out/tail; mkdir -p $O
for rep in $(seq ${REPS:-1}); do for r in ${ROBOTS:-panda fetch baxter}; do for v in $1; do
  mn=${v%,*}; dv=${v#*,}
  echo -n "min $mn div $dv rep $rep: " >> $O/out.txt
  PRRTC_TAIL_MIN=$mn PRRTC_TAIL_DIV=$dv timeout 300 python tools/batch_counters.py $r 0 ${N:-1000} 2>&1 | head -1 | cut -c1-100 >> $O/out.txt
done; done; done
