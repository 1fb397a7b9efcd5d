#!/usr/bin/env bash
# occupancy experiment: plan_kernel<128, MINB> for MINB = 4, 5, 6 (batch only)
mkdir -p gpurun_out/minb
for m in 4 5 4 5; do
  PRRTC_PLAN_MINB=$m timeout 300 python tools/batch_stats.py panda 32:128 >> gpurun_out/minb/batch_$m.txt 2>&1
done
