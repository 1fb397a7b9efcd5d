#!/usr/bin/env bash
# occupancy experiment: plan_kernel<128, MINB> for MINB = 4, 5, 6
mkdir -p gpurun_out/minb
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/minb/pytest.log 2>&1
for m in 4 5 6; do
  PRRTC_PLAN_MINB=$m timeout 300 python tools/batch_stats.py panda 32:128 > gpurun_out/minb/batch_$m.txt 2>&1
  PRRTC_PLAN_MINB=$m timeout 300 python bench.py --steps 5 --no-cpu-baseline --latency-samples 50 > gpurun_out/minb/bench_$m.json 2>gpurun_out/minb/bench_$m.err
done
