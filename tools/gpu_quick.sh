#!/usr/bin/env bash
# quick GPU loop: parity tests, phase profile, bench (no CPU baseline)
T=${1:-q}
mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$T/pytest.log 2>&1
timeout 300 python tools/phase_profile.py > gpurun_out/$T/phase.txt 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline --latency-samples 50 > gpurun_out/$T/bench.json 2>gpurun_out/$T/bench.err
timeout 300 python tools/batch_stats.py panda 32:128 > gpurun_out/$T/batch.txt 2>&1
