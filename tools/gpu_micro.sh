#!/usr/bin/env bash
# microbench + chunk profile + GPU tests + two short benches (no CPU baseline, no extras)
T=${1:-m}
mkdir -p gpurun_out/$T
python tools/chunk_profile.py panda > gpurun_out/$T/cp.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/$T/pytest.log 2>&1
for i in 1 2; do
  timeout 400 python bench.py --steps 5 --no-cpu-baseline --no-extras --latency-samples 30 > gpurun_out/$T/bench$i.json 2> gpurun_out/$T/bench.err
done
