#!/usr/bin/env bash
# One gpurun pass of the full bench line only: gpurun_out/<tag>/bench.json
#   gpurun --timeout 1200 -- 'bash tools/bench_only.sh <tag>'
TAG=${1:-bench}
mkdir -p gpurun_out/$TAG
timeout 1100 python bench.py ${BENCH_ARGS:-} > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
echo "bench rc=$?" >> gpurun_out/$TAG/bench.err
