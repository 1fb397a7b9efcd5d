#!/usr/bin/env bash
# One gpurun pass: GPU tests, smoke, bench line, ncu launch list, one ncu --set full
# capture of plan_kernel. Everything lands in gpurun_out/.
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tag]'
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"; lscpu > "$OUT/lscpu.txt" 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --latency-samples 10 --no-cpu-baseline --no-parity --no-extras \
      > "$OUT/ncu_bench.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:plan_kernel -s 2 -c 1 \
      -o "$OUT/plan_batch" python tools/profile_one.py panda 3 batch > "$OUT/ncu_full.log" 2>&1
fi
echo done > "$OUT/DONE"
