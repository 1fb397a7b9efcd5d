#!/usr/bin/env bash
# compute-sanitizer passes over the planner kernels:
#   gpurun --timeout 2400 -- 'bash tools/sanitize.sh r2'
# memcheck / synccheck / racecheck on single problems (few and many CTAs on one
# problem: concurrent tree appends) and small batches (CTAs joining problems),
# plus memcheck over the GPU parity tests (checking and debug kernels).
set -u
TAG=${1:-r2}
OUT=gpurun_out/$TAG/sanitizer
mkdir -p "$OUT"
CS="compute-sanitizer --print-limit 100"
run() { local name=$1; shift; timeout 1200 env PRRTC_WARP=${PRRTC_WARP:-} $CS "$@" > "$OUT/$name.log" 2>&1; echo "$name rc=$?" >> "$OUT/summary.txt"; tail -3 "$OUT/$name.log" >> "$OUT/summary.txt"; }
run memcheck_single16   --tool memcheck  python tools/profile_one.py panda 2 single 1 16
run memcheck_single148  --tool memcheck  python tools/profile_one.py panda 2 single 1 0
run memcheck_batch100   --tool memcheck  python tools/profile_one.py panda 2 batch 100
run memcheck_baxter     --tool memcheck  python tools/profile_one.py baxter 1 batch 40
run synccheck_single    --tool synccheck python tools/profile_one.py panda 1 single 1 8
run synccheck_batch40   --tool synccheck python tools/profile_one.py panda 1 batch 40
run racecheck_single4   --tool racecheck --racecheck-report hazard python tools/profile_one.py panda 1 single 1 4
run racecheck_batch12   --tool racecheck --racecheck-report hazard python tools/profile_one.py panda 1 batch 12
run racecheck_baxter8   --tool racecheck --racecheck-report hazard python tools/profile_one.py baxter 1 batch 8
run memcheck_parity     --tool memcheck  python -m pytest tests/test_gpu_parity.py -x -q -k "not nn_exact"
if [ "${WARP:-1}" = "1" ]; then  # the warp-worker planner (plan_warp_kernel, PRRTC_WARP=1)
  PRRTC_WARP=1 run memcheck_warp_batch100  --tool memcheck  python tools/profile_one.py panda 2 batch 100
  PRRTC_WARP=1 run memcheck_warp_fetch200  --tool memcheck  python tools/profile_one.py fetch 1 batch 200
  PRRTC_WARP=1 run memcheck_warp_baxter40  --tool memcheck  python tools/profile_one.py baxter 1 batch 40
  PRRTC_WARP=1 run synccheck_warp_batch40  --tool synccheck python tools/profile_one.py panda 1 batch 40
  PRRTC_WARP=1 run racecheck_warp_batch12  --tool racecheck --racecheck-report hazard python tools/profile_one.py panda 1 batch 12
fi
echo done >> "$OUT/summary.txt"
