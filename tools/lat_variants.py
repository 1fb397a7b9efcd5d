"""Single-problem latency (prrtc_plan wall clock) of PlannerParams variants,
alternating in one process:  python tools/lat_variants.py [robot] [n] [reps]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_06757_b200 import planner  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams, PlanStatus  # noqa: E402

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
model, scenes, S, G, kinds = bench.load_workload(robot, n)
rob = planner.device_robot(model)
dsc = [planner.device_scene(s) for s in scenes]
variants = {
    "default(512t)": bench.robot_params(robot, PlannerParams()),
    "256t": bench.robot_params(robot, PlannerParams(threads_per_cta=256)),
    "128t": bench.robot_params(robot, PlannerParams(threads_per_cta=128)),
}
for rep in range(reps):
    for name, p in variants.items():
        if p is None:
            continue
        for i in range(5):
            planner.plan(rob, dsc[i], S[i], G[i], p)
        rs = [planner.plan(rob, dsc[i], S[i], G[i], p) for i in range(len(S))]
        ok = [r for r in rs if r.status == PlanStatus.Solved]
        w = [r.wall_time_ms for r in ok]
        dv = [r.device_time_ms for r in ok]
        print(f"{robot} {name}: wall median {np.median(w):.4f} p95 {np.percentile(w, 95):.4f} | device median "
              f"{np.median(dv):.4f} | success {len(ok) / len(rs):.3f}", flush=True)
