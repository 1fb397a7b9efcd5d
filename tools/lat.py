"""Single-problem prrtc_plan latency over the bench problems (median / p95
wall and device, ms): python tools/lat.py [robot] [n] [workers]"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_06757_b200 import planner  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams, PlanStatus  # noqa: E402
robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
model, scenes, S, G, kinds = bench.load_workload(robot, 1000)
idx = list(range(0, 1000, max(1, 1000 // n)))[:n]
ds = {i: planner.device_scene(scenes[i]) for i in idx}
p = PlannerParams(workers=int(sys.argv[3]) if len(sys.argv) > 3 else 0)
for i in idx[:10]:
    planner.plan(model, ds[i], S[i], G[i], p)
wall, dev = [], []
for i in idx:
    r = planner.plan(model, ds[i], S[i], G[i], p)
    if r.status == PlanStatus.Solved:
        wall.append(r.wall_time_ms)
        dev.append(r.device_time_ms)
print(f"{robot} workers={p.workers} n={len(wall)} wall median {np.median(wall):.4f} p95 {np.percentile(wall, 95):.4f} "
      f"device median {np.median(dev):.4f} p95 {np.percentile(dev, 95):.4f}")
