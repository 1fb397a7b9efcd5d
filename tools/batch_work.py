"""Where a batch's work goes: iterations and device spans of solved vs failed
problems, per scene kind (default params, the bench batch).

    python tools/batch_work.py [robot] [n]
"""
import sys
import time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams, PlanStatus  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402
robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
scenes = [make_scene(robot, str(k), int(p))[0] for k, p in zip(d["kind"][:n], d["pid"][:n])]
p = PlannerParams()
if robot == "baxter":
    p.dd_radius = 4.0
b = planner.Batch(m, scenes, d["start"][:n], d["goal"][:n], p)
for rep in range(3):
    t = time.perf_counter()
    b.launch()
    res = b.results()
    print(f"launch+results {1e3 * (time.perf_counter() - t):.2f} ms")
ok = np.array([r.status == PlanStatus.Solved for r in res])
it = np.array([r.iterations_total for r in res], dtype=np.float64)
dv = np.array([r.device_time_ms for r in res])
print(f"{robot}: solved {ok.mean():.3f}; iterations solved {it[ok].sum():.0f} (mean {it[ok].mean():.0f}, "
      f"median {np.median(it[ok]):.0f}, p95 {np.percentile(it[ok], 95):.0f}) failed {it[~ok].sum():.0f} "
      f"({(~ok).sum()} problems); failed share of iterations {it[~ok].sum() / it.sum():.3f}")
for k in np.unique(d["kind"][:n]):
    s = d["kind"][:n] == k
    print(f"  {k}: solved {ok[s].mean():.3f} iters mean {it[s].mean():.0f} dev-span median {np.median(dv[s]):.3f} "
          f"p95 {np.percentile(dv[s], 95):.3f} max {dv[s].max():.3f}")
print("slowest spans:", np.round(np.sort(dv)[-12:], 2))
print("failed messages:", sorted({r.message for r in res if r.status != PlanStatus.Solved}))
