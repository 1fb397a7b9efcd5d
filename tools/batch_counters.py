"""Work totals of one headline batch (bench params): iterations, checked
states (fk_calls), sphere tests, fine-stage entries, algorithmic flops, and
the kernel's device time — what a launch spends its instructions on.

    python tools/batch_counters.py [robot] [threads_per_cta] [n_problems]

(n_problems > 1000 repeats the robot's 1000-problem set.)
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
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
idx = np.arange(n) % len(d["pid"])
scenes = [make_scene(robot, str(d["kind"][i]), int(d["pid"][i]))[0] for i in idx]
p = PlannerParams(workers=1, tree_capacity=20000)
if nt:
    p.threads_per_cta = nt
if robot == "baxter":
    p.dd_radius = 4.0
b = planner.Batch(m, scenes, d["start"][idx], d["goal"][idx], p)
import torch  # noqa: E402
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.current_stream()
kms = []
for rep in range(4):
    t = time.perf_counter()
    ev0.record(st)
    b.launch(st.cuda_stream)
    ev1.record(st)
    res = b.results()
    wall = (time.perf_counter() - t) * 1e3
    kms.append(ev0.elapsed_time(ev1))
ok = np.array([r.status == PlanStatus.Solved for r in res])
it = float(sum(r.iterations_total for r in res))
fl = float(sum(r.flops for r in res))
fk, st, fe = (float(sum(getattr(r.check_stats, f) for r in res)) for f in ("fk_calls", "sphere_tests", "fine_stage_entries"))
P = np.array([len(s.primitives) for s in scenes])
print(f"{robot}: n {len(res)} solved {ok.mean():.3f} kernel {min(kms[1:]):.3f} ms wall {wall:.3f} ms | iterations {it:.0f} "
      f"({it / len(res):.1f}/problem) | checked states {fk:.0f} ({fk / 32:.0f} x 32) | sphere tests {st:.0f} "
      f"({st / max(fk, 1):.1f}/state) | fine entries {fe:.0f} | flops {fl:.3e} ({fl / max(fk, 1):.0f}/state) | "
      f"primitives mean {P.mean():.1f} max {P.max()}")
dv = np.array([r.device_time_ms for r in res])
itp = np.array([r.iterations_total for r in res], dtype=float)
q = lambda x: " ".join(f"{v:.3f}" for v in np.percentile(x, [50, 90, 99, 100]))  # noqa: E731
print(f"  per-problem device ms p50/p90/p99/max: solved {q(dv[ok])} | failed {q(dv[~ok]) if (~ok).any() else '-'}")
print(f"  iterations p50/p90/p99/max: solved {q(itp[ok])} | failed {q(itp[~ok]) if (~ok).any() else '-'}")
