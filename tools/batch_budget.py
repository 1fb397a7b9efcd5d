"""How much of the batch time the failing problems' budgets cost: the bench
batch as is, without the problems that fail, and at smaller budgets
(params.workers = budget in reference workers)."""
import sys
import time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams, PlanStatus  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402
robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
scenes = [make_scene(robot, str(k), int(p))[0] for k, p in zip(d["kind"], d["pid"])]


def run(idx, params, reps=5):
    b = planner.Batch(m, [scenes[i] for i in idx], d["start"][idx], d["goal"][idx], params)
    b.launch()
    b.results()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.launch(torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    res = b.results()
    ok = np.array([r.status == PlanStatus.Solved for r in res])
    return float(np.median(ms)), ok


allidx = np.arange(len(d["pid"]))
ms, ok = run(allidx, PlannerParams())
print(f"{robot} full batch: {ms:.3f} ms, solved {ok.mean():.3f}")
ms2, ok2 = run(allidx[ok], PlannerParams())
print(f"without the {(~ok).sum()} failing problems: {ms2:.3f} ms, solved {ok2.mean():.3f}")
for w in (8, 16, 32, 64):
    ms3, ok3 = run(allidx, PlannerParams(workers=w))
    print(f"budget {w} workers x 2000: {ms3:.3f} ms, solved {ok3.mean():.3f}")
for cps in (1, 2, 3):
    ms4, ok4 = run(allidx, PlannerParams(ctas_per_sm=cps))
    print(f"ctas_per_sm {cps}: {ms4:.3f} ms, solved {ok4.mean():.3f}")
