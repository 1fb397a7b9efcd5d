"""How one problem's fixed iteration budget parallelises over CTAs: the
problem alone on the GPU, W workers of 128 threads, budget 2000 iterations
in total (max_iters_per_worker = 2000 / W). Device time and success over
seeds, per W.

    python tools/scale_one.py [robot] [problem ...]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams, PlanStatus  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
ids = [int(x) for x in sys.argv[2:]] or [978, 963, 834]
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
for i in ids:
    sc = planner.device_scene(make_scene(robot, str(d["kind"][i]), int(d["pid"][i]))[0])
    for W in (1, 2, 4, 8, 16, 32):
        t, ok, it = [], 0, []
        for seed in range(8):
            p = PlannerParams(workers=W, max_iters_per_worker=2000 // W, tree_capacity=20000, threads_per_cta=128,
                              seed=seed * (1 << 20))
            r = planner.plan(m, sc, d["start"][i], d["goal"][i], p)
            t.append(r.device_time_ms)
            ok += r.status == PlanStatus.Solved
            it.append(r.iterations_total)
        print(f"problem {i} ({d['kind'][i]}) W {W:2d}: device ms median {np.median(t):.3f} max {np.max(t):.3f} "
              f"solved {ok}/8 iterations mean {np.mean(it):.0f}")
