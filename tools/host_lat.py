"""Host-side breakdown of single-problem prrtc_plan calls (PRRTC_HOST_TRACE=1)."""
import os
import sys
from pathlib import Path

import numpy as np

os.environ["PRRTC_HOST_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402

d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "problems_panda.npz")
m = robots.get("panda")
for i in (0, 400, 700):
    sc = planner.device_scene(make_scene("panda", str(d["kind"][i]), int(d["pid"][i]))[0])
    for rep in range(6):
        r = planner.plan(m, sc, d["start"][i], d["goal"][i], PlannerParams())
        print(f"    problem {i} {r.status.name} wall {r.wall_time_ms * 1e3:.1f} us", file=sys.stderr, flush=True)

# batch e2e: python-side total vs the library's own phases
import time  # noqa: E402
scenes = [planner.device_scene(make_scene("panda", str(k), int(p))[0]) for k, p in zip(d["kind"], d["pid"])]
for rep in range(4):
    t0 = time.perf_counter()
    planner.plan_batch_arrays(m, scenes, d["start"], d["goal"], PlannerParams())
    t1 = time.perf_counter()
    print(f"    batch e2e {1e3 * (t1 - t0):.3f} ms", file=sys.stderr, flush=True)
import cProfile, pstats  # noqa: E402,E401
pr = cProfile.Profile()
pr.enable()
planner.plan_batch_arrays(m, scenes, d["start"], d["goal"], PlannerParams())
pr.disable()
pstats.Stats(pr, stream=sys.stderr).sort_stats("cumulative").print_stats(12)
