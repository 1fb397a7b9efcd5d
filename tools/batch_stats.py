"""Batch tail analysis: per-problem iterations / device time / status for
several iteration budgets (development aid, prints one line per budget)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams, PlanStatus  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
# configs "budget:threads", e.g. 1:128,32:128,32:256
configs = [tuple(int(v) for v in (x.split(":") + ["128"])[:2])
           for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "8", "32"])]
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
scenes = [make_scene(robot, str(k), int(p))[0] for k, p in zip(d["kind"], d["pid"])]
for w, nt in configs:
    params = PlannerParams(workers=w, threads_per_cta=nt)
    b = planner.Batch(m, scenes, d["start"], d["goal"], params)
    b.launch()
    b.results()
    t = time.perf_counter()
    b.launch()
    res = b.results()
    dt = (time.perf_counter() - t) * 1e3
    st = np.array([r.status == PlanStatus.Solved for r in res])
    it = np.array([r.iterations_total for r in res])
    dv = np.array([r.device_time_ms for r in res])
    nodes = np.array([sum(r.tree_nodes) for r in res])
    fl = sum(r.flops for r in res)
    print(f"{robot} budget x{w} threads {nt}: {dt:.2f} ms ({len(res) / dt * 1e3:.0f}/s) solved {st.mean():.3f} "
          f"iters p50/p90/p99/max {np.percentile(it, 50):.0f}/{np.percentile(it, 90):.0f}/"
          f"{np.percentile(it, 99):.0f}/{it.max()} sum {it.sum()} | dev ms p50/p99/max "
          f"{np.median(dv):.3f}/{np.percentile(dv, 99):.3f}/{dv.max():.3f} | nodes p50/max "
          f"{np.median(nodes):.0f}/{nodes.max()} | alg TFLOP/s {fl / dt / 1e9:.3f}", flush=True)
    for k in ("table_pick", "bookshelf", "cage"):
        sel = d["kind"] == k
        print(f"    {k}: solved {st[sel].mean():.3f} iters p50 {np.median(it[sel]):.0f} "
              f"dev ms p50 {np.median(dv[sel]):.3f}", flush=True)
    del b
