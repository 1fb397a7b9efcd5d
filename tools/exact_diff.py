"""Per-problem comparison of the exact batch mode (workers = 1,
max_workers_per_problem = 1) with the reference's workers=1 plan():
status, iterations and path, for one robot's problem set.

    python tools/exact_diff.py [robot] [n] [tree_capacity] [scalar|avx2]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2503_06757_b200 import planner  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams, PlanStatus  # noqa: E402

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
model, scenes, S, G, kinds = bench.load_workload(robot, n)
o = Oracle("ref")
scalar = len(sys.argv) <= 4 or sys.argv[4] != "avx2"
o.force_scalar(scalar)  # the device follows the scalar backend's summation order
for threads in (0, 32):
    p = bench.robot_params(robot, PlannerParams(workers=1, tree_capacity=cap, max_workers_per_problem=1,
                                                threads_per_cta=threads))
    dsc = planner.device_scenes(scenes, 0)
    be = planner.plan_batch_arrays(model, dsc, S, G, p)
    ref, _ = o.plan_many(model, scenes, S, G, bench.robot_params(robot, PlannerParams(workers=1, tree_capacity=cap)),
                         threads=16)
    paths = be.paths
    kinds_bad = {"status": 0, "iters": 0, "path": 0}
    shown = 0
    for i, r in enumerate(ref):
        st, it = int(be.status[i]), int(be.iterations_total[i])
        if st != int(r.status):
            kinds_bad["status"] += 1
        elif it != r.iterations_total:
            kinds_bad["iters"] += 1
        elif r.status == PlanStatus.Solved and not np.array_equal(paths[i], r.path):
            kinds_bad["path"] += 1
        else:
            continue
        if shown < 8:
            shown += 1
            print(f"  #{i} {kinds[i]}: dev status {st} iters {it} len {len(paths[i])} | ref status {int(r.status)} "
                  f"iters {r.iterations_total} len {len(r.path)}")
    same = len(ref) - sum(kinds_bad.values())
    print(f"{robot} threads {threads} cap {cap} ref {'scalar' if scalar else 'avx2'}: identical {same}/{len(ref)} mismatches {kinds_bad}")
