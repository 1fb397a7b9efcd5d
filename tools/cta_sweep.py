"""Batch time vs CTAs per SM (params.ctas_per_sm) at the bench headline params."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_06757_b200 import planner  # noqa: E402

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
model, scenes, S, G, kinds = bench.load_workload(robot, 1000)
for rep in range(2):
    for cps in (1, 2, 3, 4):
        p = bench.robot_params(robot, bench.headline_params(ctas_per_sm=cps))
        b = planner.Batch(model, scenes, S, G, p)
        b.launch()
        b.results()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(10):
            e0.record()
            b.launch(torch.cuda.current_stream().cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        res = b.results()
        print(f"{robot} ctas/SM {cps}: {np.median(ms):.3f} ms, {1000 / np.median(ms) * 1e3:.0f} problems/s, "
              f"solved {np.mean([r.status == 0 for r in res]):.3f}", flush=True)
        del b
