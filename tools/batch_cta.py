"""CTA size / CTAs per SM sweep of one robot's 1000-problem batch (bench params)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2503_06757_b200 import planner  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams, PlanStatus  # noqa: E402
robot = sys.argv[1] if len(sys.argv) > 1 else "baxter"
model, scenes, S, G, kinds = bench.load_workload(robot, 1000)
for tpc, cps in ((0, 0), (128, 0), (256, 0), (128, 3), (256, 1)):
    p = bench.robot_params(robot, PlannerParams(threads_per_cta=tpc, ctas_per_sm=cps))
    b = planner.Batch(model, scenes, S, G, p)
    b.launch()
    b.results()
    ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.launch(torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ok = np.mean([r.status == PlanStatus.Solved for r in b.results()])
    print(f"{robot} threads_per_cta {tpc} ctas_per_sm {cps}: {np.median(ms):.2f} ms solved {ok:.3f}", flush=True)
    del b
