"""Replanning loop frame latency (BASELINE config 5): 100 frames of
prrtc_scene_update + prrtc_plan, median / p95 ms, three repetitions."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_06757_b200 import replan  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams  # noqa: E402
model, scenes, S, G, kinds = bench.load_workload("panda", 1000)
i = int(np.where(kinds == "table_pick")[0][0])
for rep in range(3):
    frames = replan.run(model, scenes[i], S[i], G[i], frames=100, params=PlannerParams())
    w = [f.wall_ms for f in frames]
    print(f"replan frame median {np.median(w):.4f} p95 {np.percentile(w, 95):.4f} ms")
