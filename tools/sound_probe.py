import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_2503_06757_b200 import planner
from paper_2503_06757_b200.model import PlanStatus
model, scenes, S, G, kinds = bench.load_workload('panda', 1000)
drob = planner.device_robot(model)
dsc = [planner.device_scene(s) for s in scenes]
sp = bench.headline_params(validate_path=True)
planner.plan_batch_arrays(drob, dsc, S, G, sp)
ms = []
for _ in range(8):
    t = time.perf_counter(); r = planner.plan_batch_arrays(drob, dsc, S, G, sp); ms.append((time.perf_counter() - t) * 1e3)
print(sys.argv[1], 'sound ms', ' '.join(f'{x:.2f}' for x in ms), 'median', round(statistics.median(ms), 3), 'solved', np.mean(r.status == PlanStatus.Solved))
