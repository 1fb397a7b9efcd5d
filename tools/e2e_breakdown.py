"""Host-side anatomy of the e2e call (prrtc_plan_batch via plan_batch_arrays):
Python wrapper vs C-ABI (PRRTC_HOST_TRACE) vs device time."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_06757_b200 import planner  # noqa: E402
from paper_2503_06757_b200 import _lib  # noqa: E402
from paper_2503_06757_b200._lib import Result  # noqa: E402
import ctypes as C  # noqa: E402

model, scenes, S, G, kinds = bench.load_workload("panda", 1000)
params = bench.headline_params()
dsc = planner.device_scenes(scenes, 0)
for _ in range(5):
    planner.plan_batch_arrays(model, dsc, S, G, params)
tw, tc, tb = [], [], []
rob = planner.device_robot(model, 0)
for _ in range(20):
    t0 = time.perf_counter()
    rob_, res, n, hs = planner._plan_batch_raw(model, dsc, S, G, params, 0)
    t1 = time.perf_counter()
    out = planner.BatchResult(res, n, rob.dof)
    planner._free(res, n)
    t2 = time.perf_counter()
    tc.append((t1 - t0) * 1e3)
    tb.append((t2 - t1) * 1e3)
print(f"C call (incl. ctypes setup) median {np.median(tc):.3f} ms; BatchResult + free {np.median(tb):.3f} ms")
os.environ["PRRTC_HOST_TRACE"] = "1"
planner.reload_env()
planner._plan_batch_raw(model, dsc, S, G, params, 0)
