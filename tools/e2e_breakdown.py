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
model = planner.device_robot(model, 0)  # setup: the handle, as the bench holds it
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
for _ in range(30):  # medians of the traced components over 30 calls (stderr lines, parsed below)
    rob_, res, n, hs = planner._plan_batch_raw(model, dsc, S, G, params, 0)
    planner._free(res, n)

# Python-side split of one call: before the foreign call, the call, after it
import paper_2503_06757_b200.planner as P  # noqa: E402
pre, mid, post = [], [], []
os.environ.pop("PRRTC_HOST_TRACE", None)
planner.reload_env()
lib_ = _lib.load()
for _ in range(30):
    t0 = time.perf_counter()
    rob = P.device_robot(model, 0)
    S_ = np.ascontiguousarray(np.asarray(S, dtype=np.float64).reshape(-1, rob.dof))
    G_ = np.ascontiguousarray(np.asarray(G, dtype=np.float64).reshape(-1, rob.dof))
    n = S_.shape[0]
    hs, arr = P._scene_handles(dsc, n, 0)
    p = params.to_c()
    res = (Result * n)()
    t1 = time.perf_counter()
    P.check(lib_.prrtc_plan_batch(rob.h, arr, n, P._dptr(S_), P._dptr(G_), rob.dof, C.byref(p), res))
    t2 = time.perf_counter()
    out = P.BatchResult(res, n, rob.dof)
    P._free(res, n)
    t3 = time.perf_counter()
    pre.append(t1 - t0)
    mid.append(t2 - t1)
    post.append(t3 - t2)
print(f"python pre {1e6 * np.median(pre):.1f} us | C call {1e6 * np.median(mid):.1f} us | "
      f"python post {1e6 * np.median(post):.1f} us")
