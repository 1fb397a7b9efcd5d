"""One launch each of the roofline microbenchmark kernels (bench.microbench's
inputs) for an ncu capture: validate_edges_kernel dense (two_stage=0,
early_exit=0) and two-stage, debug_nn_multi_kernel with 1 and 32 queries per
pass.   ncu --set full -k regex:'validate_edges|debug_nn_multi' python tools/profile_micro.py"""
import ctypes
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_06757_b200 import _lib, planner  # noqa: E402

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
model, scenes, S, G, kinds = bench.load_workload(robot, 1000)
lib = _lib.load()
rob = planner.device_robot(model, 0)
n_edges, n_cc, delta = 4096, 32, 0.5
k = np.arange(n_edges) % len(S)
A = np.ascontiguousarray(S[k])
d = G[k] - A
B = np.ascontiguousarray(A + d * np.minimum(1.0, delta / np.linalg.norm(d, axis=1))[:, None])
sc = planner.device_scene(scenes[len(scenes) // 2], 0)
dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
for two, early in ((0, 0), (1, 1)):
    ms, fl, te = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _lib.check(lib.prrtc_bench_validate_edges(rob.h, sc.h, dp(A), dp(B), n_edges, model.dof, n_cc, two, early, 1,
                                              ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(te)))
    print(f"validate_edges two_stage={two}: {ms.value:.4f} ms, flops/state {fl.value / (n_edges * n_cc):.0f}")
rng = np.random.default_rng(7)
lim = model.limits()
T = np.ascontiguousarray(rng.uniform(lim[:, 0], lim[:, 1], size=(100000, model.dof)))
for g in (1, 32):
    Q = np.ascontiguousarray(rng.uniform(lim[:, 0], lim[:, 1], size=(2048 if g == 1 else 32 * 592, model.dof)))
    ms = ctypes.c_double()
    _lib.check(lib.prrtc_bench_nn(dp(T), T.shape[0], model.dof, dp(Q), Q.shape[0], g, 0, 1, ctypes.byref(ms)))
    print(f"nn group {g}: {ms.value:.4f} ms")
