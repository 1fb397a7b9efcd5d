"""The roofline microbenchmark hooks: they time the same
kernels the product uses and count the algorithmic work the way the
planner does. Dense mode executes every test, so its count is exact:
S * P fine-vs-primitive tests plus sum |f_a| * |f_b| over self pairs per state."""
import ctypes

import numpy as np
import pytest

from conftest import load_problems
from paper_2503_06757_b200 import _lib, planner, robots
from paper_2503_06757_b200.scenes import make_scene

pytestmark = pytest.mark.gpu


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


@pytest.mark.parametrize("robot", ["panda", "fetch"])
def test_dense_counts_every_test(gpu, robot):
    m = robots.get(robot)
    probs = load_problems(robot, 6)
    kind, pid, s, g = probs[1]
    scene = make_scene(robot, kind, pid)[0]
    A = np.ascontiguousarray(np.array([p[2] for p in probs]))
    G = np.array([p[3] for p in probs])
    d = G - A
    B = np.ascontiguousarray(A + d * np.minimum(1.0, 0.5 / np.linalg.norm(d, axis=1))[:, None])
    rob, sc = planner.device_robot(m), planner.device_scene(scene)
    lib = _lib.load()
    ms, fl, te = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    n_cc = 32
    _lib.check(lib.prrtc_bench_validate_edges(rob.h, sc.h, _dp(A), _dp(B), len(A), m.dof, n_cc, 0, 0, 2,
                                              ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(te)))
    S, P = m.fine_count(), len(scene.primitives)
    pairs = sum(len(m.spheres[a].fine) * len(m.spheres[b].fine) for a, b in m.self_pairs)
    states = len(A) * n_cc
    assert te.value == states * (S * P + pairs)
    assert ms.value > 0 and fl.value > te.value * 10
    # two-stage production mode does less work for the same edges
    ms2, fl2, te2 = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _lib.check(lib.prrtc_bench_validate_edges(rob.h, sc.h, _dp(A), _dp(B), len(A), m.dof, n_cc, 1, 0, 2,
                                              ctypes.byref(ms2), ctypes.byref(fl2), ctypes.byref(te2)))
    assert 0 < fl2.value < fl.value


def test_nn_bench_and_l2_peak(gpu):
    lib = _lib.load()
    rng = np.random.default_rng(3)
    T = np.ascontiguousarray(rng.uniform(-2, 2, size=(5000, 7)))
    Q = np.ascontiguousarray(rng.uniform(-2, 2, size=(64, 7)))
    for g in (1, 32):
        ms = ctypes.c_double()
        _lib.check(lib.prrtc_bench_nn(_dp(T), len(T), 7, _dp(Q), len(Q), g, 0, 2, ctypes.byref(ms)))
        assert ms.value > 0
    with pytest.raises(ValueError):
        _lib.check(lib.prrtc_bench_nn(_dp(T), len(T), 7, _dp(Q), len(Q), 33, 0, 2, ctypes.byref(ms)))
    assert lib.prrtc_l2_peak_gbs(0) > 1000.0
