"""CPU: the C-ABI library loads, exports every symbol include/prrtc_b200.h
declares, its struct layouts match the Python binding, and it fails loudly
(no CPU fallback) when no sm_100 device is present."""
import ctypes as C
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import has_gpu
from paper_2503_06757_b200 import _lib, robots
from paper_2503_06757_b200.model import Joint, REVOLUTE

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "prrtc_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|double)\s+\*?(prrtc_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "prrtc_b200.h"
#define P(T, f) printf(#T "." #f " %zu\\n", offsetof(T, f));
int main(void) {
  printf("prrtc_params %zu\\nprrtc_result %zu\\nprrtc_robot_desc %zu\\nprrtc_scene_desc %zu\\n",
         sizeof(prrtc_params), sizeof(prrtc_result), sizeof(prrtc_robot_desc), sizeof(prrtc_scene_desc));
  P(prrtc_params, seed) P(prrtc_params, deterministic) P(prrtc_params, nn_partitions)
  P(prrtc_params, max_workers_per_problem)
  P(prrtc_result, path) P(prrtc_result, flops) P(prrtc_result, tree_nodes) P(prrtc_result, message)
  P(prrtc_robot_desc, self_pairs) P(prrtc_scene_desc, capsules)
  return 0;
}""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    out = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                              check=True).stdout.strip().splitlines())
    assert int(out["prrtc_params"]) == C.sizeof(_lib.Params)
    assert int(out["prrtc_result"]) == C.sizeof(_lib.Result)
    assert int(out["prrtc_robot_desc"]) == C.sizeof(_lib.RobotDesc)
    assert int(out["prrtc_scene_desc"]) == C.sizeof(_lib.SceneDesc)
    assert int(out["prrtc_params.seed"]) == _lib.Params.seed.offset
    assert int(out["prrtc_params.deterministic"]) == _lib.Params.deterministic.offset
    assert int(out["prrtc_params.nn_partitions"]) == _lib.Params.nn_partitions.offset
    assert int(out["prrtc_params.max_workers_per_problem"]) == _lib.Params.max_workers_per_problem.offset
    assert int(out["prrtc_result.path"]) == _lib.Result.path.offset
    assert int(out["prrtc_result.flops"]) == _lib.Result.flops.offset
    assert int(out["prrtc_result.tree_nodes"]) == _lib.Result.tree_nodes.offset
    assert int(out["prrtc_result.message"]) == _lib.Result.message.offset
    assert int(out["prrtc_robot_desc.self_pairs"]) == _lib.RobotDesc.self_pairs.offset
    assert int(out["prrtc_scene_desc.capsules"]) == _lib.SceneDesc.capsules.offset


def test_params_default_matches_reference():
    p = _lib.Params()
    _lib.load().prrtc_params_default(C.byref(p))
    # planner.hpp:21-40
    assert (p.delta, p.n_cc, p.workers, p.max_iters_per_worker, p.tree_capacity) == (0.5, 32, 0, 2000, 200000)
    assert (p.dd_radius, p.dynamic_domain, p.balance, p.early_exit, p.two_stage, p.batched_cc) == (0.0, 1, 1, 1, 1, 0)
    assert (p.nn_partitions, p.sampler, p.seed) == (1, 0, 0)


def test_validation_mirrors_finalize_without_device():
    """RobotModel::finalize errors (kinematics.cpp:15-74) are reported before
    any device work, as ValueError (std::invalid_argument)."""
    from paper_2503_06757_b200.planner import DeviceRobot
    m = robots.get("panda")
    m.joints[3] = Joint(REVOLUTE, 2, m.joints[3].origin_quat, m.joints[3].origin_xyz, (0, 0, 2), -1, 1)
    with pytest.raises(ValueError, match="axis"):
        DeviceRobot(m)
    m = robots.get("panda")
    m.self_pairs = [(1, 2)]
    with pytest.raises(ValueError, match="adjacent"):
        DeviceRobot(m)
    m = robots.get("panda")
    m.joints[2] = Joint(REVOLUTE, 5, (1, 0, 0, 0), (0, 0, 0), (0, 0, 1), -1, 1)
    with pytest.raises(ValueError, match="parent"):
        DeviceRobot(m)


@pytest.mark.skipif(has_gpu(), reason="only meaningful without a GPU")
def test_no_cpu_fallback():
    from paper_2503_06757_b200.planner import DeviceRobot
    with pytest.raises(_lib.PrrtcError, match="no CPU fallback"):
        DeviceRobot(robots.get("panda"))


def test_missing_library_fails_loudly(tmp_path):
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2503_06757_b200 import planner, robots\n"
            "planner.DeviceRobot(robots.get('panda'))\n") % str(ROOT)
    env = dict(os.environ, PRRTC_B200_LIB=str(tmp_path / "missing.so"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.returncode != 0 and "no CPU fallback" in r.stderr


def test_result_helpers_pack_and_free():
    """prrtc_results_pack_paths / prrtc_results_free (host-only helpers used by
    the batch API): paths back to back with doubles offsets; freeing clears."""
    import numpy as np
    lib = _lib.load()
    libc = C.CDLL(None)
    libc.malloc.restype = C.c_void_p
    libc.malloc.argtypes = [C.c_size_t]
    res = (_lib.Result * 3)()
    rng = np.random.default_rng(0)
    paths = [rng.standard_normal((4, 7)), None, rng.standard_normal((2, 7))]
    for r, p in zip(res, paths):
        r.dof = 7
        if p is not None:
            buf = libc.malloc(8 * p.size)
            C.memmove(buf, p.ctypes.data, 8 * p.size)
            r.path = C.cast(buf, C.POINTER(C.c_double))
            r.path_len = p.shape[0]
    off = np.zeros(4, dtype=np.uint64)
    assert lib.prrtc_results_pack_paths(res, 3, None, off.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
    assert off.tolist() == [0, 28, 28, 42]
    flat = np.zeros(int(off[-1]))
    assert lib.prrtc_results_pack_paths(res, 3, flat.ctypes.data_as(C.POINTER(C.c_double)),
                                        off.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
    assert np.array_equal(flat[:28].reshape(4, 7), paths[0]) and np.array_equal(flat[28:].reshape(2, 7), paths[2])
    lib.prrtc_results_free(res, 3)
    assert all(not r.path and r.path_len == 0 for r in res)
    assert lib.prrtc_results_pack_paths(None, 0, None, off.ctypes.data_as(C.POINTER(C.c_uint64))) == -1
