"""ctypes binding of the C-ABI (include/prrtc_b200.h).

The shared library is built in-tree (paper_2503_06757_b200/lib/libprrtc_b200.so)
by ``python -m paper_2503_06757_b200.build``. There is no fallback: importing
the planner without the library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libprrtc_b200.so"

PRRTC_OK = 0
PRRTC_EINVAL = -1
PRRTC_ECUDA = -2
PRRTC_ENODEV = -3
PRRTC_ENOMEM = -4


class RobotDesc(C.Structure):
    _fields_ = [
        ("n_links", C.c_uint32),
        ("kind", C.POINTER(C.c_int32)),
        ("parent", C.POINTER(C.c_int32)),
        ("origin_quat", C.POINTER(C.c_double)),
        ("origin_xyz", C.POINTER(C.c_double)),
        ("axis", C.POINTER(C.c_double)),
        ("lo", C.POINTER(C.c_double)),
        ("hi", C.POINTER(C.c_double)),
        ("coarse", C.POINTER(C.c_double)),
        ("fine_offset", C.POINTER(C.c_uint32)),
        ("fine", C.POINTER(C.c_double)),
        ("n_self_pairs", C.c_uint32),
        ("self_pairs", C.POINTER(C.c_int32)),
    ]


class SceneDesc(C.Structure):
    _fields_ = [
        ("n_spheres", C.c_uint32),
        ("spheres", C.POINTER(C.c_double)),
        ("n_boxes", C.c_uint32),
        ("boxes", C.POINTER(C.c_double)),
        ("n_capsules", C.c_uint32),
        ("capsules", C.POINTER(C.c_double)),
        ("n_cylinders", C.c_uint32),
        ("cylinders", C.POINTER(C.c_double)),
    ]


class Params(C.Structure):
    _fields_ = [
        ("delta", C.c_double),
        ("n_cc", C.c_int32),
        ("workers", C.c_uint32),
        ("max_iters_per_worker", C.c_uint64),
        ("tree_capacity", C.c_uint64),
        ("dd_radius", C.c_double),
        ("dynamic_domain", C.c_uint8),
        ("balance", C.c_uint8),
        ("early_exit", C.c_uint8),
        ("two_stage", C.c_uint8),
        ("batched_cc", C.c_uint8),
        ("_pad", C.c_uint8 * 3),
        ("nn_partitions", C.c_uint32),
        ("sampler", C.c_int32),
        ("seed", C.c_uint64),
        ("threads_per_cta", C.c_uint32),
        ("ctas_per_sm", C.c_uint32),
        ("deterministic", C.c_uint32),
        ("validate_path", C.c_uint32),
        ("max_workers_per_problem", C.c_uint32),
        ("_pad2", C.c_uint32),
    ]


class Result(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("dof", C.c_uint32),
        ("path_len", C.c_uint32),
        ("path_block", C.c_uint32),
        ("path", C.POINTER(C.c_double)),
        ("cost", C.c_double),
        ("wall_time_ms", C.c_double),
        ("device_time_ms", C.c_double),
        ("iterations_total", C.c_uint64),
        ("sphere_tests", C.c_uint64),
        ("fk_calls", C.c_uint64),
        ("fine_stage_entries", C.c_uint64),
        ("flops", C.c_uint64),
        ("tree_nodes", C.c_uint64 * 2),
        ("solving_worker", C.c_int32),
        ("path_check", C.c_uint32),
        ("message", C.c_char * 128),
    ]


# (name, restype, argtypes) — every symbol include/prrtc_b200.h declares
P = C.c_void_p
DP = C.POINTER(C.c_double)
FP = C.POINTER(C.c_float)
U8P = C.POINTER(C.c_uint8)
SIGNATURES = [
    ("prrtc_api_version", C.c_int, []),
    ("prrtc_last_error", C.c_int, [C.c_char_p, C.c_size_t]),
    ("prrtc_device_count", C.c_int, []),
    ("prrtc_default_workers", C.c_int, [C.c_int]),
    ("prrtc_debug_reload_env", C.c_int, []),
    ("prrtc_last_transfer_bytes", C.c_int, [C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("prrtc_params_default", None, [C.POINTER(Params)]),
    ("prrtc_robot_create", C.c_int, [C.POINTER(RobotDesc), C.c_int, C.POINTER(P)]),
    ("prrtc_robot_destroy", C.c_int, [P]),
    ("prrtc_robot_dof", C.c_int, [P]),
    ("prrtc_robot_fine_count", C.c_int, [P]),
    ("prrtc_robot_limits", C.c_int, [P, DP]),
    ("prrtc_scene_create", C.c_int, [C.POINTER(SceneDesc), C.c_int, C.POINTER(P)]),
    ("prrtc_scene_update", C.c_int, [P, C.POINTER(SceneDesc)]),
    ("prrtc_scene_destroy", C.c_int, [P]),
    ("prrtc_plan", C.c_int, [P, P, DP, DP, C.c_uint32, C.POINTER(Params), C.POINTER(Result)]),
    ("prrtc_plan_batch", C.c_int, [P, C.POINTER(P), C.c_uint32, DP, DP, C.c_uint32, C.POINTER(Params), C.POINTER(Result)]),
    ("prrtc_plan_batch_multi", C.c_int, [C.POINTER(P), C.POINTER(P), C.c_uint32, C.c_uint32, DP, DP, C.c_uint32,
                                         C.POINTER(Params), C.c_uint32, C.POINTER(Result)]),
    ("prrtc_debug_chunk_queue", C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32),
                                          C.POINTER(C.c_int32), C.POINTER(C.c_uint32)]),
    ("prrtc_result_free", None, [C.POINTER(Result)]),
    ("prrtc_results_free", None, [C.POINTER(Result), C.c_uint32]),
    ("prrtc_results_pack_paths", C.c_int, [C.POINTER(Result), C.c_uint32, C.POINTER(C.c_double),
                                           C.POINTER(C.c_uint64)]),
    ("prrtc_batch_create", C.c_int, [P, C.POINTER(P), C.c_uint32, DP, DP, C.c_uint32, C.POINTER(Params), C.POINTER(P)]),
    ("prrtc_batch_launch", C.c_int, [P, P]),
    ("prrtc_batch_results", C.c_int, [P, C.POINTER(Result)]),
    ("prrtc_batch_launch_count", C.c_int, [P]),
    ("prrtc_batch_destroy", C.c_int, [P]),
    ("prrtc_validate_edges", C.c_int, [P, P, DP, DP, C.c_uint32, C.c_uint32, C.c_int32, C.c_int, C.c_int, U8P]),
    ("prrtc_check_configs", C.c_int, [P, P, DP, C.c_uint32, C.c_uint32, C.c_int, U8P]),
    ("prrtc_debug_fk", C.c_int, [P, DP, C.c_uint32, C.c_uint32, FP, FP]),
    ("prrtc_debug_check_edges", C.c_int, [P, P, DP, DP, C.c_uint32, C.c_uint32, C.c_int32, C.c_int, U8P, FP]),
    ("prrtc_debug_sphere_hits", C.c_int, [P, FP, DP, C.c_uint32, U8P]),
    ("prrtc_debug_nn", C.c_int, [DP, C.c_uint32, C.c_uint32, DP, C.c_uint32, C.c_int, C.POINTER(C.c_uint32), DP]),
    ("prrtc_debug_nn_multi", C.c_int, [DP, C.c_uint32, C.c_uint32, DP, C.c_uint32, C.c_uint32, C.c_int,
                                       C.POINTER(C.c_uint32), DP]),
    ("prrtc_debug_halton", C.c_int, [C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.c_uint32, C.c_int, DP]),
    ("prrtc_debug_sample", C.c_int, [P, C.c_uint64, C.c_uint32, DP]),
    ("prrtc_debug_chunk_profile", C.c_int, [P, P, DP, DP, C.c_uint32, C.c_int32, C.c_int,
                                           C.POINTER(C.c_longlong)]),
    ("prrtc_fp32_peak_tflops", C.c_double, [C.c_int]),
    ("prrtc_fp64_peak_tflops", C.c_double, [C.c_int]),
    ("prrtc_l2_peak_gbs", C.c_double, [C.c_int]),
    ("prrtc_bench_validate_edges", C.c_int, [P, P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_uint32,
                                             C.c_uint32, C.c_int32, C.c_int, C.c_int, C.c_int,
                                             C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("prrtc_bench_nn", C.c_int, [C.POINTER(C.c_double), C.c_uint32, C.c_uint32, C.POINTER(C.c_double), C.c_uint32,
                                 C.c_uint32, C.c_int, C.c_int, C.POINTER(C.c_double)]),
]

_lib = None


def load() -> C.CDLL:
    """Load the CUDA planner library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("PRRTC_B200_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2503_06757_b200.build` "
            "(the planner has no CPU fallback)")
    lib = C.CDLL(str(path))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class PrrtcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def last_error() -> str:
    buf = C.create_string_buffer(512)
    load().prrtc_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc: int) -> None:
    """Map return codes to the reference's error behaviour: PRRTC_EINVAL is
    std::invalid_argument -> ValueError; anything else is a RuntimeError."""
    if rc == PRRTC_OK:
        return
    msg = last_error()
    if rc == PRRTC_EINVAL:
        raise ValueError(msg)
    raise PrrtcError(rc, msg)
