"""Python host API over the C-ABI — the reference's planning interface.

    plan(model, scene, start, goal, params) -> PlanResult      planner.hpp:55-56
    plan_batch(model, scenes, starts, goals, params)           (many problems, one launch)
    validate_edges / check_configs                             collision.hpp:57-75
    debug_* parity hooks                                       include/prrtc_b200.h

Robot and scene uploads are setup (untimed in the reference methodology,
PAPER.md:201) and are cached per content fingerprint, so repeated plan()
calls on the same model/scene only move start/goal/params and the result.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import Params, Result, check
from .model import (CheckStatsSnapshot, PlannerParams, PlanResult, PlanStatus, RobotModel,
                    Scene)

_DP = C.POINTER(C.c_double)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_DP)


class DeviceRobot:
    """prrtc_robot handle (validated + uploaded RobotModel)."""

    def __init__(self, model: RobotModel, device: int = 0):
        lib = _lib.load()
        desc, keep = model.to_desc()
        h = C.c_void_p()
        check(lib.prrtc_robot_create(C.byref(desc), device, C.byref(h)))
        self.h = h
        self.model = model
        self.device = device
        self.dof = lib.prrtc_robot_dof(h)
        self.fine_count = lib.prrtc_robot_fine_count(h)
        self.n_links = model.link_count()
        del keep

    def __del__(self):
        if getattr(self, "h", None) and getattr(_lib, "_lib", None) is not None:  # module globals may be gone at exit
            _lib._lib.prrtc_robot_destroy(self.h)
            self.h = None


class DeviceScene:
    """prrtc_scene handle (validated + uploaded Scene)."""

    def __init__(self, scene: Scene, device: int = 0):
        lib = _lib.load()
        desc, keep = scene.to_desc()
        h = C.c_void_p()
        check(lib.prrtc_scene_create(C.byref(desc), device, C.byref(h)))
        self.h = h
        self.scene = scene
        self.device = device
        self.n_prims = len(scene.primitives)
        del keep

    def update(self, scene: Scene) -> None:
        """prrtc_scene_update: replace the primitives (dynamic obstacles)."""
        desc, keep = scene.to_desc()
        check(_lib.load().prrtc_scene_update(self.h, C.byref(desc)))
        self.scene = scene
        self.n_prims = len(scene.primitives)
        del keep

    def __del__(self):
        if getattr(self, "h", None) and getattr(_lib, "_lib", None) is not None:  # module globals may be gone at exit
            _lib._lib.prrtc_scene_destroy(self.h)
            self.h = None


_robot_cache: dict = {}
_scene_cache: dict = {}


def _fingerprint(obj) -> str:
    return repr(obj)


def device_robot(model: RobotModel | DeviceRobot, device: int = 0) -> DeviceRobot:
    if isinstance(model, DeviceRobot):
        return model
    key = (_fingerprint(model), device)
    h = _robot_cache.get(key)
    if h is None:
        h = _robot_cache[key] = DeviceRobot(model, device)
    return h


def device_scene(scene: Scene | DeviceScene, device: int = 0) -> DeviceScene:
    if isinstance(scene, DeviceScene):
        return scene
    key = (_fingerprint(scene), device)
    h = _scene_cache.get(key)
    if h is None:
        if len(_scene_cache) > 4096:
            _scene_cache.clear()
        h = _scene_cache[key] = DeviceScene(scene, device)
    return h


def _to_result(r: Result, dof: int) -> PlanResult:
    path = np.zeros((0, dof))
    if r.path_len and bool(r.path):
        path = np.ctypeslib.as_array(r.path, shape=(r.path_len * dof,)).reshape(r.path_len, dof).copy()
    return PlanResult(
        status=PlanStatus(r.status),
        path=path,
        cost=r.cost,
        wall_time_ms=r.wall_time_ms,
        iterations_total=r.iterations_total,
        check_stats=CheckStatsSnapshot(r.sphere_tests, r.fk_calls, r.fine_stage_entries),
        solving_worker=r.solving_worker,
        message=r.message.decode(errors="replace"),
        device_time_ms=r.device_time_ms,
        tree_nodes=(int(r.tree_nodes[0]), int(r.tree_nodes[1])),
        flops=int(r.flops),
        path_check=int(r.path_check),
    )


def _result_dtype() -> np.dtype:
    """numpy view of prrtc_result (pointer fields as uint64)."""
    names, formats, offsets = [], [], []
    for name, ctype in Result._fields_:
        off = getattr(Result, name).offset
        if name == "path":
            fmt = np.uint64
        elif name == "message":
            fmt = "S128"
        elif name == "tree_nodes":
            fmt = (np.uint64, 2)
        else:
            fmt = np.dtype(ctype)
        names.append(name)
        formats.append(fmt)
        offsets.append(off)
    return np.dtype({"names": names, "formats": formats, "offsets": offsets, "itemsize": C.sizeof(Result)})


_RESULT_DTYPE = None


class BatchResult:
    """Array view of a batch's results (no per-problem Python objects):
    status / cost / iterations_total / device_time_ms / flops / path_check
    arrays, and all paths back to back in `path_data` (config-major doubles)
    with `path_offsets[n + 1]` (in doubles); `paths` gives per-problem views."""

    def __init__(self, res, n: int, dof: int):
        global _RESULT_DTYPE
        if _RESULT_DTYPE is None:
            _RESULT_DTYPE = _result_dtype()
        a = np.frombuffer(res, dtype=_RESULT_DTYPE, count=n)
        self.status = a["status"].copy()
        self.cost = a["cost"].copy()
        self.iterations_total = a["iterations_total"].copy()
        self.device_time_ms = a["device_time_ms"].copy()
        self.flops = a["flops"].copy()
        self.path_check = a["path_check"].copy()
        self.dof = dof
        lib = _lib.load()
        self.path_offsets = np.zeros(n + 1, dtype=np.uint64)
        offp = self.path_offsets.ctypes.data_as(C.POINTER(C.c_uint64))
        # sized from the results' own path lengths (a result without a path has path_len 0)
        total = int(np.sum(a["path_len"].astype(np.uint64) * (a["path"] != 0))) * dof
        self.path_data = np.empty(total, dtype=np.float64)
        check(lib.prrtc_results_pack_paths(res, n, _dptr(self.path_data), offp))
        assert int(self.path_offsets[-1]) == total

    @property
    def paths(self) -> list:
        o = self.path_offsets.astype(np.int64)
        return [self.path_data[o[i]:o[i + 1]].reshape(-1, self.dof) for i in range(len(o) - 1)]


def _cfg(q, dof: int, what: str) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(q, dtype=np.float64))
    if a.ndim != 1 or a.shape[0] != dof:  # require_dim (types.hpp:16-21)
        raise ValueError(f"{what}: expected dimension {dof}, got {a.shape[-1] if a.ndim else 0}")
    return a


def plan(model, scene, start, goal, params: PlannerParams | None = None, device: int = 0) -> PlanResult:
    """Drop-in for prrtc::plan (planner.cpp:246-322), computed on the B200."""
    params = params or PlannerParams()
    rob = device_robot(model, device)
    scn = device_scene(scene, device)
    s = _cfg(start, rob.dof, "plan.start")
    g = _cfg(goal, rob.dof, "plan.goal")
    p = params.to_c()
    r = Result()
    check(_lib.load().prrtc_plan(rob.h, scn.h, _dptr(s), _dptr(g), rob.dof, C.byref(p), C.byref(r)))
    try:
        return _to_result(r, rob.dof)
    finally:
        _lib.load().prrtc_result_free(C.byref(r))


class SceneSet:
    """Per-problem scene handles packed once for repeated batch calls (setup,
    like device_scene): plan_batch* accepts it in place of a scene list."""

    def __init__(self, scenes, device: int = 0):
        self.device = device
        self.hs = [device_scene(s, device) for s in scenes]
        self.arr = (C.c_void_p * len(self.hs))(*[h.h.value for h in self.hs])

    def __len__(self) -> int:
        return len(self.hs)


def device_scenes(scenes, device: int = 0) -> SceneSet:
    return SceneSet(scenes, device)


def _scene_handles(scenes, n, device):
    if isinstance(scenes, SceneSet):
        if len(scenes) != n or scenes.device != device:
            raise ValueError("plan_batch: SceneSet must hold one scene per problem on the same device")
        return scenes.hs, scenes.arr
    if isinstance(scenes, (Scene, DeviceScene)):
        scenes = [scenes] * n
    if len(scenes) != n:
        raise ValueError("plan_batch: one scene per problem required")
    hs = [device_scene(s, device) for s in scenes]
    arr = (C.c_void_p * n)(*[h.h.value for h in hs])
    return hs, arr


def _plan_batch_raw(model, scenes, starts, goals, params, device):
    params = params or PlannerParams()
    rob = device_robot(model, device)
    S = np.ascontiguousarray(np.asarray(starts, dtype=np.float64).reshape(-1, rob.dof))
    G = np.ascontiguousarray(np.asarray(goals, dtype=np.float64).reshape(-1, rob.dof))
    n = S.shape[0]
    hs, arr = _scene_handles(scenes, n, device)
    p = params.to_c()
    res = (Result * n)()
    check(_lib.load().prrtc_plan_batch(rob.h, arr, n, _dptr(S), _dptr(G), rob.dof, C.byref(p), res))
    return rob, res, n, hs


def _free(res, n):
    _lib.load().prrtc_results_free(res, n)


def plan_batch(model, scenes, starts, goals, params: PlannerParams | None = None,
               device: int = 0) -> list[PlanResult]:
    """n independent problems (one robot, one scene each) in one device launch."""
    rob, res, n, hs = _plan_batch_raw(model, scenes, starts, goals, params, device)
    out = [_to_result(res[i], rob.dof) for i in range(n)]
    _free(res, n)
    return out


def plan_batch_arrays(model, scenes, starts, goals, params: PlannerParams | None = None,
                      device: int = 0) -> BatchResult:
    """plan_batch returning arrays (BatchResult) instead of n PlanResult objects.
    Pass DeviceScene handles (device_scene(s)) to keep scene setup out of the call."""
    rob, res, n, hs = _plan_batch_raw(model, scenes, starts, goals, params, device)
    out = BatchResult(res, n, rob.dof)
    _free(res, n)
    return out


def plan_batch_multi(model, scenes, starts, goals, params: PlannerParams | None = None,
                     devices: Sequence[int] | None = None, chunk: int = 0) -> BatchResult:
    """prrtc_plan_batch_multi: the problems spread over several devices (one
    host thread per device, a shared chunk queue, no collective; SURVEY.md
    §8e). devices = None uses every visible sm_100 device. Robot and scene
    handles are uploaded to each device (setup, cached)."""
    params = params or PlannerParams()
    devices = list(range(device_count())) if devices is None else list(devices)
    if not devices:
        raise RuntimeError("plan_batch_multi: no sm_100 device")
    robs = [device_robot(model, d) for d in devices]
    dof = robs[0].dof
    S = np.ascontiguousarray(np.asarray(starts, dtype=np.float64).reshape(-1, dof))
    G = np.ascontiguousarray(np.asarray(goals, dtype=np.float64).reshape(-1, dof))
    n = S.shape[0]
    src = scenes.hs if isinstance(scenes, SceneSet) else scenes
    if isinstance(src, (Scene, DeviceScene)):
        src = [src] * n
    if len(src) != n:
        raise ValueError("plan_batch: one scene per problem required")
    keep, handles = [], []
    for d in devices:  # per-device handles (a handle of another device is re-uploaded from its Scene)
        hs = [x if isinstance(x, DeviceScene) and x.device == d
              else device_scene(x.scene if isinstance(x, DeviceScene) else x, d) for x in src]
        keep.append(hs)
        handles.extend(h.h.value for h in hs)
    rarr = (C.c_void_p * len(devices))(*[r.h.value for r in robs])
    sarr = (C.c_void_p * len(handles))(*handles)
    p = params.to_c()
    res = (Result * n)()
    check(_lib.load().prrtc_plan_batch_multi(rarr, sarr, len(devices), n, _dptr(S), _dptr(G), dof, C.byref(p),
                                             chunk, res))
    out = BatchResult(res, n, dof)
    _free(res, n)
    return out


def debug_chunk_queue(n_workers: int, n: int, chunk: int = 0, delay_us=None):
    """The multi-device chunk queue without devices: (owner[n], chunks_taken[n_workers])."""
    owner = np.zeros(n, dtype=np.int32)
    taken = np.zeros(n_workers, dtype=np.uint32)
    dl = None
    if delay_us is not None:
        dl = np.ascontiguousarray(np.asarray(delay_us, dtype=np.uint32))
    check(_lib.load().prrtc_debug_chunk_queue(n_workers, n, chunk,
                                              dl.ctypes.data_as(C.POINTER(C.c_uint32)) if dl is not None else None,
                                              owner.ctypes.data_as(C.POINTER(C.c_int32)),
                                              taken.ctypes.data_as(C.POINTER(C.c_uint32))))
    return owner, taken


class Batch:
    """Device-resident batch: inputs uploaded once (prrtc_batch_create), then
    solved repeatedly with launch(); results() copies the outcome back."""

    def __init__(self, model, scenes, starts, goals, params: PlannerParams | None = None, device: int = 0):
        self.params = params or PlannerParams()
        self.rob = device_robot(model, device)
        S = np.ascontiguousarray(np.asarray(starts, dtype=np.float64).reshape(-1, self.rob.dof))
        G = np.ascontiguousarray(np.asarray(goals, dtype=np.float64).reshape(-1, self.rob.dof))
        self.n = S.shape[0]
        self._hs, arr = _scene_handles(scenes, self.n, device)
        p = self.params.to_c()
        h = C.c_void_p()
        check(_lib.load().prrtc_batch_create(self.rob.h, arr, self.n, _dptr(S), _dptr(G), self.rob.dof,
                                             C.byref(p), C.byref(h)))
        self.h = h

    def launch(self, stream: int = 0) -> None:
        check(_lib.load().prrtc_batch_launch(self.h, C.c_void_p(stream)))

    def launch_count(self) -> int:
        return _lib.load().prrtc_batch_launch_count(self.h)

    def results(self) -> list[PlanResult]:
        res = (Result * self.n)()
        check(_lib.load().prrtc_batch_results(self.h, res))
        out = [_to_result(res[i], self.rob.dof) for i in range(self.n)]
        for i in range(self.n):
            _lib.load().prrtc_result_free(C.byref(res[i]))
        return out

    def __del__(self):
        if getattr(self, "h", None) and getattr(_lib, "_lib", None) is not None:  # module globals may be gone at exit
            _lib._lib.prrtc_batch_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------------------
# batched collision checking (product API)
# ---------------------------------------------------------------------------
def validate_edges(model, scene, frm, to, n_cc: int = 32, two_stage: bool = True,
                   early_exit: bool = True, device: int = 0) -> np.ndarray:
    """CollisionChecker::validate_edge over many edges (collision.cpp:206-224)."""
    rob = device_robot(model, device)
    scn = device_scene(scene, device)
    F = np.ascontiguousarray(np.asarray(frm, dtype=np.float64).reshape(-1, rob.dof))
    T = np.ascontiguousarray(np.asarray(to, dtype=np.float64).reshape(-1, rob.dof))
    out = np.zeros(F.shape[0], dtype=np.uint8)
    check(_lib.load().prrtc_validate_edges(rob.h, scn.h, _dptr(F), _dptr(T), F.shape[0], rob.dof, n_cc,
                                           int(two_stage), int(early_exit),
                                           out.ctypes.data_as(C.POINTER(C.c_uint8))))
    return out.astype(bool)


def check_configs(model, scene, q, two_stage: bool = True, device: int = 0) -> np.ndarray:
    """CollisionChecker::check_config over many configurations (collision.cpp:130-204)."""
    rob = device_robot(model, device)
    scn = device_scene(scene, device)
    Q = np.ascontiguousarray(np.asarray(q, dtype=np.float64).reshape(-1, rob.dof))
    out = np.zeros(Q.shape[0], dtype=np.uint8)
    check(_lib.load().prrtc_check_configs(rob.h, scn.h, _dptr(Q), Q.shape[0], rob.dof, int(two_stage),
                                          out.ctypes.data_as(C.POINTER(C.c_uint8))))
    return out.astype(bool)


# ---------------------------------------------------------------------------
# parity hooks
# ---------------------------------------------------------------------------
def debug_fk(model, q, device: int = 0):
    """Posed fine [n,S,3] and coarse [n,L,3] sphere centers (FP32) as the
    device collision code sees them."""
    rob = device_robot(model, device)
    Q = np.ascontiguousarray(np.asarray(q, dtype=np.float64).reshape(-1, rob.dof))
    n = Q.shape[0]
    fine = np.zeros((n, rob.fine_count, 3), dtype=np.float32)
    coarse = np.zeros((n, rob.n_links, 3), dtype=np.float32)
    FPT = C.POINTER(C.c_float)
    check(_lib.load().prrtc_debug_fk(rob.h, _dptr(Q), n, rob.dof, fine.ctypes.data_as(FPT),
                                     coarse.ctypes.data_as(FPT)))
    return fine, coarse


def debug_check_edges(model, scene, frm, to, n_cc: int = 32, two_stage: bool = True, device: int = 0):
    """Per-state device verdicts [n_edges, n_cc] (no early exit) and the posed
    fine spheres [n_edges, n_cc, S, 3] (FP32) the device's checks used."""
    rob = device_robot(model, device)
    scn = device_scene(scene, device)
    F = np.ascontiguousarray(np.asarray(frm, dtype=np.float64).reshape(-1, rob.dof))
    T = np.ascontiguousarray(np.asarray(to, dtype=np.float64).reshape(-1, rob.dof))
    n = F.shape[0]
    valid = np.zeros((n, n_cc), dtype=np.uint8)
    fine = np.zeros((n, n_cc, rob.fine_count, 3), dtype=np.float32)
    check(_lib.load().prrtc_debug_check_edges(rob.h, scn.h, _dptr(F), _dptr(T), n, rob.dof, n_cc, int(two_stage),
                                              valid.ctypes.data_as(C.POINTER(C.c_uint8)),
                                              fine.ctypes.data_as(C.POINTER(C.c_float))))
    return valid.astype(bool), fine


def debug_sphere_hits(scene, centers, radii, device: int = 0) -> np.ndarray:
    """Device predicate verdicts [n, P] (primitive order: spheres, boxes, capsules)."""
    scn = device_scene(scene, device)
    X = np.ascontiguousarray(np.asarray(centers, dtype=np.float32).reshape(-1, 3))
    R = np.ascontiguousarray(np.asarray(radii, dtype=np.float64).reshape(-1))
    out = np.zeros((X.shape[0], scn.n_prims), dtype=np.uint8)
    check(_lib.load().prrtc_debug_sphere_hits(scn.h, X.ctypes.data_as(C.POINTER(C.c_float)), _dptr(R),
                                              X.shape[0], out.ctypes.data_as(C.POINTER(C.c_uint8))))
    return out.astype(bool)


def debug_nn(tree, q, device: int = 0, group: int = 0):
    """Device nearest neighbour: (index[nq], squared distance[nq]); group > 0
    runs the planner's multi-sample pass on `group` queries at a time."""
    T = np.ascontiguousarray(np.asarray(tree, dtype=np.float64))
    Q = np.ascontiguousarray(np.asarray(q, dtype=np.float64).reshape(-1, T.shape[1]))
    idx = np.zeros(Q.shape[0], dtype=np.uint32)
    d2 = np.zeros(Q.shape[0], dtype=np.float64)
    check(_lib.load().prrtc_debug_nn_multi(_dptr(T), T.shape[0], T.shape[1], _dptr(Q), Q.shape[0], group, device,
                                           idx.ctypes.data_as(C.POINTER(C.c_uint32)), _dptr(d2)))
    return idx, d2


def debug_halton(bases: Sequence[int], indices: Sequence[int], device: int = 0) -> np.ndarray:
    B = np.ascontiguousarray(np.asarray(bases, dtype=np.uint32))
    I = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
    out = np.zeros(B.shape[0], dtype=np.float64)
    check(_lib.load().prrtc_debug_halton(B.ctypes.data_as(C.POINTER(C.c_uint32)),
                                         I.ctypes.data_as(C.POINTER(C.c_uint64)), B.shape[0], device,
                                         _dptr(out)))
    return out


def debug_sample(model, index0: int, n: int, device: int = 0) -> np.ndarray:
    rob = device_robot(model, device)
    out = np.zeros((n, rob.dof), dtype=np.float64)
    check(_lib.load().prrtc_debug_sample(rob.h, index0, n, _dptr(out)))
    return out


def reload_env() -> None:
    """Make the library re-read its PRRTC_* environment switches (it caches them)."""
    check(_lib.load().prrtc_debug_reload_env())


def device_count() -> int:
    return _lib.load().prrtc_device_count()


def default_workers(device: int = 0) -> int:
    """CTAs prrtc_plan uses on one problem when params.workers == 0."""
    lib = _lib.load()
    n = lib.prrtc_default_workers(device)
    check(min(n, 0))
    return n
