"""TEST INFRASTRUCTURE — ctypes binding of the oracle libraries (see __init__)."""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
LIBS = {"ref": HERE / "_ref" / "libprrtc_ref.so", "port": HERE / "liboracle.so"}
PREFIX = {"ref": "ref_", "port": "orc_"}

if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2503_06757_b200._lib import Params, Result, RobotDesc, SceneDesc  # noqa: E402  (plain C structs)

P = C.c_void_p
DP = C.POINTER(C.c_double)
U8P = C.POINTER(C.c_uint8)
U64P = C.POINTER(C.c_uint64)

_SIGS = [
    ("last_error", C.c_int, [C.c_char_p, C.c_size_t]),
    ("robot_create", P, [C.POINTER(RobotDesc)]),
    ("robot_destroy", None, [P]),
    ("robot_dof", C.c_int, [P]),
    ("scene_create", P, [C.POINTER(SceneDesc)]),
    ("scene_destroy", None, [P]),
    ("force_scalar", C.c_int, [C.c_int]),
    ("fk_poses", C.c_int, [P, DP, DP]),
    ("fk_spheres", C.c_int, [P, DP, C.c_int, DP]),
    ("sphere_hits", C.c_int, [P, C.c_double, C.c_double, C.c_double, C.c_double, U8P]),
    ("check_config", C.c_int, [P, P, DP, C.c_int, C.c_int, U64P]),
    ("check_configs", C.c_int, [P, P, DP, C.c_uint32, C.c_int, U8P]),
    ("validate_edge", C.c_int, [P, P, DP, DP, C.c_int, C.c_int, C.c_int, U64P]),
    ("validate_edges", C.c_int, [P, P, DP, DP, C.c_uint32, C.c_int, C.c_int, C.c_int, U8P]),
    ("validate_edge_batched", C.c_int, [P, P, DP, DP, C.c_uint32, C.c_int, C.c_int, C.c_int, U8P, U64P]),
    ("nearest_serial", C.c_int64, [DP, C.c_uint64, C.c_uint32, DP, DP]),
    ("nearest_parallel", C.c_int64, [DP, C.c_uint64, C.c_uint32, DP, C.c_uint64, DP]),
    ("sq_distance", C.c_double, [DP, DP, C.c_uint32]),
    ("halton_value", C.c_double, [C.c_uint, C.c_uint64]),
    ("halton_bases", C.c_int, [C.c_uint32, C.POINTER(C.c_uint32)]),
    ("sample_config", C.c_int, [P, C.c_uint64, C.c_uint64, C.c_uint32, DP]),
    ("plan", C.c_int, [P, P, DP, DP, C.POINTER(Params), C.POINTER(Result)]),
    ("plan_many", C.c_double, [P, C.POINTER(P), C.c_uint32, DP, DP, C.POINTER(Params), C.c_uint32, C.POINTER(Result)]),
    ("result_free", None, [C.POINTER(Result)]),
    ("path_valid", C.c_int, [P, P, DP, C.c_uint32, C.c_int]),
    ("path_cost", C.c_double, [DP, C.c_uint32, C.c_uint32]),
]


def available(kind: str) -> bool:
    return LIBS[kind].exists()


def _dp(a):
    return a.ctypes.data_as(DP)


class Oracle:
    def __init__(self, kind: str = "ref"):
        path = LIBS[kind]
        if not path.exists():
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(str(path))
        self.fn = {}
        for name, res, args in _SIGS:
            f = getattr(self.lib, PREFIX[kind] + name)
            f.restype = res
            f.argtypes = args
            self.fn[name] = f
        # optional: threaded batch path check (reference build only)
        self._many = getattr(self.lib, PREFIX[kind] + "paths_valid_many", None)
        if self._many is not None:
            self._many.restype = C.c_int
            self._many.argtypes = [P, C.POINTER(P), C.c_uint32, DP, U64P, C.c_int, C.c_uint32, U8P]
        self._anyhit = getattr(self.lib, PREFIX[kind] + "sphere_any_hits", None)
        if self._anyhit is not None:
            self._anyhit.restype = C.c_int
            self._anyhit.argtypes = [P, DP, C.c_uint32, U8P]
        self._robots = {}
        self._scenes = {}

    # ---- handles ----
    def err(self) -> str:
        b = C.create_string_buffer(512)
        self.fn["last_error"](b, 512)
        return b.value.decode()

    def robot(self, model):
        key = repr(model)
        if key not in self._robots:
            d, keep = model.to_desc()
            h = self.fn["robot_create"](C.byref(d))
            if not h:
                raise ValueError(self.err())
            self._robots[key] = (h, model.dof, model)
        return self._robots[key]

    def scene(self, scene):
        key = repr(scene)
        if key not in self._scenes:
            if len(self._scenes) > 20000:
                self._scenes.clear()
            d, keep = scene.to_desc()
            h = self.fn["scene_create"](C.byref(d))
            if not h:
                raise ValueError(self.err())
            self._scenes[key] = h
        return self._scenes[key]

    def force_scalar(self, on: bool = True) -> bool:
        return bool(self.fn["force_scalar"](int(on)))

    # ---- kinematics ----
    def fk_poses(self, model, q) -> np.ndarray:
        h, dof, m = self.robot(model)
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros((m.link_count(), 12))
        if self.fn["fk_poses"](h, _dp(q), _dp(out)) < 0:
            raise ValueError(self.err())
        return out

    def fk_spheres(self, model, q, fine: bool = True) -> np.ndarray:
        h, dof, m = self.robot(model)
        q = np.ascontiguousarray(q, dtype=np.float64)
        n = m.fine_count() if fine else m.link_count()
        out = np.zeros((n, 4))
        if self.fn["fk_spheres"](h, _dp(q), int(fine), _dp(out)) < 0:
            raise ValueError(self.err())
        return out

    # ---- collision ----
    def sphere_hits(self, scene, x, y, z, r) -> np.ndarray:
        s = self.scene(scene)
        out = np.zeros(max(1, len(scene.primitives)), dtype=np.uint8)
        self.fn["sphere_hits"](s, float(x), float(y), float(z), float(r), out.ctypes.data_as(U8P))
        return out[: len(scene.primitives)].astype(bool)

    def sphere_any_hits(self, scene, xyzr) -> np.ndarray:
        """Per sphere (rows x, y, z, r): does the reference predicate
        sphere_vs_primitive flag any primitive of the scene."""
        X = np.ascontiguousarray(np.asarray(xyzr, dtype=np.float64).reshape(-1, 4))
        out = np.zeros(X.shape[0], dtype=np.uint8)
        if self._anyhit is not None:
            self._anyhit(self.scene(scene), _dp(X), X.shape[0], out.ctypes.data_as(U8P))
        else:
            for i, (x, y, z, r) in enumerate(X):
                out[i] = bool(self.sphere_hits(scene, x, y, z, r).any())
        return out.astype(bool)

    def check_config(self, model, scene, q, two_stage=True, early_exit=True, stats=False):
        h, dof, _ = self.robot(model)
        q = np.ascontiguousarray(q, dtype=np.float64)
        st = np.zeros(3, dtype=np.uint64)
        r = self.fn["check_config"](h, self.scene(scene), _dp(q), int(two_stage), int(early_exit),
                                    st.ctypes.data_as(U64P))
        if r < 0:
            raise ValueError(self.err())
        return (bool(r), st) if stats else bool(r)

    def check_configs(self, model, scene, q, two_stage=True) -> np.ndarray:
        h, dof, _ = self.robot(model)
        q = np.ascontiguousarray(np.asarray(q, dtype=np.float64).reshape(-1, dof))
        out = np.zeros(q.shape[0], dtype=np.uint8)
        if self.fn["check_configs"](h, self.scene(scene), _dp(q), q.shape[0], int(two_stage),
                                    out.ctypes.data_as(U8P)) < 0:
            raise ValueError(self.err())
        return out.astype(bool)

    def validate_edge(self, model, scene, frm, to, n=32, two_stage=True, early_exit=True, stats=False):
        h, dof, _ = self.robot(model)
        a = np.ascontiguousarray(frm, dtype=np.float64)
        b = np.ascontiguousarray(to, dtype=np.float64)
        st = np.zeros(3, dtype=np.uint64)
        r = self.fn["validate_edge"](h, self.scene(scene), _dp(a), _dp(b), n, int(two_stage),
                                     int(early_exit), st.ctypes.data_as(U64P))
        if r < 0:
            raise ValueError(self.err())
        return (bool(r), st) if stats else bool(r)

    def validate_edges(self, model, scene, frm, to, n=32, two_stage=True, early_exit=True) -> np.ndarray:
        h, dof, _ = self.robot(model)
        a = np.ascontiguousarray(np.asarray(frm, dtype=np.float64).reshape(-1, dof))
        b = np.ascontiguousarray(np.asarray(to, dtype=np.float64).reshape(-1, dof))
        out = np.zeros(a.shape[0], dtype=np.uint8)
        if self.fn["validate_edges"](h, self.scene(scene), _dp(a), _dp(b), a.shape[0], n, int(two_stage),
                                     int(early_exit), out.ctypes.data_as(U8P)) < 0:
            raise ValueError(self.err())
        return out.astype(bool)

    def validate_edge_batched(self, model, scene, frm, to, n=32, two_stage=True, early_exit=True):
        h, dof, _ = self.robot(model)
        a = np.ascontiguousarray(np.asarray(frm, dtype=np.float64).reshape(-1, dof))
        b = np.ascontiguousarray(np.asarray(to, dtype=np.float64).reshape(-1, dof))
        out = np.zeros(max(1, a.shape[0]), dtype=np.uint8)
        st = np.zeros(3, dtype=np.uint64)
        if self.fn["validate_edge_batched"](h, self.scene(scene), _dp(a), _dp(b), a.shape[0], n,
                                            int(two_stage), int(early_exit), out.ctypes.data_as(U8P),
                                            st.ctypes.data_as(U64P)) < 0:
            raise ValueError(self.err())
        return out[: a.shape[0]].astype(bool), st

    # ---- nearest neighbour / sampling ----
    def nearest_serial(self, tree, q):
        t = np.ascontiguousarray(tree, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        d = C.c_double()
        i = self.fn["nearest_serial"](_dp(t), t.shape[0], t.shape[1], _dp(q), C.byref(d))
        if i < 0:
            raise ValueError(self.err())
        return int(i), d.value

    def nearest_parallel(self, tree, q, partitions):
        t = np.ascontiguousarray(tree, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        d = C.c_double()
        i = self.fn["nearest_parallel"](_dp(t), t.shape[0], t.shape[1], _dp(q), partitions, C.byref(d))
        if i < 0:
            raise ValueError(self.err())
        return int(i), d.value

    def sq_distance(self, a, b) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return self.fn["sq_distance"](_dp(a), _dp(b), a.shape[0])

    def halton_value(self, base: int, index: int) -> float:
        return self.fn["halton_value"](base, index)

    def halton_bases(self, n: int) -> list[int]:
        out = (C.c_uint32 * n)()
        self.fn["halton_bases"](n, out)
        return list(out)

    def sample_config(self, model, offset: int, stride: int, n: int) -> np.ndarray:
        h, dof, _ = self.robot(model)
        out = np.zeros((n, dof))
        if self.fn["sample_config"](h, offset, stride, n, _dp(out)) < 0:
            raise ValueError(self.err())
        return out

    # ---- planner ----
    def plan(self, model, scene, start, goal, params=None):
        from paper_2503_06757_b200.model import PlannerParams
        from paper_2503_06757_b200.planner import _to_result
        params = params or PlannerParams()
        h, dof, _ = self.robot(model)
        s = np.ascontiguousarray(start, dtype=np.float64)
        g = np.ascontiguousarray(goal, dtype=np.float64)
        p = params.to_c()
        r = Result()
        if self.fn["plan"](h, self.scene(scene), _dp(s), _dp(g), C.byref(p), C.byref(r)) < 0:
            raise ValueError(self.err())
        try:
            return _to_result(r, dof)
        finally:
            self.fn["result_free"](C.byref(r))

    def plan_many(self, model, scenes, starts, goals, params=None, threads: int = 1):
        """Independent problems on `threads` host threads; returns (results, wall_ms)."""
        from paper_2503_06757_b200.model import PlannerParams
        from paper_2503_06757_b200.planner import _to_result
        params = params or PlannerParams()
        h, dof, _ = self.robot(model)
        S = np.ascontiguousarray(np.asarray(starts, dtype=np.float64).reshape(-1, dof))
        G = np.ascontiguousarray(np.asarray(goals, dtype=np.float64).reshape(-1, dof))
        n = S.shape[0]
        sh = (C.c_void_p * n)(*[self.scene(s) for s in scenes])
        p = params.to_c()
        res = (Result * n)()
        ms = self.fn["plan_many"](h, sh, n, _dp(S), _dp(G), C.byref(p), threads, res)
        out = []
        for i in range(n):
            if res[i].status < 0:
                raise ValueError(res[i].message.decode())
            out.append(_to_result(res[i], dof))
            self.fn["result_free"](C.byref(res[i]))
        return out, ms

    def path_valid(self, model, scene, path, n: int) -> bool:
        h, dof, _ = self.robot(model)
        p = np.ascontiguousarray(np.asarray(path, dtype=np.float64).reshape(-1, dof))
        r = self.fn["path_valid"](h, self.scene(scene), _dp(p), p.shape[0], n)
        if r < 0:
            raise ValueError(self.err())
        return bool(r)

    def paths_valid(self, model, scenes, paths, n: int, threads: int = 1) -> np.ndarray:
        """path_valid over a list of paths (one scene each): bool array."""
        h, dof, _ = self.robot(model)
        if self._many is None or threads <= 1:
            return np.array([len(p) > 0 and self.path_valid(model, s, p, n) for s, p in zip(scenes, paths)])
        ps = [np.ascontiguousarray(np.asarray(p, dtype=np.float64).reshape(-1, dof)) for p in paths]
        off = np.zeros(len(ps) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([p.size for p in ps])
        data = np.concatenate([p.ravel() for p in ps]) if off[-1] else np.zeros(1)
        sh = (P * len(ps))(*[self.scene(s) for s in scenes])
        out = np.zeros(len(ps), dtype=np.uint8)
        self._many(h, sh, len(ps), _dp(data), off.ctypes.data_as(U64P), n, threads, out.ctypes.data_as(U8P))
        if (out == 2).any():
            raise ValueError(self.err())
        return out == 1

    def path_cost(self, path) -> float:
        p = np.ascontiguousarray(path, dtype=np.float64)
        return self.fn["path_cost"](_dp(p), p.shape[0], p.shape[1])
