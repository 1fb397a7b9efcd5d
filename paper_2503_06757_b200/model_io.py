"""Model I/O drop-in: the reference's JSON robot / scene / problem / path
formats and its results and ECDF CSVs.

    load_robot / load_scene / load_problem / load_path_file   model_io.cpp:91-342
    write_robot / write_scene / write_problem / write_path    model_io.cpp:344-421
    results_csv_string / write_results_csv / write_ecdf_csv   model_io.cpp:423-465
    ParamsPatch, ProblemSpec, PathFile, BenchRecord           model_io.hpp:25-84
    robot_finalize / scene_validate                           kinematics.cpp:15-74, geometry.cpp:10-39

Files written here are byte-identical to what the reference writes
(nlohmann::json ``dump(2)``: keys sorted, two-space indent, doubles in
shortest round-trip form with nlohmann's fixed/exponent switch points) and
files the reference writes load here to the same values; IoError messages
name the file and the offending field exactly like the reference's.
``tests/test_model_io.py`` checks both directions against the compiled
reference (oracle/_ref) and against committed fixtures.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field, fields
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

from .model import (FIXED, PRISMATIC, REVOLUTE, BoxPrim, CapsulePrim, Joint, LinkSpheres,
                    PlannerParams, PlanStatus, RobotModel, SamplerKind, Scene, Sphere,
                    SpherePrim)


class IoError(RuntimeError):
    """model_io.hpp:19-22: unreadable files, malformed JSON, schema and
    invariant violations; the message names the file and offending field."""


class JsonTypeError(RuntimeError):
    """A nlohmann::json type_error escaping an unguarded ``get<T>()``
    (e.g. ``vec3_from``, model_io.cpp:48-51) — not an IoError in the reference."""


# ---------------------------------------------------------------------------
# host-side model invariants (the reference checks them in finalize/validate)
# ---------------------------------------------------------------------------

def _cpp_to_string(x: float) -> str:
    """std::to_string(double) == printf("%f")."""
    return "%f" % x


def robot_finalize(model: RobotModel) -> None:
    """RobotModel::finalize (kinematics.cpp:15-74) invariants, same messages.
    Raises ValueError (the reference's std::invalid_argument)."""
    name = model.name
    n = len(model.joints)
    if n == 0:
        raise ValueError(f"robot '{name}': joints must be non-empty")
    if len(model.spheres) != n:
        raise ValueError(f"robot '{name}': spheres must have one entry per joint "
                         f"({len(model.spheres)} vs {n})")
    for i, j in enumerate(model.joints):
        where = f"robot '{name}' joints[{i}]"
        if j.parent >= i:
            raise ValueError(where + ".parent: must be smaller than the joint index")
        if j.parent < -1:
            raise ValueError(where + ".parent: out of range")
        w, x, y, z = j.origin_quat
        qn = math.sqrt(w * w + x * x + y * y + z * z)  # Quat::norm (transform.hpp:92-95)
        if abs(qn - 1.0) > 1e-6:
            raise ValueError(where + ".origin.quaternion: norm deviates from 1 by more than 1e-6 ("
                             + _cpp_to_string(qn) + ")")
        if j.kind != FIXED:
            an = math.sqrt(j.axis[0] * j.axis[0] + j.axis[1] * j.axis[1] + j.axis[2] * j.axis[2])
            if abs(an - 1.0) > 1e-9:
                raise ValueError(where + ".axis: must be unit length, |axis| = " + _cpp_to_string(an))
            if not (j.lo <= j.hi):
                raise ValueError(where + ".limits: lo must be <= hi")
    for l, ls in enumerate(model.spheres):
        where = f"robot '{name}' spheres[{l}]"
        if not (ls.coarse.radius > 0.0):
            raise ValueError(where + ".coarse.radius: must be positive")
        cc = ls.coarse.center
        for k, f in enumerate(ls.fine):
            if not (f.radius > 0.0):
                raise ValueError(where + f".fine[{k}].radius: must be positive")
            dx, dy, dz = f.center[0] - cc[0], f.center[1] - cc[1], f.center[2] - cc[2]
            reach = math.sqrt(dx * dx + dy * dy + dz * dz) + f.radius
            if reach > ls.coarse.radius + 1e-9:
                raise ValueError(where + f".fine[{k}]: escapes the coarse bounding sphere by "
                                 + _cpp_to_string(reach - ls.coarse.radius))
    for p, (a, b) in enumerate(model.self_pairs):
        where = f"robot '{name}' self_pairs[{p}]"
        if a < 0 or b < 0 or a >= n or b >= n:
            raise ValueError(where + ": link index out of range")
        if a == b:
            raise ValueError(where + ": a link cannot pair with itself")
        if model.joints[a].parent == b or model.joints[b].parent == a:
            raise ValueError(where + ": adjacent parent-child links must not be tested")


def scene_validate(scene: Scene) -> None:
    """Scene::validate (geometry.cpp:10-39), same messages (ValueError)."""
    for i, p in enumerate(scene.primitives):
        where = f"scene '{scene.name}' primitives[{i}]"
        if isinstance(p, BoxPrim):
            h = p.half_extents
            if not (h[0] > 0.0 and h[1] > 0.0 and h[2] > 0.0):
                raise ValueError(where + ".half_extents: must be componentwise positive")
            w, x, y, z = p.quat
            if abs(math.sqrt(w * w + x * x + y * y + z * z) - 1.0) > 1e-6:
                raise ValueError(where + ".pose.quaternion: norm deviates from 1 by more than 1e-6")
        else:
            if not (p.radius > 0.0):
                raise ValueError(where + ".radius: must be positive")


# ---------------------------------------------------------------------------
# types (model_io.hpp:25-84)
# ---------------------------------------------------------------------------

_PATCH_FIELDS = ("delta", "n_cc", "workers", "max_iters_per_worker", "tree_capacity", "dd_radius",
                 "dynamic_domain", "balance", "early_exit", "two_stage", "batched_cc", "nn_partitions",
                 "sampler", "seed")


@dataclass
class ParamsPatch:
    """model_io.hpp:25-44: optional PlannerParams overrides."""
    delta: Optional[float] = None
    n_cc: Optional[int] = None
    workers: Optional[int] = None
    max_iters_per_worker: Optional[int] = None
    tree_capacity: Optional[int] = None
    dd_radius: Optional[float] = None
    dynamic_domain: Optional[bool] = None
    balance: Optional[bool] = None
    early_exit: Optional[bool] = None
    two_stage: Optional[bool] = None
    batched_cc: Optional[bool] = None
    nn_partitions: Optional[int] = None
    sampler: Optional[int] = None
    seed: Optional[int] = None

    def apply(self, p: PlannerParams) -> PlannerParams:
        """ParamsPatch::apply (model_io.cpp:195-210). Note: like the
        reference's ``if (seed)``, a set-but-zero optional still applies
        (std::optional's bool is "has value")."""
        for name in _PATCH_FIELDS:
            v = getattr(self, name)
            if v is not None:
                setattr(p, name, v)
        return p


@dataclass
class ProblemSpec:  # model_io.hpp:46-55
    name: str = ""
    robot: str = ""  # as written in the file, relative to the file's directory
    scene: str = ""
    start: np.ndarray = field(default_factory=lambda: np.zeros(0))
    goal: np.ndarray = field(default_factory=lambda: np.zeros(0))
    params: ParamsPatch = field(default_factory=ParamsPatch)


@dataclass
class PathFile:  # model_io.hpp:57-66
    robot: str = ""
    scene: str = ""
    configs: list = field(default_factory=list)
    cost: float = 0.0
    params: PlannerParams = field(default_factory=PlannerParams)
    timestamp: str = ""


@dataclass
class BenchRecord:  # model_io.hpp:68-79
    problem: str = ""
    trial: int = 0
    status: PlanStatus = PlanStatus.Failed
    time_ms: float = 0.0
    cost: float = 0.0
    iterations: int = 0
    sphere_tests: int = 0
    workers: int = 1
    seed: int = 0
    config_hash: int = 0


def sampler_to_string(k: int) -> str:
    """to_string(SamplerKind) (model_io.cpp:212-214)."""
    return "halton" if int(k) == SamplerKind.Halton else "uniform"


def status_to_string(s: int) -> str:
    """to_string(PlanStatus) (planner.cpp:14-21)."""
    return {0: "Solved", 1: "Failed", 2: "Infeasible-endpoint"}.get(int(s), "?")


# ---------------------------------------------------------------------------
# JSON value access with nlohmann semantics
# ---------------------------------------------------------------------------

class _Num(float):
    """A parsed JSON float (keeps ints and floats apart like nlohmann)."""


def _reject_constant(name):
    raise ValueError(f"invalid literal {name}")


def _parse_file(path: Path):
    """parse_file (model_io.cpp:17-25)."""
    try:
        with open(path, "r", encoding="utf-8") as f:
            text = f.read()
    except OSError:
        raise IoError(f"{path}: cannot open file") from None
    try:
        return json.loads(text, parse_constant=_reject_constant)
    except ValueError as e:
        raise IoError(f"{path}: [json.exception.parse_error] {e}") from None


def _is_number(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _as(v, kind: str):
    """nlohmann get<T>(): numbers (and booleans) convert to arithmetic
    types, strings only to strings, booleans only to bool."""
    if kind == "double":
        if _is_number(v) or isinstance(v, bool):
            return float(v)
    elif kind in ("int", "unsigned", "uint64"):
        if _is_number(v) or isinstance(v, bool):
            x = int(v)
            if kind == "unsigned":
                x &= 0xFFFFFFFF
            elif kind == "uint64":
                x &= 0xFFFFFFFFFFFFFFFF
            elif kind == "int":
                x = ((x + 2**31) % 2**32) - 2**31
            return x
    elif kind == "bool":
        if isinstance(v, bool):
            return v
    elif kind == "string":
        if isinstance(v, str):
            return v
    raise JsonTypeError(f"[json.exception.type_error.302] type must be {kind}, but is {_type_name(v)}")


def _type_name(v) -> str:
    if v is None:
        return "null"
    if isinstance(v, bool):
        return "boolean"
    if _is_number(v):
        return "number"
    if isinstance(v, str):
        return "string"
    if isinstance(v, list):
        return "array"
    return "object"


def _field(j, key: str, where: str):
    """field (model_io.cpp:33-37)."""
    if not isinstance(j, dict) or key not in j:
        if not isinstance(j, dict) and j is not None:
            # nlohmann's find() on a non-object returns end()
            pass
        raise IoError(f"{where}.{key}: missing field")
    return j[key]


def _field_as(j, key: str, kind: str, where: str):
    """field_as<T> (model_io.cpp:39-46)."""
    v = _field(j, key, where)
    try:
        return _as(v, kind)
    except JsonTypeError:
        raise IoError(f"{where}.{key}: wrong type") from None


def _value(j, key: str, default, kind: str):
    """json::value(key, default)."""
    if isinstance(j, dict) and key in j:
        return _as(j[key], kind)
    return default


def _vec3_from(j, where: str) -> tuple:
    """vec3_from (model_io.cpp:48-51)."""
    if not isinstance(j, list) or len(j) != 3:
        raise IoError(f"{where}: expected an array of 3 numbers")
    return (_as(j[0], "double"), _as(j[1], "double"), _as(j[2], "double"))


def _pose_from(j, where: str):
    """pose_from (model_io.cpp:55-64) -> (quat w,x,y,z, translation)."""
    t = _vec3_from(_field(j, "translation", where), where + ".translation")
    q = _field(j, "quaternion", where)
    if not isinstance(q, list) or len(q) != 4:
        raise IoError(where + ".quaternion: expected an array of 4 numbers [w, x, y, z]")
    return tuple(_as(x, "double") for x in q), t


def _sphere_from(j, where: str) -> Sphere:
    """sphere_from (model_io.cpp:71-74)."""
    return Sphere(_vec3_from(_field(j, "center", where), where + ".center"),
                  _field_as(j, "radius", "double", where))


def _config_from(j, where: str) -> np.ndarray:
    """config_from (model_io.cpp:78-87)."""
    if not isinstance(j, list):
        raise IoError(f"{where}: expected an array of numbers")
    out = []
    for v in j:
        if not _is_number(v):
            raise IoError(f"{where}: expected an array of numbers")
        out.append(float(v))
    return np.array(out, dtype=np.float64)


# ---------------------------------------------------------------------------
# nlohmann dump(2)
# ---------------------------------------------------------------------------

class Int(int):
    """Marks a value to be written as a JSON integer."""


def _fmt_double(x: float) -> str:
    """nlohmann::detail::to_chars: shortest round-trip digits, then
    format_buffer with min_exp = -4, max_exp = 15 (fixed vs exponent),
    ".0" appended to integral fixed output, exponent as e+NN / e-NN."""
    if not math.isfinite(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    neg = x < 0
    r = repr(abs(x))
    # extract digits and decimal exponent from Python's shortest repr
    if "e" in r:
        mant, ex = r.split("e")
        ex = int(ex)
    else:
        mant, ex = r, 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    # value = 0.digits * 10^n  with n = position of the decimal point
    lead_zeros = len(ip + fp) - len((ip + fp).lstrip("0"))
    n = len(ip) + ex - lead_zeros
    digits = digits.rstrip("0") or "0"
    k = len(digits)
    if k <= n <= 15:
        s = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        m = digits[0] + ("." + digits[1:] if k > 1 else "")
        s = m + "e" + ("-" if e < 0 else "+") + ("%02d" % abs(e))
    return ("-" if neg else "") + s


def _esc(s: str) -> str:
    return json.dumps(s, ensure_ascii=False)


def dumps(v, indent: int = 2, _lvl: int = 0) -> str:
    """nlohmann::json::dump(indent) for the value kinds these files use."""
    pad = " " * (indent * (_lvl + 1))
    end = " " * (indent * _lvl)
    if isinstance(v, bool):
        return "true" if v else "false"
    if v is None:
        return "null"
    if isinstance(v, int):
        return str(int(v))
    if isinstance(v, float):
        return _fmt_double(v)
    if isinstance(v, str):
        return _esc(v)
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(pad + dumps(x, indent, _lvl + 1) for x in v) + "\n" + end + "]"
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = sorted(v.items())  # nlohmann::json objects are std::map
        return "{\n" + ",\n".join(pad + _esc(k) + ": " + dumps(x, indent, _lvl + 1) for k, x in items) \
            + "\n" + end + "}"
    raise TypeError(f"cannot serialise {type(v)}")


def _write_file(path: Path, j) -> None:
    """write_file (model_io.cpp:27-31)."""
    try:
        with open(path, "w", encoding="utf-8", newline="\n") as f:
            f.write(dumps(j) + "\n")
    except OSError:
        raise IoError(f"{path}: cannot open file for writing") from None


def _vec3_to(v) -> list:
    return [float(v[0]), float(v[1]), float(v[2])]


def _pose_to(quat, t) -> dict:
    return {"translation": _vec3_to(t), "quaternion": [float(q) for q in quat]}


def _sphere_to(s: Sphere) -> dict:
    return {"center": _vec3_to(s.center), "radius": float(s.radius)}


# ---------------------------------------------------------------------------
# loaders (model_io.cpp:91-342)
# ---------------------------------------------------------------------------

def load_robot(path) -> RobotModel:
    """load_robot (model_io.cpp:91-158)."""
    path = Path(path)
    j = _parse_file(path)
    where = str(path)
    name = _value(j, "name", path.stem, "string")
    joints_j = _field(j, "joints", where)
    if not isinstance(joints_j, list):
        raise IoError(where + ".joints: expected an array")
    joints = []
    for i, d in enumerate(joints_j):
        jw = f"{where}.joints[{i}]"
        kind_s = _field_as(d, "kind", "string", jw)
        kind = {"revolute": REVOLUTE, "prismatic": PRISMATIC, "fixed": FIXED}.get(kind_s)
        if kind is None:
            raise IoError(f"{jw}.kind: unknown joint kind '{kind_s}'")
        parent = _field_as(d, "parent", "int", jw)
        quat, xyz = _pose_from(_field(d, "origin", jw), jw + ".origin")
        joint = Joint(kind=kind, parent=parent, origin_quat=quat, origin_xyz=xyz)
        if kind != FIXED:
            joint.axis = _vec3_from(_field(d, "axis", jw), jw + ".axis")
            lim = _field(d, "limits", jw)
            if not isinstance(lim, list) or len(lim) != 2:
                raise IoError(jw + ".limits: expected [lo, hi]")
            joint.lo, joint.hi = _as(lim[0], "double"), _as(lim[1], "double")
        else:
            # Joint defaults (robot.hpp:17-26): axis (0,0,1), limits 0
            joint.axis, joint.lo, joint.hi = (0.0, 0.0, 1.0), 0.0, 0.0
        joints.append(joint)
    sph_j = _field(j, "spheres", where)
    if not isinstance(sph_j, list):
        raise IoError(where + ".spheres: expected an array")
    spheres = []
    for l, s in enumerate(sph_j):
        sw = f"{where}.spheres[{l}]"
        coarse = _sphere_from(_field(s, "coarse", sw), sw + ".coarse")
        fine_j = _field(s, "fine", sw)
        if not isinstance(fine_j, list):
            raise IoError(sw + ".fine: expected an array")
        fine = [_sphere_from(f, f"{sw}.fine[{k}]") for k, f in enumerate(fine_j)]
        spheres.append(LinkSpheres(coarse, fine))
    pairs = []
    if isinstance(j, dict) and "self_pairs" in j:
        pj = j["self_pairs"]
        if not isinstance(pj, list):
            raise IoError(where + ".self_pairs: expected an array of [i, j] pairs")
        for p in pj:
            if not isinstance(p, list) or len(p) != 2:
                raise IoError(where + ".self_pairs: expected an array of [i, j] pairs")
            pairs.append((_as(p[0], "int"), _as(p[1], "int")))
    model = RobotModel(name=name, joints=joints, spheres=spheres, self_pairs=pairs)
    try:
        robot_finalize(model)
    except ValueError as e:
        raise IoError(f"{where}: {e}") from None
    return model


def load_scene(path) -> Scene:
    """load_scene (model_io.cpp:160-193)."""
    path = Path(path)
    j = _parse_file(path)
    where = str(path)
    scene = Scene(name=_value(j, "name", path.stem, "string"))
    prims = _field(j, "primitives", where)
    if not isinstance(prims, list):
        raise IoError(where + ".primitives: expected an array")
    for i, p in enumerate(prims):
        pw = f"{where}.primitives[{i}]"
        kind = _field_as(p, "kind", "string", pw)
        if kind == "sphere":
            scene.primitives.append(SpherePrim(_vec3_from(_field(p, "center", pw), pw + ".center"),
                                               _field_as(p, "radius", "double", pw)))
        elif kind == "box":
            quat, t = _pose_from(_field(p, "pose", pw), pw + ".pose")
            scene.primitives.append(BoxPrim(quat, t, _vec3_from(_field(p, "half_extents", pw),
                                                                pw + ".half_extents")))
        elif kind == "capsule":
            scene.primitives.append(CapsulePrim(_vec3_from(_field(p, "a", pw), pw + ".a"),
                                                _vec3_from(_field(p, "b", pw), pw + ".b"),
                                                _field_as(p, "radius", "double", pw)))
        else:
            raise IoError(f"{pw}.kind: unknown primitive kind '{kind}'")
    try:
        scene_validate(scene)
    except ValueError as e:
        raise IoError(f"{where}: {e}") from None
    return scene


def _sampler_from(s: str, where: str) -> int:
    """sampler_from (model_io.cpp:218-222)."""
    if s == "halton":
        return SamplerKind.Halton
    if s == "uniform":
        return SamplerKind.Uniform
    raise IoError(f"{where}: unknown sampler '{s}'")


_PATCH_KINDS = {"delta": "double", "n_cc": "int", "workers": "unsigned", "max_iters_per_worker": "uint64",
                "tree_capacity": "uint64", "dd_radius": "double", "dynamic_domain": "bool",
                "balance": "bool", "early_exit": "bool", "two_stage": "bool", "batched_cc": "bool",
                "nn_partitions": "unsigned", "seed": "uint64"}


def _params_patch_from(j, where: str) -> ParamsPatch:
    """params_patch_from (model_io.cpp:224-245)."""
    p = ParamsPatch()
    if not isinstance(j, dict):
        return p
    for name in _PATCH_FIELDS:
        if name not in j:
            continue
        if name == "sampler":
            p.sampler = _sampler_from(_as(j[name], "string"), where + ".sampler")
        else:
            setattr(p, name, _as(j[name], _PATCH_KINDS[name]))
    return p


def _params_patch_to(p: ParamsPatch) -> dict:
    """params_patch_to (model_io.cpp:247-264)."""
    out = {}
    for name in _PATCH_FIELDS:
        v = getattr(p, name)
        if v is None:
            continue
        if name == "sampler":
            out[name] = sampler_to_string(v)
        elif _PATCH_KINDS[name] == "double":
            out[name] = float(v)
        elif _PATCH_KINDS[name] == "bool":
            out[name] = bool(v)
        else:
            out[name] = int(v)
    return out


def _params_to(p: PlannerParams) -> dict:
    """params_to (model_io.cpp:266-281)."""
    return {"delta": float(p.delta), "n_cc": int(p.n_cc), "workers": int(p.workers),
            "max_iters_per_worker": int(p.max_iters_per_worker), "tree_capacity": int(p.tree_capacity),
            "dd_radius": float(p.dd_radius), "dynamic_domain": bool(p.dynamic_domain),
            "balance": bool(p.balance), "early_exit": bool(p.early_exit), "two_stage": bool(p.two_stage),
            "batched_cc": bool(p.batched_cc), "nn_partitions": int(p.nn_partitions),
            "sampler": sampler_to_string(p.sampler), "seed": int(p.seed)}


def _params_from(j, where: str) -> PlannerParams:
    """params_from (model_io.cpp:283-288)."""
    return _params_patch_from(j, where).apply(PlannerParams())


def load_problem(path) -> ProblemSpec:
    """load_problem (model_io.cpp:292-315): also loads the referenced robot
    and checks start/goal against its dof."""
    path = Path(path)
    j = _parse_file(path)
    where = str(path)
    pr = ProblemSpec()
    pr.name = _value(j, "name", path.stem, "string")
    pr.robot = _field_as(j, "robot", "string", where)
    pr.scene = _field_as(j, "scene", "string", where)
    pr.start = _config_from(_field(j, "start", where), where + ".start")
    pr.goal = _config_from(_field(j, "goal", where), where + ".goal")
    if isinstance(j, dict) and "params" in j:
        pr.params = _params_patch_from(j["params"], where + ".params")
    robot = load_robot(path.parent / pr.robot)
    if len(pr.start) != robot.dof:
        raise IoError(f"{where}.start: dimension {len(pr.start)} does not match robot dof {robot.dof}")
    if len(pr.goal) != robot.dof:
        raise IoError(f"{where}.goal: dimension {len(pr.goal)} does not match robot dof {robot.dof}")
    return pr


def _bitwise_equal(a, b) -> bool:
    """bitwise_equal (types.hpp:23-29)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def load_path_file(path) -> PathFile:
    """load_path_file (model_io.cpp:317-342)."""
    path = Path(path)
    j = _parse_file(path)
    where = str(path)
    f = PathFile()
    f.robot = _field_as(j, "robot", "string", where)
    f.scene = _field_as(j, "scene", "string", where)
    cj = _field(j, "path", where)
    if not isinstance(cj, list) or not cj:
        raise IoError(where + ".path: expected a non-empty array of configurations")
    f.configs = [_config_from(c, f"{where}.path[{i}]") for i, c in enumerate(cj)]
    for i in range(1, len(f.configs)):
        if _bitwise_equal(f.configs[i - 1], f.configs[i]):
            raise IoError(f"{where}.path[{i}]: duplicates the previous waypoint")
    if isinstance(j, dict) and "metadata" in j:
        m = j["metadata"]
        f.cost = _value(m, "cost", 0.0, "double")
        f.timestamp = _value(m, "timestamp", "", "string")
        if isinstance(m, dict) and "params" in m:
            f.params = _params_from(m["params"], where + ".metadata.params")
    return f


# ---------------------------------------------------------------------------
# writers (model_io.cpp:344-421)
# ---------------------------------------------------------------------------

_KIND_NAME = {REVOLUTE: "revolute", PRISMATIC: "prismatic", FIXED: "fixed"}


def robot_to_json(model: RobotModel) -> dict:
    joints = []
    for jt in model.joints:
        d = {"kind": _KIND_NAME[jt.kind], "parent": int(jt.parent),
             "origin": _pose_to(jt.origin_quat, jt.origin_xyz)}
        if jt.kind != FIXED:
            d["axis"] = _vec3_to(jt.axis)
            d["limits"] = [float(jt.lo), float(jt.hi)]
        joints.append(d)
    spheres = [{"coarse": _sphere_to(ls.coarse), "fine": [_sphere_to(f) for f in ls.fine]}
               for ls in model.spheres]
    return {"name": model.name, "joints": joints, "spheres": spheres,
            "self_pairs": [[int(a), int(b)] for a, b in model.self_pairs]}


def write_robot(path, model: RobotModel) -> None:
    """write_robot (model_io.cpp:344-370)."""
    _write_file(Path(path), robot_to_json(model))


def scene_to_json(scene: Scene) -> dict:
    prims = []
    for p in scene.primitives:
        if isinstance(p, SpherePrim):
            prims.append({"kind": "sphere", "center": _vec3_to(p.center), "radius": float(p.radius)})
        elif isinstance(p, CapsulePrim):
            prims.append({"kind": "capsule", "a": _vec3_to(p.a), "b": _vec3_to(p.b),
                          "radius": float(p.radius)})
        elif not isinstance(p, BoxPrim):
            raise IoError(f"scene '{scene.name}': the reference scene format has no "
                          f"{type(p).__name__} primitive (geometry.hpp:35)")
        else:
            prims.append({"kind": "box", "pose": _pose_to(p.quat, p.translation),
                          "half_extents": _vec3_to(p.half_extents)})
    return {"name": scene.name, "primitives": prims}


def write_scene(path, scene: Scene) -> None:
    """write_scene (model_io.cpp:372-391)."""
    _write_file(Path(path), scene_to_json(scene))


def write_problem(path, problem: ProblemSpec) -> None:
    """write_problem (model_io.cpp:393-402)."""
    j = {"name": problem.name, "robot": problem.robot, "scene": problem.scene,
         "start": [float(x) for x in problem.start], "goal": [float(x) for x in problem.goal]}
    params = _params_patch_to(problem.params)
    if params:
        j["params"] = params
    _write_file(Path(path), j)


def write_path(path, pf: PathFile) -> None:
    """write_path (model_io.cpp:404-421)."""
    if len(pf.configs) == 0:
        raise IoError(f"{path}: path must contain at least one waypoint")
    for i in range(1, len(pf.configs)):
        if _bitwise_equal(pf.configs[i - 1], pf.configs[i]):
            raise IoError(f"{path}.path[{i}]: duplicates the previous waypoint")
    _write_file(Path(path), {
        "robot": pf.robot, "scene": pf.scene,
        "path": [[float(x) for x in q] for q in pf.configs],
        "metadata": {"cost": float(pf.cost), "params": _params_to(pf.params), "timestamp": pf.timestamp},
    })


# ---------------------------------------------------------------------------
# CSVs (model_io.cpp:423-465)
# ---------------------------------------------------------------------------

def _format_double(v: float) -> str:
    """format_double (model_io.cpp:425-429): %.17g."""
    return "%.17g" % v


def _format_ms(v: float) -> str:
    """format_ms (model_io.cpp:431-435): %.3f."""
    return "%.3f" % v


def results_csv_string(rows: Sequence[BenchRecord]) -> str:
    """results_csv_string (model_io.cpp:439-449)."""
    out = ["problem,status,time_ms,cost,iterations,sphere_tests,workers,seed\n"]
    for r in rows:
        cost = _format_double(r.cost) if int(r.status) == PlanStatus.Solved else ""
        out.append(f"{r.problem},{status_to_string(r.status)},{_format_ms(r.time_ms)},{cost},"
                   f"{int(r.iterations)},{int(r.sphere_tests)},{int(r.workers)},{int(r.seed)}\n")
    return "".join(out)


def write_results_csv(path, rows: Sequence[BenchRecord]) -> None:
    """write_results_csv (model_io.cpp:451-455)."""
    try:
        with open(path, "w", newline="") as f:
            f.write(results_csv_string(rows))
    except OSError:
        raise IoError(f"{path}: cannot open file for writing") from None


def write_ecdf_csv(path, points) -> None:
    """write_ecdf_csv (model_io.cpp:457-465)."""
    try:
        with open(path, "w", newline="") as f:
            f.write("value,fraction_solved\n")
            for v, frac in points:
                f.write(f"{_format_double(v)},{_format_double(frac)}\n")
    except OSError:
        raise IoError(f"{path}: cannot open file for writing") from None
