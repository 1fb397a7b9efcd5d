"""Host-side mirror of the reference's planning types.

Same names, fields, defaults and meaning as the reference C++ types so code
written against the reference reads the same here:

  Joint / Sphere / LinkSpheres / RobotModel   robot.hpp:12-71
  SpherePrim / BoxPrim / CapsulePrim / Scene  geometry.hpp:13-46
  PlannerParams                               planner.hpp:21-40
  PlanResult / PlanStatus                     planner.hpp:15, 42-51

Each model type flattens itself into the C-ABI descriptors of
include/prrtc_b200.h (``to_desc``). Validation happens in the library
(prrtc_robot_create / prrtc_scene_create mirror RobotModel::finalize and
Scene::validate) and surfaces as ValueError, the Python analogue of the
reference's std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

REVOLUTE, PRISMATIC, FIXED = 0, 1, 2


class PlanStatus(IntEnum):
    Solved = 0
    Failed = 1
    InfeasibleEndpoint = 2


class SamplerKind(IntEnum):
    Halton = 0
    Uniform = 1


def quat_from_rpy(roll: float, pitch: float, yaw: float) -> tuple[float, float, float, float]:
    """URDF fixed-axis rpy -> unit quaternion (w, x, y, z), R = Rz(yaw) Ry(pitch) Rx(roll)."""
    cr, sr = math.cos(roll / 2), math.sin(roll / 2)
    cp, sp = math.cos(pitch / 2), math.sin(pitch / 2)
    cy, sy = math.cos(yaw / 2), math.sin(yaw / 2)
    return (cr * cp * cy + sr * sp * sy,
            sr * cp * cy - cr * sp * sy,
            cr * sp * cy + sr * cp * sy,
            cr * cp * sy - sr * sp * cy)


def quat_to_mat3(q) -> np.ndarray:
    """Quat::to_mat3 (transform.hpp:97-103), raw (unnormalised) quaternion."""
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


@dataclass
class Joint:  # robot.hpp:17-26
    kind: int = REVOLUTE
    parent: int = -1
    origin_quat: tuple = (1.0, 0.0, 0.0, 0.0)  # w, x, y, z
    origin_xyz: tuple = (0.0, 0.0, 0.0)
    axis: tuple = (0.0, 0.0, 1.0)
    lo: float = 0.0
    hi: float = 0.0


@dataclass
class Sphere:  # robot.hpp:28-33
    center: tuple
    radius: float


@dataclass
class LinkSpheres:  # robot.hpp:37-42
    coarse: Sphere
    fine: list = field(default_factory=list)


@dataclass
class RobotModel:  # robot.hpp:44-71
    name: str
    joints: list
    spheres: list
    self_pairs: list = field(default_factory=list)
    # model-specific metadata for scene/problem generation (not in the reference)
    home: tuple = ()
    ee_links: tuple = ()

    @property
    def dof(self) -> int:
        return sum(1 for j in self.joints if j.kind != FIXED)

    def link_count(self) -> int:
        return len(self.joints)

    def limits(self) -> np.ndarray:
        """RobotModel::limits (robot.hpp:57-64): [dof, 2] (lo, hi)."""
        return np.array([[j.lo, j.hi] for j in self.joints if j.kind != FIXED], dtype=np.float64)

    def fine_count(self) -> int:
        return sum(len(ls.fine) for ls in self.spheres)

    def to_desc(self):
        """Flatten into prrtc_robot_desc; returns (desc, keepalive)."""
        from ._lib import RobotDesc
        n = len(self.joints)
        keep = {}

        def arr(name, ctype, values):
            a = (ctype * max(1, len(values)))(*values)
            keep[name] = a
            return a

        offs = [0]
        fine = []
        for ls in self.spheres:
            for f in ls.fine:
                fine += [*f.center, f.radius]
            offs.append(offs[-1] + len(ls.fine))
        d = RobotDesc()
        d.n_links = n
        d.kind = arr("kind", C.c_int32, [j.kind for j in self.joints])
        d.parent = arr("parent", C.c_int32, [j.parent for j in self.joints])
        d.origin_quat = arr("oq", C.c_double, [v for j in self.joints for v in j.origin_quat])
        d.origin_xyz = arr("ox", C.c_double, [v for j in self.joints for v in j.origin_xyz])
        d.axis = arr("axis", C.c_double, [v for j in self.joints for v in j.axis])
        d.lo = arr("lo", C.c_double, [j.lo for j in self.joints])
        d.hi = arr("hi", C.c_double, [j.hi for j in self.joints])
        d.coarse = arr("coarse", C.c_double, [v for ls in self.spheres for v in (*ls.coarse.center, ls.coarse.radius)])
        d.fine_offset = arr("foff", C.c_uint32, offs)
        d.fine = arr("fine", C.c_double, fine)
        d.n_self_pairs = len(self.self_pairs)
        d.self_pairs = arr("pairs", C.c_int32, [v for p in self.self_pairs for v in p])
        return d, keep


@dataclass
class SpherePrim:  # geometry.hpp:13-18
    center: tuple
    radius: float


@dataclass
class BoxPrim:  # geometry.hpp:20-25 (pose = quaternion w,x,y,z + translation)
    quat: tuple
    translation: tuple
    half_extents: tuple


@dataclass
class CapsulePrim:  # geometry.hpp:27-33
    a: tuple
    b: tuple
    radius: float


@dataclass
class CylinderPrim:
    """Extension (BASELINE config 4): a solid cylinder about the local z axis
    of its pose. The reference has no cylinder primitive (geometry.hpp:35);
    verdicts are pinned to the C restatement (oracle/prrtc_oracle.c)."""
    quat: tuple
    translation: tuple
    radius: float
    half_length: float


@dataclass
class Scene:  # geometry.hpp:37-46
    name: str
    primitives: list = field(default_factory=list)

    def grouped(self):
        s = [p for p in self.primitives if isinstance(p, SpherePrim)]
        b = [p for p in self.primitives if isinstance(p, BoxPrim)]
        c = [p for p in self.primitives if isinstance(p, CapsulePrim)]
        return s, b, c

    def cylinders(self) -> list:
        return [p for p in self.primitives if isinstance(p, CylinderPrim)]

    def ordered(self) -> list:
        """Primitive order used by every per-primitive output: spheres, boxes,
        capsules, then cylinders."""
        s, b, c = self.grouped()
        return s + b + c + self.cylinders()

    def to_desc(self):
        from ._lib import SceneDesc
        s, b, c = self.grouped()
        y = self.cylinders()
        keep = {}
        sv = [v for p in s for v in (*p.center, p.radius)]
        bv = [v for p in b for v in (*p.quat, *p.translation, *p.half_extents)]
        cv = [v for p in c for v in (*p.a, *p.b, p.radius)]
        yv = [v for p in y for v in (*p.quat, *p.translation, p.radius, p.half_length)]
        d = SceneDesc()
        d.n_spheres, d.n_boxes, d.n_capsules, d.n_cylinders = len(s), len(b), len(c), len(y)
        keep["s"] = (C.c_double * max(1, len(sv)))(*sv)
        keep["b"] = (C.c_double * max(1, len(bv)))(*bv)
        keep["c"] = (C.c_double * max(1, len(cv)))(*cv)
        keep["y"] = (C.c_double * max(1, len(yv)))(*yv)
        d.spheres, d.boxes, d.capsules, d.cylinders = keep["s"], keep["b"], keep["c"], keep["y"]
        return d, keep


@dataclass
class PlannerParams:  # planner.hpp:21-40 (+ device knobs)
    delta: float = 0.5
    n_cc: int = 32
    workers: int = 0
    max_iters_per_worker: int = 2000
    tree_capacity: int = 200000
    dd_radius: float = 0.0
    dynamic_domain: bool = True
    balance: bool = True
    early_exit: bool = True
    two_stage: bool = True
    batched_cc: bool = False
    nn_partitions: int = 1
    sampler: int = SamplerKind.Halton
    seed: int = 0
    # device knobs
    threads_per_cta: int = 0
    ctas_per_sm: int = 0
    deterministic: bool = False
    validate_path: bool = False  # device re-validation of returned paths
    max_workers_per_problem: int = 0  # batches: 0 = elastic help; 1 with workers=1 = the reference's search

    def resolved_dd_radius(self) -> float:
        return self.dd_radius if self.dd_radius > 0.0 else 4.0 * self.delta

    def to_c(self):
        from ._lib import Params
        p = Params()
        p.delta = self.delta
        p.n_cc = self.n_cc
        p.workers = self.workers
        p.max_iters_per_worker = self.max_iters_per_worker
        p.tree_capacity = self.tree_capacity
        p.dd_radius = self.dd_radius
        p.dynamic_domain = int(self.dynamic_domain)
        p.balance = int(self.balance)
        p.early_exit = int(self.early_exit)
        p.two_stage = int(self.two_stage)
        p.batched_cc = int(self.batched_cc)
        p.nn_partitions = self.nn_partitions
        p.sampler = int(self.sampler)
        p.seed = self.seed
        p.threads_per_cta = self.threads_per_cta
        p.ctas_per_sm = self.ctas_per_sm
        p.deterministic = int(self.deterministic)
        p.validate_path = int(self.validate_path)
        p.max_workers_per_problem = self.max_workers_per_problem
        return p


@dataclass
class CheckStatsSnapshot:  # collision.hpp:27-31
    sphere_tests: int = 0
    fk_calls: int = 0
    fine_stage_entries: int = 0


@dataclass
class PlanResult:  # planner.hpp:42-51
    status: PlanStatus = PlanStatus.Failed
    path: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))
    cost: float = 0.0
    wall_time_ms: float = 0.0
    iterations_total: int = 0
    check_stats: CheckStatsSnapshot = field(default_factory=CheckStatsSnapshot)
    solving_worker: int = -1
    message: str = ""
    device_time_ms: float = 0.0
    tree_nodes: tuple = (0, 0)
    flops: int = 0
    path_check: int = 0  # validate_path: 0 not checked, 1 valid, 2 invalid
