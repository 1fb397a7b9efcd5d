"""Synthetic robot models: Panda 7-DoF, Fetch 8-DoF, Baxter 14-DoF.

The reference ships no robot models (proj/.gitignore excludes examples/), so
these are authored here: joint origins/axes/limits follow the
public URDFs (franka_description, fetch_description, baxter_description);
collision spheres are placed along each link's body segments (sphere chains,
spacing <= 0.8 r) with the coarse sphere the tight bounding sphere of the fine
ones (+1e-6 m), so RobotModel::finalize's containment invariant
(kinematics.cpp:56-57) holds with margin. Self-collision pairs are the
non-adjacent link pairs that are free at the home pose, collide in some but at
most 30% of 6000 uniformly sampled configurations (so never-colliding and
structurally overlapping pairs are pruned); derived offline
with the reference FK and hard-coded here.
"""
from __future__ import annotations

import math

import numpy as np

from .model import FIXED, PRISMATIC, REVOLUTE, Joint, LinkSpheres, RobotModel, Sphere, quat_from_rpy

PI = math.pi


def sphere_chain(segments) -> list[Sphere]:
    """segments: [(p0, p1, r)] in the link frame -> evenly spaced spheres."""
    out = []
    for p0, p1, r in segments:
        p0 = np.asarray(p0, float)
        p1 = np.asarray(p1, float)
        length = float(np.linalg.norm(p1 - p0))
        n = max(1, int(math.ceil(length / (0.8 * r)))) + 1 if length > 0 else 1
        for k in range(n):
            t = k / (n - 1) if n > 1 else 0.0
            c = p0 + t * (p1 - p0)
            out.append(Sphere(tuple(round(float(v), 6) for v in c), float(r)))
    return out


def bounding(fine: list[Sphere]) -> Sphere:
    """Coarse sphere: center = midpoint of the fine-sphere AABB, radius = max reach + 1e-6."""
    if not fine:
        return Sphere((0.0, 0.0, 0.0), 1e-3)
    c = np.array([f.center for f in fine])
    r = np.array([f.radius for f in fine])
    center = 0.5 * ((c - r[:, None]).min(0) + (c + r[:, None]).max(0))
    reach = float(np.max(np.linalg.norm(c - center, axis=1) + r))
    return Sphere(tuple(float(v) for v in center), reach + 1e-6)


def _link(segments) -> LinkSpheres:
    fine = sphere_chain(segments)
    return LinkSpheres(bounding(fine), fine)


def _j(kind, parent, xyz, rpy=(0.0, 0.0, 0.0), axis=(0.0, 0.0, 1.0), lo=0.0, hi=0.0) -> Joint:
    return Joint(kind, parent, quat_from_rpy(*rpy), tuple(float(v) for v in xyz), axis, lo, hi)


# ---------------------------------------------------------------------------
# Franka Emika Panda (franka_description panda_arm.xacro)
# ---------------------------------------------------------------------------
def panda() -> RobotModel:
    J = [
        _j(FIXED, -1, (0, 0, 0)),                                                   # 0 link0
        _j(REVOLUTE, 0, (0, 0, 0.333), lo=-2.8973, hi=2.8973),                      # 1 link1
        _j(REVOLUTE, 1, (0, 0, 0), (-PI / 2, 0, 0), lo=-1.7628, hi=1.7628),         # 2 link2
        _j(REVOLUTE, 2, (0, -0.316, 0), (PI / 2, 0, 0), lo=-2.8973, hi=2.8973),     # 3 link3
        _j(REVOLUTE, 3, (0.0825, 0, 0), (PI / 2, 0, 0), lo=-3.0718, hi=-0.0698),    # 4 link4
        _j(REVOLUTE, 4, (-0.0825, 0.384, 0), (-PI / 2, 0, 0), lo=-2.8973, hi=2.8973),  # 5 link5
        _j(REVOLUTE, 5, (0, 0, 0), (PI / 2, 0, 0), lo=-0.0175, hi=3.7525),          # 6 link6
        _j(REVOLUTE, 6, (0.088, 0, 0), (PI / 2, 0, 0), lo=-2.8973, hi=2.8973),      # 7 link7
        _j(FIXED, 7, (0, 0, 0.107), (0, 0, -PI / 4)),                               # 8 hand
    ]
    S = [
        _link([((-0.04, 0, 0.05), (0.0, 0, 0.14), 0.08)]),
        _link([((0, 0, -0.19), (0, 0, -0.02), 0.075)]),
        _link([((0, -0.02, 0), (0, -0.24, 0), 0.072)]),
        _link([((0, 0, -0.15), (0, 0, -0.03), 0.065), ((0.045, 0, 0), (0.0825, 0, 0), 0.06)]),
        _link([((0, 0, 0), (-0.055, 0.09, 0), 0.065)]),
        _link([((0, 0, -0.26), (0, 0, -0.07), 0.06), ((0, 0.075, -0.22), (0, 0.075, -0.12), 0.045)]),
        _link([((0, 0, -0.02), (0.088, 0, 0), 0.055)]),
        _link([((0, 0, 0.0), (0, 0, 0.075), 0.05)]),
        _link([((0, -0.075, 0.04), (0, 0.075, 0.04), 0.033), ((0, -0.035, 0.095), (0, 0.035, 0.095), 0.018)]),
    ]
    pairs = [(0, 5), (0, 6), (0, 7), (0, 8), (1, 5), (1, 6), (1, 7), (1, 8), (2, 5), (2, 7),
             (2, 8), (3, 5), (3, 8), (5, 7), (5, 8)]
    return RobotModel("panda", J, S, pairs,
                      home=(0.0, -0.785, 0.0, -2.356, 0.0, 1.571, 0.785), ee_links=(8,))


# ---------------------------------------------------------------------------
# Fetch (fetch_description fetch.urdf): prismatic torso + 7-DoF arm
# ---------------------------------------------------------------------------
def fetch() -> RobotModel:
    X, Y = (1.0, 0.0, 0.0), (0.0, 1.0, 0.0)
    J = [
        _j(FIXED, -1, (0, 0, 0)),                                                   # 0 base
        _j(PRISMATIC, 0, (-0.086875, 0, 0.37743), lo=0.0, hi=0.38615),              # 1 torso
        _j(FIXED, 1, (0.053125, 0, 0.603001)),                                      # 2 head
        _j(REVOLUTE, 1, (0.119525, 0, 0.34858), lo=-1.6056, hi=1.6056),             # 3 shoulder_pan
        _j(REVOLUTE, 3, (0.117, 0, 0.06), axis=Y, lo=-1.221, hi=1.518),             # 4 shoulder_lift
        _j(REVOLUTE, 4, (0.219, 0, 0), axis=X, lo=-PI, hi=PI),                      # 5 upperarm_roll
        _j(REVOLUTE, 5, (0.133, 0, 0), axis=Y, lo=-2.251, hi=2.251),                # 6 elbow_flex
        _j(REVOLUTE, 6, (0.197, 0, 0), axis=X, lo=-PI, hi=PI),                      # 7 forearm_roll
        _j(REVOLUTE, 7, (0.1245, 0, 0), axis=Y, lo=-2.16, hi=2.16),                 # 8 wrist_flex
        _j(REVOLUTE, 8, (0.1385, 0, 0), axis=X, lo=-PI, hi=PI),                     # 9 wrist_roll
        _j(FIXED, 9, (0.16645, 0, 0)),                                              # 10 gripper
    ]
    S = [
        _link([((-0.12, -0.12, 0.18), (0.12, -0.12, 0.18), 0.15), ((-0.12, 0.12, 0.18), (0.12, 0.12, 0.18), 0.15)]),
        _link([((-0.07, 0, 0.05), (-0.07, 0, 0.55), 0.12)]),
        _link([((0.02, 0, 0.08), (0.12, 0, 0.08), 0.12)]),
        _link([((0.0, 0, 0.0), (0.1, 0, 0.05), 0.07)]),
        _link([((0.0, 0, 0.0), (0.13, 0, 0.0), 0.066)]),
        _link([((0.0, 0, 0.0), (0.12, 0, 0.0), 0.062)]),
        _link([((0.0, 0, 0.0), (0.15, 0, 0.0), 0.06)]),
        _link([((0.0, 0, 0.0), (0.1, 0, 0.0), 0.056)]),
        _link([((0.0, 0, 0.0), (0.1, 0, 0.0), 0.055)]),
        _link([((0.0, 0, 0.0), (0.05, 0, 0.0), 0.05)]),
        _link([((-0.09, -0.06, 0), (-0.09, 0.06, 0), 0.045), ((-0.02, -0.05, 0), (-0.02, 0.05, 0), 0.025)]),
    ]
    pairs = [(0, 6), (0, 7), (0, 8), (0, 9), (0, 10), (1, 6), (1, 7), (1, 8), (1, 9), (1, 10),
             (2, 5), (2, 6), (2, 7), (2, 8), (2, 9), (2, 10), (3, 8), (3, 9), (3, 10), (4, 9),
             (4, 10), (5, 10)]
    return RobotModel("fetch", J, S, pairs,
                      home=(0.2, 1.32, 1.4, -0.2, 1.72, 0.0, 1.66, 0.0), ee_links=(10,))


# ---------------------------------------------------------------------------
# Rethink Baxter (baxter_description): two 7-DoF arms as one forest
# ---------------------------------------------------------------------------
def _baxter_arm(sign: float, first: int) -> tuple[list, list]:
    mount = np.array([0.024645, sign * 0.219645, 0.118588])
    yaw = sign * PI / 4
    s0 = mount + np.array([math.cos(yaw) * 0.055695, math.sin(yaw) * 0.055695, 0.011038])
    J = [
        _j(REVOLUTE, 0, tuple(s0), (0, 0, yaw), lo=-1.7016, hi=1.7016),                     # s0
        _j(REVOLUTE, first, (0.069, 0, 0.27035), (-PI / 2, 0, 0), lo=-2.147, hi=1.047),     # s1
        _j(REVOLUTE, first + 1, (0.102, 0, 0), (PI / 2, 0, PI / 2), lo=-3.0541, hi=3.0541),  # e0
        _j(REVOLUTE, first + 2, (0.069, 0, 0.26242), (-PI / 2, -PI / 2, 0), lo=-0.05, hi=2.618),  # e1
        _j(REVOLUTE, first + 3, (0.10359, 0, 0), (PI / 2, 0, PI / 2), lo=-3.059, hi=3.059),  # w0
        _j(REVOLUTE, first + 4, (0.01, 0, 0.2707), (-PI / 2, -PI / 2, 0), lo=-1.5707, hi=2.094),  # w1
        _j(REVOLUTE, first + 5, (0.115975, 0, 0), (PI / 2, 0, PI / 2), lo=-3.059, hi=3.059),  # w2
        _j(FIXED, first + 6, (0, 0, 0.11355)),                                               # hand
    ]
    S = [
        _link([((0, 0, 0.05), (0.04, 0, 0.22), 0.09)]),
        _link([((0, 0, 0), (0.09, 0, 0), 0.08)]),
        _link([((0, 0, 0.03), (0.04, 0, 0.22), 0.072)]),
        _link([((0, 0, 0), (0.095, 0, 0), 0.068)]),
        _link([((0, 0, 0.03), (0.01, 0, 0.23), 0.062)]),
        _link([((0, 0, 0), (0.1, 0, 0), 0.058)]),
        _link([((0, 0, 0.0), (0, 0, 0.09), 0.052)]),
        _link([((0, -0.05, 0.04), (0, 0.05, 0.04), 0.04), ((0, -0.03, 0.1), (0, 0.03, 0.1), 0.02)]),
    ]
    return J, S


def baxter() -> RobotModel:
    J = [_j(FIXED, -1, (0, 0, 0))]
    S = [_link([((-0.06, 0, -0.55), (-0.06, 0, 0.2), 0.17), ((0.02, 0, 0.45), (0.02, 0, 0.6), 0.12)])]
    jl, sl = _baxter_arm(+1.0, 1)
    jr, sr = _baxter_arm(-1.0, 9)
    J += jl + jr
    S += sl + sr
    pairs = [(0, 2), (0, 3), (0, 4), (0, 5), (0, 6), (0, 7), (0, 8), (0, 10), (0, 11), (0, 12),
             (0, 13), (0, 14), (0, 15), (0, 16), (1, 3), (1, 4), (1, 5), (1, 6), (1, 7), (1, 8),
             (1, 12), (1, 13), (1, 14), (1, 15), (1, 16), (2, 7), (2, 8), (2, 11), (2, 12),
             (2, 13), (2, 14), (2, 15), (2, 16), (3, 5), (3, 10), (3, 11), (3, 12), (3, 13),
             (3, 14), (3, 15), (3, 16), (4, 9), (4, 10), (4, 11), (4, 12), (4, 13), (4, 14),
             (4, 15), (4, 16), (5, 7), (5, 9), (5, 10), (5, 11), (5, 12), (5, 13), (5, 14),
             (5, 15), (5, 16), (6, 9), (6, 10), (6, 11), (6, 12), (6, 13), (6, 14), (6, 15),
             (6, 16), (7, 9), (7, 10), (7, 11), (7, 12), (7, 13), (7, 14), (7, 15), (7, 16),
             (8, 9), (8, 10), (8, 11), (8, 12), (8, 13), (8, 14), (8, 15), (8, 16), (9, 11),
             (9, 13), (9, 14), (9, 15), (9, 16), (10, 15), (10, 16), (11, 13), (11, 15),
             (11, 16), (13, 15)]
    home = (0.3, -0.55, 0.0, 1.2, 0.0, 0.9, 0.0, -0.3, -0.55, 0.0, 1.2, 0.0, 0.9, 0.0)
    return RobotModel("baxter", J, S, pairs, home=home, ee_links=(8, 16))


ROBOTS = {"panda": panda, "fetch": fetch, "baxter": baxter}


def get(name: str) -> RobotModel:
    return ROBOTS[name]()
