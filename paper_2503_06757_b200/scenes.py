"""Synthetic MotionBenchMaker-shaped scenes.

The reference bundles no scenes (proj/.gitignore excludes examples/) and MBM
itself is an external dataset, so the three archetypes the paper evaluates on
(Fig. 3) are generated procedurally, deterministically from
(robot, kind, problem id):

  table_pick  table + 4..12 objects (boxes, upright cylinders as capsules,
              spheres); goal: end effector above one object
  bookshelf   side/back boards + 3..5 shelves; goal: end effector in a cell
  cage        a cube of 8..12 bars (capsules) on a table; goal: inside it

Per-problem jitter: +-5 cm position and +-15 deg yaw of the whole scene about
its anchor, from numpy's PCG64 seeded with 1000 + problem_id. Primitives are
spheres, oriented boxes and capsules only — the reference has no cylinder
primitive (geometry.hpp:35), so cylinders are expressed as capsules (a
conservative superset) and stay oracle-checkable.

Each scene also returns goal regions (axis-aligned boxes, world frame), one
per end-effector link of the robot, used by the problem generator.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .model import BoxPrim, CapsulePrim, CylinderPrim, Scene, SpherePrim

KINDS = ("table_pick", "bookshelf", "cage")


@dataclass
class GoalRegion:
    center: np.ndarray
    half: np.ndarray

    def contains(self, p) -> bool:
        return bool(np.all(np.abs(np.asarray(p) - self.center) <= self.half))


@dataclass
class Frame:
    """Where the archetype sits relative to the robot base."""
    offset: tuple  # added to every coordinate
    yscale: float  # lateral spread (dual-arm robots)
    arms: int      # goal regions to emit


FRAMES = {
    "panda": Frame((0.0, 0.0, 0.0), 1.0, 1),
    "fetch": Frame((0.2, 0.0, 0.72), 1.0, 1),
    "baxter": Frame((0.05, 0.0, 0.3), 1.7, 2),
}


def _yaw_quat(yaw: float):
    return (math.cos(yaw / 2), 0.0, 0.0, math.sin(yaw / 2))


def _qmul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return (aw * bw - ax * bx - ay * by - az * bz,
            aw * bx + ax * bw + ay * bz - az * by,
            aw * by - ax * bz + ay * bw + az * bx,
            aw * bz + ax * by - ay * bx + az * bw)


class _Builder:
    def __init__(self, frame: Frame, anchor, rng):
        self.f = frame
        self.prims = []
        self.anchor = np.asarray(anchor, float)
        self.yaw = float(rng.uniform(-math.radians(15), math.radians(15)))
        self.shift = np.array([rng.uniform(-0.05, 0.05), rng.uniform(-0.05, 0.05), 0.0])
        c, s = math.cos(self.yaw), math.sin(self.yaw)
        self.R = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]])

    def P(self, p) -> tuple:
        """archetype coordinates -> world (scale, jitter about the anchor, robot offset)."""
        p = np.array(p, float)
        p[1] *= self.f.yscale
        w = self.anchor + self.R @ (p - self.anchor) + self.shift + np.asarray(self.f.offset)
        return tuple(float(round(v, 9)) for v in w)

    def box(self, center, half):
        h = (half[0], half[1] * (self.f.yscale if half[1] > 0.2 else 1.0), half[2])
        self.prims.append(BoxPrim(_yaw_quat(self.yaw), self.P(center), tuple(float(v) for v in h)))

    def capsule(self, a, b, r):
        self.prims.append(CapsulePrim(self.P(a), self.P(b), float(r)))

    def sphere(self, c, r):
        self.prims.append(SpherePrim(self.P(c), float(r)))

    def region(self, center, half) -> GoalRegion:
        # regions stay axis-aligned in the world; shrink by the yaw-induced spread
        return GoalRegion(np.array(self.P(center)), np.asarray(half, float))


def _objects(b: _Builder, rng, n, xr, yr, z0):
    tops = []
    for _ in range(n):
        x, y = rng.uniform(*xr), rng.uniform(*yr)
        kind = rng.integers(3)
        if kind == 0:
            hx, hy, hz = rng.uniform(0.02, 0.05), rng.uniform(0.02, 0.05), rng.uniform(0.03, 0.08)
            b.box((x, y, z0 + hz), (hx, hy, hz))
            tops.append((x, y, z0 + 2 * hz))
        elif kind == 1:  # upright cylinder as a capsule
            r, h = rng.uniform(0.02, 0.04), rng.uniform(0.08, 0.2)
            b.capsule((x, y, z0 + r), (x, y, z0 + h - r), r)
            tops.append((x, y, z0 + h))
        else:
            r = rng.uniform(0.03, 0.06)
            b.sphere((x, y, z0 + r), r)
            tops.append((x, y, z0 + 2 * r))
    return tops


def table_pick(frame: Frame, rng):
    b = _Builder(frame, (0.6, 0.0, 0.0), rng)
    b.box((0.68, 0.0, -0.04), (0.3, 0.6, 0.04))
    tops = _objects(b, rng, int(rng.integers(4, 13)), (0.42, 0.85), (-0.42, 0.42), 0.0)
    regions = []
    order = sorted(range(len(tops)), key=lambda i: tops[i][1], reverse=True)
    picks = [order[0], order[-1]] if frame.arms == 2 else [int(rng.integers(len(tops)))]
    for i in picks[: frame.arms]:
        x, y, zt = tops[i]
        regions.append(b.region((x, y, zt + 0.13), (0.04, 0.04, 0.04)))
    return b.prims, regions


def bookshelf(frame: Frame, rng):
    b = _Builder(frame, (0.75, 0.0, 0.45), rng)
    depth, x0 = 0.15, 0.77
    n = int(rng.integers(3, 6))
    zs = np.sort(np.concatenate([[-0.05], rng.uniform(0.12, 0.85, n - 2), [1.0]]))
    # enforce >= 0.24 m clear cells
    for k in range(1, len(zs)):
        zs[k] = max(zs[k], zs[k - 1] + 0.26)
    for z in zs:
        b.box((x0, 0.0, z), (depth, 0.47, 0.01))
    top = float(zs[-1])
    b.box((x0, -0.47, (top - 0.05) / 2), (depth, 0.01, (top + 0.05) / 2 + 0.01))
    b.box((x0, 0.47, (top - 0.05) / 2), (depth, 0.01, (top + 0.05) / 2 + 0.01))
    b.box((x0 + depth + 0.01, 0.0, (top - 0.05) / 2), (0.01, 0.48, (top + 0.05) / 2 + 0.01))
    if frame.arms == 2:
        b.box((x0, 0.0, (top - 0.05) / 2), (depth, 0.01, (top + 0.05) / 2))  # divider
    cells = [(zs[k], zs[k + 1]) for k in range(len(zs) - 1) if 0.05 <= zs[k] + 0.1 <= 0.75]
    if not cells:
        cells = [(zs[0], zs[1])]
    lo, hi = cells[int(rng.integers(len(cells)))]
    zc = 0.5 * (lo + hi)
    hz = max(0.02, 0.5 * (hi - lo) - 0.1)
    regions = []
    ys = [0.22, -0.22] if frame.arms == 2 else [float(rng.uniform(-0.2, 0.2))]
    for y in ys:
        regions.append(b.region((x0 - 0.06, y, zc), (0.06, 0.12, hz)))
    if frame.arms == 2:  # clutter: upright cylinders on the shelves
        for _ in range(int(rng.integers(2, 6))):
            k = int(rng.integers(len(zs) - 1))
            r = rng.uniform(0.02, 0.035)
            x, y = rng.uniform(x0 + 0.02, x0 + 0.12), rng.uniform(-0.4, 0.4)
            b.capsule((x, y, zs[k] + 0.01 + r), (x, y, zs[k] + min(0.18, zs[k + 1] - zs[k] - 0.05)), r)
    return b.prims, regions


def cage(frame: Frame, rng):
    c = np.array([0.52, 0.0, 0.3])
    b = _Builder(frame, c, rng)
    b.box((0.55, 0.0, -0.04), (0.32, 0.55, 0.04))
    h = 0.19
    corners = [c + h * np.array([sx, sy, sz]) for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)]
    edges = []
    for i in range(8):
        for j in range(i + 1, 8):
            if np.sum(np.abs(corners[i] - corners[j]) > 1e-9) == 1:
                edges.append((i, j))
    drop = set(rng.choice(len(edges), size=int(rng.integers(0, 5)), replace=False).tolist())
    for e, (i, j) in enumerate(edges):
        if e not in drop:
            b.capsule(corners[i], corners[j], 0.012)
    regions = []
    if frame.arms == 2:
        regions.append(b.region(c + np.array([0.0, 0.06, 0.0]), (0.06, 0.04, 0.07)))
        regions.append(b.region(c + np.array([0.0, -0.06, 0.0]), (0.06, 0.04, 0.07)))
    else:
        regions.append(b.region(c, (0.07, 0.07, 0.07)))
    return b.prims, regions


GENERATORS = {"table_pick": table_pick, "bookshelf": bookshelf, "cage": cage}


def make_scene(robot: str, kind: str, problem_id: int, cylinders: bool = False) -> tuple[Scene, list[GoalRegion]]:
    """cylinders=True: the upright objects become true solid cylinders (the
    primitive extension, BASELINE config 4) instead of capsules."""
    rng = np.random.default_rng(1000 + int(problem_id))
    prims, regions = GENERATORS[kind](FRAMES[robot], rng)
    if cylinders:
        prims = [as_cylinder(p) for p in prims]
    return Scene(f"{robot}_{kind}_{problem_id}" + ("_cyl" if cylinders else ""), prims), regions


def as_cylinder(p):
    """An upright capsule (a, b share x, y) -> the solid cylinder spanning the
    same height (its caps' extent) with the same radius; other primitives
    unchanged."""
    if not isinstance(p, CapsulePrim) or p.a[0] != p.b[0] or p.a[1] != p.b[1]:
        return p
    lo, hi = min(p.a[2], p.b[2]) - p.radius, max(p.a[2], p.b[2]) + p.radius
    return CylinderPrim((1.0, 0.0, 0.0, 0.0), (p.a[0], p.a[1], 0.5 * (lo + hi)), p.radius, 0.5 * (hi - lo))


def kind_for(problem_id: int, n_problems: int) -> str:
    """1000 problems split 334/333/333 over table_pick/bookshelf/cage."""
    per = [(n_problems + 2) // 3, (n_problems + 1) // 3]
    if problem_id < per[0]:
        return "table_pick"
    if problem_id < per[0] + per[1]:
        return "bookshelf"
    return "cage"
