"""Dynamic-obstacle replanning loop (BASELINE config 5).

Each frame moves the dynamic obstacles, pushes the new primitive set into the
resident device scene (prrtc_scene_update: one small H2D, no reallocation)
and plans again from the current start (prrtc_plan) — the per-frame work of
the paper's real-time replanning demo minus perception. The
scene is the static part plus `moving` spheres that translate by `step`
metres per frame.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import planner
from .model import PlannerParams, PlanResult, Scene, SpherePrim


@dataclass
class FrameResult:
    frame: int
    wall_ms: float          # scene update + plan, host wall clock
    result: PlanResult
    scene: Scene


@dataclass
class MovingSpheres:
    """`n` spheres on parallel tracks, moving `step` m per frame along `direction`."""
    origin: tuple = (0.45, -0.45, 0.45)
    direction: tuple = (0.0, 1.0, 0.0)
    spacing: tuple = (0.0, 0.0, 0.12)
    radius: float = 0.05
    n: int = 3
    step: float = 0.01

    def at(self, frame: int) -> list:
        o, d, s = (np.asarray(v, dtype=np.float64) for v in (self.origin, self.direction, self.spacing))
        return [SpherePrim(tuple(o + s * k + d * self.step * frame), self.radius) for k in range(self.n)]


def scene_at(static: Scene, obstacles: MovingSpheres, frame: int) -> Scene:
    return Scene(f"{static.name}_frame{frame}", list(static.primitives) + obstacles.at(frame))


def run(model, static: Scene, start, goal, frames: int = 100, obstacles: MovingSpheres | None = None,
        params: PlannerParams | None = None, device: int = 0) -> list[FrameResult]:
    """The replanning loop: per frame prrtc_scene_update + prrtc_plan."""
    obstacles = obstacles or MovingSpheres()
    params = params or PlannerParams()
    rob = planner.device_robot(model, device)
    dscene = planner.DeviceScene(scene_at(static, obstacles, 0), device)
    out = []
    for f in range(frames):
        sc = scene_at(static, obstacles, f)
        t0 = time.perf_counter()
        dscene.update(sc)
        r = planner.plan(rob, dscene, start, goal, params, device=device)
        out.append(FrameResult(f, (time.perf_counter() - t0) * 1e3, r, sc))
    return out
