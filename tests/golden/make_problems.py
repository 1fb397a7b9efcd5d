"""Generates the committed planning-problem fixtures (TEST/BENCH INFRASTRUCTURE).

    python tests/golden/make_problems.py [robot ...] [--n N] [--set K]

--set K (K >= 1) writes problems_<robot>_s<K>.npz: another N problems with
problem ids from K * 100000 (disjoint scenes, starts and goals), the shard of
rank K in the multi-GPU weak-scaling bench (rank 0 uses problems_<robot>.npz).

For every problem id p: the scene is make_scene(robot, kind_for(p, N), p)
(deterministic, so only start/goal are stored). Start = the robot's home pose
+ U(-0.2, 0.2) rad jitter, collision-free; goal = a uniformly sampled
configuration whose end-effector frame origin(s) lie in the scene's goal
region(s), collision-free — both checked by the reference oracle
(oracle/_ref: CollisionChecker::check_config, forward_kinematics). No IK is
needed. Output: tests/golden/problems_<robot>.npz.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import Oracle  # noqa: E402
from paper_2503_06757_b200 import robots  # noqa: E402
from paper_2503_06757_b200.model import quat_to_mat3  # noqa: E402
from paper_2503_06757_b200.scenes import kind_for, make_scene  # noqa: E402

DEFAULT_N = {"panda": 1000, "fetch": 1000, "baxter": 1000}


def arm_joints(model, ee_link):
    """Actuated-joint slots on the chain root -> ee_link."""
    qidx, k = {}, 0
    for i, j in enumerate(model.joints):
        if j.kind != 2:
            qidx[i] = k
            k += 1
    out, l = [], ee_link
    while l >= 0:
        if l in qidx:
            out.append(qidx[l])
        l = model.joints[l].parent
    return sorted(out)


def fk_positions(model, Q):
    """Batched FK (link-frame origins) in numpy, the reference's formulas
    (kinematics.cpp:78-103, transform.hpp:56-80). Only used to pre-filter
    goal candidates by end-effector position; the oracle re-checks."""
    n, L = Q.shape[0], model.link_count()
    R = np.zeros((L, n, 3, 3))
    T = np.zeros((L, n, 3))
    k = 0
    for i, j in enumerate(model.joints):
        Ro = quat_to_mat3(j.origin_quat)
        to = np.array(j.origin_xyz)
        if j.kind == 0:
            q = Q[:, k]
            k += 1
            ax, ay, az = j.axis
            c, s = np.cos(q), np.sin(q)
            t = 1 - c
            Rm = np.stack([np.stack([t * ax * ax + c, t * ax * ay - s * az, t * ax * az + s * ay], -1),
                           np.stack([t * ax * ay + s * az, t * ay * ay + c, t * ay * az - s * ax], -1),
                           np.stack([t * ax * az - s * ay, t * ay * az + s * ax, t * az * az + c], -1)], -2)
            Rl, tl = Ro @ Rm, np.broadcast_to(to, (n, 3))
        elif j.kind == 1:
            q = Q[:, k]
            k += 1
            Rl = np.broadcast_to(Ro, (n, 3, 3))
            tl = to + (Ro @ np.array(j.axis))[None] * q[:, None]
        else:
            Rl, tl = np.broadcast_to(Ro, (n, 3, 3)), np.broadcast_to(to, (n, 3))
        if j.parent < 0:
            R[i], T[i] = Rl, tl
        else:
            R[i] = R[j.parent] @ Rl
            T[i] = np.einsum("nij,nj->ni", R[j.parent], tl) + T[j.parent]
    return T


def sample_goal(o, model, scene, regions, rng, batch=40000, rounds=25):
    lim = model.limits()
    home = np.array(model.home)
    arms = [arm_joints(model, l) for l in model.ee_links]
    cands = []
    for arm, ee, reg in zip(arms, model.ee_links, regions):
        found = []
        for _ in range(rounds):
            Q = np.tile(home, (batch, 1))
            Q[:, arm] = lim[arm, 0] + rng.random((batch, len(arm))) * (lim[arm, 1] - lim[arm, 0])
            P = fk_positions(model, Q)[ee]
            inside = np.all(np.abs(P - reg.center) <= reg.half, axis=1)
            found.extend(Q[inside][:, arm])
            if len(found) >= 64:
                break
        if not found:
            return None
        cands.append(np.array(found))
    for _ in range(200):
        q = home.copy()
        for arm, c in zip(arms, cands):
            q[arm] = c[rng.integers(len(c))]
        if o.check_config(model, scene, q, two_stage=False, early_exit=True):
            return q
    return None


def sample_start(o, model, scene, rng):
    lim = model.limits()
    home = np.array(model.home)
    for _ in range(2000):
        q = np.clip(home + rng.uniform(-0.2, 0.2, model.dof), lim[:, 0], lim[:, 1])
        if o.check_config(model, scene, q, two_stage=False, early_exit=True):
            return q
    return None


def generate(robot: str, n: int, o: Oracle, p0: int = 0):
    model = robots.get(robot)
    starts, goals, kinds, pids = [], [], [], []
    t0 = time.time()
    p = p0
    while len(pids) < n:
        kind = kind_for(len(pids), n)
        scene, regions = make_scene(robot, kind, p)
        rng = np.random.default_rng(7_000_000 + p)
        s = sample_start(o, model, scene, rng)
        g = sample_goal(o, model, scene, regions, rng) if s is not None else None
        if s is not None and g is not None:
            starts.append(s)
            goals.append(g)
            kinds.append(kind)
            pids.append(p)
        p += 1
        if (p - p0) % 100 == 0:
            print(f"{robot}: {len(pids)}/{p} problems, {time.time() - t0:.1f}s", flush=True)
    return (np.array(kinds), np.array(pids, dtype=np.int64), np.array(starts), np.array(goals))


def main(argv):
    n_override = None
    set_k = 0
    if "--set" in argv:
        i = argv.index("--set")
        set_k = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    if "--n" in argv:
        i = argv.index("--n")
        n_override = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    names = argv or list(DEFAULT_N)
    o = Oracle("ref")
    for r in names:
        n = n_override or DEFAULT_N[r]
        kinds, pids, S, G = generate(r, n, o, p0=100000 * set_k)
        out = Path(__file__).resolve().parent / (f"problems_{r}_s{set_k}.npz" if set_k else f"problems_{r}.npz")
        np.savez_compressed(out, kind=kinds, pid=pids, start=S, goal=G, n=n)
        print(f"wrote {out}: {len(pids)} problems (ids up to {pids.max()})")


if __name__ == "__main__":
    main(sys.argv[1:])
