"""Generates tests/golden/golden_ref.npz from the COMPILED REFERENCE (oracle/_ref)
— TEST INFRASTRUCTURE.

    python tests/golden/make_golden.py

The reference ships no golden vectors or fixtures (proj/CMakeLists.txt:6,
proj/.gitignore:1-2), so these are produced by running the unmodified
reference sources (oracle/Makefile) with the scalar backend forced
(kernels.hpp:107-110). They pin the C restatement (oracle/prrtc_oracle.c) on
machines where /root/reference is absent (tests/test_oracle_port.py).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import Oracle  # noqa: E402
from paper_2503_06757_b200 import robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402

ROBOTS = ["panda", "fetch", "baxter"]
KINDS = ["table_pick", "bookshelf", "cage"]


def configs(m, n, seed):
    lim = m.limits()
    rng = np.random.default_rng(seed)
    return lim[:, 0] + rng.random((n, m.dof)) * (lim[:, 1] - lim[:, 0])


def build(o: Oracle) -> dict:
    out = {}
    rng = np.random.default_rng(123)
    bases = np.array(o.halton_bases(16), dtype=np.uint32)
    hb = np.repeat(bases, 40)
    hi = np.concatenate([np.arange(0, 320), rng.integers(0, 2**44, len(hb) - 320)]).astype(np.uint64)
    out["halton_base"], out["halton_index"] = hb, hi
    out["halton_value"] = np.array([o.halton_value(int(b), int(i)) for b, i in zip(hb, hi)])
    for r in ROBOTS:
        m = robots.get(r)
        out[f"{r}_sample"] = o.sample_config(m, 1, 3, 60)
        Q = configs(m, 40, 1)
        out[f"{r}_fk_q"] = Q
        out[f"{r}_fk_poses"] = np.stack([o.fk_poses(m, q) for q in Q])
        out[f"{r}_fk_fine"] = np.stack([o.fk_spheres(m, q, True) for q in Q])
        out[f"{r}_fk_coarse"] = np.stack([o.fk_spheres(m, q, False) for q in Q])
        Qc = configs(m, 60, 2)
        out[f"{r}_cc_q"] = Qc
        res, stats = [], []
        for k in KINDS:
            sc, _ = make_scene(r, k, 7)
            for ts in (0, 1):
                for ee in (0, 1):
                    for q in Qc:
                        v, st = o.check_config(m, sc, q, ts, ee, stats=True)
                        res.append(v)
                        stats.append(st)
        out[f"{r}_cc_valid"] = np.array(res)
        out[f"{r}_cc_stats"] = np.array(stats)
        lim = m.limits()
        E0 = configs(m, 40, 3)
        E1 = np.clip(E0 + rng.normal(size=E0.shape) * 0.25, lim[:, 0], lim[:, 1])
        E1[0] = E0[0]
        out[f"{r}_edge_from"], out[f"{r}_edge_to"] = E0, E1
        sc, _ = make_scene(r, "cage", 9)
        out[f"{r}_edge_valid"] = o.validate_edges(m, sc, E0, E1, 32)
        vb, st = o.validate_edge_batched(m, sc, E0, E1, 32)
        out[f"{r}_edge_batched"], out[f"{r}_edge_batched_stats"] = vb, st
        # planner, workers = 1 (deterministic, planner.cpp:295-296)
        d = np.load(ROOT / "tests" / "golden" / f"problems_{r}.npz")
        st_, it_, cost_, paths, lens, stats_ = [], [], [], [], [], []
        for i in range(8):
            sc, _ = make_scene(r, str(d["kind"][i]), int(d["pid"][i]))
            res = o.plan(m, sc, d["start"][i], d["goal"][i], PlannerParams(workers=1, tree_capacity=20000))
            st_.append(int(res.status))
            it_.append(res.iterations_total)
            cost_.append(res.cost)
            paths.append(res.path.reshape(-1, m.dof))
            lens.append(len(res.path))
            cs = res.check_stats
            stats_.append([cs.sphere_tests, cs.fk_calls, cs.fine_stage_entries])
        out[f"{r}_plan_status"] = np.array(st_)
        out[f"{r}_plan_iters"] = np.array(it_)
        out[f"{r}_plan_cost"] = np.array(cost_)
        out[f"{r}_plan_len"] = np.array(lens)
        out[f"{r}_plan_path"] = np.concatenate(paths) if paths else np.zeros((0, m.dof))
        out[f"{r}_plan_stats"] = np.array(stats_)
        out[f"{r}_plan_start"] = d["start"][:8]
        out[f"{r}_plan_goal"] = d["goal"][:8]
        out[f"{r}_plan_kind"] = d["kind"][:8]
        out[f"{r}_plan_pid"] = d["pid"][:8]
    tree = rng.uniform(-3, 3, (700, 7))
    tree[350] = tree[10]
    q = rng.uniform(-3, 3, (30, 7))
    q[0] = tree[10]
    out["nn_tree"], out["nn_q"] = tree, q
    out["nn_index"] = np.array([o.nearest_serial(tree, x)[0] for x in q])
    out["nn_dist"] = np.array([o.nearest_serial(tree, x)[1] for x in q])
    out["nn_par_index"] = np.array([o.nearest_parallel(tree, x, 7)[0] for x in q])
    return out


def main():
    o = Oracle("ref")
    o.force_scalar(True)
    out = build(o)
    path = ROOT / "tests" / "golden" / "golden_ref.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size // 1024} KiB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
