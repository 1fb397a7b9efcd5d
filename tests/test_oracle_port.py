"""CPU: the oracle itself is pinned before it is trusted.

* the C restatement (oracle/liboracle.so) reproduces the golden vectors that
  the compiled reference produced (tests/golden/golden_ref.npz) bit for bit;
* the compiled reference, when present, still reproduces them;
* the SPEC known-answer examples hold.
"""
import math
from pathlib import Path

import numpy as np
import pytest

from paper_2503_06757_b200 import robots
from paper_2503_06757_b200.model import (FIXED, REVOLUTE, BoxPrim, CapsulePrim, Joint, LinkSpheres,
                                         PlannerParams, RobotModel, Scene, Sphere, SpherePrim)
from paper_2503_06757_b200.scenes import make_scene

GOLD = Path(__file__).resolve().parent / "golden" / "golden_ref.npz"
KINDS = ["table_pick", "bookshelf", "cage"]


def oracles():
    from oracle import Oracle, available
    out = [Oracle("port")]
    if available("ref"):
        o = Oracle("ref")
        o.force_scalar(True)
        out.append(o)
    return out


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("kind", ["port", "ref"])
def test_golden_vectors(gold, kind):
    from oracle import Oracle, available
    if kind == "ref" and not available("ref"):
        pytest.skip("reference build not present")
    o = Oracle(kind)
    o.force_scalar(True)
    hv = np.array([o.halton_value(int(b), int(i)) for b, i in zip(gold["halton_base"], gold["halton_index"])])
    assert np.array_equal(hv, gold["halton_value"])
    for r in ["panda", "fetch", "baxter"]:
        m = robots.get(r)
        assert np.array_equal(o.sample_config(m, 1, 3, 60), gold[f"{r}_sample"])
        Q = gold[f"{r}_fk_q"]
        assert np.array_equal(np.stack([o.fk_poses(m, q) for q in Q]), gold[f"{r}_fk_poses"])
        assert np.array_equal(np.stack([o.fk_spheres(m, q, True) for q in Q]), gold[f"{r}_fk_fine"])
        assert np.array_equal(np.stack([o.fk_spheres(m, q, False) for q in Q]), gold[f"{r}_fk_coarse"])
        res, stats = [], []
        for k in KINDS:
            sc, _ = make_scene(r, k, 7)
            for ts in (0, 1):
                for ee in (0, 1):
                    for q in gold[f"{r}_cc_q"]:
                        v, st = o.check_config(m, sc, q, ts, ee, stats=True)
                        res.append(v)
                        stats.append(st)
        assert np.array_equal(np.array(res), gold[f"{r}_cc_valid"])
        assert np.array_equal(np.array(stats), gold[f"{r}_cc_stats"])
        sc, _ = make_scene(r, "cage", 9)
        E0, E1 = gold[f"{r}_edge_from"], gold[f"{r}_edge_to"]
        assert np.array_equal(o.validate_edges(m, sc, E0, E1, 32), gold[f"{r}_edge_valid"])
        vb, st = o.validate_edge_batched(m, sc, E0, E1, 32)
        assert np.array_equal(vb, gold[f"{r}_edge_batched"])
        assert np.array_equal(st, gold[f"{r}_edge_batched_stats"])
        off = 0
        for i in range(len(gold[f"{r}_plan_status"])):
            sc, _ = make_scene(r, str(gold[f"{r}_plan_kind"][i]), int(gold[f"{r}_plan_pid"][i]))
            res = o.plan(m, sc, gold[f"{r}_plan_start"][i], gold[f"{r}_plan_goal"][i],
                         PlannerParams(workers=1, tree_capacity=20000))
            n = int(gold[f"{r}_plan_len"][i])
            assert int(res.status) == gold[f"{r}_plan_status"][i]
            assert res.iterations_total == gold[f"{r}_plan_iters"][i]
            assert res.cost == gold[f"{r}_plan_cost"][i]
            cs = res.check_stats
            assert [cs.sphere_tests, cs.fk_calls, cs.fine_stage_entries] == list(gold[f"{r}_plan_stats"][i])
            assert np.array_equal(res.path.reshape(-1, m.dof), gold[f"{r}_plan_path"][off:off + n])
            off += n
    tree, q = gold["nn_tree"], gold["nn_q"]
    assert [o.nearest_serial(tree, x)[0] for x in q] == list(gold["nn_index"])
    assert np.array_equal([o.nearest_serial(tree, x)[1] for x in q], gold["nn_dist"])
    assert [o.nearest_parallel(tree, x, 7)[0] for x in q] == list(gold["nn_par_index"])


def planar2():
    """planar 2-link, revolute z axes, origins +1 m along x."""
    J = [Joint(REVOLUTE, -1, (1, 0, 0, 0), (0, 0, 0), (0, 0, 1), -4, 4),
         Joint(REVOLUTE, 0, (1, 0, 0, 0), (1, 0, 0), (0, 0, 1), -4, 4),
         Joint(FIXED, 1, (1, 0, 0, 0), (1, 0, 0))]
    S = [LinkSpheres(Sphere((0, 0, 0), 0.1), [Sphere((0, 0, 0), 0.05)]) for _ in J]
    return RobotModel("planar2", J, S, [])


@pytest.mark.parametrize("o", oracles(), ids=lambda o: o.kind)
def test_spec_known_answers(o):
    # Halton
    assert [o.halton_value(2, i) for i in (1, 2, 3, 4)] == [0.5, 0.25, 0.75, 0.125]
    assert o.halton_value(3, 1) == 1 / 3 and o.halton_value(2, 0) == 0.0
    # FK planar closed form: tip at (0, 2, 0)
    P = o.fk_poses(planar2(), np.array([math.pi / 2, 0.0]))
    assert np.allclose(P[2, 9:], [0, 2, 0], atol=1e-9)
    # sphere (3,0,0) r=1 vs unit box: clearance 1 -> free; inside -> hit
    sc = Scene("box", [BoxPrim((1, 0, 0, 0), (0, 0, 0), (1, 1, 1))])
    assert not o.sphere_hits(sc, 3, 0, 0, 1)[0]
    assert not o.sphere_hits(sc, 2, 0, 0, 1)[0]      # touching is free
    assert o.sphere_hits(sc, 0.2, 0.1, 0, 0.05)[0]
    # capsule tangency free, 1e-6 closer hit
    cap = Scene("cap", [CapsulePrim((0, 0, 0), (0, 0, 1), 0.5)])
    assert not o.sphere_hits(cap, 1.5, 0, 0.5, 1.0)[0]
    assert o.sphere_hits(cap, 1.5 - 1e-6, 0, 0.5, 1.0)[0]
    sp = Scene("sp", [SpherePrim((0, 0, 0), 1.0)])
    assert not o.sphere_hits(sp, 2, 0, 0, 1)[0] and o.sphere_hits(sp, 2 - 1e-9, 0, 0, 1)[0]
    # NN tie-break: distances (2, 1, 1) -> index 1
    tree = np.array([[2.0, 0.0], [1.0, 0.0], [-1.0, 0.0]])
    assert o.nearest_serial(tree, np.zeros(2)) == (1, 1.0)
    assert o.nearest_parallel(tree, np.zeros(2), 3)[0] == 1
    # empty scene, no pairs -> always free
    m = robots.get("panda")
    assert o.check_config(m, Scene("e", []), np.array(m.home))
    # engulfing primitive -> never free
    assert not o.check_config(m, Scene("big", [SpherePrim((0, 0, 0), 100.0)]), np.array(m.home))


@pytest.mark.parametrize("o", oracles(), ids=lambda o: o.kind)
def test_plan_degenerate_cases(o):
    m = robots.get("panda")
    sc = Scene("e", [])
    home = np.array(m.home)
    r = o.plan(m, sc, home, home, PlannerParams(workers=1, tree_capacity=2000))
    assert r.status == 0 and r.path.shape == (1, 7) and r.cost == 0.0
    bad = home.copy()
    bad[0] = 9.0
    r = o.plan(m, sc, bad, home, PlannerParams(workers=1, tree_capacity=2000))
    assert r.status == 2 and "start" in r.message
    with pytest.raises(ValueError, match="delta"):
        o.plan(m, sc, home, home, PlannerParams(delta=0.0))
