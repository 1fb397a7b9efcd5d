"""Parity of the sm_100a hot-path pieces against the CPU oracle.

Bars (BASELINE.json north_star):
  * FK sphere centres within 1e-5 m of the reference FK;
  * collision verdicts bit-exact on identical collision-sphere sets (the
    device's posed spheres fed to the reference predicate
    sphere_vs_primitive, geometry.cpp:41-66);
  * NN index exact with ties to the lowest index, squared distance bitwise
    equal to the scalar backend (kernels_scalar.cpp:9-37);
  * Halton values / samples bit-exact (sampling.cpp:8-51).
"""
import numpy as np
import pytest

from conftest import load_problems
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.scenes import make_scene

pytestmark = pytest.mark.gpu

ROBOTS = ["panda", "fetch", "baxter"]


def random_configs(model, n, seed):
    lim = model.limits()
    rng = np.random.default_rng(seed)
    return lim[:, 0] + rng.random((n, model.dof)) * (lim[:, 1] - lim[:, 0])


def fine_radii(model):
    return np.array([f.radius for ls in model.spheres for f in ls.fine])


def link_of_fine(model):
    return np.concatenate([[l] * len(ls.fine) for l, ls in enumerate(model.spheres)]).astype(int)


@pytest.mark.parametrize("robot", ROBOTS)
def test_fk_sphere_centres_within_1e5(gpu, oracle, robot):
    m = robots.get(robot)
    Q = random_configs(m, 1000, 1)
    fine, coarse = planner.debug_fk(m, Q)
    err = 0.0
    for i in range(0, len(Q), 7):
        ref = oracle.fk_spheres(m, Q[i], fine=True)
        err = max(err, np.abs(fine[i].astype(np.float64) - ref[:, :3]).max())
        refc = oracle.fk_spheres(m, Q[i], fine=False)
        err = max(err, np.abs(coarse[i].astype(np.float64) - refc[:, :3]).max())
    assert err < 1e-5, err


def oracle_brute_on_spheres(oracle, model, scene, centers):
    """check_config_brute (collision.cpp:100-128) evaluated by the reference
    predicates on the device's posed sphere set."""
    r = fine_radii(model)
    link = link_of_fine(model)
    env = any(oracle.sphere_hits(scene, *map(float, centers[j]), r[j]).any() for j in range(len(r)))
    if env:
        return False
    for a, b in model.self_pairs:
        ia, ib = np.where(link == a)[0], np.where(link == b)[0]
        for i in ia:
            for j in ib:
                pa, pb = centers[i].astype(np.float64), centers[j].astype(np.float64)
                dx, dy, dz = pa[0] - pb[0], pa[1] - pb[1], pa[2] - pb[2]
                d2 = dx * dx + dy * dy + dz * dz  # kernels_detail.hpp:17-23, same order
                rr = r[i] + r[j]
                if d2 < rr * rr:
                    return False
    return True


@pytest.mark.parametrize("robot", ROBOTS)
def test_predicates_bitexact_on_device_spheres(gpu, oracle, robot):
    m = robots.get(robot)
    scene, _ = make_scene(robot, "cage", 3)
    Q = random_configs(m, 64, 2)
    fine, _ = planner.debug_fk(m, Q)
    X = fine.reshape(-1, 3)
    R = np.tile(fine_radii(m), len(Q))
    dev = planner.debug_sphere_hits(scene, X, R)
    ref = np.array([oracle.sphere_hits(scene, *map(float, X[i]), R[i]) for i in range(len(X))])
    assert dev.shape == ref.shape
    assert np.array_equal(dev, ref)


@pytest.mark.parametrize("kind", ["table_pick", "bookshelf", "cage"])
def test_predicates_bitexact_near_boundary(gpu, oracle, kind):
    """Spheres placed within +-2e-5 m of tangency to every primitive: the
    guard band must route them to the exact FP64 path."""
    scene, _ = make_scene("panda", kind, 11)
    rng = np.random.default_rng(5)
    pts, rad = [], []
    for p in scene.ordered():
        for _ in range(40):
            r = float(rng.uniform(0.02, 0.08))
            off = float(rng.uniform(-2e-5, 2e-5))
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            if hasattr(p, "half_extents"):
                from paper_2503_06757_b200.model import quat_to_mat3
                Rb = quat_to_mat3(p.quat)
                h = np.array(p.half_extents)
                local = np.clip(d * 2.0, -h, h)  # a surface point
                out = d / np.linalg.norm(d)
                c = np.array(p.translation) + Rb @ (local + out * (r + off))
            elif hasattr(p, "a"):
                a, b = np.array(p.a), np.array(p.b)
                t = rng.uniform(0, 1)
                n = np.cross(b - a, d)
                n /= np.linalg.norm(n)
                c = a + t * (b - a) + n * (p.radius + r + off)
            else:
                c = np.array(p.center) + d * (p.radius + r + off)
            pts.append(c)
            rad.append(r)
    X = np.array(pts, dtype=np.float32)
    R = np.array(rad)
    dev = planner.debug_sphere_hits(scene, X, R)
    ref = np.array([oracle.sphere_hits(scene, *map(float, X[i]), R[i]) for i in range(len(X))])
    assert np.array_equal(dev, ref)


@pytest.mark.parametrize("robot", ROBOTS)
def test_check_configs_bitexact_on_device_spheres(gpu, oracle, robot):
    m = robots.get(robot)
    for kind, seed in [("table_pick", 1), ("bookshelf", 2), ("cage", 3)]:
        scene, _ = make_scene(robot, kind, seed)
        Q = random_configs(m, 96, seed)
        fine, _ = planner.debug_fk(m, Q)
        two = planner.check_configs(m, scene, Q, two_stage=True)
        brute = planner.check_configs(m, scene, Q, two_stage=False)
        assert np.array_equal(two, brute)  # two-stage == fine-only
        ref = np.array([oracle_brute_on_spheres(oracle, m, scene, fine[i]) for i in range(len(Q))])
        assert np.array_equal(two, ref)
        # and against the reference's own FP64 FK (statistically identical)
        ref64 = oracle.check_configs(m, scene, Q, two_stage=True)
        assert np.mean(ref64 == two) >= 0.99


@pytest.mark.parametrize("robot", ROBOTS)
def test_validate_edges_matches_oracle(gpu, oracle, robot):
    m = robots.get(robot)
    probs = load_problems(robot, 30)
    rng = np.random.default_rng(9)
    for kind, pid, s, g in probs[::3]:
        scene, _ = make_scene(robot, kind, pid)
        lim = m.limits()
        frm = np.repeat(s[None], 64, 0)
        d = rng.normal(size=(64, m.dof))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        to = np.clip(frm + d * rng.uniform(0.05, 1.0, (64, 1)), lim[:, 0], lim[:, 1])
        to[0] = frm[0]  # bitwise-equal edge collapses to one check (collision.cpp:215)
        for two_stage in (True, False):
            for ee in (True, False):
                dev = planner.validate_edges(m, scene, frm, to, 32, two_stage, ee)
                if two_stage and ee:
                    base = dev
                assert np.array_equal(dev, base)  # options never change verdicts
        ref = oracle.validate_edges(m, scene, frm, to, 32)
        assert np.mean(ref == base) >= 0.98, (kind, pid)


def ref_state_verdicts(oracle, model, scene, fine):
    """Reference predicates (sphere_vs_primitive, geometry.cpp:41-66, and the
    self-pair sphere test, kernels_detail.hpp:17-23 in its FP64 operation
    order) on given posed fine spheres: fine [n, S, 3] -> valid [n]."""
    r = fine_radii(model)
    n, S = fine.shape[:2]
    X = np.concatenate([fine.reshape(-1, 3).astype(np.float64), np.tile(r, n)[:, None]], axis=1)
    env = oracle.sphere_any_hits(scene, X).reshape(n, S).any(axis=1)
    off = np.concatenate([[0], np.cumsum([len(ls.fine) for ls in model.spheres])])
    selfhit = np.zeros(n, dtype=bool)
    P = fine.astype(np.float64)
    for a, b in model.self_pairs:
        A, B = P[:, off[a]:off[a + 1]], P[:, off[b]:off[b + 1]]
        ra, rb = r[off[a]:off[a + 1]], r[off[b]:off[b + 1]]
        dx = A[:, :, None, 0] - B[:, None, :, 0]
        dy = A[:, :, None, 1] - B[:, None, :, 1]
        dz = A[:, :, None, 2] - B[:, None, :, 2]
        d2 = (dx * dx + dy * dy) + dz * dz
        rr = ra[:, None] + rb[None, :]
        selfhit |= (d2 < rr * rr).any(axis=(1, 2))
    return ~(env | selfhit)


@pytest.mark.parametrize("robot", ROBOTS)
def test_check_edges_bitexact_on_device_spheres(gpu, oracle, robot):
    """prrtc_debug_check_edges: every state's device verdict
    equals the reference predicates evaluated on the device's own posed
    spheres (bit-exact, two-stage and brute force), and the AND over an
    edge's states is prrtc_validate_edges' verdict."""
    m = robots.get(robot)
    rng = np.random.default_rng(17)
    lim = m.limits()
    for kind, pid, s, g in load_problems(robot, 1000)[::200]:
        scene, _ = make_scene(robot, kind, pid)
        frm = np.repeat(s[None], 24, 0)
        d = rng.normal(size=(24, m.dof))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        to = np.clip(frm + d * rng.uniform(0.1, 1.5, (24, 1)), lim[:, 0], lim[:, 1])
        to[0] = frm[0]
        for two_stage in (True, False):
            valid, fine = planner.debug_check_edges(m, scene, frm, to, 32, two_stage)
            ref = ref_state_verdicts(oracle, m, scene, fine.reshape(-1, fine.shape[2], 3)).reshape(valid.shape)
            assert np.array_equal(valid, ref), (kind, pid, two_stage, np.argwhere(valid != ref)[:5])
            edge = planner.validate_edges(m, scene, frm, to, 32, two_stage, True)
            assert np.array_equal(edge, valid.all(axis=1))
        assert (~valid).any() and valid.any()  # both outcomes exercised


def test_nn_exact_with_ties(gpu, oracle):
    rng = np.random.default_rng(3)
    for dof in (7, 8, 14):
        for count in (1, 2, 3, 31, 32, 33, 257, 1000, 4099):
            tree = rng.uniform(-3, 3, (count, dof))
            if count > 4:  # duplicates and equal-distance nodes
                tree[count // 2] = tree[1]
                tree[-1] = tree[1]
            q = rng.uniform(-3, 3, (8, dof))
            q[0] = tree[min(1, count - 1)]  # zero distance, first index wins
            q[1] = tree[count // 2]
            for group in (0, 1, 2, 3, 5, 8):  # one query per pass (0 = 1) and the planner's multi-sample passes
                idx, d2 = planner.debug_nn(tree, q, group=group)
                for i in range(len(q)):
                    ri, rd = oracle.nearest_serial(tree, q[i])
                    assert idx[i] == ri, (dof, count, i, group)
                    assert d2[i] == oracle.sq_distance(tree[ri], q[i])
    # near-ties below FP32 resolution: the FP32 filter must hand them to the
    # exact FP64 refinement (several candidates per thread included)
    for dof in (7, 14):
        q = rng.uniform(-2, 2, (32, dof))
        for count in (64, 1000, 5000):
            d = rng.normal(size=(count, dof))
            d /= np.linalg.norm(d, axis=1, keepdims=True)
            r = 0.7 + rng.integers(0, 3, count)[:, None] * 1e-12 + rng.uniform(0, 1e-9, (count, 1))
            tree = q[0] + d * r
            for group in (0, 16, 18, 32):
                idx, d2 = planner.debug_nn(tree, q, group=group)
                for i in range(len(q)):
                    ri, _ = oracle.nearest_serial(tree, q[i])
                    assert idx[i] == ri, (dof, count, i, group)
                    assert d2[i] == oracle.sq_distance(tree[ri], q[i])
    # distances (2, 1, 1) -> first distance-1 index
    tree = np.array([[2.0, 0.0], [1.0, 0.0], [-1.0, 0.0]])
    idx, _ = planner.debug_nn(tree, np.zeros((1, 2)))
    assert idx[0] == 1


def test_halton_bitexact(gpu, oracle):
    rng = np.random.default_rng(4)
    bases = np.array(oracle.halton_bases(14) * 200, dtype=np.uint32)
    idx = np.concatenate([np.arange(0, 700), rng.integers(0, 2**40, len(bases) - 700)]).astype(np.uint64)
    dev = planner.debug_halton(bases, idx)
    ref = np.array([oracle.halton_value(int(b), int(i)) for b, i in zip(bases, idx)])
    assert np.array_equal(dev, ref)
    assert list(planner.debug_halton([2, 2, 2, 2, 3], [1, 2, 3, 4, 1])) == [0.5, 0.25, 0.75, 0.125, 1 / 3]


@pytest.mark.parametrize("robot", ROBOTS)
def test_sample_config_bitexact(gpu, oracle, robot):
    m = robots.get(robot)
    dev = planner.debug_sample(m, 1, 500)
    ref = oracle.sample_config(m, 1, 1, 500)
    assert np.array_equal(dev, ref)
    lim = m.limits()
    assert np.all(dev >= lim[:, 0]) and np.all(dev < lim[:, 1])
