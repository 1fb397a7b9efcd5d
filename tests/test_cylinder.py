"""The cylinder primitive extension (BASELINE config 4 asks for
"cylinders+cuboids"; the reference has no cylinder, geometry.hpp:35).

Its verdicts cannot be pinned to the reference, so they are pinned twice:
the C restatement's FP64 predicate against an independent numpy distance
computation (CPU), and the device against the restatement — bit-exact
verdicts on the device's own posed spheres, two-stage == brute force, and
planned paths re-validated (GPU)."""
import numpy as np
import pytest

from conftest import ROOT
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.model import CylinderPrim, PlannerParams, PlanStatus, Scene, quat_from_rpy, quat_to_mat3
from paper_2503_06757_b200.scenes import make_scene


@pytest.fixture(scope="module")
def port():
    from oracle import Oracle
    o = Oracle("port")  # the compiled reference has no cylinder primitive
    return o


def _cyl_scene(rng, n=6):
    prims = []
    for _ in range(n):
        q = quat_from_rpy(*rng.uniform(-np.pi, np.pi, 3))
        prims.append(CylinderPrim(q, tuple(rng.uniform(-0.6, 0.6, 3)), float(rng.uniform(0.02, 0.2)),
                                  float(rng.uniform(0.02, 0.3))))
    return Scene("cylinders", prims)


def _np_distance(p, c: CylinderPrim):
    """Distance from point p to the solid cylinder (independent formulation:
    closest point by clamping in the cylinder frame)."""
    R = quat_to_mat3(c.quat)
    l = R.T @ (np.asarray(p) - np.asarray(c.translation))
    rho = np.hypot(l[0], l[1])
    q = l.copy()
    if rho > c.radius:
        q[:2] *= c.radius / rho
    q[2] = np.clip(l[2], -c.half_length, c.half_length)
    return np.linalg.norm(l - q)


def test_port_cylinder_predicate_matches_geometry(port):
    rng = np.random.default_rng(0)
    scene = _cyl_scene(rng)
    for _ in range(3000):
        p = rng.uniform(-1.0, 1.0, 3)
        r = float(rng.uniform(0.01, 0.15))
        hits = port.sphere_hits(scene, *p, r)
        for h, c in zip(hits, scene.ordered()):
            d = _np_distance(p, c)
            if abs(d - r) > 1e-9:  # away from tangency the verdicts must agree
                assert bool(h) == (d < r), (p, r, c, d)


def test_reference_rejects_cylinder_scenes():
    from oracle import Oracle, available
    if not available("ref"):
        pytest.skip("reference build absent")
    with pytest.raises(ValueError, match="no cylinder"):
        Oracle("ref").scene(_cyl_scene(np.random.default_rng(1), 1))


def test_cylinder_scene_validation():
    from paper_2503_06757_b200 import _lib
    from conftest import has_gpu
    if not has_gpu():
        pytest.skip("scene handles bind to a device")
    bad = Scene("bad", [CylinderPrim((1.0, 0, 0, 0), (0, 0, 0), 0.1, 0.0)])
    with pytest.raises(ValueError, match="half_length: must be positive"):
        planner.DeviceScene(bad)


@pytest.mark.gpu
def test_cylinder_verdicts_bitexact_on_device_spheres(gpu, port):
    rng = np.random.default_rng(2)
    scene = _cyl_scene(rng, 8)
    m = robots.get("panda")
    lim = m.limits()
    Q = rng.uniform(lim[:, 0], lim[:, 1], (64, m.dof))
    fine, _ = planner.debug_fk(m, Q)
    X = fine.reshape(-1, 3)
    R = np.tile(np.array([f.radius for ls in m.spheres for f in ls.fine]), len(Q))
    dev = planner.debug_sphere_hits(scene, X, R)
    ref = np.array([port.sphere_hits(scene, *map(float, X[i]), R[i]) for i in range(len(X))])
    assert np.array_equal(dev, ref)
    # near tangency: every sphere within +-2e-5 m of a cylinder's surface
    pts, rad = [], []
    for c in scene.ordered():
        Rc = quat_to_mat3(c.quat)
        for _ in range(60):
            r = float(rng.uniform(0.02, 0.08))
            off = float(rng.uniform(-2e-5, 2e-5))
            side = rng.integers(3)
            ang = rng.uniform(0, 2 * np.pi)
            if side == 0:  # mantle
                l = np.array([np.cos(ang) * (c.radius + r + off), np.sin(ang) * (c.radius + r + off),
                              rng.uniform(-c.half_length, c.half_length)])
            else:  # caps
                s = 1.0 if side == 1 else -1.0
                rr = rng.uniform(0, c.radius)
                l = np.array([np.cos(ang) * rr, np.sin(ang) * rr, s * (c.half_length + r + off)])
            pts.append(np.asarray(c.translation) + Rc @ l)
            rad.append(r)
    X = np.array(pts, dtype=np.float32)
    R = np.array(rad)
    dev = planner.debug_sphere_hits(scene, X, R)
    ref = np.array([port.sphere_hits(scene, *map(float, X[i]), R[i]) for i in range(len(X))])
    assert np.array_equal(dev, ref)


@pytest.mark.gpu
def test_cylinder_scene_checks_and_plans(gpu, port):
    """Two-stage == brute force on cylinder scenes, verdicts equal the
    restatement's on the device's spheres, and plans through table-top
    scenes whose upright objects are true cylinders re-validate."""
    m = robots.get("panda")
    d = np.load(ROOT / "tests" / "golden" / "problems_panda.npz")
    rng = np.random.default_rng(3)
    lim = m.limits()
    idx = [int(i) for i in np.where(d["kind"] == "table_pick")[0][:40]]
    solved = tried = 0
    for i in idx:
        scene, _ = make_scene("panda", "table_pick", int(d["pid"][i]), cylinders=True)
        if not any(isinstance(p, CylinderPrim) for p in scene.primitives) or tried >= 12:
            continue
        tried += 1
        Q = rng.uniform(lim[:, 0], lim[:, 1], (96, m.dof))
        two = planner.check_configs(m, scene, Q, two_stage=True)
        brute = planner.check_configs(m, scene, Q, two_stage=False)
        assert np.array_equal(two, brute)
        s, g = d["start"][i], d["goal"][i]
        if not (port.check_config(m, scene, s) and port.check_config(m, scene, g)):
            continue  # the cylinder variant may cover an endpoint
        r = planner.plan(m, scene, s, g, PlannerParams(tree_capacity=20000))
        if r.status == PlanStatus.Solved:
            solved += 1
            assert np.array_equal(r.path[0], s) and np.array_equal(r.path[-1], g)
            ok = port.validate_edges(m, scene, r.path[:-1], r.path[1:], 32, False, False)
            assert ok.all()
    assert solved >= 6
