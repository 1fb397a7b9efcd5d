"""CPU: the synthetic robots, scenes and committed problem fixtures are valid
inputs for the reference (checked with the oracle)."""
import importlib.util
from pathlib import Path

import numpy as np
import pytest

from conftest import load_problems
from paper_2503_06757_b200 import robots
from paper_2503_06757_b200.model import Scene
from paper_2503_06757_b200.scenes import KINDS, make_scene

ROOT = Path(__file__).resolve().parents[1]
ROBOTS = ["panda", "fetch", "baxter"]


def _make_problems_module():
    spec = importlib.util.spec_from_file_location("make_problems", ROOT / "tests" / "golden" / "make_problems.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("robot", ROBOTS)
def test_robot_finalizes_and_home_is_free(oracle, robot):
    m = robots.get(robot)
    assert m.dof == {"panda": 7, "fetch": 8, "baxter": 14}[robot]
    assert oracle.check_config(m, Scene("empty", []), np.array(m.home), two_stage=False, early_exit=False)
    # coarse spheres contain the fine ones (kinematics.cpp:56-57)
    for ls in m.spheres:
        for f in ls.fine:
            assert np.linalg.norm(np.subtract(f.center, ls.coarse.center)) + f.radius <= ls.coarse.radius + 1e-9


@pytest.mark.parametrize("robot", ROBOTS)
@pytest.mark.parametrize("kind", KINDS)
def test_scenes_deterministic_and_valid(oracle, robot, kind):
    a, ra = make_scene(robot, kind, 17)
    b, rb = make_scene(robot, kind, 17)
    assert a == b and np.array_equal(ra[0].center, rb[0].center)
    assert make_scene(robot, kind, 18)[0] != a
    assert 1 <= len(a.primitives) <= 64
    oracle.scene(a)  # Scene::validate


@pytest.mark.parametrize("robot", ROBOTS)
def test_problem_fixtures_are_feasible(oracle, robot):
    mp = _make_problems_module()
    m = robots.get(robot)
    lim = m.limits()
    probs = load_problems(robot)
    assert len(probs) >= 12
    rng = np.random.default_rng(0)
    for i in rng.choice(len(probs), size=min(15, len(probs)), replace=False):
        kind, pid, s, g = probs[i]
        scene, regions = make_scene(robot, kind, pid)
        for q in (s, g):
            assert np.all(q >= lim[:, 0]) and np.all(q <= lim[:, 1])
            assert oracle.check_config(m, scene, q, two_stage=False, early_exit=False)
        P = mp.fk_positions(m, g[None])
        for ee, reg in zip(m.ee_links, regions):
            assert reg.contains(P[ee][0])
            assert np.allclose(P[ee][0], oracle.fk_poses(m, g)[ee, 9:], atol=1e-9)
