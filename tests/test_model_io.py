"""CPU: the model I/O drop-in (paper_2503_06757_b200/model_io.py) against the
reference's own model_io.cpp (oracle/_ref/libprrtc_ref_io.so, compiled in
place) and against committed fixtures written by it (tests/golden/io/).

* files we write load in the reference and re-serialise to the same text
  (byte-identical except the one cosmetic difference of the image's
  nlohmann copy, see _normalise);
* files the reference writes load here to bit-identical values;
* every schema / invariant error carries the reference's exact message.
"""
import json
import re
import shutil
from pathlib import Path

import numpy as np
import pytest

from paper_2503_06757_b200 import model_io as mio
from paper_2503_06757_b200 import robots
from paper_2503_06757_b200.model import BoxPrim, CapsulePrim, PlannerParams, PlanStatus, SpherePrim
from paper_2503_06757_b200.scenes import make_scene

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden" / "io"

try:
    from oracle.refio import RefIO, available as refio_available
except Exception:  # pragma: no cover
    refio_available = lambda: False  # noqa: E731

needs_ref = pytest.mark.skipif(not refio_available(), reason="reference model_io build absent (oracle/_ref)")


def _normalise(text: str) -> str:
    """The only nlohmann copy in this image (cudnn_frontend's, 3.11.3) is
    patched to print integer arrays on one line ("Custom from FE" in its
    serializer); stock 3.11.3, which the reference pins, expands them like
    any other array. Our writer follows stock; collapse integer arrays in
    both texts before comparing."""
    return re.sub(r"\[\s*(-?\d+)\s*,\s*(-?\d+)\s*\]", r"[\1,\2]", text)


@pytest.fixture(scope="module")
def ref():
    return RefIO()


def _robot_equal(a, b):
    assert a.name == b.name and len(a.joints) == len(b.joints)
    for ja, jb in zip(a.joints, b.joints):
        assert (ja.kind, ja.parent) == (jb.kind, jb.parent)
        assert tuple(ja.origin_quat) == tuple(jb.origin_quat) and tuple(ja.origin_xyz) == tuple(jb.origin_xyz)
        if ja.kind != 2:
            assert tuple(ja.axis) == tuple(jb.axis) and (ja.lo, ja.hi) == (jb.lo, jb.hi)
    for sa, sb in zip(a.spheres, b.spheres):
        assert tuple(sa.coarse.center) == tuple(sb.coarse.center) and sa.coarse.radius == sb.coarse.radius
        assert [(tuple(f.center), f.radius) for f in sa.fine] == [(tuple(f.center), f.radius) for f in sb.fine]
    assert [tuple(p) for p in a.self_pairs] == [tuple(p) for p in b.self_pairs]


# ---------------------------------------------------------------------------
# number formatting (nlohmann::detail::to_chars)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("x,s", [(1.0, "1.0"), (0.5, "0.5"), (-2.8973, "-2.8973"), (0.0, "0.0"), (-0.0, "-0.0"),
                                 (1e-5, "1e-05"), (0.0001234, "0.0001234"), (123456789012345.0, "123456789012345.0"),
                                 (1e15, "1e+15"), (1.5e16, "1.5e+16"), (0.1 + 0.2, "0.30000000000000004"),
                                 (2.5e-300, "2.5e-300"), (1e100, "1e+100")])
def test_double_format(x, s):
    assert mio._fmt_double(x) == s
    assert float(s) == x


def test_double_format_roundtrips_random():
    rng = np.random.default_rng(5)
    for x in np.concatenate([rng.standard_normal(2000), rng.standard_normal(500) * 1e-6,
                             rng.standard_normal(500) * 1e12]):
        assert float(mio._fmt_double(float(x))) == float(x)


# ---------------------------------------------------------------------------
# writers -> reference loaders -> reference writers
# ---------------------------------------------------------------------------
@needs_ref
@pytest.mark.parametrize("name", ["panda", "fetch", "baxter"])
def test_robot_roundtrip_through_reference(ref, tmp_path, name):
    m = robots.get(name)
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    mio.write_robot(a, m)
    assert ref.roundtrip("robot", a, b) is None
    assert _normalise(a.read_text()) == _normalise(b.read_text())
    assert ref.robot_dof(a) == m.dof
    _robot_equal(mio.load_robot(b), m)


@needs_ref
@pytest.mark.parametrize("robot,kind,pid", [("panda", "table_pick", 0), ("panda", "bookshelf", 7), ("panda", "cage", 3),
                                            ("fetch", "bookshelf", 2), ("baxter", "cage", 1)])
def test_scene_roundtrip_through_reference(ref, tmp_path, robot, kind, pid):
    try:
        s, _ = make_scene(robot, kind, pid)
    except Exception:
        pytest.skip(f"no {kind} scenes for {robot}")
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    mio.write_scene(a, s)
    assert ref.roundtrip("scene", a, b) is None
    assert a.read_text() == b.read_text()  # no integer arrays: byte-identical
    s2 = mio.load_scene(b)
    assert s2.name == s.name and len(s2.primitives) == len(s.primitives)
    for p, q in zip(s.primitives, s2.primitives):
        assert type(p) is type(q) and repr(p) == repr(q)


def _write_problem_dir(d: Path, robot="panda", n=3, patch=None):
    m = robots.get(robot)
    mio.write_robot(d / f"{robot}.json", m)
    data = np.load(ROOT / "tests" / "golden" / f"problems_{robot}.npz")
    for i in range(n):
        s, _ = make_scene(robot, str(data["kind"][i]), int(data["pid"][i]))
        mio.write_scene(d / f"scene_{i}.json", s)
        p = mio.ProblemSpec(name=f"{robot}_{i:03d}", robot=f"{robot}.json", scene=f"scene_{i}.json",
                            start=data["start"][i], goal=data["goal"][i],
                            params=patch if patch is not None else mio.ParamsPatch())
        mio.write_problem(d / f"problem_{i:03d}.json", p)
    return m


@needs_ref
def test_problem_and_path_roundtrip_through_reference(ref, tmp_path):
    patch = mio.ParamsPatch(delta=0.25, n_cc=16, workers=4, max_iters_per_worker=500, tree_capacity=4000,
                            dd_radius=1.5, dynamic_domain=False, balance=True, early_exit=False, two_stage=True,
                            batched_cc=True, nn_partitions=2, sampler=0, seed=9)
    _write_problem_dir(tmp_path, patch=patch)
    a, b = tmp_path / "problem_000.json", tmp_path / "rt.json"
    assert ref.roundtrip("problem", a, b) is None
    assert a.read_text() == b.read_text()
    pr = mio.load_problem(b)
    assert pr.params == patch and pr.robot == "panda.json"
    # effective params of the bundle equal the reference's
    base = PlannerParams(seed=3)
    rp, name = ref.problem_bundle(a, base)
    from paper_2503_06757_b200 import suite
    lp = suite.load_problem_bundle(a, base)
    assert name == lp.spec.name
    for f in ("delta", "n_cc", "workers", "max_iters_per_worker", "tree_capacity", "dd_radius", "nn_partitions", "seed"):
        assert getattr(rp, f) == getattr(lp.params, f), f
    for f in ("dynamic_domain", "balance", "early_exit", "two_stage", "batched_cc"):
        assert bool(getattr(rp, f)) == bool(getattr(lp.params, f)), f
    # path file
    rng = np.random.default_rng(0)
    pf = mio.PathFile(robot="panda.json", scene="scene_0.json", configs=list(rng.standard_normal((5, 7))),
                      cost=3.25, params=PlannerParams(delta=0.3, seed=11), timestamp="2026-10-17T00:00:00Z")
    pa, pb = tmp_path / "path.json", tmp_path / "path_rt.json"
    mio.write_path(pa, pf)
    assert ref.roundtrip("path", pa, pb) is None
    assert pa.read_text() == pb.read_text()
    back = mio.load_path_file(pb)
    assert np.array_equal(np.array(back.configs), np.array(pf.configs))
    assert back.cost == pf.cost and back.params == pf.params and back.timestamp == pf.timestamp


@needs_ref
def test_problem_dir_order_matches_reference(ref, tmp_path):
    _write_problem_dir(tmp_path, n=4)
    (tmp_path / "notes.txt").write_text("not a problem")
    from paper_2503_06757_b200 import suite
    # robot/scene files are *.json too: load_problem_dir treats every *.json
    # in the directory as a problem, exactly like bench.cpp:47-61 -> both fail
    with pytest.raises(mio.IoError) as e:
        suite.load_problem_dir(tmp_path, PlannerParams())
    with pytest.raises(RuntimeError) as r:
        ref.problem_dir(tmp_path)
    assert str(e.value) == str(r.value)
    d = tmp_path / "problems"
    d.mkdir()
    for f in sorted(tmp_path.glob("problem_*.json")):
        txt = json.loads(f.read_text())
        txt["robot"], txt["scene"] = "../" + txt["robot"], "../" + txt["scene"]
        (d / f.name).write_text(json.dumps(txt))
    names = [lp.spec.name for lp in suite.load_problem_dir(d, PlannerParams())]
    assert names == ref.problem_dir(d) and len(names) == 4


# ---------------------------------------------------------------------------
# error behaviour: identical messages
# ---------------------------------------------------------------------------
_BAD_ROBOTS = {
    "missing_joints": {"name": "r", "spheres": []},
    "joints_not_array": {"name": "r", "joints": 3, "spheres": []},
    "bad_kind": {"joints": [{"kind": "spherical", "parent": -1}], "spheres": []},
    "kind_wrong_type": {"joints": [{"kind": 1, "parent": -1}], "spheres": []},
    "missing_origin": {"joints": [{"kind": "fixed", "parent": -1}], "spheres": []},
    "short_translation": {"joints": [{"kind": "fixed", "parent": -1, "origin": {"translation": [0, 0],
                                                                                  "quaternion": [1, 0, 0, 0]}}],
                          "spheres": []},
    "bad_quat_len": {"joints": [{"kind": "fixed", "parent": -1, "origin": {"translation": [0, 0, 0],
                                                                             "quaternion": [1, 0, 0]}}],
                     "spheres": []},
    "bad_limits": {"joints": [{"kind": "revolute", "parent": -1, "axis": [0, 0, 1], "limits": [1],
                               "origin": {"translation": [0, 0, 0], "quaternion": [1, 0, 0, 0]}}], "spheres": []},
    "quat_norm": {"joints": [{"kind": "fixed", "parent": -1, "origin": {"translation": [0, 0, 0],
                                                                          "quaternion": [1.1, 0, 0, 0]}}],
                  "spheres": [{"coarse": {"center": [0, 0, 0], "radius": 1}, "fine": []}]},
    "axis_norm": {"joints": [{"kind": "revolute", "parent": -1, "axis": [0, 0, 2], "limits": [-1, 1],
                              "origin": {"translation": [0, 0, 0], "quaternion": [1, 0, 0, 0]}}],
                  "spheres": [{"coarse": {"center": [0, 0, 0], "radius": 1}, "fine": []}]},
    "sphere_count": {"joints": [{"kind": "fixed", "parent": -1, "origin": {"translation": [0, 0, 0],
                                                                             "quaternion": [1, 0, 0, 0]}}],
                     "spheres": []},
    "escape": {"joints": [{"kind": "fixed", "parent": -1, "origin": {"translation": [0, 0, 0],
                                                                       "quaternion": [1, 0, 0, 0]}}],
               "spheres": [{"coarse": {"center": [0, 0, 0], "radius": 0.1},
                            "fine": [{"center": [0.05, 0, 0], "radius": 0.07}]}]},
    "fine_radius": {"joints": [{"kind": "fixed", "parent": -1, "origin": {"translation": [0, 0, 0],
                                                                            "quaternion": [1, 0, 0, 0]}}],
                    "spheres": [{"coarse": {"center": [0, 0, 0], "radius": 0.1},
                                 "fine": [{"center": [0, 0, 0], "radius": 0}]}]},
    "pair_adjacent": {"joints": [{"kind": "fixed", "parent": -1, "origin": {"translation": [0, 0, 0],
                                                                              "quaternion": [1, 0, 0, 0]}},
                                 {"kind": "fixed", "parent": 0, "origin": {"translation": [0, 0, 0],
                                                                           "quaternion": [1, 0, 0, 0]}}],
                      "spheres": [{"coarse": {"center": [0, 0, 0], "radius": 0.1}, "fine": []}] * 2,
                      "self_pairs": [[0, 1]]},
    "pair_shape": {"joints": [{"kind": "fixed", "parent": -1, "origin": {"translation": [0, 0, 0],
                                                                           "quaternion": [1, 0, 0, 0]}}],
                   "spheres": [{"coarse": {"center": [0, 0, 0], "radius": 0.1}, "fine": []}],
                   "self_pairs": [[0, 1, 2]]},
    "parent_order": {"joints": [{"kind": "fixed", "parent": 0, "origin": {"translation": [0, 0, 0],
                                                                            "quaternion": [1, 0, 0, 0]}}],
                     "spheres": [{"coarse": {"center": [0, 0, 0], "radius": 0.1}, "fine": []}]},
    "radius_type": {"joints": [{"kind": "fixed", "parent": -1, "origin": {"translation": [0, 0, 0],
                                                                            "quaternion": [1, 0, 0, 0]}}],
                    "spheres": [{"coarse": {"center": [0, 0, 0], "radius": "big"}, "fine": []}]},
}
_BAD_SCENES = {
    "missing_prims": {"name": "s"},
    "bad_kind": {"primitives": [{"kind": "cylinder"}]},
    "sphere_radius": {"primitives": [{"kind": "sphere", "center": [0, 0, 0], "radius": -1}]},
    "box_extent": {"primitives": [{"kind": "box", "pose": {"translation": [0, 0, 0], "quaternion": [1, 0, 0, 0]},
                                   "half_extents": [1, 0, 1]}]},
    "box_quat": {"primitives": [{"kind": "box", "pose": {"translation": [0, 0, 0], "quaternion": [0.5, 0, 0, 0]},
                                 "half_extents": [1, 1, 1]}]},
    "capsule_radius": {"primitives": [{"kind": "capsule", "a": [0, 0, 0], "b": [0, 0, 1], "radius": 0}]},
    "capsule_missing_b": {"primitives": [{"kind": "capsule", "a": [0, 0, 0], "radius": 1}]},
}


def _messages(tmp_path, ref, kind, cases):
    out = {}
    for name, body in cases.items():
        f = tmp_path / f"{name}.json"
        f.write_text(json.dumps(body))
        loader = mio.load_robot if kind == "robot" else mio.load_scene
        with pytest.raises(mio.IoError) as e:
            loader(f)
        got = str(e.value).replace(str(tmp_path) + "/", "")
        if ref is not None:
            want = ref.roundtrip(kind, f, tmp_path / "out.json")
            assert want is not None, name
            assert got == want.replace(str(tmp_path) + "/", ""), name
        out[name] = got
    return out


@needs_ref
def test_error_messages_match_reference(ref, tmp_path):
    _messages(tmp_path, ref, "robot", _BAD_ROBOTS)
    _messages(tmp_path, ref, "scene", _BAD_SCENES)


def test_error_messages_match_golden(tmp_path):
    """Pinned without the reference build: messages recorded from it."""
    want = json.loads((GOLD / "errors.json").read_text())
    assert _messages(tmp_path, None, "robot", _BAD_ROBOTS) == want["robot"]
    assert _messages(tmp_path, None, "scene", _BAD_SCENES) == want["scene"]


@needs_ref
def test_problem_and_path_errors_match_reference(ref, tmp_path):
    m = _write_problem_dir(tmp_path, n=1)
    good = json.loads((tmp_path / "problem_000.json").read_text())
    cases = {
        "dim": dict(good, start=good["start"][:-1]),
        "goal_dim": dict(good, goal=good["goal"] + [0.0]),
        "start_type": dict(good, start=["a"] * m.dof),
        "sampler": dict(good, params={"sampler": "sobol"}),
        "robot_missing": {k: v for k, v in good.items() if k != "robot"},
    }
    for name, body in cases.items():
        f = tmp_path / f"bad_{name}.json"
        f.write_text(json.dumps(body))
        with pytest.raises(mio.IoError) as e:
            mio.load_problem(f)
        want = ref.roundtrip("problem", f, tmp_path / "o.json")
        assert str(e.value) == want, name
    pcases = {"empty": {"robot": "r", "scene": "s", "path": []},
              "dup": {"robot": "r", "scene": "s", "path": [[0.0, 1.0], [0.0, 1.0]]},
              "notnum": {"robot": "r", "scene": "s", "path": [[0.0, "x"]]}}
    for name, body in pcases.items():
        f = tmp_path / f"badpath_{name}.json"
        f.write_text(json.dumps(body))
        with pytest.raises(mio.IoError) as e:
            mio.load_path_file(f)
        assert str(e.value) == ref.roundtrip("path", f, tmp_path / "o.json"), name
    with pytest.raises(mio.IoError) as e:
        mio.write_path(tmp_path / "w.json", mio.PathFile(configs=[np.zeros(2), np.zeros(2)]))
    assert str(e.value) == f"{tmp_path}/w.json.path[1]: duplicates the previous waypoint"
    with pytest.raises(mio.IoError) as e:
        mio.load_robot(tmp_path / "nope.json")
    assert str(e.value) == f"{tmp_path}/nope.json: cannot open file"


# ---------------------------------------------------------------------------
# committed fixtures written by the reference
# ---------------------------------------------------------------------------
def test_golden_files_load_and_rewrite(tmp_path):
    """tests/golden/io/*.json were written by the reference's writers
    (make_io_golden.py); loading and rewriting them reproduces the text."""
    for f in sorted(GOLD.glob("robot_*.json")):
        m = mio.load_robot(f)
        mio.write_robot(tmp_path / f.name, m)
        assert _normalise((tmp_path / f.name).read_text()) == _normalise(f.read_text()), f.name
        assert m.dof == {"panda": 7, "fetch": 8, "baxter": 14}[m.name]
    for f in sorted(GOLD.glob("scene_*.json")):
        mio.write_scene(tmp_path / f.name, mio.load_scene(f))
        assert (tmp_path / f.name).read_text() == f.read_text(), f.name
    for f in sorted(GOLD.glob("problem_*.json")):
        mio.write_problem(tmp_path / f.name, mio.load_problem(f))
        assert (tmp_path / f.name).read_text() == f.read_text(), f.name
    for f in sorted(GOLD.glob("path_*.json")):
        mio.write_path(tmp_path / f.name, mio.load_path_file(f))
        assert (tmp_path / f.name).read_text() == f.read_text(), f.name


# ---------------------------------------------------------------------------
# CSVs
# ---------------------------------------------------------------------------
def _records(n=40, seed=0):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        st = PlanStatus(int(rng.choice([0, 0, 0, 1, 2])))
        out.append(mio.BenchRecord(problem=f"p{i % 7}", trial=i // 7, status=st, time_ms=float(rng.exponential(2.0)),
                                   cost=float(rng.uniform(1, 9)), iterations=int(rng.integers(0, 5000)),
                                   sphere_tests=int(rng.integers(0, 10**9)), workers=int(rng.integers(1, 300)),
                                   seed=int(rng.integers(0, 2**63))))
    return out


@needs_ref
def test_results_csv_matches_reference(ref):
    recs = _records()
    assert mio.results_csv_string(recs) == ref.results_csv(recs)


def test_results_csv_format(tmp_path):
    recs = [mio.BenchRecord(problem="a", trial=0, status=PlanStatus.Solved, time_ms=1.23456, cost=0.1, iterations=5,
                            sphere_tests=7, workers=2, seed=3),
            mio.BenchRecord(problem="b", status=PlanStatus.InfeasibleEndpoint, time_ms=0.5, cost=9.0)]
    s = mio.results_csv_string(recs)
    assert s == ("problem,status,time_ms,cost,iterations,sphere_tests,workers,seed\n"
                 "a,Solved,1.235,0.10000000000000001,5,7,2,3\n"
                 "b,Infeasible-endpoint,0.500,,0,0,1,0\n")
    mio.write_results_csv(tmp_path / "r.csv", recs)
    assert (tmp_path / "r.csv").read_text() == s
    mio.write_ecdf_csv(tmp_path / "e.csv", [(0.5, 0.25), (1.0, 0.5)])
    assert (tmp_path / "e.csv").read_text() == "value,fraction_solved\n0.5,0.25\n1,0.5\n"
