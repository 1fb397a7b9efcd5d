"""The C++ drop-in (prrtc::b200::plan, reference types) against the reference
prrtc::plan in the same process (tests/cpp/dropin_demo.cpp)."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import load_problems
from paper_2503_06757_b200 import robots
from paper_2503_06757_b200.model import BoxPrim, CapsulePrim, SpherePrim
from paper_2503_06757_b200.scenes import make_scene

ROOT = Path(__file__).resolve().parents[1]
DEMO = ROOT / "tests" / "cpp" / "bin" / "dropin_demo"
DROPIN = ROOT / "paper_2503_06757_b200" / "lib" / "libprrtc_b200_dropin.so"


def fmt(x):
    return repr(float(x))


def write_problems(path, model, problems):
    out = [f"{model.link_count()} {len(model.self_pairs)}"]
    for j, ls in zip(model.joints, model.spheres):
        vals = [j.kind, j.parent, *j.origin_quat, *j.origin_xyz, *j.axis, j.lo, j.hi,
                *ls.coarse.center, ls.coarse.radius, len(ls.fine)]
        for f in ls.fine:
            vals += [*f.center, f.radius]
        out.append(" ".join(str(v) if isinstance(v, int) else fmt(v) for v in vals))
    out.append(" ".join(f"{a} {b}" for a, b in model.self_pairs))
    out.append(str(len(problems)))
    for scene, s, g in problems:
        sp = [p for p in scene.primitives if isinstance(p, SpherePrim)]
        bp = [p for p in scene.primitives if isinstance(p, BoxPrim)]
        cp = [p for p in scene.primitives if isinstance(p, CapsulePrim)]
        vals = [len(sp), len(bp), len(cp)]
        out.append(" ".join(map(str, vals)))
        out.append(" ".join(fmt(v) for p in sp for v in (*p.center, p.radius)))
        out.append(" ".join(fmt(v) for p in bp for v in (*p.quat, *p.translation, *p.half_extents)))
        out.append(" ".join(fmt(v) for p in cp for v in (*p.a, *p.b, p.radius)))
        out.append(" ".join(fmt(v) for v in s))
        out.append(" ".join(fmt(v) for v in g))
    path.write_text("\n".join(out) + "\n")


def test_dropin_library_exports_reference_signature():
    if not DROPIN.exists():
        pytest.skip("drop-in not built (needs the reference headers at build time)")
    syms = subprocess.run(["nm", "-DC", str(DROPIN)], capture_output=True, text=True).stdout
    assert ("prrtc::b200::plan(prrtc::RobotModel const&, prrtc::Scene const&, std::span<double const, "
            "18446744073709551615ul>, std::span<double const, 18446744073709551615ul>, "
            "prrtc::PlannerParams const&)") in syms


@pytest.mark.gpu
def test_dropin_matches_reference_contract(gpu, oracle, tmp_path):
    if not DEMO.exists():
        pytest.skip("drop-in demo not built")
    m = robots.get("panda")
    probs = load_problems("panda")
    pick = [probs[i] for i in range(0, len(probs), 90)][:10]
    items = [(make_scene("panda", k, p)[0], s, g) for k, p, s, g in pick]
    f = tmp_path / "p.txt"
    write_problems(f, m, items)
    r = subprocess.run([str(DEMO), str(f)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.strip().splitlines()]
    assert lines[-1]["invalid_argument"] and "expected dimension" in lines[-1]["what"]
    # 4 concurrent host threads and the multi-device batch: every problem
    # answered (Solved / Failed), solved paths run start -> goal (9 = not)
    conc = next(x["concurrent"] for x in lines if "concurrent" in x)
    multi = next(x["multi"] for x in lines if "multi" in x)
    assert len(conc) == len(multi) == len(items)
    assert all(v in (0, 1) for v in conc + multi)
    b200 = [x for x in lines if x.get("impl") == "b200"]
    ref = [x for x in lines if x.get("impl") == "reference"]
    assert len(b200) == len(ref) == len(items)
    assert sum(x["status"] == 0 for x in b200) >= sum(x["status"] == 0 for x in ref)
    for x, (scene, s, g) in zip(b200, items):
        if x["status"] != 0:
            continue
        P = np.array(x["path"])
        assert np.array_equal(P[0], s) and np.array_equal(P[-1], g)
        # sound at the planner's resolution (the reference planner's own
        # guarantee; the 4 x n_cc sound mode is tested in test_gpu_planner.py)
        assert oracle.path_valid(m, scene, P, 32)
        assert abs(x["cost"] - np.linalg.norm(np.diff(P, axis=0), axis=1).sum()) < 1e-9
