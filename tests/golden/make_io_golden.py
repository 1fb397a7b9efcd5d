"""Generates tests/golden/io/: model files WRITTEN BY THE REFERENCE's own
writers (model_io.cpp:344-421, compiled in place as oracle/_ref/
libprrtc_ref_io.so) and the reference's error messages for the malformed
inputs of tests/test_model_io.py. Run in the build container (needs
/root/reference):  python tests/golden/make_io_golden.py
"""
import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.refio import RefIO  # noqa: E402
from paper_2503_06757_b200 import model_io as mio  # noqa: E402
from paper_2503_06757_b200 import robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402

OUT = ROOT / "tests" / "golden" / "io"


def main():
    ref = RefIO()
    OUT.mkdir(exist_ok=True)
    for f in OUT.glob("*.json"):
        f.unlink()
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)

        def via_ref(kind, write, name):
            write(td / name)
            err = ref.roundtrip(kind, td / name, OUT / name)
            assert err is None, err

        for r in ("panda", "fetch", "baxter"):
            via_ref("robot", lambda p, r=r: mio.write_robot(p, robots.get(r)), f"robot_{r}.json")
        for i, kind in enumerate(("table_pick", "bookshelf", "cage")):
            s, _ = make_scene("panda", kind, i)
            via_ref("scene", lambda p, s=s: mio.write_scene(p, s), f"scene_{kind}.json")
        d = np.load(ROOT / "tests" / "golden" / "problems_panda.npz")
        shutil.copy(OUT / "robot_panda.json", td / "robot_panda.json")
        for i, (kind, patch) in enumerate((("table_pick", mio.ParamsPatch()),
                                           ("bookshelf", mio.ParamsPatch(delta=0.25, seed=4, early_exit=False)))):
            shutil.copy(OUT / f"scene_{kind}.json", td / f"scene_{kind}.json")
            spec = mio.ProblemSpec(name=f"panda_{kind}", robot="robot_panda.json", scene=f"scene_{kind}.json",
                                   start=d["start"][0], goal=d["goal"][0], params=patch)
            via_ref("problem", lambda p, spec=spec: mio.write_problem(p, spec), f"problem_{kind}.json")
        rng = np.random.default_rng(1)
        pf = mio.PathFile(robot="robot_panda.json", scene="scene_cage.json", configs=list(rng.standard_normal((6, 7))),
                          cost=4.75, params=PlannerParams(delta=0.4, n_cc=24, seed=2), timestamp="2026-10-17T00:00:00Z")
        via_ref("path", lambda p: mio.write_path(p, pf), "path_panda.json")

        import test_model_io as t
        errs = {}
        for kind, cases in (("robot", t._BAD_ROBOTS), ("scene", t._BAD_SCENES)):
            errs[kind] = {}
            for name, body in cases.items():
                f = td / f"{name}.json"
                f.write_text(json.dumps(body))
                e = ref.roundtrip(kind, f, td / "o.json")
                errs[kind][name] = e.replace(str(td) + "/", "")
        (OUT / "errors.json").write_text(json.dumps(errs, indent=1, sort_keys=True) + "\n")
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
