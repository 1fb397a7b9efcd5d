"""Per-phase cycle breakdown of one 32-state validation chunk (one CTA)."""
import ctypes as C
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import _lib, planner, robots
from paper_2503_06757_b200.scenes import make_scene
robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
rob = planner.device_robot(m)
names = {0: "start", 7: "setup", 8: "gen", 1: "chk", 2: "fkA", 3: "fkB", 4: "fkC", 10: "coarse_env(w0)",
         11: "self_pairs(w0)", 5: "coarse_sync", 6: "fine_env", 9: "end"}
order = [0, 7, 8, 1, 2, 3, 4, 10, 11, 5, 6, 9]
for i in (0, 400, 700):
    sc = planner.device_scene(make_scene(robot, str(d["kind"][i]), int(d["pid"][i]))[0])
    s, g = d["start"][i], d["goal"][i]
    to = s + (g - s) * (0.5 / np.linalg.norm(g - s))
    for rep in range(3):
        st = (C.c_longlong * 16)()
        _lib.check(_lib.load().prrtc_debug_chunk_profile(rob.h, sc.h, s.ctypes.data_as(C.POINTER(C.c_double)),
                                                        to.ctypes.data_as(C.POINTER(C.c_double)), m.dof, 32, 1, st))
    t = list(st)
    prev = t[0]
    parts = []
    for k in order[1:]:
        if t[k]:
            parts.append(f"{names[k]} {t[k] - prev}")
            prev = t[k]
    print(f"{robot} problem {i}: total {t[9] - t[0]} cycles | " + ", ".join(parts))
