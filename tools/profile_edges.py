"""One-CTA chunk latency probe: validate_edges on 1 edge (32 states), for ncu."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.scenes import make_scene
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "problems_panda.npz")
m = robots.get("panda")
i = 400
sc = make_scene("panda", str(d["kind"][i]), int(d["pid"][i]))[0]
s, g = d["start"][i], d["goal"][i]
to = s + (g - s) * (0.5 / np.linalg.norm(g - s))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for rep in range(3):
    v = planner.validate_edges(m, sc, np.repeat(s[None], n, 0), np.repeat(to[None], n, 0), 32)
print(v[:4])
