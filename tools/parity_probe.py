"""Equal-budget planner parity probe: GPU batch vs the
reference planner at identical PlannerParams, per robot and workers W.

    python tools/parity_probe.py [--robots panda,fetch,baxter] [--n 1000] [--ws 1,16]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--robots", default="panda,fetch,baxter")
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--ws", default="1,16")
    ap.add_argument("--cap", type=int, default=200000)
    a = ap.parse_args()
    t0 = time.time()
    out = bench.parity_block(a.robots.split(","), [int(w) for w in a.ws.split(",")], a.n, device=0,
                             tree_capacity=a.cap)
    out["probe_s"] = time.time() - t0
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
