"""Quick latency/throughput probe on the GPU (development aid)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.model import PlannerParams, PlanStatus
from paper_2503_06757_b200.scenes import make_scene

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
scenes = [make_scene(robot, str(k), int(p))[0] for k, p in zip(d["kind"], d["pid"])]
S, G = d["start"], d["goal"]
params = PlannerParams(tree_capacity=cap, threads_per_cta=int(sys.argv[3]) if len(sys.argv) > 3 else 0)
sel = list(range(0, len(S), max(1, len(S) // 60)))[:60]
for w in (0, 32, 64, 148, 296, 592):
    params.workers = w
    walls, devs, st, its = [], [], [], []
    for i in sel:
        r = planner.plan(m, scenes[i], S[i], G[i], params)
        walls.append(r.wall_time_ms); devs.append(r.device_time_ms); st.append(r.status); its.append(r.iterations_total)
    walls, devs, st = np.array(walls), np.array(devs), np.array(st)
    ok = st == 0
    print(f"{robot} workers={w}: solved {ok.mean():.2f} wall median {np.median(walls[ok]):.3f} p95 {np.percentile(walls[ok],95):.3f} "
          f"dev median {np.median(devs[ok]):.3f} iters med {np.median(its):.0f}", flush=True)
params.workers = 0
b = planner.Batch(m, scenes, S, G, params)
for rep in range(3):
    t = time.perf_counter(); b.launch(); res = b.results(); dt = time.perf_counter() - t
    ok = np.array([r.status == PlanStatus.Solved for r in res])
    fl = sum(r.flops for r in res)
    print(f"batch {len(S)}: {dt*1e3:.2f} ms -> {len(S)/dt:.0f} problems/s, solved {ok.mean():.3f}, "
          f"TFLOP/s(alg) {fl/dt/1e12:.3f}, per-problem dev median {np.median([r.device_time_ms for r in res]):.3f} ms", flush=True)
