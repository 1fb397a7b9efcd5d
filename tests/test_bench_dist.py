"""CPU: the N>1 plumbing of bench.py (one process per GPU, weak scaling over
independent problems, max-over-ranks timing) on a world_size-2 gloo group.
No collective touches the planning data path; the only collectives are the
barrier and the timing max-reduction."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

WORKER = r"""
import json, os, sys
sys.path.insert(0, %(root)r)
import bench
import torch.distributed as dist
world, rank, local = bench.dist_setup()
bench.dist_barrier(world)
m = bench.dist_max(10.0 + 5 * rank, world)
t = bench.dist_sum(100.0 + rank, world)
print(json.dumps({"rank": rank, "world": world, "max": m, "sum": t}))
dist.destroy_process_group()
"""


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_max_over_ranks(tmp_path):
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, WORLD_SIZE="2", RANK=str(r), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), PRRTC_BENCH_BACKEND="gloo")
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER % {"root": str(ROOT)}], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    assert sorted(r["rank"] for r in res) == [0, 1]
    assert all(r["world"] == 2 and r["max"] == 15.0 and r["sum"] == 201.0 for r in res)


def test_weak_scaling_value_definition():
    import bench
    # value = whole-job problems/s: N ranks x problems per rank / max step time
    assert bench.UNIT == "problems/s"
    assert "problems/sec" in bench.METRIC


def test_shard_partitions_problems():
    """Config 5 sharding: every problem lands on exactly one rank, shares
    differ by at most one (weak per-GPU load), no exchange needed."""
    import bench
    for n in (0, 1, 7, 10000):
        for world in (1, 2, 4, 8):
            parts = [bench.shard(n, world, r) for r in range(world)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= (1 if n else 0)


def test_ranks_solve_distinct_problem_sets():
    """Weak scaling over DISTINCT problems: rank r's set (problems_panda_s<r>)
    shares no problem (scene id, start, goal) with any other rank's, and every
    set keeps the 334/333/333 scene-kind mix."""
    import numpy as np

    import bench
    seen, starts = set(), []
    for r in range(8):
        (m, scenes, S, G, kinds), name = bench.problem_set("panda", r, 1000)
        assert "replica" not in name
        ids = {sc.name for sc in scenes}
        assert len(ids) == 1000 and not (ids & seen)
        seen |= ids
        starts.append(S)
        assert [int((kinds == k).sum()) for k in ("table_pick", "bookshelf", "cage")] == [334, 333, 333]
    allS = np.concatenate(starts)
    assert len(np.unique(allS, axis=0)) == len(allS)
