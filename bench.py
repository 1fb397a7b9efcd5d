#!/usr/bin/env python
"""bench.py — B200 pRRTC planning benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Metric (BASELINE.json): "median/p95 ms-to-first-solution per problem;
problems/sec at 1/2/4/8 B200". Workload = BASELINE configs[1]: Panda 7-DoF,
a batch of 1000 synthetic MotionBenchMaker-shaped problems (334 table_pick /
333 bookshelf / 333 cage, tests/golden/problems_panda.npz), reference default
PlannerParams (delta 0.5, n_cc 32, tree_capacity 200000, dynamic domain,
two-stage, early exit, Halton).

A step = one full solve of the 1000-problem batch (every problem to Solved
or Failed) by one persistent plan_kernel launch on inputs already resident
in HBM; `value` = problems/s of the whole job (N ranks x 1000 problems / the
max-over-ranks step time; weak scaling, no collective on the data path).
`e2e` = the same through the host-buffer C-ABI call prrtc_plan_batch
(packed H2D of starts/goals/scene table, kernel, D2H of results/paths).
`latency_ms` = median / p95 of single-problem prrtc_plan calls (host wall
clock around the C call, setup excluded as in PAPER.md:201).

--impl reference times the reference's own CPU planner (oracle/_ref, the
unmodified reference sources; the C restatement oracle/liboracle.so when the
reference build is absent) on the host cores, same problems and params.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "median/p95 ms-to-first-solution per problem; problems/sec at 1/2/4/8 B200"
UNIT = "problems/s"


def load_workload(robot: str, n: int, set_k: int = 0):
    """The first n problems of the robot's 1000-problem set (all of it for
    n >= 1000); a smaller n takes an evenly spread subset, so every scene
    kind (the set is ordered table_pick / bookshelf / cage) stays represented."""
    from paper_2503_06757_b200 import robots
    from paper_2503_06757_b200.scenes import make_scene
    d = np.load(ROOT / "tests" / "golden" / (f"problems_{robot}_s{set_k}.npz" if set_k else f"problems_{robot}.npz"))
    N = len(d["pid"])
    idx = np.arange(N) if n >= N else np.unique(np.linspace(0, N - 1, n).round().astype(int))
    scenes = [make_scene(robot, str(d["kind"][i]), int(d["pid"][i]))[0] for i in idx]
    return robots.get(robot), scenes, d["start"][idx].copy(), d["goal"][idx].copy(), d["kind"][idx]


def workload_config(robot, n, params, world):
    """The workload description, identical on both arms (same keys, same values)."""
    return {
        "workload": f"{robot}_mbm_{n}",
        "robot": robot,
        "problems_per_gpu": n,
        "scenes": "table_pick/bookshelf/cage 334/333/333 (synthetic MBM-shaped, tests/golden)",
        "params": {"delta": params.delta, "n_cc": params.n_cc, "workers": params.workers,
                   "max_iters_per_worker": params.max_iters_per_worker, "tree_capacity": params.tree_capacity,
                   "dynamic_domain": True, "dd_radius": params.resolved_dd_radius(), "two_stage": True,
                   "early_exit": True, "sampler": "halton"},
        "l2": "flushed between timed steps (256 MiB write)",
        "parallelism": f"dp{world} (independent problems per GPU, no collective)",
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 5 + i and s[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    """One process per GPU; the process group (gloo, host memory) carries only
    the timing barrier and the max / sum of per-rank numbers — nothing on the
    planning path needs a collective (north_star: no NCCL)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    return world, rank, local


def dist_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def shard(n: int, world: int, rank: int) -> list:
    """This rank's share of n independent problems (round robin, no exchange)."""
    return list(range(rank, n, world))


def dist_barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_reference(model, scenes, S, G, params, threads):
    """Reference CPU planner (oracle/_ref when built, else the C port)."""
    from oracle import Oracle, available
    kind = "reference" if available("ref") else "port"
    o = Oracle("ref" if kind == "reference" else "port")
    res, ms = o.plan_many(model, scenes, S, G, params, threads=threads)
    return o, kind, res, ms


def ncu_summary() -> dict:
    """profiles/ncu_summary.json: the committed ncu --set full capture of
    plan_kernel (tools/summarize_profile.py), or {}."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return {}
    return {}


def traffic_from_profiles():
    return ncu_summary().get("plan_kernel_dram_bytes_per_launch")


def microbench(model, scenes, S, G, dev, fp32_peak):
    """SURVEY.md §8(d) roofline microbenchmarks of the two kernels inside the
    planner: the collision path (prrtc_validate_edges' kernel) in dense mode
    (two_stage off, early_exit off: every test executed, the unambiguous
    FP32-pipe figure) and in the production two-stage mode, and the NN scan
    (FP64 SoA tree, 100k nodes = one tree at the default capacity) against the
    measured L2 read bandwidth. Device-resident inputs, CUDA events."""
    import ctypes
    from paper_2503_06757_b200 import _lib, planner
    lib = _lib.load()
    rob = planner.device_robot(model, dev)
    out = {}
    # 32768 edges = 1M states: ~14 rounds of the 2368 warp checkers (4096
    # left the last of ~2 rounds 40% idle)
    n_edges, n_cc, delta = 32768, 32, 0.5
    k = np.arange(n_edges) % len(S)
    A = np.ascontiguousarray(S[k])
    d = G[k] - A
    B = np.ascontiguousarray(A + d * np.minimum(1.0, delta / np.linalg.norm(d, axis=1))[:, None])
    sc = planner.device_scene(scenes[len(scenes) // 2], dev)  # a bookshelf scene
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    for name, two, early in (("collision_dense", 0, 0), ("collision_two_stage", 1, 1)):
        ms, fl, te = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        _lib.check(lib.prrtc_bench_validate_edges(rob.h, sc.h, dp(A), dp(B), n_edges, model.dof, n_cc, two, early, 5,
                                                  ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(te)))
        states = n_edges * n_cc
        tf = fl.value / (ms.value * 1e-3) / 1e12
        out[name] = {"kernel": "validate_edges_warp_kernel (one edge per warp, one state per lane)",
                     "edges": n_edges, "states": states, "ms": ms.value,
                     "states_per_s": states / (ms.value * 1e-3), "flops_per_state": fl.value / states,
                     "tests_per_state": te.value / states, "achieved_tflops": tf,
                     "frac_fp32_peak": tf / fp32_peak if fp32_peak else None,
                     "mode": f"two_stage={two} early_exit={early}"}
    l2 = lib.prrtc_l2_peak_gbs(dev)
    fp64 = lib.prrtc_fp64_peak_tflops(dev)
    rng = np.random.default_rng(7)
    lim = model.limits()
    T = np.ascontiguousarray(rng.uniform(lim[:, 0], lim[:, 1], size=(100000, model.dof)))
    for g in (1, 32):
        # enough queries for >= 592 CTAs (one CTA takes g queries per pass)
        Q = np.ascontiguousarray(rng.uniform(lim[:, 0], lim[:, 1], size=(2048 if g == 1 else 32 * 592, model.dof)))
        ms = ctypes.c_double()
        _lib.check(lib.prrtc_bench_nn(dp(T), T.shape[0], model.dof, dp(Q), Q.shape[0], g, dev, 3, ctypes.byref(ms)))
        # the reference's arithmetic: FP64 keys, 3 un-fused ops (sub, mul, add)
        # per (query, node, dimension); node coordinates 8 B each (FP64 SoA)
        pairs = Q.shape[0] * T.shape[0]
        tf = pairs * model.dof * 3 / (ms.value * 1e-3) / 1e12
        gbs = pairs * model.dof * 8 / (ms.value * 1e-3) / 1e9
        out[f"nn_group{g}"] = {"kernel": "debug_nn_multi_kernel (the planner's nn_scan_multi)", "tree_nodes": T.shape[0],
                               "queries": Q.shape[0], "queries_per_pass": g, "ms": ms.value,
                               "bound": "fp64", "achieved_fp64_tflops": tf,
                               "frac_fp64_peak": tf / fp64 if fp64 else None,
                               "bytes_per_query_fp64": T.shape[0] * model.dof * 8,
                               "query_node_bytes_per_s_gbs": gbs,
                               "note": f"{g} queries share each node load (L1): per-query bytes exceed the L2 "
                                       "peak by that reuse, so the FP64 pipe is the bound"}
    out["l2_peak_gbs"] = l2
    out["fp32_peak_tflops"] = fp32_peak
    out["fp64_peak_tflops"] = fp64
    return out


def bench_extras(dev, params):
    """BASELINE config 5's dynamic-obstacle replanning loop beside the headline
    (informational, untimed by the driver), rank 0: 100 frames, 3 spheres
    moving 1 cm/frame, prrtc_scene_update + prrtc_plan per frame. Configs 3-4
    (Fetch / Baxter) are table_one; the 10k mixed batch is mixed_sharded
    (every rank)."""
    import torch
    from paper_2503_06757_b200 import planner, replan
    from paper_2503_06757_b200.model import PlannerParams, PlanStatus

    out = {}
    # replanning loop
    model, scenes, S, G, kinds = load_workload("panda", 1000)
    i = int(np.where(kinds == "table_pick")[0][0])
    rp = PlannerParams()  # latency scenario: workers = 0 (one CTA per SM)
    frames = replan.run(model, scenes[i], S[i], G[i], frames=100, params=rp, device=dev)
    wall = [f.wall_ms for f in frames]
    ok = [f.result.status == PlanStatus.Solved for f in frames]
    out["replanning"] = {"frames": len(frames), "frame_ms_median": float(np.median(wall)),
                         "frame_ms_p95": float(np.percentile(wall, 95)), "success_rate": float(np.mean(ok)),
                         "api": "prrtc_scene_update + prrtc_plan per frame (host wall clock), workers = 0",
                         "obstacles": "3 spheres r=0.05 moving 1 cm/frame through a table_pick scene"}
    return out


def robot_params(robot, base):
    """Per-robot planner settings of the extras. The reference's default
    dynamic-domain radius (4 delta = 2.0, planner.hpp:37) starves exploration
    in 14-D (uniform samples are almost never within 2.0 of a failed node):
    the reference itself solves ~6% of these Baxter problems with it. Scale
    it with the dimension (4 delta * dof / 7) for the dual-arm robot."""
    import copy
    p = copy.copy(base)
    if robot == "baxter":
        p.dd_radius = 4.0 * p.delta * 14 / 7
    return p


def _stats(ok, cost, res_paths):
    c = [x for x, o in zip(cost, ok) if o]
    return {"success": float(np.mean(ok)) if len(ok) else None,
            "cost_median": float(np.median(c)) if c else None, "cost_mean": float(np.mean(c)) if c else None}


PARITY_SUBSET = {("baxter", 16): 300}  # bounds the reference's 16-thread Baxter arm's time (~0.2 s per problem)


def _z(p1, p2, n1, n2):
    """Two-proportion z score of p1 - p2 (pooled): |z| < 2 is within sampling noise."""
    if p1 is None or p2 is None:
        return None
    p = (p1 * n1 + p2 * n2) / (n1 + n2)
    se = (p * (1 - p) * (1 / n1 + 1 / n2)) ** 0.5
    return (p1 - p2) / se if se > 0 else 0.0


def parity_block(robot_names, workers_list, n, device=0, tree_capacity=200000, threads=None, subset=None):
    """Equal-budget statistical parity (north_star: success no lower than the
    reference's, initial path cost reported alongside; every returned path
    re-validated by the reference checker). Per robot and W: the B200 batch
    and the reference planner (oracle/_ref, the unmodified sources) run the
    SAME problems at IDENTICAL PlannerParams — workers = W, so both get the
    iteration budget max_iters_per_worker x W (planner.cpp:199,287-288) —
    and the reference checker re-validates every returned path of both at
    n_cc and at 4 n_cc (fine only, early exit off). The B200
    arm also runs in sound mode (validate_path). Untimed by the driver:
    correctness evidence beside the headline."""
    from paper_2503_06757_b200 import planner
    from paper_2503_06757_b200.model import PlannerParams, PlanStatus
    threads = threads or os.cpu_count() or 1
    out = {"params": "reference defaults (delta 0.5, n_cc 32, max_iters_per_worker 2000, dynamic domain, "
                     "two-stage, early exit, Halton) with workers = W on both arms",
           "tree_capacity": tree_capacity, "host_threads": threads, "robots": {}}
    o = None
    subset = PARITY_SUBSET if subset is None else subset
    for robot in robot_names:
        model, scenes_all, S_all, G_all, kinds = load_workload(robot, n)
        dsc_all = planner.device_scenes(scenes_all, device)
        rr = {"problems": len(S_all)}
        for W in workers_list:
            k = min(len(S_all), subset.get((robot, W), len(S_all)))
            idx = np.unique(np.linspace(0, len(S_all) - 1, k).round().astype(int))
            scenes, S, G = [scenes_all[i] for i in idx], S_all[idx], G_all[idx]
            dsc = planner.device_scenes(scenes, device) if k < len(S_all) else dsc_all
            params = robot_params(robot, PlannerParams(workers=W, tree_capacity=tree_capacity))
            planner.plan_batch_arrays(model, dsc.hs[:8], S[:8], G[:8], params, device=device)  # workspace warm-up
            t0 = time.perf_counter()
            br = planner.plan_batch_arrays(model, dsc, S, G, params, device=device)
            g_ms = (time.perf_counter() - t0) * 1e3
            sound = robot_params(robot, PlannerParams(workers=W, tree_capacity=tree_capacity, validate_path=True))
            t0 = time.perf_counter()
            bs = planner.plan_batch_arrays(model, dsc, S, G, sound, device=device)
            s_ms = (time.perf_counter() - t0) * 1e3
            if o is None:
                from oracle import Oracle, available
                o = Oracle("ref" if available("ref") else "port")
                out["reference_kind"] = o.kind
            rth = max(1, threads // W)  # W threads per problem, problems side by side
            t0 = time.perf_counter()
            ref, _ = o.plan_many(model, scenes, S, G, params, threads=rth)
            r_ms = (time.perf_counter() - t0) * 1e3
            g_ok = br.status == PlanStatus.Solved
            r_ok = np.array([r.status == PlanStatus.Solved for r in ref])
            g_paths = [p for p, k in zip(br.paths, g_ok) if k]
            r_paths = [r.path for r in ref if r.status == PlanStatus.Solved]
            g_sc = [s for s, k in zip(scenes, g_ok) if k]
            r_sc = [s for s, k in zip(scenes, r_ok) if k]
            nc = params.n_cc

            def valid(sc, ps, m):
                return float(np.mean(o.paths_valid(model, sc, ps, m, threads=threads))) if ps else None
            both = g_ok & r_ok
            row = {
                "b200": {**_stats(g_ok, br.cost, None), "valid_ncc": valid(g_sc, g_paths, nc),
                         "valid_4ncc": valid(g_sc, g_paths, 4 * nc),
                         "iterations_mean": float(np.mean(br.iterations_total)),
                         "problems_per_s_e2e": len(S) / (g_ms / 1e3)},
                "b200_sound": {**_stats(bs.status == PlanStatus.Solved, bs.cost, None),
                               "valid_4ncc_device": float(np.mean(bs.path_check[bs.status == PlanStatus.Solved] == 1))
                               if (bs.status == PlanStatus.Solved).any() else None,
                               "problems_per_s_e2e": len(S) / (s_ms / 1e3)},
                "reference": {**_stats(r_ok, [r.cost for r in ref], None), "valid_ncc": valid(r_sc, r_paths, nc),
                              "valid_4ncc": valid(r_sc, r_paths, 4 * nc),
                              "iterations_mean": float(np.mean([r.iterations_total for r in ref])),
                              "problems_per_s": len(S) / (r_ms / 1e3), "threads_per_problem": W,
                              "problems_in_parallel": rth},
                "both_solved": int(both.sum()),
                "cost_mean_both_solved": {"b200": float(np.mean(br.cost[both])) if both.any() else None,
                                          "reference": float(np.mean([r.cost for r, b in zip(ref, both) if b]))
                                          if both.any() else None},
                "dd_radius": params.resolved_dd_radius(),
                "problems": len(S),
            }
            if W == 1:
                # exact mode: max_workers_per_problem = 1 keeps every problem on one
                # worker (no help joins), which is the reference's workers=1 search
                # itself: same Halton stream, same accept loop, exact FP64 nodes —
                # so status, iteration count and path match problem by problem
                # (up to an FP32-FK verdict within ~1e-6 m of a contact)
                exact = robot_params(robot, PlannerParams(workers=1, tree_capacity=tree_capacity,
                                                          max_workers_per_problem=1))
                t0 = time.perf_counter()
                be = planner.plan_batch_arrays(model, dsc, S, G, exact, device=device)
                e_ms = (time.perf_counter() - t0) * 1e3
                e_ok = be.status == PlanStatus.Solved
                e_paths = be.paths
                # the reference arm above uses its default kernel dispatch (AVX2),
                # whose sq_distance summation order differs from the scalar one in
                # the last bits; the device follows the scalar
                # order, so the bitwise path identity is taken against a
                # scalar-backend reference run (kernels.hpp:109 force_backend)
                o.force_scalar(True)
                try:
                    ref_s, _ = o.plan_many(model, scenes, S, G, params, threads=threads)
                finally:
                    o.force_scalar(False)

                def same_as(rs, paths_too):
                    return sum(1 for i, r in enumerate(rs)
                               if int(be.status[i]) == int(r.status) and int(be.iterations_total[i]) == r.iterations_total
                               and (not paths_too or r.status != PlanStatus.Solved or np.array_equal(e_paths[i], r.path)))
                same = same_as(ref_s, True)
                row["b200_exact"] = {**_stats(e_ok, be.cost, None),
                                     "iterations_mean": float(np.mean(be.iterations_total)),
                                     "identical_to_reference": same,
                                     "identical_to": "reference plan() workers=1, scalar backend: status, "
                                                     "iterations and path bitwise",
                                     "status_and_iterations_equal_default_backend": same_as(ref, False),
                                     "problems_per_s_e2e": len(S) / (e_ms / 1e3),
                                     "max_workers_per_problem": 1}
            if W > 1:
                # single-problem mode: prrtc_plan puts W CTAs on the problem at once,
                # W concurrent workers like the reference's W threads (the batch
                # arm above shares its CTAs elastically over 1000 problems, so a
                # problem there mostly runs as one worker with the W-fold budget)
                t0 = time.perf_counter()
                sr = [planner.plan(model, dsc.hs[i], S[i], G[i], params, device=device) for i in range(len(S))]
                p_ms = (time.perf_counter() - t0) * 1e3
                s_ok = np.array([r.status == PlanStatus.Solved for r in sr])
                s_paths = [r.path for r in sr if r.status == PlanStatus.Solved]
                s_sc = [sc for sc, k in zip(scenes, s_ok) if k]
                row["b200_single"] = {**_stats(s_ok, [r.cost for r in sr], None),
                                      "valid_ncc": valid(s_sc, s_paths, nc), "valid_4ncc": valid(s_sc, s_paths, 4 * nc),
                                      "iterations_mean": float(np.mean([r.iterations_total for r in sr])),
                                      "problems_per_s_e2e": len(S) / (p_ms / 1e3), "ctas_per_problem": W}
            row["success_not_below_reference"] = row["b200"]["success"] >= row["reference"]["success"]
            row["success_z_b200_minus_ref"] = _z(row["b200"]["success"], row["reference"]["success"], len(S), len(S))
            if "b200_single" in row:
                row["success_z_single_minus_ref"] = _z(row["b200_single"]["success"], row["reference"]["success"],
                                                       len(S), len(S))
            rr[f"W{W}"] = row
        out["robots"][robot] = rr
    return out


def planners_block(dev, peak=None):
    """The two device planners on the same device-resident batches at the
    headline params: CTA workers (the default, plan_kernel)
    and warp workers (threads_per_cta = 32, plan_warp_kernel); kernel time by
    CUDA events on the launching stream (best of 3 after a warm-up)."""
    import torch
    from paper_2503_06757_b200 import planner
    from paper_2503_06757_b200.model import PlanStatus
    out = {}
    st = torch.cuda.Stream(device=dev)
    for robot, n in (("panda", 1000), ("fetch", 1000), ("fetch", 10000)):
        model, scenes, S, G, _ = load_workload(robot, 1000)
        ds = [planner.device_scene(s, dev) for s in scenes]
        idx = np.arange(n) % len(S)
        row = {}
        for name, nt in (("cta", 128), ("warp", 32)):  # (0 would be the automatic choice between them)
            b = planner.Batch(model, [ds[i] for i in idx], S[idx], G[idx],
                              robot_params(robot, headline_params(threads_per_cta=nt)), device=dev)
            ms = []
            for rep in range(4):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                b.launch(st.cuda_stream)
                e1.record(st)
                st.synchronize()
                ms.append(e0.elapsed_time(e1))
            res = b.results()
            ok = np.mean([r.status == PlanStatus.Solved for r in res])
            tf = float(sum(r.flops for r in res)) / (ms[-1] * 1e-3) / 1e12  # the last launch's counted flops
            row[name] = {"kernel_ms": min(ms[1:]), "problems_per_s": n / (min(ms[1:]) / 1e3), "success": float(ok),
                         "achieved_tflops": tf, "fp32_frac": tf / peak if peak else None}
            del b
        out[f"{robot}_{n}"] = row
    return out


def mixed_sharded(dev, world, rank, total=10000):
    """BASELINE config 5: a 10k-problem mixed three-robot batch (1/3 per
    robot) sharded round robin across the ranks (one GPU each, no data-path
    collective). Each rank solves its share as three device batches on three
    streams (tree_capacity 20000 so the resident problems fit in HBM); the
    time is the host wall clock from a barrier to the rank's sync, max over
    ranks; problems/s is whole-job."""
    import torch
    from paper_2503_06757_b200 import planner
    from paper_2503_06757_b200.model import PlannerParams, PlanStatus
    mp = headline_params()  # workers = 1, tree_capacity 20000: the headline's params
    per = (total - 2 * (total // 3), total // 3, total // 3)
    batches, streams, mine = [], [], 0
    for robot, n in zip(("panda", "fetch", "baxter"), per):
        model, scenes, S, G, _ = load_workload(robot, 1000)
        idx = [i % len(S) for i in shard(n, world, rank)]
        mine += len(idx)
        batches.append(planner.Batch(model, [scenes[i] for i in idx], S[idx], G[idx],
                                     robot_params(robot, mp), device=dev))
        streams.append(torch.cuda.Stream(device=dev))
    for b, st in zip(batches, streams):  # warm (workspace, first-touch)
        b.launch(st.cuda_stream)
    torch.cuda.synchronize()
    dist_barrier(world)
    t0 = time.perf_counter()
    for b, st in zip(batches, streams):
        b.launch(st.cuda_stream)
    torch.cuda.synchronize()
    ms = dist_max((time.perf_counter() - t0) * 1e3, world)
    ok = sum(r.status == PlanStatus.Solved for b in batches for r in b.results())
    solved, count = dist_sum(float(ok), world), dist_sum(float(mine), world)
    del batches
    return {"problems": int(count), "problems_per_s": count / (ms / 1e3), "ms": ms,
            "success_rate": solved / count, "params": "headline (workers 1, tree_capacity 20000)", "n_gpus": world,
            "sharding": "round robin over ranks, no collective on the data path",
            "timing": "host wall clock, barrier -> three concurrent stream launches + sync, max over ranks"}


HEADLINE_WORKERS = 1  # workers per problem on BOTH arms (identical PlannerParams)


HEADLINE_CAPACITY = 20000  # right-sized (both arms); the default 200000 is reported beside it


def headline_params(**kw):
    """The headline's PlannerParams, identical on both arms: the reference
    defaults (planner.hpp:21-40) with workers = 1 (per-problem iteration budget
    max_iters_per_worker x 1 = 2000, planner.cpp:199) and tree_capacity 20000
    (ample for 2000 iterations; the reference allocates its trees inside the
    timed plan() call, planner.cpp:254,290-291, so the default 200000 would
    mostly time that allocation — its figures are reported alongside)."""
    from paper_2503_06757_b200.model import PlannerParams
    kw.setdefault("tree_capacity", HEADLINE_CAPACITY)
    return PlannerParams(workers=HEADLINE_WORKERS, **kw)


def problem_set(robot: str, rank: int, n: int):
    """Rank r's problems: set 0 = tests/golden/problems_<robot>.npz, set r >= 1 =
    problems_<robot>_s<r>.npz (disjoint problem ids, same scene-kind mix), so
    the weak-scaling job solves distinct problems on every GPU. Falls back to
    set 0 (noted in the config) when a set is not generated."""
    if rank > 0 and (ROOT / "tests" / "golden" / f"problems_{robot}_s{rank}.npz").exists():
        return load_workload(robot, n, set_k=rank), f"set {rank}"
    return load_workload(robot, n), "set 0" + (" (replica: no distinct set generated)" if rank else "")


def lscpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _lat(vals):
    v = [x for x in vals if x is not None]
    return {"median": float(np.median(v)) if v else None, "p95": float(np.percentile(v, 95)) if v else None,
            "n": len(v)}


def cpu_baseline_block(model, scenes, S, G, kinds, gpu_single=None):
    """SURVEY.md §8(d) / BASELINE.md §3 CPU-baseline protocol on the box's host
    cores, reference = oracle/_ref (the unmodified reference sources):
    throughput (nproc threads, workers = 1 per problem) at tree_capacity 200000
    (the default; its allocation is inside the reference's timer,
    planner.cpp:254,290-291) and at the right-sized 20000; single-problem
    latency (the reference's own wall_time_ms, one problem at a time) at
    workers = 1 and workers = nproc on a 200-problem spread sample at both
    capacities; BASELINE config 1 (one Panda table_pick problem, seed 0)."""
    from oracle import Oracle, available
    from paper_2503_06757_b200.model import PlannerParams, PlanStatus
    threads = os.cpu_count() or 1
    o = Oracle("ref" if available("ref") else "port")
    n = len(S)
    out = {"kind": "reference" if o.kind == "ref" else "port", "cores": threads, "cpu_model": lscpu_model()}
    for cap in (200000, 20000):
        p = PlannerParams(workers=1, tree_capacity=cap)
        res, ms = o.plan_many(model, scenes, S, G, p, threads=threads)
        ok = [r.status == PlanStatus.Solved for r in res]
        out[f"throughput_cap{cap}"] = {
            "problems_per_s": n / (ms / 1e3), "success": float(np.mean(ok)),
            "cost_mean": float(np.mean([r.cost for r in res if r.status == PlanStatus.Solved])),
            "sample": f"all {n} problems, workers=1 per problem, {threads} problems in parallel"}
    sub = np.unique(np.linspace(0, n - 1, min(n, 200)).round().astype(int))
    for W in (1, threads):
        for cap in (200000, 20000):
            p = PlannerParams(workers=W, tree_capacity=cap)
            res, _ = o.plan_many(model, [scenes[i] for i in sub], S[sub], G[sub], p, threads=1)
            ok = [r.status == PlanStatus.Solved for r in res]
            out[f"latency_w{W}_cap{cap}"] = {
                **_lat([r.wall_time_ms for r in res if r.status == PlanStatus.Solved]),
                "success": float(np.mean(ok)),
                "cost_mean": float(np.mean([r.cost for r in res if r.status == PlanStatus.Solved])),
                "sample": f"{len(sub)} problems spread over the set, one at a time, reference wall_time_ms"}
    # BASELINE config 1: Panda table_pick, seed 0 (problem 0 of the set), 20 trials per arm
    i0 = int(np.where(kinds == "table_pick")[0][0])
    c1 = {"problem": f"{kinds[i0]} index {i0}", "seed": 0}
    for W in (1, threads):
        p = PlannerParams(workers=W)
        rs = [o.plan(model, scenes[i0], S[i0], G[i0], p) for _ in range(20)]
        c1[f"reference_w{W}"] = {**_lat([r.wall_time_ms for r in rs if r.status == PlanStatus.Solved]),
                                 "success": float(np.mean([r.status == PlanStatus.Solved for r in rs])),
                                 "cost_mean": float(np.mean([r.cost for r in rs if r.status == PlanStatus.Solved]))
                                 if any(r.status == PlanStatus.Solved for r in rs) else None}
    if gpu_single is not None:
        c1.update(gpu_single(i0))
    out["config1"] = c1
    return out


def run_reference(args):
    """--impl reference: the reference's own CPU planner (oracle/_ref) on the
    host cores, on the headline's workload, metric and PlannerParams. Under
    torchrun only rank 0 runs; the others exit without work."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2503_06757_b200.model import PlanStatus
    model, scenes, S, G, kinds = load_workload(args.robot, args.problems)
    params = headline_params()
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference(model, scenes[:64], S[:64], G[:64], params, threads)
    times, solved, lat, cost = [], [], [], []
    kind = None
    for _ in range(args.steps):
        o, kind, res, ms = cpu_reference(model, scenes, S, G, params, threads)
        times.append(ms)
        solved.append(np.mean([r.status == PlanStatus.Solved for r in res]))
        lat += [r.wall_time_ms for r in res if r.status == PlanStatus.Solved]
        cost += [r.cost for r in res if r.status == PlanStatus.Solved]
    ms = statistics.median(times)
    value = len(S) / (ms / 1e3)
    # the reference's default tree capacity (its allocation is inside plan())
    r20, ms20 = o.plan_many(model, scenes, S, G, headline_params(tree_capacity=200000), threads=threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.robot, len(S), params, args.gpus),
        "success_rate": float(np.mean(solved)), "mean_cost": float(np.mean(cost)),
        "host_threads": threads, "cpu_model": lscpu_model(),
        "tree_capacity_200000": {"problems_per_s": len(S) / (ms20 / 1e3),
                                 "success_rate": float(np.mean([r.status == PlanStatus.Solved for r in r20]))},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"all {len(S)} problems x {args.steps} steps, workers=1 per problem, "
                                   f"{threads} problems in parallel"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "latency_ms": {**_lat(lat), "note": "reference wall_time_ms of each problem inside the "
                                            f"{threads}-thread throughput run (workers=1)"},
    }
    print(json.dumps(line))
    return 0


def table_one(dev, robot, params_fn, n_lat, peak):
    """Table-I figures of one robot (statistics as
    bench.cpp:90-109): single-problem prrtc_plan latency at the device's
    default worker count (one 512-thread CTA per SM) on a spread sample, its
    success and cost, and the FP32 roofline fraction of plan_kernel over those
    launches (algorithmic flops / device time); plus the 1000-problem batch at
    the headline params (problems/s, success)."""
    import torch
    from paper_2503_06757_b200 import planner, suite
    from paper_2503_06757_b200.model import PlannerParams, PlanStatus
    model, scenes, S, G, kinds = load_workload(robot, 1000)
    out = {"dof": model.dof}
    bp = params_fn(robot, headline_params())
    b = planner.Batch(model, scenes, S, G, bp, device=dev)
    b.launch()
    b.results()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(3):
        e0.record()
        b.launch(torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    res = b.results()
    fl = float(sum(r.flops for r in res))
    out["batch"] = {"problems_per_s": len(S) / (statistics.median(ms) / 1e3),
                    "success_rate": float(np.mean([r.status == PlanStatus.Solved for r in res])),
                    "fp32_frac": fl / (statistics.median(ms) * 1e-3) / 1e12 / peak if peak else None,
                    "params": f"workers={bp.workers}, dd_radius={bp.resolved_dd_radius()}"}
    del b
    sp = params_fn(robot, PlannerParams())  # workers = 0: one CTA per SM
    idx = np.unique(np.linspace(0, len(S) - 1, n_lat).round().astype(int))
    for i in idx[:3]:
        planner.plan(model, scenes[i], S[i], G[i], sp, device=dev)
    rs = [planner.plan(model, scenes[i], S[i], G[i], sp, device=dev) for i in idx]
    ok = [r for r in rs if r.status == PlanStatus.Solved]
    q = suite.summarize_values([r.wall_time_ms for r in ok])
    dsum = sum(r.device_time_ms for r in rs)
    out["single"] = {"median_ms": q.median, "p95_ms": q.p95, "mean_ms": q.mean,
                     "device_median_ms": float(np.median([r.device_time_ms for r in ok])) if ok else None,
                     "success_rate": len(ok) / len(rs), "cost_mean": float(np.mean([r.cost for r in ok])) if ok else None,
                     "fp32_frac": (sum(r.flops for r in rs) / (dsum * 1e-3) / 1e12 / peak) if dsum and peak else None,
                     "samples": len(rs), "workers": planner.default_workers(dev),
                     "params": f"workers=0 (budget {planner.default_workers(dev)} x 2000), "
                               f"dd_radius={sp.resolved_dd_radius()}"}
    if robot == "baxter":  # also at the reference's default dynamic-domain radius (4 delta)
        from paper_2503_06757_b200.model import PlannerParams as PP
        b = planner.plan_batch_arrays(model, planner.device_scenes(scenes, dev), S, G, headline_params(), device=dev)
        out["batch_reference_dd"] = {"success_rate": float(np.mean(b.status == PlanStatus.Solved)),
                                     "dd_radius": PP().resolved_dd_radius()}
    return out


def run_b200(args):
    import torch
    # one GPU per rank (ranks beyond the visible GPUs share them: functional runs only)
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count()))
    world, rank, local = dist_setup()
    from paper_2503_06757_b200 import _lib, planner
    from paper_2503_06757_b200.model import PlannerParams, PlanStatus
    from paper_2503_06757_b200.planner import Batch

    dev = local % max(1, torch.cuda.device_count())
    (model, scenes, S, G, kinds), set_name = problem_set(args.robot, rank, args.problems)
    n = len(S)
    params = headline_params()
    batch = Batch(model, scenes, S, G, params, device=dev)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{dev}")
    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            batch.launch(stream.cuda_stream)
        stream.synchronize()
    batch.results()
    # ---- timed region: K steps, L2 flushed between steps (untimed) ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    dist_barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                flush.zero_()
                ev[k][0].record(stream)
                batch.launch(stream.cuda_stream)
                ev[k][1].record(stream)
        torch.cuda.synchronize()
    dist_barrier(world)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    res = batch.results()  # last step's outcome (copied after the timed region)
    ms = dist_max(sum(step_ms) / len(step_ms), world)
    total_n = dist_sum(float(n), world)  # problems of the whole job (every rank's own set)
    value = total_n / (ms / 1e3)
    solved = [r.status == PlanStatus.Solved for r in res]
    flops = float(sum(r.flops for r in res))
    del batch

    # ---- e2e through the host-buffer C-ABI (prrtc_plan_batch), every rank,
    # barrier + max over ranks (whole-job problems/s) ----
    # setup: robot and scene handles uploaded once — a call
    # then costs the inputs' H2D, the kernel, the results' D2H and unpacking
    # (passing the RobotModel itself would re-fingerprint it, ~0.12 ms of
    # Python per call, to catch mutation)
    drob = planner.device_robot(model, dev)
    dscenes = planner.device_scenes(scenes, dev)
    planner.plan_batch_arrays(drob, dscenes, S, G, params, device=dev)  # workspace warm
    e2e_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        dist_barrier(world)
        t0 = time.perf_counter()
        er = planner.plan_batch_arrays(drob, dscenes, S, G, params, device=dev)
        e2e_ms.append(dist_max((time.perf_counter() - t0) * 1e3, world))
    e2e_solved = dist_sum(float(np.sum(er.status == PlanStatus.Solved)), world) / total_n
    # sound mode (validate_path: every path re-checked on the device at 4 n_cc, failures re-planned)
    sp = headline_params(validate_path=True)
    for _ in range(3):  # warm-up: re-plans grow the pinned path-block pool once
        planner.plan_batch_arrays(drob, dscenes, S, G, sp, device=dev)
    s_ms = []
    for _ in range(9):  # re-plans of rejected paths make single calls noisy (1.9-5.6 ms): median of 9
        dist_barrier(world)
        t0 = time.perf_counter()
        sr = planner.plan_batch_arrays(drob, dscenes, S, G, sp, device=dev)
        s_ms.append(dist_max((time.perf_counter() - t0) * 1e3, world))
    s_solved = dist_sum(float(np.sum(sr.status == PlanStatus.Solved)), world) / total_n
    mixed = None if args.no_extras else mixed_sharded(dev, world, rank)

    if rank == 0:
        lib = _lib.load()
        peak = lib.prrtc_fp32_peak_tflops(dev)
        kernel_ms = statistics.median(step_ms)
        achieved = flops / (kernel_ms * 1e-3) / 1e12
        import ctypes
        h2d_c, d2h_c = ctypes.c_uint64(), ctypes.c_uint64()
        planner.plan_batch_arrays(drob, dscenes, S, G, params, device=dev)  # the e2e call, for its byte count
        _lib.check(lib.prrtc_last_transfer_bytes(dev, ctypes.byref(h2d_c), ctypes.byref(d2h_c)))
        # ---- single-problem latency (prrtc_plan, host wall clock), per worker count ----
        from paper_2503_06757_b200 import suite
        idx = np.unique(np.linspace(0, n - 1, args.latency_samples).round().astype(int))
        lat = {}
        for W in (0, 16, 1):
            lp = PlannerParams(workers=W)
            for i in idx[:3]:
                planner.plan(model, scenes[i], S[i], G[i], lp, device=dev)
            rs = [planner.plan(model, scenes[i], S[i], G[i], lp, device=dev) for i in idx]
            ok = [r for r in rs if r.status == PlanStatus.Solved]
            q = suite.summarize_values([r.wall_time_ms for r in ok])  # Table-I statistics (bench.cpp:90-109)
            dsum = sum(r.device_time_ms for r in rs)
            lat[f"workers{W}"] = {
                "median": q.median, "p95": q.p95, "mean": q.mean, "q1": q.q1, "q3": q.q3,
                "device_median": float(np.median([r.device_time_ms for r in ok])) if ok else None,
                "success_rate": len(ok) / len(rs), "cost_mean": float(np.mean([r.cost for r in ok])) if ok else None,
                "fp32_frac": (sum(r.flops for r in rs) / (dsum * 1e-3) / 1e12 / peak) if dsum and peak else None,
                "ctas": planner.default_workers(dev) if W == 0 else W, "samples": len(rs)}

        def gpu_single(i0):
            out = {}
            for W in (1, 16, 0):
                lp = PlannerParams(workers=W)
                planner.plan(model, scenes[i0], S[i0], G[i0], lp, device=dev)
                rs = [planner.plan(model, scenes[i0], S[i0], G[i0], lp, device=dev) for _ in range(20)]
                out[f"b200_w{W}"] = {**_lat([r.wall_time_ms for r in rs if r.status == PlanStatus.Solved]),
                                     "success": float(np.mean([r.status == PlanStatus.Solved for r in rs]))}
            return out

        extras = {}
        if not args.no_extras:
            extras["robots"] = {r: table_one(dev, r, robot_params, 100, peak) for r in ("panda", "fetch", "baxter")}
            extras.update(bench_extras(dev, params))
            extras["planners"] = planners_block(dev, peak)
        micro = microbench(model, scenes, S, G, dev, peak)
        parity = None
        if not args.no_parity:
            parity = parity_block(["panda", "fetch", "baxter"], [1, 16], args.parity_problems, device=dev)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": workload_config(args.robot, n, params, world),
            "problem_sets": f"rank r solves its own {n}-problem set ({world} sets, rank 0: {set_name})",
            "success_rate": float(np.mean(solved)),
            "mean_cost": float(np.mean([r.cost for r in res if r.status == PlanStatus.Solved])),
            "e2e": {"value": total_n / (statistics.median(e2e_ms) / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d_c.value), "d2h_bytes_per_step": int(d2h_c.value),
                    "success_rate": float(e2e_solved),
                    "api": "prrtc_plan_batch (host buffers), every rank, max over ranks"},
            "sound_mode": {"problems_per_s_e2e": total_n / (statistics.median(s_ms) / 1e3),
                           "success_rate": float(s_solved),
                           "calls_ms": [round(x, 3) for x in s_ms],
                           "api": "prrtc_plan_batch, params.validate_path = 1 (every path re-checked on the "
                                  "device at 4 n_cc, failures re-planned)"},
            "roofline": {"bound": "fp32", "kernel": "plan_kernel", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "peak_source": "measured FFMA-chain microbenchmark (prrtc_fp32_peak_tflops); "
                                        "MEASURED_PEAKS.json has no FP32 figure",
                         "algorithmic_flops_per_launch": flops, "traffic": traffic_from_profiles(),
                         "ncu": {k.replace("plan_kernel_", ""): v for k, v in ncu_summary().items()
                                 if k.startswith("plan_kernel_") and k != "plan_kernel_dram_bytes_per_launch"},
                         "ncu_source": ncu_summary().get("source")},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "microbench": micro,
            **extras,
        }
        if mixed is not None:
            line["mixed_10k"] = mixed
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline_block(model, scenes, S, G, kinds, gpu_single)
            t = cb[f"throughput_cap{HEADLINE_CAPACITY}"]
            line["cpu_baseline"] = {"value": t["problems_per_s"], "unit": UNIT, "cores": cb["cores"],
                                    "kind": cb["kind"], "sample": t["sample"], **cb}
        if parity is not None:
            line["parity"] = parity
            line["parity_summary"] = {
                f"{r}_W{w}": {"success_b200": v[f"W{w}"]["b200"]["success"],
                              "success_ref": v[f"W{w}"]["reference"]["success"],
                              "success_b200_single": v[f"W{w}"].get("b200_single", {}).get("success"),
                              "success_b200_exact": v[f"W{w}"].get("b200_exact", {}).get("success"),
                              "identical_to_reference": v[f"W{w}"].get("b200_exact", {}).get("identical_to_reference"),
                              "z_batch": v[f"W{w}"]["success_z_b200_minus_ref"],
                              "z_single": v[f"W{w}"].get("success_z_single_minus_ref"),
                              "problems": v[f"W{w}"]["problems"],
                              "cost_med_b200_single": v[f"W{w}"].get("b200_single", {}).get("cost_median"),
                              "cost_med_b200": v[f"W{w}"]["b200"]["cost_median"],
                              "cost_med_ref": v[f"W{w}"]["reference"]["cost_median"],
                              "valid_ncc": [v[f"W{w}"]["b200"]["valid_ncc"], v[f"W{w}"]["reference"]["valid_ncc"]],
                              "valid_4ncc": [v[f"W{w}"]["b200"]["valid_4ncc"], v[f"W{w}"]["reference"]["valid_4ncc"]]}
                for r, v in parity["robots"].items() for w in (1, 16)}
        line["latency_ms"] = {**lat["workers0"], "by_workers": lat,
                              "api": "prrtc_plan, host wall clock; workers0 = one 512-thread CTA per SM"}
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--robot", default="panda")
    ap.add_argument("--problems", type=int, default=1000)
    ap.add_argument("--latency-samples", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the Fetch/Baxter/mixed/replanning extras")
    ap.add_argument("--no-parity", action="store_true", help="skip the equal-budget parity block")
    ap.add_argument("--parity-problems", type=int, default=1000)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
