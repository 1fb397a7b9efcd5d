"""The persistent planner kernel against the reference planner.

Random trees cannot be bit-reproduced under parallel insertion, so the bar is
statistical (BASELINE.json north_star): every returned path re-validates
collision-free with the reference checker at 4 x n_cc, fine-only, early exit
off, success rate >= the reference's on the same problems, and
the deterministic single-CTA mode replays the reference's workers=1 run.
"""
import numpy as np
import pytest

from conftest import load_problems
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.model import PlannerParams, PlanStatus
from paper_2503_06757_b200.scenes import make_scene

pytestmark = pytest.mark.gpu


def dump_failure(m, scene, P, params, tag):
    """Save a failing path (gpurun_out/ is merged back) with per-edge verdicts."""
    import pickle
    from pathlib import Path
    out = Path(__file__).resolve().parents[1] / "gpurun_out"
    out.mkdir(exist_ok=True)
    dev32 = planner.validate_edges(m, scene, P[:-1], P[1:], params.n_cc)
    with open(out / f"fail_{tag}.pkl", "wb") as f:
        pickle.dump({"model": m.name, "scene": scene, "path": P, "dev32": dev32}, f)
    return dev32


def check_path(oracle, m, scene, res, start, goal, params, strict4=True):
    """The path is sound at the planner's resolution (every edge re-validates
    with the reference checker at n_cc, fine-only, early exit off — what the
    reference planner itself guarantees) and, when strict4, at 4 x n_cc
    (SPEC.md:367). Returns whether the 4 x n_cc check passed."""
    assert res.status == PlanStatus.Solved
    P = res.path
    assert P.shape[1] == m.dof and len(P) >= 1
    assert np.array_equal(P[0], start) and np.array_equal(P[-1], goal)
    if len(P) > 1:
        ok32 = oracle.validate_edges(m, scene, P[:-1], P[1:], params.n_cc, False, False)
        assert ok32.all(), f"path fails the reference checker at n_cc: {ok32.tolist()}"
    ok4 = oracle.path_valid(m, scene, P, 4 * params.n_cc)
    if strict4 and not ok4:
        dev32 = dump_failure(m, scene, P, params, f"{m.name}_{scene.name}")
        ref32 = oracle.validate_edges(m, scene, P[:-1], P[1:], params.n_cc, False, False)
        ref128 = oracle.validate_edges(m, scene, P[:-1], P[1:], 4 * params.n_cc, False, False)
        raise AssertionError(f"path fails 4x re-validation: device@n_cc {dev32.tolist()} "
                             f"oracle@n_cc {ref32.tolist()} oracle@4n_cc {ref128.tolist()}")
    if len(P) > 1:
        seg = np.linalg.norm(np.diff(P, axis=0), axis=1)
        assert np.all(seg > 0) and np.all(seg <= params.delta + 1e-9)
        assert abs(res.cost - seg.sum()) < 1e-9
    return ok4


def not_below(ok, ok_ref, n):
    """Success no lower than the reference's (north_star), at equal budgets, up
    to sampling noise: the two-proportion 2-sigma band of n problems. The
    full 1000-problem sets are compared in bench.py's parity block."""
    p = max(ok, ok_ref) / n
    return ok / n >= ok_ref / n - 2.0 * np.sqrt(max(p * (1 - p), 1.0 / n) * 2.0 / n)


@pytest.mark.parametrize("robot", ["panda", "fetch", "baxter"])
def test_plan_paths_revalidate(gpu, oracle, robot):
    """Single-problem mode at the reference's budget: W = 16 CTAs on the
    problem, budget 16 x max_iters_per_worker, against the reference with
    workers = 16 (planner.cpp:199,287-288). Every path sound at n_cc (the
    reference planner's own guarantee) and >= 90% at 4 x n_cc (edges are
    checked at n_cc samples, so a contact between two samples can slip
    through — for the reference too). Sound mode (validate_path): every path
    sound at 4 x n_cc."""
    m = robots.get(robot)
    params = PlannerParams(workers=16)  # reference defaults otherwise (planner.hpp:21-40)
    sound = PlannerParams(workers=16, validate_path=True)
    probs = load_problems(robot, 1000)[::40]  # 25 problems spread over the scene kinds
    solved = solved_ref = 0
    ok4 = []
    for kind, pid, s, g in probs:
        scene, _ = make_scene(robot, kind, pid)
        r = planner.plan(m, scene, s, g, params)
        assert r.status in (PlanStatus.Solved, PlanStatus.Failed)
        assert r.iterations_total <= 16 * params.max_iters_per_worker + 64  # (ticket blocks in flight)
        if r.status == PlanStatus.Solved:
            solved += 1
            ok4.append(check_path(oracle, m, scene, r, s, g, params, strict4=False))
        rs = planner.plan(m, scene, s, g, sound)
        if rs.status == PlanStatus.Solved:
            assert rs.path_check == 1
            check_path(oracle, m, scene, rs, s, g, sound, strict4=True)
        ref = oracle.plan(m, scene, s, g, params)
        solved_ref += ref.status == PlanStatus.Solved
    assert not_below(solved, solved_ref, len(probs)), (solved, solved_ref)
    assert np.mean(ok4) >= 0.9, f"4 x n_cc soundness {np.mean(ok4):.2f}"


def test_batch_success_not_below_reference(gpu, oracle):
    """Batch mode at the reference's budget (workers = 1: 2000 iterations per
    problem on both planners), 300 problems spread over the scene kinds."""
    m = robots.get("panda")
    probs = load_problems("panda", 1000)[::3][:300]
    scenes = [make_scene("panda", k, p)[0] for k, p, _, _ in probs]
    S = np.array([p[2] for p in probs])
    G = np.array([p[3] for p in probs])
    params = PlannerParams(workers=1, tree_capacity=20000)
    res = planner.plan_batch(m, scenes, S, G, params)
    ref, _ = oracle.plan_many(m, scenes, S, G, params, threads=8)
    ok = sum(r.status == PlanStatus.Solved for r in res)
    ok_ref = sum(r.status == PlanStatus.Solved for r in ref)
    assert not_below(ok, ok_ref, len(probs)), (ok, ok_ref)
    assert all(r.iterations_total <= params.max_iters_per_worker for r in res if r.status != PlanStatus.Solved)
    ok4 = [check_path(oracle, m, sc, r, s, g, params, strict4=False)
           for sc, r, s, g in zip(scenes, res, S, G) if r.status == PlanStatus.Solved]
    assert np.mean(ok4) >= 0.9
    # initial path cost reported alongside: same order as the reference's on the common solved set
    both = [(r.cost, q.cost) for r, q in zip(res, ref) if r.status == q.status == PlanStatus.Solved]
    assert len(both) > 0.5 * len(probs)
    cg, cr = np.mean([b[0] for b in both]), np.mean([b[1] for b in both])
    assert cg <= 1.25 * cr, (cg, cr)
    # sound mode: every returned path passes 4 x n_cc
    sound = PlannerParams(workers=1, tree_capacity=20000, validate_path=True)
    for sc, r, s, g in zip(scenes[:60], planner.plan_batch(m, scenes[:60], S[:60], G[:60], sound), S, G):
        if r.status == PlanStatus.Solved:
            check_path(oracle, m, sc, r, s, g, sound, strict4=True)


@pytest.mark.parametrize("robot,threads", [("panda", 0), ("panda", 32), ("fetch", 0), ("fetch", 32)])
def test_batch_one_worker_per_problem_replays_reference(gpu, oracle, robot, threads):
    """A batch with workers = 1 and max_workers_per_problem = 1 (no help
    joins) runs, in ONE launch, each problem's reference workers=1 search:
    one worker draws Halton indices 1 + seed + k in order (planner.cpp:192-
    193), the multi-sample NN pass equals the sequential accept loop, tree
    nodes are the exact FP64 checked configs — so status, iteration count
    and the path itself equal the reference's, problem by problem, on both
    device planners (CTA workers, threads 0; warp workers, threads 32). The
    reference runs its scalar backend (its AVX2 sq_distance sums in another
    order, kernels_avx2.cpp:26-39; the device follows the scalar order).
    Measured: 1000/1000 identical for each robot on both planners
    (tools/exact_diff.py); the search is deterministic, so the bar is all."""
    m = robots.get(robot)
    probs = load_problems(robot, 1000)[::5]  # 200 problems over the scene kinds
    scenes = [make_scene(robot, k, p)[0] for k, p, _, _ in probs]
    S = np.array([p[2] for p in probs])
    G = np.array([p[3] for p in probs])
    params = PlannerParams(workers=1, tree_capacity=20000, max_workers_per_problem=1, threads_per_cta=threads)
    res = planner.plan_batch(m, scenes, S, G, params)
    ref, _ = oracle.plan_many(m, scenes, S, G, PlannerParams(workers=1, tree_capacity=20000), threads=8)
    same = 0
    for r, q in zip(res, ref):
        if r.status == q.status and r.iterations_total == q.iterations_total and (
                r.status != PlanStatus.Solved or np.array_equal(r.path, q.path)):
            same += 1
    assert same == len(probs), f"{same}/{len(probs)} problems replay the reference"


def test_deterministic_mode_replays_reference(gpu, oracle):
    """One CTA, Halton stride 1, balanced pick: the device replays the
    reference's workers=1 run (scalar backend) node for node, except where an
    FP32-FK verdict differs from the FP64 one within ~1e-6 m of a boundary."""
    m = robots.get("panda")
    probs = load_problems("panda", 30)
    same = 0
    params = PlannerParams(tree_capacity=20000, deterministic=True, workers=1)
    for kind, pid, s, g in probs:
        scene, _ = make_scene("panda", kind, pid)
        r = planner.plan(m, scene, s, g, params)
        ref = oracle.plan(m, scene, s, g, PlannerParams(workers=1, tree_capacity=20000))
        assert r.status == ref.status or r.status == PlanStatus.Solved
        if r.status == ref.status and (r.status != PlanStatus.Solved or np.array_equal(r.path, ref.path)):
            same += 1
            assert r.iterations_total == ref.iterations_total
            # CheckStats follow the reference's counting semantics in this mode
            # (collision.hpp:14-37, collision.cpp:73-84,133,158,179,189)
            assert r.check_stats == ref.check_stats, (kind, pid, r.check_stats, ref.check_stats)
    assert same >= len(probs) * 0.9


@pytest.mark.parametrize("two_stage,early_exit", [(False, True), (True, False), (False, False)])
def test_deterministic_check_stats_variants(gpu, oracle, two_stage, early_exit):
    """CheckStats parity under the CheckOptions variants (brute force, no early
    exit): wherever the deterministic device run replays the reference's
    workers=1 run, sphere_tests / fk_calls / fine_stage_entries are equal."""
    m = robots.get("panda")
    params = PlannerParams(tree_capacity=20000, deterministic=True, workers=1, two_stage=two_stage,
                           early_exit=early_exit)
    same = 0
    probs = load_problems("panda", 1000)[::100]
    for kind, pid, s, g in probs:
        scene, _ = make_scene("panda", kind, pid)
        r = planner.plan(m, scene, s, g, params)
        ref = oracle.plan(m, scene, s, g, PlannerParams(workers=1, tree_capacity=20000, two_stage=two_stage,
                                                        early_exit=early_exit))
        if r.status == ref.status and (r.status != PlanStatus.Solved or np.array_equal(r.path, ref.path)):
            same += 1
            assert r.iterations_total == ref.iterations_total
            assert r.check_stats == ref.check_stats, (kind, pid, r.check_stats, ref.check_stats)
    assert same >= 0.8 * len(probs)


def test_endpoint_statuses(gpu, oracle):
    m = robots.get("panda")
    kind, pid, s, g = load_problems("panda", 1)[0]
    scene, _ = make_scene("panda", kind, pid)
    # start == goal -> Solved, [start], cost 0 (planner.cpp:279-285)
    r = planner.plan(m, scene, s, s)
    assert r.status == PlanStatus.Solved and r.path.shape == (1, m.dof) and r.cost == 0.0
    # out of limits -> InfeasibleEndpoint, start message first (planner.cpp:263-277)
    bad = s.copy()
    bad[0] = 10.0
    r = planner.plan(m, scene, bad, g)
    assert r.status == PlanStatus.InfeasibleEndpoint and "start" in r.message
    r = planner.plan(m, scene, s, bad)
    assert r.status == PlanStatus.InfeasibleEndpoint and "goal" in r.message
    # colliding goal: find a config in collision
    lim = m.limits()
    rng = np.random.default_rng(0)
    for _ in range(1000):
        q = lim[:, 0] + rng.random(m.dof) * (lim[:, 1] - lim[:, 0])
        if not oracle.check_config(m, scene, q):
            break
    r = planner.plan(m, scene, s, q)
    assert r.status == PlanStatus.InfeasibleEndpoint and "goal" in r.message


def test_invalid_arguments_raise(gpu):
    m = robots.get("panda")
    kind, pid, s, g = load_problems("panda", 1)[0]
    scene, _ = make_scene("panda", kind, pid)
    with pytest.raises(ValueError, match="delta"):
        planner.plan(m, scene, s, g, PlannerParams(delta=0.0))
    with pytest.raises(ValueError, match="n_cc"):
        planner.plan(m, scene, s, g, PlannerParams(n_cc=0))
    with pytest.raises(ValueError, match="tree_capacity"):
        planner.plan(m, scene, s, g, PlannerParams(tree_capacity=1))
    with pytest.raises(ValueError, match="dimension"):
        planner.plan(m, scene, s[:3], g)


def test_capacity_exhaustion_fails_cleanly(gpu):
    m = robots.get("panda")
    probs = load_problems("panda")
    kind, pid, s, g = next(p for p in probs if p[0] == "cage")
    scene, _ = make_scene("panda", kind, pid)
    r = planner.plan(m, scene, s, g, PlannerParams(tree_capacity=4))
    assert r.status in (PlanStatus.Solved, PlanStatus.Failed)
    assert r.tree_nodes[0] <= 2 and r.tree_nodes[1] <= 2


@pytest.mark.parametrize("robot", ["panda", "baxter"])
def test_device_path_validation_agrees_with_reference(gpu, oracle, robot):
    """validate_path: the second kernel re-checks every returned path at
    4 x n_cc, fine-only, early exit off; its verdict must
    equal the reference checker's on the same path."""
    m = robots.get(robot)
    probs = load_problems(robot, 40)
    scenes = [make_scene(robot, k, p)[0] for k, p, _, _ in probs]
    S = np.array([p[2] for p in probs])
    G = np.array([p[3] for p in probs])
    params = PlannerParams(tree_capacity=20000, validate_path=True)
    res = planner.plan_batch(m, scenes, S, G, params)
    checked = 0
    for sc, r in zip(scenes, res):
        if r.status == PlanStatus.Solved:
            assert r.path_check in (1, 2)
            assert (r.path_check == 1) == oracle.path_valid(m, sc, r.path, 4 * params.n_cc)
            checked += 1
        else:
            assert r.path_check == 0
    assert checked >= 10
    # single-problem call and the array API carry the verdict too
    r1 = planner.plan(m, scenes[0], S[0], G[0], params)
    assert r1.status != PlanStatus.Solved or r1.path_check == 1
    ba = planner.plan_batch_arrays(m, scenes[:8], S[:8], G[:8], params)
    assert all(c == 1 for c, st in zip(ba.path_check, ba.status) if st == PlanStatus.Solved)
    # pre-packed scene handles (SceneSet) give the same results as the list
    bs = planner.plan_batch_arrays(m, planner.device_scenes(scenes[:8]), S[:8], G[:8],
                                   PlannerParams(tree_capacity=20000, validate_path=True, deterministic=True))
    bl = planner.plan_batch_arrays(m, scenes[:8], S[:8], G[:8],
                                   PlannerParams(tree_capacity=20000, validate_path=True, deterministic=True))
    assert (bs.status == bl.status).all() and np.array_equal(bs.path_data, bl.path_data)
    with pytest.raises(ValueError):
        planner.plan_batch_arrays(m, planner.device_scenes(scenes[:4]), S[:8], G[:8], params)
    # off by default: nothing is checked
    off = PlannerParams(tree_capacity=20000)
    r0 = planner.plan_batch(m, scenes[:4], S[:4], G[:4], off)
    assert all(r.path_check == 0 for r in r0)


def test_replanning_loop_with_scene_updates(gpu, oracle):
    """BASELINE config 5: moving obstacles pushed with prrtc_scene_update
    between plans; every frame's path re-validates in THAT frame's scene."""
    from paper_2503_06757_b200 import replan
    m = robots.get("panda")
    kind, pid, s, g = next(p for p in load_problems("panda", 50) if p[0] == "table_pick")
    static, _ = make_scene("panda", kind, pid)
    params = PlannerParams(tree_capacity=20000)
    frames = replan.run(m, static, s, g, frames=12, obstacles=replan.MovingSpheres(step=0.08), params=params)
    solved = 0
    for f in frames:
        assert len(f.scene.primitives) == len(static.primitives) + 3
        r = f.result
        if r.status == PlanStatus.Solved:
            solved += 1
            check_path(oracle, m, f.scene, r, s, g, params, strict4=False)
        else:
            ref = oracle.plan(m, f.scene, s, g, PlannerParams(workers=1, tree_capacity=20000))
            assert ref.status != PlanStatus.Solved or r.status == PlanStatus.Failed
    assert solved >= 8


@pytest.mark.parametrize("robot", ["panda", "fetch"])
def test_single_problem_result_paths_agree(gpu, oracle, robot, monkeypatch):
    """A single problem's result comes back three ways: published by the
    kernel into mapped host memory (default), the same launch with a mapped
    block too small for the path (PRRTC_MAP_BYTES: publish_result raises the
    flag without the payload, the host copies back), and the plain D2H
    copy-back (PRRTC_NO_MAP). Deterministic mode makes the three runs the
    same search: identical status, path, iterations, FK and fine-stage
    counters; repeated calls on the same workspace stay identical."""
    m = robots.get(robot)
    probs = load_problems(robot, 12)
    params = PlannerParams(deterministic=True, tree_capacity=20000)
    for kind, pid, s, g in probs[:6]:
        scene, _ = make_scene(robot, kind, pid)
        runs = []
        for env in ({}, {"PRRTC_MAP_BYTES": "300"}, {"PRRTC_NO_MAP": "1"}, {}):
            for k in ("PRRTC_MAP_BYTES", "PRRTC_NO_MAP"):
                monkeypatch.delenv(k, raising=False)
            for k, v in env.items():
                monkeypatch.setenv(k, v)
            planner.reload_env()  # the library caches its switches
            runs.append(planner.plan(m, scene, s, g, params))
        for k in ("PRRTC_MAP_BYTES", "PRRTC_NO_MAP"):
            monkeypatch.delenv(k, raising=False)
        planner.reload_env()
        r0 = runs[0]
        for r in runs[1:]:
            assert r.status == r0.status and r.message == r0.message
            assert np.array_equal(r.path, r0.path)
            assert r.iterations_total == r0.iterations_total
            # (deterministic mode counts CheckStats with the reference's
            # semantics, so all three counters repeat exactly)
            assert r.check_stats == r0.check_stats
            assert r.check_stats.fk_calls == r0.check_stats.fk_calls
            assert r.check_stats.fine_stage_entries == r0.check_stats.fine_stage_entries
            assert r.tree_nodes == r0.tree_nodes
        if r0.status == PlanStatus.Solved:
            assert oracle.path_valid(m, scene, r0.path, params.n_cc)


@pytest.mark.parametrize("robot", ["panda", "baxter"])
def test_chunk_size_does_not_change_the_search(gpu, oracle, robot, monkeypatch):
    """Edge states are validated NS at a time (32, 64 or 128 per chunk; the
    fixed-offset shared region holds per-state buffers for 128). The chunk
    size is a schedule, not a semantic: in deterministic mode a single
    problem with 32-, 64- (default) and 128-state chunks is the same search —
    identical status, path, iterations and reference-semantics CheckStats."""
    m = robots.get(robot)
    probs = load_problems(robot, 10)
    params = PlannerParams(deterministic=True, tree_capacity=20000)
    if robot == "baxter":
        params.dd_radius = 4.0
    knobs = ("PRRTC_NS32", "PRRTC_NS64", "PRRTC_NS128")
    try:
        for kind, pid, s, g in probs[:5]:
            scene, _ = make_scene(robot, kind, pid)
            runs = []
            for env in ({}, {"PRRTC_NS32": "1"}, {"PRRTC_NS128": "1"}):
                for k in knobs:
                    monkeypatch.delenv(k, raising=False)
                for k, v in env.items():
                    monkeypatch.setenv(k, v)
                planner.reload_env()
                runs.append(planner.plan(m, scene, s, g, params))
            r0 = runs[0]
            for r in runs[1:]:
                assert r.status == r0.status
                assert np.array_equal(r.path, r0.path)
                assert r.iterations_total == r0.iterations_total
                assert r.check_stats == r0.check_stats
            if r0.status == PlanStatus.Solved:
                assert oracle.path_valid(m, scene, r0.path, params.n_cc)
    finally:
        for k in knobs:
            monkeypatch.delenv(k, raising=False)
        planner.reload_env()


def test_tree_invariants_under_concurrent_appends(gpu, monkeypatch):
    """Lock-free tree protocol under load: with
    PRRTC_DEBUG_FLAGS bit 2 every CTA checks, at every snapshot it acquires,
    that each published slot of both trees is ready (this launch's epoch), has
    a parent below itself and an edge no longer than delta (SPEC.md:368,
    tree.hpp:27-53). All SMs on one problem (maximum append contention), then
    a batch where CTAs join running problems."""
    monkeypatch.setenv("PRRTC_DEBUG_FLAGS", "4")
    planner.reload_env()
    try:
        _invariant_runs()
    finally:
        monkeypatch.delenv("PRRTC_DEBUG_FLAGS")
        planner.reload_env()


def _invariant_runs():
    m = robots.get("panda")
    probs = load_problems("panda", 1000)[::50]
    for kind, pid, s, g in probs:
        scene, _ = make_scene("panda", kind, pid)
        r = planner.plan(m, scene, s, g, PlannerParams(workers=0, tree_capacity=20000))
        assert "invariant" not in r.message, r.message
        assert r.status in (PlanStatus.Solved, PlanStatus.Failed)
    scenes = [make_scene("panda", k, p)[0] for k, p, _, _ in probs]
    S = np.array([p[2] for p in probs])
    G = np.array([p[3] for p in probs])
    res = planner.plan_batch(m, scenes, S, G, PlannerParams(tree_capacity=20000))
    assert all("invariant" not in r.message for r in res)


def test_uniform_sampler_replays_reference(gpu, oracle):
    """SamplerKind::Uniform (sampling.hpp:40-54: std::mt19937_64 seeded
    seed * 0x9e3779b97f4a7c15 + worker, libstdc++ uniform_real_distribution)
    in deterministic mode: the device's draws equal the reference's, so the
    run replays the reference's workers=1 uniform run node for node (up to
    FP32-FK verdict flips near contact), CheckStats included."""
    from paper_2503_06757_b200.model import SamplerKind
    if oracle.kind != "ref":
        pytest.skip("the uniform sampler is checked against the compiled reference")
    m = robots.get("panda")
    probs = load_problems("panda", 1000)[::50]
    same = 0
    for seed in (0, 7):
        for kind, pid, s, g in probs:
            scene, _ = make_scene("panda", kind, pid)
            p = PlannerParams(tree_capacity=20000, workers=1, sampler=SamplerKind.Uniform, seed=seed)
            r = planner.plan(m, scene, s, g, PlannerParams(**{**p.__dict__, "deterministic": True}))
            ref = oracle.plan(m, scene, s, g, p)
            if r.status == ref.status and (r.status != PlanStatus.Solved or np.array_equal(r.path, ref.path)):
                same += 1
                assert r.iterations_total == ref.iterations_total
                assert r.check_stats == ref.check_stats
    assert same >= 0.9 * 2 * len(probs), same


def test_batch_paths_live_until_freed(gpu):
    """A batch's paths share one pooled pinned block (prrtc_capi.cu
    PathBlock): every path stays valid until its own prrtc_result_free, while
    later batches take blocks from the pool, and frees in any order release
    the block once (exercised over repeated batches so blocks are reused)."""
    import ctypes as C
    from paper_2503_06757_b200 import _lib
    m = robots.get("panda")
    probs = load_problems("panda", 1000)[::10]
    scenes = planner.device_scenes([make_scene("panda", k, p)[0] for k, p, _, _ in probs])
    S = np.array([p[2] for p in probs])
    G = np.array([p[3] for p in probs])
    params = PlannerParams(workers=1, tree_capacity=20000, max_workers_per_problem=1)
    lib = _lib.load()
    kept = []
    for rep in range(6):
        _, res, n, _ = planner._plan_batch_raw(m, scenes, S, G, params, 0)
        copies = [planner._to_result(res[i], m.dof).path for i in range(n)]
        assert sum(res[i].path_block != 0 for i in range(n)) == sum(len(c) > 0 for c in copies)
        kept.append((res, n, copies))
        if rep % 2 == 1:  # free an earlier batch in a scrambled order, one result at a time
            old, k, _ = kept.pop(0)
            for i in np.random.default_rng(rep).permutation(k):
                lib.prrtc_result_free(C.byref(old[int(i)]))
                assert not old[int(i)].path and old[int(i)].path_block == 0
    for res, n, copies in kept:  # still intact after the later batches reused the pool
        for i in range(n):
            now = planner._to_result(res[i], m.dof).path
            assert np.array_equal(now, copies[i])
        planner._free(res, n)
