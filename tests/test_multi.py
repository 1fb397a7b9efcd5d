"""Multi-device batches: prrtc_plan_batch_multi's chunk queue
and its equivalence with prrtc_plan_batch."""
import numpy as np
import pytest

from conftest import load_problems
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.model import PlannerParams, PlanStatus
from paper_2503_06757_b200.scenes import make_scene


@pytest.mark.parametrize("workers", [1, 2, 4, 8])
@pytest.mark.parametrize("n,chunk", [(1000, 64), (100, 7), (5, 0), (64, 64), (65, 64)])
def test_chunk_queue_hands_out_every_problem_once(workers, n, chunk):
    owner, taken = planner.debug_chunk_queue(workers, n, chunk, [20] * workers)
    assert (owner >= 0).all() and (owner < workers).all()
    c = chunk or max(64, -(-n // (4 * workers)))
    assert taken.sum() == -(-n // c)
    # chunks are contiguous runs owned by one worker
    for b in range(0, n, c):
        assert len(set(owner[b:b + c].tolist())) == 1


def test_chunk_queue_slow_worker_takes_fewer_chunks():
    # worker 1 is 20x slower per problem: the dynamic queue gives it fewer chunks
    owner, taken = planner.debug_chunk_queue(4, 2048, 64, [50, 1000, 50, 50])
    assert (owner >= 0).all()
    assert taken[1] <= min(taken[0], taken[2], taken[3])


@pytest.mark.gpu
def test_plan_batch_multi_equals_plan_batch_deterministic(gpu):
    """One device, deterministic mode (one CTA, tickets in order): the chunked
    multi-device call returns exactly what one prrtc_plan_batch returns."""
    m = robots.get("panda")
    probs = load_problems("panda", 1000)[::50]
    scenes = [make_scene("panda", k, p)[0] for k, p, _, _ in probs]
    S = np.array([p[2] for p in probs])
    G = np.array([p[3] for p in probs])
    params = PlannerParams(workers=1, tree_capacity=20000, deterministic=True)
    ref = planner.plan_batch_arrays(m, scenes, S, G, params)
    got = planner.plan_batch_multi(m, scenes, S, G, params, devices=[0], chunk=3)
    assert np.array_equal(ref.status, got.status)
    assert np.array_equal(ref.iterations_total, got.iterations_total)
    for a, b in zip(ref.paths, got.paths):
        assert np.array_equal(a, b)
    assert (got.status == PlanStatus.Solved).mean() > 0.5


@pytest.mark.gpu
def test_plan_batch_multi_rejects_duplicate_device(gpu):
    m = robots.get("panda")
    k, p, s, g = load_problems("panda", 1)[0]
    sc = make_scene("panda", k, p)[0]
    with pytest.raises(ValueError):
        planner.plan_batch_multi(m, [sc], s[None], g[None], PlannerParams(), devices=[0, 0])
