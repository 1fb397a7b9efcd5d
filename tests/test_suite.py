"""The bench-harness drop-in (paper_2503_06757_b200/suite.py) against the
reference's bench.cpp (oracle/_ref/libprrtc_ref_io.so): statistics,
summary table, ECDF, ablation parsing and the run records' seeds / hashes /
order. CPU, except the last test which runs the suite on the B200."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2503_06757_b200 import model_io as mio
from paper_2503_06757_b200 import robots, suite
from paper_2503_06757_b200.model import PlannerParams, PlanStatus
from paper_2503_06757_b200.scenes import make_scene

ROOT = Path(__file__).resolve().parents[1]

try:
    from oracle.refio import RefIO, available as refio_available
except Exception:  # pragma: no cover
    refio_available = lambda: False  # noqa: E731

needs_ref = pytest.mark.skipif(not refio_available(), reason="reference bench build absent (oracle/_ref)")


@pytest.fixture(scope="module")
def ref():
    return RefIO()


def _records(n=60, seed=1, names=7):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        out.append(mio.BenchRecord(problem=f"prob_{(i * 5) % names}", trial=i // names,
                                   status=PlanStatus(int(rng.choice([0, 0, 0, 0, 1, 2]))),
                                   time_ms=float(rng.lognormal(0, 1)), cost=float(rng.uniform(2, 9)),
                                   iterations=int(rng.integers(1, 4000)), sphere_tests=int(rng.integers(0, 10**8)),
                                   workers=1, seed=i))
    return out


def test_summarize_values_known_answers():
    q = suite.summarize_values([3.0, 1.0, 2.0, 4.0])
    assert (q.n, q.mean, q.q1, q.median, q.q3, q.max) == (4, 2.5, 1.75, 2.5, 3.25, 4.0)
    assert q.p95 == pytest.approx(3.85)
    one = suite.summarize_values([7.0])
    assert (one.q1, one.median, one.p95, one.max) == (7.0, 7.0, 7.0, 7.0)
    with pytest.raises(ValueError, match="summarize_values: empty input"):
        suite.summarize_values([])
    with pytest.raises(ValueError, match="summarize: empty input"):
        suite.summarize([])


@needs_ref
def test_summarize_values_bitexact_vs_reference(ref):
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 5, 19, 20, 21, 100, 1001):
        v = rng.lognormal(0, 2, n)
        q = suite.summarize_values(v)
        r = ref.summarize_values(v)
        got = np.array([q.n, q.mean, q.q1, q.median, q.q3, q.p95, q.max])
        assert got.tobytes() == r.tobytes(), n


@needs_ref
def test_summary_table_matches_reference(ref):
    recs = _records()
    assert suite.summary_table(suite.summarize(recs)) == ref.summary_table(recs)
    # a problem with no solved run keeps zeroed quantiles
    recs2 = recs + [mio.BenchRecord(problem="never", status=PlanStatus.Failed, time_ms=1.0)]
    assert suite.summary_table(suite.summarize(recs2)) == ref.summary_table(recs2)


def test_summarize_groups():
    recs = _records()
    rows = suite.summarize(recs)
    assert rows[-1].problem == "" and rows[-1].runs == len(recs)
    assert [r.problem for r in rows[:-1]] == list(dict.fromkeys(r.problem for r in recs))
    assert sum(r.solved for r in rows[:-1]) == rows[-1].solved


@needs_ref
@pytest.mark.parametrize("use_cost", [False, True])
def test_ecdf_matches_reference(ref, use_cost):
    recs = _records(80)
    got = suite.ecdf_points(recs, use_cost)
    want = ref.ecdf([int(r.status) for r in recs], [r.time_ms for r in recs], [r.cost for r in recs], use_cost)
    assert got == want
    assert got[-1][1] == sum(int(r.status) == 0 for r in recs) / len(recs)


@needs_ref
def test_ablation_values_match_reference(ref):
    for axis, values in (("workers", ["1", "8", "256", " 12", "+3"]), ("early_exit", ["on", "off", "true", "0"]),
                         ("two_stage", ["1", "false"]), ("dynamic_domain", ["off", "on"]),
                         ("batched_cc", ["true", "off"])):
        for v in values:
            p = PlannerParams()
            suite.apply_ablation_value(p, suite.ablation_axis_from(axis), v)
            r = ref.apply_ablation(axis, v, PlannerParams())
            assert (p.workers, p.early_exit, p.two_stage, p.dynamic_domain, p.batched_cc) == \
                (r.workers, bool(r.early_exit), bool(r.two_stage), bool(r.dynamic_domain), bool(r.batched_cc))
    for axis, v in (("early_exit", "maybe"), ("speed", "1")):
        with pytest.raises(ValueError) as e:
            suite.apply_ablation_value(PlannerParams(), suite.ablation_axis_from(axis), v)
        with pytest.raises(ValueError) as r:
            ref.apply_ablation(axis, v, PlannerParams())
        assert str(e.value) == str(r.value)
    with pytest.raises(ValueError, match="values must be non-empty"):
        suite.run_ablation(suite.AblationSpec(suite.AblationAxis.Workers, []), [], 1)


def _problem_dir(d: Path, n=2):
    m = robots.get("panda")
    mio.write_robot(d / "robot.json", m)
    data = np.load(ROOT / "tests" / "golden" / "problems_panda.npz")
    (d / "problems").mkdir()
    for i in range(n):
        s, _ = make_scene("panda", str(data["kind"][i]), int(data["pid"][i]))
        mio.write_scene(d / f"scene_{i}.json", s)
        patch = mio.ParamsPatch(tree_capacity=4000, seed=5 * i) if i % 2 else mio.ParamsPatch(tree_capacity=4000)
        mio.write_problem(d / "problems" / f"p{i}.json",
                          mio.ProblemSpec(name=f"panda_{i}", robot="../robot.json", scene=f"../scene_{i}.json",
                                          start=data["start"][i], goal=data["goal"][i], params=patch))
    return d / "problems"


@pytest.mark.parametrize("p", [PlannerParams(), PlannerParams(delta=0.125, n_cc=7, dd_radius=1.0 / 3.0, workers=3,
                                                                 dynamic_domain=False, batched_cc=True),
                               PlannerParams(tree_capacity=123456789, max_iters_per_worker=10**12, delta=1e-7)])
def test_params_hash_stream_format(p):
    s = "|".join(["%g" % p.delta, str(p.n_cc), str(p.workers), str(p.max_iters_per_worker), str(p.tree_capacity),
                  "%g" % p.dd_radius, str(int(p.dynamic_domain)), str(int(p.balance)), str(int(p.early_exit)),
                  str(int(p.two_stage)), str(int(p.batched_cc)), str(p.nn_partitions), str(int(p.sampler))])
    assert suite.params_hash(p) == suite._fnv1a(s)
    assert suite._fnv1a("") == 1469598103934665603


@needs_ref
def test_run_records_match_reference(ref, tmp_path):
    """The reference's run_suite (its CPU planner, workers=1) over a problem
    directory: our records carry the same order, trials, seeds and
    config hashes (bench.cpp:63-88)."""
    d = _problem_dir(tmp_path)
    base = PlannerParams(workers=1, seed=2)
    want = ref.run_suite(d, base, trials=2)
    probs = suite.load_problem_dir(d, base)
    recs = []
    for lp in probs:
        for t in range(2):
            p = PlannerParams(**{**lp.params.__dict__})
            p.seed = lp.params.seed + t
            recs.append((suite.params_hash(p), 1, p.seed, t))
    assert [(h, w, s, tr) for h, w, s, st, tr in want] == recs


@pytest.mark.gpu
def test_run_suite_on_b200(tmp_path, oracle):
    """run_suite / run_suite_batched through the B200 planner: every run
    solves, paths re-validate with the reference checker, and both runners
    produce the same record keys; the summary table renders."""
    d = _problem_dir(tmp_path, n=3)
    probs = suite.load_problem_dir(d, PlannerParams())
    recs = suite.run_suite(probs, 2)
    assert [(r.problem, r.trial) for r in recs] == [(lp.spec.name, t) for lp in probs for t in range(2)]
    assert all(r.status == PlanStatus.Solved and r.time_ms > 0 for r in recs)
    assert [r.seed for r in recs] == [lp.params.seed + t for lp in probs for t in range(2)]
    brecs = suite.run_suite_batched(probs, 2)
    assert [(r.problem, r.trial, r.seed, r.config_hash) for r in brecs] == \
        [(r.problem, r.trial, r.seed, r.config_hash) for r in recs]
    assert all(r.status == PlanStatus.Solved for r in brecs)
    table = suite.summary_table(suite.summarize(recs))
    assert "(pooled)" in table and "100.0%" in table
    groups = suite.run_ablation(suite.AblationSpec(suite.AblationAxis.EarlyExit, ["on", "off"]), probs[:1], 1,
                                batched=True)
    assert [g.value for g in groups] == ["on", "off"]
    assert all(r.status == PlanStatus.Solved for g in groups for r in g.records)
    pts = suite.ecdf_points(recs, False)
    assert pts[-1][1] == 1.0
