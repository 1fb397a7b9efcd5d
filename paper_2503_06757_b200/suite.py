"""Bench-harness drop-in: the reference's suite runner,
Table-I statistics, ablation sweeps and ECDF, over the B200 planner.

    load_problem_bundle / load_problem_dir       bench.cpp:36-61
    run_suite                                    bench.cpp:63-88   (one prrtc_plan per run)
    run_suite_batched                            (B200-native: every run of a params group in
                                                  one prrtc_plan_batch launch)
    summarize_values / Quantiles                 bench.cpp:90-109
    summarize / ProblemSummary / summary_table   bench.cpp:111-173
    AblationAxis / apply_ablation_value /
    run_ablation                                 bench.cpp:175-239
    ecdf_points                                  bench.cpp:241-255
    params_hash                                  bench.cpp:23-30

The statistics are exact restatements (tests/test_suite.py compares them
with the compiled reference harness). Only the planner underneath differs:
``run_suite`` calls ``planner.plan`` (the B200 persistent kernel) where the
reference calls its CPU ``plan``; the recorded time is the planning call
only, never setup (bench.cpp:60-61).
"""
from __future__ import annotations

import copy
import enum
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Sequence

import numpy as np

from . import model_io
from .model import PlannerParams, PlanStatus, RobotModel, Scene
from .model_io import BenchRecord, IoError, ProblemSpec


@dataclass
class LoadedProblem:  # bench.hpp:14-20
    spec: ProblemSpec
    robot: RobotModel
    scene: Scene
    params: PlannerParams


def load_problem_bundle(path, base: PlannerParams) -> LoadedProblem:
    """bench.cpp:36-45: problem + referenced robot/scene, base params patched."""
    path = Path(path)
    spec = model_io.load_problem(path)
    robot = model_io.load_robot(path.parent / spec.robot)
    scene = model_io.load_scene(path.parent / spec.scene)
    params = spec.params.apply(copy.copy(base))
    return LoadedProblem(spec, robot, scene, params)


def load_problem_dir(d, base: PlannerParams) -> list[LoadedProblem]:
    """bench.cpp:47-61: every regular *.json file, sorted by path."""
    d = Path(d)
    if not d.is_dir():
        raise IoError(f"{d}: not a directory")
    files = sorted((p for p in d.iterdir() if p.is_file() and p.suffix == ".json"), key=lambda p: str(p))
    return [load_problem_bundle(f, base) for f in files]


def _fnv1a(s: str) -> int:
    """fnv1a (bench.cpp:14-21)."""
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def _ostream_double(x: float) -> str:
    """operator<<(ostream&, double) with the default precision 6 (%g)."""
    return "%g" % x


def params_hash(p: PlannerParams) -> int:
    """params_hash (bench.cpp:23-30); bools stream as 0/1, the sampler as its int."""
    s = "|".join([_ostream_double(p.delta), str(int(p.n_cc)), str(int(p.workers)), str(int(p.max_iters_per_worker)),
                  str(int(p.tree_capacity)), _ostream_double(p.dd_radius), str(int(bool(p.dynamic_domain))),
                  str(int(bool(p.balance))), str(int(bool(p.early_exit))), str(int(bool(p.two_stage))),
                  str(int(bool(p.batched_cc))), str(int(p.nn_partitions)), str(int(p.sampler))])
    return _fnv1a(s)


def _workers(p: PlannerParams, device: int) -> int:
    """bench.cpp:81-82 records hardware_concurrency for workers = 0; on the
    device workers = 0 means one CTA per SM (include/prrtc_b200.h)."""
    if p.workers:
        return int(p.workers)
    from . import planner
    return planner.default_workers(device)


def _record(name: str, trial: int, params: PlannerParams, r, device: int) -> BenchRecord:
    return BenchRecord(problem=name, trial=trial, status=PlanStatus(int(r.status)), time_ms=float(r.wall_time_ms),
                       cost=float(r.cost), iterations=int(r.iterations_total),
                       sphere_tests=int(r.check_stats.sphere_tests), workers=_workers(params, device),
                       seed=int(params.seed), config_hash=params_hash(params))


def run_suite(problems: Sequence[LoadedProblem], trials: int, device: int = 0) -> list[BenchRecord]:
    """run_suite (bench.cpp:63-88): every problem `trials` times, trial t with
    seed base + t, ordered (problem, trial); time = the planning call only."""
    from . import planner
    out = []
    for lp in problems:
        for t in range(trials):
            params = copy.copy(lp.params)
            params.seed = lp.params.seed + t
            r = planner.plan(lp.robot, lp.scene, lp.spec.start, lp.spec.goal, params, device=device)
            out.append(_record(lp.spec.name, t, params, r, device))
    return out


def run_suite_batched(problems: Sequence[LoadedProblem], trials: int, device: int = 0) -> list[BenchRecord]:
    """run_suite with the runs solved as device batches: runs sharing a robot
    and effective params (seed included) go to one prrtc_plan_batch launch.
    Records (order, seeds, hashes) are those of run_suite; time_ms is each
    problem's on-device time-to-solution inside the batch."""
    from . import planner
    runs = []
    for lp in problems:
        for t in range(trials):
            params = copy.copy(lp.params)
            params.seed = lp.params.seed + t
            runs.append((lp, t, params))
    groups: dict = {}
    for i, (lp, t, params) in enumerate(runs):
        key = (id(lp.robot), params_hash(params), params.seed, params.threads_per_cta, params.ctas_per_sm)
        groups.setdefault(key, []).append(i)
    results = [None] * len(runs)
    for idx in groups.values():
        lp0, _, params = runs[idx[0]]
        res = planner.plan_batch(lp0.robot, [runs[i][0].scene for i in idx],
                                 np.stack([runs[i][0].spec.start for i in idx]),
                                 np.stack([runs[i][0].spec.goal for i in idx]), params, device=device)
        for i, r in zip(idx, res):
            r.wall_time_ms = r.device_time_ms
            results[i] = r
    return [_record(lp.spec.name, t, params, results[i], device) for i, (lp, t, params) in enumerate(runs)]


# ---------------------------------------------------------------------------
# statistics (bench.cpp:90-173)
# ---------------------------------------------------------------------------

@dataclass
class Quantiles:  # bench.hpp:33-41
    n: int = 0
    mean: float = 0.0
    q1: float = 0.0
    median: float = 0.0
    q3: float = 0.0
    p95: float = 0.0
    max: float = 0.0


def summarize_values(values: Sequence[float]) -> Quantiles:
    """summarize_values (bench.cpp:90-109): linear interpolation between the
    sorted neighbours at h = p (n - 1); mean by a left-to-right sum of the
    sorted values (std::accumulate)."""
    if len(values) == 0:
        raise ValueError("summarize_values: empty input")
    s = sorted(float(v) for v in values)
    n = len(s)

    def quantile(p: float) -> float:
        h = p * float(n - 1)
        lo = int(h)
        if lo + 1 >= n:
            return s[-1]
        return s[lo] + (h - float(lo)) * (s[lo + 1] - s[lo])

    acc = 0.0
    for v in s:
        acc += v
    return Quantiles(n=n, mean=acc / float(n), q1=quantile(0.25), median=quantile(0.5), q3=quantile(0.75),
                     p95=quantile(0.95), max=s[-1])


@dataclass
class ProblemSummary:  # bench.hpp:45-52
    problem: str = ""
    runs: int = 0
    solved: int = 0
    success_rate: float = 0.0
    time_ms: Quantiles = field(default_factory=Quantiles)
    cost: Quantiles = field(default_factory=Quantiles)


def _summarize_group(name: str, records: Sequence[BenchRecord]) -> ProblemSummary:
    """summarize_group (bench.cpp:113-132)."""
    s = ProblemSummary(problem=name, runs=len(records))
    times = [r.time_ms for r in records if int(r.status) == PlanStatus.Solved]
    costs = [r.cost for r in records if int(r.status) == PlanStatus.Solved]
    s.solved = len(times)
    s.success_rate = 0.0 if s.runs == 0 else s.solved / s.runs
    if times:
        s.time_ms = summarize_values(times)
        s.cost = summarize_values(costs)
    return s


def summarize(records: Sequence[BenchRecord]) -> list[ProblemSummary]:
    """summarize (bench.cpp:136-156): per problem in first-seen order, then the
    pooled row (problem == "")."""
    if len(records) == 0:
        raise ValueError("summarize: empty input")
    order = []
    for r in records:
        if r.problem not in order:
            order.append(r.problem)
    out = [_summarize_group(name, [r for r in records if r.problem == name]) for name in order]
    out.append(_summarize_group("", list(records)))
    return out


def summary_table(rows: Sequence[ProblemSummary]) -> str:
    """summary_table (bench.cpp:158-173), same printf formats."""
    out = ["%-28s %5s %7s | %9s %9s %9s | %9s %9s\n" % ("problem", "runs", "succ", "t_mean", "t_med", "t_max",
                                                         "c_mean", "c_med")]
    for s in rows:
        out.append("%-28s %5d %6.1f%% | %9.3f %9.3f %9.3f | %9.3f %9.3f\n" % (
            "(pooled)" if s.problem == "" else s.problem, s.runs, 100.0 * s.success_rate, s.time_ms.mean,
            s.time_ms.median, s.time_ms.max, s.cost.mean, s.cost.median))
    return "".join(out)


# ---------------------------------------------------------------------------
# ablations (bench.cpp:175-239)
# ---------------------------------------------------------------------------

class AblationAxis(enum.Enum):  # bench.hpp:60
    Workers = "workers"
    EarlyExit = "early_exit"
    TwoStage = "two_stage"
    DynamicDomain = "dynamic_domain"
    BatchedCc = "batched_cc"


def ablation_axis_from(name: str) -> AblationAxis:
    """ablation_axis_from (bench.cpp:175-182)."""
    for a in AblationAxis:
        if a.value == name:
            return a
    raise ValueError(f"unknown ablation axis '{name}'")


def _parse_on_off(v: str) -> bool:
    """parse_on_off (bench.cpp:197-201)."""
    if v in ("on", "true", "1"):
        return True
    if v in ("off", "false", "0"):
        return False
    raise ValueError(f"expected on/off, got '{v}'")


def _stoul(v: str) -> int:
    """std::stoul: optional leading whitespace/sign, then digits (prefix parse)."""
    s = v.lstrip()
    i = 0
    neg = False
    if i < len(s) and s[i] in "+-":
        neg = s[i] == "-"
        i += 1
    j = i
    while j < len(s) and s[j].isdigit():
        j += 1
    if j == i:
        raise ValueError("stoul")
    x = int(s[i:j])
    if x > 0xFFFFFFFFFFFFFFFF:
        raise OverflowError("stoul")
    return ((-x) if neg else x) & 0xFFFFFFFF


@dataclass
class AblationSpec:  # bench.hpp:66-69
    axis: AblationAxis = AblationAxis.Workers
    values: list = field(default_factory=list)


def apply_ablation_value(params: PlannerParams, axis: AblationAxis, value: str) -> None:
    """apply_ablation_value (bench.cpp:205-222)."""
    if axis == AblationAxis.Workers:
        params.workers = _stoul(value)
    elif axis == AblationAxis.EarlyExit:
        params.early_exit = _parse_on_off(value)
    elif axis == AblationAxis.TwoStage:
        params.two_stage = _parse_on_off(value)
    elif axis == AblationAxis.DynamicDomain:
        params.dynamic_domain = _parse_on_off(value)
    elif axis == AblationAxis.BatchedCc:
        params.batched_cc = _parse_on_off(value)


@dataclass
class AblationGroup:  # bench.hpp:76-79
    value: str
    records: list


def run_ablation(spec: AblationSpec, problems: Sequence[LoadedProblem], trials: int, device: int = 0,
                 batched: bool = False) -> list[AblationGroup]:
    """run_ablation (bench.cpp:225-239): sweep one axis, everything else fixed."""
    if not spec.values:
        raise ValueError("run_ablation: values must be non-empty")
    groups = []
    for value in spec.values:
        adjusted = []
        for p in problems:
            q = copy.copy(p)
            q.params = copy.copy(p.params)
            apply_ablation_value(q.params, spec.axis, value)
            adjusted.append(q)
        runner = run_suite_batched if batched else run_suite
        groups.append(AblationGroup(value, runner(adjusted, trials, device)))
    return groups


def ecdf_points(records: Sequence[BenchRecord], use_cost: bool) -> list[tuple[float, float]]:
    """ecdf_points (bench.cpp:241-255): sorted solved values, fraction of ALL
    runs solved within each."""
    vals = sorted((r.cost if use_cost else r.time_ms) for r in records if int(r.status) == PlanStatus.Solved)
    total = float(len(records))
    return [(v, (i + 1) / total) for i, v in enumerate(vals)]
