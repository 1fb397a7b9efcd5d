// oracle/ref_io_capi.cpp — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// extern "C" wrapper over the UNMODIFIED reference model I/O and bench
// harness sources (/root/reference/proj/src/model_io.cpp, bench.cpp), compiled
// in place by oracle/Makefile into oracle/_ref/libprrtc_ref_io.so together
// with the reference planner (namespace renamed prrtc -> prrtc_ref). It pins
// the Python drop-in paper_2503_06757_b200/model_io.py and suite.py: the
// tests round-trip files through the reference loaders/writers and compare
// the harness statistics. Only tests/ may load it.
//
// Every function forwards to the reference symbol cited beside it.

#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "prrtc/bench.hpp"
#include "prrtc/model_io.hpp"
#include "prrtc/planner.hpp"

#include "prrtc_b200.h"

using namespace prrtc;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}

int put_string(const std::string& s, char* out, size_t len) {
    if (!out || len == 0) return (int)s.size();
    std::snprintf(out, len, "%s", s.c_str());
    return (int)s.size();
}

PlannerParams to_params(const prrtc_params* p) {
    PlannerParams q;
    q.delta = p->delta;
    q.n_cc = p->n_cc;
    q.workers = p->workers;
    q.max_iters_per_worker = p->max_iters_per_worker;
    q.tree_capacity = p->tree_capacity;
    q.dd_radius = p->dd_radius;
    q.dynamic_domain = p->dynamic_domain;
    q.balance = p->balance;
    q.early_exit = p->early_exit;
    q.two_stage = p->two_stage;
    q.batched_cc = p->batched_cc;
    q.nn_partitions = p->nn_partitions;
    q.sampler = p->sampler == PRRTC_SAMPLER_UNIFORM ? SamplerKind::Uniform : SamplerKind::Halton;
    q.seed = p->seed;
    return q;
}

std::vector<BenchRecord> to_records(uint32_t n, const char* const* problems, const int32_t* trials,
                                    const int32_t* statuses, const double* time_ms, const double* cost,
                                    const uint64_t* iterations, const uint64_t* sphere_tests,
                                    const uint32_t* workers, const uint64_t* seeds) {
    std::vector<BenchRecord> rows(n);
    for (uint32_t i = 0; i < n; ++i) {
        rows[i].problem = problems[i];
        rows[i].trial = trials[i];
        rows[i].status = statuses[i] == 0 ? PlanStatus::Solved
                         : statuses[i] == 1 ? PlanStatus::Failed
                                            : PlanStatus::InfeasibleEndpoint;
        rows[i].time_ms = time_ms[i];
        rows[i].cost = cost[i];
        rows[i].iterations = iterations[i];
        rows[i].sphere_tests = sphere_tests[i];
        rows[i].workers = workers[i];
        rows[i].seed = seeds[i];
    }
    return rows;
}
}  // namespace

extern "C" {

int refio_last_error(char* buf, size_t len) { return put_string(g_err, buf, len); }

// load_robot/load_scene/load_problem/load_path_file then the matching writer
// (model_io.cpp:91-421). kind: 0 robot, 1 scene, 2 problem, 3 path.
int refio_roundtrip(int kind, const char* in_path, const char* out_path) {
    try {
        switch (kind) {
            case 0: write_robot(out_path, load_robot(in_path)); break;
            case 1: write_scene(out_path, load_scene(in_path)); break;
            case 2: write_problem(out_path, load_problem(in_path)); break;
            case 3: write_path(out_path, load_path_file(in_path)); break;
            default: g_err = "bad kind"; return -1;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// load_robot then RobotModel::dof (robot.hpp:53).
int refio_robot_dof(const char* path) {
    try {
        return load_robot(path).dof;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// load_problem_bundle (bench.cpp:36-45): the effective params as JSON-like
// values written into a prrtc_params plus the problem name.
int refio_problem_bundle(const char* path, const prrtc_params* base, prrtc_params* out, char* name,
                         size_t name_len) {
    try {
        const LoadedProblem lp = load_problem_bundle(path, to_params(base));
        const PlannerParams& p = lp.params;
        *out = *base;
        out->delta = p.delta;
        out->n_cc = p.n_cc;
        out->workers = p.workers;
        out->max_iters_per_worker = p.max_iters_per_worker;
        out->tree_capacity = p.tree_capacity;
        out->dd_radius = p.dd_radius;
        out->dynamic_domain = p.dynamic_domain;
        out->balance = p.balance;
        out->early_exit = p.early_exit;
        out->two_stage = p.two_stage;
        out->batched_cc = p.batched_cc;
        out->nn_partitions = p.nn_partitions;
        out->sampler = p.sampler == SamplerKind::Uniform ? PRRTC_SAMPLER_UNIFORM : PRRTC_SAMPLER_HALTON;
        out->seed = p.seed;
        put_string(lp.spec.name, name, name_len);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// load_problem_dir (bench.cpp:47-61): number of problems and their names,
// '\n'-separated, in the reference's order.
int refio_problem_dir(const char* dir, char* names, size_t len) {
    try {
        const auto ps = load_problem_dir(dir, PlannerParams{});
        std::string s;
        for (const auto& p : ps) s += p.spec.name + "\n";
        put_string(s, names, len);
        return (int)ps.size();
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// results_csv_string (model_io.cpp:439-449).
int refio_results_csv(uint32_t n, const char* const* problems, const int32_t* trials,
                      const int32_t* statuses, const double* time_ms, const double* cost,
                      const uint64_t* iterations, const uint64_t* sphere_tests, const uint32_t* workers,
                      const uint64_t* seeds, char* out, size_t len) {
    const auto rows = to_records(n, problems, trials, statuses, time_ms, cost, iterations, sphere_tests,
                                 workers, seeds);
    return put_string(results_csv_string(rows), out, len);
}

// summarize_values (bench.cpp:90-109): n, mean, q1, median, q3, p95, max.
int refio_summarize_values(const double* v, uint32_t n, double* out7) {
    try {
        const Quantiles q = summarize_values(std::span<const double>(v, n));
        const double r[7] = {(double)q.n, q.mean, q.q1, q.median, q.q3, q.p95, q.max};
        std::memcpy(out7, r, sizeof r);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// summarize + summary_table (bench.cpp:136-173).
int refio_summary_table(uint32_t n, const char* const* problems, const int32_t* trials,
                        const int32_t* statuses, const double* time_ms, const double* cost,
                        const uint64_t* iterations, const uint64_t* sphere_tests, const uint32_t* workers,
                        const uint64_t* seeds, char* out, size_t len) {
    try {
        const auto rows = to_records(n, problems, trials, statuses, time_ms, cost, iterations, sphere_tests,
                                     workers, seeds);
        return put_string(summary_table(summarize(rows)), out, len);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ecdf_points (bench.cpp:241-255) -> pairs written to out[2*k]; returns k.
int refio_ecdf(uint32_t n, const int32_t* statuses, const double* time_ms, const double* cost, int use_cost,
               double* out) {
    std::vector<const char*> names(n, "p");
    std::vector<int32_t> zeros(n, 0);
    std::vector<uint64_t> z64(n, 0);
    std::vector<uint32_t> ones(n, 1);
    const auto rows = to_records(n, names.data(), zeros.data(), statuses, time_ms, cost, z64.data(),
                                 z64.data(), ones.data(), z64.data());
    const auto pts = ecdf_points(rows, use_cost != 0);
    for (size_t i = 0; i < pts.size(); ++i) {
        out[2 * i] = pts[i].first;
        out[2 * i + 1] = pts[i].second;
    }
    return (int)pts.size();
}

// ablation_axis_from + apply_ablation_value (bench.cpp:175-222).
int refio_apply_ablation(const char* axis, const char* value, prrtc_params* p) {
    try {
        PlannerParams q = to_params(p);
        apply_ablation_value(q, ablation_axis_from(axis), value);
        p->workers = q.workers;
        p->early_exit = q.early_exit;
        p->two_stage = q.two_stage;
        p->dynamic_domain = q.dynamic_domain;
        p->batched_cc = q.batched_cc;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// run_suite (bench.cpp:63-88) over a problem directory with the reference's
// own CPU plan(): records' config_hash (params_hash, bench.cpp:23-30),
// workers, seed, status, iterations — for the harness parity test.
int refio_run_suite(const char* dir, const prrtc_params* base, int trials, uint32_t cap, uint64_t* hashes,
                    uint32_t* workers, uint64_t* seeds, int32_t* statuses, int32_t* trial_out) {
    try {
        const auto ps = load_problem_dir(dir, to_params(base));
        const auto recs = run_suite(ps, trials);
        if (recs.size() > cap) {
            g_err = "capacity";
            return -1;
        }
        for (size_t i = 0; i < recs.size(); ++i) {
            hashes[i] = recs[i].config_hash;
            workers[i] = recs[i].workers;
            seeds[i] = recs[i].seed;
            statuses[i] = (int32_t)recs[i].status;
            trial_out[i] = recs[i].trial;
        }
        return (int)recs.size();
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
