// oracle/ref_capi.cpp — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// extern "C" wrapper over the UNMODIFIED reference sources compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libprrtc_ref.so
// (namespace renamed prrtc -> prrtc_ref with -Dprrtc=prrtc_ref so it can share
// a process with the B200 drop-in). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it, and only as the
// checker / the CPU baseline — never as the thing measured or shipped.
//
// Every function forwards to the reference symbol cited beside it.

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>
#include <atomic>

#include "prrtc/collision.hpp"
#include "prrtc/geometry.hpp"
#include "prrtc/kernels.hpp"
#include "prrtc/kinematics.hpp"
#include "prrtc/nn.hpp"
#include "prrtc/planner.hpp"
#include "prrtc/sampling.hpp"

#include "prrtc_b200.h"

using namespace prrtc;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}

}  // namespace

extern "C" {

int ref_last_error(char* buf, size_t len) {
    if (!buf || len == 0) return 0;
    std::snprintf(buf, len, "%s", g_err.c_str());
    return 0;
}

// Builds and finalizes a RobotModel (robot.hpp:44-71, kinematics.cpp:15-74).
void* ref_robot_create(const prrtc_robot_desc* d) {
    try {
        auto* m = new RobotModel();
        m->name = "robot";
        for (uint32_t i = 0; i < d->n_links; ++i) {
            Joint j;
            j.kind = d->kind[i] == PRRTC_JOINT_REVOLUTE    ? JointKind::Revolute
                     : d->kind[i] == PRRTC_JOINT_PRISMATIC ? JointKind::Prismatic
                                                           : JointKind::Fixed;
            j.parent = d->parent[i];
            j.origin.rotation = {d->origin_quat[4 * i], d->origin_quat[4 * i + 1],
                                 d->origin_quat[4 * i + 2], d->origin_quat[4 * i + 3]};
            j.origin.translation = {d->origin_xyz[3 * i], d->origin_xyz[3 * i + 1],
                                    d->origin_xyz[3 * i + 2]};
            j.axis = {d->axis[3 * i], d->axis[3 * i + 1], d->axis[3 * i + 2]};
            j.lo = d->lo[i];
            j.hi = d->hi[i];
            m->joints.push_back(j);
            LinkSpheres ls;
            ls.coarse.center = {d->coarse[4 * i], d->coarse[4 * i + 1], d->coarse[4 * i + 2]};
            ls.coarse.radius = d->coarse[4 * i + 3];
            for (uint32_t k = d->fine_offset[i]; k < d->fine_offset[i + 1]; ++k) {
                Sphere s;
                s.center = {d->fine[4 * k], d->fine[4 * k + 1], d->fine[4 * k + 2]};
                s.radius = d->fine[4 * k + 3];
                ls.fine.push_back(s);
            }
            m->spheres.push_back(ls);
        }
        for (uint32_t p = 0; p < d->n_self_pairs; ++p) {
            m->self_pairs.emplace_back(d->self_pairs[2 * p], d->self_pairs[2 * p + 1]);
        }
        m->finalize();
        return m;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_robot_destroy(void* r) { delete static_cast<RobotModel*>(r); }

int ref_robot_dof(void* r) { return static_cast<RobotModel*>(r)->dof; }

// Scene (geometry.hpp:37-46); primitive order: spheres, boxes, capsules.
void* ref_scene_create(const prrtc_scene_desc* d) {
    if (d->cylinders && d->n_cylinders) {  // the reference has no cylinder (geometry.hpp:35)
        g_err = "the reference scene has no cylinder primitive (geometry.hpp:35)";
        return nullptr;
    }
    try {
        auto* s = new Scene();
        s->name = "scene";
        for (uint32_t i = 0; i < d->n_spheres; ++i) {
            const double* p = d->spheres + 4 * i;
            s->primitives.push_back(SpherePrim{{p[0], p[1], p[2]}, p[3]});
        }
        for (uint32_t i = 0; i < d->n_boxes; ++i) {
            const double* p = d->boxes + 10 * i;
            BoxPrim b;
            b.pose.rotation = {p[0], p[1], p[2], p[3]};
            b.pose.translation = {p[4], p[5], p[6]};
            b.half_extents = {p[7], p[8], p[9]};
            s->primitives.push_back(b);
        }
        for (uint32_t i = 0; i < d->n_capsules; ++i) {
            const double* p = d->capsules + 7 * i;
            s->primitives.push_back(CapsulePrim{{p[0], p[1], p[2]}, {p[3], p[4], p[5]}, p[6]});
        }
        s->validate();
        return s;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_scene_destroy(void* s) { delete static_cast<Scene*>(s); }

// kernels::force_backend / reset_backend (kernels.hpp:107-110).
int ref_force_scalar(int on) {
    if (on) {
        kernels::force_backend(kernels::Backend::Scalar);
    } else {
        kernels::reset_backend();
    }
    return kernels::active_backend() == kernels::Backend::Scalar ? 1 : 0;
}

// forward_kinematics (kinematics.cpp:92-103): out[L*12] = R row-major, t.
int ref_fk_poses(void* robot, const double* q, double* out) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        auto poses = forward_kinematics(m, ConfigView(q, m.dof));
        for (size_t l = 0; l < poses.size(); ++l) {
            for (int k = 0; k < 9; ++k) out[12 * l + k] = poses[l].rotation.m[k];
            out[12 * l + 9] = poses[l].translation.x;
            out[12 * l + 10] = poses[l].translation.y;
            out[12 * l + 11] = poses[l].translation.z;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// sphere_positions (kinematics.cpp:111-126): out[n*4]; level 0 coarse, 1 fine.
int ref_fk_spheres(void* robot, const double* q, int level, double* out) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        auto s = sphere_positions(m, ConfigView(q, m.dof),
                                  level == 0 ? SphereLevel::Coarse : SphereLevel::Fine);
        for (size_t i = 0; i < s.size(); ++i) {
            out[4 * i] = s[i].center.x;
            out[4 * i + 1] = s[i].center.y;
            out[4 * i + 2] = s[i].center.z;
            out[4 * i + 3] = s[i].radius;
        }
        return static_cast<int>(s.size());
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// sphere_vs_primitive (geometry.cpp:41-66) for every primitive of the scene.
int ref_sphere_hits(void* scene, double x, double y, double z, double r, uint8_t* hits) {
    const auto& s = *static_cast<Scene*>(scene);
    PosedSphere ps{{x, y, z}, r};
    int any = 0;
    for (size_t i = 0; i < s.primitives.size(); ++i) {
        hits[i] = sphere_vs_primitive(ps, s.primitives[i]) ? 1 : 0;
        any |= hits[i];
    }
    return any;
}

// any_hit[i] = 1 iff sphere i (xyzr[4i..4i+3]) hits some primitive, by the
// reference predicate sphere_vs_primitive (geometry.cpp:41-66).
int ref_sphere_any_hits(void* scene, const double* xyzr, uint32_t n, uint8_t* any_hit) {
    const auto& s = *static_cast<Scene*>(scene);
    for (uint32_t i = 0; i < n; ++i) {
        PosedSphere ps{{xyzr[4 * i], xyzr[4 * i + 1], xyzr[4 * i + 2]}, xyzr[4 * i + 3]};
        uint8_t h = 0;
        for (size_t k = 0; k < s.primitives.size() && !h; ++k) h = sphere_vs_primitive(ps, s.primitives[k]) ? 1 : 0;
        any_hit[i] = h;
    }
    return 0;
}

static void put_stats(const CheckStats& st, uint64_t* out) {
    if (!out) return;
    auto s = snapshot(st);
    out[0] = s.sphere_tests;
    out[1] = s.fk_calls;
    out[2] = s.fine_stage_entries;
}

// CollisionChecker::check_config (collision.cpp:130-204); 1 = free.
int ref_check_config(void* robot, void* scene, const double* q, int two_stage, int early_exit,
                     uint64_t* stats) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        CollisionChecker c(m, *static_cast<Scene*>(scene));
        CheckStats st;
        bool ok = c.check_config(ConfigView(q, m.dof), st,
                                 CheckOptions{two_stage != 0, early_exit != 0});
        put_stats(st, stats);
        return ok ? 1 : 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Many configs through one checker: out[n] (1 = free).
int ref_check_configs(void* robot, void* scene, const double* q, uint32_t n, int two_stage,
                      uint8_t* out) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        CollisionChecker c(m, *static_cast<Scene*>(scene));
        CheckStats st;
        for (uint32_t i = 0; i < n; ++i) {
            out[i] = c.check_config(ConfigView(q + size_t(i) * m.dof, m.dof), st,
                                    CheckOptions{two_stage != 0, true})
                         ? 1
                         : 0;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// CollisionChecker::validate_edge (collision.cpp:206-224); 1 = valid.
int ref_validate_edge(void* robot, void* scene, const double* from, const double* to, int n,
                      int two_stage, int early_exit, uint64_t* stats) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        CollisionChecker c(m, *static_cast<Scene*>(scene));
        CheckStats st;
        bool ok = c.validate_edge(ConfigView(from, m.dof), ConfigView(to, m.dof), n, st,
                                  CheckOptions{two_stage != 0, early_exit != 0});
        put_stats(st, stats);
        return ok ? 1 : 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Many edges through one checker, one validate_edge call each.
int ref_validate_edges(void* robot, void* scene, const double* from, const double* to,
                       uint32_t n_edges, int n, int two_stage, int early_exit, uint8_t* out) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        CollisionChecker c(m, *static_cast<Scene*>(scene));
        CheckStats st;
        for (uint32_t e = 0; e < n_edges; ++e) {
            out[e] = c.validate_edge(ConfigView(from + size_t(e) * m.dof, m.dof),
                                     ConfigView(to + size_t(e) * m.dof, m.dof), n, st,
                                     CheckOptions{two_stage != 0, early_exit != 0})
                         ? 1
                         : 0;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// CollisionChecker::validate_edge_batched (collision.cpp:226-262).
int ref_validate_edge_batched(void* robot, void* scene, const double* from, const double* to,
                              uint32_t n_edges, int n, int two_stage, int early_exit,
                              uint8_t* out, uint64_t* stats) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        CollisionChecker c(m, *static_cast<Scene*>(scene));
        CheckStats st;
        std::vector<EdgeCheckRequest> reqs(n_edges);
        for (uint32_t e = 0; e < n_edges; ++e) {
            reqs[e].from.assign(from + size_t(e) * m.dof, from + size_t(e + 1) * m.dof);
            reqs[e].to.assign(to + size_t(e) * m.dof, to + size_t(e + 1) * m.dof);
            reqs[e].resolution_count = n;
        }
        auto v = c.validate_edge_batched(reqs, st, CheckOptions{two_stage != 0, early_exit != 0});
        std::copy(v.begin(), v.end(), out);
        put_stats(st, stats);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// nearest_serial (nn.cpp:22-29) over an AoS snapshot.
int64_t ref_nearest_serial(const double* cfgs, uint64_t count, uint32_t dof, const double* q,
                           double* dist) {
    try {
        auto r = nearest_serial(TreeView{cfgs, dof, count}, ConfigView(q, dof));
        if (dist) *dist = r.distance;
        return static_cast<int64_t>(r.index);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// nearest_parallel (nn.cpp:31-69).
int64_t ref_nearest_parallel(const double* cfgs, uint64_t count, uint32_t dof, const double* q,
                             uint64_t partitions, double* dist) {
    try {
        auto r = nearest_parallel(TreeView{cfgs, dof, count}, ConfigView(q, dof), partitions);
        if (dist) *dist = r.distance;
        return static_cast<int64_t>(r.index);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// sq_distance (nn.cpp:12-16) with the active backend.
double ref_sq_distance(const double* a, const double* b, uint32_t dof) {
    return sq_distance(ConfigView(a, dof), ConfigView(b, dof));
}

// halton_value (sampling.cpp:8-18).
double ref_halton_value(unsigned base, uint64_t index) { return halton_value(base, index); }

int ref_halton_bases(uint32_t n, uint32_t* out) {
    auto b = halton_bases(n);
    for (uint32_t i = 0; i < n; ++i) out[i] = b[i];
    return 0;
}

// sample_config (sampling.cpp:39-51): n draws at offset, offset+stride, ...
int ref_sample_config(void* robot, uint64_t offset, uint64_t stride, uint32_t n, double* out) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        auto lims = m.limits();
        HaltonState h = HaltonState::make(m.dof, offset, stride);
        for (uint32_t i = 0; i < n; ++i) {
            sample_config(h, lims, std::span<double>(out + size_t(i) * m.dof, m.dof));
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

static PlannerParams to_params(const prrtc_params* p) {
    PlannerParams q;
    q.delta = p->delta;
    q.n_cc = p->n_cc;
    q.workers = p->workers;
    q.max_iters_per_worker = p->max_iters_per_worker;
    q.tree_capacity = p->tree_capacity;
    q.dd_radius = p->dd_radius;
    q.dynamic_domain = p->dynamic_domain != 0;
    q.balance = p->balance != 0;
    q.early_exit = p->early_exit != 0;
    q.two_stage = p->two_stage != 0;
    q.batched_cc = p->batched_cc != 0;
    q.nn_partitions = p->nn_partitions;
    q.sampler = p->sampler == PRRTC_SAMPLER_UNIFORM ? SamplerKind::Uniform : SamplerKind::Halton;
    q.seed = p->seed;
    return q;
}

static void to_result(const PlanResult& r, int dof, prrtc_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->status = r.status == PlanStatus::Solved   ? PRRTC_SOLVED
                  : r.status == PlanStatus::Failed ? PRRTC_FAILED
                                                   : PRRTC_INFEASIBLE_ENDPOINT;
    out->dof = dof;
    out->path_len = static_cast<uint32_t>(r.path.size());
    if (!r.path.empty()) {
        out->path = static_cast<double*>(std::malloc(sizeof(double) * dof * r.path.size()));
        for (size_t i = 0; i < r.path.size(); ++i) {
            std::copy(r.path[i].begin(), r.path[i].end(), out->path + i * dof);
        }
    }
    out->cost = r.cost;
    out->wall_time_ms = r.wall_time_ms;
    out->iterations_total = r.iterations_total;
    out->sphere_tests = r.check_stats.sphere_tests;
    out->fk_calls = r.check_stats.fk_calls;
    out->fine_stage_entries = r.check_stats.fine_stage_entries;
    out->solving_worker = r.solving_worker;
    std::snprintf(out->message, sizeof(out->message), "%s", r.message.c_str());
}

void ref_result_free(prrtc_result* r) {
    if (r && r->path) {
        std::free(r->path);
        r->path = nullptr;
    }
}

// plan (planner.cpp:246-322). Returns 0, or -1 for std::invalid_argument.
int ref_plan(void* robot, void* scene, const double* start, const double* goal,
             const prrtc_params* params, prrtc_result* out) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        auto r = plan(m, *static_cast<Scene*>(scene), ConfigView(start, m.dof),
                      ConfigView(goal, m.dof), to_params(params));
        to_result(r, m.dof, out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// n independent problems on n_threads host threads (each plan() call uses
// params->workers workers, normally 1). The bench's CPU-throughput baseline.
// Returns the wall time in ms of the whole batch.
double ref_plan_many(void* robot, void* const* scenes, uint32_t n, const double* starts,
                     const double* goals, const prrtc_params* params, uint32_t n_threads,
                     prrtc_result* out) {
    const auto& m = *static_cast<RobotModel*>(robot);
    const PlannerParams pp = to_params(params);
    std::atomic<uint32_t> next{0};
    auto work = [&]() {
        for (;;) {
            uint32_t i = next.fetch_add(1);
            if (i >= n) break;
            try {
                auto r = plan(m, *static_cast<Scene*>(scenes[i]),
                              ConfigView(starts + size_t(i) * m.dof, m.dof),
                              ConfigView(goals + size_t(i) * m.dof, m.dof), pp);
                to_result(r, m.dof, &out[i]);
            } catch (const std::exception& e) {
                std::memset(&out[i], 0, sizeof(out[i]));
                out[i].status = -1;
                std::snprintf(out[i].message, sizeof(out[i].message), "%s", e.what());
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (uint32_t t = 1; t < std::max(1u, n_threads); ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
        .count();
}

// Soundness re-validation: every consecutive edge of the path
// with the fine-only, early-exit-off checker at `n` samples. 1 = valid.
int ref_path_valid(void* robot, void* scene, const double* path, uint32_t len, int n) {
    try {
        const auto& m = *static_cast<RobotModel*>(robot);
        CollisionChecker c(m, *static_cast<Scene*>(scene));
        CheckStats st;
        const CheckOptions opt{false, false};
        if (len == 0) return 0;
        if (!c.check_config(ConfigView(path, m.dof), st, opt)) return 0;
        for (uint32_t i = 1; i < len; ++i) {
            if (!c.validate_edge(ConfigView(path + size_t(i - 1) * m.dof, m.dof),
                                 ConfigView(path + size_t(i) * m.dof, m.dof), n, st, opt)) {
                return 0;
            }
        }
        return 1;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ref_path_valid over many paths (path i = doubles [off[i], off[i+1]) of
// path_data, scene i) on n_threads host threads: out[i] = 1 valid, 0 invalid
// or empty, 2 error. The per-path check is the reference checker exactly as
// in ref_path_valid (fine-only, early exit off).
int ref_paths_valid_many(void* robot, void* const* scenes, uint32_t n, const double* path_data,
                         const uint64_t* off, int n_cc, uint32_t n_threads, uint8_t* out) {
    const auto& m = *static_cast<RobotModel*>(robot);
    std::atomic<uint32_t> next{0};
    auto work = [&]() {
        for (;;) {
            const uint32_t i = next.fetch_add(1);
            if (i >= n) break;
            const uint32_t len = (uint32_t)((off[i + 1] - off[i]) / m.dof);
            const int r = ref_path_valid(robot, scenes[i], path_data + off[i], len, n_cc);
            out[i] = r < 0 ? 2 : (uint8_t)r;
        }
    };
    std::vector<std::thread> th;
    for (uint32_t t = 1; t < std::max(1u, n_threads); ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    return 0;
}

// path_cost (planner.cpp:152-158) with the active backend.
double ref_path_cost(const double* path, uint32_t len, uint32_t dof) {
    std::vector<Config> p;
    for (uint32_t i = 0; i < len; ++i) p.emplace_back(path + size_t(i) * dof, path + size_t(i + 1) * dof);
    return path_cost(p);
}

}  // extern "C"
