// prrtc_dropin.cpp — reference-typed C++ host side over the C-ABI.
//
// Converts the reference's RobotModel / Scene / PlannerParams (robot.hpp,
// geometry.hpp, planner.hpp) into the flat C-ABI descriptors, caches the
// uploaded device copies (setup, untimed in the reference methodology,
// PAPER.md:201), calls prrtc_plan / prrtc_plan_batch, and converts the result
// back into PlanResult. Errors map back to the reference's exceptions.
#include "prrtc_dropin.hpp"

#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "prrtc_b200.h"

namespace prrtc::b200 {
namespace {

// Concurrency (the reference's plan() is safe to call from many threads,
// planner.cpp:246-322): the handle caches are guarded per device and only
// while a handle is looked up or created; the plan call itself runs
// unlocked (the C-ABI serialises calls per device on its workspace), so one
// host thread per GPU plans in parallel. The device is the calling thread's
// choice (set_thread_device) or else the process default (set_device).
constexpr int kMaxDev = 64;
std::mutex g_cache_mu[kMaxDev];
std::atomic<int> g_default_device{0};
thread_local int t_device = -1;

int current_device() {
    const int d = t_device >= 0 ? t_device : g_default_device.load(std::memory_order_relaxed);
    if (d < 0 || d >= kMaxDev) throw std::invalid_argument("prrtc_b200: device ordinal out of range");
    return d;
}

std::string last_error() {
    char buf[512];
    prrtc_last_error(buf, sizeof(buf));
    return buf;
}

[[noreturn]] void raise(int rc) {
    if (rc == PRRTC_EINVAL) throw std::invalid_argument(last_error());
    throw std::runtime_error("prrtc_b200: " + last_error());
}

// FNV-1a over the bytes of every field the device copy depends on.
struct Hasher {
    uint64_t h = 1469598103934665603ull;
    void bytes(const void* p, size_t n) {
        const auto* c = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
    }
    template <class T>
    void v(const T& x) { bytes(&x, sizeof(x)); }
};

uint64_t fingerprint(const RobotModel& m) {
    Hasher h;
    for (const Joint& j : m.joints) {
        h.v(j.kind); h.v(j.parent); h.v(j.origin.rotation.w); h.v(j.origin.rotation.x);
        h.v(j.origin.rotation.y); h.v(j.origin.rotation.z); h.v(j.origin.translation.x);
        h.v(j.origin.translation.y); h.v(j.origin.translation.z); h.v(j.axis.x); h.v(j.axis.y);
        h.v(j.axis.z); h.v(j.lo); h.v(j.hi);
    }
    for (const LinkSpheres& ls : m.spheres) {
        h.v(ls.coarse.center.x); h.v(ls.coarse.center.y); h.v(ls.coarse.center.z); h.v(ls.coarse.radius);
        for (const Sphere& f : ls.fine) {
            h.v(f.center.x); h.v(f.center.y); h.v(f.center.z); h.v(f.radius);
        }
        h.v(ls.fine.size());
    }
    for (const auto& p : m.self_pairs) { h.v(p.first); h.v(p.second); }
    return h.h;
}

struct SceneFlat {
    std::vector<double> s, b, c;
};

SceneFlat flatten(const Scene& scene) {  // SceneIndex grouping (geometry.cpp:68-99)
    SceneFlat f;
    for (const Primitive& p : scene.primitives) {
        if (const auto* s = std::get_if<SpherePrim>(&p)) {
            f.s.insert(f.s.end(), {s->center.x, s->center.y, s->center.z, s->radius});
        } else if (const auto* b = std::get_if<BoxPrim>(&p)) {
            f.b.insert(f.b.end(), {b->pose.rotation.w, b->pose.rotation.x, b->pose.rotation.y,
                                   b->pose.rotation.z, b->pose.translation.x, b->pose.translation.y,
                                   b->pose.translation.z, b->half_extents.x, b->half_extents.y,
                                   b->half_extents.z});
        } else {
            const auto& c = std::get<CapsulePrim>(p);
            f.c.insert(f.c.end(), {c.a.x, c.a.y, c.a.z, c.b.x, c.b.y, c.b.z, c.radius});
        }
    }
    return f;
}

uint64_t fingerprint(const SceneFlat& f) {
    Hasher h;
    h.bytes(f.s.data(), 8 * f.s.size());
    h.v(f.s.size());
    h.bytes(f.b.data(), 8 * f.b.size());
    h.v(f.b.size());
    h.bytes(f.c.data(), 8 * f.c.size());
    h.v(f.c.size());
    return h.h;
}

struct RobotEntry {
    uint64_t fp;
    prrtc_robot* h;
};
struct SceneEntry {
    uint64_t fp;
    prrtc_scene* h;
};
std::map<std::pair<const RobotModel*, int>, RobotEntry> g_robots;
std::map<std::pair<const Scene*, int>, SceneEntry> g_scenes;

// (caller holds g_cache_mu[device])
prrtc_robot* robot_handle(const RobotModel& m, int device) {
    const uint64_t fp = fingerprint(m);
    auto key = std::make_pair(&m, device);
    auto it = g_robots.find(key);
    if (it != g_robots.end() && it->second.fp == fp) return it->second.h;
    const size_t L = m.joints.size();
    if (m.spheres.size() != L)
        throw std::invalid_argument("robot '" + m.name + "': spheres must have one entry per joint");
    std::vector<int32_t> kind(L), parent(L), pairs;
    std::vector<double> oq(4 * L), ox(3 * L), axis(3 * L), lo(L), hi(L), coarse(4 * L), fine;
    std::vector<uint32_t> foff(L + 1, 0);
    for (size_t i = 0; i < L; ++i) {
        const Joint& j = m.joints[i];
        kind[i] = j.kind == JointKind::Revolute ? PRRTC_JOINT_REVOLUTE
                  : j.kind == JointKind::Prismatic ? PRRTC_JOINT_PRISMATIC
                                                   : PRRTC_JOINT_FIXED;
        parent[i] = j.parent;
        oq[4 * i] = j.origin.rotation.w;
        oq[4 * i + 1] = j.origin.rotation.x;
        oq[4 * i + 2] = j.origin.rotation.y;
        oq[4 * i + 3] = j.origin.rotation.z;
        ox[3 * i] = j.origin.translation.x;
        ox[3 * i + 1] = j.origin.translation.y;
        ox[3 * i + 2] = j.origin.translation.z;
        axis[3 * i] = j.axis.x;
        axis[3 * i + 1] = j.axis.y;
        axis[3 * i + 2] = j.axis.z;
        lo[i] = j.lo;
        hi[i] = j.hi;
        const LinkSpheres& ls = m.spheres[i];
        coarse[4 * i] = ls.coarse.center.x;
        coarse[4 * i + 1] = ls.coarse.center.y;
        coarse[4 * i + 2] = ls.coarse.center.z;
        coarse[4 * i + 3] = ls.coarse.radius;
        for (const Sphere& f : ls.fine) fine.insert(fine.end(), {f.center.x, f.center.y, f.center.z, f.radius});
        foff[i + 1] = foff[i] + static_cast<uint32_t>(ls.fine.size());
    }
    for (const auto& p : m.self_pairs) pairs.insert(pairs.end(), {p.first, p.second});
    prrtc_robot_desc d{};
    d.n_links = static_cast<uint32_t>(L);
    d.kind = kind.data();
    d.parent = parent.data();
    d.origin_quat = oq.data();
    d.origin_xyz = ox.data();
    d.axis = axis.data();
    d.lo = lo.data();
    d.hi = hi.data();
    d.coarse = coarse.data();
    d.fine_offset = foff.data();
    d.fine = fine.data();
    d.n_self_pairs = static_cast<uint32_t>(m.self_pairs.size());
    d.self_pairs = pairs.data();
    prrtc_robot* h = nullptr;
    const int rc = prrtc_robot_create(&d, device, &h);
    if (rc) raise(rc);
    if (it != g_robots.end()) prrtc_robot_destroy(it->second.h);
    g_robots[key] = {fp, h};
    return h;
}

// (caller holds g_cache_mu[device])
prrtc_scene* scene_handle(const Scene& s, int device) {
    const SceneFlat f = flatten(s);
    const uint64_t fp = fingerprint(f);
    auto key = std::make_pair(&s, device);
    auto it = g_scenes.find(key);
    if (it != g_scenes.end() && it->second.fp == fp) return it->second.h;
    prrtc_scene_desc d{};
    d.n_spheres = static_cast<uint32_t>(f.s.size() / 4);
    d.spheres = f.s.data();
    d.n_boxes = static_cast<uint32_t>(f.b.size() / 10);
    d.boxes = f.b.data();
    d.n_capsules = static_cast<uint32_t>(f.c.size() / 7);
    d.capsules = f.c.data();
    prrtc_scene* h = nullptr;
    int rc;
    if (it != g_scenes.end()) {  // same Scene object, new content: dynamic obstacles
        rc = prrtc_scene_update(it->second.h, &d);
        if (rc) raise(rc);
        it->second.fp = fp;
        return it->second.h;
    }
    rc = prrtc_scene_create(&d, device, &h);
    if (rc) raise(rc);
    g_scenes[key] = {fp, h};
    return h;
}

prrtc_params to_c(const PlannerParams& p) {
    prrtc_params c;
    prrtc_params_default(&c);
    c.delta = p.delta;
    c.n_cc = p.n_cc;
    c.workers = p.workers;
    c.max_iters_per_worker = p.max_iters_per_worker;
    c.tree_capacity = p.tree_capacity;
    c.dd_radius = p.dd_radius;
    c.dynamic_domain = p.dynamic_domain;
    c.balance = p.balance;
    c.early_exit = p.early_exit;
    c.two_stage = p.two_stage;
    c.batched_cc = p.batched_cc;
    c.nn_partitions = p.nn_partitions;
    c.sampler = p.sampler == SamplerKind::Uniform ? PRRTC_SAMPLER_UNIFORM : PRRTC_SAMPLER_HALTON;
    c.seed = p.seed;
    return c;
}

PlanResult from_c(prrtc_result& r) {
    PlanResult out;
    out.status = r.status == PRRTC_SOLVED   ? PlanStatus::Solved
                 : r.status == PRRTC_FAILED ? PlanStatus::Failed
                                            : PlanStatus::InfeasibleEndpoint;
    for (uint32_t i = 0; i < r.path_len; ++i)
        out.path.emplace_back(r.path + static_cast<size_t>(i) * r.dof, r.path + static_cast<size_t>(i + 1) * r.dof);
    out.cost = r.cost;
    out.wall_time_ms = r.wall_time_ms;
    out.iterations_total = r.iterations_total;
    out.check_stats.sphere_tests = r.sphere_tests;
    out.check_stats.fk_calls = r.fk_calls;
    out.check_stats.fine_stage_entries = r.fine_stage_entries;
    out.solving_worker = r.solving_worker;
    out.message = r.message;
    prrtc_result_free(&r);
    return out;
}

}  // namespace

void set_device(int device) {
    if (device < 0 || device >= kMaxDev) throw std::invalid_argument("prrtc_b200: device ordinal out of range");
    g_default_device.store(device, std::memory_order_relaxed);
}

void set_thread_device(int device) {
    if (device >= kMaxDev) throw std::invalid_argument("prrtc_b200: device ordinal out of range");
    t_device = device;
}

void clear_cache() {
    for (int d = 0; d < kMaxDev; ++d) {
        std::lock_guard<std::mutex> lk(g_cache_mu[d]);
        for (auto it = g_robots.begin(); it != g_robots.end();) {
            if (it->first.second == d) {
                prrtc_robot_destroy(it->second.h);
                it = g_robots.erase(it);
            } else {
                ++it;
            }
        }
        for (auto it = g_scenes.begin(); it != g_scenes.end();) {
            if (it->first.second == d) {
                prrtc_scene_destroy(it->second.h);
                it = g_scenes.erase(it);
            } else {
                ++it;
            }
        }
    }
}

PlanResult plan(const RobotModel& model, const Scene& scene, ConfigView start, ConfigView goal,
                const PlannerParams& params) {
    require_dim(start, static_cast<size_t>(model.dof), "plan.start");  // planner.cpp:248-249
    require_dim(goal, static_cast<size_t>(model.dof), "plan.goal");
    const int dev = current_device();
    prrtc_robot* r;
    prrtc_scene* s;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu[dev]);
        r = robot_handle(model, dev);
        s = scene_handle(scene, dev);
    }
    const prrtc_params p = to_c(params);
    prrtc_result res{};
    const int rc = prrtc_plan(r, s, start.data(), goal.data(), static_cast<uint32_t>(start.size()), &p, &res);
    if (rc) raise(rc);
    return from_c(res);
}

namespace {
void flatten_inputs(const RobotModel& model, const std::vector<const Scene*>& scenes,
                    const std::vector<Config>& starts, const std::vector<Config>& goals, std::vector<double>& S,
                    std::vector<double>& G) {
    if (scenes.size() != starts.size() || starts.size() != goals.size())
        throw std::invalid_argument("plan_batch: scenes, starts and goals must have the same length");
    for (size_t i = 0; i < scenes.size(); ++i) {
        require_dim(starts[i], static_cast<size_t>(model.dof), "plan.start");
        require_dim(goals[i], static_cast<size_t>(model.dof), "plan.goal");
        S.insert(S.end(), starts[i].begin(), starts[i].end());
        G.insert(G.end(), goals[i].begin(), goals[i].end());
    }
}
}  // namespace

std::vector<PlanResult> plan_batch(const RobotModel& model, const std::vector<const Scene*>& scenes,
                                   const std::vector<Config>& starts, const std::vector<Config>& goals,
                                   const PlannerParams& params) {
    std::vector<double> S, G;
    flatten_inputs(model, scenes, starts, goals, S, G);
    const int dev = current_device();
    prrtc_robot* r;
    std::vector<const prrtc_scene*> sh;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu[dev]);
        r = robot_handle(model, dev);
        for (const Scene* sc : scenes) sh.push_back(scene_handle(*sc, dev));
    }
    const prrtc_params p = to_c(params);
    std::vector<prrtc_result> res(scenes.size());
    const int rc = prrtc_plan_batch(r, sh.data(), static_cast<uint32_t>(sh.size()), S.data(), G.data(),
                                    static_cast<uint32_t>(model.dof), &p, res.data());
    if (rc) raise(rc);
    std::vector<PlanResult> out;
    for (auto& x : res) out.push_back(from_c(x));
    return out;
}

std::vector<PlanResult> plan_batch(const RobotModel& model, const std::vector<const Scene*>& scenes,
                                   const std::vector<Config>& starts, const std::vector<Config>& goals,
                                   const PlannerParams& params, const std::vector<int>& devices,
                                   uint32_t chunk) {
    if (devices.empty()) throw std::invalid_argument("plan_batch: no devices");
    std::vector<double> S, G;
    flatten_inputs(model, scenes, starts, goals, S, G);
    std::vector<const prrtc_robot*> rs;
    std::vector<const prrtc_scene*> sh;
    for (int dev : devices) {
        if (dev < 0 || dev >= kMaxDev) throw std::invalid_argument("prrtc_b200: device ordinal out of range");
        std::lock_guard<std::mutex> lk(g_cache_mu[dev]);
        rs.push_back(robot_handle(model, dev));
        for (const Scene* sc : scenes) sh.push_back(scene_handle(*sc, dev));
    }
    const prrtc_params p = to_c(params);
    std::vector<prrtc_result> res(scenes.size());
    const int rc = prrtc_plan_batch_multi(rs.data(), sh.data(), static_cast<uint32_t>(devices.size()),
                                          static_cast<uint32_t>(scenes.size()), S.data(), G.data(),
                                          static_cast<uint32_t>(model.dof), &p, chunk, res.data());
    if (rc) raise(rc);
    std::vector<PlanResult> out;
    for (auto& x : res) out.push_back(from_c(x));
    return out;
}

}  // namespace prrtc::b200
