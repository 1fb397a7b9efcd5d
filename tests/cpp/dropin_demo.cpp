// tests/cpp/dropin_demo.cpp — TEST INFRASTRUCTURE.
//
// Exercises the C++ drop-in with the reference's own types: builds
// prrtc::RobotModel / prrtc::Scene (reference headers, RobotModel::finalize
// from the reference's kinematics.cpp compiled in place), then solves every
// problem with prrtc::b200::plan (B200) and prrtc::plan (reference CPU,
// workers = 1). One JSON line per problem on stdout.
//
// Input (whitespace separated, doubles printed with 17 significant digits):
//   L npairs
//   L x: kind parent qw qx qy qz tx ty tz ax ay az lo hi cx cy cz cr nfine {x y z r}*
//   npairs x: a b
//   N
//   N x: ns nb nc {x y z r}* {qw qx qy qz tx ty tz hx hy hz}* {ax ay az bx by bz r}* start goal
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <string>
#include <thread>
#include <vector>

#include "prrtc/planner.hpp"
#include "prrtc_dropin.hpp"

using namespace prrtc;

static void print_result(const char* impl, int i, const PlanResult& r, double ms) {
    std::printf("{\"impl\": \"%s\", \"problem\": %d, \"status\": %d, \"cost\": %.17g, \"iterations\": %llu, "
                "\"ms\": %.6f, \"message\": \"%s\", \"path\": [",
                impl, i, static_cast<int>(r.status), r.cost, static_cast<unsigned long long>(r.iterations_total),
                ms, r.message.c_str());
    for (size_t k = 0; k < r.path.size(); ++k) {
        std::printf("%s[", k ? ", " : "");
        for (size_t d = 0; d < r.path[k].size(); ++d) std::printf("%s%.17g", d ? ", " : "", r.path[k][d]);
        std::printf("]");
    }
    std::printf("]}\n");
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: dropin_demo <problems.txt> [workers]\n");
        return 2;
    }
    std::ifstream in(argv[1]);
    size_t L, np;
    in >> L >> np;
    RobotModel m;
    m.name = "dropin";
    for (size_t i = 0; i < L; ++i) {
        Joint j;
        int kind;
        in >> kind >> j.parent >> j.origin.rotation.w >> j.origin.rotation.x >> j.origin.rotation.y >>
            j.origin.rotation.z >> j.origin.translation.x >> j.origin.translation.y >> j.origin.translation.z >>
            j.axis.x >> j.axis.y >> j.axis.z >> j.lo >> j.hi;
        j.kind = kind == 0 ? JointKind::Revolute : kind == 1 ? JointKind::Prismatic : JointKind::Fixed;
        m.joints.push_back(j);
        LinkSpheres ls;
        size_t nf;
        in >> ls.coarse.center.x >> ls.coarse.center.y >> ls.coarse.center.z >> ls.coarse.radius >> nf;
        for (size_t k = 0; k < nf; ++k) {
            Sphere s;
            in >> s.center.x >> s.center.y >> s.center.z >> s.radius;
            ls.fine.push_back(s);
        }
        m.spheres.push_back(ls);
    }
    for (size_t p = 0; p < np; ++p) {
        int a, b;
        in >> a >> b;
        m.self_pairs.emplace_back(a, b);
    }
    m.finalize();  // reference kinematics.cpp:15-74
    size_t N;
    in >> N;
    PlannerParams b200p;      // reference defaults (planner.hpp:21-40)
    b200p.workers = argc > 2 ? static_cast<unsigned>(std::stoul(argv[2])) : 0;
    PlannerParams cpup;
    cpup.workers = 1;
    std::vector<Scene> scenes;
    std::vector<Config> starts, goals;
    scenes.reserve(N);
    for (size_t i = 0; i < N; ++i) {
        Scene sc;
        sc.name = "scene";
        size_t ns, nb, nc;
        in >> ns >> nb >> nc;
        for (size_t k = 0; k < ns; ++k) {
            SpherePrim s;
            in >> s.center.x >> s.center.y >> s.center.z >> s.radius;
            sc.primitives.push_back(s);
        }
        for (size_t k = 0; k < nb; ++k) {
            BoxPrim b;
            in >> b.pose.rotation.w >> b.pose.rotation.x >> b.pose.rotation.y >> b.pose.rotation.z >>
                b.pose.translation.x >> b.pose.translation.y >> b.pose.translation.z >> b.half_extents.x >>
                b.half_extents.y >> b.half_extents.z;
            sc.primitives.push_back(b);
        }
        for (size_t k = 0; k < nc; ++k) {
            CapsulePrim c;
            in >> c.a.x >> c.a.y >> c.a.z >> c.b.x >> c.b.y >> c.b.z >> c.radius;
            sc.primitives.push_back(c);
        }
        Config s(m.dof), g(m.dof);
        for (auto& v : s) in >> v;
        for (auto& v : g) in >> v;
        auto t0 = std::chrono::steady_clock::now();
        PlanResult rb = b200::plan(m, sc, s, g, b200p);
        double ms_b = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        print_result("b200", static_cast<int>(i), rb, ms_b);
        t0 = std::chrono::steady_clock::now();
        PlanResult rc = prrtc::plan(m, sc, s, g, cpup);
        double ms_c = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        print_result("reference", static_cast<int>(i), rc, ms_c);
        scenes.push_back(sc);
        starts.push_back(s);
        goals.push_back(g);
    }
    // concurrent callers (the reference's plan() is safe to call from many
    // threads): 4 host threads plan all problems at once on the thread's device
    {
        std::vector<int> st(N, -1);
        std::vector<std::thread> th;
        for (int t = 0; t < 4; ++t)
            th.emplace_back([&, t] {
                b200::set_thread_device(0);
                for (size_t i = t; i < N; i += 4) {
                    PlanResult r = b200::plan(m, scenes[i], starts[i], goals[i], b200p);
                    const bool ends = r.path.empty() || (r.path.front() == starts[i] && r.path.back() == goals[i]);
                    st[i] = ends ? static_cast<int>(r.status) : 9;
                }
            });
        for (auto& x : th) x.join();
        std::printf("{\"concurrent\": [");
        for (size_t i = 0; i < N; ++i) std::printf("%s%d", i ? ", " : "", st[i]);
        std::printf("]}\n");
    }
    // the multi-device batch entry on the visible device(s)
    {
        std::vector<const Scene*> sp;
        for (auto& sc : scenes) sp.push_back(&sc);
        std::vector<PlanResult> rs = b200::plan_batch(m, sp, starts, goals, b200p, std::vector<int>{0}, 2);
        std::printf("{\"multi\": [");
        for (size_t i = 0; i < rs.size(); ++i) {
            const bool ends = rs[i].path.empty() || (rs[i].path.front() == starts[i] && rs[i].path.back() == goals[i]);
            std::printf("%s%d", i ? ", " : "", ends ? static_cast<int>(rs[i].status) : 9);
        }
        std::printf("]}\n");
    }
    // the reference's error behaviour: a dimension mismatch throws std::invalid_argument
    try {
        Config bad(m.dof + 1, 0.0);
        b200::plan(m, Scene{}, bad, bad, b200p);
        std::printf("{\"invalid_argument\": false}\n");
    } catch (const std::invalid_argument& e) {
        std::printf("{\"invalid_argument\": true, \"what\": \"%s\"}\n", e.what());
    }
    b200::clear_cache();
    return 0;
}
