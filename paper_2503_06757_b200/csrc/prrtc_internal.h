// prrtc_internal.h — layouts shared by the host C-ABI (prrtc_capi.cu) and the
// sm_100a kernels (prrtc_kernels.cu). Not part of the public ABI.
//
// Data layout in HBM:
//   robot  : one packed 32-bit word buffer (header + per-link info + FP32
//            geometry + fine spheres + self pairs) copied whole into shared
//            memory by every CTA; FP64 fine radii / limits stay in global.
//   scene  : one packed FP32 word buffer (≤ PRRTC_MAX_PRIMS primitives, staged
//            in shared memory) + an FP64 mirror read only by the guard-band
//            fallback of the exact predicates.
//   trees  : per problem, per tree (start=0, goal=1): FP64 SoA configs
//            cfg[dof][cap], int32 parent[cap], uint32 ready[cap] (epoch
//            tagged), uint8-as-int32 dynamic-domain flag[cap].
//   control: one ProbCtl (128 B) per problem: counters, flags, result.
#pragma once
#include <stdint.h>

namespace prrtc_b200 {

// ---- robot words ----
enum RobotHdr : int {
    RH_NLINKS = 0,
    RH_DOF,
    RH_NFINE,
    RH_NPAIRS,
    RH_MAXFINE,
    RH_WORDS,     // total words of the packed buffer
    RH_OFF_INFO,  // int[L][4]: kind, parent, q_index, fine_off
    RH_OFF_NFINE, // int[L]
    RH_OFF_GEO,   // float[L][GEO_STRIDE]
    RH_OFF_FINE,  // float4[S] (link-frame center, radius)
    RH_OFF_PAIRS, // int2[n_pairs]
    RH_OFF_BASES, // uint32[dof] Halton bases
    RH_OFF_FLINK, // int[S] link of each fine sphere
    RH_FKFLOPS,   // algorithmic FP32 flops of FK + coarse posing per state
    RH_OFF_MAGIC, // uint64[dof] ceil(2^64 / base): exact 32-bit division by the Halton bases
    RH_OFF_FUNITS, // int2[n]: fine-stage work units (link, first sphere | count << 16), <= 3 spheres each
    RH_NFUNITS,
    RH_COUNT = 16
};

// per-link FP32 geometry (GEO_STRIDE floats). Revolute local rotation
// R_o * Rodrigues(a, q) = cos(q) M1 + sin(q) M2 + (1 - cos(q)) M3
// (transform.hpp:56-66 expanded):
//   [0..8]   M1 = R_o            (origin rotation, row major)
//   [9..17]  M2 = R_o [a]x
//   [18..26] M3 = (R_o a) a^T
//   [27..29] t_o                 (origin translation)
//   [30..32] v = R_o a           (prismatic: t_local = t_o + v q)
//   [33..35] coarse center (link frame)
//   [36]     coarse radius
constexpr int GEO_STRIDE = 40;

// ---- scene words ----
enum SceneHdr : int {
    SH_NS = 0,
    SH_NB,
    SH_NC,
    SH_WORDS,
    SH_OFF_S,  // float4[ns]: x,y,z,r
    SH_OFF_B,  // float[nb][16]: M(world->box, 9), t(3), h(3), pad
    SH_OFF_C,  // float[nc][8]: a(3), ab(3), inv_ab2, r
    SH_EPS,    // float bits: guard band (m)
    SH_CPAD,   // float bits: coarse padding (m)
    SH_NY,     // cylinders (extension)
    SH_OFF_Y,  // float[ny][16]: M(world->cylinder, 9), t(3), r, h, pad
    SH_COUNT = 12
};
constexpr int BOX_STRIDE = 16;
constexpr int CAP_STRIDE = 8;
constexpr int CYL_STRIDE = 16;
constexpr int SCENE_MAX_WORDS = SH_COUNT + 16 * 64 + 4;  // ≤ PRRTC_MAX_PRIMS boxes

// FP64 mirror: spheres [ns][4], boxes [nb][16], capsules [nc][8], same order.
struct SceneF64 {
    const double* s;
    const double* b;
    const double* c;
    const double* y;  // cylinders: m[9], t[3], r, h (CYL_STRIDE)
};

// ---- per-problem control block ----
struct ProbCtl {
    int started;      // 1 once roots are written
    int done;         // 0 running, 1 solved, 2 failed, 3 infeasible endpoint
    int winner;       // 1 + CTA id that connected, 0 = none
    int active;       // CTAs currently working on it
    int reserved[2];  // tree slot reservation counters
    int published[2]; // fully-ready prefix lengths
    unsigned long long iters_used;  // iterations actually run (tickets are claimed in blocks)
    unsigned long long iters;
    unsigned long long sphere_tests;
    unsigned long long fk_calls;
    unsigned long long fine_entries;
    unsigned long long flops;     // algorithmic FP32 flops
    int meet[2];
    unsigned long long path_off;  // doubles into the path arena
    int path_len;
    int msg;          // 0 none, 1 start infeasible, 2 goal infeasible, 3 capacity, 4 budget, 5 path arena
    long long t_start_ns;
    long long t_end_ns;
    int path_bad;     // validate_paths_kernel: some edge of the returned path collides
    int inv_bad;      // PRRTC_DEBUG_FLAGS bit 2: tree invariant violations seen at snapshots
};
static_assert(sizeof(ProbCtl) <= 128, "ProbCtl must fit 128 bytes");

struct PlanParamsDev {
    double delta;
    double dd_radius;
    int n_cc;
    int dynamic_domain;
    int balance;
    int early_exit;
    int two_stage;
    int deterministic;
    unsigned long long budget;  // total iterations per problem
    unsigned long long seed;
    int uniform;                // SamplerKind::Uniform (else Halton)
};

// Halton reciprocal-power table length per dimension: stored after the
// [dof][2] limits in the robot's device buffer (prrtc_robot_create).
constexpr int HALTON_TAB = 40;

struct PlanArgs {
    const uint32_t* robot;     // packed robot words
    const double* fine_r64;    // [S]
    const double* limits;      // [dof][2]
    const uint32_t* const* scene_words;  // per scene
    const SceneF64* scene_f64;           // per scene
    const int* prob_scene;     // [n] scene index
    const double* starts;      // [n][dof]
    const double* goals;       // [n][dof]
    int n_problems;
    ProbCtl* ctl;              // [n]
    double* cfg;               // [n][2][dof][cap]
    int* parent;               // [n][2][cap]
    unsigned* ready;           // [n][2][cap]
    int* dd;                   // [n][2][cap]
    long long cap;             // per tree (planner.cpp:290), fullness limit
    long long stride;          // per tree allocation stride (multiple of 32)
    double* arena;             // path arena (doubles)
    unsigned long long* arena_used;
    unsigned long long arena_cap;
    int* next_problem;         // unstarted-problem ticket
    int* n_done;               // finished problems (helpers exit when all are done)
    unsigned long long* trace; // [2]: LLONG_MAX - first CTA start, last CTA exit (globaltimer ns)
    long long* cta_trace;      // [grid][4]: per-CTA stamps (PRRTC_TRACE only, else null)
    unsigned epoch;
    unsigned dbg;              // PRRTC_DEBUG_FLAGS: bit 0 = fence at every snapshot (protocol check; 0 in
                               // production); bit 2 = check the trees' invariants at every snapshot
    PlanParamsDev p;
    int ns_max;                // states per validation chunk
    int nthreads;
    // single-problem result publication (null out_map: the host copies back):
    // the last CTA to finish copies the out-header, controls and used arena
    // to out_map + 64 (mapped pinned host memory) and raises out_map[0] = epoch
    unsigned char* out_map;
    unsigned long long out_map_bytes;
    const unsigned char* out_dev;       // device out-header; controls and arena follow contiguously
    unsigned long long out_hdr_bytes;   // 128 + sizeof(ProbCtl) * n_problems
    unsigned* exit_count;               // CTAs finished (zeroed with the controls)
    int mnn_nodes;                      // multi-sample NN bound: m <= mnn_nodes / tree size
    int ref_stats;                      // exact CheckStats (reference counting semantics): deterministic mode
    int tail_claim;                     // smaller ticket blocks near a problem's budget end
    int tail_min, tail_div;             // ... block = max(tail_min, min(32, unclaimed / (tail_div * workers)))
    int scene_words_max;                // warp-worker planner: words of the largest bound scene
    int help_cap;                       // help mode joins only problems with fewer active workers (0 = any)
    int help_policy;                    // which problem help joins: 1 most unclaimed budget per worker, 0 fewest workers
    // Halton samples of tickets [0, stab_n): [ticket][dof], computed once per
    // (robot, seed) by the planner's own sampler (null: compute in the loop)
    const double* stab;
    unsigned long long stab_n;
    // single-problem launches with inline inputs (no H2D copy): start and goal
    // travel in the kernel parameters, CTA 0 zeroes the out-header and the
    // controls and releases *init_flag = epoch, the other CTAs acquire it
    int inline_inputs;
    unsigned* init_flag;
    const uint32_t* scene_words1;
    SceneF64 scene_f64_1;
    double in_sg[2 * 32];               // start[dof], then goal[dof]
};

// Dynamic shared memory bytes for a robot/scene/ns_max combination.
size_t plan_smem_bytes(int robot_words, int dof, int n_links, int ns_max, int nthreads);

}  // namespace prrtc_b200
