/*
 * prrtc_b200.h — C-ABI boundary of the B200-native pRRTC planner.
 *
 * This is the drop-in boundary for the reference's planning call
 *
 *     prrtc::PlanResult prrtc::plan(const RobotModel&, const Scene&,
 *                                   ConfigView start, ConfigView goal,
 *                                   const PlannerParams&);
 *     (reference: proj/include/prrtc/planner.hpp:55-56, proj/src/planner.cpp:246-322)
 *
 * Everything below `plan()` (worker loop, sampling, nearest neighbour, steering,
 * edge validation, connect, termination) runs inside one persistent sm_100a
 * kernel. The host side only converts the reference types into the flat
 * descriptors below, uploads them once (setup, untimed in the reference's
 * methodology) and calls prrtc_plan / prrtc_plan_batch.
 *
 * Conventions
 *   - Plain C types only; no exceptions cross the ABI. Every entry point
 *     returns PRRTC_OK (0) or a negative error code; the message for the last
 *     failure on the calling thread is available from prrtc_last_error().
 *   - Error codes mirror the reference's error behaviour:
 *       PRRTC_EINVAL  <-> std::invalid_argument (types.hpp:16-21,
 *                         planner.cpp:248-252, kinematics.cpp:15-74,
 *                         geometry.cpp:10-39)
 *       PRRTC_ECUDA   a CUDA runtime failure (no reference equivalent)
 *       PRRTC_ENODEV  no usable sm_100 device: there is NO CPU fallback.
 *   - Planning outcomes are statuses, not errors (planner.hpp:15):
 *       PRRTC_SOLVED, PRRTC_FAILED, PRRTC_INFEASIBLE_ENDPOINT.
 *   - All configurations are FP64 (reference Config = std::vector<double>,
 *     types.hpp:13). Robot/scene handles are bound to one CUDA device.
 *   - Calls are synchronous (like the reference's plan(), which joins its
 *     workers before returning, planner.cpp:295-304). Handles are read-only
 *     during a plan call; concurrent calls on distinct handles are safe.
 */
#ifndef PRRTC_B200_H
#define PRRTC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRRTC_API_VERSION 2

/* Limits of the device implementation (checked at handle creation). */
#define PRRTC_MAX_DOF 32
#define PRRTC_MAX_LINKS 48
#define PRRTC_MAX_FINE_PER_LINK 64
#define PRRTC_MAX_FINE 512
#define PRRTC_MAX_PRIMS 64   /* primitives per scene, all kinds together */
#define PRRTC_MAX_SELF_PAIRS 512

/* ---- return codes ---- */
#define PRRTC_OK 0
#define PRRTC_EINVAL (-1)
#define PRRTC_ECUDA (-2)
#define PRRTC_ENODEV (-3)
#define PRRTC_ENOMEM (-4)
#define PRRTC_EINTERNAL (-5)

/* ---- plan statuses (reference PlanStatus, planner.hpp:15) ---- */
#define PRRTC_SOLVED 0
#define PRRTC_FAILED 1
#define PRRTC_INFEASIBLE_ENDPOINT 2

/* ---- joint kinds (reference JointKind, robot.hpp:12) ---- */
#define PRRTC_JOINT_REVOLUTE 0
#define PRRTC_JOINT_PRISMATIC 1
#define PRRTC_JOINT_FIXED 2

/* ---- samplers (reference SamplerKind, planner.hpp:19) ---- */
#define PRRTC_SAMPLER_HALTON 0
#define PRRTC_SAMPLER_UNIFORM 1

/*
 * Robot description: the flattened reference RobotModel (robot.hpp:44-71).
 * One joint per link; joint i defines the frame of link i; parent == -1 roots
 * a chain (forest allowed, robot.hpp:14-16). Validated with the same
 * invariants as RobotModel::finalize (kinematics.cpp:15-74).
 */
typedef struct prrtc_robot_desc {
    uint32_t n_links;            /* = joints.size() = spheres.size() */
    const int32_t* kind;         /* [n_links] PRRTC_JOINT_* */
    const int32_t* parent;       /* [n_links] -1 = world */
    const double* origin_quat;   /* [n_links*4] w,x,y,z   (Joint::origin.rotation) */
    const double* origin_xyz;    /* [n_links*3]           (Joint::origin.translation) */
    const double* axis;          /* [n_links*3] unit; ignored for fixed joints */
    const double* lo;            /* [n_links] limits; ignored for fixed joints */
    const double* hi;            /* [n_links] */
    const double* coarse;        /* [n_links*4] cx,cy,cz,r in link frame */
    const uint32_t* fine_offset; /* [n_links+1] prefix offsets into `fine` */
    const double* fine;          /* [fine_offset[n_links]*4] cx,cy,cz,r */
    uint32_t n_self_pairs;
    const int32_t* self_pairs;   /* [n_self_pairs*2] link indices */
} prrtc_robot_desc;

/*
 * Scene description: the reference Scene (geometry.hpp:37-46) grouped by
 * primitive kind, which is exactly how SceneIndex lays it out
 * (geometry.cpp:68-99). Boxes are given as pose (unit quaternion w,x,y,z +
 * translation) + half extents (geometry.hpp:20-25); capsules as endpoints a,b
 * + radius (geometry.hpp:27-33).
 */
typedef struct prrtc_scene_desc {
    uint32_t n_spheres;
    const double* spheres;   /* [n*4]  x,y,z,r */
    uint32_t n_boxes;
    const double* boxes;     /* [n*10] qw,qx,qy,qz, tx,ty,tz, hx,hy,hz */
    uint32_t n_capsules;
    const double* capsules;  /* [n*7]  ax,ay,az, bx,by,bz, r */
    /* Extension (BASELINE config 4; the reference has no cylinder primitive,
       geometry.hpp:35, so its verdicts are pinned to the C restatement only):
       solid cylinders about the pose's local z axis. */
    uint32_t n_cylinders;
    const double* cylinders; /* [n*9]  qw,qx,qy,qz, tx,ty,tz, radius, half_length */
} prrtc_scene_desc;

/*
 * Planner parameters: reference PlannerParams (planner.hpp:21-40), same
 * meaning and defaults, plus device knobs.
 *
 *  workers          reference: concurrent worker iterations (0 = hardware
 *                   concurrency). Here: CTAs working on one problem in
 *                   prrtc_plan (0 = one 512-thread CTA per SM). The per-problem iteration
 *                   budget is workers_effective * max_iters_per_worker.
 *  tree_capacity    total across both trees, split in half (planner.cpp:290).
 *  nn_partitions    accepted for API parity; the device scan always splits
 *                   the tree over all threads of a CTA (result identical by
 *                   construction, nn.cpp:31-69).
 */
typedef struct prrtc_params {
    double delta;                  /* 0.5 */
    int32_t n_cc;                  /* 32 */
    uint32_t workers;              /* 0 */
    uint64_t max_iters_per_worker; /* 2000 */
    uint64_t tree_capacity;        /* 200000 */
    double dd_radius;              /* <= 0 selects 4*delta */
    uint8_t dynamic_domain;        /* 1 */
    uint8_t balance;               /* 1 */
    uint8_t early_exit;            /* 1 */
    uint8_t two_stage;             /* 1 */
    uint8_t batched_cc;            /* 0 */
    uint8_t _pad[3];
    uint32_t nn_partitions;        /* 1 */
    int32_t sampler;               /* PRRTC_SAMPLER_HALTON */
    uint64_t seed;                 /* 0 */
    /* --- device knobs (no reference equivalent) --- */
    uint32_t threads_per_cta;      /* 0 = automatic: 512 for one problem; a batch runs on
                                      128-thread CTAs, or on the warp-worker planner (one
                                      worker per warp) when it holds at least as many
                                      problems as the device has warp workers and at
                                      least 2048; else 128, 256 or
                                      512, or 32 = the warp-worker planner (not for
                                      deterministic / Uniform-sampler runs) */
    uint32_t ctas_per_sm;          /* 0 = as many as co-reside */
    uint32_t deterministic;        /* 1 = single CTA, Halton stride 1: replays
                                      the reference's workers=1 mode */
    uint32_t validate_path;        /* 1 = sound mode: re-validate every path on the device
                                      at 4*n_cc states per edge, fine spheres only, no
                                      early exit, by a second kernel on the
                                      same stream (result: prrtc_result.path_check);
                                      prrtc_plan / prrtc_plan_batch re-plan a problem whose
                                      path fails it with the next seed (up to 4 times) and
                                      never return such a path (status FAILED instead) */
    uint32_t max_workers_per_problem; /* batches: the most workers (CTAs or warp workers)
                                      one problem may have at once. 0 = elastic: a worker
                                      that finds no unstarted problem joins the running
                                      problem with the fewest workers that still has
                                      budget (shorter batch tails, more parallel search).
                                      W = at most W; with workers = 1 and 1 here each
                                      problem runs exactly the reference's workers=1
                                      search (planner.cpp:186-242: Halton stream
                                      1+seed+k, same iterations, same result) */
    uint32_t _pad2;
} prrtc_params;

/* Result of one planning problem: reference PlanResult (planner.hpp:42-51). */
typedef struct prrtc_result {
    int32_t status;              /* PRRTC_SOLVED / FAILED / INFEASIBLE_ENDPOINT */
    uint32_t dof;
    uint32_t path_len;           /* number of configs */
    uint32_t path_block;         /* library-internal: a batch's paths share one host
                                    block (0 = the path is its own allocation) */
    double* path;                /* [path_len*dof], library-owned; free with
                                    prrtc_result_free() (never free() it: the paths
                                    of one batch call share a pinned block that
                                    lives until the last of them is freed) */
    double cost;                 /* arclength (planner.cpp:152-158) */
    double wall_time_ms;         /* host wall clock around the call */
    double device_time_ms;       /* CUDA-event time of the device work */
    uint64_t iterations_total;
    uint64_t sphere_tests;       /* CheckStats (collision.hpp:17-25) */
    uint64_t fk_calls;
    uint64_t fine_stage_entries;
    uint64_t flops;              /* algorithmic FP32 flops executed on the device
                                    (SURVEY.md §8d), for the roofline */
    uint64_t tree_nodes[2];      /* published nodes in start/goal tree */
    int32_t solving_worker;      /* CTA that connected the trees, -1 if none */
    uint32_t path_check;         /* validate_path: 0 not checked, 1 valid, 2 invalid */
    char message[128];
} prrtc_result;

typedef struct prrtc_robot prrtc_robot;
typedef struct prrtc_scene prrtc_scene;
typedef struct prrtc_batch prrtc_batch;

/* ---------------- library ---------------- */
int prrtc_api_version(void);
/* Copies the last error message of the calling thread (NUL-terminated). */
int prrtc_last_error(char* buf, size_t len);
/* Number of usable devices, or a negative error. */
int prrtc_device_count(void);
/* CTAs prrtc_plan puts on one problem for params.workers == 0 (the analogue of
 * the reference's hardware_concurrency default, planner.cpp:287-288); or an error. */
int prrtc_default_workers(int device);
/* Re-reads the PRRTC_* diagnostic environment switches,
   which the library otherwise reads once: for callers that change one
   in-process (tests). */
int prrtc_debug_reload_env(void);
/* Host<->device bytes the last prrtc_plan / prrtc_plan_batch call on this
 * device copied (inputs up; result header, controls and paths down). */
int prrtc_last_transfer_bytes(int device, uint64_t* h2d, uint64_t* d2h);
void prrtc_params_default(prrtc_params* p);

/* ---------------- setup (untimed) ---------------- */
/* Validates like RobotModel::finalize (kinematics.cpp:15-74) and uploads. */
int prrtc_robot_create(const prrtc_robot_desc* desc, int device, prrtc_robot** out);
int prrtc_robot_destroy(prrtc_robot* robot);
int prrtc_robot_dof(const prrtc_robot* robot);
int prrtc_robot_fine_count(const prrtc_robot* robot);
/* limits[2*dof] = lo,hi per actuated joint (RobotModel::limits, robot.hpp:57-64) */
int prrtc_robot_limits(const prrtc_robot* robot, double* limits);

/* Validates like Scene::validate (geometry.cpp:10-39) and uploads. */
int prrtc_scene_create(const prrtc_scene_desc* desc, int device, prrtc_scene** out);
/* Replaces the primitives of an existing scene (dynamic obstacles). The
   primitive count per kind may change within PRRTC_MAX_PRIMS. */
int prrtc_scene_update(prrtc_scene* scene, const prrtc_scene_desc* desc);
int prrtc_scene_destroy(prrtc_scene* scene);

/* ---------------- planning ---------------- */
/* Drop-in for prrtc::plan (planner.cpp:246-322). Host buffers in and out. */
int prrtc_plan(const prrtc_robot* robot, const prrtc_scene* scene, const double* start,
               const double* goal, uint32_t dof, const prrtc_params* params,
               prrtc_result* result);

/* n independent problems for one robot, each with its own scene; problems
   are spread over all SMs of the robot's device (one launch). out[n]. */
int prrtc_plan_batch(const prrtc_robot* robot, const prrtc_scene* const* scenes,
                     uint32_t n_problems, const double* starts, const double* goals,
                     uint32_t dof, const prrtc_params* params, prrtc_result* out);

/* n independent problems spread over several devices (the
   reference's plan() is safe to call concurrently, planner.cpp:246-322):
   one host thread per device pulls chunks of `chunk` consecutive problems
   from a shared atomic queue (0 = automatic: about 4 chunks per device, at
   least 64 problems) and solves each chunk with prrtc_plan_batch on its
   device, so a device that draws hard problems takes fewer chunks (the
   per-problem time is heavy-tailed). No collective and no cross-device
   traffic: handles are per device. robots[d] and scenes[d * n_problems + i]
   are the robot and problem i's scene uploaded to device d (d < n_devices,
   one entry per participating device, each on a distinct device). Results
   land in out[i] in caller order; on error the first failing device's code
   is returned and the other devices stop taking chunks. */
int prrtc_plan_batch_multi(const prrtc_robot* const* robots, const prrtc_scene* const* scenes,
                           uint32_t n_devices, uint32_t n_problems, const double* starts,
                           const double* goals, uint32_t dof, const prrtc_params* params,
                           uint32_t chunk, prrtc_result* out);
/* The chunk queue of prrtc_plan_batch_multi run without devices (host-side
   logic, testable anywhere): `n_workers` threads take chunks until
   n_problems are handed out; owner[i] = the worker that took problem i,
   chunks_taken[w] = chunks of worker w (worker w sleeps delay_us[w]
   microseconds per problem it takes, to emulate slow devices; may be NULL). */
int prrtc_debug_chunk_queue(uint32_t n_workers, uint32_t n_problems, uint32_t chunk,
                            const uint32_t* delay_us, int32_t* owner, uint32_t* chunks_taken);

void prrtc_result_free(prrtc_result* result);
/* Frees the paths of n results (prrtc_plan_batch output) in one call. */
void prrtc_results_free(prrtc_result* results, uint32_t n);
/* Copies the paths of n results back to back into out (doubles, config-major;
   NULL to only size) and writes offsets[n + 1] (in doubles). */
int prrtc_results_pack_paths(const prrtc_result* results, uint32_t n, double* out, uint64_t* offsets);

/* Device-resident batches: inputs uploaded once, then run repeatedly. Used to
   time the device work alone (bench `value`); prrtc_plan_batch is the same
   path with the copies inside. */
int prrtc_batch_create(const prrtc_robot* robot, const prrtc_scene* const* scenes,
                       uint32_t n_problems, const double* starts, const double* goals,
                       uint32_t dof, const prrtc_params* params, prrtc_batch** out);
/* Enqueues one full solve of every problem of the batch on `stream`
   (a cudaStream_t, 0 = legacy default). Asynchronous. */
int prrtc_batch_launch(prrtc_batch* batch, void* stream);
/* Waits for the batch and copies results out (out[n_problems]). */
int prrtc_batch_results(prrtc_batch* batch, prrtc_result* out);
/* Kernel launches enqueued by the last prrtc_batch_launch. */
int prrtc_batch_launch_count(const prrtc_batch* batch);
int prrtc_batch_destroy(prrtc_batch* batch);

/* ---------------- batched collision checking (product API) ---------------- */
/* Reference CollisionChecker::validate_edge_batched (collision.cpp:226-262):
   valid[e] = 1 iff every sample i/n_cc (i=1..n_cc, the far endpoint copied
   exactly) of from[e]->to[e] is collision-free. A bitwise-equal edge collapses
   to one check of `to` (collision.cpp:215). */
int prrtc_validate_edges(const prrtc_robot* robot, const prrtc_scene* scene,
                         const double* from, const double* to, uint32_t n_edges,
                         uint32_t dof, int32_t n_cc, int two_stage, int early_exit,
                         uint8_t* valid);
/* Reference CollisionChecker::check_config (collision.cpp:130-204). */
int prrtc_check_configs(const prrtc_robot* robot, const prrtc_scene* scene, const double* q,
                        uint32_t n_configs, uint32_t dof, int two_stage, uint8_t* valid);

/* ---------------- parity hooks ---------------- */
/* Posed fine (and coarse) spheres exactly as the device collision code sees
   them: centers from the FP32 FK, radii from the model (reference
   sphere_positions, kinematics.cpp:111-126). fine_out[n*S*3], coarse_out[n*L*3]
   (either may be NULL). */
int prrtc_debug_fk(const prrtc_robot* robot, const double* q, uint32_t n_configs,
                   uint32_t dof, float* fine_out, float* coarse_out);
/* Edge-level parity hook (CollisionChecker::validate_edge,
   collision.cpp:206-224): for every edge, every sample i = 1..n_cc
   (edge_sample, the far endpoint copied exactly) is checked on the device
   with no early exit; state_valid[e*n_cc + i-1] = the device's verdict of that
   state and fine_out[((e*n_cc + i-1)*S + j)*3 + k] = the posed centre of fine
   sphere j exactly as the device's collision code saw it (FP32; NULL to skip).
   The edge verdict of prrtc_validate_edges is the AND over its states (a
   bitwise-equal edge is one check of `to`, whose state is every sample). */
int prrtc_debug_check_edges(const prrtc_robot* robot, const prrtc_scene* scene, const double* from,
                            const double* to, uint32_t n_edges, uint32_t dof, int32_t n_cc, int two_stage,
                            uint8_t* state_valid, float* fine_out);
/* Per-(config, fine sphere, primitive) verdicts of the device predicate
   (FP32 with FP64 guard band) for posed spheres given in FP32: hits[n*P]
   with primitive order spheres, boxes, capsules. */
int prrtc_debug_sphere_hits(const prrtc_scene* scene, const float* centers,
                            const double* radii, uint32_t n_spheres, uint8_t* hits);
/* Device nearest-neighbour scan: tree[count*dof] AoS (reference TreeView,
   nn.hpp:21-25) uploaded into the SoA layout, one query per q[i*dof].
   Exact FP64 keys in the scalar op order (kernels_scalar.cpp:9-37), ties to
   the lowest index. */
int prrtc_debug_nn(const double* tree, uint32_t count, uint32_t dof, const double* q,
                   uint32_t n_queries, int device, uint32_t* index, double* sq_dist);
/* The planner's multi-sample NN pass: queries evaluated `group` (1..32) at a
   time against the same tree, as the planner evaluates the samples of a
   Halton ticket block; group 0 = 1 (prrtc_debug_nn). */
int prrtc_debug_nn_multi(const double* tree, uint32_t count, uint32_t dof, const double* q,
                         uint32_t n_queries, uint32_t group, int device, uint32_t* index, double* sq_dist);
/* Device Halton values (reference halton_value, sampling.cpp:8-18). */
int prrtc_debug_halton(const uint32_t* bases, const uint64_t* indices, uint32_t n, int device,
                       double* out);
/* Device sample_config (sampling.cpp:39-51): out[n*dof] for sequence indices
   index0 .. index0+n-1 against the robot's limits. */
int prrtc_debug_sample(const prrtc_robot* robot, uint64_t index0, uint32_t n, double* out);

/* clock64 stamps of one 32-state validation chunk in one CTA (latency
   profiling): [0] kernel start, [7] after setup, [8] after state generation,
   [1] check start, [2] FK local transforms, [3] FK compose, [4] FK done,
   [10] warp 0's coarse environment tests done, [11] its coarse self pairs
   done, [5] coarse stage done (all warps), [6] fine env stage done (if
   reached), [9] chunk done. */
int prrtc_debug_chunk_profile(const prrtc_robot* robot, const prrtc_scene* scene, const double* from,
                              const double* to, uint32_t dof, int32_t n_cc, int two_stage,
                              long long* stamps);

/* ---------------- measurement utility ---------------- */
/* FP32 FMA-pipe peak of the device in TFLOP/s, measured with an FFMA-chain
   microbenchmark (the roofline denominator of the FK / collision work). */
double prrtc_fp32_peak_tflops(int device);
/* FP64 peak in TFLOP/s from un-fused DMUL + DADD chains (the NN scan's keys:
   FP64 multiplies and adds in the reference's order, no FMA). */
double prrtc_fp64_peak_tflops(int device);
/* L2 read bandwidth of the device in GB/s (float4 streaming over a 32 MiB
   L2-resident buffer from 4 CTAs per SM): the NN scan's roofline denominator. */
double prrtc_l2_peak_gbs(int device);
/* Roofline microbenchmark of the collision path: the
   prrtc_validate_edges kernel over n_edges device-resident edges, `reps`
   timed launches after a warm-up (CUDA events). ms = mean per launch; flops /
   tests = algorithmic FLOPs and sphere tests of one launch (device counters;
   NULL to skip). Dense mode = two_stage 0, early_exit 0. */
int prrtc_bench_validate_edges(const prrtc_robot* robot, const prrtc_scene* scene, const double* from,
                               const double* to, uint32_t n_edges, uint32_t dof, int32_t n_cc, int two_stage,
                               int early_exit, int reps, double* ms, double* flops, double* tests);
/* NN scan throughput: n_queries queries over a count-node tree (AoS input,
   scanned in the planner's SoA FP64 layout), `group` queries per pass (the
   planner's multi-sample pass; 1 = one query per pass), `reps` timed
   launches. Algorithmic bytes per query = count * dof * 8. */
int prrtc_bench_nn(const double* tree, uint32_t count, uint32_t dof, const double* q, uint32_t n_queries,
                   uint32_t group, int device, int reps, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* PRRTC_B200_H */
