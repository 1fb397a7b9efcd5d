// prrtc_launch.h — host-side launchers of the sm_100a kernels
// (implemented in prrtc_kernels.cu, called by the C-ABI in prrtc_capi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "prrtc_internal.h"

namespace prrtc_b200 {

// Robot-side kernel inputs shared by every launcher.
struct RobotArgs {
    const uint32_t* words;  // packed robot (device)
    int n_words;
    const double* fine_r64; // device
    const double* limits;   // device [dof][2]
    int n_links, dof, n_fine;
    const uint32_t* host_words;  // the same packed robot on the host (launch sizing)
};

struct SceneArgs {
    const uint32_t* words;  // packed scene (device)
    SceneF64 f64;           // device
    int n_words;            // packed scene words (launch sizing)
};

size_t smem_bytes(const RobotArgs& r, int ns_max, int nthreads, int scene_words, bool with_mt);

// Persistent planner: grid CTAs solve a.n_problems problems.
cudaError_t launch_plan(const RobotArgs& r, PlanArgs a, int grid, cudaStream_t st);
// Warp-worker planner (batches): warps per CTA that fit the shared memory
// (one CTA per SM; 0 = does not fit), and its launch.
int warp_workers_per_sm(const uint32_t* robot_words_host, int scene_words_max, int max_smem);
cudaError_t launch_plan_warp(const RobotArgs& r, const uint32_t* robot_words_host, PlanArgs a, int grid, int warps,
                             cudaStream_t st);
// Device re-validation of the solved problems' paths (after launch_plan on
// the same stream): prefix = [n_problems + 1] ints of scratch.
cudaError_t launch_validate_paths(const RobotArgs& r, const PlanArgs& a, int* prefix, int grid, cudaStream_t st);
// Max co-resident planner CTAs per SM for this configuration.
int plan_occupancy(const RobotArgs& r, int ns_max, int nthreads, int scene_words, bool with_mt);

cudaError_t launch_check_configs(const RobotArgs& r, const SceneArgs& s, const double* q, int n,
                                 int two_stage, uint8_t* out, cudaStream_t st);
cudaError_t launch_validate_edges(const RobotArgs& r, const SceneArgs& s, const double* from,
                                  const double* to, int n_edges, int n_cc, int two_stage,
                                  int early_exit, uint8_t* out, cudaStream_t st,
                                  long long* prof = nullptr, unsigned long long* counters = nullptr);
cudaError_t launch_debug_check_edges(const RobotArgs& r, const SceneArgs& s, const double* from,
                                     const double* to, int n_edges, int n_cc, int two_stage,
                                     uint8_t* state_valid, float* fine_out, cudaStream_t st);
cudaError_t launch_debug_fk(const RobotArgs& r, const double* q, int n, float* fine_out,
                            float* coarse_out, cudaStream_t st);
cudaError_t launch_debug_hits(const SceneArgs& s, const float* centers, const double* radii,
                              int n, int n_prims, uint8_t* hits, cudaStream_t st);
cudaError_t launch_debug_nn_multi(const double* soa, long long cap, int count, int dof, const double* q,
                                  int nq, int group, uint32_t* idx, double* d2, cudaStream_t st);
cudaError_t launch_debug_halton(const uint32_t* bases, const uint64_t* idx, int n, double* out,
                                cudaStream_t st);
double measure_fp32_peak(int sms, cudaStream_t st);
double measure_fp64_peak(int sms, cudaStream_t st);
double measure_l2_gbs(int sms, cudaStream_t st);

cudaError_t launch_debug_sample(const RobotArgs& r, uint64_t index0, int n, double* out,
                                cudaStream_t st);

}  // namespace prrtc_b200
