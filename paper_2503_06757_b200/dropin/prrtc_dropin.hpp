// prrtc_dropin.hpp — C++ drop-in for the reference's planning call.
//
// Same signature, types and error behaviour as
//   prrtc::PlanResult prrtc::plan(const RobotModel&, const Scene&, ConfigView,
//                                 ConfigView, const PlannerParams&)
//   (reference proj/include/prrtc/planner.hpp:55-56, proj/src/planner.cpp:246-322)
// computed by the B200 planner through the C-ABI (include/prrtc_b200.h).
//
// Build against the reference's own headers (-I proj/include); see
// INTEGRATION.md for the one-line switch in a reference build.
#pragma once

#include "prrtc/planner.hpp"

namespace prrtc::b200 {

// Drop-in for prrtc::plan. Throws std::invalid_argument exactly where the
// reference does (types.hpp:16-21, planner.cpp:248-252, RobotModel::finalize
// invariants); std::runtime_error if no sm_100 device is usable (there is no
// CPU fallback). `params.workers` = CTAs on the problem (0 = one per SM).
// Safe to call concurrently from several threads (like the reference).
PlanResult plan(const RobotModel& model, const Scene& scene, ConfigView start, ConfigView goal,
                const PlannerParams& params);

// Many independent problems for one robot in one device launch (one scene
// per problem); results in input order.
std::vector<PlanResult> plan_batch(const RobotModel& model, const std::vector<const Scene*>& scenes,
                                   const std::vector<Config>& starts, const std::vector<Config>& goals,
                                   const PlannerParams& params);

// The same problems spread over several devices (prrtc_plan_batch_multi: one
// host thread per device, a shared chunk queue; chunk 0 = automatic).
std::vector<PlanResult> plan_batch(const RobotModel& model, const std::vector<const Scene*>& scenes,
                                   const std::vector<Config>& starts, const std::vector<Config>& goals,
                                   const PlannerParams& params, const std::vector<int>& devices,
                                   uint32_t chunk = 0);

// CUDA device the drop-in plans on: the process default (initially 0) ...
void set_device(int device);
// ... unless the calling thread chose its own (-1 = back to the default):
// one host thread per GPU, each planning concurrently on its device.
void set_thread_device(int device);

// Drops the cached device copies of robots and scenes.
void clear_cache();

}  // namespace prrtc::b200
