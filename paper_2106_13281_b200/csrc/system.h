// system.h — the immutable system object behind brax_system.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "config.h"
#include "device_tables.h"

namespace brax {

struct LaunchConfig {
  int plan = 0;     // index into DHeader::plan
  int regs = 0;     // register budget variant
  bool tuned = false;
  bool fixed = false;  // fixed-shape body gathers (kFixed instantiation, V = 2 plans)
  bool lean = false;   // the lean kernel (step_lean.cu; V = 2, G = 2 / 4, ≤ 1 item and body step per warp)
};

struct System {
  Config cfg;
  int device = 0;
  DHeader hd{};
  std::vector<uint32_t> blob;          // host copy of the table blob
  uint32_t* d_blob = nullptr;          // device copy
  std::vector<float> dqp_pos, dqp_rot, dqp_vel, dqp_ang;  // default_qp, fp32, B rows
  float* d_default_qp = nullptr;       // device: pos[B][3] rot[B][4] (vel/ang are zero)
  std::vector<float> d_masks_host;     // per body mpos[3] mrot[3] + static flag (reset kernel)
  float* d_masks = nullptr;
  std::vector<std::string> lint;
  int n_dynamic = 0;
  int num_sms = 0;                     // of `device` (launch heuristics)
  bool trace = false;                  // per-phase cycle tracing (brax_system_set_tracing)
  unsigned long long* d_phase_cycles = nullptr;  // device [4]
  uint32_t* d_gran = nullptr;          // device [2][kMaxGranules]: launches started / finished per env granule
  size_t smem_bytes = 0;
  // the lean kernel's reach per plan: the most item steps any warp has (1 or 2; 0 = more,
  // or a warp with more than one body step)
  int lean_items[kNumPlans] = {};
  // launch configuration per batch size, measured by brax_system_tune
  // (every plan gives the same bits, so the choice only affects speed)
  bool autotune = true;
  mutable std::mutex tune_mu;
  mutable std::map<int64_t, LaunchConfig> tuned;
  ~System();
};

// Host-side construction: tables, plan, default_qp, lint (no GPU needed).
System* build_host(const Config& cfg);
// build_host + upload to `device`.
System* build_system(const Config& cfg, int device);

// default_qp in double precision (host), B rows.
void default_qp(const Config& cfg, std::vector<double>& pos, std::vector<double>& rot);


// Lane-group plan index chosen by the size heuristic for n_envs envs (step.cu).
int choose_plan(const System& sys, int64_t n_envs);
// The configuration the next launch of n_envs envs uses (tuned, overridden or heuristic).
LaunchConfig launch_config(const System& sys, int64_t n_envs);

// Kernel launchers (step.cu, reset.cu).  Return cudaSuccess or the launch error.
cudaError_t launch_step(const System& sys, const StepArgs& a, cudaStream_t stream);
// The lean kernel (step_lean.cu): whether it can run launch `a` with plan `plan`, and its launcher.
bool lean_applies(const System& sys, int plan, const StepArgs& a);
cudaError_t launch_lean(const System& sys, const StepArgs& a, int plan, int regs, cudaStream_t stream);
// brax_system_tune: time every launch plan on a's input (scratch outputs), remember the fastest.
cudaError_t tune_system(const System& sys, const StepArgs& a, cudaStream_t stream);
// Forward-mode derivative (JVP) of the step: StepArgs' d*_in tangents -> d*_out (NEXT-4).
cudaError_t launch_step_jvp(const System& sys, const StepArgs& a, cudaStream_t stream);
// Reverse-mode cotangent of one step in one launch (vjp.cu): g_in = Jᵀ·g_out.
cudaError_t launch_step_vjp_fused(const System& sys, const StepArgs& primal, const float* const g_out[4],
                                  float* const g_in[4], float* g_action, cudaStream_t stream);
// The same from the JVP columns (diff.cu), 13B + A JVP launches: the cross-check.
cudaError_t launch_step_vjp(const System& sys, const StepArgs& primal, const float* const g_out[4],
                            float* const g_in[4], float* g_action, cudaStream_t stream);
// Launch-order bookkeeping for the lean kernel's overlapped launches (step_lean.cu):
// every kernel launch on `stream` that is not a lean step launch records itself here,
// so the next lean launch waits for it in full (griddepcontrol.wait).
void note_other_launch(const System& sys, cudaStream_t stream);
// Held across a launch that calls note_other_launch, so the record order is the stream order.
std::unique_lock<std::recursive_mutex> launch_order_lock();
// Launch overlap (step_lean.cu): under launch_order_lock(), whether a step
// launch registers on the env-granule counters (participant, batch within their range)
// and whether it may skip the grid-wide dependent-launch wait; then record the launch.
struct OverlapDecision {
  bool reg = false;
  bool overlap = false;
};
OverlapDecision overlap_decide(const System& sys, const StepArgs& a, cudaStream_t stream, bool participant);
void overlap_commit(const System& sys, const StepArgs& a, cudaStream_t stream, const OverlapDecision& d,
                    cudaError_t launched);
// Drops the records of a system being destroyed.
void forget_system(const System* sys);
cudaError_t launch_reset(const System& sys, float* pos, float* rot, float* vel, float* ang, int64_t n,
                         uint64_t seed, float vel_noise, float ang_noise, cudaStream_t stream,
                         int64_t env_offset = 0, bool goal = false);  // goal: brax_env_reset's marker placement (R36)

}  // namespace brax

struct brax_system {
  brax::System* impl;
};
