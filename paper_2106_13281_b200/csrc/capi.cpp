// capi.cpp — the C ABI declared in include/brax_b200.h.  Argument validation,
// error translation (C++ exceptions → brax_status + thread-local detail), and
// dispatch to the kernel launchers.  No compute happens here.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "brax_b200.h"
#include "config.h"
#include "system.h"

namespace {
thread_local std::string g_detail;

brax_status fail(brax_status s, const std::string& detail) {
  g_detail = detail;
  return s;
}

template <class F>
brax_status guarded(F&& f) {
  try {
    return f();
  } catch (const brax::Error& e) {
    return fail(e.status, e.what());
  } catch (const std::bad_alloc&) {
    return fail(BRAX_E_OUT_OF_MEMORY, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(BRAX_E_INVALID_ARGUMENT, e.what());
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

brax_status check_qp(const brax_qp& q, const char* which) {
  if (!q.pos || !q.rot || !q.vel || !q.ang) return fail(BRAX_E_INVALID_ARGUMENT, std::string(which) + ": NULL pointer");
  if (!aligned16(q.pos) || !aligned16(q.rot) || !aligned16(q.vel) || !aligned16(q.ang))
    return fail(BRAX_E_MISALIGNED, std::string(which) + ": pointers must be 16-byte aligned");
  return BRAX_OK;
}

// Makes `device` current for the lifetime of the guard and restores the caller's
// current device afterwards (header convention "Device").
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != device) err = cudaSetDevice(device);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

brax_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return BRAX_OK;
  return fail(e == cudaErrorMemoryAllocation ? BRAX_E_OUT_OF_MEMORY : BRAX_E_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

brax_status step_common(const brax_system* sys, brax_qp in, const float* actions, int64_t n_steps, brax_qp out,
                        int64_t n_envs, const brax_step_extras* x, void* stream, const brax_env_io* io = nullptr,
                        float* observe_only = nullptr, const brax_random_actions* ra = nullptr) {
  if (!sys || !sys->impl) return fail(BRAX_E_INVALID_ARGUMENT, "sys is NULL");
  if (n_envs < 0 || n_steps < 0) return fail(BRAX_E_INVALID_ARGUMENT, "n_envs and n_steps must be >= 0");
  const bool env = io != nullptr || observe_only != nullptr;
  if (env && !sys->impl->cfg.task.present) return fail(BRAX_E_INVALID_ARGUMENT, "system has no task block");
  if (io && (!io->steps || !io->episode)) return fail(BRAX_E_INVALID_ARGUMENT, "env io: steps and episode are required");
  if (n_envs == 0 || (n_steps == 0 && !observe_only)) return BRAX_OK;
  if (n_envs > (int64_t(1) << 40)) return fail(BRAX_E_INVALID_ARGUMENT, "n_envs too large");
  brax_status st = check_qp(in, "in");
  if (st != BRAX_OK) return st;
  if ((st = check_qp(out, "out")) != BRAX_OK) return st;
  const brax::System& s = *sys->impl;
  if (s.hd.A > 0 && !actions && !observe_only && !ra)
    return fail(BRAX_E_INVALID_ARGUMENT, "action is NULL but act_dim > 0");
  if (ra && actions) return fail(BRAX_E_INVALID_ARGUMENT, "give either actions or random actions");
  if (actions && !aligned16(actions)) return fail(BRAX_E_MISALIGNED, "action must be 16-byte aligned");
  // aliasing: identical (in == out for all four arrays) is fine, any other overlap is not
  const float* ins[4] = {in.pos, in.rot, in.vel, in.ang};
  const float* outs[4] = {out.pos, out.rot, out.vel, out.ang};
  bool same = true;
  for (int i = 0; i < 4; ++i) same = same && ins[i] == outs[i];
  if (!same) {
    const int64_t B = s.hd.B;
    const int64_t bytes[4] = {n_envs * B * 12, n_envs * B * 16, n_envs * B * 12, n_envs * B * 12};
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        uintptr_t a0 = uintptr_t(ins[i]), a1 = a0 + uintptr_t(bytes[i]);
        uintptr_t b0 = uintptr_t(outs[j]), b1 = b0 + uintptr_t(bytes[j]);
        if (a0 < b1 && b0 < a1) return fail(BRAX_E_INVALID_ARGUMENT, "in and out overlap partially");
      }
    for (int i = 0; i < 4; ++i)
      for (int j = i + 1; j < 4; ++j) {
        uintptr_t a0 = uintptr_t(outs[i]), a1 = a0 + uintptr_t(bytes[i]);
        uintptr_t b0 = uintptr_t(outs[j]), b1 = b0 + uintptr_t(bytes[j]);
        if (a0 < b1 && b0 < a1) return fail(BRAX_E_INVALID_ARGUMENT, "out arrays overlap");
      }
  }
  if (x && x->contact_dp && !aligned16(x->contact_dp)) return fail(BRAX_E_MISALIGNED, "contact_dp must be 16-byte aligned");
  if (x && x->contact_dp && env) return fail(BRAX_E_INVALID_ARGUMENT, "contact_dp is not an env-step output");
  brax::StepArgs a{in.pos, in.rot, in.vel, in.ang, out.pos, out.rot, out.vel, out.ang, actions,
                   x ? x->status : nullptr, x ? x->contact_active : nullptr, n_envs, n_steps, 0, 0, nullptr};
  if (a.contact_active && s.hd.C == 0) a.contact_active = nullptr;
  a.contact_dp = x ? x->contact_dp : nullptr;
  if (ra && s.hd.A > 0) {
    a.act_random = 1;
    a.act_seed = ra->seed;
    a.act_env_offset = ra->env_offset;
    a.act_step0 = ra->step0;
  }
  if (env) {
    a.env = 1;
    a.dqp = s.d_default_qp;
    a.masks = s.d_masks;
    if (observe_only) {
      a.n_steps = 0;
      a.actions = nullptr;
      a.obs = observe_only;
    } else {
      a.obs = io->obs;
      a.reward = io->reward;
      a.done = io->done;
      a.steps = io->steps;
      a.episode = io->episode;
      a.seed = io->seed;
      a.env_offset = io->env_offset;
    }
  }
  DeviceGuard dg(s.device);
  if (dg.err != cudaSuccess) return cuda_status(dg.err, "cudaSetDevice");
  return cuda_status(brax::launch_step(s, a, static_cast<cudaStream_t>(stream)), "brax_step launch");
}
}  // namespace

extern "C" {

const char* brax_status_string(brax_status s) {
  switch (s) {
    case BRAX_OK: return "BRAX_OK";
    case BRAX_E_INVALID_ARGUMENT: return "BRAX_E_INVALID_ARGUMENT";
    case BRAX_E_PARSE: return "BRAX_E_PARSE";
    case BRAX_E_VALIDATION: return "BRAX_E_VALIDATION";
    case BRAX_E_CYCLIC_JOINT_GRAPH: return "BRAX_E_CYCLIC_JOINT_GRAPH";
    case BRAX_E_UNSUPPORTED_PAIR: return "BRAX_E_UNSUPPORTED_PAIR";
    case BRAX_E_MISALIGNED: return "BRAX_E_MISALIGNED";
    case BRAX_E_CUDA: return "BRAX_E_CUDA";
    case BRAX_E_OUT_OF_MEMORY: return "BRAX_E_OUT_OF_MEMORY";
  }
  return "unknown brax_status";
}

const char* brax_last_error_detail(void) { return g_detail.c_str(); }
int brax_abi_version(void) { return BRAX_ABI_VERSION; }

brax_status brax_config_parse(const char* text, size_t len, brax_config** out) {
  if (!text || !out) return fail(BRAX_E_INVALID_ARGUMENT, "text and out must be non-NULL");
  return guarded([&] {
    brax_config* c = new brax_config{brax::parse_config(std::string(text, len))};
    *out = c;
    return BRAX_OK;
  });
}

void brax_config_destroy(brax_config* cfg) { delete cfg; }

brax_status brax_config_from_desc(const brax_config_desc* desc, brax_config** out) {
  if (!desc || !out) return fail(BRAX_E_INVALID_ARGUMENT, "desc and out must be non-NULL");
  return guarded([&] {
    brax_config* c = new brax_config{brax::config_from_desc(*desc)};
    *out = c;
    return BRAX_OK;
  });
}

brax_status brax_config_slot_table(const brax_config* cfg, int32_t* out) {
  if (!cfg || !out) return fail(BRAX_E_INVALID_ARGUMENT, "cfg and out must be non-NULL");
  const auto& sl = cfg->cfg.slots;
  for (size_t i = 0; i < sl.size(); ++i) {
    int32_t row[7] = {sl[i].pair, sl[i].type, sl[i].a, sl[i].b, sl[i].col_a, sl[i].col_b, sl[i].point};
    std::memcpy(out + 7 * i, row, sizeof row);
  }
  return BRAX_OK;
}

brax_status brax_config_counts(const brax_config* cfg, int32_t* n_bodies, int32_t* n_joints, int32_t* act_dim,
                               int32_t* n_slots) {
  if (!cfg) return fail(BRAX_E_INVALID_ARGUMENT, "cfg is NULL");
  if (n_bodies) *n_bodies = int32_t(cfg->cfg.bodies.size());
  if (n_joints) *n_joints = int32_t(cfg->cfg.joints.size());
  if (act_dim) *act_dim = cfg->cfg.act_dim;
  if (n_slots) *n_slots = int32_t(cfg->cfg.slots.size());
  return BRAX_OK;
}

brax_status brax_config_default_qp(const brax_config* cfg, double* pos, double* rot) {
  if (!cfg || !pos || !rot) return fail(BRAX_E_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    std::vector<double> p, r;
    brax::default_qp(cfg->cfg, p, r);
    std::memcpy(pos, p.data(), p.size() * sizeof(double));
    std::memcpy(rot, r.data(), r.size() * sizeof(double));
    return BRAX_OK;
  });
}

brax_status brax_system_create(const brax_config* cfg, int cuda_device, brax_system** out) {
  if (!cfg || !out) return fail(BRAX_E_INVALID_ARGUMENT, "cfg and out must be non-NULL");
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
      throw brax::Error(BRAX_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (cuda_device < 0 || cuda_device >= n) throw brax::Error(BRAX_E_INVALID_ARGUMENT, "cuda_device out of range");
    brax_system* s = new brax_system{brax::build_system(cfg->cfg, cuda_device)};
    *out = s;
    return BRAX_OK;
  });
}

void brax_system_destroy(brax_system* sys) {
  if (!sys) return;
  delete sys->impl;
  delete sys;
}

brax_status brax_system_get_info(const brax_system* sys, brax_system_info* out) {
  if (!sys || !out) return fail(BRAX_E_INVALID_ARGUMENT, "NULL argument");
  const brax::System& s = *sys->impl;
  out->n_bodies = s.hd.B;
  out->n_dynamic = s.n_dynamic;
  out->n_joints = s.hd.J;
  out->act_dim = s.hd.A;
  out->n_contact_slots = s.hd.C;
  out->substeps = s.hd.S;
  out->dt = float(s.cfg.dt);
  out->warps_per_block = s.hd.plan[0].W;
  out->n_lint_warnings = int32_t(s.lint.size());
  out->smem_bytes = int32_t(s.smem_bytes);
  return BRAX_OK;
}

brax_status brax_system_slot_table(const brax_system* sys, int32_t* out) {
  if (!sys) return fail(BRAX_E_INVALID_ARGUMENT, "sys is NULL");
  brax_config tmp{sys->impl->cfg};
  return brax_config_slot_table(&tmp, out);
}

brax_status brax_system_set_tracing(brax_system* sys, int enable) {
  if (!sys) return fail(BRAX_E_INVALID_ARGUMENT, "sys is NULL");
  sys->impl->trace = enable != 0;
  return BRAX_OK;
}

brax_status brax_system_phase_cycles(brax_system* sys, uint64_t out[4]) {
  if (!sys || !out) return fail(BRAX_E_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard dg(sys->impl->device);
  unsigned long long h[4];
  cudaError_t e = cudaMemcpy(h, sys->impl->d_phase_cycles, sizeof h, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(sys->impl->d_phase_cycles, 0, sizeof h);
  if (e != cudaSuccess) return cuda_status(e, "brax_system_phase_cycles");
  for (int k = 0; k < 4; ++k) out[k] = h[k];
  return BRAX_OK;
}

brax_status brax_system_set_autotune(brax_system* sys, int enable) {
  if (!sys) return fail(BRAX_E_INVALID_ARGUMENT, "sys is NULL");
  sys->impl->autotune = enable != 0;
  return BRAX_OK;
}

brax_status brax_system_tune(brax_system* sys, brax_qp in, const float* action, int64_t n_envs, void* stream) {
  if (!sys || !sys->impl) return fail(BRAX_E_INVALID_ARGUMENT, "sys is NULL");
  if (n_envs < 0) return fail(BRAX_E_INVALID_ARGUMENT, "n_envs must be >= 0");
  if (n_envs == 0 || !sys->impl->autotune) return BRAX_OK;
  brax_status st = check_qp(in, "in");
  if (st != BRAX_OK) return st;
  const brax::System& s = *sys->impl;
  if (s.hd.A > 0 && !action) return fail(BRAX_E_INVALID_ARGUMENT, "action is NULL but act_dim > 0");
  if (action && !aligned16(action)) return fail(BRAX_E_MISALIGNED, "action must be 16-byte aligned");
  DeviceGuard dg(s.device);
  if (dg.err != cudaSuccess) return cuda_status(dg.err, "cudaSetDevice");
  brax::StepArgs a{in.pos, in.rot, in.vel, in.ang, nullptr, nullptr, nullptr, nullptr, action,
                   nullptr, nullptr, n_envs, 1, 0, 0, nullptr};
  return cuda_status(brax::tune_system(s, a, static_cast<cudaStream_t>(stream)), "brax_system_tune");
}

brax_status brax_system_launch_config(const brax_system* sys, int64_t n_envs, int32_t out[6]) {
  if (!sys || !out) return fail(BRAX_E_INVALID_ARGUMENT, "NULL argument");
  if (n_envs < 0) return fail(BRAX_E_INVALID_ARGUMENT, "n_envs < 0");
  const brax::System& s = *sys->impl;
  const brax::LaunchConfig c = brax::launch_config(s, n_envs);
  const brax::DPlan& P = s.hd.plan[c.plan];
  out[0] = P.G;
  out[1] = P.V;
  out[2] = P.E;
  out[3] = P.W;
  out[4] = c.regs;
  out[5] = (c.tuned ? 1 : 0) | (c.fixed && P.V == 2 ? 2 : 0) | (c.lean ? 4 : 0);
  return BRAX_OK;
}

const char* brax_system_lint_warning(const brax_system* sys, int32_t i) {
  if (!sys || i < 0 || size_t(i) >= sys->impl->lint.size()) return nullptr;
  return sys->impl->lint[i].c_str();
}

brax_status brax_default_qp(const brax_system* sys, float* h_pos, float* h_rot, float* h_vel, float* h_ang) {
  if (!sys || !h_pos || !h_rot || !h_vel || !h_ang) return fail(BRAX_E_INVALID_ARGUMENT, "NULL argument");
  const brax::System& s = *sys->impl;
  std::memcpy(h_pos, s.dqp_pos.data(), s.dqp_pos.size() * 4);
  std::memcpy(h_rot, s.dqp_rot.data(), s.dqp_rot.size() * 4);
  std::memcpy(h_vel, s.dqp_vel.data(), s.dqp_vel.size() * 4);
  std::memcpy(h_ang, s.dqp_ang.data(), s.dqp_ang.size() * 4);
  return BRAX_OK;
}

brax_status brax_reset(const brax_system* sys, brax_qp out, int64_t n_envs, uint64_t seed, float vel_noise,
                       float ang_noise, void* stream) {
  if (!sys) return fail(BRAX_E_INVALID_ARGUMENT, "sys is NULL");
  if (n_envs < 0) return fail(BRAX_E_INVALID_ARGUMENT, "n_envs must be >= 0");
  if (n_envs == 0) return BRAX_OK;
  brax_status st = check_qp(out, "out");
  if (st != BRAX_OK) return st;
  DeviceGuard dg(sys->impl->device);
  return cuda_status(brax::launch_reset(*sys->impl, out.pos, out.rot, out.vel, out.ang, n_envs, seed, vel_noise,
                                        ang_noise, static_cast<cudaStream_t>(stream)),
                     "brax_reset launch");
}

brax_status brax_step(const brax_system* sys, brax_qp in, const float* action, brax_qp out, int64_t n_envs,
                      void* stream) {
  return step_common(sys, in, action, 1, out, n_envs, nullptr, stream);
}

brax_status brax_step_ex(const brax_system* sys, brax_qp in, const float* action, brax_qp out, int64_t n_envs,
                         const brax_step_extras* extras, void* stream) {
  return step_common(sys, in, action, 1, out, n_envs, extras, stream);
}

brax_status brax_rollout(const brax_system* sys, brax_qp in, const float* actions, int64_t n_steps, brax_qp out,
                         int64_t n_envs, const brax_step_extras* extras, void* stream) {
  return step_common(sys, in, actions, n_steps, out, n_envs, extras, stream);
}

brax_status brax_rollout_random(const brax_system* sys, brax_qp in, int64_t n_steps, brax_qp out, int64_t n_envs,
                                const brax_random_actions* ra, const brax_step_extras* extras, void* stream) {
  if (!ra) return fail(BRAX_E_INVALID_ARGUMENT, "ra is NULL");
  return step_common(sys, in, nullptr, n_steps, out, n_envs, extras, stream, nullptr, nullptr, ra);
}

brax_status brax_env_step_random(const brax_system* sys, brax_qp in, int64_t n_steps, brax_qp out, int64_t n_envs,
                                 const brax_random_actions* ra, const brax_env_io* io, void* stream) {
  if (!ra || !io) return fail(BRAX_E_INVALID_ARGUMENT, "NULL argument");
  return step_common(sys, in, nullptr, n_steps, out, n_envs, nullptr, stream, io, nullptr, ra);
}

brax_status brax_step_jvp(const brax_system* sys, brax_qp in, const float* action, brax_qp din,
                          const float* daction, brax_qp out, brax_qp dout, int64_t n_envs, void* stream) {
  if (!sys || !sys->impl) return fail(BRAX_E_INVALID_ARGUMENT, "sys is NULL");
  if (n_envs < 0) return fail(BRAX_E_INVALID_ARGUMENT, "n_envs must be >= 0");
  if (n_envs == 0) return BRAX_OK;
  brax_status st = check_qp(in, "in");
  if (st != BRAX_OK) return st;
  if ((st = check_qp(out, "out")) != BRAX_OK) return st;
  if ((st = check_qp(dout, "dout")) != BRAX_OK) return st;
  const brax::System& s = *sys->impl;
  if (s.hd.A > 0 && !action) return fail(BRAX_E_INVALID_ARGUMENT, "action is NULL but act_dim > 0");
  brax::StepArgs a{in.pos, in.rot, in.vel, in.ang, out.pos, out.rot, out.vel, out.ang, action,
                   nullptr, nullptr, n_envs, 1, 0, 0, nullptr};
  a.dpos_in = din.pos;
  a.drot_in = din.rot;
  a.dvel_in = din.vel;
  a.dang_in = din.ang;
  a.dactions = daction;
  a.dpos_out = dout.pos;
  a.drot_out = dout.rot;
  a.dvel_out = dout.vel;
  a.dang_out = dout.ang;
  DeviceGuard dg(s.device);
  cudaError_t e = brax::launch_step_jvp(s, a, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorInvalidValue) return fail(BRAX_E_VALIDATION, "brax_step_jvp: system too large for the JVP kernel");
  return cuda_status(e, "brax_step_jvp launch");
}

brax_status brax_step_vjp(const brax_system* sys, brax_qp in, const float* action, brax_qp g_out, brax_qp g_in,
                          float* g_action, int64_t n_envs, void* stream) {
  if (!sys || !sys->impl) return fail(BRAX_E_INVALID_ARGUMENT, "sys is NULL");
  if (n_envs < 0) return fail(BRAX_E_INVALID_ARGUMENT, "n_envs must be >= 0");
  if (n_envs == 0) return BRAX_OK;
  brax_status st = check_qp(in, "in");
  if (st != BRAX_OK) return st;
  if ((st = check_qp(g_in, "g_in")) != BRAX_OK) return st;
  const brax::System& s = *sys->impl;
  if (s.hd.A > 0 && !action) return fail(BRAX_E_INVALID_ARGUMENT, "action is NULL but act_dim > 0");
  brax::StepArgs a{in.pos, in.rot, in.vel, in.ang, nullptr, nullptr, nullptr, nullptr, action,
                   nullptr, nullptr, n_envs, 1, 0, 0, nullptr};
  const float* go[4] = {g_out.pos, g_out.rot, g_out.vel, g_out.ang};
  float* gi[4] = {g_in.pos, g_in.rot, g_in.vel, g_in.ang};
  DeviceGuard dg(s.device);
  cudaError_t e = std::getenv("BRAX_VJP_COLUMNS")
                      ? brax::launch_step_vjp(s, a, go, gi, g_action, static_cast<cudaStream_t>(stream))
                      : brax::launch_step_vjp_fused(s, a, go, gi, g_action, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorInvalidValue) return fail(BRAX_E_VALIDATION, "brax_step_vjp: system too large for the JVP kernel");
  return cuda_status(e, "brax_step_vjp");
}

brax_status brax_system_task_info(const brax_system* sys, int32_t out[4]) {
  if (!sys || !out) return fail(BRAX_E_INVALID_ARGUMENT, "NULL argument");
  const brax::Config& c = sys->impl->cfg;
  out[0] = c.task.present ? 1 : 0;
  out[1] = c.obs_dim();
  out[2] = c.task.present ? c.task.episode_length : 0;
  out[3] = c.task.present ? c.task.torso : -1;
  return BRAX_OK;
}

brax_status brax_env_step(const brax_system* sys, brax_qp in, const float* actions, int64_t n_steps, brax_qp out,
                          int64_t n_envs, const brax_env_io* io, void* stream) {
  if (!io) return fail(BRAX_E_INVALID_ARGUMENT, "io is NULL");
  return step_common(sys, in, actions, n_steps, out, n_envs, nullptr, stream, io);
}

brax_status brax_env_observe(const brax_system* sys, brax_qp qp, int64_t n_envs, float* obs, void* stream) {
  if (!obs) return fail(BRAX_E_INVALID_ARGUMENT, "obs is NULL");
  return step_common(sys, qp, nullptr, 0, qp, n_envs, nullptr, stream, nullptr, obs);
}

brax_status brax_env_reset(const brax_system* sys, brax_qp out, int64_t n_envs, const brax_env_io* io,
                           void* stream) {
  if (!sys || !io) return fail(BRAX_E_INVALID_ARGUMENT, "NULL argument");
  const brax::System& s = *sys->impl;
  if (!s.cfg.task.present) return fail(BRAX_E_INVALID_ARGUMENT, "system has no task block");
  if (!io->steps || !io->episode) return fail(BRAX_E_INVALID_ARGUMENT, "env io: steps and episode are required");
  if (n_envs < 0) return fail(BRAX_E_INVALID_ARGUMENT, "n_envs must be >= 0");
  if (n_envs == 0) return BRAX_OK;
  brax_status st = check_qp(out, "out");
  if (st != BRAX_OK) return st;
  DeviceGuard dg(s.device);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  cudaError_t e = brax::launch_reset(s, out.pos, out.rot, out.vel, out.ang, n_envs, io->seed,
                                     float(s.cfg.task.noise_vel), float(s.cfg.task.noise_ang), cs, io->env_offset,
                                     true);
  if (e == cudaSuccess) e = cudaMemsetAsync(io->steps, 0, size_t(n_envs) * 4, cs);
  if (e == cudaSuccess) e = cudaMemsetAsync(io->episode, 0, size_t(n_envs) * 4, cs);
  if (e != cudaSuccess) return cuda_status(e, "brax_env_reset");
  if (!io->obs) return BRAX_OK;
  return step_common(sys, out, nullptr, 0, out, n_envs, nullptr, stream, nullptr, io->obs);
}

}  // extern "C"
