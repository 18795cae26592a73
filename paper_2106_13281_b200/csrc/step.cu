// step.cu — the generic (table-driven) batched Brax step kernel for sm_100a,
// and its launcher.
//
// Computes Alg. 1 of the paper `substeps` times per step for
// n independent envs (device code in step_device.cuh).  Mapping:
//   * one block = E envs; a warp's 32 lanes form G = 32/E groups; group g of
//     warp w runs one work item (a body, a joint, a contact slot) on the E envs,
//     lane = env.  The items sharing a warp have the same code class, so
//     control flow is group-uniform; the only divergence is whether a contact
//     is active in a given env.  G > 1 gives more, smaller blocks for small
//     batches (choose_plan).
//   * each env's QP is read from HBM once (coalesced, float4), kept in shared
//     memory as [body][field][lane] for all substeps (and all steps of
//     brax_rollout), and written back once.
//   * per-body sums are gathers over static incidence lists in a fixed order
//     (joints by index, then contact slots by index): no atomics.
//   * per substep: phase 1 joints+actuators and contacts (item warps) | barrier |
//     phase 2 gather + potential + collision integrators, fused with the next
//     substep's kinematic integrator (body warps) | barrier.
// The static tables are staged into shared memory and read with broadcast
// LDS.128; the code is shared by all warps, which keeps the instruction
// footprint small (a per-system specialised variant with the
// tables as immediates ran 2x slower: ~160 KB of per-warp code thrashes the
// instruction caches — DESIGN.md §5).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <vector>
#include <cstdlib>

#include "device_rng.cuh"
#include "step_device.cuh"
#include "system.h"

namespace brax {
namespace {

using namespace dev;

__device__ __forceinline__ float diag_val(F1 v) { return v.x; }
__device__ __forceinline__ float diag_val(F2 v) { return v.x; }
__device__ __forceinline__ float diag_val(D1 v) { return v.v; }

struct KArgs {
  StepArgs a;
  const uint32_t* blob;
  DHeader hd;
  int32_t plan;  // index into hd.plan (G = 1 << plan lane groups per warp)
  // launch overlap (as in step_lean.cu): env-granule counters
  uint32_t* gs;
  uint32_t* gd;
  int32_t reg;
  int32_t overlap;
};

// Register budget: 80 per thread keeps 2 blocks of up to 12 warps resident per SM.
// S = float: one env per lane; F2: two envs per lane.  R: register budget per
// thread (instantiated for several budgets; launch_step picks the largest that
// keeps two blocks resident per SM).
// kFixed: body gathers with compile-time list lengths for the common incidence shapes
// (a separate instantiation the autotuner may pick: the extra code costs instruction-
// cache space that some systems do not win back; same bits either way).
template <class S, int R, bool kEnv, bool kFixed = false>
__global__ void __maxnreg__(R) brax_step_kernel(const __grid_constant__ KArgs ka) {
  extern __shared__ __align__(16) uint32_t smem[];
  const DHeader& H = ka.hd;
  const DPlan& P = H.plan[ka.plan];
  const StepArgs& a = ka.a;
  // V: layout id of the lane type (1: F1, 2: F2 env pairs, 3: D1 value/tangent pairs);
  // SL: words per lane slot in per-env arrays; RW = LG·SL: their row width
  constexpr int V = Lanes<S>::V, SL = Lanes<S>::SL, QS = Lanes<S>::QS, JS = Lanes<S>::JS, CS = Lanes<S>::CS;
  const int B = H.B, J = H.J, C = H.C, A = H.A, E = P.E, G = P.G;
  const DTask& T = H.task;
  const int LG = 32 / G;  // lanes per group = records per item
  const int RW = LG * SL;
  const bool cdp = !kEnv && a.contact_dp != nullptr;  // brax_step_extras.contact_dp (physics kernel)
  const SmemLayout L =
      smem_layout(B, J, C, A, E, LG, SL == 2, H.blob_words, kEnv ? T.obs_dim : 0, kEnv ? T.contact_obs : 0, cdp);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // [0] tables + QP, [1] actions
  uint32_t* sBlob = smem + L.blob;
  float* sQ = reinterpret_cast<float*>(smem + L.q);
  float* sJ = reinterpret_cast<float*>(smem + L.u);
  float* sC = sJ + J * LG * JS;
  float* stg = reinterpret_cast<float*>(smem + L.u);  // aliases sJ/sC outside the substeps
  float* sA = reinterpret_cast<float*>(smem + L.a);
  float* sAstg = reinterpret_cast<float*>(smem + L.astg);
  float* sCnt = reinterpret_cast<float*>(smem + L.cnt);
  uint32_t* sStat = smem + L.stat;
  // env epilogue (NEXT-1): torso position at the step start, steps / episode / reset flag
  // per env, contact Δv [B][6][E] of the last substep, observation rows (alias U)
  float* sX0 = reinterpret_cast<float*>(smem + L.x0);
  int32_t* sSteps = reinterpret_cast<int32_t*>(smem + L.steps);
  uint32_t* sEp = smem + L.ep;
  int32_t* sRst = reinterpret_cast<int32_t*>(smem + L.rst);
  float* sCo = reinterpret_cast<float*>(smem + L.co);
  float* sObs = reinterpret_cast<float*>(smem + L.u);
  constexpr bool envm = kEnv;  // env epilogue compiled in (a.env != 0) or out
  const bool save_co = envm && T.contact_obs;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tracing (brax_system_phase_cycles): thread 0 times prologue / joints+contacts /
  // integrate / epilogue with clock64 (uniform branch; off unless requested)
  // (the sums live in shared memory, not in registers held across the whole kernel)
  // the specialised (kFixed) variants carry no tracing code: a traced launch uses the generic one
  constexpr bool kTraceable = !kFixed;
  const bool trace = kTraceable && a.phase_cycles != nullptr && tid == 0;
  __shared__ long long sTr[5];  // per-phase sums, last mark
#ifdef BRAX_DIAG
  __shared__ float sDiag[kMaxWarps];  // diagnostics (a.diag_block) only
#endif
  if (trace) {
    for (int k = 0; k < 4; ++k) sTr[k] = 0;
    sTr[4] = clock64();
  }
  auto lap = [&](int k) {  // re-tests the (uniform) argument instead of holding `trace` in a register
    if (kTraceable && a.phase_cycles != nullptr && threadIdx.x == 0) {
      const long long t = clock64();
      sTr[k] += t - sTr[4];
      sTr[4] = t;
    }
  };
  const int grp = lane / LG, el = lane - grp * LG;  // lane group; this lane's record slot (envs el, el + LG)
  const int64_t e0 = int64_t(blockIdx.x) * E;
  const int nvalid = (a.n_envs - e0 < E) ? int(a.n_envs - e0) : E;
  constexpr bool kJvp = V == 3;                        // D1: value + tangent staging, per-row copies
  const bool bulk = !kJvp && a.bulk_ok && nvalid == E;  // block-uniform
  const bool act_bulk = bulk && a.act_bulk_ok && A > 0;
  const uint32_t qp_bytes = uint32_t(E * B) * 13u * 4u, act_bytes = uint32_t(E * A) * 4u;

  // S1: tables and (full blocks) the four contiguous QP chunks arrive by TMA bulk copies
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {  // the tables are constant: load them before waiting for the previous grid
    mbar_expect_tx(&bars[0], uint32_t(H.blob_words) * 4u + (bulk ? qp_bytes : 0u));
    tma_load(sBlob, ka.blob, uint32_t(H.blob_words) * 4u, &bars[0]);
  }
  // programmatic dependent launch: everything above overlapped the previous kernel's
  // tail; the QP and actions may be its outputs, so wait for it to complete here — or,
  // for an overlapped launch, only for the earlier launches on this block's env granules
  if (!ka.overlap) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int g0 = int(e0 / kGranule), ng = (nvalid + kGranule - 1) / kGranule;
  uint32_t gprev = 0, gdone = 0;
  if (ka.reg && tid < ng) {
    // register, and read the finished count in the same round trip: completions counted
    // before our registration are all of earlier launches (a later one waits for us)
    gprev = atomicAdd(ka.gs + g0 + tid, 1u);
    gdone = ld_acquire_gpu(ka.gd + g0 + tid);
  }
  if (ka.reg) __syncthreads();  // every registration performed before the trigger
  asm volatile("griddepcontrol.launch_dependents;");
  if (ka.reg) {
    if (tid < ng)
      while (int32_t(gdone - gprev) < 0) {
        __nanosleep(64);
        gdone = ld_acquire_gpu(ka.gd + g0 + tid);
      }
    __syncthreads();
    if (tid == 0) fence_proxy_async_global();
  }
  if (tid == 0) {
    if (bulk) {
      float* sp = stg;
      float* sr = sp + E * B * 3;
      float* sv = sr + E * B * 4;
      float* sw = sv + E * B * 3;
      tma_load(sp, a.pos_in + e0 * B * 3, uint32_t(E * B) * 12u, &bars[0]);
      tma_load(sr, a.rot_in + e0 * B * 4, uint32_t(E * B) * 16u, &bars[0]);
      tma_load(sv, a.vel_in + e0 * B * 3, uint32_t(E * B) * 12u, &bars[0]);
      tma_load(sw, a.ang_in + e0 * B * 3, uint32_t(E * B) * 12u, &bars[0]);
    }
    if (act_bulk) {
      mbar_expect_tx(&bars[1], act_bytes);
      tma_load(sAstg, a.actions + e0 * A, act_bytes, &bars[1]);
    }
  }
  if (!bulk) {  // ragged tail / unaligned / JVP: per-row loads
    if constexpr (kJvp) load_block_d(a, sQ, B, E, e0, nvalid);
    else load_block<V>(a, sQ, B, E, e0, nvalid);
  }
  mbar_wait(&bars[0], 0);
  if (bulk) stg_to_records<V>(stg, sQ, B, E);
  for (int i = tid; i < E; i += blockDim.x) sStat[i] = 0u;
  if (envm) {
    for (int i = tid; i < E; i += blockDim.x) {
      sSteps[i] = i < nvalid && a.steps ? a.steps[e0 + i] : 0;
      sEp[i] = i < nvalid && a.episode ? a.episode[e0 + i] : 0u;
    }
    if (save_co)
      for (int i = tid; i < 6 * B * RW; i += blockDim.x) sCo[i] = 0.f;
  }
  if (cdp)  // static bodies keep 0; dynamic bodies store at substep 0 of every step
    for (int i = tid; i < 6 * B * RW; i += blockDim.x) sCo[i] = 0.f;
  __syncthreads();
  lap(0);

  const DBody* bodies = reinterpret_cast<const DBody*>(sBlob + H.off_bodies);
  const DJoint* joints = reinterpret_cast<const DJoint*>(sBlob + H.off_joints);
  const DSlot* slots = reinterpret_cast<const DSlot*>(sBlob + H.off_slots);
  const int32_t* item_begin = reinterpret_cast<const int32_t*>(sBlob + P.off_item_begin);
  const int32_t* items = reinterpret_cast<const int32_t*>(sBlob + P.off_items) + grp;
  const int32_t* body_begin = reinterpret_cast<const int32_t*>(sBlob + P.off_body_begin);
  const int32_t* bodies_of_warp = reinterpret_cast<const int32_t*>(sBlob + P.off_bodies_of_warp) + grp;
  const int32_t* jinc_begin = reinterpret_cast<const int32_t*>(sBlob + H.off_jinc_begin);
  const int32_t* jinc = reinterpret_cast<const int32_t*>(sBlob + H.off_jinc);
  const int32_t* cinc_begin = reinterpret_cast<const int32_t*>(sBlob + H.off_cinc_begin);
  const int32_t* cinc = reinterpret_cast<const int32_t*>(sBlob + H.off_cinc);
  const float* sJe = sJ + el * JS;  // this lane's record of joint 0 (joint j: + j·LG·JS)
  const float* sCe = sC + el * CS;
  const int it0 = item_begin[warp], it1 = item_begin[warp + 1];
  const int bw0 = body_begin[warp], bw1 = body_begin[warp + 1];

  const int od = T.obs_dim;
  // ---- NEXT-1 env epilogue pieces (R30-R35; per-env scalar code spells out its rounding) ----
  auto save_x0 = [&]() {  // torso position at the step boundary (before S2)
    for (int i = tid; i < E; i += blockDim.x)
      for (int k = 0; k < 3; ++k) sX0[3 * i + k] = sQ[qword<V>(T.obj, i, 0, k, LG)];
  };
  auto observe = [&](float* obs_out) {  // obs rows of the block's envs -> obs_out [nvalid][od]
    // joints: angles and rates, by the warps that own them
    for (int it = it0; it < it1; ++it) {
      int item = items[it * G];
      if (item < 0 || item >= J) continue;
      const DJoint& jt = joints[item];
      joint_obs<S>(jt, Row<S>{sQ + (jt.parent * LG + el) * QS}, Row<S>{sQ + (jt.child * LG + el) * QS},
                   sObs + el * od, LG * od, 5 + jt.obs_off, 11 + T.nq + jt.obs_off);
    }
    // torso and contact parts, one thread per (env, word)
    const int nco = T.contact_obs ? 6 * B : 0, ng = T.has_goal ? 9 : 0, nw = 11 + ng + nco;
    for (int i = tid; i < E * nw; i += blockDim.x) {
      const int env = i / nw, k = i - env * nw;
      float v;
      int at;
      if (k < 11) {
        const int f = k == 0 ? 0 : k < 5 ? 1 : k < 8 ? 2 : 3;
        const int c = k == 0 ? 2 : k < 5 ? k - 1 : k < 8 ? k - 5 : k - 8;
        v = sQ[qword<V>(T.torso, env, f, c, LG)];
        at = k < 5 ? k : 5 + T.nq + (k - 5);
      } else if (k < 11 + ng) {  // goal block (R36): x_T − x_O, x_O − x_torso, v_O
        const int g = (k - 11) / 3, c = (k - 11) - 3 * g;
        const float xo = sQ[qword<V>(T.obj, env, 0, c, LG)];
        v = g == 0 ? __fadd_rn(sQ[qword<V>(T.target, env, 0, c, LG)], -xo)
          : g == 1 ? __fadd_rn(xo, -sQ[qword<V>(T.torso, env, 0, c, LG)])
                   : sQ[qword<V>(T.obj, env, 2, c, LG)];
        at = 11 + 2 * T.nq + (k - 11);
      } else {
        const int b = (k - 11 - ng) / 6, kk = (k - 11 - ng) - 6 * b;
        v = fminf(fmaxf(sCo[(b * 6 + kk) * RW + eslot<V>(env, LG)], -1.f), 1.f);
        at = 11 + 2 * T.nq + (k - 11);
      }
      sObs[env * od + at] = v;
    }
    __syncthreads();
    for (int i = tid; i < nvalid * od; i += blockDim.x) obs_out[i] = sObs[i];
    __syncthreads();
  };

  if (envm && a.n_steps == 0) {  // observe only (brax_env_observe / brax_env_reset): QP not written
    observe(a.obs + e0 * od);
    if (ka.reg && tid == 0) {  // (the host does not register these launches; never leave a granule open)
      __threadfence();
      for (int k = 0; k < ng; ++k) atomicAdd(ka.gd + g0 + k, 1u);
    }
    return;
  }
  // S2 of the first substep; every later S2 is fused into the previous substep's integrate()
  if (envm) {
    save_x0();
    __syncthreads();
  }
  for (int i = bw0; i < bw1; ++i) {
    int b = bodies_of_warp[i * G];
    if (b >= 0) kinematic<S>(bodies[b], Row<S>{sQ + (b * LG + el) * QS}, H.h);
  }
  for (int64_t step = 0; step < a.n_steps; ++step) {
    if (envm && step > 0) {  // env mode ends every step at the boundary: its S2 runs here
      save_x0();
      __syncthreads();
      for (int i = bw0; i < bw1; ++i) {
        int b = bodies_of_warp[i * G];
        if (b >= 0) kinematic<S>(bodies[b], Row<S>{sQ + (b * LG + el) * QS}, H.h);
      }
    }
    if (act_bulk) {  // this step's actions arrived in sAstg [E][A]; transpose to sA [A][E]
      mbar_wait(&bars[1], uint32_t(step & 1));
      for (int i = tid; i < E * A; i += blockDim.x) {
        const int env = i / A, k = i - env * A;
        sA[k * RW + eslot<V>(env, LG)] = sAstg[i];
      }
    } else if (kJvp) {
      load_actions_d(a, sA, A, E, step, e0, nvalid);
    } else if (a.act_random) {  // NEXT-2: this step's actions from the counter-based generator
      const uint2 key = make_uint2(uint32_t(a.act_seed & 0xffffffffu), uint32_t(a.act_seed >> 32));
      const int A4 = (A + 3) >> 2;
      const uint32_t t = uint32_t(a.act_step0 + step);
      for (int i = tid; i < E * A4; i += blockDim.x) {
        const int env = i / A4, g = i - env * A4;
        const uint4 x = philox4x32_10(make_uint4(uint32_t(a.act_env_offset + e0 + env), t, uint32_t(g), kActTag), key);
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
        for (int j = 0; j < 4 && 4 * g + j < A; ++j) sA[(4 * g + j) * RW + eslot<V>(env, LG)] = u_pm1(xs[j]);
      }
    } else {
      load_actions<V>(a, sA, A, E, LG, step, e0, nvalid);
    }  // sA is read in phase 2, after a barrier
    for (int it = it0; it < it1; ++it) {
      int item = items[it * G];
      if (item >= J) {
        for (int k = 0; k < SL; ++k) sCnt[(item - J) * RW + el * SL + k] = 0.f;
      }
    }
    const bool pf_act = act_bulk && tid == 0 && step + 1 < a.n_steps;
    for (int s = 0; s < H.S; ++s) {
      __syncthreads();
      lap(2);
#ifdef BRAX_DIAG  // per-warp clock stamps of substep 3 of step 0 in one block (build with BRAX_NVCC_FLAGS=-DBRAX_DIAG)
      const bool dg = a.diag_block && step == 0 && s == 3 && int(blockIdx.x) == a.diag_block - 1 && lane == 0;
      long long dt0 = dg ? clock64() : 0, dt1 = 0, dt2 = 0, dtg = 0, dts = 0;
#endif
      if (s == 0 && pf_act) {  // prefetch next step's actions
        mbar_expect_tx(&bars[1], act_bytes);
        tma_load(sAstg, a.actions + ((step + 1) * a.n_envs + e0) * A, act_bytes, &bars[1]);
      }
      for (int it = it0; it < it1; ++it) {
        int item = items[it * G];
        if (item < 0) continue;
        if (item < J) {
          const DJoint& jt = joints[item];
          const Row<S> rp{sQ + (jt.parent * LG + el) * QS}, rc{sQ + (jt.child * LG + el) * QS};
          float* rec = sJ + (item * LG + el) * JS;
          if constexpr (kFixed) {  // specialised variant: torque-actuated joints with dof at compile time
            const int4 h0 = *reinterpret_cast<const int4*>(&jt);
            if (h0.w == 0 && h0.z == 1) joint<S, 1, 0>(jt, rp, rc, sA + el * SL, RW, rec);
            else if (h0.w == 0 && h0.z == 2) joint<S, 2, 0>(jt, rp, rc, sA + el * SL, RW, rec);
            else if (h0.w == 0 && h0.z == 3) joint<S, 3, 0>(jt, rp, rc, sA + el * SL, RW, rec);
            else joint<S>(jt, rp, rc, sA + el * SL, RW, rec);
          } else {
            joint<S>(jt, rp, rc, sA + el * SL, RW, rec);
          }
        } else {
          int c = item - J;
          const DSlot& sl = slots[c];
          float* cp = sCnt + c * RW + el * SL;
          S cnt = Lanes<S>::ld(cp);
          const Row<S> ra{sQ + (sl.a * LG + el) * QS}, rb{sQ + (sl.b * LG + el) * QS};
          float* rec = sC + (c * LG + el) * CS;
          if constexpr (kFixed) {  // specialised variant: capsule ends and spheres on the ground at compile time
            const int4 h0 = *reinterpret_cast<const int4*>(&sl), h1 = reinterpret_cast<const int4*>(&sl)[1];
            const bool ground = h1.x == 0 && h1.y == 1 && (h1.z & kCapsuleOnGroundFlags) == kCapsuleOnGroundFlags;
            if (ground && h0.x == 1)
              contact<S, 1>(sl, ra, rb, 1.f + H.e, H.beta_over_h, H.mu, rec, cnt);
            else if (ground && h0.x == 0)
              contact<S, 2>(sl, ra, rb, 1.f + H.e, H.beta_over_h, H.mu, rec, cnt);
            else if (ground && h0.x == 2)
              contact<S, 3>(sl, ra, rb, 1.f + H.e, H.beta_over_h, H.mu, rec, cnt);
            else
              contact<S>(sl, ra, rb, 1.f + H.e, H.beta_over_h, H.mu, rec, cnt);
          } else {
            contact<S>(sl, ra, rb, 1.f + H.e, H.beta_over_h, H.mu, rec, cnt);
          }
          Lanes<S>::st(cp, cnt);
        }
      }
#ifdef BRAX_DIAG
      if (dg) dt1 = clock64();
#endif
      __syncthreads();
      lap(1);
#ifdef BRAX_DIAG
      if (dg) dt2 = clock64();
#endif
      const bool last = s + 1 == H.S;
      const bool kin = !(last && (envm || step + 1 == a.n_steps));  // fused S2 of the next substep
      for (int i = bw0; i < bw1; ++i) {
        int b = bodies_of_warp[i * G];
        if (b < 0) continue;
        Acc<S> acc{typename Acc<S>::NoInit{}};
        const int j0 = jinc_begin[b], j1 = jinc_begin[b + 1], c0 = cinc_begin[b], c1 = cinc_begin[b + 1];
        const int nj = j1 - j0, nc = c1 - c0;  // warp-uniform: bodies sharing a step have one shape
        auto general = [&]() {
          if (nj > 0) acc.template gather<false>(jinc + j0, nj, sJe, LG * JS);
          else acc.zero_joints();
          if (nc > 0) acc.template gather<true>(cinc + c0, nc, sCe, LG * CS);
          else acc.zero_slots();
        };
        if constexpr (kFixed) {
#define BRAX_GF(NJ, NC) \
  if (nj == NJ && nc == NC) acc.template gather_fixed<NJ, NC>(jinc + j0, cinc + c0, sJe, LG * JS, sCe, LG * CS); else
          BRAX_GF(1, 2) BRAX_GF(2, 0) BRAX_GF(2, 2) BRAX_GF(3, 2) BRAX_GF(4, 1) general();
#undef BRAX_GF
        } else {
          general();
        }
#ifdef BRAX_DIAG
        if (dg) {  // stamp once the gathered sums exist (the store waits for them)
          dts = clock64();
          sDiag[warp] = diag_val(acc.F.x) + diag_val(acc.dV.x) + diag_val(acc.cnt);
          dtg = clock64();
        }
#endif
        float* co = (save_co && last) || cdp ? sCo + b * 6 * RW + el * SL : nullptr;
        const bool co_acc = cdp && s > 0;
        const Row<S> rb{sQ + (b * LG + el) * QS};
        if constexpr (kFixed) {  // specialised variant: isotropic bodies without frozen axes at compile time
          const int fl = bodies[b].flags;
          constexpr int kFreeFlags = kFlagIso | kFlagFreePos | kFlagFreeRot;
          if ((fl & kFreeFlags) == kFreeFlags && !bodies[b].rot_frozen)
            integrate<S, true>(bodies[b], rb, acc, H.h, H.g, kin, co, RW, co_acc);
          else
            integrate<S>(bodies[b], rb, acc, H.h, H.g, kin, co, RW, co_acc);
        } else {
          integrate<S>(bodies[b], rb, acc, H.h, H.g, kin, co, RW, co_acc);
        }
      }
#ifdef BRAX_DIAG
      if (dg) {
        unsigned smid, wid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
        printf("DIAG sm %u warp %d slot %u items %d bodies %d: p1 %lld wait1 %lld p2 %lld (setup+gather issue %lld, ready %lld)\n",
               smid, warp, wid, it1 - it0, bw1 - bw0, dt1 - dt0, dt2 - dt1, clock64() - dt2, dts - dt2, dtg - dt2);
      }
#endif
    }
    if (envm) {
      const uint2 key = make_uint2(uint32_t(a.seed & 0xffffffffu), uint32_t(a.seed >> 32));  // reset / marker draws
      __syncthreads();
      // reward, done, step / episode counters (one thread per env; goal tasks R36)
      for (int i = tid; i < E; i += blockDim.x) {
        float x1[3];  // the torso's (goal tasks: the object's) position after the step
        for (int k = 0; k < 3; ++k) x1[k] = sQ[qword<V>(T.obj, i, 0, k, LG)];
        const int32_t st1 = sSteps[i] + 1;
        float prog;
        if (T.has_goal) {  // R36: progress towards the marker (+ bonus and a new marker on a hit)
          float xt[3], s0 = 0.f, s1 = 0.f;
          for (int k = 0; k < 3; ++k) {
            xt[k] = sQ[qword<V>(T.target, i, 0, k, LG)];
            const float e0k = __fadd_rn(sX0[3 * i + k], -xt[k]), e1k = __fadd_rn(x1[k], -xt[k]);
            s0 = __fmaf_rn(e0k, e0k, s0);
            s1 = __fmaf_rn(e1k, e1k, s1);
          }
          const float d1 = __fsqrt_rn(s1);
          prog = __fdiv_rn(__fadd_rn(__fsqrt_rn(s0), -d1), T.dt);
          if (d1 < T.radius) {
            prog = __fadd_rn(prog, T.bonus);
            place_target(a.dqp, T.target, T.range, uint32_t(a.env_offset + e0 + i), uint32_t(2 + st1), sEp[i], key, xt);
            for (int k = 0; k < 3; ++k) sQ[qword<V>(T.target, i, 0, k, LG)] = xt[k];
          }
        } else {
          float fwd = __fmul_rn(__fadd_rn(x1[0], -sX0[3 * i]), T.fwd[0]);
          fwd = __fmaf_rn(__fadd_rn(x1[1], -sX0[3 * i + 1]), T.fwd[1], fwd);
          fwd = __fmaf_rn(__fadd_rn(x1[2], -sX0[3 * i + 2]), T.fwd[2], fwd);
          prog = __fdiv_rn(fwd, T.dt);
        }
        float ctrl = 0.f;
        for (int k = 0; k < A; ++k) {
          const float u = sA[k * RW + eslot<V>(i, LG)];
          ctrl = __fmaf_rn(u, u, ctrl);
        }
        const float reward = __fadd_rn(__fadd_rn(prog, T.survive), -__fmul_rn(T.ctrl_cost, ctrl));
        bool done = st1 >= T.episode_length;
        const float tz = sQ[qword<V>(T.torso, i, 0, 2, LG)];
        if (T.has_healthy) done = done || tz < T.z_lo || tz > T.z_hi;
        sRst[i] = done ? 1 : 0;
        sSteps[i] = done ? 0 : st1;
        if (done) sEp[i] += 1u;
        if (i < nvalid) {
          if (a.reward) a.reward[step * a.n_envs + e0 + i] = reward;
          if (a.done) a.done[step * a.n_envs + e0 + i] = done ? 1 : 0;
        }
      }
      __syncthreads();
      // auto-reset of done envs (R34): default_qp + noise, Philox counter (env, b, f, episode)
      for (int i = tid; i < E * B; i += blockDim.x) {
        const int env = i / B, b = i - env * B;
        if (!sRst[env]) continue;
        float x[3], q[4], v[3], w[3];
        reset_body(a.dqp, a.masks, B, b, uint32_t(a.env_offset + e0 + env), sEp[env], key, T.noise_vel,
                   T.noise_ang, x, q, v, w);
        if (T.has_goal && b == T.target)  // R36: the new episode's marker placement
          place_target(a.dqp, b, T.range, uint32_t(a.env_offset + e0 + env), 2u, sEp[env], key, x);
        for (int k = 0; k < 3; ++k) {
          sQ[qword<V>(b, env, 0, k, LG)] = x[k];
          sQ[qword<V>(b, env, 2, k, LG)] = v[k];
          sQ[qword<V>(b, env, 3, k, LG)] = w[k];
        }
        for (int k = 0; k < 4; ++k) sQ[qword<V>(b, env, 1, k, LG)] = q[k];
        if (save_co)
          for (int k = 0; k < 6; ++k) sCo[(b * 6 + k) * RW + eslot<V>(env, LG)] = 0.f;
      }
      __syncthreads();
      if (a.obs) observe(a.obs + (step * a.n_envs + e0) * od);
    }
  }
  if (envm) {
    for (int i = tid; i < nvalid; i += blockDim.x) {
      if (a.steps) a.steps[e0 + i] = sSteps[i];
      if (a.episode) a.episode[e0 + i] = sEp[i];
    }
  }
  lap(2);
  __syncthreads();
  // S9: status bits, contact counts, contact Δv sums, and the single write-back of the QP (TMA bulk for full blocks)
  block_extras<V>(a, sQ, sCnt, sStat, B, C, E, LG, e0, nvalid);
  if (cdp)
    for (int i = tid; i < nvalid * B * 6; i += blockDim.x) {
      const int env = i / (B * 6), r = i - env * (B * 6);
      a.contact_dp[(e0 + env) * B * 6 + r] = sCo[r * RW + eslot<V>(env, LG)];
    }
  if (bulk) {
    records_to_stg<V>(sQ, stg, B, E);
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      const float* sp = stg;
      const float* sr = sp + E * B * 3;
      const float* sv = sr + E * B * 4;
      const float* sw = sv + E * B * 3;
      tma_store(a.pos_out + e0 * B * 3, sp, uint32_t(E * B) * 12u);
      tma_store(a.rot_out + e0 * B * 4, sr, uint32_t(E * B) * 16u);
      tma_store(a.vel_out + e0 * B * 3, sv, uint32_t(E * B) * 12u);
      tma_store(a.ang_out + e0 * B * 3, sw, uint32_t(E * B) * 12u);
      if (ka.reg) tma_store_commit_wait_all();
      else tma_store_commit_wait();
    }
  } else if constexpr (kJvp) {
    store_block_d(a, sQ, B, E, e0, nvalid);
  } else {
    store_block<V>(a, sQ, B, E, e0, nvalid);
  }
  if (a.status) {
    __syncthreads();
    for (int i = tid; i < nvalid; i += blockDim.x) a.status[e0 + i] = sStat[i];
  }
  if (trace) {
    lap(3);
    for (int k = 0; k < 4; ++k) atomicAdd(&a.phase_cycles[k], (unsigned long long)sTr[k]);
  }
  if (ka.reg) {  // release this block's granules to the next launch
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async_global();
      __threadfence();
      for (int k = 0; k < ng; ++k) atomicAdd(ka.gd + g0 + k, 1u);
    }
  }
}

}  // namespace

// Lane-group plan for a launch: more, smaller blocks (G = 2, 4) when the batch
// alone would leave the SMs with few independent env groups to overlap their
// per-substep barriers; G = 1 once the grid fills the GPU.
int choose_plan(const System& sys, int64_t n_envs) {
  auto fits = [&](int i) { return sys.hd.plan[i].smem_bytes <= kMaxDynSmem; };
  if (const char* e = std::getenv("BRAX_PLAN")) {  // "G,V" override (experiments; ignored if it does not fit)
    int g = 0, v = 0;
    if (std::sscanf(e, "%d,%d", &g, &v) == 2)
      for (int i = 0; i < kNumPlans; ++i)
        if (sys.hd.plan[i].G == g && sys.hd.plan[i].V == v && fits(i)) return i;
  }
  int sms = sys.num_sms > 0 ? sys.num_sms : 148;
  int64_t blocks32 = (n_envs + 31) / 32;
  // measured (profiles/): lane groups help only while the smaller blocks still
  // fit one per SM (the batch is too small to fill the GPU with 32-env blocks)
  int p = 0;
  if (4 * blocks32 <= sms) p = 2;
  else if (2 * blocks32 <= sms) p = 1;
  else if (blocks32 >= 4 * sms) p = 3;  // large batches: two envs per lane (G = 1, V = 2)
  if (fits(p)) return p;
  // large systems: the biggest one-env-per-lane block that fits (plan 2, 8 envs, always does)
  for (int q : {0, 1, 2})
    if (fits(q)) return q;
  return 2;
}

// Register budget per thread: as many as possible while the SM still holds the
// number of blocks the grid can use (B200: 148 SMs, 64 K registers = 4 SMSPs x
// 16 K, 228 KB shared memory, 64 warps).  Measured (profiles/): more registers
// buy ILP for latency-bound small batches, occupancy wins for large ones.
int choose_regs(const System& sys, const DPlan& P, int64_t grid) {
  if (const char* e = std::getenv("BRAX_MAXREG")) return std::atoi(e);
  const int sms = sys.num_sms > 0 ? sys.num_sms : 148;
  const int64_t want = (grid + sms - 1) / sms;
  const int by_smem = (228 * 1024) / (P.smem_bytes + 1024);
  const int by_warps = 64 / P.W;
  int blocks = int(want < 8 ? want : 8);
  blocks = blocks < by_smem ? blocks : by_smem;
  blocks = blocks < by_warps ? blocks : by_warps;
  blocks = blocks < 1 ? 1 : blocks;
  const int warps_per_smsp = (blocks * P.W + 3) / 4;
  return (16384 / (warps_per_smsp * 32)) & ~7;
}

namespace {
template <class S, int R, bool kEnv = false, bool kFixed = false>
cudaError_t launch_variant(const KArgs& ka, dim3 grid, dim3 block, size_t smem, cudaStream_t stream) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(brax_step_kernel<S, R, kEnv, kFixed>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kMaxDynSmem);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: prologue overlaps the previous kernel
  attr[0].val.programmaticStreamSerializationAllowed = std::getenv("BRAX_NO_PDL") ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, brax_step_kernel<S, R, kEnv, kFixed>, ka);
}

cudaError_t launch_with_args(const System& sys, KArgs& ka, int regs, bool fixed, cudaStream_t stream);

cudaError_t launch_with(const System& sys, const StepArgs& a, int plan, int regs, bool fixed, cudaStream_t stream) {
  auto order = launch_order_lock();  // held across the launch: recorded order = stream order
  // observe-only env launches return early and do not take part in the granule protocol
  const OverlapDecision d = overlap_decide(sys, a, stream, !(a.env && a.n_steps == 0));
  KArgs ka{a, sys.d_blob, sys.hd, plan, sys.d_gran, sys.d_gran + kMaxGranules, d.reg ? 1 : 0, d.overlap ? 1 : 0};
  const cudaError_t e = launch_with_args(sys, ka, regs, fixed, stream);
  overlap_commit(sys, a, stream, d, e);
  return e;
}

cudaError_t launch_with_args(const System& sys, KArgs& ka, int regs, bool fixed, cudaStream_t stream) {
  const StepArgs& a = ka.a;
  const int plan = ka.plan;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  ka.a.bulk_ok = al16(a.pos_in) && al16(a.rot_in) && al16(a.vel_in) && al16(a.ang_in) && al16(a.pos_out) &&
                 al16(a.rot_out) && al16(a.vel_out) && al16(a.ang_out);
  ka.a.act_bulk_ok = a.actions && al16(a.actions) && ((a.n_envs * sys.hd.A) % 4 == 0);
  if (std::getenv("BRAX_NO_BULK")) ka.a.bulk_ok = ka.a.act_bulk_ok = 0;
  ka.a.phase_cycles = sys.trace ? sys.d_phase_cycles : nullptr;
  if (sys.trace) fixed = false;  // tracing is compiled into the generic variants only
  if (const char* e = std::getenv("BRAX_DIAG_BLOCK")) ka.a.diag_block = std::atoi(e);
  const DPlan& P = sys.hd.plan[plan];
  dim3 grid(unsigned((a.n_envs + P.E - 1) / P.E)), block(unsigned(P.W * 32));
  const size_t smem = size_t(a.env ? P.smem_bytes_env : a.contact_dp ? P.smem_bytes_cdp : P.smem_bytes);
  if (a.env) {  // env-epilogue instantiations (fewer register variants)
    if (P.V == 2) {
      if (fixed) {
        if (regs >= 128) return launch_variant<F2, 128, true, true>(ka, grid, block, smem, stream);
        return launch_variant<F2, 96, true, true>(ka, grid, block, smem, stream);
      }
      if (regs >= 128) return launch_variant<F2, 128, true>(ka, grid, block, smem, stream);
      return launch_variant<F2, 96, true>(ka, grid, block, smem, stream);
    }
    if (regs >= 128) return launch_variant<F1, 128, true>(ka, grid, block, smem, stream);
    if (regs >= 96) return launch_variant<F1, 96, true>(ka, grid, block, smem, stream);
    return launch_variant<F1, 64, true>(ka, grid, block, smem, stream);
  }
  if (P.V == 2) {
    if (fixed) {
      if (regs >= 128) return launch_variant<F2, 128, false, true>(ka, grid, block, smem, stream);
      if (regs >= 96) return launch_variant<F2, 96, false, true>(ka, grid, block, smem, stream);
      return launch_variant<F2, 80, false, true>(ka, grid, block, smem, stream);
    }
    if (regs >= 128) return launch_variant<F2, 128>(ka, grid, block, smem, stream);
    if (regs >= 96) return launch_variant<F2, 96>(ka, grid, block, smem, stream);
    return launch_variant<F2, 80>(ka, grid, block, smem, stream);
  }
  if (regs >= 128) return launch_variant<F1, 128>(ka, grid, block, smem, stream);
  if (regs >= 112) return launch_variant<F1, 112>(ka, grid, block, smem, stream);
  if (regs >= 96) return launch_variant<F1, 96>(ka, grid, block, smem, stream);
  if (regs >= 80) return launch_variant<F1, 80>(ka, grid, block, smem, stream);
  if (regs >= 64) return launch_variant<F1, 64>(ka, grid, block, smem, stream);
  return launch_variant<F1, 56>(ka, grid, block, smem, stream);
}

// the register budget of the instantiated variant launch_with runs for `regs`
int variant_regs(int V, int regs) {
  static const int v2[] = {128, 96, 80}, v1[] = {128, 112, 96, 80, 64, 56};
  const int* t = V == 2 ? v2 : v1;
  const int n = V == 2 ? 3 : 6;
  for (int i = 0; i < n; ++i)
    if (regs >= t[i]) return t[i];
  return t[n - 1];
}

bool plan_fits(const System& sys, int p) { return sys.hd.plan[p].smem_bytes <= kMaxDynSmem; }

int64_t grid_of(const System& sys, int p, int64_t n) { return (n + sys.hd.plan[p].E - 1) / sys.hd.plan[p].E; }

LaunchConfig heuristic_config(const System& sys, int64_t n) {
  LaunchConfig c;
  c.plan = choose_plan(sys, n);
  if (const char* e = std::getenv("BRAX_FIXED_GATHER")) c.fixed = std::atoi(e) != 0;  // experiments / tests
  if (const char* e = std::getenv("BRAX_LEAN")) c.lean = std::atoi(e) != 0;
  const char* e = std::getenv("BRAX_MAXREG");
  c.regs = variant_regs(sys.hd.plan[c.plan].V,
                        e ? std::atoi(e) : choose_regs(sys, sys.hd.plan[c.plan], grid_of(sys, c.plan, n)));
  return c;
}

// Times one step of every plan that fits (at its register budget), reading the
// caller's state and actions and writing scratch buffers; the caller's buffers are
// not written.
LaunchConfig tune(const System& sys, const StepArgs& a, cudaStream_t stream) {
  LaunchConfig best = heuristic_config(sys, a.n_envs);
  if (!sys.autotune || std::getenv("BRAX_PLAN") || std::getenv("BRAX_MAXREG")) return best;
  const int64_t n = a.n_envs, B = sys.hd.B;
  const size_t fbytes[4] = {size_t(n * B * 3 * 4), size_t(n * B * 4 * 4), size_t(n * B * 3 * 4),
                            size_t(n * B * 3 * 4)};
  float* buf = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), fbytes[0] + fbytes[1] + fbytes[2] + fbytes[3], stream) !=
      cudaSuccess) {
    cudaGetLastError();
    return best;
  }
  float* f[4] = {buf, nullptr, nullptr, nullptr};
  for (int k = 1; k < 4; ++k) f[k] = f[k - 1] + fbytes[k - 1] / 4;
  // the trials step a scratch copy of the caller's state in place (the caller's buffers are
  // not written): stepping one fixed input out of place ranked the plans differently from a
  // trajectory (ant 8192: (2,2) chosen, 1 µs slower per step in bench.py than (4,2)); the
  // candidates are timed in interleaved rounds, so the state's drift reaches all alike
  StepArgs t = a;
  const float* src[4] = {a.pos_in, a.rot_in, a.vel_in, a.ang_in};
  for (int k = 0; k < 4; ++k) cudaMemcpyAsync(f[k], src[k], fbytes[k], cudaMemcpyDeviceToDevice, stream);
  t.pos_in = t.pos_out = f[0];
  t.rot_in = t.rot_out = f[1];
  t.vel_in = t.vel_out = f[2];
  t.ang_in = t.ang_out = f[3];
  t.n_steps = 1;
  t.status = nullptr;
  t.contact_active = nullptr;
  t.contact_dp = nullptr;
  t.env = 0;
  // candidates: every plan that fits, its generic / specialised / lean kernels at the plan's
  // register budget; each warmed up (and checked feasible) once
  std::vector<LaunchConfig> cands;
  auto run = [&](const LaunchConfig& c) {
    return c.lean ? launch_lean(sys, t, c.plan, c.regs, stream) : launch_with(sys, t, c.plan, c.regs, c.fixed, stream);
  };
  for (int p = 0; p < kNumPlans; ++p) {
    if (!plan_fits(sys, p)) continue;
    const int regs = variant_regs(sys.hd.plan[p].V, choose_regs(sys, sys.hd.plan[p], grid_of(sys, p, n)));
    std::vector<LaunchConfig> cs;
    for (int fx = 0; fx < (sys.hd.plan[p].V == 2 ? 2 : 1); ++fx) {
      LaunchConfig c;
      c.plan = p;
      c.regs = regs;
      c.fixed = fx != 0;
      cs.push_back(c);
    }
    if (lean_applies(sys, p, t)) {  // the lean kernel of this plan (same bits) at each of its
      // register budgets: with overlapped launches the best budget is not the one the
      // occupancy heuristic picks (ant 65 k: 96 registers 155 µs, 80 registers 162 µs)
      const int lean_regs[3] = {80, 96, 128};
      for (int r : lean_regs) {
        LaunchConfig c;
        c.plan = p;
        c.regs = sys.hd.plan[p].V == 2 ? r : (r == 80 ? 64 : r);  // F1 instantiations: 64 / 96 / 128
        c.fixed = true;
        c.lean = true;
        cs.push_back(c);
      }
    }
    for (const LaunchConfig& c : cs) {
      if (run(c) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      cands.push_back(c);
    }
  }
  // interleaved timing of CUDA graphs of 32 launches per candidate (the way a caller replays
  // steps; long enough that the first launch's missing overlap with a predecessor does not
  // decide), five rounds, each candidate's fastest round; on a private stream
  // ordered after the caller's work (graph capture needs a non-legacy stream)
  cudaEvent_t e0, e1, ready;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
  cudaStream_t ts = nullptr;
  cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking);
  cudaEventRecord(ready, stream);
  cudaStreamWaitEvent(ts, ready, 0);
  std::vector<cudaGraphExec_t> gx(cands.size(), nullptr);
  for (size_t i = 0; i < cands.size(); ++i) {
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(ts, cudaStreamCaptureModeThreadLocal) != cudaSuccess) break;
    cudaStream_t keep = stream;
    stream = ts;  // run() launches on `stream`
    for (int r = 0; r < 32; ++r) run(cands[i]);
    stream = keep;
    if (cudaStreamEndCapture(ts, &g) == cudaSuccess && g) {
      if (cudaGraphInstantiate(&gx[i], g, 0) != cudaSuccess) gx[i] = nullptr;
      cudaGraphDestroy(g);
    }
    cudaGetLastError();
  }
  std::vector<float> best_of(cands.size(), 1e30f);
  for (int round = 0; round < 5; ++round)
    for (size_t i = 0; i < cands.size(); ++i) {
      if (!gx[i]) continue;
      cudaEventRecord(e0, ts);
      cudaGraphLaunch(gx[i], ts);
      cudaEventRecord(e1, ts);
      float m = 0.f;
      if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&m, e0, e1) != cudaSuccess) {
        cudaGetLastError();
        m = 1e30f;
      }
      if (round > 0) best_of[i] = std::min(best_of[i], m);  // round 0 uploads the graphs
    }
  for (cudaGraphExec_t x : gx)
    if (x) cudaGraphExecDestroy(x);
  cudaStreamSynchronize(ts);
  cudaStreamDestroy(ts);
  cudaEventDestroy(ready);
  float best_ms = 1e30f;
  for (size_t i = 0; i < cands.size(); ++i)
    if (best_of[i] < best_ms) {
      best_ms = best_of[i];
      best = cands[i];
    }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(buf, stream);
  cudaStreamSynchronize(stream);
  best.tuned = true;
  return best;
}
}  // namespace

// NEXT-4 JVP: lane type D1 on the one-env-per-lane plan of the heuristic's lane-group count
cudaError_t launch_step_jvp(const System& sys, const StepArgs& a, cudaStream_t stream) {
  if (a.n_envs <= 0 || a.n_steps <= 0) return cudaSuccess;
  int p = choose_plan(sys, a.n_envs);
  if (sys.hd.plan[p].V == 2) p -= 3;  // plans 3-5 are the V = 2 versions of plans 0-2
  while (p < 2 && sys.hd.plan[p].smem_bytes_jvp > kMaxDynSmem) ++p;  // smaller blocks for large systems
  DPlan P = sys.hd.plan[p];
  if (P.smem_bytes_jvp > kMaxDynSmem) return cudaErrorInvalidValue;
  P.smem_bytes = P.smem_bytes_jvp;
  auto order = launch_order_lock();
  note_other_launch(sys, stream);
  KArgs ka{a, sys.d_blob, sys.hd, p};
  ka.a.bulk_ok = ka.a.act_bulk_ok = 0;
  ka.a.phase_cycles = nullptr;
  dim3 grid(unsigned((a.n_envs + P.E - 1) / P.E)), block(unsigned(P.W * 32));
  const int regs = choose_regs(sys, P, int64_t(grid.x));
  if (regs >= 255) return launch_variant<D1, 255>(ka, grid, block, size_t(P.smem_bytes), stream);
  return launch_variant<D1, 128>(ka, grid, block, size_t(P.smem_bytes), stream);
}

LaunchConfig launch_config(const System& sys, int64_t n_envs) {
  if (std::getenv("BRAX_PLAN") || std::getenv("BRAX_MAXREG")) return heuristic_config(sys, n_envs);
  {
    std::lock_guard<std::mutex> g(sys.tune_mu);
    auto it = sys.tuned.find(n_envs);
    if (it != sys.tuned.end()) return it->second;
  }
  return heuristic_config(sys, n_envs);
}

// Explicit tuning (brax_system_tune): measures every plan on the caller's state and
// remembers the fastest for a.n_envs.  Allocates stream-ordered scratch and
// synchronises the stream; brax_step itself never does either.
cudaError_t tune_system(const System& sys, const StepArgs& a, cudaStream_t stream) {
  if (a.n_envs <= 0) return cudaSuccess;
  LaunchConfig c = tune(sys, a, stream);
  cudaError_t e = cudaGetLastError();
  std::lock_guard<std::mutex> g(sys.tune_mu);
  sys.tuned[a.n_envs] = c;
  return e;
}

cudaError_t launch_step(const System& sys, const StepArgs& a, cudaStream_t stream) {
  if (a.n_envs <= 0 || (a.n_steps <= 0 && !a.env)) return cudaSuccess;
  LaunchConfig c = launch_config(sys, a.n_envs);
  // the env epilogue / contact_dp regions may not fit the tuned plan: the largest block that does
  auto bytes = [&](int p) { return a.env ? sys.hd.plan[p].smem_bytes_env
                                         : a.contact_dp ? sys.hd.plan[p].smem_bytes_cdp : sys.hd.plan[p].smem_bytes; };
  if (bytes(c.plan) > kMaxDynSmem) {
    int q = -1;
    for (int p = kNumPlans - 1; p >= 0; --p)
      if (bytes(p) <= kMaxDynSmem && (q < 0 || sys.hd.plan[p].E > sys.hd.plan[q].E)) q = p;
    if (q < 0) return cudaErrorInvalidValue;
    c.plan = q;
    c.regs = variant_regs(sys.hd.plan[q].V, choose_regs(sys, sys.hd.plan[q], grid_of(sys, q, a.n_envs)));
    c.lean = false;
  }
  if (c.lean && lean_applies(sys, c.plan, a)) return launch_lean(sys, a, c.plan, c.regs, stream);
  return launch_with(sys, a, c.plan, c.regs, c.fixed, stream);
}

}  // namespace brax
