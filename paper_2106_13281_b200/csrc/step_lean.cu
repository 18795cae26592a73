// step_lean.cu — the lean step kernel: the same physics as brax_step_kernel
// (Alg. 1; device code in step_device.cuh, identical operations in
// the identical order, so identical bits) with the per-substep scaffolding cut down
// for the common launch shape (DESIGN.md §5 "Lean kernel").
//
// Applies to the plans whose work plan gives every warp at most one body step and at
// most one item step (the planner's G > 1 rule W = max(item steps, body steps) does, up
// to 16 warps) or, for the one-lane-group two-envs-per-lane plans of large batches
// (W = ⌈item steps / 2⌉), two item steps (kItems = 2, physics launches).  Then:
//   * G, the lanes per group, E and every record stride are compile-time constants;
//   * each warp's item and body, their code class (the specialised classes of the
//     kFixed variant, else the generic code) and their shared-memory record addresses
//     are resolved once, before the substep loop, instead of once per substep;
//   * no JVP, tracing or contact-Δv code is compiled in (those launches use
//     brax_step_kernel); the env epilogue (NEXT-1) is a separate instantiation (kEnv),
//     with brax_step_kernel's epilogue code in the same order (same bits).
// Measured on B200 (tools/experiments/ab.sh): see DESIGN.md §5.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>
#include <vector>

#include "device_rng.cuh"
#include "step_device.cuh"
#include "system.h"

namespace brax {
namespace {

using namespace dev;

struct LeanArgs {
  StepArgs a;
  const uint32_t* blob;
  DHeader hd;
  int32_t plan;
  SmemLayout L;
  // launch overlap: per env granule, launches started (gs) / finished (gd)
  uint32_t* gs;
  uint32_t* gd;
  int32_t reg;       // this launch registers on the granule counters
  int32_t overlap;   // skip griddepcontrol.wait: wait for the granules' earlier launches instead
};

#ifdef BRAX_DIAG
// block timelines (tools/experiments/overlap_timeline.sh): [launch tag][block][entry, after
// the wait, staged, loop end, stored, smid, overlap, exit] in globaltimer ns
constexpr int kDiagLaunches = 16, kDiagBlocks = 4096;
__device__ long long g_diag_tl[kDiagLaunches * kDiagBlocks * 8];
#endif

// item classes (warp-uniform: the items sharing a warp step share a class)
enum : int {
  kItemNone = 0, kJointHinge = 1, kJoint2 = 2, kJoint3 = 3, kJointGeneric = 4,
  kCapsuleGround = 5, kSphereGround = 6, kBoxGround = 7, kContactGeneric = 8,
};
// body gather shapes with compile-time list lengths (as in the kFixed variant)
enum : int { kGatherGeneral = 0, kG12 = 1, kG20 = 2, kG22 = 3, kG32 = 4, kG41 = 5 };

// kItems: the most item steps a warp of the plan has (2: the one-lane-group plans of large
// batches, W = ⌈item steps / 2⌉; physics launches only)
template <class S, int G, int R, bool kEnv, int kItems = 1>
__global__ void __maxnreg__(R) brax_step_lean(const __grid_constant__ LeanArgs ka) {
  // S = F2: two envs per lane (packed FP32); F1: one env per lane (small batches)
  constexpr int V = Lanes<S>::V, SL = Lanes<S>::SL, LG = 32 / G, E = V * LG, RW = LG * SL;
  constexpr int LGS = G == 1 ? 5 : G == 2 ? 4 : 3;  // log2(LG)
  constexpr int QS = Lanes<S>::QS, JS = Lanes<S>::JS, CS = Lanes<S>::CS;
  extern __shared__ __align__(16) uint32_t smem[];
  const DHeader& H = ka.hd;
  const DPlan& P = H.plan[ka.plan];
  const StepArgs& a = ka.a;
  const SmemLayout& L = ka.L;
  const int B = H.B, J = H.J, C = H.C, A = H.A;
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
  // env epilogue (kEnv): torso position at the step start, steps / episode / reset flag per
  // env, contact Δv of the last substep, observation rows (alias U)
  const DTask& T = H.task;
  float* sX0 = reinterpret_cast<float*>(smem + L.x0);
  int32_t* sSteps = reinterpret_cast<int32_t*>(smem + L.steps);
  uint32_t* sEp = smem + L.ep;
  int32_t* sRst = reinterpret_cast<int32_t*>(smem + L.rst);
  float* sCo = reinterpret_cast<float*>(smem + L.co);
  float* sObs = reinterpret_cast<float*>(smem + L.u);
  const bool save_co = kEnv && T.contact_obs;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane >> LGS, el = lane & (LG - 1);
  const int64_t e0 = int64_t(blockIdx.x) * E;
  const int nvalid = (a.n_envs - e0 < E) ? int(a.n_envs - e0) : E;
  const bool bulk = a.bulk_ok && nvalid == E;  // block-uniform
  const bool act_bulk = bulk && a.act_bulk_ok && A > 0;
  const uint32_t qp_bytes = uint32_t(E * B) * 13u * 4u, act_bytes = uint32_t(E * A) * 4u;

#ifdef BRAX_DIAG  // block timeline (globaltimer, ns): entry, after griddepcontrol.wait, staged, loop end, exit
  __shared__ long long sDg[kMaxWarps][4];
  long long tl[5] = {0, 0, 0, 0, 0};
  const bool dgb = a.diag_block && tid == 0 && (a.diag_block >= 1000 || (blockIdx.x % 64) == 0);
  auto gtime = []() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
  if (dgb) tl[0] = gtime();
#endif
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
  // The QP may be the previous launch's output.  Default: PDL's grid-wide wait.  Overlapped
  // launches (host-checked: the launches of this system still in flight on this stream use
  // buffers that are this launch's, env for env, or disjoint from them): register as
  // the next launch of each of the block's env granules, let the next launch be scheduled,
  // and wait only until every earlier launch on these granules has finished.
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
#ifndef BRAX_OVERLAP_NO_SPIN  // (negative control for tests/test_gpu_overlap.py only: races on purpose)
    if (tid < ng)
      while (int32_t(gdone - gprev) < 0) {
        __nanosleep(64);
        gdone = ld_acquire_gpu(ka.gd + g0 + tid);
      }
#endif
    __syncthreads();
    if (tid == 0) fence_proxy_async_global();  // the TMA loads below read what the acquire made visible
  }
#ifdef BRAX_DIAG
  if (dgb) tl[1] = gtime();
#endif
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
  if (!bulk) load_block<V>(a, sQ, B, E, e0, nvalid);  // ragged tail / unaligned: per-row loads
  mbar_wait(&bars[0], 0);
  if (bulk) stg_to_records<V>(stg, sQ, B, E);
  for (int i = tid; i < E; i += blockDim.x) sStat[i] = 0u;
  if (kEnv) {
    for (int i = tid; i < E; i += blockDim.x) {
      sSteps[i] = i < nvalid && a.steps ? a.steps[e0 + i] : 0;
      sEp[i] = i < nvalid && a.episode ? a.episode[e0 + i] : 0u;
    }
    if (save_co)
      for (int i = tid; i < 6 * B * RW; i += blockDim.x) sCo[i] = 0.f;
  }
  __syncthreads();
#ifdef BRAX_DIAG
  if (dgb) tl[2] = gtime();
#endif

  // ---- this warp's program, resolved once: at most kItems items and one body ----
  const DBody* bodies = reinterpret_cast<const DBody*>(sBlob + H.off_bodies);
  const int32_t* item_begin = reinterpret_cast<const int32_t*>(sBlob + P.off_item_begin);
  const int32_t* body_begin = reinterpret_cast<const int32_t*>(sBlob + P.off_body_begin);
  const int it0 = item_begin[warp], nit = item_begin[warp + 1] - it0;
  const int bw0 = body_begin[warp];
  const int body = bw0 < body_begin[warp + 1]
                       ? reinterpret_cast<const int32_t*>(sBlob + P.off_bodies_of_warp)[bw0 * G + grp]
                       : -1;
  struct ItemProg {
    int cls = kItemNone;
    const uint32_t* params = nullptr;  // the item's parameter record (DJoint / DSlot) in shared memory
    float *p = nullptr, *c = nullptr, *rec = nullptr, *cnt = nullptr;  // record addresses
  };
  auto resolve = [&](int k) {
    ItemProg r;
    const int item = k < nit ? reinterpret_cast<const int32_t*>(sBlob + P.off_items)[(it0 + k) * G + grp] : -1;
    if (item >= 0 && item < J) {
      const DJoint& jt = reinterpret_cast<const DJoint*>(sBlob + H.off_joints)[item];
      const int4 h0 = *reinterpret_cast<const int4*>(&jt);
      r.cls = h0.w == 0 ? (h0.z == 1 ? kJointHinge : h0.z == 2 ? kJoint2 : h0.z == 3 ? kJoint3 : kJointGeneric)
                        : kJointGeneric;
      r.params = reinterpret_cast<const uint32_t*>(&jt);
      r.p = sQ + ((h0.x << LGS) + el) * QS;
      r.c = sQ + ((h0.y << LGS) + el) * QS;
      r.rec = sJ + ((item << LGS) + el) * JS;
    } else if (item >= J) {
      const int c = item - J;
      const DSlot& sl = reinterpret_cast<const DSlot*>(sBlob + H.off_slots)[c];
      const int4 h0 = *reinterpret_cast<const int4*>(&sl), h1 = reinterpret_cast<const int4*>(&sl)[1];
      const bool ground = h1.x == 0 && h1.y == 1 && (h1.z & kCapsuleOnGroundFlags) == kCapsuleOnGroundFlags;
      r.cls = !ground ? kContactGeneric : h0.x == 1 ? kCapsuleGround : h0.x == 0 ? kSphereGround
                                        : h0.x == 2 ? kBoxGround : kContactGeneric;
      r.params = reinterpret_cast<const uint32_t*>(&sl);
      r.p = sQ + ((h0.y << LGS) + el) * QS;
      r.c = sQ + ((h0.z << LGS) + el) * QS;
      r.rec = sC + ((c << LGS) + el) * CS;
      r.cnt = sCnt + c * RW + el * SL;
    }
    return r;
  };
  const ItemProg it_a = resolve(0);
  const ItemProg it_b = kItems > 1 ? resolve(1) : ItemProg{};
  const int icls = it_a.cls;
  const uint32_t* iparams = it_a.params;
  float *ip = it_a.p, *ic = it_a.c;
  int gcls = kGatherGeneral, j0 = 0, nj = 0, c0 = 0, nc = 0;
  bool free_body = false;
  float* brow = nullptr;
  if (body >= 0) {
    const int32_t* jinc_begin = reinterpret_cast<const int32_t*>(sBlob + H.off_jinc_begin);
    const int32_t* cinc_begin = reinterpret_cast<const int32_t*>(sBlob + H.off_cinc_begin);
    j0 = jinc_begin[body];
    nj = jinc_begin[body + 1] - j0;
    c0 = cinc_begin[body];
    nc = cinc_begin[body + 1] - c0;
    gcls = nj == 1 && nc == 2 ? kG12 : nj == 2 && nc == 0 ? kG20 : nj == 2 && nc == 2 ? kG22
         : nj == 3 && nc == 2 ? kG32 : nj == 4 && nc == 1 ? kG41 : kGatherGeneral;
    constexpr int kFreeFlags = kFlagIso | kFlagFreePos | kFlagFreeRot;
    free_body = (bodies[body].flags & kFreeFlags) == kFreeFlags && !bodies[body].rot_frozen;
    brow = sQ + ((body << LGS) + el) * QS;
  }
  const float* sJe = sJ + el * JS;  // this lane's record of joint 0 (joint j: + j·LG·JS)
  const float* sCe = sC + el * CS;

  const int od = T.obs_dim;
  // NEXT-1: the torso's (goal tasks: the object's) position at the step boundary, before S2,
  // saved by the lane group that integrates that body (program order: no barrier needed)
  auto save_x0 = [&]() {
    if (body != T.obj) return;
    const V3T<S> x = Row<S>{brow}.pos();
    if constexpr (V == 2) {
      const float a0[3] = {x.x.x, x.y.x, x.z.x}, a1[3] = {x.x.y, x.y.y, x.z.y};
      for (int k = 0; k < 3; ++k) {
        sX0[3 * el + k] = a0[k];
        sX0[3 * (el + LG) + k] = a1[k];
      }
    } else {
      const float a0[3] = {x.x.x, x.y.x, x.z.x};
      for (int k = 0; k < 3; ++k) sX0[3 * el + k] = a0[k];
    }
  };
  auto observe = [&](float* obs_out) {  // NEXT-1: obs rows of the block's envs -> obs_out [nvalid][od]
    if (icls != kItemNone && icls <= kJointGeneric) {  // joints: angles and rates, by the warps that own them
      const DJoint& jt = *reinterpret_cast<const DJoint*>(iparams);
      joint_obs<S>(jt, Row<S>{ip}, Row<S>{ic}, sObs + el * od, LG * od, 5 + jt.obs_off, 11 + T.nq + jt.obs_off);
    }
    // torso, goal and contact parts, one thread per (env, word)
    const int nco = T.contact_obs ? 6 * B : 0, ng = T.has_goal ? 9 : 0, nw = 11 + ng + nco;
    for (int i = tid; i < E * nw; i += blockDim.x) {
      const int k = i / E, env = i - k * E;  // E is a compile-time power of two: shifts, not a division
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

  // S2 of the first substep; every later S2 is fused into the previous substep's integrate()
  // (env mode ends every step at the boundary: its S2 runs at the next step's start)
  if (kEnv) save_x0();
  if (body >= 0) kinematic<S>(bodies[body], Row<S>{brow}, H.h);
  for (int64_t step = 0; step < a.n_steps; ++step) {
    if (kEnv && step > 0) {
      save_x0();
      if (body >= 0) kinematic<S>(bodies[body], Row<S>{brow}, H.h);
    }
    if (act_bulk) {  // this step's actions arrived in sAstg [E][A]; transpose to sA [A][E]
      mbar_wait(&bars[1], uint32_t(step & 1));
      for (int i = tid; i < E * A; i += blockDim.x) {
        const int env = i / A, k = i - env * A;
        sA[k * RW + eslot<V>(env, LG)] = sAstg[i];
      }
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
    }  // sA is read after the next barrier
    if (it_a.cnt) Lanes<S>::st(it_a.cnt, bc<S>(0.f));
    if (kItems > 1 && it_b.cnt) Lanes<S>::st(it_b.cnt, bc<S>(0.f));
    const bool pf_act = act_bulk && tid == 0 && step + 1 < a.n_steps;
    for (int s = 0; s < H.S; ++s) {
      __syncthreads();
#ifdef BRAX_DIAG  // per-warp clock stamps of substep 3 of step 0 in one block (build with -DBRAX_DIAG)
      const bool dg = a.diag_block && step == 0 && s == 3 && int(blockIdx.x) == a.diag_block - 1 && lane == 0;
      if (dg) sDg[warp][0] = clock64();
#endif
      if (s == 0 && pf_act) {  // prefetch next step's actions
        mbar_expect_tx(&bars[1], act_bytes);
        tma_load(sAstg, a.actions + ((step + 1) * a.n_envs + e0) * A, act_bytes, &bars[1]);
      }
      // phase 1: this warp's joint (with its actuator) or contact slot (S3-S5); kItems = 2:
      // the second one after it (one call site per class: the loop is not unrolled)
#pragma unroll 1
      for (int k = 0; k < kItems; ++k) {
        const ItemProg& it = k == 0 ? it_a : it_b;
        const int cls = it.cls;
        if (cls == kItemNone) break;
        const Row<S> rp{it.p}, rc{it.c};
        float* const irec = it.rec;
        if (cls <= kJointGeneric) {
          const DJoint& jt = *reinterpret_cast<const DJoint*>(it.params);
          const float* act = sA + el * SL;
          if (cls == kJointHinge) joint<S, 1, 0>(jt, rp, rc, act, RW, irec);
          else if (cls == kJoint2) joint<S, 2, 0>(jt, rp, rc, act, RW, irec);
          else if (cls == kJoint3) joint<S, 3, 0>(jt, rp, rc, act, RW, irec);
          else joint<S>(jt, rp, rc, act, RW, irec);
        } else {
          const DSlot& sl = *reinterpret_cast<const DSlot*>(it.params);
          float* const icnt = it.cnt;
          S cnt = Lanes<S>::ld(icnt);
          if (cls == kCapsuleGround) contact<S, 1>(sl, rp, rc, 1.f + H.e, H.beta_over_h, H.mu, irec, cnt);
          else if (cls == kSphereGround) contact<S, 2>(sl, rp, rc, 1.f + H.e, H.beta_over_h, H.mu, irec, cnt);
          else if (cls == kBoxGround) contact<S, 3>(sl, rp, rc, 1.f + H.e, H.beta_over_h, H.mu, irec, cnt);
          else contact<S>(sl, rp, rc, 1.f + H.e, H.beta_over_h, H.mu, irec, cnt);
          Lanes<S>::st(icnt, cnt);
        }
      }
#ifdef BRAX_DIAG
      if (dg) sDg[warp][1] = clock64();
#endif
      __syncthreads();
#ifdef BRAX_DIAG
      if (dg) sDg[warp][2] = clock64();
#endif
      // phase 2: this warp's body — gather (S6), potential + collision integrators
      // (S7, S8) fused with the next substep's kinematic integrator (S2)
      if (body >= 0) {
        const bool last = s + 1 == H.S;
        const bool kin = !(last && (kEnv || step + 1 == a.n_steps));
        float* const co = save_co && last ? sCo + body * 6 * RW + el * SL : nullptr;
        const int32_t* jl = reinterpret_cast<const int32_t*>(sBlob + H.off_jinc) + j0;
        const int32_t* cl = reinterpret_cast<const int32_t*>(sBlob + H.off_cinc) + c0;
        Acc<S> acc{typename Acc<S>::NoInit{}};
        switch (gcls) {
          case kG12: acc.template gather_fixed<1, 2>(jl, cl, sJe, LG * JS, sCe, LG * CS); break;
          case kG20: acc.template gather_fixed<2, 0>(jl, cl, sJe, LG * JS, sCe, LG * CS); break;
          case kG22: acc.template gather_fixed<2, 2>(jl, cl, sJe, LG * JS, sCe, LG * CS); break;
          case kG32: acc.template gather_fixed<3, 2>(jl, cl, sJe, LG * JS, sCe, LG * CS); break;
          case kG41: acc.template gather_fixed<4, 1>(jl, cl, sJe, LG * JS, sCe, LG * CS); break;
          default:
            if (nj > 0) acc.template gather<false>(jl, nj, sJe, LG * JS);
            else acc.zero_joints();
            if (nc > 0) acc.template gather<true>(cl, nc, sCe, LG * CS);
            else acc.zero_slots();
        }
        if (free_body) integrate<S, true>(bodies[body], Row<S>{brow}, acc, H.h, H.g, kin, co, RW);
        else integrate<S>(bodies[body], Row<S>{brow}, acc, H.h, H.g, kin, co, RW);
      }
#ifdef BRAX_DIAG
      if (dg) sDg[warp][3] = clock64();  // printed after the substep loop (printf would skew the stamps)
#endif
    }
    if (kEnv) {  // NEXT-1 epilogue of this step (R30-R34, R36), brax_step_kernel's code and order
      const uint2 key = make_uint2(uint32_t(a.seed & 0xffffffffu), uint32_t(a.seed >> 32));  // reset / marker draws
      __syncthreads();
      for (int i = tid; i < E; i += blockDim.x) {  // reward, done, step / episode counters
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
        const int b = i / E, env = i - b * E;
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
  if (kEnv)
    for (int i = tid; i < nvalid; i += blockDim.x) {
      if (a.steps) a.steps[e0 + i] = sSteps[i];
      if (a.episode) a.episode[e0 + i] = sEp[i];
    }
  __syncthreads();
#ifdef BRAX_DIAG
  if (dgb) tl[3] = gtime();
  if (a.diag_block && int(blockIdx.x) == a.diag_block - 1 && tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    for (int w = 0; w < int(blockDim.x >> 5); ++w)
      printf("LEAN sm %u warp %d: p1 %lld wait %lld p2 %lld (from substep start: p1 end %lld, p2 end %lld)\n", smid, w,
             sDg[w][1] - sDg[w][0], sDg[w][2] - sDg[w][1], sDg[w][3] - sDg[w][2], sDg[w][1] - sDg[0][0],
             sDg[w][3] - sDg[0][0]);
  }
#endif
  // S9: status bits, contact counts, and the single write-back of the QP (TMA bulk for full blocks)
  block_extras<V>(a, sQ, sCnt, sStat, B, C, E, LG, e0, nvalid);
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
      if (ka.reg) tma_store_commit_wait_all();  // written, not just read: a later launch may run now
      else tma_store_commit_wait();
#ifdef BRAX_DIAG
      if (dgb) tl[4] = gtime();
#endif
    }
  } else {
    store_block<V>(a, sQ, B, E, e0, nvalid);
  }
  if (a.status) {
    __syncthreads();
    for (int i = tid; i < nvalid; i += blockDim.x) a.status[e0 + i] = sStat[i];
  }
  if (ka.reg) {  // this launch is done with its granules: release them to the next launch
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async_global();
      __threadfence();
      for (int k = 0; k < ng; ++k) atomicAdd(ka.gd + g0 + k, 1u);
    }
  }
#ifdef BRAX_DIAG  // block timeline of launch tag (diag_block - 1000) into g_diag_tl, no printf in the way
  if (dgb && tl[4] && a.diag_block >= 1000 && a.diag_block < 1000 + kDiagLaunches && blockIdx.x < kDiagBlocks) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    long long* r = g_diag_tl + (size_t(a.diag_block - 1000) * kDiagBlocks + blockIdx.x) * 8;
    for (int k = 0; k < 5; ++k) r[k] = tl[k];
    r[5] = smid;
    r[6] = ka.overlap;
    r[7] = gtime();
  }
#endif
}

template <class S, int G, int R, bool kEnv = false, int kItems = 1>
cudaError_t launch_lean_variant(const LeanArgs& ka, dim3 grid, dim3 block, size_t smem, cudaStream_t stream) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
#ifdef BRAX_DIAG
    const int max_dyn = kMaxDynSmem - 1024;  // the diagnostics' static shared stamps
#else
    const int max_dyn = kMaxDynSmem;
#endif
    cudaError_t e =
        cudaFuncSetAttribute(brax_step_lean<S, G, R, kEnv, kItems>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
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
  return cudaLaunchKernelEx(&cfg, brax_step_lean<S, G, R, kEnv, kItems>, ka);
}

// ---- launch-order bookkeeping for overlapped launches (DESIGN.md §5 "Launch overlap") ----
// Per (device, stream): the window of lean launches that may still be in flight — every
// launch since the last one that waited for its predecessor in full (griddepcontrol.wait).
// A launch may skip that wait only if the stream's last kernel is the window's last member,
// it belongs to the same system and batch size, and every buffer it touches is, for every
// window member, either disjoint from that member's buffers or the same array of the same
// field (env i <-> env i): then the per-granule counters order every dependency, and a
// later full-waiting launch that waits for the window's last member waits, transitively
// through the granule counters, for all of them.  Kernels of other code on the stream do
// not trigger their dependents early, so they serialise as usual; this library's other
// kernels reset the window (note_other_launch).
struct Span {
  uintptr_t lo, hi;
  int kind;
  bool operator==(const Span& o) const { return lo == o.lo && hi == o.hi && kind == o.kind; }
};
struct LaunchRecord {
  std::vector<Span> reads, writes;
  bool operator==(const LaunchRecord& o) const { return reads == o.reads && writes == o.writes; }
};
struct StreamWindow {
  const System* sys = nullptr;
  int64_t n = -1;
  bool valid = false;               // the stream's last kernel is the window's last member
  std::vector<LaunchRecord> members;  // distinct buffer sets of the launches in the window
};
constexpr size_t kMaxWindow = 64;
std::recursive_mutex g_track_mu;  // held across each launch: recorded order = stream order
// keyed by (device, stream, capture sequence id or 0): a stream capture tracks its own
// launch order (its first node has no in-graph predecessor; the graph launch serialises
// with the stream's earlier work) and leaves the stream's eager record alone
using TrackKey = std::tuple<int, cudaStream_t, unsigned long long>;
std::map<TrackKey, StreamWindow> g_track;

TrackKey track_key(cudaStream_t stream) {
  int d = 0;
  cudaGetDevice(&d);
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(stream, &st, &id) != cudaSuccess) {
    cudaGetLastError();
    id = 0;
  }
  const TrackKey key{d, stream, st == cudaStreamCaptureStatusActive ? id : 0ull};
  if (std::get<2>(key) != 0 && g_track.size() > 1024 && !g_track.count(key))
    for (auto it = g_track.begin(); it != g_track.end();)  // finished captures' windows
      it = std::get<2>(it->first) != 0 ? g_track.erase(it) : std::next(it);
  return key;
}

void spans_of(const System& sys, const StepArgs& a, std::vector<Span>& rd, std::vector<Span>& wr) {
  const int64_t n = a.n_envs, B = sys.hd.B, T = a.n_steps > 0 ? a.n_steps : 1;
  auto add = [](std::vector<Span>& v, const void* p, int64_t bytes, int kind) {
    if (p && bytes > 0) v.push_back({reinterpret_cast<uintptr_t>(p), reinterpret_cast<uintptr_t>(p) + uintptr_t(bytes), kind});
  };
  const int w[4] = {3, 4, 3, 3};
  const void* in[4] = {a.pos_in, a.rot_in, a.vel_in, a.ang_in};
  const void* out[4] = {a.pos_out, a.rot_out, a.vel_out, a.ang_out};
  for (int f = 0; f < 4; ++f) {
    add(rd, in[f], n * B * w[f] * 4, f);
    add(wr, out[f], n * B * w[f] * 4, f);
  }
  add(rd, a.actions, T * n * sys.hd.A * 4, 4);
  add(wr, a.status, n * 4, 5);
  add(wr, a.contact_active, n * sys.hd.C, 6);
  add(wr, a.contact_dp, n * B * 6 * 4, 12);
  if (a.env) {
    add(rd, a.steps, n * 4, 7);
    add(wr, a.steps, n * 4, 7);
    add(rd, a.episode, n * 4, 8);
    add(wr, a.episode, n * 4, 8);
    add(wr, a.obs, T * n * sys.hd.task.obs_dim * 4, 9);
    add(wr, a.reward, T * n * 4, 10);
    add(wr, a.done, T * n, 11);
  }
}

bool compatible(const LaunchRecord& cur, const LaunchRecord& prev) {
  auto ok = [](const Span& x, const Span& y) {
    return x.hi <= y.lo || y.hi <= x.lo || (x.lo == y.lo && x.hi == y.hi && x.kind == y.kind);
  };
  for (const Span& y : prev.writes) {
    for (const Span& x : cur.reads)
      if (!ok(x, y)) return false;
    for (const Span& x : cur.writes)
      if (!ok(x, y)) return false;
  }
  for (const Span& y : prev.reads)
    for (const Span& x : cur.writes)
      if (!ok(x, y)) return false;
  return true;
}

}  // namespace

std::unique_lock<std::recursive_mutex> launch_order_lock() { return std::unique_lock<std::recursive_mutex>(g_track_mu); }

OverlapDecision overlap_decide(const System& sys, const StepArgs& a, cudaStream_t stream, bool participant) {
  std::lock_guard<std::recursive_mutex> g(g_track_mu);
  OverlapDecision d;
  d.reg = participant && sys.d_gran != nullptr && a.n_envs <= int64_t(kMaxGranules) * kGranule;
  if (!d.reg || std::getenv("BRAX_NO_OVERLAP")) return d;
  const StreamWindow& w = g_track[track_key(stream)];
  if (!w.valid || w.sys != &sys || w.n != a.n_envs) return d;
  LaunchRecord cur;
  spans_of(sys, a, cur.reads, cur.writes);
  bool known = false;
  for (const LaunchRecord& m : w.members) {
    if (!compatible(cur, m)) return d;
    known = known || cur == m;
  }
  if (!known && w.members.size() >= kMaxWindow) return d;  // start a new window
  d.overlap = true;
  return d;
}

void overlap_commit(const System& sys, const StepArgs& a, cudaStream_t stream, const OverlapDecision& d,
                    cudaError_t launched) {
  std::lock_guard<std::recursive_mutex> g(g_track_mu);
  StreamWindow& w = g_track[track_key(stream)];
  if (launched != cudaSuccess || !d.reg) {  // nothing to order by counters: the next launch waits in full
    w = StreamWindow{};
    return;
  }
  LaunchRecord cur;
  spans_of(sys, a, cur.reads, cur.writes);
  if (d.overlap) {
    for (const LaunchRecord& m : w.members)
      if (cur == m) return;
    w.members.push_back(std::move(cur));
    return;
  }
  w = StreamWindow{};  // this launch waited in full: it opens the window
  w.sys = &sys;
  w.n = a.n_envs;
  w.valid = true;
  w.members.push_back(std::move(cur));
}

void note_other_launch(const System&, cudaStream_t stream) {
  std::lock_guard<std::recursive_mutex> g(g_track_mu);
  g_track[track_key(stream)] = StreamWindow{};
}

void forget_system(const System* sys) {
  std::lock_guard<std::recursive_mutex> g(g_track_mu);
  for (auto it = g_track.begin(); it != g_track.end();)
    it = it->second.sys == sys ? g_track.erase(it) : std::next(it);
}

bool lean_applies(const System& sys, int plan, const StepArgs& a) {
  const DPlan& P = sys.hd.plan[plan];
  if (P.V != 2 && P.G == 1) return false;  // one env per lane: the lane-group plans only
  if ((a.env && a.n_steps == 0) || a.contact_dp || sys.trace || a.dpos_out) return false;  // observe-only: generic
  if (a.env && P.G == 1) return false;  // env instantiations: the lane-group plans
  const int items = sys.lean_items[plan];
  if (items == 0 || (items == 2 && (a.env || P.G != 1 || P.V != 2))) return false;  // kItems = 2: G = 1, F2, physics
  return (a.env ? P.smem_bytes_env : P.smem_bytes) <= kMaxDynSmem;
}

namespace {
cudaError_t dispatch_lean(const LeanArgs& ka, const DPlan& P, bool env, int items, int regs, dim3 grid, dim3 block,
                          size_t smem, cudaStream_t stream) {
  if (env) {  // env-epilogue instantiations (register budgets 128 / 96)
    if (P.V == 2) {
      if (P.G == 2) {
        if (regs >= 128) return launch_lean_variant<F2, 2, 128, true>(ka, grid, block, smem, stream);
        return launch_lean_variant<F2, 2, 96, true>(ka, grid, block, smem, stream);
      }
      if (regs >= 128) return launch_lean_variant<F2, 4, 128, true>(ka, grid, block, smem, stream);
      return launch_lean_variant<F2, 4, 96, true>(ka, grid, block, smem, stream);
    }
    if (P.G == 2) {
      if (regs >= 128) return launch_lean_variant<F1, 2, 128, true>(ka, grid, block, smem, stream);
      return launch_lean_variant<F1, 2, 96, true>(ka, grid, block, smem, stream);
    }
    if (regs >= 128) return launch_lean_variant<F1, 4, 128, true>(ka, grid, block, smem, stream);
    return launch_lean_variant<F1, 4, 96, true>(ka, grid, block, smem, stream);
  }
  // register budgets: the largest instantiation not above `regs` (F2 128 / 96 / 80; F1 128 / 96 / 64)
  if (P.V == 2) {
    if (P.G == 1 && items == 2) {
      if (regs >= 128) return launch_lean_variant<F2, 1, 128, false, 2>(ka, grid, block, smem, stream);
      if (regs >= 96) return launch_lean_variant<F2, 1, 96, false, 2>(ka, grid, block, smem, stream);
      return launch_lean_variant<F2, 1, 80, false, 2>(ka, grid, block, smem, stream);
    }
    if (P.G == 1) {
      if (regs >= 128) return launch_lean_variant<F2, 1, 128>(ka, grid, block, smem, stream);
      if (regs >= 96) return launch_lean_variant<F2, 1, 96>(ka, grid, block, smem, stream);
      return launch_lean_variant<F2, 1, 80>(ka, grid, block, smem, stream);
    }
    if (P.G == 2) {
      if (regs >= 128) return launch_lean_variant<F2, 2, 128>(ka, grid, block, smem, stream);
      if (regs >= 96) return launch_lean_variant<F2, 2, 96>(ka, grid, block, smem, stream);
      return launch_lean_variant<F2, 2, 80>(ka, grid, block, smem, stream);
    }
    if (regs >= 128) return launch_lean_variant<F2, 4, 128>(ka, grid, block, smem, stream);
    if (regs >= 96) return launch_lean_variant<F2, 4, 96>(ka, grid, block, smem, stream);
    return launch_lean_variant<F2, 4, 80>(ka, grid, block, smem, stream);
  }
  if (P.G == 2) {
    if (regs >= 128) return launch_lean_variant<F1, 2, 128>(ka, grid, block, smem, stream);
    if (regs >= 96) return launch_lean_variant<F1, 2, 96>(ka, grid, block, smem, stream);
    return launch_lean_variant<F1, 2, 64>(ka, grid, block, smem, stream);
  }
  if (regs >= 128) return launch_lean_variant<F1, 4, 128>(ka, grid, block, smem, stream);
  if (regs >= 96) return launch_lean_variant<F1, 4, 96>(ka, grid, block, smem, stream);
  return launch_lean_variant<F1, 4, 64>(ka, grid, block, smem, stream);
}
}  // namespace

cudaError_t launch_lean(const System& sys, const StepArgs& a, int plan, int regs, cudaStream_t stream) {
  const DPlan& P = sys.hd.plan[plan];
  const DHeader& H = sys.hd;
  LeanArgs ka{a, sys.d_blob, sys.hd, plan, {}};
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  ka.a.bulk_ok = al16(a.pos_in) && al16(a.rot_in) && al16(a.vel_in) && al16(a.ang_in) && al16(a.pos_out) &&
                 al16(a.rot_out) && al16(a.vel_out) && al16(a.ang_out);
  ka.a.act_bulk_ok = a.actions && al16(a.actions) && ((a.n_envs * H.A) % 4 == 0);
  if (std::getenv("BRAX_NO_BULK")) ka.a.bulk_ok = ka.a.act_bulk_ok = 0;
  if (const char* e = std::getenv("BRAX_DIAG_BLOCK")) ka.a.diag_block = std::atoi(e);
  ka.L = smem_layout(H.B, H.J, H.C, H.A, P.E, 32 / P.G, P.V == 2 ? 1 : 0, H.blob_words,
                     a.env ? H.task.obs_dim : 0, a.env ? H.task.contact_obs : 0, 0);
  dim3 grid(unsigned((a.n_envs + P.E - 1) / P.E)), block(unsigned(P.W * 32));
  const size_t smem = size_t(a.env ? P.smem_bytes_env : P.smem_bytes);
  // granule registration and launch overlap (DESIGN.md §5 "Launch overlap"); the record and
  // the launch happen under one lock, so the recorded order is the stream order
  auto order = launch_order_lock();
  const OverlapDecision d = overlap_decide(sys, a, stream, true);
  ka.gs = sys.d_gran;
  ka.gd = sys.d_gran + kMaxGranules;
  ka.reg = d.reg ? 1 : 0;
  ka.overlap = d.overlap ? 1 : 0;
  const cudaError_t e = dispatch_lean(ka, P, a.env != 0, sys.lean_items[plan], regs, grid, block, smem, stream);
  overlap_commit(sys, a, stream, d, e);
  return e;
}

}  // namespace brax

#ifdef BRAX_DIAG
extern "C" int brax_diag_timeline(long long* out, long long n) {  // diagnostic builds only
  const long long total = (long long)brax::kDiagLaunches * brax::kDiagBlocks * 8;
  return cudaMemcpyFromSymbol(out, brax::g_diag_tl, size_t(n < total ? n : total) * sizeof(long long)) == cudaSuccess
             ? 0 : 1;
}
#endif
