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

#include <cstdio>
#include <cstdlib>

#include "step_device.cuh"
#include "system.h"

namespace brax {
namespace {

using namespace dev;

struct KArgs {
  StepArgs a;
  const uint32_t* blob;
  DHeader hd;
  int32_t plan;  // index into hd.plan (G = 1 << plan lane groups per warp)
};

// Register budget: 80 per thread keeps 2 blocks of up to 12 warps resident per SM.
// S = float: one env per lane; F2: two envs per lane.  R: register budget per
// thread (instantiated for several budgets; launch_step picks the largest that
// keeps two blocks resident per SM).
template <class S, int R>
__global__ void __maxnreg__(R) brax_step_kernel(const __grid_constant__ KArgs ka) {
  extern __shared__ __align__(16) uint32_t smem[];
  const DHeader& H = ka.hd;
  const DPlan& P = H.plan[ka.plan];
  const StepArgs& a = ka.a;
  const int B = H.B, J = H.J, C = H.C, A = H.A, E = P.E, G = P.G;
  const SmemLayout L = smem_layout(B, J, C, A, E, H.blob_words);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // [0] tables + QP, [1] actions
  uint32_t* sBlob = smem + L.blob;
  float* sQ = reinterpret_cast<float*>(smem + L.q);
  float* sJ = reinterpret_cast<float*>(smem + L.u);
  float* sC = sJ + J * E * kJS;
  float* stg = reinterpret_cast<float*>(smem + L.u);  // aliases sJ/sC outside the substeps
  float* sA = reinterpret_cast<float*>(smem + L.a);
  float* sAstg = reinterpret_cast<float*>(smem + L.astg);
  float* sCnt = reinterpret_cast<float*>(smem + L.cnt);
  uint32_t* sStat = smem + L.stat;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tracing (brax_system_phase_cycles): thread 0 times prologue / joints+contacts /
  // integrate / epilogue with clock64 (uniform branch; off unless requested)
  const bool trace = a.phase_cycles != nullptr && tid == 0;
  long long tr_mark = trace ? clock64() : 0, tr[4] = {0, 0, 0, 0};
  auto lap = [&](int k) {
    if (trace) {
      long long t = clock64();
      tr[k] += t - tr_mark;
      tr_mark = t;
    }
  };
  const int LG = 32 / G;                                 // lanes per group
  const int grp = lane / LG, el = lane - grp * LG;       // lane group; first env slot of this lane
  const int o2q = LG * kQS, o2j = LG * kJS, o2c = LG * kCS;  // second env (S = F2): + LG slots
  const int64_t e0 = int64_t(blockIdx.x) * E;
  const int nvalid = (a.n_envs - e0 < E) ? int(a.n_envs - e0) : E;
  const bool bulk = a.bulk_ok && nvalid == E;          // block-uniform
  const bool act_bulk = bulk && a.act_bulk_ok && A > 0;
  const uint32_t qp_bytes = uint32_t(E * B) * 13u * 4u, act_bytes = uint32_t(E * A) * 4u;

  // S1: tables and (full blocks) the four contiguous QP chunks arrive by TMA bulk copies
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&bars[0], uint32_t(H.blob_words) * 4u + (bulk ? qp_bytes : 0u));
    tma_load(sBlob, ka.blob, uint32_t(H.blob_words) * 4u, &bars[0]);
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
  if (!bulk) load_block(a, sQ, sStat, B, E, e0, nvalid);  // ragged tail / unaligned: per-row loads
  mbar_wait(&bars[0], 0);
  if (bulk) stg_to_records(stg, sQ, B, E, E);
  for (int i = tid; i < E; i += blockDim.x) sStat[i] = 0u;
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
  const float* sJe = sJ + el * kJS;  // this env's record of joint 0 (joint j: + j*E*kJS)
  const float* sCe = sC + el * kCS;
  const int it0 = item_begin[warp], it1 = item_begin[warp + 1];
  const int bw0 = body_begin[warp], bw1 = body_begin[warp + 1];

  // S2 of the first substep; every later S2 is fused into the previous substep's integrate()
  for (int i = bw0; i < bw1; ++i) {
    int b = bodies_of_warp[i * G];
    if (b >= 0) kinematic<S>(bodies[b], Row<S>{sQ + (b * E + el) * kQS, o2q}, H.h);
  }
  for (int64_t step = 0; step < a.n_steps; ++step) {
    if (act_bulk) {  // this step's actions arrived in sAstg [E][A]; transpose to sA [A][E]
      mbar_wait(&bars[1], uint32_t(step & 1));
      for (int i = tid; i < E * A; i += blockDim.x) {
        const int env = i / A, k = i - env * A;
        sA[k * E + env] = sAstg[i];
      }
    } else {
      load_actions(a, sA, A, E, step, e0, nvalid);
    }  // sA is read in phase 2, after a barrier
    for (int it = it0; it < it1; ++it) {
      int item = items[it * G];
      if (item >= J) {
        sCnt[(item - J) * E + el] = 0.f;
        if (LG != E) sCnt[(item - J) * E + el + LG] = 0.f;
      }
    }
    for (int s = 0; s < H.S; ++s) {
      __syncthreads();
      lap(2);
      if (act_bulk && s == 0 && tid == 0 && step + 1 < a.n_steps) {  // prefetch next step's actions
        mbar_expect_tx(&bars[1], act_bytes);
        tma_load(sAstg, a.actions + ((step + 1) * a.n_envs + e0) * A, act_bytes, &bars[1]);
      }
      for (int it = it0; it < it1; ++it) {
        int item = items[it * G];
        if (item < 0) continue;
        if (item < J) {
          const DJoint& jt = joints[item];
          joint<S>(jt, Row<S>{sQ + (jt.parent * E + el) * kQS, o2q}, Row<S>{sQ + (jt.child * E + el) * kQS, o2q},
                   sA + el, E, LG, sJ + (item * E + el) * kJS, o2j);
        } else {
          int c = item - J;
          const DSlot& sl = slots[c];
          float* cp = sCnt + c * E + el;
          S cnt = Lanes<S>::ld(cp, LG);
          contact<S>(sl, Row<S>{sQ + (sl.a * E + el) * kQS, o2q}, Row<S>{sQ + (sl.b * E + el) * kQS, o2q},
                     1.f + H.e, H.beta_over_h, H.mu, sC + (c * E + el) * kCS, o2c, cnt);
          store_count(cp, LG, cnt);
        }
      }
      __syncthreads();
      lap(1);
      for (int i = bw0; i < bw1; ++i) {
        int b = bodies_of_warp[i * G];
        if (b < 0) continue;
        Acc<S> acc;
#pragma unroll 4
        for (int k = jinc_begin[b]; k < jinc_begin[b + 1]; ++k) {
          int e = jinc[k];
          acc.joint(sJe + (e >> 4) * (E * kJS), o2j, e);
        }
#pragma unroll 4
        for (int k = cinc_begin[b]; k < cinc_begin[b + 1]; ++k) {
          int e = cinc[k];
          acc.slot(sCe + (e >> 4) * (E * kCS), o2c, e);
        }
        const bool kin = !(step + 1 == a.n_steps && s + 1 == H.S);  // fused S2 of the next substep
        integrate<S>(bodies[b], Row<S>{sQ + (b * E + el) * kQS, o2q}, acc, H.h, H.g, kin);
      }
    }
  }
  lap(2);
  __syncthreads();
  // S9: status bits, contact counts, and the single write-back of the QP (TMA bulk for full blocks)
  block_extras(a, sQ, sCnt, sStat, B, C, E, e0, nvalid);
  if (bulk) {
    records_to_stg(sQ, stg, B, E, E);
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
      tma_store_commit_wait();
    }
  } else {
    store_block(a, sQ, B, E, e0, nvalid);
  }
  if (a.status) {
    __syncthreads();
    for (int i = tid; i < nvalid; i += blockDim.x) a.status[e0 + i] = sStat[i];
  }
  if (trace) {
    lap(3);
    for (int k = 0; k < 4; ++k) atomicAdd(&a.phase_cycles[k], (unsigned long long)tr[k]);
  }
}

}  // namespace

// Lane-group plan for a launch: more, smaller blocks (G = 2, 4) when the batch
// alone would leave the SMs with few independent env groups to overlap their
// per-substep barriers; G = 1 once the grid fills the GPU.
int choose_plan(const System& sys, int64_t n_envs) {
  if (const char* e = std::getenv("BRAX_PLAN")) {  // "G,V" override (experiments)
    int g = 0, v = 0;
    if (std::sscanf(e, "%d,%d", &g, &v) == 2)
      for (int i = 0; i < kNumPlans; ++i)
        if (sys.hd.plan[i].G == g && sys.hd.plan[i].V == v) return i;
  }
  int sms = sys.num_sms > 0 ? sys.num_sms : 148;
  int64_t blocks32 = (n_envs + 31) / 32;
  // measured (profiles/): lane groups help only while the smaller blocks still
  // fit one per SM (the batch is too small to fill the GPU with 32-env blocks)
  if (4 * blocks32 <= sms) return 2;
  if (2 * blocks32 <= sms) return 1;
  if (blocks32 >= 4 * sms) return 3;  // large batches: two envs per lane (G = 1, V = 2)
  return 0;
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
template <class S, int R>
cudaError_t launch_variant(const KArgs& ka, dim3 grid, dim3 block, size_t smem, cudaStream_t stream) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !attr_set[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(brax_step_kernel<S, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  brax_step_kernel<S, R><<<grid, block, smem, stream>>>(ka);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_step(const System& sys, const StepArgs& a, cudaStream_t stream) {
  if (a.n_envs <= 0 || a.n_steps <= 0) return cudaSuccess;
  KArgs ka{a, sys.d_blob, sys.hd, choose_plan(sys, a.n_envs)};
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  ka.a.bulk_ok = al16(a.pos_in) && al16(a.rot_in) && al16(a.vel_in) && al16(a.ang_in) && al16(a.pos_out) &&
                 al16(a.rot_out) && al16(a.vel_out) && al16(a.ang_out);
  ka.a.act_bulk_ok = a.actions && al16(a.actions) && ((a.n_envs * sys.hd.A) % 4 == 0);
  if (std::getenv("BRAX_NO_BULK")) ka.a.bulk_ok = ka.a.act_bulk_ok = 0;
  ka.a.phase_cycles = sys.trace ? sys.d_phase_cycles : nullptr;
  const DPlan& P = sys.hd.plan[ka.plan];
  dim3 grid(unsigned((a.n_envs + P.E - 1) / P.E)), block(unsigned(P.W * 32));
  const size_t smem = size_t(P.smem_bytes);
  const int regs = choose_regs(sys, P, int64_t(grid.x));
  if (P.V == 2) {
    if (regs >= 128) return launch_variant<F2, 128>(ka, grid, block, smem, stream);
    if (regs >= 96) return launch_variant<F2, 96>(ka, grid, block, smem, stream);
    return launch_variant<F2, 80>(ka, grid, block, smem, stream);
  }
  if (regs >= 128) return launch_variant<float, 128>(ka, grid, block, smem, stream);
  if (regs >= 112) return launch_variant<float, 112>(ka, grid, block, smem, stream);
  if (regs >= 96) return launch_variant<float, 96>(ka, grid, block, smem, stream);
  if (regs >= 80) return launch_variant<float, 80>(ka, grid, block, smem, stream);
  if (regs >= 64) return launch_variant<float, 64>(ka, grid, block, smem, stream);
  return launch_variant<float, 56>(ka, grid, block, smem, stream);
}

}  // namespace brax
