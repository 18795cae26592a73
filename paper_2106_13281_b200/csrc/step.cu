// step.cu — the batched Brax physics step for sm_100a.
//
// Computes Alg. 1 of the paper `substeps` times per step for
// n independent envs, with the formulas of SURVEY.md §8(c).1 (DESIGN.md
// "Readings").  Mapping:
//   * one block = 32 envs; lane = env; warp = work item (a body, a joint, a
//     contact slot).  All lanes of a warp run the same item of the same scene,
//     so control flow and static parameters are warp-uniform; the only
//     divergence is whether a contact is active in a given env.
//   * each env's QP is read from HBM once (coalesced, float4), kept in shared
//     memory as [body][field][lane] for all substeps (and, for brax_rollout,
//     all steps), and written back once.
//   * per-body sums are gathers over static incidence lists in a fixed order
//     (joints by index, then contact slots by index): no atomics.
//   * per substep: phase 1 kinematic integrator (body warps) | barrier |
//     phase 2 joints+actuators and contacts (item warps) | barrier |
//     phase 3 gather + potential + collision integrators (body warps).
// fp32 throughout, IEEE div/sqrt (R28).  No tensor cores: nothing here is a
// dense contraction.
#include <cuda_runtime.h>
#include <stdint.h>

#include "system.h"

namespace brax {
namespace {

struct V3 { float x, y, z; };
struct Q4 { float w, x, y, z; };

__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 operator*(float s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ V3 had(V3 a, V3 b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
__device__ __forceinline__ float dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ Q4 qmul(Q4 a, Q4 b) {
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x, a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
__device__ __forceinline__ Q4 qconj(Q4 q) { return {q.w, -q.x, -q.y, -q.z}; }
// rotate(q, v) = v + w·t + u×t, t = 2u×v
__device__ __forceinline__ V3 rotate(Q4 q, V3 v) {
  V3 u{q.x, q.y, q.z};
  V3 t = 2.f * cross(u, v);
  return v + q.w * t + cross(u, t);
}
// I_w⁻¹(q)·v = rotate(q, inv_rotate(q, v) ⊙ I_b⁻¹)   (R4)
__device__ __forceinline__ V3 iw(Q4 q, V3 inv_i, V3 v) { return rotate(q, had(rotate(qconj(q), v), inv_i)); }
__device__ __forceinline__ V3 v3(const float* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ Q4 q4(const float* p) { return {p[0], p[1], p[2], p[3]}; }
__device__ __forceinline__ float clampf(float x, float lo, float hi) { return fminf(fmaxf(x, lo), hi); }

// shared-memory QP: [body][field][lane]
struct Row {
  float* p;  // = sQ + b*13*32 + lane
  __device__ __forceinline__ V3 ld3(int f) const { return {p[f * 32], p[(f + 1) * 32], p[(f + 2) * 32]}; }
  __device__ __forceinline__ Q4 ldq() const { return {p[3 * 32], p[4 * 32], p[5 * 32], p[6 * 32]}; }
  __device__ __forceinline__ void st3(int f, V3 v) const { p[f * 32] = v.x; p[(f + 1) * 32] = v.y; p[(f + 2) * 32] = v.z; }
  __device__ __forceinline__ void stq(Q4 q) const { p[3 * 32] = q.w; p[4 * 32] = q.x; p[5 * 32] = q.y; p[6 * 32] = q.z; }
};

struct Tables {
  const DBody* bodies;
  const DJoint* joints;
  const DSlot* slots;
  const int32_t* item_begin;
  const int32_t* items;
  const int32_t* body_begin;
  const int32_t* bodies_of_warp;
  const int32_t* inc_begin;
  const int32_t* inc;
};

// ---- S2: kinematic integrator (R3, R21) -------------------------
__device__ __forceinline__ void kinematic(const DBody& bd, Row r, float h) {
  V3 x = r.ld3(0), v = r.ld3(7);
  r.st3(0, x + h * had(v3(bd.mpos), v));
  if (!bd.rot_frozen) {
    V3 w = had(v3(bd.mrot), r.ld3(10));
    Q4 q = r.ldq();
    Q4 dq = qmul(Q4{0.f, w.x, w.y, w.z}, q);
    float hh = 0.5f * h;
    q = Q4{q.w + hh * dq.w, q.x + hh * dq.x, q.y + hh * dq.y, q.z + hh * dq.z};
    float inv = 1.f / sqrtf(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
    r.stq(Q4{q.w * inv, q.x * inv, q.y * inv, q.z * inv});
  }
}

// ---- S3 + S4: joint spring/limits with its actuator (R5, R7-R12)
__device__ __forceinline__ void joint(const DJoint& J, Row P, Row C, const float* act, float* out) {
  Q4 qp = P.ldq(), qc = C.ldq();
  V3 xp = P.ld3(0), xc = C.ld3(0);
  V3 rp = rotate(qp, v3(J.o_p)), rc = rotate(qc, v3(J.o_c));
  V3 dx = (xp - xc) + (rp - rc);
  V3 wp = P.ld3(10), wc = C.ld3(10);
  V3 dv = (P.ld3(7) + cross(wp, rp)) - (C.ld3(7) + cross(wc, rc));
  V3 f = J.k * dx + J.c_l * dv;
  Q4 fp = qmul(qp, q4(J.jp)), fc = qmul(qc, q4(J.jc));
  Q4 qr = qmul(qconj(fp), fc);
  if (qr.w < 0.f) qr = Q4{-qr.w, -qr.x, -qr.y, -qr.z};
  float R02 = 2.f * (qr.x * qr.z + qr.w * qr.y);
  float R12 = 2.f * (qr.y * qr.z - qr.w * qr.x);
  float R22 = 1.f - 2.f * (qr.x * qr.x + qr.y * qr.y);
  float R01 = 2.f * (qr.x * qr.y - qr.w * qr.z);
  float R00 = 1.f - 2.f * (qr.y * qr.y + qr.z * qr.z);
  float th[3] = {atan2f(-R12, R22), asinf(clampf(R02, -1.f, 1.f)), atan2f(-R01, R00)};
  float tau[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (i < J.dof) {
      tau[i] = J.k_l * (clampf(th[i], J.lo[i], J.hi[i]) - th[i]);
      if (J.act_kind >= 0) {
        float a = act[(J.act_offset + i) * 32];
        tau[i] += (J.act_kind == 0) ? J.strength * clampf(a, -1.f, 1.f)
                                    : J.strength * (clampf(a, J.lo[i], J.hi[i]) - th[i]);
      }
    } else {
      tau[i] = -(J.k_a * th[i]);
    }
  }
  V3 twd = rotate(fp, V3{tau[0], tau[1], tau[2]}) + J.c_a * (wp - wc);
  V3 tc = twd + cross(rc, f);
  V3 tp = (-1.f) * (twd + cross(rp, f));
  out[0 * 32] = f.x; out[1 * 32] = f.y; out[2 * 32] = f.z;
  out[3 * 32] = tc.x; out[4 * 32] = tc.y; out[5 * 32] = tc.z;
  out[6 * 32] = tp.x; out[7 * 32] = tp.y; out[8 * 32] = tp.z;
}

// Closest points between segments (Ericson, Real-Time Collision Detection §5.1.9).
__device__ __forceinline__ void seg_seg(V3 p1, V3 q1, V3 p2, V3 q2, V3& c1, V3& c2) {
  V3 d1 = q1 - p1, d2 = q2 - p2, r = p1 - p2;
  float a = dot(d1, d1), e = dot(d2, d2), f = dot(d2, r);
  float s = 0.f, t = 0.f;
  if (a <= 0.f && e <= 0.f) {
  } else if (a <= 0.f) {
    t = clampf(f / e, 0.f, 1.f);
  } else {
    float c = dot(d1, r);
    if (e <= 0.f) {
      s = clampf(-c / a, 0.f, 1.f);
    } else {
      float b = dot(d1, d2);
      float denom = a * e - b * b;
      s = (denom == 0.f) ? 0.f : clampf((b * f - c * e) / denom, 0.f, 1.f);
      t = (b * s + f) / e;
      if (t < 0.f) {
        t = 0.f;
        s = clampf(-c / a, 0.f, 1.f);
      } else if (t > 1.f) {
        t = 1.f;
        s = clampf((b - c) / a, 0.f, 1.f);
      }
    }
  }
  c1 = p1 + s * d1;
  c2 = p2 + t * d2;
}

// ---- S5: contact slot, velocity-level impulse + Baumgarte (R13-R19)
__device__ __forceinline__ void contact(const DSlot& S, Row A, Row B, const DHeader& H, float* out, int* cnt) {
  Q4 qa = A.ldq(), qb = B.ldq();
  V3 xa = A.ld3(0), xb = B.ld3(0);
  V3 cA = xa + rotate(qa, v3(S.ca_pos));
  V3 cB = xb + rotate(qb, v3(S.cb_pos));
  Q4 qA = qmul(qa, q4(S.ca_rot)), qB = qmul(qb, q4(S.cb_rot));
  const V3 zhat{0.f, 0.f, 1.f};
  V3 n, pt;
  float d;
  if (S.type <= 2) {  // sphere / capsule end / box corner vs plane: plane is B
    n = rotate(qB, zhat);
    V3 c;
    float r;
    if (S.type == 2) {
      V3 sg{(S.point & 1) ? S.hs[0] : -S.hs[0], (S.point & 2) ? S.hs[1] : -S.hs[1],
            (S.point & 4) ? S.hs[2] : -S.hs[2]};
      c = cA + rotate(qA, sg);
      r = 0.f;
    } else {
      c = cA;
      if (S.type == 1) {
        V3 ax = rotate(qA, zhat);
        c = (S.point == 0) ? cA + S.ella * ax : cA - S.ella * ax;
      }
      r = S.ra;
    }
    if (S.type == 2) {
      d = -dot(c - cB, n);
      pt = c;
    } else {
      d = r - dot(c - cB, n);
      pt = c - r * n;
    }
  } else {
    V3 pa = cA, pb = cB;
    if (S.type == 4) {  // sphere (A) – capsule (B)
      V3 axb = rotate(qB, zhat);
      V3 e0 = cB + S.ellb * axb, e1 = cB - S.ellb * axb;
      V3 seg = e0 - e1;
      float L2 = dot(seg, seg);
      float t = (L2 > 0.f) ? clampf(dot(cA - e1, seg) / L2, 0.f, 1.f) : 0.f;
      pb = e1 + t * seg;
    } else if (S.type == 5) {  // capsule – capsule
      V3 axa = rotate(qA, zhat), axb = rotate(qB, zhat);
      seg_seg(cA + S.ella * axa, cA - S.ella * axa, cB + S.ellb * axb, cB - S.ellb * axb, pa, pb);
    }
    V3 delta = pa - pb;
    float dist = sqrtf(dot(delta, delta));
    n = (dist > 0.f) ? (1.f / dist) * delta : zhat;
    d = S.ra + S.rb - dist;
    pt = 0.5f * ((pa - S.ra * n) + (pb + S.rb * n));
  }
  bool active = false;
  V3 P{0.f, 0.f, 0.f}, ta{0.f, 0.f, 0.f}, tb{0.f, 0.f, 0.f};
  if (d > 0.f) {
    V3 rA = pt - xa, rB = pt - xb;
    V3 ia = v3(S.inv_inertia_a), ib = v3(S.inv_inertia_b);
    V3 u = (A.ld3(7) + cross(A.ld3(10), rA)) - (B.ld3(7) + cross(B.ld3(10), rB));
    float un = dot(u, n);
    auto eff = [&](V3 dir) {
      float k = 0.f;
      if (!S.a_static) {
        V3 rn = cross(rA, dir);
        k = k + S.inv_mass_a + dot(rn, iw(qa, ia, rn));
      }
      if (!S.b_static) {
        V3 rn = cross(rB, dir);
        k = k + S.inv_mass_b + dot(rn, iw(qb, ib, rn));
      }
      return k;
    };
    float kn = eff(n);
    float jn = fmaxf(0.f, (-(1.f + H.e) * un + H.beta_over_h * d) / kn);
    if (jn > 0.f) {
      active = true;
      V3 ut = u - un * n;
      float st = sqrtf(dot(ut, ut));
      P = jn * n;
      if (st > 0.f) {
        V3 th = (1.f / st) * ut;
        float jt = fminf(st / eff(th), H.mu * jn);
        P = P - jt * th;
      }
      ta = cross(rA, P);
      tb = cross(rB, P);
    }
  }
  out[0 * 32] = P.x; out[1 * 32] = P.y; out[2 * 32] = P.z;
  out[3 * 32] = ta.x; out[4 * 32] = ta.y; out[5 * 32] = ta.z;
  out[6 * 32] = tb.x; out[7 * 32] = tb.y; out[8 * 32] = tb.z;
  out[9 * 32] = active ? 1.f : 0.f;
  *cnt += active ? 1 : 0;
}

// ---- S6 + S7 + S8: gather, potential integrator, collision integrator
// sJ, sC: this lane's column of the joint / slot outputs.
__device__ __forceinline__ void integrate(const DBody& bd, Row r, const Tables& T, int b, const float* sJ,
                                          const float* sC, const DHeader& H) {
  V3 F{0.f, 0.f, 0.f}, Tq{0.f, 0.f, 0.f}, dV{0.f, 0.f, 0.f}, dW{0.f, 0.f, 0.f};
  float cnt = 0.f;
  const int i0 = T.inc_begin[b], i1 = T.inc_begin[b + 1];
  for (int i = i0; i < i1; ++i) {
    int e = T.inc[i];
    int kind = e >> 16, ix = e & 0xffff;
    if (kind <= kIncJointParent) {
      const float* o = sJ + ix * kJointOut * 32;
      V3 f{o[0], o[32], o[64]};
      if (kind == kIncJointChild) {
        F = F + f;
        Tq = Tq + V3{o[96], o[128], o[160]};
      } else {
        F = F - f;
        Tq = Tq + V3{o[192], o[224], o[256]};
      }
    } else {
      const float* o = sC + ix * kSlotOut * 32;
      V3 p{o[0], o[32], o[64]};
      cnt += o[288];
      if (kind == kIncSlotA) {
        dV = dV + p;
        dW = dW + V3{o[96], o[128], o[160]};
      } else {
        dV = dV - p;
        dW = dW - V3{o[192], o[224], o[256]};
      }
    }
  }
  Q4 q = r.ldq();
  V3 mp = v3(bd.mpos), mr = v3(bd.mrot), ii = v3(bd.inv_inertia);
  V3 g{H.g[0], H.g[1], H.g[2]};
  V3 v = had(mp, r.ld3(7) + H.h * (bd.inv_mass * F + g));
  V3 w = had(mr, r.ld3(10) + H.h * iw(q, ii, Tq));
  if (cnt > 0.f) {
    float ic = 1.f / cnt;  // R14: mean over the body's active contacts
    v = had(mp, v + (bd.inv_mass * ic) * dV);
    w = had(mr, w + ic * iw(q, ii, dW));
  }
  r.st3(7, v);
  r.st3(10, w);
}

// Coalesced staging of one QP field [n][B][K] <-> sQ[b][f0 + k][lane].
template <int K, bool kLoad>
__device__ __forceinline__ void stage(const float* gin, float* gout, float* sQ, int f0, int64_t e0, int nvalid,
                                      int B, uint32_t magic) {
  const int row = B * K;
  const int count = nvalid * row;
  const float* src = gin + e0 * row;
  float* dst = gout + e0 * row;
  const int n4 = count >> 2;
  for (int i4 = threadIdx.x; i4 < n4; i4 += blockDim.x) {
    float vals[4];
    if (kLoad) {
      float4 v = __ldg(reinterpret_cast<const float4*>(src) + i4);
      vals[0] = v.x; vals[1] = v.y; vals[2] = v.z; vals[3] = v.w;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int i = 4 * i4 + c;
      int env = __umulhi(uint32_t(i), magic);
      int rem = i - env * row;
      int b = rem / K;
      int k = rem - b * K;
      float* s = sQ + (b * kQPFields + f0 + k) * 32 + env;
      if (kLoad) *s = vals[c]; else vals[c] = *s;
    }
    if (!kLoad) reinterpret_cast<float4*>(dst)[i4] = make_float4(vals[0], vals[1], vals[2], vals[3]);
  }
  for (int i = 4 * n4 + threadIdx.x; i < count; i += blockDim.x) {
    int env = __umulhi(uint32_t(i), magic);
    int rem = i - env * row;
    int b = rem / K;
    int k = rem - b * K;
    float* s = sQ + (b * kQPFields + f0 + k) * 32 + env;
    if (kLoad) *s = __ldg(src + i); else dst[i] = *s;
  }
}

struct KArgs {
  StepArgs a;
  const uint32_t* blob;
  DHeader hd;
};

__global__ void __launch_bounds__(kMaxWarps * 32) brax_step_kernel(const KArgs ka) {
  extern __shared__ __align__(16) uint32_t smem[];
  const DHeader& H = ka.hd;
  const StepArgs& a = ka.a;
  const int B = H.B, J = H.J, C = H.C, A = H.A;
  uint32_t* sBlob = smem;
  float* sQ = reinterpret_cast<float*>(smem + H.blob_words);
  float* sJ = sQ + B * kQPFields * 32;
  float* sC = sJ + J * kJointOut * 32;
  float* sA = sC + C * kSlotOut * 32;
  int* sCnt = reinterpret_cast<int*>(sA + A * 32);
  uint32_t* sStat = reinterpret_cast<uint32_t*>(sCnt + C * 32);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t e0 = int64_t(blockIdx.x) * 32;
  const int nvalid = (a.n_envs - e0 < 32) ? int(a.n_envs - e0) : 32;

  // stage the static tables (≈2-7 KB) and this block's 32 envs' QP
  {
    const uint4* src = reinterpret_cast<const uint4*>(ka.blob);
    uint4* dst = reinterpret_cast<uint4*>(sBlob);
    for (int i = tid; i < H.blob_words / 4; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  if (nvalid < 32) {  // identity state for lanes past the end of the batch
    for (int i = tid; i < B * kQPFields * 32; i += blockDim.x) {
      int f = (i >> 5) % kQPFields;
      sQ[i] = (f == 3) ? 1.f : 0.f;
    }
    __syncthreads();
  }
  stage<3, true>(a.pos_in, nullptr, sQ, 0, e0, nvalid, B, H.row_magic[0]);
  stage<4, true>(a.rot_in, nullptr, sQ, 3, e0, nvalid, B, H.row_magic[1]);
  stage<3, true>(a.vel_in, nullptr, sQ, 7, e0, nvalid, B, H.row_magic[0]);
  stage<3, true>(a.ang_in, nullptr, sQ, 10, e0, nvalid, B, H.row_magic[0]);
  if (tid < 32) sStat[tid] = 0u;
  __syncthreads();

  Tables T;
  T.bodies = reinterpret_cast<const DBody*>(sBlob + H.off_bodies);
  T.joints = reinterpret_cast<const DJoint*>(sBlob + H.off_joints);
  T.slots = reinterpret_cast<const DSlot*>(sBlob + H.off_slots);
  T.item_begin = reinterpret_cast<const int32_t*>(sBlob + H.off_item_begin);
  T.items = reinterpret_cast<const int32_t*>(sBlob + H.off_items);
  T.body_begin = reinterpret_cast<const int32_t*>(sBlob + H.off_body_begin);
  T.bodies_of_warp = reinterpret_cast<const int32_t*>(sBlob + H.off_bodies_of_warp);
  T.inc_begin = reinterpret_cast<const int32_t*>(sBlob + H.off_inc_begin);
  T.inc = reinterpret_cast<const int32_t*>(sBlob + H.off_inc);
  const int it0 = T.item_begin[warp], it1 = T.item_begin[warp + 1];
  const int bw0 = T.body_begin[warp], bw1 = T.body_begin[warp + 1];

  for (int64_t step = 0; step < a.n_steps; ++step) {
    // S1: this step's action, [n][A] -> sA[k][lane] (read in phase 2, after a barrier)
    if (A > 0) {
      const float* act = a.actions + (step * a.n_envs + e0) * A;
      for (int i = tid; i < nvalid * A; i += blockDim.x) {
        int env = (A == 1) ? i : int(__umulhi(uint32_t(i), H.row_magic[2]));  // magic(1) would overflow
        int k = i - env * A;
        sA[k * 32 + env] = __ldg(act + i);
      }
    }
    for (int it = it0; it < it1; ++it) {
      int item = T.items[it];
      if (item >= J) sCnt[(item - J) * 32 + lane] = 0;
    }
    for (int s = 0; s < H.S; ++s) {
      for (int i = bw0; i < bw1; ++i) {
        int b = T.bodies_of_warp[i];
        kinematic(T.bodies[b], Row{sQ + b * kQPFields * 32 + lane}, H.h);
      }
      __syncthreads();
      for (int it = it0; it < it1; ++it) {
        int item = T.items[it];
        if (item < J) {
          const DJoint& jt = T.joints[item];
          joint(jt, Row{sQ + jt.parent * kQPFields * 32 + lane}, Row{sQ + jt.child * kQPFields * 32 + lane},
                sA + lane, sJ + item * kJointOut * 32 + lane);
        } else {
          int c = item - J;
          const DSlot& sl = T.slots[c];
          contact(sl, Row{sQ + sl.a * kQPFields * 32 + lane}, Row{sQ + sl.b * kQPFields * 32 + lane}, H,
                  sC + c * kSlotOut * 32 + lane, sCnt + c * 32 + lane);
        }
      }
      __syncthreads();
      for (int i = bw0; i < bw1; ++i) {
        int b = T.bodies_of_warp[i];
        integrate(T.bodies[b], Row{sQ + b * kQPFields * 32 + lane}, T, b, sJ + lane, sC + lane, H);
      }
    }
  }
  __syncthreads();

  // S9: status bits, contact counts, and the single write-back of the QP
  if (a.status) {
    for (int i = tid; i < B * kQPFields * 32; i += blockDim.x) {
      float v = sQ[i];
      uint32_t bit = isfinite(v) ? (fabsf(v) > 1e6f ? 2u : 0u) : 1u;
      if (bit) atomicOr(&sStat[i & 31], bit);
    }
  }
  if (a.contact_active) {
    for (int i = tid; i < nvalid * C; i += blockDim.x) {
      int env = i / C, c = i - env * C;
      a.contact_active[(e0 + env) * C + c] = uint8_t(sCnt[c * 32 + env]);
    }
  }
  stage<3, false>(nullptr, a.pos_out, sQ, 0, e0, nvalid, B, H.row_magic[0]);
  stage<4, false>(nullptr, a.rot_out, sQ, 3, e0, nvalid, B, H.row_magic[1]);
  stage<3, false>(nullptr, a.vel_out, sQ, 7, e0, nvalid, B, H.row_magic[0]);
  stage<3, false>(nullptr, a.ang_out, sQ, 10, e0, nvalid, B, H.row_magic[0]);
  if (a.status) {
    __syncthreads();
    if (tid < nvalid) a.status[e0 + tid] = sStat[tid];
  }
}

}  // namespace

cudaError_t launch_step(const System& sys, const StepArgs& a, cudaStream_t stream) {
  if (a.n_envs <= 0 || a.n_steps <= 0) return cudaSuccess;
  static bool attr_set[64] = {};
  if (sys.device >= 0 && sys.device < 64 && !attr_set[sys.device]) {
    cudaError_t e = cudaFuncSetAttribute(brax_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set[sys.device] = true;
  }
  KArgs ka{a, sys.d_blob, sys.hd};
  dim3 grid(unsigned((a.n_envs + 31) / 32)), block(unsigned(sys.hd.W * 32));
  brax_step_kernel<<<grid, block, sys.smem_bytes, stream>>>(ka);
  return cudaGetLastError();
}

}  // namespace brax
