// step_device.cuh — device code of the batched Brax step (sm_100a).
//
// Formulas: Alg. 1 of the paper with SURVEY.md §8(c).1 /
// DESIGN.md "Readings"; see the per-function citations.  Shared-memory
// records are float4-aligned (device_tables.h: kQS, kJS, kCS) so state,
// parameters and per-item outputs move with LDS.128 / STS.128.
#pragma once
#include <stdint.h>

#include "device_tables.h"

namespace brax {
namespace dev {

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
// I_w⁻¹(q)·v = rotate(q, inv_rotate(q, v) ⊙ I_b⁻¹)   (R4); isotropic: i·v exactly
__device__ __forceinline__ V3 iw(Q4 q, const float* inv_i, bool iso, V3 v) {
  if (iso) return inv_i[0] * v;
  return rotate(q, had(rotate(qconj(q), v), V3{inv_i[0], inv_i[1], inv_i[2]}));
}
__device__ __forceinline__ V3 v3(const float* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ Q4 q4(const float* p) {
  float4 v = *reinterpret_cast<const float4*>(p);
  return {v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ float clampf(float x, float lo, float hi) { return fminf(fmaxf(x, lo), hi); }

// atan2 for fp32: range reduction to [0, 1] and a degree-8 polynomial in a²
// (least-squares/minimax fit of atan(a)/a; max error ≈ 1.0e-7 rad in fp32).
__device__ __forceinline__ float atan2_f(float y, float x) {
  float ax = fabsf(x), ay = fabsf(y);
  float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  float a = (mx > 0.f) ? __fdividef(mn, mx) : 0.f;
  float s = a * a;
  float p = 0.002456719521433115f;
  p = fmaf(p, s, -0.014401338994503021f);
  p = fmaf(p, s, 0.03978119418025017f);
  p = fmaf(p, s, -0.07234854996204376f);
  p = fmaf(p, s, 0.1049894466996193f);
  p = fmaf(p, s, -0.14161229133605957f);
  p = fmaf(p, s, 0.19985906779766083f);
  p = fmaf(p, s, -0.33332598209381104f);
  p = fmaf(p, s, 0.9999998807907104f);
  float r = p * a;
  r = (ay > ax) ? 1.5707963267948966f - r : r;
  r = (x < 0.f) ? 3.141592653589793f - r : r;
  return copysignf(r, y);
}
// asin(x) = atan2(x, √((1−x)(1+x))), x already clamped to [−1, 1]
__device__ __forceinline__ float asin_f(float x) { return atan2_f(x, sqrtf((1.f - x) * (1.f + x))); }

// QP record of one (body, lane) in shared memory: pos | rot | vel | ang, float4 each
struct Row {
  float* p;  // = sQ + (b*E + env) * kQS
  __device__ __forceinline__ V3 pos() const { float4 v = *reinterpret_cast<float4*>(p); return {v.x, v.y, v.z}; }
  __device__ __forceinline__ Q4 rot() const { float4 v = *reinterpret_cast<float4*>(p + 4); return {v.x, v.y, v.z, v.w}; }
  __device__ __forceinline__ V3 vel() const { float4 v = *reinterpret_cast<float4*>(p + 8); return {v.x, v.y, v.z}; }
  __device__ __forceinline__ V3 ang() const { float4 v = *reinterpret_cast<float4*>(p + 12); return {v.x, v.y, v.z}; }
  __device__ __forceinline__ void set_pos(V3 v) const { *reinterpret_cast<float4*>(p) = make_float4(v.x, v.y, v.z, 0.f); }
  __device__ __forceinline__ void set_rot(Q4 q) const { *reinterpret_cast<float4*>(p + 4) = make_float4(q.w, q.x, q.y, q.z); }
  __device__ __forceinline__ void set_vel(V3 v) const { *reinterpret_cast<float4*>(p + 8) = make_float4(v.x, v.y, v.z, 0.f); }
  __device__ __forceinline__ void set_ang(V3 v) const { *reinterpret_cast<float4*>(p + 12) = make_float4(v.x, v.y, v.z, 0.f); }
};
// record of body b for env-slot `el` of a block holding E envs
__device__ __forceinline__ Row row(float* sQ, int b, int el, int E) { return Row{sQ + (b * E + el) * kQS}; }

// ---- S2: kinematic integrator (R3, R21) -------------------------
__device__ __forceinline__ void kinematic(const DBody& bd, Row r, float h) {
  V3 v = r.vel();
  if (!(bd.flags & kFlagFreePos)) v = had(v3(bd.mpos), v);
  r.set_pos(r.pos() + h * v);
  if (!bd.rot_frozen) {
    V3 w = r.ang();
    if (!(bd.flags & kFlagFreeRot)) w = had(v3(bd.mrot), w);
    Q4 q = r.rot();
    Q4 dq = qmul(Q4{0.f, w.x, w.y, w.z}, q);
    float hh = 0.5f * h;
    q = Q4{q.w + hh * dq.w, q.x + hh * dq.x, q.y + hh * dq.y, q.z + hh * dq.z};
    float n2 = q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z;
    float inv = rsqrtf(n2);
    inv = inv * (1.5f - 0.5f * n2 * inv * inv);  // one Newton step: ≈ correctly rounded 1/√n2
    r.set_rot(Q4{q.w * inv, q.x * inv, q.y * inv, q.z * inv});
  }
}

// ---- S3 + S4: joint spring/limits with its actuator (R5, R7-R12)
// act: this env's column of the block's actions sA[k][env] (stride E).
// out: this (joint, env) record: F on child | T child | T parent.
// Zero offsets / identity frames are computed through (exact results, no
// branches: better ILP); only the optional damping term and the actuator are
// guarded, by flags that are uniform across a warp's lane groups.
__device__ __forceinline__ void joint(const DJoint& J, Row P, Row C, const float* act, int E, float* out) {
  Q4 qp = P.rot(), qc = C.rot();
  V3 rp = rotate(qp, v3(J.o_p));
  V3 rc = rotate(qc, v3(J.o_c));
  V3 dx = (P.pos() - C.pos()) + (rp - rc);
  V3 wp = P.ang(), wc = C.ang();
  V3 f = J.k * dx;
  if (!(J.flags & kJNoCl)) f = f + J.c_l * ((P.vel() + cross(wp, rp)) - (C.vel() + cross(wc, rc)));
  Q4 fp = qmul(qp, q4(J.jp));
  Q4 fc = qmul(qc, q4(J.jc));
  Q4 qr = qmul(qconj(fp), fc);
  float sg = (qr.w < 0.f) ? -1.f : 1.f;  // canonicalise q_r to w >= 0 (R25)
  qr = Q4{sg * qr.w, sg * qr.x, sg * qr.y, sg * qr.z};
  float R02 = 2.f * (qr.x * qr.z + qr.w * qr.y);
  float R12 = 2.f * (qr.y * qr.z - qr.w * qr.x);
  float R22 = 1.f - 2.f * (qr.x * qr.x + qr.y * qr.y);
  float R01 = 2.f * (qr.x * qr.y - qr.w * qr.z);
  float R00 = 1.f - 2.f * (qr.y * qr.y + qr.z * qr.z);
  float th[3] = {atan2_f(-R12, R22), asin_f(clampf(R02, -1.f, 1.f)), atan2_f(-R01, R00)};
  float tau[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const bool free_axis = i < J.dof;
    tau[i] = free_axis ? J.k_l * (clampf(th[i], J.lo[i], J.hi[i]) - th[i]) : -(J.k_a * th[i]);
  }
  if (J.act_kind >= 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (i < J.dof) {
        float a = act[(J.act_offset + i) * E];
        tau[i] += (J.act_kind == 0) ? J.strength * clampf(a, -1.f, 1.f)
                                    : J.strength * (clampf(a, J.lo[i], J.hi[i]) - th[i]);
      }
    }
  }
  V3 twd = rotate(fp, V3{tau[0], tau[1], tau[2]});
  if (!(J.flags & kJNoCa)) twd = twd + J.c_a * (wp - wc);
  V3 tc = twd + cross(rc, f);
  V3 tp = twd + cross(rp, f);
  float4* o = reinterpret_cast<float4*>(out);
  o[0] = make_float4(f.x, f.y, f.z, 0.f);
  o[1] = make_float4(tc.x, tc.y, tc.z, 0.f);
  o[2] = make_float4(-tp.x, -tp.y, -tp.z, 0.f);
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
// out: this (slot, env) record: P, active | r_A×P | r_B×P; cnt: substeps active.
__device__ __forceinline__ void contact(const DSlot& S, Row A, Row B, float opl_e, float beta_over_h, float mu,
                                        float* out, int* cnt) {
  const int fl = S.flags;
  Q4 qa = A.rot(), qb = B.rot();
  V3 xa = A.pos(), xb = B.pos();
  V3 cA = (fl & kSZeroPa) ? xa : xa + rotate(qa, v3(S.ca_pos));
  V3 cB = (fl & kSZeroPb) ? xb : xb + rotate(qb, v3(S.cb_pos));
  Q4 qA = (fl & kSIdentA) ? qa : qmul(qa, q4(S.ca_rot));
  Q4 qB = (fl & kSIdentB) ? qb : qmul(qb, q4(S.cb_rot));
  const V3 zhat{0.f, 0.f, 1.f};
  V3 n, pt;
  float d;
  if (S.type <= 2) {  // sphere / capsule end / box corner vs plane: plane is B
    n = rotate(qB, zhat);
    if (S.type == 2) {
      V3 c = cA + rotate(qA, v3(S.corner));
      d = -dot(c - cB, n);
      pt = c;
    } else {
      V3 c = (S.type == 1) ? cA + S.ell_a * rotate(qA, zhat) : cA;
      d = S.ra - dot(c - cB, n);
      pt = c - S.ra * n;
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
      seg_seg(cA + S.ell_a * axa, cA - S.ell_a * axa, cB + S.ellb * axb, cB - S.ellb * axb, pa, pb);
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
    V3 u = (A.vel() + cross(A.ang(), rA)) - (B.vel() + cross(B.ang(), rB));
    float un = dot(u, n);
    const bool isa = fl & kSIsoA, isb = fl & kSIsoB;
    auto eff = [&](V3 dir) {  // k(dir) = Σ_X not static [1/m_X + (r_X×dir)·I_w⁻¹(r_X×dir)]
      float k = 0.f;
      if (!S.a_static) {
        V3 rn = cross(rA, dir);
        k = k + S.inv_mass_a + dot(rn, iw(qa, S.inv_inertia_a, isa, rn));
      }
      if (!S.b_static) {
        V3 rn = cross(rB, dir);
        k = k + S.inv_mass_b + dot(rn, iw(qb, S.inv_inertia_b, isb, rn));
      }
      return k;
    };
    float kn = eff(n);
    float jn = fmaxf(0.f, __fdividef(-opl_e * un + beta_over_h * d, kn));
    if (jn > 0.f) {
      active = true;
      V3 ut = u - un * n;
      float st2 = dot(ut, ut);
      P = jn * n;
      if (st2 > 0.f) {
        float ist = rsqrtf(st2);
        float st = st2 * ist;
        V3 th = ist * ut;
        float jt = fminf(__fdividef(st, eff(th)), mu * jn);
        P = P - jt * th;
      }
      ta = cross(rA, P);
      tb = cross(rB, P);
    }
  }
  float4* o = reinterpret_cast<float4*>(out);
  o[0] = make_float4(P.x, P.y, P.z, active ? 1.f : 0.f);
  o[1] = make_float4(ta.x, ta.y, ta.z, 0.f);
  o[2] = make_float4(tb.x, tb.y, tb.z, 0.f);
  *cnt += active ? 1 : 0;
}

// ---- S6: per-body accumulation over the static incidence lists (fixed order) --
// e = (item << 4) | t with t = 4 (child / A side: sign +1) or 8 (parent / B side:
// sign −1); rec: this env's record of the item; the torque vector sits at word t.
struct Acc {
  V3 F{0.f, 0.f, 0.f}, T{0.f, 0.f, 0.f}, dV{0.f, 0.f, 0.f}, dW{0.f, 0.f, 0.f};
  float cnt = 0.f;
  __device__ __forceinline__ void joint(const float* rec, int e) {
    float4 f = *reinterpret_cast<const float4*>(rec), t = *reinterpret_cast<const float4*>(rec + (e & 15));
    float sg = (e & 8) ? -1.f : 1.f;
    F = V3{fmaf(sg, f.x, F.x), fmaf(sg, f.y, F.y), fmaf(sg, f.z, F.z)};
    T = T + V3{t.x, t.y, t.z};
  }
  __device__ __forceinline__ void slot(const float* rec, int e) {
    float4 p = *reinterpret_cast<const float4*>(rec), t = *reinterpret_cast<const float4*>(rec + (e & 15));
    float sg = (e & 8) ? -1.f : 1.f;
    dV = V3{fmaf(sg, p.x, dV.x), fmaf(sg, p.y, dV.y), fmaf(sg, p.z, dV.z)};
    dW = V3{fmaf(sg, t.x, dW.x), fmaf(sg, t.y, dW.y), fmaf(sg, t.z, dW.z)};
    cnt += p.w;
  }
};

// ---- S7 + S8: potential integrator then collision integrator (R14, R21)
__device__ __forceinline__ void integrate(const DBody& bd, Row r, const Acc& acc, float h, V3 g) {
  const bool iso = bd.flags & kFlagIso, fp = bd.flags & kFlagFreePos, fr = bd.flags & kFlagFreeRot;
  Q4 q = r.rot();
  V3 v = r.vel() + h * (bd.inv_mass * acc.F + g);
  V3 w = r.ang() + h * iw(q, bd.inv_inertia, iso, acc.T);
  if (!fp) v = had(v3(bd.mpos), v);
  if (!fr) w = had(v3(bd.mrot), w);
  if (acc.cnt > 0.f) {
    float ic = __fdividef(1.f, acc.cnt);  // R14: mean over the body's active contacts
    v = v + (bd.inv_mass * ic) * acc.dV;
    w = w + ic * iw(q, bd.inv_inertia, iso, acc.dW);
    if (!fp) v = had(v3(bd.mpos), v);
    if (!fr) w = had(v3(bd.mrot), w);
  }
  r.set_vel(v);
  r.set_ang(w);
}

// ---- S1 / S9: staging of one QP field [n][B][K] <-> sQ record words foff..foff+K-1.
// One env row (B·K contiguous floats) per warp iteration, lanes along the row:
// coalesced, and no integer division (K is a compile-time constant).
template <int K, bool kLoad>
__device__ __forceinline__ void stage(const float* gin, float* gout, float* sQ, int foff, int64_t e0, int nvalid,
                                      int B, int E) {
  const int row_len = B * K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int env = warp; env < nvalid; env += nw) {
    const int64_t g0 = (e0 + env) * row_len;
    for (int k = lane; k < row_len; k += 32) {
      const int b = k / K, c = k - (k / K) * K;
      float* s = sQ + (b * E + env) * kQS + foff + c;
      if (kLoad) *s = __ldg(gin + g0 + k);
      else gout[g0 + k] = *s;
    }
  }
}

// ---- TMA 1-D bulk copies (cp.async.bulk) + mbarrier, sm_90+/sm_100a ----------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared, completion signalled on `bar` (bytes and addresses multiples of 16)
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
// shared -> global (bulk group); the caller commits and waits
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Staging area layout (words): the block's contiguous global chunks
// pos [E][B][3] | rot [E][B][4] | vel [E][B][3] | ang [E][B][3].
__device__ __forceinline__ void stg_to_records(const float* stg, float* sQ, int B, int E, int nvalid) {
  const float* sp = stg;
  const float* sr = stg + E * B * 3;
  const float* sv = sr + E * B * 4;
  const float* sw = sv + E * B * 3;
  for (int i = threadIdx.x; i < nvalid * B; i += blockDim.x) {
    const int env = i / B, b = i - env * B;
    float4* r = reinterpret_cast<float4*>(sQ + (b * E + env) * kQS);
    r[0] = make_float4(sp[3 * i], sp[3 * i + 1], sp[3 * i + 2], 0.f);
    r[1] = make_float4(sr[4 * i], sr[4 * i + 1], sr[4 * i + 2], sr[4 * i + 3]);
    r[2] = make_float4(sv[3 * i], sv[3 * i + 1], sv[3 * i + 2], 0.f);
    r[3] = make_float4(sw[3 * i], sw[3 * i + 1], sw[3 * i + 2], 0.f);
  }
}
__device__ __forceinline__ void records_to_stg(const float* sQ, float* stg, int B, int E, int nvalid) {
  float* sp = stg;
  float* sr = stg + E * B * 3;
  float* sv = sr + E * B * 4;
  float* sw = sv + E * B * 3;
  for (int i = threadIdx.x; i < nvalid * B; i += blockDim.x) {
    const int env = i / B, b = i - env * B;
    const float4* r = reinterpret_cast<const float4*>(sQ + (b * E + env) * kQS);
    float4 p = r[0], q = r[1], v = r[2], w = r[3];
    sp[3 * i] = p.x; sp[3 * i + 1] = p.y; sp[3 * i + 2] = p.z;
    sr[4 * i] = q.x; sr[4 * i + 1] = q.y; sr[4 * i + 2] = q.z; sr[4 * i + 3] = q.w;
    sv[3 * i] = v.x; sv[3 * i + 1] = v.y; sv[3 * i + 2] = v.z;
    sw[3 * i] = w.x; sw[3 * i + 1] = w.y; sw[3 * i + 2] = w.z;
  }
}

// S1: the block's E envs' QP -> shared memory (env slots past the batch end get identity state)
__device__ __forceinline__ void load_block(const StepArgs& a, float* sQ, uint32_t* sStat, int B, int E, int64_t e0,
                                           int nvalid) {
  if (nvalid < E) {
    for (int i = threadIdx.x; i < B * E; i += blockDim.x) {
      float4* p = reinterpret_cast<float4*>(sQ + i * kQS);
      p[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      p[1] = make_float4(1.f, 0.f, 0.f, 0.f);
      p[2] = make_float4(0.f, 0.f, 0.f, 0.f);
      p[3] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
  }
  stage<3, true>(a.pos_in, nullptr, sQ, 0, e0, nvalid, B, E);
  stage<4, true>(a.rot_in, nullptr, sQ, 4, e0, nvalid, B, E);
  stage<3, true>(a.vel_in, nullptr, sQ, 8, e0, nvalid, B, E);
  stage<3, true>(a.ang_in, nullptr, sQ, 12, e0, nvalid, B, E);
}

// S1 (per step): this step's action [n][A] -> sA[k][env] (one env row per warp iteration)
__device__ __forceinline__ void load_actions(const StepArgs& a, float* sA, int A, int E, int64_t step, int64_t e0,
                                             int nvalid) {
  if (A <= 0) return;
  const float* act = a.actions + (step * a.n_envs + e0) * A;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int env = warp; env < nvalid; env += nw)
    for (int k = lane; k < A; k += 32) sA[k * E + env] = __ldg(act + env * A + k);
}

// S9: status bits and contact counts (after a barrier)
__device__ __forceinline__ void block_extras(const StepArgs& a, const float* sQ, const int* sCnt, uint32_t* sStat,
                                             int B, int C, int E, int64_t e0, int nvalid) {
  if (a.status) {
    for (int i = threadIdx.x; i < B * E; i += blockDim.x) {
      const float* p = sQ + i * kQS;
      uint32_t bits = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k == 3 || k == 11 || k == 15) continue;  // padding words
        float v = p[k];
        bits |= isfinite(v) ? (fabsf(v) > 1e6f ? 2u : 0u) : 1u;
      }
      if (bits) atomicOr(&sStat[i % E], bits);
    }
  }
  if (a.contact_active) {
    for (int i = threadIdx.x; i < nvalid * C; i += blockDim.x) {
      int env = i / C, c = i - env * C;
      a.contact_active[(e0 + env) * C + c] = uint8_t(sCnt[c * E + env]);
    }
  }
}

// S9 fallback (ragged tail / unaligned): per-row stores of the QP
__device__ __forceinline__ void store_block(const StepArgs& a, float* sQ, int B, int E, int64_t e0, int nvalid) {
  stage<3, false>(nullptr, a.pos_out, sQ, 0, e0, nvalid, B, E);
  stage<4, false>(nullptr, a.rot_out, sQ, 4, e0, nvalid, B, E);
  stage<3, false>(nullptr, a.vel_out, sQ, 8, e0, nvalid, B, E);
  stage<3, false>(nullptr, a.ang_out, sQ, 12, e0, nvalid, B, E);
}

}  // namespace dev
}  // namespace brax
