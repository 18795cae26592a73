// step_device.cuh — device code of the batched Brax step (sm_100a).
//
// Formulas: Alg. 1 of the paper with SURVEY.md §8(c).1 /
// DESIGN.md "Readings"; see the per-function citations.  Shared-memory
// records are float4-aligned (device_tables.h: kQS, kJS, kCS) so state and
// per-item outputs move with LDS.128 / STS.128.
//
// The physics is templated on the per-lane scalar S: `float` (one env per
// lane) or `F2` (two envs per lane: every parameter load, branch and address
// computation then serves two envs, and the two independent dependency chains
// double the instruction-level parallelism).  Conditions that differ between
// envs (contact activity, clamps, signs) are selects, never branches.
#pragma once
#include <stdint.h>

#include "device_tables.h"

namespace brax {
namespace dev {

// ---- per-lane scalar types -----------------------------------------------------
struct F2 { float x, y; };
struct B2 { bool x, y; };

__device__ __forceinline__ F2 operator+(F2 a, F2 b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ F2 operator-(F2 a, F2 b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ F2 operator*(F2 a, F2 b) { return {a.x * b.x, a.y * b.y}; }
__device__ __forceinline__ F2 operator-(F2 a) { return {-a.x, -a.y}; }
__device__ __forceinline__ F2 operator+(F2 a, float b) { return {a.x + b, a.y + b}; }
__device__ __forceinline__ F2 operator+(float a, F2 b) { return {a + b.x, a + b.y}; }
__device__ __forceinline__ F2 operator-(F2 a, float b) { return {a.x - b, a.y - b}; }
__device__ __forceinline__ F2 operator-(float a, F2 b) { return {a - b.x, a - b.y}; }
__device__ __forceinline__ F2 operator*(float a, F2 b) { return {a * b.x, a * b.y}; }
__device__ __forceinline__ F2 operator*(F2 a, float b) { return {a.x * b, a.y * b}; }

__device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ F2 vmin(F2 a, F2 b) { return {fminf(a.x, b.x), fminf(a.y, b.y)}; }
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ F2 vmax(F2 a, F2 b) { return {fmaxf(a.x, b.x), fmaxf(a.y, b.y)}; }
__device__ __forceinline__ float vabs(float a) { return fabsf(a); }
__device__ __forceinline__ F2 vabs(F2 a) { return {fabsf(a.x), fabsf(a.y)}; }
__device__ __forceinline__ float vsqrt(float a) { return sqrtf(a); }
__device__ __forceinline__ F2 vsqrt(F2 a) { return {sqrtf(a.x), sqrtf(a.y)}; }
__device__ __forceinline__ float vrsqrt(float a) { return rsqrtf(a); }
__device__ __forceinline__ F2 vrsqrt(F2 a) { return {rsqrtf(a.x), rsqrtf(a.y)}; }
__device__ __forceinline__ float vdiv(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ F2 vdiv(F2 a, F2 b) { return {__fdividef(a.x, b.x), __fdividef(a.y, b.y)}; }
__device__ __forceinline__ float vcopysign(float a, float b) { return copysignf(a, b); }
__device__ __forceinline__ F2 vcopysign(F2 a, F2 b) { return {copysignf(a.x, b.x), copysignf(a.y, b.y)}; }
__device__ __forceinline__ bool lt(float a, float b) { return a < b; }
__device__ __forceinline__ B2 lt(F2 a, F2 b) { return {a.x < b.x, a.y < b.y}; }
__device__ __forceinline__ bool gt(float a, float b) { return a > b; }
__device__ __forceinline__ B2 gt(F2 a, F2 b) { return {a.x > b.x, a.y > b.y}; }
__device__ __forceinline__ float sel(bool m, float a, float b) { return m ? a : b; }
__device__ __forceinline__ F2 sel(B2 m, F2 a, F2 b) { return {m.x ? a.x : b.x, m.y ? a.y : b.y}; }
__device__ __forceinline__ bool both(bool m, bool n) { return m && n; }
__device__ __forceinline__ B2 both(B2 m, B2 n) { return {m.x && n.x, m.y && n.y}; }
__device__ __forceinline__ bool any(bool m) { return m; }
__device__ __forceinline__ bool any(B2 m) { return m.x || m.y; }
__device__ __forceinline__ float as_count(bool m) { return m ? 1.f : 0.f; }
__device__ __forceinline__ F2 as_count(B2 m) { return {m.x ? 1.f : 0.f, m.y ? 1.f : 0.f}; }
template <class S> __device__ __forceinline__ S bc(float f);
template <> __device__ __forceinline__ float bc<float>(float f) { return f; }
template <> __device__ __forceinline__ F2 bc<F2>(float f) { return {f, f}; }
template <class S> __device__ __forceinline__ S clampv(S x, float lo, float hi) {
  return vmin(vmax(x, bc<S>(lo)), bc<S>(hi));
}

template <class S> struct V3T { S x, y, z; };
template <class S> struct Q4T { S w, x, y, z; };
template <class S> __device__ __forceinline__ V3T<S> operator+(V3T<S> a, V3T<S> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class S> __device__ __forceinline__ V3T<S> operator-(V3T<S> a, V3T<S> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class S> __device__ __forceinline__ V3T<S> operator*(S s, V3T<S> a) { return {s * a.x, s * a.y, s * a.z}; }
template <class S> __device__ __forceinline__ V3T<S> scale(float s, V3T<S> a) { return {s * a.x, s * a.y, s * a.z}; }
template <class S> __device__ __forceinline__ V3T<S> had(const float* m, V3T<S> a) { return {m[0] * a.x, m[1] * a.y, m[2] * a.z}; }
template <class S> __device__ __forceinline__ S dot(V3T<S> a, V3T<S> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class S> __device__ __forceinline__ V3T<S> cross(V3T<S> a, V3T<S> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class S> __device__ __forceinline__ V3T<S> bc3(const float* p) { return {bc<S>(p[0]), bc<S>(p[1]), bc<S>(p[2])}; }
template <class S> __device__ __forceinline__ Q4T<S> bcq(const float* p) {
  return {bc<S>(p[0]), bc<S>(p[1]), bc<S>(p[2]), bc<S>(p[3])};
}
template <class S> __device__ __forceinline__ V3T<S> sel3(decltype(lt(S(), S())) m, V3T<S> a, V3T<S> b) {
  return {sel(m, a.x, b.x), sel(m, a.y, b.y), sel(m, a.z, b.z)};
}
template <class S> __device__ __forceinline__ Q4T<S> qmul(Q4T<S> a, Q4T<S> b) {
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x, a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w};
}
template <class S> __device__ __forceinline__ Q4T<S> qconj(Q4T<S> q) { return {q.w, -q.x, -q.y, -q.z}; }
// c + a×b with the products fused into the accumulation (2 FFMA per component)
template <class S> __device__ __forceinline__ V3T<S> cross_add(V3T<S> a, V3T<S> b, V3T<S> c) {
  return {a.y * b.z + (c.x - a.z * b.y), a.z * b.x + (c.y - a.x * b.z), a.x * b.y + (c.z - a.y * b.x)};
}
// rotate(q, v) = v + w·t + u×t, t = 2u×v, evaluated as v + (2w)·c + (2u)×c with
// c = u×v: 7 FMUL + 12 FFMA instead of 9 FMUL + 9 FFMA + 3 FADD.
template <class S> __device__ __forceinline__ V3T<S> rotate(Q4T<S> q, V3T<S> v) {
  V3T<S> u{q.x, q.y, q.z};
  V3T<S> c = cross(u, v);
  S w2 = 2.f * q.w;
  V3T<S> u2{2.f * q.x, 2.f * q.y, 2.f * q.z};
  V3T<S> r{w2 * c.x + v.x, w2 * c.y + v.y, w2 * c.z + v.z};
  return cross_add(u2, c, r);
}
// rotate(q, ẑ): the third column of R(q)
template <class S> __device__ __forceinline__ V3T<S> rotate_z(Q4T<S> q) {
  return {2.f * (q.x * q.z + q.w * q.y), 2.f * (q.y * q.z - q.w * q.x), 1.f - 2.f * (q.x * q.x + q.y * q.y)};
}
// I_w⁻¹(q)·v = rotate(q, inv_rotate(q, v) ⊙ I_b⁻¹)   (R4); isotropic: i·v exactly
template <class S> __device__ __forceinline__ V3T<S> iw(Q4T<S> q, const float* inv_i, bool iso, V3T<S> v) {
  if (iso) return scale(inv_i[0], v);
  return rotate(q, had(inv_i, rotate(qconj(q), v)));
}

// atan2 for fp32: range reduction to [0, 1] and a degree-8 polynomial in a²
// (least-squares/minimax fit of atan(a)/a; max error ≈ 1.0e-7 rad in fp32).
template <class S> __device__ __forceinline__ S atan2_f(S y, S x) {
  S ax = vabs(x), ay = vabs(y);
  S mx = vmax(ax, ay), mn = vmin(ax, ay);
  S a = sel(gt(mx, bc<S>(0.f)), vdiv(mn, mx), bc<S>(0.f));
  S s = a * a;
  S p = bc<S>(0.002456719521433115f);
  p = p * s + -0.014401338994503021f;
  p = p * s + 0.03978119418025017f;
  p = p * s + -0.07234854996204376f;
  p = p * s + 0.1049894466996193f;
  p = p * s + -0.14161229133605957f;
  p = p * s + 0.19985906779766083f;
  p = p * s + -0.33332598209381104f;
  p = p * s + 0.9999998807907104f;
  S r = p * a;
  r = sel(gt(ay, ax), 1.5707963267948966f - r, r);
  r = sel(lt(x, bc<S>(0.f)), 3.141592653589793f - r, r);
  return vcopysign(r, y);
}
// asin(x) = atan2(x, √((1−x)(1+x))), x already clamped to [−1, 1]
template <class S> __device__ __forceinline__ S asin_f(S x) {
  S c2 = (1.f - x) * (1.f + x);  // ≥ 0; √ via rsqrt (no IEEE slow-path call), exact 0 at |x| = 1
  return atan2_f(x, sel(gt(c2, bc<S>(0.f)), c2 * vrsqrt(c2), bc<S>(0.f)));
}

// ---- shared-memory access for V = 1 or 2 envs per lane ---------------------------
// A lane of a group of L lanes handles env slot `el` and (S = F2) `el + L`; the
// second env's record sits `o2` words after the first's.
__device__ __forceinline__ float ld1(const float* p, int) { return *p; }
__device__ __forceinline__ F2 ld2(const float* p, int o2) { return {p[0], p[o2]}; }
template <class S> struct Lanes;
template <> struct Lanes<float> {
  static __device__ __forceinline__ float4 ld4(const float* p, int) { return *reinterpret_cast<const float4*>(p); }
  static __device__ __forceinline__ V3T<float> ld3(const float* p, int o2) {
    float4 a = ld4(p, o2);
    return {a.x, a.y, a.z};
  }
  static __device__ __forceinline__ Q4T<float> ldq(const float* p, int o2) {
    float4 a = ld4(p, o2);
    return {a.x, a.y, a.z, a.w};
  }
  static __device__ __forceinline__ void st3(float* p, int, V3T<float> v, float w = 0.f) {
    *reinterpret_cast<float4*>(p) = make_float4(v.x, v.y, v.z, w);
  }
  static __device__ __forceinline__ void stq(float* p, int, Q4T<float> q) {
    *reinterpret_cast<float4*>(p) = make_float4(q.w, q.x, q.y, q.z);
  }
  static __device__ __forceinline__ float ld(const float* p, int) { return *p; }
  static __device__ __forceinline__ float w4(const float* p, int) { return p[3]; }
};
template <> struct Lanes<F2> {
  static __device__ __forceinline__ V3T<F2> ld3(const float* p, int o2) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + o2);
    return {{a.x, b.x}, {a.y, b.y}, {a.z, b.z}};
  }
  static __device__ __forceinline__ Q4T<F2> ldq(const float* p, int o2) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + o2);
    return {{a.x, b.x}, {a.y, b.y}, {a.z, b.z}, {a.w, b.w}};
  }
  static __device__ __forceinline__ void st3(float* p, int o2, V3T<F2> v, F2 w = {0.f, 0.f}) {
    *reinterpret_cast<float4*>(p) = make_float4(v.x.x, v.y.x, v.z.x, w.x);
    *reinterpret_cast<float4*>(p + o2) = make_float4(v.x.y, v.y.y, v.z.y, w.y);
  }
  static __device__ __forceinline__ void stq(float* p, int o2, Q4T<F2> q) {
    *reinterpret_cast<float4*>(p) = make_float4(q.w.x, q.x.x, q.y.x, q.z.x);
    *reinterpret_cast<float4*>(p + o2) = make_float4(q.w.y, q.x.y, q.y.y, q.z.y);
  }
  static __device__ __forceinline__ F2 ld(const float* p, int o2) { return {p[0], p[o2]}; }
  static __device__ __forceinline__ F2 w4(const float* p, int o2) { return {p[3], p[o2 + 3]}; }
};

// QP record of one (body, env) in shared memory: pos | rot | vel | ang, float4 each
template <class S> struct Row {
  float* p;  // = sQ + (b*E + env) * kQS
  int o2;    // second env's record (S = F2): + L·kQS words
  __device__ __forceinline__ V3T<S> pos() const { return Lanes<S>::ld3(p, o2); }
  __device__ __forceinline__ Q4T<S> rot() const { return Lanes<S>::ldq(p + 4, o2); }
  __device__ __forceinline__ V3T<S> vel() const { return Lanes<S>::ld3(p + 8, o2); }
  __device__ __forceinline__ V3T<S> ang() const { return Lanes<S>::ld3(p + 12, o2); }
  __device__ __forceinline__ void set_pos(V3T<S> v) const { Lanes<S>::st3(p, o2, v); }
  __device__ __forceinline__ void set_rot(Q4T<S> q) const { Lanes<S>::stq(p + 4, o2, q); }
  __device__ __forceinline__ void set_vel(V3T<S> v) const { Lanes<S>::st3(p + 8, o2, v); }
  __device__ __forceinline__ void set_ang(V3T<S> v) const { Lanes<S>::st3(p + 12, o2, v); }
};

// ---- S2: kinematic integrator (R3, R21) -------------------------
template <class S> __device__ __forceinline__ void kinematic(const DBody& bd, Row<S> r, float h) {
  V3T<S> v = r.vel();
  if (!(bd.flags & kFlagFreePos)) v = had(bd.mpos, v);
  r.set_pos(r.pos() + scale(h, v));
  if (!bd.rot_frozen) {
    V3T<S> w = r.ang();
    if (!(bd.flags & kFlagFreeRot)) w = had(bd.mrot, w);
    Q4T<S> q = r.rot();
    Q4T<S> dq = qmul(Q4T<S>{bc<S>(0.f), w.x, w.y, w.z}, q);
    const float hh = 0.5f * h;
    q = Q4T<S>{q.w + hh * dq.w, q.x + hh * dq.x, q.y + hh * dq.y, q.z + hh * dq.z};
    S n2 = q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z;
    S inv = vrsqrt(n2);
    inv = inv * (1.5f - 0.5f * n2 * inv * inv);  // one Newton step: ≈ correctly rounded 1/√n2
    r.set_rot(Q4T<S>{q.w * inv, q.x * inv, q.y * inv, q.z * inv});
  }
}

// ---- S3 + S4: joint spring/limits with its actuator (R5, R7-R12)
// act: this env's column of the block's actions sA[k][env] (row stride E, second env + L).
// out: this (joint, env) record: F on child | T child | T parent.
template <class S>
__device__ __forceinline__ void joint(const DJoint& Jm, Row<S> P, Row<S> C, const float* act, int E, int L,
                                      float* out, int o2) {
  // the parameter record, read with LDS.128 (struct fields at fixed float4 slots)
  const float4* J4 = reinterpret_cast<const float4*>(&Jm);
  const int4 h0 = *reinterpret_cast<const int4*>(&Jm), h1 = reinterpret_cast<const int4*>(&Jm)[1];
  const int dof = h0.z, act_kind = h0.w, act_offset = h1.x, flags = h1.y;
  const float4 op_k = J4[2], oc_cl = J4[3], jp = J4[4], jc = J4[5], lo_kl = J4[6], hi_ka = J4[7], ca_s = J4[8];
  const float lo[3] = {lo_kl.x, lo_kl.y, lo_kl.z}, hi[3] = {hi_ka.x, hi_ka.y, hi_ka.z};
  Q4T<S> qp = P.rot(), qc = C.rot();
  V3T<S> rp = rotate(qp, V3T<S>{bc<S>(op_k.x), bc<S>(op_k.y), bc<S>(op_k.z)});
  V3T<S> rc = rotate(qc, V3T<S>{bc<S>(oc_cl.x), bc<S>(oc_cl.y), bc<S>(oc_cl.z)});
  V3T<S> dx = (P.pos() - C.pos()) + (rp - rc);
  V3T<S> wp = P.ang(), wc = C.ang();
  V3T<S> f = scale(op_k.w, dx);
  if (!(flags & kJNoCl))
    f = f + scale(oc_cl.w, cross_add(wp, rp, P.vel()) - cross_add(wc, rc, C.vel()));
  Q4T<S> fp = qmul(qp, Q4T<S>{bc<S>(jp.x), bc<S>(jp.y), bc<S>(jp.z), bc<S>(jp.w)});
  Q4T<S> fc = qmul(qc, Q4T<S>{bc<S>(jc.x), bc<S>(jc.y), bc<S>(jc.z), bc<S>(jc.w)});
  Q4T<S> qr = qmul(qconj(fp), fc);
  S sg = sel(lt(qr.w, bc<S>(0.f)), bc<S>(-1.f), bc<S>(1.f));  // canonicalise q_r to w >= 0 (R25)
  qr = Q4T<S>{sg * qr.w, sg * qr.x, sg * qr.y, sg * qr.z};
  S R02 = 2.f * (qr.x * qr.z + qr.w * qr.y);
  S R12 = 2.f * (qr.y * qr.z - qr.w * qr.x);
  S R22 = 1.f - 2.f * (qr.x * qr.x + qr.y * qr.y);
  S R01 = 2.f * (qr.x * qr.y - qr.w * qr.z);
  S R00 = 1.f - 2.f * (qr.y * qr.y + qr.z * qr.z);
  S th[3] = {atan2_f(-R12, R22), asin_f(clampv(R02, -1.f, 1.f)), atan2_f(-R01, R00)};
  S tau[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (i < dof) tau[i] = lo_kl.w * (clampv(th[i], lo[i], hi[i]) - th[i]);
    else tau[i] = -(hi_ka.w * th[i]);
  }
  if (act_kind >= 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (i < dof) {
        S a = Lanes<S>::ld(act + (act_offset + i) * E, L);
        tau[i] = tau[i] + ((act_kind == 0) ? ca_s.y * clampv(a, -1.f, 1.f)
                                           : ca_s.y * (clampv(a, lo[i], hi[i]) - th[i]));
      }
    }
  }
  // τ_i is the generalised force conjugate to θ_i (R7 as amended): the parent-
  // joint-frame torque is Σ τ_i b_i, b the dual basis of the rotation axes of Rx Ry Rz.
  // With c1 = cos θ1 = √(R12² + R22²), sin θ0 = −R12/c1, cos θ0 = R22/c1, sin θ1 = R02:
  //   tj = (τ0, u·R12 + t·R22, u·R22 − t·R12),  u = (τ2 − τ0·R02)/max(c1², 0.01),  t = τ1/c1.
  S c2 = R12 * R12 + R22 * R22;  // cos² θ1
  S ic = sel(gt(c2, bc<S>(0.f)), vrsqrt(c2), bc<S>(0.f));
  S t1 = tau[1] * ic;
  S u = (tau[2] - tau[0] * R02) * vmin(ic * ic, bc<S>(100.f));
  V3T<S> tj{tau[0], u * R12 + t1 * R22, u * R22 - t1 * R12};
  V3T<S> twd = rotate(fp, tj);
  if (!(flags & kJNoCa)) twd = twd + scale(ca_s.x, wp - wc);
  V3T<S> tc = cross_add(rc, f, twd);
  V3T<S> tp = cross_add(rp, f, twd);
  Lanes<S>::st3(out, o2, f);
  Lanes<S>::st3(out + 4, o2, tc);
  Lanes<S>::st3(out + 8, o2, V3T<S>{-tp.x, -tp.y, -tp.z});
}

// Closest points between segments (Ericson, Real-Time Collision Detection §5.1.9),
// with the per-env branches written as selects.  Degenerate (zero-length)
// segments are a parameter property (uniform): a = |d1|², e = |d2|² > 0 unless ℓ = 0.
template <class S>
__device__ __forceinline__ void seg_seg(V3T<S> p1, V3T<S> q1, V3T<S> p2, V3T<S> q2, bool degA, bool degB,
                                        V3T<S>& c1, V3T<S>& c2) {
  V3T<S> d1 = q1 - p1, d2 = q2 - p2, r = p1 - p2;
  S a = dot(d1, d1), e = dot(d2, d2), f = dot(d2, r);
  const S zero = bc<S>(0.f);
  S s = zero, t = zero;
  if (degA && degB) {
  } else if (degA) {
    t = clampv(vdiv(f, e), 0.f, 1.f);
  } else {
    S c = dot(d1, r);
    if (degB) {
      s = clampv(vdiv(-c, a), 0.f, 1.f);
    } else {
      S b = dot(d1, d2);
      S denom = a * e - b * b;
      s = sel(gt(vabs(denom), zero), clampv(vdiv(b * f - c * e, denom), 0.f, 1.f), zero);
      t = vdiv(b * s + f, e);
      S s_lo = clampv(vdiv(-c, a), 0.f, 1.f), s_hi = clampv(vdiv(b - c, a), 0.f, 1.f);
      auto tl = lt(t, zero), th = gt(t, bc<S>(1.f));
      s = sel(tl, s_lo, sel(th, s_hi, s));
      t = sel(tl, zero, sel(th, bc<S>(1.f), t));
    }
  }
  c1 = p1 + s * d1;
  c2 = p2 + t * d2;
}

// ---- S5: contact slot, velocity-level impulse + Baumgarte (R13-R19)
// out: this (slot, env) record: P, active | r_A×P | r_B×P; cnt: substeps active.
template <class S>
__device__ __forceinline__ void contact(const DSlot& SLm, Row<S> A, Row<S> B, float opl_e, float beta_over_h,
                                        float mu, float* out, int o2, S& cnt) {
  // the parameter record, read with LDS.128 at its fixed float4 slots
  const float4* S4 = reinterpret_cast<const float4*>(&SLm);
  const int4 h0 = *reinterpret_cast<const int4*>(&SLm), h1 = reinterpret_cast<const int4*>(&SLm)[1];
  const int type = h0.x, a_static = h1.x, b_static = h1.y, fl = h1.z;
  const float4 ca = S4[2], cb = S4[4], ells = S4[6];  // ca_pos|ra, cb_pos|rb, ell_a ellb 1/m_a 1/m_b
  const float ra = ca.w, rb = cb.w;
  Q4T<S> qa = A.rot(), qb = B.rot();
  V3T<S> xa = A.pos(), xb = B.pos();
  V3T<S> cA = (fl & kSZeroPa) ? xa : xa + rotate(qa, V3T<S>{bc<S>(ca.x), bc<S>(ca.y), bc<S>(ca.z)});
  V3T<S> cB = (fl & kSZeroPb) ? xb : xb + rotate(qb, V3T<S>{bc<S>(cb.x), bc<S>(cb.y), bc<S>(cb.z)});
  Q4T<S> qA = qa, qB = qb;
  if (!(fl & kSIdentA)) {
    const float4 r = S4[3];
    qA = qmul(qa, Q4T<S>{bc<S>(r.x), bc<S>(r.y), bc<S>(r.z), bc<S>(r.w)});
  }
  if (!(fl & kSIdentB)) {
    const float4 r = S4[5];
    qB = qmul(qb, Q4T<S>{bc<S>(r.x), bc<S>(r.y), bc<S>(r.z), bc<S>(r.w)});
  }
  const S zero = bc<S>(0.f);
  V3T<S> n, pt;
  S d;
  if (type <= 2) {  // sphere / capsule end / box corner vs plane: plane is B
    n = rotate_z(qB);
    if (type == 2) {
      const float4 k = S4[7];
      V3T<S> c = cA + rotate(qA, V3T<S>{bc<S>(k.x), bc<S>(k.y), bc<S>(k.z)});
      d = -dot(c - cB, n);
      pt = c;
    } else {
      V3T<S> c = (type == 1) ? cA + scale(ells.x, rotate_z(qA)) : cA;
      d = ra - dot(c - cB, n);
      pt = c - scale(ra, n);
    }
  } else {
    V3T<S> pa = cA, pb = cB;
    if (type == 4) {  // sphere (A) – capsule (B)
      V3T<S> axb = rotate_z(qB);
      V3T<S> e0 = cB + scale(ells.y, axb), e1 = cB - scale(ells.y, axb);
      V3T<S> seg = e0 - e1;
      if (ells.y > 0.f) pb = e1 + clampv(vdiv(dot(cA - e1, seg), dot(seg, seg)), 0.f, 1.f) * seg;
      else pb = e1;
    } else if (type == 5) {  // capsule – capsule
      V3T<S> axa = rotate_z(qA), axb = rotate_z(qB);
      seg_seg(cA + scale(ells.x, axa), cA - scale(ells.x, axa), cB + scale(ells.y, axb), cB - scale(ells.y, axb),
              !(ells.x > 0.f), !(ells.y > 0.f), pa, pb);
    }
    V3T<S> delta = pa - pb;
    S dist2 = dot(delta, delta);
    auto nz = gt(dist2, zero);
    S idist = sel(nz, vrsqrt(dist2), zero);
    S dist = dist2 * idist;
    V3T<S> zhat{zero, zero, bc<S>(1.f)};
    n = sel3<S>(nz, idist * delta, zhat);  // R16: ẑ when the centres coincide
    d = (ra + rb) - dist;
    pt = scale(0.5f, (pa - scale(ra, n)) + (pb + scale(rb, n)));
  }
  auto pen = gt(d, zero);  // R16: strict d > 0
  V3T<S> P{zero, zero, zero}, ta{zero, zero, zero}, tb{zero, zero, zero};
  S active = zero;
  if (any(pen)) {
    V3T<S> rA = pt - xa, rB = pt - xb;
    V3T<S> u = cross_add(A.ang(), rA, A.vel()) - cross_add(B.ang(), rB, B.vel());
    S un = dot(u, n);
    const bool isa = fl & kSIsoA, isb = fl & kSIsoB;
    const float4 iia4 = S4[8], iib4 = S4[9];
    const float iia[3] = {iia4.x, iia4.y, iia4.z}, iib[3] = {iib4.x, iib4.y, iib4.z};
    auto eff = [&](V3T<S> dir) {  // k(dir) = Σ_X not static [1/m_X + (r_X×dir)·I_w⁻¹(r_X×dir)]
      S k = zero;
      if (!a_static) {
        V3T<S> rn = cross(rA, dir);
        k = k + ells.z + dot(rn, iw(qa, iia, isa, rn));
      }
      if (!b_static) {
        V3T<S> rn = cross(rB, dir);
        k = k + ells.w + dot(rn, iw(qb, iib, isb, rn));
      }
      return k;
    };
    S jn = vmax(zero, vdiv(-opl_e * un + beta_over_h * d, eff(n)));
    auto act = both(pen, gt(jn, zero));  // R15
    if (any(act)) {
      jn = sel(act, jn, zero);
      V3T<S> ut = u - un * n;
      S st2 = dot(ut, ut);
      auto sl = gt(st2, zero);  // R16: j_t = 0 when s_t = 0
      S ist = sel(sl, vrsqrt(st2), zero);
      S st = st2 * ist;
      V3T<S> th = ist * ut;
      S kt = sel(sl, eff(th), bc<S>(1.f));
      S jt = vmin(vdiv(st, kt), mu * jn);
      P = jn * n - jt * th;
      ta = cross(rA, P);
      tb = cross(rB, P);
      active = as_count(act);
    }
  }
  Lanes<S>::st3(out, o2, P, active);
  Lanes<S>::st3(out + 4, o2, ta);
  Lanes<S>::st3(out + 8, o2, tb);
  cnt = cnt + active;
}

__device__ __forceinline__ void store_count(float* p, int, float c) { *p = c; }
__device__ __forceinline__ void store_count(float* p, int o2, F2 c) {
  p[0] = c.x;
  p[o2] = c.y;
}

// ---- S6: per-body accumulation over the static incidence lists (fixed order) --
// e = (item << 4) | t with t = 4 (child / A side: sign +1) or 8 (parent / B side:
// sign −1); rec: this env's record of the item; the torque vector sits at word t.
template <class S> struct Acc {
  V3T<S> F, T, dV, dW;
  S cnt;
  __device__ __forceinline__ Acc() {
    const S z = bc<S>(0.f);
    F = T = dV = dW = V3T<S>{z, z, z};
    cnt = z;
  }
  __device__ __forceinline__ void joint(const float* rec, int o2, int e) {
    const float sg = (e & 8) ? -1.f : 1.f;
    F = F + scale(sg, Lanes<S>::ld3(rec, o2));
    T = T + Lanes<S>::ld3(rec + (e & 15), o2);
  }
  __device__ __forceinline__ void slot(const float* rec, int o2, int e) {
    const float sg = (e & 8) ? -1.f : 1.f;
    dV = dV + scale(sg, Lanes<S>::ld3(rec, o2));
    dW = dW + scale(sg, Lanes<S>::ld3(rec + (e & 15), o2));
    cnt = cnt + Lanes<S>::w4(rec, o2);
  }
};

// ---- S7 + S8: potential integrator then collision integrator (R14, R21),
// fused (kin = true) with the next substep's S2 kinematic integrator of the same
// body: same arithmetic as kinematic(), with v and ω still in registers.
template <class S> __device__ __forceinline__ void integrate(const DBody& bd, Row<S> r, const Acc<S>& acc, float h,
                                                             const float* g, bool kin) {
  const bool iso = bd.flags & kFlagIso, fp = bd.flags & kFlagFreePos, fr = bd.flags & kFlagFreeRot;
  Q4T<S> q = r.rot();
  V3T<S> v = r.vel() + scale(h, scale(bd.inv_mass, acc.F) + bc3<S>(g));
  V3T<S> w = r.ang() + scale(h, iw(q, bd.inv_inertia, iso, acc.T));
  if (!fp) v = had(bd.mpos, v);
  if (!fr) w = had(bd.mrot, w);
  auto hit = gt(acc.cnt, bc<S>(0.f));
  if (any(hit)) {
    S ic = sel(hit, vdiv(bc<S>(1.f), acc.cnt), bc<S>(0.f));  // R14: mean over the body's active contacts
    v = v + (bd.inv_mass * ic) * acc.dV;
    w = w + ic * iw(q, bd.inv_inertia, iso, acc.dW);
    if (!fp) v = had(bd.mpos, v);
    if (!fr) w = had(bd.mrot, w);
  }
  r.set_vel(v);
  r.set_ang(w);
  if (kin) {  // next substep's kinematic integrator (v, ω already masked)
    r.set_pos(r.pos() + scale(h, v));
    if (!bd.rot_frozen) {
      Q4T<S> dq = qmul(Q4T<S>{bc<S>(0.f), w.x, w.y, w.z}, q);
      const float hh = 0.5f * h;
      Q4T<S> qn{q.w + hh * dq.w, q.x + hh * dq.x, q.y + hh * dq.y, q.z + hh * dq.z};
      S n2 = qn.w * qn.w + qn.x * qn.x + qn.y * qn.y + qn.z * qn.z;
      S inv = vrsqrt(n2);
      inv = inv * (1.5f - 0.5f * n2 * inv * inv);
      r.set_rot(Q4T<S>{qn.w * inv, qn.x * inv, qn.y * inv, qn.z * inv});
    }
  }
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
__device__ __forceinline__ void block_extras(const StepArgs& a, const float* sQ, const float* sCnt, uint32_t* sStat,
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
