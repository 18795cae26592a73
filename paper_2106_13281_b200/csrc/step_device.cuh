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
// F1: one env per lane; F2: two envs per lane.  Both spell out every rounding
// step the same way — products are lazy (M1 / M2) and contract into an FMA
// exactly where the source writes `a*b + c`, `c - a*b` or `a*b + c*d`, every other
// add / mul is rounded on its own (__fadd_rn / __fmul_rn / add.rn.f32x2 are never
// re-fused by the compiler) — so a given env's result is bitwise the same under
// every launch plan (V = 1 or 2), i.e. independent of the batch size.
struct F1 { float x; };
struct F2 { float x, y; };
struct B2 { bool x, y; };

struct M1 {  // the product a*b, not yet rounded
  F1 a, b;
  __device__ __forceinline__ operator F1() const { return {__fmul_rn(a.x, b.x)}; }
};
__device__ __forceinline__ F1 fma1(F1 a, F1 b, F1 c) { return {__fmaf_rn(a.x, b.x, c.x)}; }
__device__ __forceinline__ F1 neg1(F1 a) { return {-a.x}; }
__device__ __forceinline__ F1 bc1(float f) { return {f}; }
__device__ __forceinline__ M1 operator*(F1 a, F1 b) { return {a, b}; }
__device__ __forceinline__ M1 operator*(float a, F1 b) { return {bc1(a), b}; }
__device__ __forceinline__ M1 operator*(F1 a, float b) { return {a, bc1(b)}; }
__device__ __forceinline__ M1 operator*(M1 m, F1 b) { return {F1(m), b}; }
__device__ __forceinline__ M1 operator*(F1 a, M1 m) { return {a, F1(m)}; }
__device__ __forceinline__ M1 operator*(M1 m, float b) { return {F1(m), bc1(b)}; }
__device__ __forceinline__ M1 operator*(float a, M1 m) { return {bc1(a), F1(m)}; }
__device__ __forceinline__ M1 operator*(M1 m, M1 n) { return {F1(m), F1(n)}; }
__device__ __forceinline__ M1 operator-(M1 m) { return {neg1(m.a), m.b}; }
__device__ __forceinline__ F1 operator-(F1 a) { return neg1(a); }
__device__ __forceinline__ F1 operator+(F1 a, F1 b) { return {__fadd_rn(a.x, b.x)}; }
__device__ __forceinline__ F1 operator-(F1 a, F1 b) { return {__fadd_rn(a.x, -b.x)}; }
__device__ __forceinline__ F1 operator+(F1 a, float b) { return {__fadd_rn(a.x, b)}; }
__device__ __forceinline__ F1 operator+(float a, F1 b) { return {__fadd_rn(a, b.x)}; }
__device__ __forceinline__ F1 operator-(F1 a, float b) { return {__fadd_rn(a.x, -b)}; }
__device__ __forceinline__ F1 operator-(float a, F1 b) { return {__fadd_rn(a, -b.x)}; }
__device__ __forceinline__ F1 operator+(M1 m, F1 c) { return fma1(m.a, m.b, c); }
__device__ __forceinline__ F1 operator+(F1 c, M1 m) { return fma1(m.a, m.b, c); }
__device__ __forceinline__ F1 operator-(M1 m, F1 c) { return fma1(m.a, m.b, neg1(c)); }
__device__ __forceinline__ F1 operator-(F1 c, M1 m) { return fma1(neg1(m.a), m.b, c); }
__device__ __forceinline__ F1 operator+(M1 m, float c) { return fma1(m.a, m.b, bc1(c)); }
__device__ __forceinline__ F1 operator+(float c, M1 m) { return fma1(m.a, m.b, bc1(c)); }
__device__ __forceinline__ F1 operator-(M1 m, float c) { return fma1(m.a, m.b, bc1(-c)); }
__device__ __forceinline__ F1 operator-(float c, M1 m) { return fma1(neg1(m.a), m.b, bc1(c)); }
__device__ __forceinline__ F1 operator+(M1 m, M1 n) { return fma1(n.a, n.b, F1(m)); }
__device__ __forceinline__ F1 operator-(M1 m, M1 n) { return fma1(neg1(n.a), n.b, F1(m)); }

// F2 arithmetic runs on the packed FP32 pipes of sm_100a (FADD2 / FMUL2 / FFMA2: one
// instruction for both envs), same contraction rules as F1; ptxas folds operand
// negation and uniform / immediate scalars into the packed instruction.
__device__ __forceinline__ F2 add2(F2 a, F2 b) {
  F2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// The rounded product as fma(a, b, −0): ptxas fuses a mul.rn.f32x2 into a following
// add.rn.f32x2 (it does not for the scalar .rn forms), which would round differently
// from F1.  The −0 addend is a __constant__ (a runtime value to ptxas), so the FFMA2
// is neither simplified back to a multiply nor fused; fma(a, b, −0) = round(a·b)
// including the sign of zero.
__constant__ float kNegZero = -0.0f;
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
  F2 d;
  const float z = kNegZero;
  asm("{.reg .b64 ra, rb, rz, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mov.b64 rz, {%6,%6};\n\tfma.rn.f32x2 rd, ra, rb, rz;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(z));
  return d;
}
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mov.b64 rc, {%6,%7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ F2 neg2(F2 a) { return {-a.x, -a.y}; }
__device__ __forceinline__ F2 bc2(float f) { return {f, f}; }
struct M2 {  // the product a*b, not yet rounded
  F2 a, b;
  __device__ __forceinline__ operator F2() const { return mul2(a, b); }
};
__device__ __forceinline__ M2 operator*(F2 a, F2 b) { return {a, b}; }
__device__ __forceinline__ M2 operator*(float a, F2 b) { return {bc2(a), b}; }
__device__ __forceinline__ M2 operator*(F2 a, float b) { return {a, bc2(b)}; }
__device__ __forceinline__ M2 operator*(M2 m, F2 b) { return {F2(m), b}; }
__device__ __forceinline__ M2 operator*(F2 a, M2 m) { return {a, F2(m)}; }
__device__ __forceinline__ M2 operator*(M2 m, float b) { return {F2(m), bc2(b)}; }
__device__ __forceinline__ M2 operator*(float a, M2 m) { return {bc2(a), F2(m)}; }
__device__ __forceinline__ M2 operator*(M2 m, M2 n) { return {F2(m), F2(n)}; }
__device__ __forceinline__ M2 operator-(M2 m) { return {neg2(m.a), m.b}; }
__device__ __forceinline__ F2 operator-(F2 a) { return neg2(a); }
__device__ __forceinline__ F2 operator+(F2 a, F2 b) { return add2(a, b); }
__device__ __forceinline__ F2 operator-(F2 a, F2 b) { return add2(a, neg2(b)); }
__device__ __forceinline__ F2 operator+(F2 a, float b) { return add2(a, bc2(b)); }
__device__ __forceinline__ F2 operator+(float a, F2 b) { return add2(bc2(a), b); }
__device__ __forceinline__ F2 operator-(F2 a, float b) { return add2(a, bc2(-b)); }
__device__ __forceinline__ F2 operator-(float a, F2 b) { return add2(bc2(a), neg2(b)); }
__device__ __forceinline__ F2 operator+(M2 m, F2 c) { return fma2(m.a, m.b, c); }
__device__ __forceinline__ F2 operator+(F2 c, M2 m) { return fma2(m.a, m.b, c); }
__device__ __forceinline__ F2 operator-(M2 m, F2 c) { return fma2(m.a, m.b, neg2(c)); }
__device__ __forceinline__ F2 operator-(F2 c, M2 m) { return fma2(neg2(m.a), m.b, c); }
__device__ __forceinline__ F2 operator+(M2 m, float c) { return fma2(m.a, m.b, bc2(c)); }
__device__ __forceinline__ F2 operator+(float c, M2 m) { return fma2(m.a, m.b, bc2(c)); }
__device__ __forceinline__ F2 operator-(M2 m, float c) { return fma2(m.a, m.b, bc2(-c)); }
__device__ __forceinline__ F2 operator-(float c, M2 m) { return fma2(neg2(m.a), m.b, bc2(c)); }
__device__ __forceinline__ F2 operator+(M2 m, M2 n) { return fma2(n.a, n.b, F2(m)); }
__device__ __forceinline__ F2 operator-(M2 m, M2 n) { return fma2(neg2(n.a), n.b, F2(m)); }

// ---- D1: one env per lane carrying (value, tangent): the forward-mode derivative
// (JVP) of the step (NEXT-4).  The value part rounds exactly like F1 (the same
// contraction pattern), so the JVP's primal output is brax_step's, bit for bit.
// Derivative conventions at the method's kinks (R35):
// min / max / clamp take the tangent of the selected argument (the first on ties),
// selects take the selected branch's tangent, comparisons use values.
// One MUFU instruction each: the .ftz forms skip the denormal-input rescaling that
// rsqrtf / __fdividef wrap around MUFU.RSQ / MUFU.RCP (4 extra instructions per call).
// For normal inputs the result is the same MUFU value (and a/b the same single-rounded
// product a·rcp(b)); the inputs here (squared norms, clamped ratios, effective masses,
// contact counts) are normal or exactly 0, which every call site guards.
__device__ __forceinline__ float rsqrt_mufu(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_mufu(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float div_mufu(float a, float b) { return __fmul_rn(a, rcp_mufu(b)); }

struct D1 { float v, t; };
__device__ __forceinline__ D1 d1mul(D1 a, D1 b) {
  return {__fmul_rn(a.v, b.v), __fmaf_rn(a.t, b.v, __fmul_rn(a.v, b.t))};
}
__device__ __forceinline__ D1 d1fma(D1 a, D1 b, D1 c) {
  return {__fmaf_rn(a.v, b.v, c.v), __fmaf_rn(a.t, b.v, __fmaf_rn(a.v, b.t, c.t))};
}
__device__ __forceinline__ D1 d1neg(D1 a) { return {-a.v, -a.t}; }
__device__ __forceinline__ D1 d1bc(float f) { return {f, 0.f}; }
struct MD1 {  // the product a*b, not yet rounded
  D1 a, b;
  __device__ __forceinline__ operator D1() const { return d1mul(a, b); }
};
__device__ __forceinline__ MD1 operator*(D1 a, D1 b) { return {a, b}; }
__device__ __forceinline__ MD1 operator*(float a, D1 b) { return {d1bc(a), b}; }
__device__ __forceinline__ MD1 operator*(D1 a, float b) { return {a, d1bc(b)}; }
__device__ __forceinline__ MD1 operator*(MD1 m, D1 b) { return {D1(m), b}; }
__device__ __forceinline__ MD1 operator*(D1 a, MD1 m) { return {a, D1(m)}; }
__device__ __forceinline__ MD1 operator*(MD1 m, float b) { return {D1(m), d1bc(b)}; }
__device__ __forceinline__ MD1 operator*(float a, MD1 m) { return {d1bc(a), D1(m)}; }
__device__ __forceinline__ MD1 operator*(MD1 m, MD1 n) { return {D1(m), D1(n)}; }
__device__ __forceinline__ MD1 operator-(MD1 m) { return {d1neg(m.a), m.b}; }
__device__ __forceinline__ D1 operator-(D1 a) { return d1neg(a); }
__device__ __forceinline__ D1 operator+(D1 a, D1 b) { return {__fadd_rn(a.v, b.v), __fadd_rn(a.t, b.t)}; }
__device__ __forceinline__ D1 operator-(D1 a, D1 b) { return {__fadd_rn(a.v, -b.v), __fadd_rn(a.t, -b.t)}; }
__device__ __forceinline__ D1 operator+(D1 a, float b) { return {__fadd_rn(a.v, b), a.t}; }
__device__ __forceinline__ D1 operator+(float a, D1 b) { return {__fadd_rn(a, b.v), b.t}; }
__device__ __forceinline__ D1 operator-(D1 a, float b) { return {__fadd_rn(a.v, -b), a.t}; }
__device__ __forceinline__ D1 operator-(float a, D1 b) { return {__fadd_rn(a, -b.v), -b.t}; }
__device__ __forceinline__ D1 operator+(MD1 m, D1 c) { return d1fma(m.a, m.b, c); }
__device__ __forceinline__ D1 operator+(D1 c, MD1 m) { return d1fma(m.a, m.b, c); }
__device__ __forceinline__ D1 operator-(MD1 m, D1 c) { return d1fma(m.a, m.b, d1neg(c)); }
__device__ __forceinline__ D1 operator-(D1 c, MD1 m) { return d1fma(d1neg(m.a), m.b, c); }
__device__ __forceinline__ D1 operator+(MD1 m, float c) { return d1fma(m.a, m.b, d1bc(c)); }
__device__ __forceinline__ D1 operator+(float c, MD1 m) { return d1fma(m.a, m.b, d1bc(c)); }
__device__ __forceinline__ D1 operator-(MD1 m, float c) { return d1fma(m.a, m.b, d1bc(-c)); }
__device__ __forceinline__ D1 operator-(float c, MD1 m) { return d1fma(d1neg(m.a), m.b, d1bc(c)); }
__device__ __forceinline__ D1 operator+(MD1 m, MD1 n) { return d1fma(n.a, n.b, D1(m)); }
__device__ __forceinline__ D1 operator-(MD1 m, MD1 n) { return d1fma(d1neg(n.a), n.b, D1(m)); }
__device__ __forceinline__ D1 vmin(D1 a, D1 b) { return {fminf(a.v, b.v), b.v < a.v ? b.t : a.t}; }
__device__ __forceinline__ D1 vmax(D1 a, D1 b) { return {fmaxf(a.v, b.v), b.v > a.v ? b.t : a.t}; }
__device__ __forceinline__ D1 vabs(D1 a) { return {fabsf(a.v), a.v < 0.f ? -a.t : a.t}; }
__device__ __forceinline__ D1 vrsqrt(D1 a) {  // d(a^-1/2) = −½ a^-3/2 da
  const float r = rsqrt_mufu(a.v);
  return {r, __fmul_rn(__fmul_rn(-0.5f, __fmul_rn(r, __fmul_rn(r, r))), a.t)};
}
__device__ __forceinline__ D1 vdiv(D1 a, D1 b) {  // d(a/b) = (da − q db)/b
  const float q = div_mufu(a.v, b.v);
  return {q, div_mufu(__fmaf_rn(-q, b.t, a.t), b.v)};
}
__device__ __forceinline__ D1 vcopysign(D1 a, D1 b) {
  return {copysignf(a.v, b.v), (signbit(a.v) != signbit(b.v)) ? -a.t : a.t};
}
__device__ __forceinline__ bool lt(D1 a, D1 b) { return a.v < b.v; }
__device__ __forceinline__ bool gt(D1 a, D1 b) { return a.v > b.v; }
__device__ __forceinline__ D1 sel(bool m, D1 a, D1 b) { return m ? a : b; }

__device__ __forceinline__ F1 vmin(F1 a, F1 b) { return {fminf(a.x, b.x)}; }
__device__ __forceinline__ F2 vmin(F2 a, F2 b) { return {fminf(a.x, b.x), fminf(a.y, b.y)}; }
__device__ __forceinline__ F1 vmax(F1 a, F1 b) { return {fmaxf(a.x, b.x)}; }
__device__ __forceinline__ F2 vmax(F2 a, F2 b) { return {fmaxf(a.x, b.x), fmaxf(a.y, b.y)}; }
__device__ __forceinline__ F1 vabs(F1 a) { return {fabsf(a.x)}; }
__device__ __forceinline__ F2 vabs(F2 a) { return {fabsf(a.x), fabsf(a.y)}; }
__device__ __forceinline__ F1 vrsqrt(F1 a) { return {rsqrt_mufu(a.x)}; }
__device__ __forceinline__ F2 vrsqrt(F2 a) { return {rsqrt_mufu(a.x), rsqrt_mufu(a.y)}; }
__device__ __forceinline__ F1 vdiv(F1 a, F1 b) { return {div_mufu(a.x, b.x)}; }
__device__ __forceinline__ F2 vdiv(F2 a, F2 b) { return {div_mufu(a.x, b.x), div_mufu(a.y, b.y)}; }
__device__ __forceinline__ F1 vcopysign(F1 a, F1 b) { return {copysignf(a.x, b.x)}; }
__device__ __forceinline__ F2 vcopysign(F2 a, F2 b) { return {copysignf(a.x, b.x), copysignf(a.y, b.y)}; }
__device__ __forceinline__ bool lt(F1 a, F1 b) { return a.x < b.x; }
__device__ __forceinline__ B2 lt(F2 a, F2 b) { return {a.x < b.x, a.y < b.y}; }
__device__ __forceinline__ bool gt(F1 a, F1 b) { return a.x > b.x; }
__device__ __forceinline__ B2 gt(F2 a, F2 b) { return {a.x > b.x, a.y > b.y}; }
__device__ __forceinline__ F1 sel(bool m, F1 a, F1 b) { return m ? a : b; }
__device__ __forceinline__ F2 sel(B2 m, F2 a, F2 b) { return {m.x ? a.x : b.x, m.y ? a.y : b.y}; }
__device__ __forceinline__ bool both(bool m, bool n) { return m && n; }
__device__ __forceinline__ B2 both(B2 m, B2 n) { return {m.x && n.x, m.y && n.y}; }
__device__ __forceinline__ bool any(bool m) { return m; }
__device__ __forceinline__ bool any(B2 m) { return m.x || m.y; }
__device__ __forceinline__ F1 as_count(bool m) { return {m ? 1.f : 0.f}; }
__device__ __forceinline__ F2 as_count(B2 m) { return {m.x ? 1.f : 0.f, m.y ? 1.f : 0.f}; }
template <class S> __device__ __forceinline__ S bc(float f);
template <> __device__ __forceinline__ F1 bc<F1>(float f) { return {f}; }
template <> __device__ __forceinline__ F2 bc<F2>(float f) { return {f, f}; }
template <> __device__ __forceinline__ D1 bc<D1>(float f) { return {f, 0.f}; }
template <class S> __device__ __forceinline__ S clampv(S x, float lo, float hi) {
  return vmin(vmax(x, bc<S>(lo)), bc<S>(hi));
}

template <class S> struct V3T { S x, y, z; };
template <class S> struct Q4T { S w, x, y, z; };
template <class S> __device__ __forceinline__ V3T<S> operator+(V3T<S> a, V3T<S> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class S> __device__ __forceinline__ V3T<S> operator-(V3T<S> a, V3T<S> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class S> __device__ __forceinline__ V3T<S> operator*(S s, V3T<S> a) { return {s * a.x, s * a.y, s * a.z}; }
template <class S> __device__ __forceinline__ V3T<S> scale(float s, V3T<S> a) { return {s * a.x, s * a.y, s * a.z}; }
// c + s·a with the products fused (one FMA per component)
template <class S> __device__ __forceinline__ V3T<S> axpy(float s, V3T<S> a, V3T<S> c) {
  return {s * a.x + c.x, s * a.y + c.y, s * a.z + c.z};
}
template <class S> __device__ __forceinline__ V3T<S> axpy(S s, V3T<S> a, V3T<S> c) {
  return {s * a.x + c.x, s * a.y + c.y, s * a.z + c.z};
}
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
  return atan2_f(x, sel(gt(c2, bc<S>(0.f)), S(c2 * vrsqrt(c2)), bc<S>(0.f)));
}

// Small-argument forms for the joint angles of the constrained (alignment) axes, whose
// values are small: odd Taylor polynomials, truncation ≤ 3e-10 (|x| ≤ 0.25) — exact to
// fp32 like the general forms above.  joint_f evaluates the general forms only when a
// lane of the warp is outside the range and selects per lane, so an env's result
// depends on its own state alone (bitwise the same under every launch plan).
template <class S> __device__ __forceinline__ S asin_small(S x) {  // |x| ≤ 0.25
  S s = x * x;
  S p = bc<S>(0.017352764423076924f);  // 231/13312
  p = p * s + 0.022372159090909091f;    // 63/2816
  p = p * s + 0.030381944444444444f;    // 35/1152
  p = p * s + 0.044642857142857144f;    // 5/112
  p = p * s + 0.075f;                   // 3/40
  p = p * s + 0.16666666666666666f;     // 1/6
  return S(x * s) * p + x;
}
template <class S> __device__ __forceinline__ S atan_small(S t) {  // |t| ≤ 0.25
  S s = t * t;
  S p = bc<S>(0.07692307692307693f);  // 1/13
  p = p * s + -0.09090909090909091f;   // −1/11
  p = p * s + 0.1111111111111111f;     // 1/9
  p = p * s + -0.14285714285714285f;   // −1/7
  p = p * s + 0.2f;                    // 1/5
  p = p * s + -0.3333333333333333f;    // −1/3
  return S(t * s) * p + t;
}
__device__ __forceinline__ bool allv(bool m) { return m; }
__device__ __forceinline__ bool allv(B2 m) { return m.x && m.y; }

// ---- shared-memory access for V = 1 or 2 envs per lane ---------------------------
// Records (device_tables.h): V = 1 — field f at words 4f..4f+3 of the env's record;
// V = 2 — one record per lane, both envs interleaved: field f at words 8f..8f+7 as
// (c0 env0, c0 env1, c1 env0, c1 env1 | c2 env0, c2 env1, c3 env0, c3 env1).
template <class S> struct Lanes;
template <> struct Lanes<F1> {
  static constexpr int V = 1, SL = 1, M = 4;  // layout id, words per lane slot, words per record field
  static constexpr int QS = kQS, JS = kJS, CS = kCS;
  static __device__ __forceinline__ V3T<F1> ld3(const float* p) {
    float4 a = *reinterpret_cast<const float4*>(p);
    return {{a.x}, {a.y}, {a.z}};
  }
  static __device__ __forceinline__ Q4T<F1> ldq(const float* p) {
    float4 a = *reinterpret_cast<const float4*>(p);
    return {{a.x}, {a.y}, {a.z}, {a.w}};
  }
  static __device__ __forceinline__ void st3(float* p, V3T<F1> v, F1 w = {0.f}) {
    *reinterpret_cast<float4*>(p) = make_float4(v.x.x, v.y.x, v.z.x, w.x);
  }
  static __device__ __forceinline__ void stq(float* p, Q4T<F1> q) {
    *reinterpret_cast<float4*>(p) = make_float4(q.w.x, q.x.x, q.y.x, q.z.x);
  }
  static __device__ __forceinline__ F1 ld(const float* p) { return {*p}; }  // per-env scalar arrays
  static __device__ __forceinline__ void st(float* p, F1 v) { *p = v.x; }
  static __device__ __forceinline__ F1 w4(const float* p) { return {p[3]}; }  // 4th word of field 0
  static __device__ __forceinline__ V3T<F1> ld3w(const float* p, F1& w) {
    float4 a = *reinterpret_cast<const float4*>(p);
    w = {a.w};
    return {{a.x}, {a.y}, {a.z}};
  }
};
template <> struct Lanes<F2> {
  static constexpr int V = 2, SL = 2, M = 8;
  static constexpr int QS = kQS2, JS = kJS2, CS = kCS2;
  static __device__ __forceinline__ V3T<F2> ld3(const float* p) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    return {{a.x, a.y}, {a.z, a.w}, {b.x, b.y}};
  }
  static __device__ __forceinline__ Q4T<F2> ldq(const float* p) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    return {{a.x, a.y}, {a.z, a.w}, {b.x, b.y}, {b.z, b.w}};
  }
  static __device__ __forceinline__ void st3(float* p, V3T<F2> v, F2 w = {0.f, 0.f}) {
    *reinterpret_cast<float4*>(p) = make_float4(v.x.x, v.x.y, v.y.x, v.y.y);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v.z.x, v.z.y, w.x, w.y);
  }
  static __device__ __forceinline__ void stq(float* p, Q4T<F2> q) {
    *reinterpret_cast<float4*>(p) = make_float4(q.w.x, q.w.y, q.x.x, q.x.y);
    *reinterpret_cast<float4*>(p + 4) = make_float4(q.y.x, q.y.y, q.z.x, q.z.y);
  }
  // per-env scalar arrays hold a lane's two envs in adjacent words
  static __device__ __forceinline__ F2 ld(const float* p) {
    float2 a = *reinterpret_cast<const float2*>(p);
    return {a.x, a.y};
  }
  static __device__ __forceinline__ void st(float* p, F2 v) { *reinterpret_cast<float2*>(p) = make_float2(v.x, v.y); }
  static __device__ __forceinline__ F2 w4(const float* p) {
    float2 a = *reinterpret_cast<const float2*>(p + 6);
    return {a.x, a.y};
  }
  static __device__ __forceinline__ V3T<F2> ld3w(const float* p, F2& w) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    w = {b.z, b.w};
    return {{a.x, a.y}, {a.z, a.w}, {b.x, b.y}};
  }
};

template <> struct Lanes<D1> {  // one env per lane; records hold (value, tangent) pairs like F2's env pairs
  static constexpr int V = 3, SL = 2, M = 8;
  static constexpr int QS = kQS2, JS = kJS2, CS = kCS2;
  static __device__ __forceinline__ V3T<D1> ld3(const float* p) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    return {{a.x, a.y}, {a.z, a.w}, {b.x, b.y}};
  }
  static __device__ __forceinline__ Q4T<D1> ldq(const float* p) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    return {{a.x, a.y}, {a.z, a.w}, {b.x, b.y}, {b.z, b.w}};
  }
  static __device__ __forceinline__ void st3(float* p, V3T<D1> v, D1 w = {0.f, 0.f}) {
    *reinterpret_cast<float4*>(p) = make_float4(v.x.v, v.x.t, v.y.v, v.y.t);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v.z.v, v.z.t, w.v, w.t);
  }
  static __device__ __forceinline__ void stq(float* p, Q4T<D1> q) {
    *reinterpret_cast<float4*>(p) = make_float4(q.w.v, q.w.t, q.x.v, q.x.t);
    *reinterpret_cast<float4*>(p + 4) = make_float4(q.y.v, q.y.t, q.z.v, q.z.t);
  }
  static __device__ __forceinline__ D1 ld(const float* p) {
    float2 a = *reinterpret_cast<const float2*>(p);
    return {a.x, a.y};
  }
  static __device__ __forceinline__ void st(float* p, D1 v) { *reinterpret_cast<float2*>(p) = make_float2(v.v, v.t); }
  static __device__ __forceinline__ D1 w4(const float* p) {
    float2 a = *reinterpret_cast<const float2*>(p + 6);
    return {a.x, a.y};
  }
  static __device__ __forceinline__ V3T<D1> ld3w(const float* p, D1& w) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    w = {b.z, b.w};
    return {{a.x, a.y}, {a.z, a.w}, {b.x, b.y}};
  }
};

// QP record of one (body, lane) in shared memory: pos | rot | vel | ang
template <class S> struct Row {
  float* p;  // = sQ + (b·L + lane slot) · Lanes<S>::QS
  static constexpr int M = Lanes<S>::M;
  __device__ __forceinline__ V3T<S> pos() const { return Lanes<S>::ld3(p); }
  __device__ __forceinline__ Q4T<S> rot() const { return Lanes<S>::ldq(p + M); }
  __device__ __forceinline__ V3T<S> vel() const { return Lanes<S>::ld3(p + 2 * M); }
  __device__ __forceinline__ V3T<S> ang() const { return Lanes<S>::ld3(p + 3 * M); }
  __device__ __forceinline__ void set_pos(V3T<S> v) const { Lanes<S>::st3(p, v); }
  __device__ __forceinline__ void set_rot(Q4T<S> q) const { Lanes<S>::stq(p + M, q); }
  __device__ __forceinline__ void set_vel(V3T<S> v) const { Lanes<S>::st3(p + 2 * M, v); }
  __device__ __forceinline__ void set_ang(V3T<S> v) const { Lanes<S>::st3(p + 3 * M, v); }
};

// ---- S2: kinematic integrator (R3, R21) -------------------------
// rotation part: q' = normalize(q + ½h (0, ω)⊗q) (ω already masked)
// (0, ω)⊗q written out without the products by the zero scalar part (same values)
template <class S> __device__ __forceinline__ Q4T<S> qmul_pure(V3T<S> a, Q4T<S> b) {
  return {-(a.x * b.x) - a.y * b.y - a.z * b.z, a.x * b.w + a.y * b.z - a.z * b.y,
          a.y * b.w - a.x * b.z + a.z * b.x, a.z * b.w + a.x * b.y - a.y * b.x};
}
template <class S> __device__ __forceinline__ Q4T<S> kin_rot(Q4T<S> q, V3T<S> w, float h) {
  Q4T<S> dq = qmul_pure(w, q);
  const float hh = 0.5f * h;
  q = Q4T<S>{q.w + hh * dq.w, q.x + hh * dq.x, q.y + hh * dq.y, q.z + hh * dq.z};
  S n2 = q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z;
  S inv = vrsqrt(n2);
  inv = inv * (1.5f - 0.5f * n2 * inv * inv);  // one Newton step: ≈ correctly rounded 1/√n2
  return Q4T<S>{q.w * inv, q.x * inv, q.y * inv, q.z * inv};
}
template <class S> __device__ __forceinline__ void kinematic(const DBody& bd, Row<S> r, float h) {
  V3T<S> v = r.vel();
  if (!(bd.flags & kFlagFreePos)) v = had(bd.mpos, v);
  r.set_pos(axpy(h, v, r.pos()));
  if (!bd.rot_frozen) {
    V3T<S> w = r.ang();
    if (!(bd.flags & kFlagFreeRot)) w = had(bd.mrot, w);
    r.set_rot(kin_rot(r.rot(), w, h));
  }
}

// ---- S3 + S4: joint spring/limits with its actuator (R5, R7-R12)
// Computed by joint_f from any row type with pos() / rot() / vel() / ang() (shared-memory
// records for the step, register rows for the adjoint's local derivatives) and an
// action accessor act(k) for action component k; returns F on the child, T on the
// child and T on the parent (already negated, as stored).
template <class S> struct JointOut { V3T<S> f, tc, tp; };
// kDof > 0 / kAct > -2: the joint's dof / actuator kind known at compile time (the
// specialised kernel variant's common class: hinge with a torque actuator), else read.
template <class S, class RowT, class ActF, int kDof = 0, int kAct = -2>
__device__ __forceinline__ JointOut<S> joint_f(const DJoint& Jm, const RowT& P, const RowT& C, ActF act) {
  // the parameter record, read with LDS.128 (struct fields at fixed float4 slots)
  const float4* J4 = reinterpret_cast<const float4*>(&Jm);
  const int4 h0 = *reinterpret_cast<const int4*>(&Jm), h1 = reinterpret_cast<const int4*>(&Jm)[1];
  const int dof = kDof > 0 ? kDof : h0.z, act_kind = kAct > -2 ? kAct : h0.w, act_offset = h1.x, flags = h1.y;
  const float4 op_k = J4[2], oc_cl = J4[3], jp = J4[4], jc = J4[5], lo_kl = J4[6], hi_ka = J4[7], ca_s = J4[8];
  const float lo[3] = {lo_kl.x, lo_kl.y, lo_kl.z}, hi[3] = {hi_ka.x, hi_ka.y, hi_ka.z};
  Q4T<S> qp = P.rot(), qc = C.rot();
  V3T<S> rp = rotate(qp, V3T<S>{bc<S>(op_k.x), bc<S>(op_k.y), bc<S>(op_k.z)});
  V3T<S> rc = rotate(qc, V3T<S>{bc<S>(oc_cl.x), bc<S>(oc_cl.y), bc<S>(oc_cl.z)});
  V3T<S> dx = (P.pos() - C.pos()) + (rp - rc);
  V3T<S> wp = P.ang(), wc = C.ang();
  V3T<S> f = scale(op_k.w, dx);
  if (!(flags & kJNoCl))
    f = axpy(oc_cl.w, cross_add(wp, rp, P.vel()) - cross_add(wc, rc, C.vel()), f);
  Q4T<S> fp = qmul(qp, Q4T<S>{bc<S>(jp.x), bc<S>(jp.y), bc<S>(jp.z), bc<S>(jp.w)});
  Q4T<S> fc = qmul(qc, Q4T<S>{bc<S>(jc.x), bc<S>(jc.y), bc<S>(jc.z), bc<S>(jc.w)});
  // q_r's canonicalisation to w >= 0 (R25) is not evaluated: every entry of R(q_r) below is a
  // sum of products of two components, which flipping all four signs leaves bit-identical
  Q4T<S> qr = qmul(qconj(fp), fc);
  S R02 = 2.f * (qr.x * qr.z + qr.w * qr.y);
  S R12 = 2.f * (qr.y * qr.z - qr.w * qr.x);
  S R22 = 1.f - 2.f * (qr.x * qr.x + qr.y * qr.y);
  S R01 = 2.f * (qr.x * qr.y - qr.w * qr.z);
  S R00 = 1.f - 2.f * (qr.y * qr.y + qr.z * qr.z);
  // θ1 and θ2: small-argument forms where every lane's argument is small (the
  // alignment errors of constrained axes), else the general forms, selected per lane
  const S x1 = clampv(R02, -1.f, 1.f);
  const auto small1 = gt(bc<S>(0.25f), vabs(x1));
  const auto small2 = both(gt(R00, bc<S>(0.f)), gt(S(0.25f * R00), vabs(R01)));
  S th[3] = {atan2_f(-R12, R22), asin_small(x1), atan_small(vdiv(-R01, R00))};
  if (__any_sync(__activemask(), !(allv(small1) && allv(small2)))) {
    th[1] = sel(small1, th[1], asin_f(x1));
    th[2] = sel(small2, th[2], atan2_f(-R01, R00));
  }
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
        S a = act(act_offset + i);
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
  S u = (tau[2] - tau[0] * R02) * vmin(S(ic * ic), bc<S>(100.f));
  V3T<S> tj{tau[0], u * R12 + t1 * R22, u * R22 - t1 * R12};
  V3T<S> twd = rotate(fp, tj);
  if (!(flags & kJNoCa)) twd = axpy(ca_s.x, wp - wc, twd);
  V3T<S> tc = cross_add(rc, f, twd);
  V3T<S> tp = cross_add(rp, f, twd);
  return JointOut<S>{f, tc, V3T<S>{-tp.x, -tp.y, -tp.z}};
}
// act: this lane's column of the block's actions sA[k][slot] (row stride E).
// out: this (joint, lane) record: F on child | T child | T parent.
template <class S, int kDof = 0, int kAct = -2>
__device__ __forceinline__ void joint(const DJoint& Jm, Row<S> P, Row<S> C, const float* act, int E, float* out) {
  auto actf = [&](int k) { return Lanes<S>::ld(act + k * E); };
  const JointOut<S> o = joint_f<S, Row<S>, decltype(actf), kDof, kAct>(Jm, P, C, actf);
  constexpr int M = Lanes<S>::M;
  Lanes<S>::st3(out, o.f);
  Lanes<S>::st3(out + M, o.tc);
  Lanes<S>::st3(out + 2 * M, o.tp);
}

// ---- NEXT-1 observation of one joint (R32): its free axes' angles θ_i (R7) and
// rates θ̇_i = b_i·ω_r, ω_r = R(q_p⊗J_p)ᵀ(ω_c − ω_p), b the dual basis of the rotation
// axes (as in joint()).  rows: obs row of this lane's first env; the second env's
// (S = F2) is `second` words further; angle i at word ang0 + i, rate i at rate0 + i.
template <class S> __device__ __forceinline__ void st_rows(float* p, int second, S v);
template <> __device__ __forceinline__ void st_rows<F1>(float* p, int, F1 v) { *p = v.x; }
template <> __device__ __forceinline__ void st_rows<F2>(float* p, int second, F2 v) {
  p[0] = v.x;
  p[second] = v.y;
}
template <class S>
__device__ __forceinline__ void joint_obs(const DJoint& Jm, Row<S> P, Row<S> C, float* rows, int second, int ang0,
                                          int rate0) {
  const float4* J4 = reinterpret_cast<const float4*>(&Jm);
  const int dof = reinterpret_cast<const int4*>(&Jm)->z;
  const float4 jp = J4[4], jc = J4[5];
  Q4T<S> fp = qmul(P.rot(), Q4T<S>{bc<S>(jp.x), bc<S>(jp.y), bc<S>(jp.z), bc<S>(jp.w)});
  Q4T<S> fc = qmul(C.rot(), Q4T<S>{bc<S>(jc.x), bc<S>(jc.y), bc<S>(jc.z), bc<S>(jc.w)});
  Q4T<S> qr = qmul(qconj(fp), fc);
  S sg = sel(lt(qr.w, bc<S>(0.f)), bc<S>(-1.f), bc<S>(1.f));
  qr = Q4T<S>{sg * qr.w, sg * qr.x, sg * qr.y, sg * qr.z};
  S R02 = 2.f * (qr.x * qr.z + qr.w * qr.y);
  S R12 = 2.f * (qr.y * qr.z - qr.w * qr.x);
  S R22 = 1.f - 2.f * (qr.x * qr.x + qr.y * qr.y);
  S R01 = 2.f * (qr.x * qr.y - qr.w * qr.z);
  S R00 = 1.f - 2.f * (qr.y * qr.y + qr.z * qr.z);
  S s1 = clampv(R02, -1.f, 1.f);
  S th[3] = {atan2_f(-R12, R22), asin_f(s1), atan2_f(-R01, R00)};
  S c2 = R12 * R12 + R22 * R22;
  S ic = sel(gt(c2, bc<S>(0.f)), vrsqrt(c2), bc<S>(0.f));   // 1 / cos θ1
  S c0 = sel(gt(c2, bc<S>(0.f)), R22 * ic, bc<S>(1.f));      // cos θ0
  S s0 = sel(gt(c2, bc<S>(0.f)), -(R12 * ic), bc<S>(0.f));   // sin θ0
  S c1 = c2 * ic;                                             // cos θ1
  S icg = c1 * vdiv(bc<S>(1.f), vmax(c2, bc<S>(0.01f)));      // cos θ1 / max(cos² θ1, 0.01)
  V3T<S> wr = rotate(qconj(fp), C.ang() - P.ang());
  S t = s1 * icg;
  S rate[3] = {wr.x + (s0 * t) * wr.y - (c0 * t) * wr.z, c0 * wr.y + s0 * wr.z, c0 * icg * wr.z - s0 * icg * wr.y};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (i < dof) {
      st_rows<S>(rows + ang0 + i, second, th[i]);
      st_rows<S>(rows + rate0 + i, second, rate[i]);
    }
  }
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
  c1 = axpy(s, d1, p1);
  c2 = axpy(t, d2, p2);
}

// ---- S5: contact slot, velocity-level impulse + Baumgarte (R13-R19)
// out: this (slot, lane) record: P, active | r_A×P | r_B×P; cnt: substeps active.
template <class S> struct ContactOut { V3T<S> P; S active; V3T<S> ta, tb; };
// Slot classes known at compile time (the specialised kernel variant): kCls = 1 / 2 / 3
// is a capsule end / sphere / box corner of an isotropic dynamic body, collider not
// offset, on a static plane collider at its body's origin, unrotated (the feet and
// torsos of the locomotion scenes); kCls = 0: everything read from the record.
constexpr int kCapsuleOnGroundFlags = kSZeroPa | kSZeroPb | kSIdentB | kSIsoA;
template <class S, class RowT, int kCls = 0>
__device__ __forceinline__ ContactOut<S> contact_f(const DSlot& SLm, const RowT& A, const RowT& B, float opl_e,
                                                   float beta_over_h, float mu) {
  // the parameter record, read with LDS.128 at its fixed float4 slots
  const float4* S4 = reinterpret_cast<const float4*>(&SLm);
  const int4 h0 = *reinterpret_cast<const int4*>(&SLm), h1 = reinterpret_cast<const int4*>(&SLm)[1];
  const int type = kCls == 1 ? 1 : kCls == 2 ? 0 : kCls == 3 ? 2 : h0.x, a_static = kCls ? 0 : h1.x,
            b_static = kCls ? 1 : h1.y;
  const int fl = kCls ? ((h1.z & kSIdentA) | kCapsuleOnGroundFlags) : h1.z;
  const float4 ca = S4[2], cb = S4[4], ells = S4[6];  // ca_pos|ra, cb_pos|rb, ell_a ellb 1/m_a 1/m_b
  const float ra = ca.w, rb = cb.w;
  Q4T<S> qa = A.rot(), qb = B.rot();
  V3T<S> xa = A.pos(), xb = B.pos();
  V3T<S> cB = (fl & kSZeroPb) ? xb : xb + rotate(qb, V3T<S>{bc<S>(cb.x), bc<S>(cb.y), bc<S>(cb.z)});
  Q4T<S> qB = qb;
  if (!(fl & kSIdentB)) {
    const float4 r = S4[5];
    qB = qmul(qb, Q4T<S>{bc<S>(r.x), bc<S>(r.y), bc<S>(r.z), bc<S>(r.w)});
  }
  const S zero = bc<S>(0.f);
  V3T<S> n, pt;
  S d;
  if (type <= 2) {  // sphere / capsule end / box corner vs plane: plane is B
    n = rotate_z(qB);
    // the A-side point x_A + rotate(q_A, pa_local) (DSlot::pa_local; a sphere at its body's origin: x_A)
    V3T<S> c = xa;
    if (kCls == 1 || kCls == 3 || (kCls == 0 && !(fl & kSZeroLa))) {
      const float4 l = S4[10];
      c = xa + rotate(qa, V3T<S>{bc<S>(l.x), bc<S>(l.y), bc<S>(l.z)});
    }
    if (type == 2) {
      d = -dot(c - cB, n);
      pt = c;
    } else {
      d = ra - dot(c - cB, n);
      pt = axpy(-ra, n, c);
    }
  } else {
    V3T<S> cA = (fl & kSZeroPa) ? xa : xa + rotate(qa, V3T<S>{bc<S>(ca.x), bc<S>(ca.y), bc<S>(ca.z)});
    Q4T<S> qA = qa;
    if (!(fl & kSIdentA)) {
      const float4 r = S4[3];
      qA = qmul(qa, Q4T<S>{bc<S>(r.x), bc<S>(r.y), bc<S>(r.z), bc<S>(r.w)});
    }
    V3T<S> pa = cA, pb = cB;
    if (type == 4) {  // sphere (A) – capsule (B)
      V3T<S> axb = rotate_z(qB);
      V3T<S> e0 = axpy(ells.y, axb, cB), e1 = axpy(-ells.y, axb, cB);
      V3T<S> seg = e0 - e1;
      if (ells.y > 0.f) pb = e1 + clampv(vdiv(dot(cA - e1, seg), dot(seg, seg)), 0.f, 1.f) * seg;
      else pb = e1;
    } else if (type == 5) {  // capsule – capsule
      V3T<S> axa = rotate_z(qA), axb = rotate_z(qB);
      seg_seg(axpy(ells.x, axa, cA), axpy(-ells.x, axa, cA), axpy(ells.y, axb, cB), axpy(-ells.y, axb, cB),
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
    pt = scale(0.5f, axpy(-ra, n, pa) + axpy(rb, n, pb));
  }
  auto pen = gt(d, zero);  // R16: strict d > 0
  // the impulse is evaluated for every env of a warp in which any env penetrates and
  // masked (no lane divergence, no merge moves; a non-penetrating env gets jn = 0,
  // hence P = 0); warps without a penetrating env skip it
  V3T<S> P{zero, zero, zero}, ta{zero, zero, zero}, tb{zero, zero, zero};
  S active = zero;
  if (__any_sync(__activemask(), any(pen))) {
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
  jn = sel(act, jn, zero);
  V3T<S> ut = u - un * n;
  S st2 = dot(ut, ut);
  auto sl = gt(st2, zero);  // R16: j_t = 0 when s_t = 0
  S ist = sel(sl, vrsqrt(st2), zero);
  S st = st2 * ist;
  V3T<S> th = ist * ut;
  S kt = sel(sl, eff(th), bc<S>(1.f));
  S jt = vmin(vdiv(st, kt), S(mu * jn));
  P = jn * n - jt * th;
  ta = cross(rA, P);
  if (kCls == 0) tb = cross(rB, P);  // the specialised classes' B side is static: r_B×P is never gathered
  active = sel(act, bc<S>(1.f), bc<S>(0.f));
  }
  return ContactOut<S>{P, active, ta, tb};
}
template <class S, int kCls = 0>
__device__ __forceinline__ void contact(const DSlot& SLm, Row<S> A, Row<S> B, float opl_e, float beta_over_h,
                                        float mu, float* out, S& cnt) {
  const ContactOut<S> o = contact_f<S, Row<S>, kCls>(SLm, A, B, opl_e, beta_over_h, mu);
  constexpr int M = Lanes<S>::M;
  Lanes<S>::st3(out, o.P, o.active);
  Lanes<S>::st3(out + M, o.ta);
  if (kCls == 0) Lanes<S>::st3(out + 2 * M, o.tb);  // a static B side's record field is never read
  cnt = cnt + o.active;
}


// ---- S6: per-body accumulation over the static incidence lists (fixed order) --
// e = (item << 4) | t with t = 4 (child / A side: sign +1) or 8 (parent / B side:
// sign −1); rec: this lane's record of the item; the torque vector is field t/4.
template <class S> struct Acc {
  V3T<S> F, T, dV, dW;
  S cnt;
  static constexpr int M = Lanes<S>::M;
  __device__ __forceinline__ Acc() {
    const S z = bc<S>(0.f);
    F = T = dV = dW = V3T<S>{z, z, z};
    cnt = z;
  }
  __device__ __forceinline__ void joint(const float* rec, int e) {
    const float sg = (e & 8) ? -1.f : 1.f;
    F = axpy(sg, Lanes<S>::ld3(rec), F);
    T = T + Lanes<S>::ld3(rec + (e & 15) * (M / 4));
  }
  __device__ __forceinline__ void slot(const float* rec, int e) {
    const float sg = (e & 8) ? -1.f : 1.f;
    S act;
    dV = axpy(sg, Lanes<S>::ld3w(rec, act), dV);  // P with its "active" word in the same loads
    dW = axpy(sg, Lanes<S>::ld3(rec + (e & 15) * (M / 4)), dW);
    cnt = cnt + act;
  }
  // the first entry of a list initialises the sums (no zero registers, one op less)
  __device__ __forceinline__ void joint_first(const float* rec, int e) {
    const float sg = (e & 8) ? -1.f : 1.f;
    F = scale(sg, Lanes<S>::ld3(rec));
    T = Lanes<S>::ld3(rec + (e & 15) * (M / 4));
  }
  __device__ __forceinline__ void slot_first(const float* rec, int e) {
    const float sg = (e & 8) ? -1.f : 1.f;
    dV = scale(sg, Lanes<S>::ld3w(rec, cnt));
    dW = scale(sg, Lanes<S>::ld3(rec + (e & 15) * (M / 4)));
  }
  // Gather of a whole incidence list (joints: jl[0..nj), slots: cl[0..nc)) in pairs:
  // a pair's list entries and records are all loaded before the first of them is
  // summed (one shared-memory round trip per chunk instead of one per entry; the sums
  // keep the list order, R29).  jrec / crec: this lane's record of joint / slot 0;
  // jstride / cstride: words between consecutive items' records.
  template <bool kSlot>
  __device__ __forceinline__ void add(const V3T<S>& a, const V3T<S>& b, S w, float sg) {
    if (kSlot) {
      dV = axpy(sg, a, dV);
      dW = axpy(sg, b, dW);
      cnt = cnt + w;
    } else {
      F = axpy(sg, a, F);
      T = T + b;
    }
  }
  template <bool kSlot>
  __device__ __forceinline__ void ld(const float* rec0, int stride, int e, V3T<S>& a, V3T<S>& b, S& w) {
    const float* rec = rec0 + (e >> 4) * stride;
    if (kSlot) a = Lanes<S>::ld3w(rec, w);
    else a = Lanes<S>::ld3(rec);
    b = Lanes<S>::ld3(rec + (e & 15) * (M / 4));
  }
  template <bool kSlot>
  __device__ __forceinline__ void gather(const int32_t* list, int n, const float* rec0, int stride) {
    V3T<S> a0, b0, a1, b1;
    S w0, w1;
    int e0 = list[0], e1 = list[n > 1 ? 1 : 0];
    ld<kSlot>(rec0, stride, e0, a0, b0, w0);
    ld<kSlot>(rec0, stride, e1, a1, b1, w1);
    const float s0 = (e0 & 8) ? -1.f : 1.f;
    if (kSlot) {
      dV = scale(s0, a0);
      dW = scale(s0, b0);
      cnt = w0;
    } else {
      F = scale(s0, a0);
      T = b0;
    }
    if (n > 1) add<kSlot>(a1, b1, w1, (e1 & 8) ? -1.f : 1.f);
    for (int k = 2; k < n; k += 2) {
      e0 = list[k];
      e1 = list[k + 1 < n ? k + 1 : k];
      ld<kSlot>(rec0, stride, e0, a0, b0, w0);
      ld<kSlot>(rec0, stride, e1, a1, b1, w1);
      add<kSlot>(a0, b0, w0, (e0 & 8) ? -1.f : 1.f);
      if (k + 1 < n) add<kSlot>(a1, b1, w1, (e1 & 8) ? -1.f : 1.f);
    }
  }
  // gather with the list lengths known at compile time (NJ joints, NC slots): every
  // entry, then every record is loaded before the sums (two shared-memory round trips
  // for the whole body); same operations and order as gather(), so the same bits
  template <int NJ, int NC>
  __device__ __forceinline__ void gather_fixed(const int32_t* jl, const int32_t* cl, const float* jrec0, int jstride,
                                               const float* crec0, int cstride) {
    int ej[NJ > 0 ? NJ : 1], ec[NC > 0 ? NC : 1];
#pragma unroll
    for (int k = 0; k < NJ; ++k) ej[k] = jl[k];
#pragma unroll
    for (int k = 0; k < NC; ++k) ec[k] = cl[k];
    V3T<S> fa[NJ > 0 ? NJ : 1], ta[NJ > 0 ? NJ : 1], pa[NC > 0 ? NC : 1], ra[NC > 0 ? NC : 1];
    S wa[NC > 0 ? NC : 1];
#pragma unroll
    for (int k = 0; k < NJ; ++k) {
      const float* rec = jrec0 + (ej[k] >> 4) * jstride;
      fa[k] = Lanes<S>::ld3(rec);
      ta[k] = Lanes<S>::ld3(rec + (ej[k] & 15) * (M / 4));
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const float* rec = crec0 + (ec[k] >> 4) * cstride;
      pa[k] = Lanes<S>::ld3w(rec, wa[k]);
      ra[k] = Lanes<S>::ld3(rec + (ec[k] & 15) * (M / 4));
    }
    if (NJ > 0) {
      F = scale((ej[0] & 8) ? -1.f : 1.f, fa[0]);
      T = ta[0];
    } else {
      zero_joints();
    }
#pragma unroll
    for (int k = 1; k < NJ; ++k) {
      F = axpy((ej[k] & 8) ? -1.f : 1.f, fa[k], F);
      T = T + ta[k];
    }
    if (NC > 0) {
      const float sg = (ec[0] & 8) ? -1.f : 1.f;
      dV = scale(sg, pa[0]);
      dW = scale(sg, ra[0]);
      cnt = wa[0];
    } else {
      zero_slots();
    }
#pragma unroll
    for (int k = 1; k < NC; ++k) {
      const float sg = (ec[k] & 8) ? -1.f : 1.f;
      dV = axpy(sg, pa[k], dV);
      dW = axpy(sg, ra[k], dW);
      cnt = cnt + wa[k];
    }
  }
  struct NoInit {};
  __device__ __forceinline__ explicit Acc(NoInit) {}
  __device__ __forceinline__ void zero_joints() {
    const S z = bc<S>(0.f);
    F = T = V3T<S>{z, z, z};
  }
  __device__ __forceinline__ void zero_slots() {
    const S z = bc<S>(0.f);
    dV = dW = V3T<S>{z, z, z};
    cnt = z;
  }
};

// ---- S7 + S8: potential integrator then collision integrator (R14, R21),
// fused (kin = true) with the next substep's S2 kinematic integrator of the same
// body: same arithmetic as kinematic(), with v and ω still in registers.
// co (env epilogue with contact observations, last substep of a step): this body's
// and lane's [6][E] slot for the collision integrator's velocity change; else NULL.
// kFree: an isotropic body with no frozen axis, known at compile time (the specialised
// kernel variant's common body class), else the flags are read.
template <class S, bool kFree = false>
__device__ __forceinline__ void integrate(const DBody& bd, Row<S> r, const Acc<S>& acc, float h, const float* g,
                                          bool kin, float* co, int E, bool co_acc = false) {
  const bool iso = kFree || (bd.flags & kFlagIso), fp = kFree || (bd.flags & kFlagFreePos),
             fr = kFree || (bd.flags & kFlagFreeRot);
  Q4T<S> q = r.rot();
  V3T<S> v = axpy(h, axpy(bd.inv_mass, acc.F, bc3<S>(g)), r.vel());
  V3T<S> w = axpy(h, iw(q, bd.inv_inertia, iso, acc.T), r.ang());
  if (!fp) v = had(bd.mpos, v);
  if (!fr) w = had(bd.mrot, w);
  const V3T<S> v_pre = v, w_pre = w;
  auto hit = gt(acc.cnt, bc<S>(0.f));
  if (any(hit)) {
    S ic = sel(hit, vdiv(bc<S>(1.f), acc.cnt), bc<S>(0.f));  // R14: mean over the body's active contacts
    const S mic = bd.inv_mass * ic;
    v = axpy(mic, acc.dV, v);
    w = axpy(ic, iw(q, bd.inv_inertia, iso, acc.dW), w);
    if (!fp) v = had(bd.mpos, v);
    if (!fr) w = had(bd.mrot, w);
  }
  r.set_vel(v);
  r.set_ang(w);
  if (co) {  // collision integrator's velocity change: after − before (R32); co_acc: summed over substeps
    const V3T<S> dv = v - v_pre, dw = w - w_pre;
    const S d[6] = {dv.x, dv.y, dv.z, dw.x, dw.y, dw.z};
#pragma unroll
    for (int k = 0; k < 6; ++k) Lanes<S>::st(co + k * E, co_acc ? Lanes<S>::ld(co + k * E) + d[k] : d[k]);
  }
  if (kin) {  // next substep's kinematic integrator (v, ω already masked)
    r.set_pos(axpy(h, v, r.pos()));
    if (kFree || !bd.rot_frozen) r.set_rot(kin_rot(q, w, h));
  }
}

// Word of (body b, env slot env, field f, component c) in the QP records for layout
// V (1: F1; 2: F2, envs el and el + LG share lane el's record; 3: D1, value half of
// the env's value/tangent record) with LG records per body.
template <int V> __device__ __forceinline__ int qword(int b, int env, int f, int c, int LG) {
  if (V == 1) return (b * LG + env) * kQS + 4 * f + c;
  const int h = (V == 2 && env >= LG) ? 1 : 0, el = env - h * LG;
  return (b * LG + el) * kQS2 + 8 * f + 4 * (c >> 1) + 2 * (c & 1) + h;
}
// Position of env slot `env` in a per-env row (actions, contact counts, contact Δv):
// V = 2 keeps a lane's two envs (el, el + LG) adjacent; V = 3 (D1) the value word of
// the env's (value, tangent) pair.
template <int V> __device__ __forceinline__ int eslot(int env, int LG) {
  if (V == 1) return env;
  if (V == 3) return 2 * env;
  const int h = env >= LG ? 1 : 0;
  return 2 * (env - h * LG) + h;
}

// ---- S1 / S9: staging of one QP field [n][B][K] <-> record field f.
// One env row (B·K contiguous floats) per warp iteration, lanes along the row:
// coalesced, and no integer division (K is a compile-time constant).
template <int K, bool kLoad, int V>
__device__ __forceinline__ void stage(const float* gin, float* gout, float* sQ, int f, int64_t e0, int nvalid, int B,
                                      int E) {
  const int row_len = B * K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int env = warp; env < nvalid; env += nw) {
    const int64_t g0 = (e0 + env) * row_len;
    for (int k = lane; k < row_len; k += 32) {
      const int b = k / K, c = k - (k / K) * K;
      float* s = sQ + qword<V>(b, env, f, c, V == 2 ? E / 2 : E);
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
// waits until the bulk stores have READ shared memory (the CTA may then exit; the
// global writes complete with the grid, as for any store)
__device__ __forceinline__ void tma_store_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// waits until the bulk stores have WRITTEN global memory (a later launch may read them
// before this grid completes: the lean kernel's granule protocol)
__device__ __forceinline__ void tma_store_commit_wait_all() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;" ::: "memory");
}
// orders this thread's generic-proxy accesses with async-proxy (TMA) accesses to global memory
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Staging area layout (words): the block's contiguous global chunks
// pos [E][B][3] | rot [E][B][4] | vel [E][B][3] | ang [E][B][3].  Full blocks only.
template <int V> __device__ __forceinline__ void stg_to_records(const float* stg, float* sQ, int B, int E) {
  const float* sp = stg;
  const float* sr = stg + E * B * 3;
  const float* sv = sr + E * B * 4;
  const float* sw = sv + E * B * 3;
  // consecutive threads take consecutive envs of one body: the record stores are
  // bank-conflict free (record stride 20 / 36 words)
  if (V == 1) {
    for (int t = threadIdx.x; t < E * B; t += blockDim.x) {
      const int b = t / E, env = t - b * E, i = env * B + b;
      float4* r = reinterpret_cast<float4*>(sQ + (b * E + env) * kQS);
      r[0] = make_float4(sp[3 * i], sp[3 * i + 1], sp[3 * i + 2], 0.f);
      r[1] = make_float4(sr[4 * i], sr[4 * i + 1], sr[4 * i + 2], sr[4 * i + 3]);
      r[2] = make_float4(sv[3 * i], sv[3 * i + 1], sv[3 * i + 2], 0.f);
      r[3] = make_float4(sw[3 * i], sw[3 * i + 1], sw[3 * i + 2], 0.f);
    }
  } else {
    const int LG = E >> 1;
    for (int t = threadIdx.x; t < LG * B; t += blockDim.x) {
      const int b = t / LG, el = t - b * LG, i = el * B + b;
      const int i0 = i, i1 = i + LG * B;  // staging rows of envs el and el + LG
      float4* r = reinterpret_cast<float4*>(sQ + (b * LG + el) * kQS2);
      r[0] = make_float4(sp[3 * i0], sp[3 * i1], sp[3 * i0 + 1], sp[3 * i1 + 1]);
      r[1] = make_float4(sp[3 * i0 + 2], sp[3 * i1 + 2], 0.f, 0.f);
      r[2] = make_float4(sr[4 * i0], sr[4 * i1], sr[4 * i0 + 1], sr[4 * i1 + 1]);
      r[3] = make_float4(sr[4 * i0 + 2], sr[4 * i1 + 2], sr[4 * i0 + 3], sr[4 * i1 + 3]);
      r[4] = make_float4(sv[3 * i0], sv[3 * i1], sv[3 * i0 + 1], sv[3 * i1 + 1]);
      r[5] = make_float4(sv[3 * i0 + 2], sv[3 * i1 + 2], 0.f, 0.f);
      r[6] = make_float4(sw[3 * i0], sw[3 * i1], sw[3 * i0 + 1], sw[3 * i1 + 1]);
      r[7] = make_float4(sw[3 * i0 + 2], sw[3 * i1 + 2], 0.f, 0.f);
    }
  }
}
template <int V> __device__ __forceinline__ void records_to_stg(const float* sQ, float* stg, int B, int E) {
  float* sp = stg;
  float* sr = stg + E * B * 3;
  float* sv = sr + E * B * 4;
  float* sw = sv + E * B * 3;
  if (V == 1) {
    for (int t = threadIdx.x; t < E * B; t += blockDim.x) {
      const int b = t / E, env = t - b * E, i = env * B + b;
      const float4* r = reinterpret_cast<const float4*>(sQ + (b * E + env) * kQS);
      float4 p = r[0], q = r[1], v = r[2], w = r[3];
      sp[3 * i] = p.x; sp[3 * i + 1] = p.y; sp[3 * i + 2] = p.z;
      sr[4 * i] = q.x; sr[4 * i + 1] = q.y; sr[4 * i + 2] = q.z; sr[4 * i + 3] = q.w;
      sv[3 * i] = v.x; sv[3 * i + 1] = v.y; sv[3 * i + 2] = v.z;
      sw[3 * i] = w.x; sw[3 * i + 1] = w.y; sw[3 * i + 2] = w.z;
    }
  } else {
    const int LG = E >> 1;
    for (int t = threadIdx.x; t < LG * B; t += blockDim.x) {
      const int b = t / LG, el = t - b * LG, i = el * B + b;
      const int i0 = i, i1 = i + LG * B;
      const float4* r = reinterpret_cast<const float4*>(sQ + (b * LG + el) * kQS2);
      float4 p0 = r[0], p1 = r[1], q0 = r[2], q1 = r[3], v0 = r[4], v1 = r[5], w0 = r[6], w1 = r[7];
      sp[3 * i0] = p0.x; sp[3 * i0 + 1] = p0.z; sp[3 * i0 + 2] = p1.x;
      sp[3 * i1] = p0.y; sp[3 * i1 + 1] = p0.w; sp[3 * i1 + 2] = p1.y;
      sr[4 * i0] = q0.x; sr[4 * i0 + 1] = q0.z; sr[4 * i0 + 2] = q1.x; sr[4 * i0 + 3] = q1.z;
      sr[4 * i1] = q0.y; sr[4 * i1 + 1] = q0.w; sr[4 * i1 + 2] = q1.y; sr[4 * i1 + 3] = q1.w;
      sv[3 * i0] = v0.x; sv[3 * i0 + 1] = v0.z; sv[3 * i0 + 2] = v1.x;
      sv[3 * i1] = v0.y; sv[3 * i1 + 1] = v0.w; sv[3 * i1 + 2] = v1.y;
      sw[3 * i0] = w0.x; sw[3 * i0 + 1] = w0.z; sw[3 * i0 + 2] = w1.x;
      sw[3 * i1] = w0.y; sw[3 * i1 + 1] = w0.w; sw[3 * i1 + 2] = w1.y;
    }
  }
}

// S1: the block's E envs' QP -> shared memory (env slots past the batch end get identity state)
template <int V>
__device__ __forceinline__ void load_block(const StepArgs& a, float* sQ, int B, int E, int64_t e0, int nvalid) {
  if (nvalid < E) {
    const int nrec = B * (E / V), RS = V == 2 ? kQS2 : kQS;
    for (int i = threadIdx.x; i < nrec; i += blockDim.x) {
      float4* p = reinterpret_cast<float4*>(sQ + i * RS);
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      if (V == 1) {
        p[0] = z; p[1] = make_float4(1.f, 0.f, 0.f, 0.f); p[2] = z; p[3] = z;
      } else {
        p[0] = z; p[1] = z; p[2] = make_float4(1.f, 1.f, 0.f, 0.f); p[3] = z;
        p[4] = z; p[5] = z; p[6] = z; p[7] = z;
      }
    }
    __syncthreads();
  }
  stage<3, true, V>(a.pos_in, nullptr, sQ, 0, e0, nvalid, B, E);
  stage<4, true, V>(a.rot_in, nullptr, sQ, 1, e0, nvalid, B, E);
  stage<3, true, V>(a.vel_in, nullptr, sQ, 2, e0, nvalid, B, E);
  stage<3, true, V>(a.ang_in, nullptr, sQ, 3, e0, nvalid, B, E);
}

// S1 (per step): this step's action [n][A] -> sA[k][eslot(env)] (one env row per warp iteration)
template <int V>
__device__ __forceinline__ void load_actions(const StepArgs& a, float* sA, int A, int E, int LG, int64_t step,
                                             int64_t e0, int nvalid) {
  if (A <= 0) return;
  const int RW = V == 1 ? LG : 2 * LG;
  const float* act = a.actions + (step * a.n_envs + e0) * A;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int env = warp; env < nvalid; env += nw) {
    const int slot = eslot<V>(env, LG);
    for (int k = lane; k < A; k += 32) sA[k * RW + slot] = __ldg(act + env * A + k);
  }
}

// S9: status bits and contact counts (after a barrier)
template <int V>
__device__ __forceinline__ void block_extras(const StepArgs& a, const float* sQ, const float* sCnt, uint32_t* sStat,
                                             int B, int C, int E, int LG, int64_t e0, int nvalid) {
  const int RW = V == 1 ? LG : 2 * LG;
  auto word_bits = [](float v) -> uint32_t { return isfinite(v) ? (fabsf(v) > 1e6f ? 2u : 0u) : 1u; };
  if (a.status) {
    if (V == 1) {
      for (int i = threadIdx.x; i < B * E; i += blockDim.x) {
        const float* p = sQ + i * kQS;
        uint32_t bits = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (k == 3 || k == 11 || k == 15) continue;  // padding words
          bits |= word_bits(p[k]);
        }
        if (bits) atomicOr(&sStat[i % E], bits);
      }
    } else if (V == 3) {  // value words of the (value, tangent) records
      for (int i = threadIdx.x; i < B * E; i += blockDim.x) {
        const float* p = sQ + i * kQS2;
        uint32_t bits = 0;
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          if (k == 6 || k == 22 || k == 30) continue;
          bits |= word_bits(p[k]);
        }
        if (bits) atomicOr(&sStat[i % E], bits);
      }
    } else {
      const int LG = E >> 1;
      for (int i = threadIdx.x; i < B * LG; i += blockDim.x) {
        const float* p = sQ + i * kQS2;
        uint32_t bits0 = 0, bits1 = 0;
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          if (k == 6 || k == 22 || k == 30) continue;  // padding words (pos, vel, ang 4th component)
          bits0 |= word_bits(p[k]);
          bits1 |= word_bits(p[k + 1]);
        }
        const int el = i % LG;
        if (bits0) atomicOr(&sStat[el], bits0);
        if (bits1) atomicOr(&sStat[el + LG], bits1);
      }
    }
  }
  if (a.contact_active) {
    for (int i = threadIdx.x; i < nvalid * C; i += blockDim.x) {
      int env = i / C, c = i - env * C;
      a.contact_active[(e0 + env) * C + c] = uint8_t(sCnt[c * RW + eslot<V>(env, LG)]);
    }
  }
}

// ---- JVP staging (lane type D1, layout 3): value and tangent of every QP word,
// per-row loads / stores (a NULL tangent pointer reads as zero / is not written).
template <int K, bool kLoad>
__device__ __forceinline__ void stage_d(const float* gin, const float* dgin, float* gout, float* dgout, float* sQ,
                                        int f, int64_t e0, int nvalid, int B, int LG) {
  const int row_len = B * K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int env = warp; env < nvalid; env += nw) {
    const int64_t g0 = (e0 + env) * row_len;
    for (int k = lane; k < row_len; k += 32) {
      const int b = k / K, c = k - (k / K) * K;
      float* s = sQ + qword<3>(b, env, f, c, LG);
      if (kLoad) {
        s[0] = __ldg(gin + g0 + k);
        s[1] = dgin ? __ldg(dgin + g0 + k) : 0.f;
      } else {
        gout[g0 + k] = s[0];
        if (dgout) dgout[g0 + k] = s[1];
      }
    }
  }
}
__device__ __forceinline__ void load_block_d(const StepArgs& a, float* sQ, int B, int E, int64_t e0, int nvalid) {
  if (nvalid < E) {  // identity state, zero tangent
    for (int i = threadIdx.x; i < B * E; i += blockDim.x) {
      float4* p = reinterpret_cast<float4*>(sQ + i * kQS2);
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      p[0] = z; p[1] = z; p[2] = make_float4(1.f, 0.f, 0.f, 0.f); p[3] = z;
      p[4] = z; p[5] = z; p[6] = z; p[7] = z;
    }
    __syncthreads();
  }
  stage_d<3, true>(a.pos_in, a.dpos_in, nullptr, nullptr, sQ, 0, e0, nvalid, B, E);
  stage_d<4, true>(a.rot_in, a.drot_in, nullptr, nullptr, sQ, 1, e0, nvalid, B, E);
  stage_d<3, true>(a.vel_in, a.dvel_in, nullptr, nullptr, sQ, 2, e0, nvalid, B, E);
  stage_d<3, true>(a.ang_in, a.dang_in, nullptr, nullptr, sQ, 3, e0, nvalid, B, E);
}
__device__ __forceinline__ void store_block_d(const StepArgs& a, float* sQ, int B, int E, int64_t e0, int nvalid) {
  stage_d<3, false>(nullptr, nullptr, a.pos_out, a.dpos_out, sQ, 0, e0, nvalid, B, E);
  stage_d<4, false>(nullptr, nullptr, a.rot_out, a.drot_out, sQ, 1, e0, nvalid, B, E);
  stage_d<3, false>(nullptr, nullptr, a.vel_out, a.dvel_out, sQ, 2, e0, nvalid, B, E);
  stage_d<3, false>(nullptr, nullptr, a.ang_out, a.dang_out, sQ, 3, e0, nvalid, B, E);
}
// this step's action value and tangent -> sA[k][2·env + {0, 1}]
__device__ __forceinline__ void load_actions_d(const StepArgs& a, float* sA, int A, int E, int64_t step, int64_t e0,
                                               int nvalid) {
  if (A <= 0) return;
  const int64_t off = (step * a.n_envs + e0) * A;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int env = warp; env < nvalid; env += nw)
    for (int k = lane; k < A; k += 32) {
      sA[k * 2 * E + 2 * env] = __ldg(a.actions + off + env * A + k);
      sA[k * 2 * E + 2 * env + 1] = a.dactions ? __ldg(a.dactions + off + env * A + k) : 0.f;
    }
}

// S9 fallback (ragged tail / unaligned): per-row stores of the QP
template <int V> __device__ __forceinline__ void store_block(const StepArgs& a, float* sQ, int B, int E, int64_t e0,
                                                             int nvalid) {
  stage<3, false, V>(nullptr, a.pos_out, sQ, 0, e0, nvalid, B, E);
  stage<4, false, V>(nullptr, a.rot_out, sQ, 1, e0, nvalid, B, E);
  stage<3, false, V>(nullptr, a.vel_out, sQ, 2, e0, nvalid, B, E);
  stage<3, false, V>(nullptr, a.ang_out, sQ, 3, e0, nvalid, B, E);
}

}  // namespace dev
}  // namespace brax
