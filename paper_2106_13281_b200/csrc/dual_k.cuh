// dual_k.cuh — DK<K>: a value with K tangents, the lane type of the reverse kernel's
// local derivatives (vjp.cu): one evaluation of an item's code yields K columns of
// its local Jacobian.  Same rounding pattern and kink conventions as D1
// (step_device.cuh, R35): products are lazy and contract into an FMA where
// the source writes `a*b + c`; min / max / clamp / select take the selected
// argument's tangents (the first on ties); comparisons use values.
#pragma once
#include "step_device.cuh"

namespace brax {
namespace dev {

template <int K> struct DK {
  float v;
  float t[K];
};

template <int K> __device__ __forceinline__ DK<K> dkbc(float f) {
  DK<K> r;
  r.v = f;
#pragma unroll
  for (int k = 0; k < K; ++k) r.t[k] = 0.f;
  return r;
}
template <int K> __device__ __forceinline__ DK<K> dkneg(DK<K> a) {
  a.v = -a.v;
#pragma unroll
  for (int k = 0; k < K; ++k) a.t[k] = -a.t[k];
  return a;
}
template <int K> __device__ __forceinline__ DK<K> dkmul(DK<K> a, DK<K> b) {
  DK<K> r;
  r.v = __fmul_rn(a.v, b.v);
#pragma unroll
  for (int k = 0; k < K; ++k) r.t[k] = __fmaf_rn(a.t[k], b.v, __fmul_rn(a.v, b.t[k]));
  return r;
}
template <int K> __device__ __forceinline__ DK<K> dkfma(DK<K> a, DK<K> b, DK<K> c) {
  DK<K> r;
  r.v = __fmaf_rn(a.v, b.v, c.v);
#pragma unroll
  for (int k = 0; k < K; ++k) r.t[k] = __fmaf_rn(a.t[k], b.v, __fmaf_rn(a.v, b.t[k], c.t[k]));
  return r;
}
template <int K> __device__ __forceinline__ DK<K> dkadd(DK<K> a, DK<K> b) {
  DK<K> r;
  r.v = __fadd_rn(a.v, b.v);
#pragma unroll
  for (int k = 0; k < K; ++k) r.t[k] = __fadd_rn(a.t[k], b.t[k]);
  return r;
}

template <int K> struct MDK {  // the product a*b, not yet rounded
  DK<K> a, b;
  __device__ __forceinline__ operator DK<K>() const { return dkmul(a, b); }
};
template <int K> __device__ __forceinline__ MDK<K> operator*(DK<K> a, DK<K> b) { return {a, b}; }
template <int K> __device__ __forceinline__ MDK<K> operator*(float a, DK<K> b) { return {dkbc<K>(a), b}; }
template <int K> __device__ __forceinline__ MDK<K> operator*(DK<K> a, float b) { return {a, dkbc<K>(b)}; }
template <int K> __device__ __forceinline__ MDK<K> operator*(MDK<K> m, DK<K> b) { return {DK<K>(m), b}; }
template <int K> __device__ __forceinline__ MDK<K> operator*(DK<K> a, MDK<K> m) { return {a, DK<K>(m)}; }
template <int K> __device__ __forceinline__ MDK<K> operator*(MDK<K> m, float b) { return {DK<K>(m), dkbc<K>(b)}; }
template <int K> __device__ __forceinline__ MDK<K> operator*(float a, MDK<K> m) { return {dkbc<K>(a), DK<K>(m)}; }
template <int K> __device__ __forceinline__ MDK<K> operator*(MDK<K> m, MDK<K> n) { return {DK<K>(m), DK<K>(n)}; }
template <int K> __device__ __forceinline__ MDK<K> operator-(MDK<K> m) { return {dkneg(m.a), m.b}; }
template <int K> __device__ __forceinline__ DK<K> operator-(DK<K> a) { return dkneg(a); }
template <int K> __device__ __forceinline__ DK<K> operator+(DK<K> a, DK<K> b) { return dkadd(a, b); }
template <int K> __device__ __forceinline__ DK<K> operator-(DK<K> a, DK<K> b) { return dkadd(a, dkneg(b)); }
template <int K> __device__ __forceinline__ DK<K> operator+(DK<K> a, float b) {
  a.v = __fadd_rn(a.v, b);
  return a;
}
template <int K> __device__ __forceinline__ DK<K> operator+(float a, DK<K> b) {
  b.v = __fadd_rn(a, b.v);
  return b;
}
template <int K> __device__ __forceinline__ DK<K> operator-(DK<K> a, float b) {
  a.v = __fadd_rn(a.v, -b);
  return a;
}
template <int K> __device__ __forceinline__ DK<K> operator-(float a, DK<K> b) { return dkneg(b) + a; }
template <int K> __device__ __forceinline__ DK<K> operator+(MDK<K> m, DK<K> c) { return dkfma(m.a, m.b, c); }
template <int K> __device__ __forceinline__ DK<K> operator+(DK<K> c, MDK<K> m) { return dkfma(m.a, m.b, c); }
template <int K> __device__ __forceinline__ DK<K> operator-(MDK<K> m, DK<K> c) { return dkfma(m.a, m.b, dkneg(c)); }
template <int K> __device__ __forceinline__ DK<K> operator-(DK<K> c, MDK<K> m) { return dkfma(dkneg(m.a), m.b, c); }
template <int K> __device__ __forceinline__ DK<K> operator+(MDK<K> m, float c) { return dkfma(m.a, m.b, dkbc<K>(c)); }
template <int K> __device__ __forceinline__ DK<K> operator+(float c, MDK<K> m) { return dkfma(m.a, m.b, dkbc<K>(c)); }
template <int K> __device__ __forceinline__ DK<K> operator-(MDK<K> m, float c) { return dkfma(m.a, m.b, dkbc<K>(-c)); }
template <int K> __device__ __forceinline__ DK<K> operator-(float c, MDK<K> m) {
  return dkfma(dkneg(m.a), m.b, dkbc<K>(c));
}
template <int K> __device__ __forceinline__ DK<K> operator+(MDK<K> m, MDK<K> n) { return dkfma(n.a, n.b, DK<K>(m)); }
template <int K> __device__ __forceinline__ DK<K> operator-(MDK<K> m, MDK<K> n) {
  return dkfma(dkneg(n.a), n.b, DK<K>(m));
}

template <int K> __device__ __forceinline__ DK<K> vmin(DK<K> a, DK<K> b) {
  DK<K> r = b.v < a.v ? b : a;
  r.v = fminf(a.v, b.v);
  return r;
}
template <int K> __device__ __forceinline__ DK<K> vmax(DK<K> a, DK<K> b) {
  DK<K> r = b.v > a.v ? b : a;
  r.v = fmaxf(a.v, b.v);
  return r;
}
template <int K> __device__ __forceinline__ DK<K> vabs(DK<K> a) {
  DK<K> r = a.v < 0.f ? dkneg(a) : a;
  r.v = fabsf(a.v);
  return r;
}
template <int K> __device__ __forceinline__ DK<K> vrsqrt(DK<K> a) {  // d(a^-1/2) = −½ a^-3/2 da
  const float r = rsqrt_mufu(a.v);
  const float d = __fmul_rn(-0.5f, __fmul_rn(r, __fmul_rn(r, r)));
  DK<K> o;
  o.v = r;
#pragma unroll
  for (int k = 0; k < K; ++k) o.t[k] = __fmul_rn(d, a.t[k]);
  return o;
}
template <int K> __device__ __forceinline__ DK<K> vdiv(DK<K> a, DK<K> b) {  // d(a/b) = (da − q db)/b
  DK<K> o;
  o.v = div_mufu(a.v, b.v);
#pragma unroll
  for (int k = 0; k < K; ++k) o.t[k] = div_mufu(__fmaf_rn(-o.v, b.t[k], a.t[k]), b.v);
  return o;
}
template <int K> __device__ __forceinline__ DK<K> vcopysign(DK<K> a, DK<K> b) {
  DK<K> r = (signbit(a.v) != signbit(b.v)) ? dkneg(a) : a;
  r.v = copysignf(a.v, b.v);
  return r;
}
template <int K> __device__ __forceinline__ bool lt(DK<K> a, DK<K> b) { return a.v < b.v; }
template <int K> __device__ __forceinline__ bool gt(DK<K> a, DK<K> b) { return a.v > b.v; }
template <int K> __device__ __forceinline__ DK<K> sel(bool m, DK<K> a, DK<K> b) { return m ? a : b; }
template <> __device__ __forceinline__ DK<2> bc<DK<2>>(float f) { return dkbc<2>(f); }
template <> __device__ __forceinline__ DK<4> bc<DK<4>>(float f) { return dkbc<4>(f); }
template <> __device__ __forceinline__ DK<8> bc<DK<8>>(float f) { return dkbc<8>(f); }

}  // namespace dev
}  // namespace brax
