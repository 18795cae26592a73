// device_rng.cuh — Philox4x32-10 (Salmon et al., SC'11) for the reset noise of
// brax_reset and of the env epilogue's auto-reset (R34).
#pragma once
#include <stdint.h>

namespace brax {
namespace dev {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k.x += W0; k.y += W1; }
    uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__device__ __forceinline__ float u_pm1(uint32_t x) {  // (x >> 8)·2⁻²⁴·2 − 1, exact in fp32
  return float(x >> 8) * (2.0f / 16777216.0f) - 1.0f;
}

// Reset state of body b (default_qp + noise) for the Philox counter
// (env, b, field, episode), key = seed; writes x[3], q[4], v[3], w[3].
__device__ __forceinline__ void reset_body(const float* dqp, const float* masks, int B, int b, uint32_t env,
                                           uint32_t episode, uint2 key, float sv, float sw, float* x, float* q,
                                           float* v, float* w) {
  const float* m = masks + 7 * b;
  for (int k = 0; k < 3; ++k) { v[k] = 0.f; w[k] = 0.f; }
  if (m[6] == 0.f) {
    uint4 xv = philox4x32_10(make_uint4(env, uint32_t(b), 0u, episode), key);
    uint4 xw = philox4x32_10(make_uint4(env, uint32_t(b), 1u, episode), key);
    uint32_t rv[3] = {xv.x, xv.y, xv.z}, rw[3] = {xw.x, xw.y, xw.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v[k] = __fadd_rn(v[k], __fmul_rn(m[k], __fmul_rn(sv, u_pm1(rv[k]))));
      w[k] = __fadd_rn(w[k], __fmul_rn(m[3 + k], __fmul_rn(sw, u_pm1(rw[k]))));
    }
  }
  for (int k = 0; k < 3; ++k) x[k] = dqp[3 * b + k];
  for (int k = 0; k < 4; ++k) q[k] = dqp[3 * B + 4 * b + k];
}

// Goal-task marker placement (R36): x = x̄_T + range ⊙ u(env, T, field, episode);
// field 2 at a reset of episode k, 2 + steps' at a hit (steps' ≥ 1: steps after the step).
__device__ __forceinline__ void place_target(const float* dqp, int tb, const float* range, uint32_t env,
                                             uint32_t field, uint32_t episode, uint2 key, float* x) {
  const uint4 r = philox4x32_10(make_uint4(env, uint32_t(tb), field, episode), key);
  const uint32_t rr[3] = {r.x, r.y, r.z};
#pragma unroll
  for (int k = 0; k < 3; ++k) x[k] = __fadd_rn(dqp[3 * tb + k], __fmul_rn(range[k], u_pm1(rr[k])));
}

}  // namespace dev
}  // namespace brax
