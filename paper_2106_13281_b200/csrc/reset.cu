// reset.cu — brax_reset: broadcast default_qp and add velocity
// noise drawn from Philox4x32-10 (Salmon et al., SC'11), keyed by the seed and
// counted by (env, body, field, 0).
#include <cuda_runtime.h>
#include <stdint.h>

#include "system.h"

namespace brax {
namespace {

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

__global__ void brax_reset_kernel(float* pos, float* rot, float* vel, float* ang, const float* dqp,
                                  const float* masks, int B, int64_t n, uint2 key, float sv, float sw) {
  int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * B) return;
  int64_t e = t / B;
  int b = int(t - e * B);
  const float* m = masks + 7 * b;
  float v[3] = {0.f, 0.f, 0.f}, w[3] = {0.f, 0.f, 0.f};
  if (m[6] == 0.f) {
    uint4 xv = philox4x32_10(make_uint4(uint32_t(e), uint32_t(b), 0u, 0u), key);
    uint4 xw = philox4x32_10(make_uint4(uint32_t(e), uint32_t(b), 1u, 0u), key);
    uint32_t rv[3] = {xv.x, xv.y, xv.z}, rw[3] = {xw.x, xw.y, xw.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v[k] += m[k] * (sv * u_pm1(rv[k]));
      w[k] += m[3 + k] * (sw * u_pm1(rw[k]));
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    pos[t * 3 + k] = dqp[3 * b + k];
    vel[t * 3 + k] = v[k];
    ang[t * 3 + k] = w[k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) rot[t * 4 + k] = dqp[3 * B + 4 * b + k];
}

}  // namespace

cudaError_t launch_reset(const System& sys, float* pos, float* rot, float* vel, float* ang, int64_t n,
                         uint64_t seed, float vel_noise, float ang_noise, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int B = sys.hd.B;
  int64_t total = n * B;
  unsigned blocks = unsigned((total + 255) / 256);
  uint2 key = make_uint2(uint32_t(seed & 0xffffffffu), uint32_t(seed >> 32));
  brax_reset_kernel<<<blocks, 256, 0, stream>>>(pos, rot, vel, ang, sys.d_default_qp, sys.d_masks, B, n, key,
                                                vel_noise, ang_noise);
  return cudaGetLastError();
}

}  // namespace brax
