// reset.cu — brax_reset: broadcast default_qp and add velocity
// noise drawn from Philox4x32-10 (Salmon et al., SC'11), keyed by the seed and
// counted by (env, body, field, 0); for
// brax_env_reset of a goal task also the marker's episode-0 placement (R36).
#include <cuda_runtime.h>
#include <stdint.h>

#include "system.h"

#include "device_rng.cuh"

namespace brax {
namespace {

__global__ void brax_reset_kernel(float* pos, float* rot, float* vel, float* ang, const float* dqp,
                                  const float* masks, int B, int64_t n, int64_t env_offset, uint2 key, float sv,
                                  float sw, int target, float rx, float ry, float rz) {
  int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * B) return;
  int64_t e = t / B;
  int b = int(t - e * B);
  float x[3], q[4], v[3], w[3];
  dev::reset_body(dqp, masks, B, b, uint32_t(env_offset + e), 0u, key, sv, sw, x, q, v, w);
  if (b == target) {  // goal task (R36): the episode-0 marker placement
    const float range[3] = {rx, ry, rz};
    dev::place_target(dqp, b, range, uint32_t(env_offset + e), 2u, 0u, key, x);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    pos[t * 3 + k] = x[k];
    vel[t * 3 + k] = v[k];
    ang[t * 3 + k] = w[k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) rot[t * 4 + k] = q[k];
}

}  // namespace

cudaError_t launch_reset(const System& sys, float* pos, float* rot, float* vel, float* ang, int64_t n,
                         uint64_t seed, float vel_noise, float ang_noise, cudaStream_t stream, int64_t env_offset,
                         bool goal) {
  if (n <= 0) return cudaSuccess;
  note_other_launch(sys, stream);
  const int B = sys.hd.B;
  int64_t total = n * B;
  unsigned blocks = unsigned((total + 255) / 256);
  uint2 key = make_uint2(uint32_t(seed & 0xffffffffu), uint32_t(seed >> 32));
  const DTask& T = sys.hd.task;
  const bool g = goal && T.has_goal;
  brax_reset_kernel<<<blocks, 256, 0, stream>>>(pos, rot, vel, ang, sys.d_default_qp, sys.d_masks, B, n,
                                                env_offset, key, vel_noise, ang_noise, g ? T.target : -1,
                                                T.range[0], T.range[1], T.range[2]);
  return cudaGetLastError();
}

}  // namespace brax
