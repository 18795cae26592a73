// diff.cu — reverse-mode cotangent of one step from forward-mode columns (NEXT-4):
// g_in[e][j] = Σ_o (∂out_o/∂in_j)·g_out[e][o], the column ∂out/∂in_j being the JVP
// (step.cu, lane type D1) along the unit tangent of input coordinate j.  Exact
// (no finite differences), O(13B + A) step launches per call: the fused adjoint
// kernel is the next step.
#include <cuda_runtime.h>
#include <stdint.h>

#include "system.h"

namespace brax {
namespace {

// coordinate j of (pos [B][3] | rot [B][4] | vel [B][3] | ang [B][3] | action [A]) -> (field, offset)
__device__ __forceinline__ void coord(int j, int B, int& field, int& off) {
  const int w[4] = {3, 4, 3, 3};
  for (field = 0; field < 4; ++field) {
    if (j < w[field] * B) {
      off = j;
      return;
    }
    j -= w[field] * B;
  }
  off = j;  // field 4: action index
}

__global__ void set_unit_kernel(float* pos, float* rot, float* vel, float* ang, float* act, int64_t n, int B, int A,
                                int j, float value) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n || j < 0) return;
  int f, off;
  coord(j, B, f, off);
  float* base[5] = {pos, rot, vel, ang, act};
  const int w[5] = {3, 4, 3, 3, 1};
  const int64_t stride = f < 4 ? int64_t(w[f]) * B : A;
  base[f][e * stride + off] = value;
}

__global__ void dot_column_kernel(const float* dpos, const float* drot, const float* dvel, const float* dang,
                                  const float* gpos, const float* grot, const float* gvel, const float* gang,
                                  float* opos, float* orot, float* ovel, float* oang, float* oact, int64_t n, int B,
                                  int A, int j) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const float* d[4] = {dpos, drot, dvel, dang};
  const float* g[4] = {gpos, grot, gvel, gang};
  const int w[4] = {3, 4, 3, 3};
  float s = 0.f;
  for (int f = 0; f < 4; ++f) {
    if (!g[f]) continue;  // a NULL cotangent member is zero
    const int64_t m = int64_t(w[f]) * B;
    for (int64_t k = 0; k < m; ++k) s = __fmaf_rn(d[f][e * m + k], g[f][e * m + k], s);
  }
  int f, off;
  coord(j, B, f, off);
  float* o[5] = {opos, orot, ovel, oang, oact};
  const int64_t stride = f < 4 ? int64_t(w[f]) * B : A;
  if (o[f]) o[f][e * stride + off] = s;
}

}  // namespace

cudaError_t launch_step_vjp(const System& sys, const StepArgs& primal, const float* const g_out[4],
                            float* const g_in[4], float* g_action, cudaStream_t stream) {
  const int64_t n = primal.n_envs;
  if (n <= 0) return cudaSuccess;
  note_other_launch(sys, stream);
  const int B = sys.hd.B, A = sys.hd.A;
  const int64_t qf = n * B * 13, K = int64_t(13) * B + A;
  float* buf = nullptr;
  const size_t words = size_t(2 * qf + qf + n * A);  // din, dout, primal out, daction
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), words * 4, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(buf, 0, words * 4, stream);
  float* din[4];
  float* dout[4];
  float* pout[4];
  float* p = buf;
  const int64_t sz[4] = {n * B * 3, n * B * 4, n * B * 3, n * B * 3};
  for (int k = 0; k < 4; ++k) { din[k] = p; p += sz[k]; }
  for (int k = 0; k < 4; ++k) { dout[k] = p; p += sz[k]; }
  for (int k = 0; k < 4; ++k) { pout[k] = p; p += sz[k]; }
  float* da = A > 0 ? p : nullptr;
  StepArgs a = primal;
  a.pos_out = pout[0];
  a.rot_out = pout[1];
  a.vel_out = pout[2];
  a.ang_out = pout[3];
  a.dpos_in = din[0];
  a.drot_in = din[1];
  a.dvel_in = din[2];
  a.dang_in = din[3];
  a.dactions = da;
  a.dpos_out = dout[0];
  a.drot_out = dout[1];
  a.dvel_out = dout[2];
  a.dang_out = dout[3];
  const unsigned blocks = unsigned((n + 127) / 128);
  for (int64_t j = 0; j < K && e == cudaSuccess; ++j) {
    set_unit_kernel<<<blocks, 128, 0, stream>>>(din[0], din[1], din[2], din[3], da, n, B, A, int(j - 1), 0.f);
    set_unit_kernel<<<blocks, 128, 0, stream>>>(din[0], din[1], din[2], din[3], da, n, B, A, int(j), 1.f);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = launch_step_jvp(sys, a, stream);
    if (e == cudaSuccess) {
      dot_column_kernel<<<blocks, 128, 0, stream>>>(dout[0], dout[1], dout[2], dout[3], g_out[0], g_out[1], g_out[2],
                                                    g_out[3], g_in[0], g_in[1], g_in[2], g_in[3], g_action, n, B, A,
                                                    int(j));
      e = cudaGetLastError();
    }
  }
  cudaError_t f = cudaFreeAsync(buf, stream);
  return e != cudaSuccess ? e : f;
}

}  // namespace brax
