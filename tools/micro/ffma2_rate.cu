// Issue-rate microbenchmark: FFMA vs FFMA2 (packed f32x2, sm_100a) with 8
// independent chains per thread, 8 warps per SMSP.  Prints warp-instructions per
// cycle per SM for each form.
#include <cstdio>
#include <cuda_runtime.h>
struct F2 { float x, y; };
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 d;
  asm volatile("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tmov.b64 rc, {%6,%7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
constexpr int kIters = 4096, kChains = 8;
__global__ void k1(float* out, float b, float c, long long* cyc) {
  float a[kChains];
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < kChains; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < kChains; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k2(float* out, float b, float c, float d, long long* cyc) {
  F2 a[kChains];
  F2 bb{b, d}, cc{c, b};
  for (int i = 0; i < kChains; ++i) a[i] = F2{float(threadIdx.x + i), float(i)};
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = fma2(a[i], bb, cc);
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < kChains; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  for (int warps : {4, 8, 16, 32}) {
    for (int form = 1; form <= 2; ++form) {
      if (form == 1) k1<<<148, warps * 32>>>(out, 1.0001f, 0.5f, cyc);
      else k2<<<148, warps * 32>>>(out, 1.0001f, 0.5f, 0.999f, cyc);
      cudaDeviceSynchronize();
      if (form == 1) k1<<<148, warps * 32>>>(out, 1.0001f, 0.5f, cyc);
      else k2<<<148, warps * 32>>>(out, 1.0001f, 0.5f, 0.999f, cyc);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double c = double(h[0]);
      double inst = double(warps) * kIters * kChains;
      printf("{\"form\": \"%s\", \"warps_per_sm\": %d, \"warp_inst_per_cycle_per_sm\": %.3f, \"fp32_lane_flops_per_cycle_per_sm\": %.1f}\n",
             form == 1 ? "FFMA" : "FFMA2", warps, inst / c, inst / c * 32 * 2 * form);
    }
  }
  return 0;
}
