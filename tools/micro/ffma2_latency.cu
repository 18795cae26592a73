// Dependent-chain latency of FFMA vs FFMA2 (fma.rn.f32x2) on one warp: cycles per
// link of a 4096-long chain.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2_latency.cu
#include <cstdio>
__global__ void chain1(float* out, float a, float b, long long* cyc) {
  float x = threadIdx.x * 1e-3f;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) x = __fmaf_rn(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain2(float* out, float a, float b, long long* cyc) {
  float x = threadIdx.x * 1e-3f, y = x + 1.f;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) {
    asm volatile("{.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%0,%1};\n\tmov.b64 rb, {%2,%2};\n\tmov.b64 rc, {%3,%3};\n\t"
                 "fma.rn.f32x2 ra, ra, rb, rc;\n\tmov.b64 {%0,%1}, ra;}"
                 : "+f"(x), "+f"(y) : "f"(a), "f"(b));
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + y;
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
}
__global__ void chainlds(float* out, long long* cyc) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < 4096; ++i) p = s[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
}
__global__ void chainmufu(float* out, float a, long long* cyc) {
  float x = 1.f + threadIdx.x * 1e-3f;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(x));
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
}
__global__ void chains2r(float* out, long long* cyc) {
  unsigned acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) {
    unsigned v;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(v));
    acc = acc * 3u + v + i;
    asm volatile("" : "+r"(acc));
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
}
struct P { int v[64]; };
__global__ void chainldc(float* out, const __grid_constant__ P p, long long* cyc) {
  int x = (int)out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) {
    x = p.v[(x + i) & 63] & 63;
    asm volatile("" : "+r"(x));
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
}
int main() {
  float* o; long long* c; long long h[6]; P pp; for (int i = 0; i < 64; ++i) pp.v[i] = (i * 7 + 1) & 63;
  cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  for (int r = 0; r < 2; ++r) {
    chain1<<<1, 32>>>(o, 0.999f, 1e-3f, c);
    chain2<<<1, 32>>>(o, 0.999f, 1e-3f, c);
    chainlds<<<1, 32>>>(o, c);
    chainmufu<<<1, 32>>>(o, 0.5f, c);
    chains2r<<<1, 32>>>(o, c);
    chainldc<<<1, 32>>>(o, pp, c);
  }
  cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("{\"ffma_dep_cyc\": %.2f, \"ffma2_dep_cyc\": %.2f, \"lds_dep_cyc\": %.2f, \"mufu_rsq_dep_cyc\": %.2f, \"s2r_loop_cyc\": %.2f, \"ldc_indexed_dep_cyc\": %.2f}\n",
         h[0] / 4096.0, h[1] / 4096.0, h[2] / 4096.0, h[3] / 4096.0, h[4] / 1024.0, h[5] / 1024.0);
  return 0;
}
