// How the CTA scheduler spreads a one-wave grid over the SMs: 512 blocks of 160
// threads with 33 KB of dynamic shared memory and 96 registers (the ant 8192 lean
// launch shape: at most 4 resident per SM), each spinning ~20 us; histogram of
// blocks per SM (%smid).  Also the 96-register / 4-warp shape (5 per SM possible).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __maxnreg__(96) spin(unsigned* smid_out, long long ns) {
  extern __shared__ float sm[];
  unsigned id;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) smid_out[blockIdx.x] = id;
  sm[threadIdx.x] = float(t);
}

static void run(int blocks, int threads, int smem) {
  unsigned* d;
  cudaMalloc(&d, blocks * 4);
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  spin<<<blocks, threads, smem>>>(d, 20000);
  cudaDeviceSynchronize();
  unsigned h[4096];
  cudaMemcpy(h, d, blocks * 4, cudaMemcpyDeviceToHost);
  int cnt[256] = {0}, hist[16] = {0};
  for (int i = 0; i < blocks; ++i) cnt[h[i] & 255]++;
  int used = 0;
  for (int s = 0; s < 148; ++s) { hist[cnt[s] < 15 ? cnt[s] : 15]++; used += cnt[s] > 0; }
  printf("blocks %d threads %d smem %d: SMs used %d; SMs holding k blocks:", blocks, threads, smem, used);
  for (int k = 0; k < 16; ++k) if (hist[k]) printf(" %d:%d", k, hist[k]);
  printf("\n");
  cudaFree(d);
}

int main() {
  run(512, 160, 33152);  // ant 8192 lean: 4 per SM by registers and shared memory
  run(512, 128, 33152);  // 4 warps: 5 per SM by registers, 6 by shared memory
  run(512, 128, 20000);
  run(444, 160, 33152);
  run(592, 160, 33152);
  return 0;
}
