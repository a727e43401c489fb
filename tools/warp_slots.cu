// Which hardware warp slots (%warpid) do the warps of a 256-thread CTA get when 3 CTAs share an SM (sm_100a)?
// The scheduler (sub-partition) of a slot is %warpid % 4; roles that must not share an FP64 pipe are assigned from it.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 3) k(int *out, int rounds) {
  extern __shared__ double sm[];
  unsigned wid, smid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if ((threadIdx.x & 31) == 0) {
    int *o = out + (blockIdx.x * 8 + (threadIdx.x >> 5)) * 2;
    o[0] = smid, o[1] = wid;
  }
  // stay resident a while so all 3 CTAs of an SM coexist
  long long t0 = clock64();
  while (clock64() - t0 < 200000) {}
  sm[threadIdx.x] = 0;
}
int main() {
  const int grid = 148 * 3;
  int *out;
  cudaMallocManaged(&out, grid * 8 * 2 * sizeof(int));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 72000);
  k<<<grid, 256, 72000>>>(out, 1);
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  int hist[8][4] = {};
  for (int b = 0; b < grid; ++b) {
    if (b < 9 || out[b * 16] == 0) {
      printf("cta %3d sm %3d warpids:", b, out[b * 16]);
      for (int w = 0; w < 8; ++w) printf(" %2d", out[(b * 8 + w) * 2 + 1]);
      printf("\n");
    }
    for (int w = 0; w < 8; ++w) hist[w][out[(b * 8 + w) * 2 + 1] & 3]++;
  }
  for (int w = 0; w < 8; ++w) printf("warp %d: slot%%4 histogram %d %d %d %d\n", w, hist[w][0], hist[w][1], hist[w][2], hist[w][3]);
  return 0;
}
