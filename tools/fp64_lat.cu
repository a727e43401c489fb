// Dependent-issue latencies of the FP64 building blocks of the potrf pivot chain on B200 (sm_100a):
// DFMA, DMUL, MUFU.RSQ64H (+ Newton), 64-bit SHFL, DMMA m8n8k4 (accumulator chain), LDS.64, mbarrier hop.
// One warp, clock64 around N dependent ops.   nvcc -arch=sm_100a -O3 -o fp64_lat fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
#define N 512
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__global__ void lat(double *out, long long *t, double a, double b) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = a; sm[lane + 32] = b;
  __syncwarp();
  double x = a + lane;
  long long t0, t1;
  // DFMA
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = fma(x, b, a);
  t1 = clock64(); t[0] = t1 - t0;
  // DMUL
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = __dmul_rn(x, b);
  t1 = clock64(); t[1] = t1 - t0;
  // rsqrt.approx.f64
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x));
  t1 = clock64(); t[2] = t1 - t0;
  // shfl 64-bit
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64(); t[3] = t1 - t0;
  // DMMA accumulator chain
  double c[2] = {x, a};
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) dmma(c, a, b);
  t1 = clock64(); t[4] = t1 - t0;
  // DMMA with A operand dependent on previous result
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) { double d2[2] = {0.0, 0.0}; dmma(d2, c[0], b); c[0] = d2[0]; c[1] = d2[1]; }
  t1 = clock64(); t[5] = t1 - t0;
  // LDS.64 pointer chase
  int idx = lane;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) { double v = ((volatile double *)sm)[idx]; idx = (idx + (int)v) & 31; }
  t1 = clock64(); t[6] = t1 - t0;
  // 2 independent DMMA chains
  double c2[2] = {b, a};
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) { dmma(c, a, b); dmma(c2, b, a); }
  t1 = clock64(); t[7] = t1 - t0;
  // 4 independent DFMA chains
  double y0 = a, y1 = b, y2 = a + 1, y3 = b + 1;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) { y0 = fma(y0, b, a); y1 = fma(y1, b, a); y2 = fma(y2, b, a); y3 = fma(y3, b, a); }
  t1 = clock64(); t[8] = t1 - t0;
  // IEEE sqrt + div
  t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) x = __ddiv_rn(1.0, __dsqrt_rn(x + 2.0));
  t1 = clock64(); t[9] = t1 - t0;
  out[lane] = x + c[0] + c[1] + idx + c2[0] + c2[1] + y0 + y1 + y2 + y3;
}
// mbarrier hop: warp 0 arrives, warp 1 waits, ping-pong
__global__ void hop(long long *t) {
  __shared__ unsigned long long bar[2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned b0 = (unsigned)__cvta_generic_to_shared(&bar[0]), b1 = (unsigned)__cvta_generic_to_shared(&bar[1]);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b1));
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) {
    unsigned mine = w == 0 ? b0 : b1, other = w == 0 ? b1 : b0;
    if (w == 0) {
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mine) : "memory");
      asm volatile("{\n .reg .pred p;\nW1_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W1_%=;\n}\n" ::"r"(other), "r"(i & 1) : "memory");
    } else {
      asm volatile("{\n .reg .pred p;\nW2_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W2_%=;\n}\n" ::"r"(other), "r"(i & 1) : "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mine) : "memory");
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) t[0] = t1 - t0;
}
int main() {
  double *out; long long *t;
  cudaMalloc(&out, 32 * 8); cudaMallocManaged(&t, 16 * 8);
  for (int rep = 0; rep < 2; ++rep) { lat<<<1, 32>>>(out, t, 1.0000001, 0.9999999); cudaDeviceSynchronize(); }
  const char *nm[] = {"DFMA", "DMUL", "MUFU.RSQ64H", "SHFL64", "DMMA acc-chain", "DMMA A-dep chain", "LDS.64 chase", "2x DMMA chains (per pair)", "4x DFMA chains (per 4)", "dsqrt_rn+ddiv_rn"};
  for (int i = 0; i < 10; ++i) printf("%-28s %.1f clk/op\n", nm[i], (double)t[i] / N);
  hop<<<1, 64>>>(t); cudaDeviceSynchronize();
  printf("mbarrier round trip (2 hops)  %.1f clk\n", (double)t[0] / 256);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
