// DMMA throughput vs warps per SM and independent chains per warp (B200).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double *out, int iters) {
  double acc[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) t += acc[i][0] + acc[i][1];
  if (t == 1.2345) out[0] = t;
}
template <int CH>
void run(int warps_per_sm, double *out) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int tpb = 32 * (warps_per_sm < 8 ? warps_per_sm : 8);
  int blocks = sms * (warps_per_sm * 32 / tpb);
  int iters = 4096 / CH * 64;
  k<CH><<<blocks, tpb>>>(out, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<CH><<<blocks, tpb>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 512.0 * CH * iters * blocks * (tpb / 32);
  printf("chains=%2d warps/SM=%2d : %6.1f TF/s\n", CH, warps_per_sm, fl / ms / 1e9);
}
int main() {
  double *o; cudaMalloc(&o, 8);
  for (int w : {4, 8, 12, 16, 32}) { run<1>(w, o); run<2>(w, o); run<4>(w, o); run<8>(w, o); run<16>(w, o); }
  return 0;
}
