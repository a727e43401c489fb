// FP64 peak microbenchmark for B200 (sm_100a): DFMA pipe vs DMMA (mma.sync m8n8k4 f64).
// Prints GFLOP/s for each; used to fix the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = s, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += a[i];
  if (t == 12345.0) out[0] = t;
}

__global__ void dmma_kernel(double *out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
      }
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += acc[i][0] + acc[i][1];
  if (t == 12345.0) out[0] = t;
}

__global__ void copy_kernel(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    int iters = 4000;
    dfma_kernel<<<blocks, tpb>>>(out, 10, 1.0000001);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, tpb>>>(out, iters, 1.0000001);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * tpb;
    printf("DFMA tpb=%d blocks=%d: %.1f GFLOP/s\n", tpb, blocks, flops / ms / 1e6);
  }
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (1024 / tpb);
    int iters = 2000;
    dmma_kernel<<<blocks, tpb>>>(out, 10);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, tpb>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * 4 * (double)iters * blocks * (tpb / 32);
    printf("DMMA tpb=%d blocks=%d: %.1f GFLOP/s\n", tpb, blocks, flops / ms / 1e6);
  }
  size_t n = (size_t)1 << 28;  // 4 GiB per buffer as double2? 2^28 * 16 = 4 GiB
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 256>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 2.0 * n * 16 / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
