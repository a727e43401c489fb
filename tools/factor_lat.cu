// Latency of the 8x8 diagonal factor + inverse sweeps of pb_tri.cuh (clock64): one warp alone on an SM, and three
// warps on the same scheduler (warps 0, 4, 8 of one CTA) as in the potrf chain kernel with 3 CTAs/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1704_02457_b200/csrc -o tools/factor_lat tools/factor_lat.cu
#include <cstdio>
#include "pb_tri.cuh"
using namespace pb;
template <int MODE>
__global__ void k(double *out, long long *t, int reps, int nactive) {
  __shared__ double dinv[12][8];
  if (threadIdx.x < 96) dinv[threadIdx.x / 8][threadIdx.x % 8] = 0.3;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, fr = lane >> 2, fc = lane & 3;
  if ((w & 3) != 0 || (w >> 2) >= nactive) return;
  double x0[2], wv[2];
  for (int e = 0; e < 2; ++e) x0[e] = (fr == 2 * fc + e ? 9.0 : 0.0) + 0.1 / (1 + fr + 2 * fc + e);
  double acc = 0;
  long long a = clock64();
  for (int i = 0; i < reps; ++i) {
    double x[2] = {x0[0] + acc * 1e-300, x0[1]};
    if (MODE == 0) inv_tile_regs(x, dinv[w], 8, wv, lane);  // inverse of a given factor (trsm kernels)
    else factor_inv_tile_u(x, wv, 8, dinv[w], lane);        // factor + inverse (potrf chain)
    acc += x[0] + wv[1];
  }
  long long b = clock64();
  if (lane == 0 && w == 0) t[0] = (b - a) / reps;
  out[threadIdx.x] = acc;
}
int main() {
  double *out; long long *t;
  cudaMalloc(&out, 8 * 384); cudaMallocManaged(&t, 64);
  for (int na = 1; na <= 3; ++na) {
    for (int r = 0; r < 2; ++r) { k<0><<<1, 384>>>(out, t, 64, na); cudaDeviceSynchronize(); }
    long long t0 = t[0];
    for (int r = 0; r < 2; ++r) { k<1><<<1, 384>>>(out, t, 64, na); cudaDeviceSynchronize(); }
    printf("%d warp(s) on one scheduler: inv_tile_regs %lld clk, factor_inv_tile_u %lld clk (%s)\n", na, t0, t[0], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
