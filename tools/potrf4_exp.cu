// Memory-system experiment for batched dpotrf_l at n = 4 (the dominant
// launch of the C2 sweep): how the store pattern of D (lower triangle only,
// strict upper untouched -> partial 32-byte sectors) and the diag_inv tail
// change achieved DRAM throughput.  Not part of the product; numbers go to
// profiles/.  Items use the reference layout: 16 doubles of data, 4 of
// diag_inv, 4 of slack (192 B per item).
//
//   V0  masked stores of the lower triangle + 32 B diag_inv     (product semantics)
//   V1  V0, but the diag_inv sector pair written as one full 64 B chunk (slack zeroed)
//   V2  software read-modify-write: D's data loaded with C, full 128 B + 64 B stored
//   V3  upper bound: full 128 B + 64 B stores, no RMW (wrong semantics)
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/potrf4_exp tools/potrf4_exp.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int STRIDE = 24;  // doubles per item

__device__ __forceinline__ double2 ldcs(const double *p) {
  double2 v;
  asm volatile("ld.global.cs.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

template <int V, int CS>
__global__ void __launch_bounds__(256) k4(const double *__restrict__ C, double *__restrict__ D, long long nitems) {
  __shared__ double sm[8][32 * 17];  // per warp: 32 items x 16 (+1 pad)
  __shared__ double sd[8][32 * 4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double *S = sm[w];
  double *SD = sd[w];
  const long long ngroups = (nitems + 31) / 32;
  const long long gw = (long long)blockIdx.x * 8 + w, nw = (long long)gridDim.x * 8;
  // register prefetch: 8 pieces of 16 B per lane (C), and 8 of D for V2
  double2 pc[8], pd[8];
  auto load = [&](long long g) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int p = lane + 32 * k, it = p >> 3, wd = p & 7;
      const long long b = g * 32 + it;
      if (b < nitems) {
        const double *src = C + b * STRIDE + 2 * wd;
        pc[k] = CS ? ldcs(src) : *reinterpret_cast<const double2 *>(src);
        if (V == 2) pd[k] = *reinterpret_cast<const double2 *>(D + b * STRIDE + 2 * wd);
      }
    }
  };
  long long g = gw;
  if (g < ngroups) load(g);
  for (; g < ngroups; g += nw) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int p = lane + 32 * k, it = p >> 3, wd = p & 7;
      S[it * 17 + 2 * wd] = pc[k].x;
      S[it * 17 + 2 * wd + 1] = pc[k].y;
    }
    double2 dd[8];
    if (V == 2) {
#pragma unroll
      for (int k = 0; k < 8; ++k) dd[k] = pd[k];
    }
    const long long gn = g + nw;
    if (gn < ngroups) load(gn);
    __syncwarp();
    // factor item `lane` (4x4, element (i,j) at 4j+i), reference order
    {
      double a[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) a[j][i] = S[lane * 17 + 4 * j + i];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double d = a[c][c];
        const double l = __dsqrt_rn(d);
        const double inv = __ddiv_rn(1.0, l);
        a[c][c] = l;
        SD[lane * 4 + c] = inv;
#pragma unroll
        for (int r = c + 1; r < 4; ++r) a[c][r] = __dmul_rn(a[c][r], inv);
#pragma unroll
        for (int c2 = c + 1; c2 < 4; ++c2)
#pragma unroll
          for (int r = c2; r < 4; ++r) a[c2][r] = __dsub_rn(a[c2][r], __dmul_rn(a[c][r], a[c][c2]));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i >= j) S[lane * 17 + 4 * j + i] = a[j][i];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int p = lane + 32 * k, it = p >> 3, wd = p & 7;
      const long long b = g * 32 + it;
      if (b >= nitems) continue;
      double *dst = D + b * STRIDE + 2 * wd;
      const int col = wd >> 1, r0 = 2 * (wd & 1);
      double2 v = make_double2(S[it * 17 + 2 * wd], S[it * 17 + 2 * wd + 1]);
      if (V == 0 || V == 1) {
        const bool w0 = r0 >= col, w1 = r0 + 1 >= col;
        if (w0 && w1) *reinterpret_cast<double2 *>(dst) = v;
        else if (w1) dst[1] = v.y;
      } else if (V == 2) {
        if (r0 < col) v.x = dd[k].x;
        if (r0 + 1 < col) v.y = dd[k].y;
        *reinterpret_cast<double2 *>(dst) = v;
      } else {
        *reinterpret_cast<double2 *>(dst) = v;
      }
    }
    // diag_inv: 32 items x 4 doubles; V>=1 also the 4 slack doubles
    if (V == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int q = lane + 32 * k, it = q >> 2, c = q & 3;
        const long long b = g * 32 + it;
        if (b < nitems) D[b * STRIDE + 16 + c] = SD[q];
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int q = lane + 32 * k, it = q >> 2, pc2 = q & 3;  // 16-byte piece pc2 of the 64 B chunk
        const long long b = g * 32 + it;
        if (b < nitems) {
          double2 v = pc2 < 2 ? make_double2(SD[it * 4 + 2 * pc2], SD[it * 4 + 2 * pc2 + 1]) : make_double2(0.0, 0.0);
          *reinterpret_cast<double2 *>(D + b * STRIDE + 16 + 2 * pc2) = v;
        }
      }
    }
    __syncwarp();
  }
}

template <int V, int CS>
float run(const double *C, double *D, long long n, int blocksPerSM, int reps) {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = sms * blocksPerSM;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  k4<V, CS><<<grid, 256>>>(C, D, n);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) k4<V, CS><<<grid, 256>>>(C, D, n);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

__global__ void fill(double *C, long long n) {
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < n; b += (long long)gridDim.x * blockDim.x) {
    double *c = C + b * STRIDE;
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 4; ++i) c[4 * j + i] = (i == j) ? 4.0 + 0.001 * (b & 7) : 0.5;
  }
}

int main(int argc, char **argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 30973322LL;
  double *C, *D;
  CK(cudaMalloc(&C, n * STRIDE * 8));
  CK(cudaMalloc(&D, n * STRIDE * 8));
  fill<<<4096, 256>>>(C, n);
  CK(cudaMemset(D, 0, n * STRIDE * 8));
  CK(cudaDeviceSynchronize());
  const double alg = 192.0 * n;  // 8*(n(n+1)+n) bytes per item, SURVEY §8d
  for (int gran : {-1, 32, 64, 128}) {
  if (gran > 0) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran));
  size_t cur = 0;
  CK(cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity));
  printf("-- L2 fetch granularity %zu\n", cur);
  for (int bps : {2}) {
    float t;
#define R(V, CS)                                                                                       \
  t = run<V, CS>(C, D, n, bps, 10);                                                                    \
  printf("V%d cs=%d blocks/SM=%d  %.3f ms  alg %.0f GB/s  frac %.3f\n", V, CS, bps, t, alg / t / 1e6, \
         alg / t / 1e6 / 6549.4);
    R(0, 0) R(2, 0) R(3, 0)
  }
  }
  return 0;
}
