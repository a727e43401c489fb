// Probe: SM-initiated PCIe traffic to pinned host memory (UVA), by access
// pattern -- full-line reads, per-item partial reads, full writes, and the
// masked writes a potrf n=4 item needs (lower triangle + diag_inv with the
// strict upper untouched).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/zc_bw.cu -o tools/zc_bw ; run on the GPU box.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// every thread reads 8 B words; `use` = words of each 24-word item that are read
__global__ void rd_items(const double *__restrict__ h, int64_t items, unsigned long long use, double *out) {
  double acc = 0;
  const int64_t words = items * 24;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(w % 24);
    if ((use >> k) & 1) acc += __ldcg(h + w);
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void wr_items(double *__restrict__ h, int64_t items, unsigned long long use) {
  const int64_t words = items * 24;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(w % 24);
    if ((use >> k) & 1) h[w] = (double)k;
  }
}

// 16-B vector variants over the whole buffer
__global__ void rd_vec(const double2 *__restrict__ h, int64_t n, double *out) {
  double acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = __ldcg(h + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}
__global__ void wr_vec(double2 *__restrict__ h, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    h[i] = make_double2(1.0, 2.0);
}

int main() {
  const int64_t items = 8000000;  // n=4 items, 192 B each -> 1.536 GB
  const size_t bytes = items * 192;
  double *h, *out;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&out, 8));
  for (size_t i = 0; i < bytes / 8; i += 512) h[i] = 0;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // n=4 lower: word offsets element (i,j) = 4j+i for i>=j, plus diag_inv 16..19
  unsigned long long lower = 0;
  for (int j = 0; j < 4; ++j)
    for (int i = j; i < 4; ++i) lower |= 1ull << (4 * j + i);
  unsigned long long dinv = 0xFull << 16;
  const unsigned long long all = (1ull << 24) - 1, data = 0xFFFFull;
  struct Case { const char *name; int kind; unsigned long long use; double algbytes; };
  Case cs[] = {
      {"read  all 192B/item (8B lanes)", 0, all, 192.0},
      {"read  data 128B/item", 0, data, 128.0},
      {"write all 192B/item (8B lanes)", 1, all, 192.0},
      {"write data+dinv 160B contiguous", 1, data | dinv, 160.0},
      {"write lower+dinv (masked, n=4)", 1, lower | dinv, 112.0},
      {"read  16B vectors, whole buffer", 2, 0, 192.0},
      {"write 16B vectors, whole buffer", 3, 0, 192.0},
  };
  for (int threads : {256, 1024}) {
    for (int per_sm : {4, 16}) {
      const int grid = sms * per_sm;
      for (auto &c : cs) {
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
          cudaEventRecord(a);
          if (c.kind == 0) rd_items<<<grid, threads>>>(h, items, c.use, out);
          else if (c.kind == 1) wr_items<<<grid, threads>>>(h, items, c.use);
          else if (c.kind == 2) rd_vec<<<grid, threads>>>((const double2 *)h, bytes / 16, out);
          else wr_vec<<<grid, threads>>>((double2 *)h, bytes / 16);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        printf("threads=%4d grid=%5d %-34s %8.2f ms  %6.1f GB/s useful  %6.1f GB/s item-eq\n", threads, grid, c.name,
               best, items * c.algbytes / best / 1e6, bytes / best / 1e6);
      }
    }
  }
  // copy engine reference
  double *d;
  CK(cudaMalloc(&d, bytes));
  for (int dir = 0; dir < 2; ++dir) {
    cudaEventRecord(a);
    if (dir == 0) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
    else cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("copy engine %s %.2f ms %.1f GB/s\n", dir ? "D2H" : "H2D", ms, bytes / ms / 1e6);
  }
  return 0;
}
