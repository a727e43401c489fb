// Batched pack / unpack / window copy between dense strided storage and
// panel-major storage (sm_100a).  Bit-exact element moves.
//
// Reference semantics: kpack_cm ccore.pyx:718-723, kunpack_cm :734-739,
// kgecp :677-682 (pack.py:45-82, 215-237).  Only in-window elements are
// written; padding is never touched.
//
// Traversal order is chosen per call so the side with unit stride is read
// or written contiguously by consecutive threads, and the panel side is
// walked so that every 32-byte sector (one panel column = 4 doubles) is
// fully used.  These kernels are HBM-bound: 16 bytes moved per element.
#include "pb_gemm.cuh"

namespace pb {

// Index decomposition: `ifast` selects whether row index i (true) or
// column index j (false) varies fastest across consecutive threads.
template <bool PACK>
__global__ void __launch_bounds__(256) dense_panel_kernel(CopyArgs g, bool ifast) {
  const ix per = g.m * g.n;
  const ix total = per * g.batch;
  for (ix t = (ix)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (ix)gridDim.x * blockDim.x) {
    const ix b = t / per, w = t - b * per;
    ix i, j;
    if (ifast) {
      j = w / g.m;
      i = w - j * g.m;
    } else {
      i = w / g.n;
      j = w - i * g.n;
    }
    const ix xo = b * g.x_stride + i * g.x_row + j * g.x_col;
    if (PACK) {
      g.D.item(b)[eo(g.di + i, g.dj + j, g.D.cn)] = g.X[xo];
    } else {
      g.Xw[xo] = g.S.item(b)[eo(g.si + i, g.sj + j, g.S.cn)];
    }
  }
}

__global__ void __launch_bounds__(256) gecp_kernel(CopyArgs g) {
  const ix per = g.m * g.n;
  const ix total = per * g.batch;
  for (ix t = (ix)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (ix)gridDim.x * blockDim.x) {
    const ix b = t / per, w = t - b * per;
    const ix j = w / g.m, i = w - j * g.m;
    g.D.item(b)[eo(g.di + i, g.dj + j, g.D.cn)] = g.S.item(b)[eo(g.si + i, g.sj + j, g.S.cn)];
  }
}

static unsigned copy_grid(ix total) {
  ix blocks = (total + 255) / 256;
  const ix cap = (ix)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

cudaError_t run_pack(const CopyArgs &g, cudaStream_t st) {
  const ix total = g.m * g.n * g.batch;
  if (total == 0) return cudaSuccess;
  const bool ifast = !(g.x_col == 1 && g.x_row != 1);
  dense_panel_kernel<true><<<copy_grid(total), 256, 0, st>>>(g, ifast);
  note_launch();
  return cudaGetLastError();
}

cudaError_t run_unpack(const CopyArgs &g, cudaStream_t st) {
  const ix total = g.m * g.n * g.batch;
  if (total == 0) return cudaSuccess;
  const bool ifast = !(g.x_col == 1 && g.x_row != 1);
  dense_panel_kernel<false><<<copy_grid(total), 256, 0, st>>>(g, ifast);
  note_launch();
  return cudaGetLastError();
}

cudaError_t run_gecp(const CopyArgs &g, cudaStream_t st) {
  const ix total = g.m * g.n * g.batch;
  if (total == 0) return cudaSuccess;
  gecp_kernel<<<copy_grid(total), 256, 0, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pb
