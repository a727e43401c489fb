// Batched pack / unpack / window copy between dense strided storage and
// panel-major storage (sm_100a).  Bit-exact element moves.
//
// Reference semantics: kpack_cm ccore.pyx:718-723, kunpack_cm :734-739,
// kgecp :677-682 (pack.py:45-82, 215-237).  Only in-window elements are
// written; padding is never touched.
//
// These kernels are HBM-bound: 16 bytes moved per element.  The product
// path (panel_chunk_kernel) moves one 32-byte CHUNK per thread: rows
// 4p..4p+3 of one column of a panel-aligned window -- exactly one sector of
// the panel side.  On the dense side the same four elements are one 32-byte
// run of a column-major item (two 16-byte accesses; consecutive threads walk
// the panels of a column, so a warp streams contiguous memory) or four
// elements of four rows of a row-major item (consecutive threads walk the
// columns, so each of the four accesses is a coalesced row segment).  Every
// sector moved is fully used on both sides; no shared-memory staging and no
// 64-bit index division (the grid walks items, threads walk an item's
// chunks).  A last panel with m % 4 rows moves its real rows only, so the
// padding rows of D are never written.  Windows starting inside a panel
// (i0 % 4 != 0) take the element-wise kernels below.
#include "pb_gemm.cuh"

namespace pb {

// One 32-byte chunk per (thread, k): rows 4p..4p+3 (rows < m only) of
// column j of item b.  Each thread gathers K chunks (all loads first, then
// all stores) so every thread keeps 2K memory requests in flight.  The
// write side is walked contiguously: the panel side (pack, gecp: columns
// fastest) or the dense side (unpack: panels fastest when column-major).
template <int MODE, int K = 4>  // 0 = pack (dense -> panel), 1 = unpack (panel -> dense), 2 = panel -> panel
__global__ void __launch_bounds__(256) panel_chunk_kernel(CopyArgs g, int np, int cpi, int ipb, int dense_vec) {
  // window rows m, columns n; np = ceil(m/4) panels; cpi = np * n chunks per item
  const bool pfast = MODE == 1 && g.x_row == 1;
  const int span = ipb * cpi;
  for (ix b0 = (ix)blockIdx.x * ipb; b0 < g.batch; b0 += (ix)gridDim.x * ipb) {
    for (int c0 = threadIdx.x; c0 < span; c0 += K * blockDim.x) {
      double v[K][4];
      ix bk[K];
      int pk[K], jk[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int c = c0 + k * blockDim.x;
        const int bi = c / cpi, w = c - bi * cpi;
        bk[k] = (c < span) ? b0 + bi : g.batch;  // out of range -> skipped
        if (pfast) {
          jk[k] = w / np;
          pk[k] = w - jk[k] * np;
        } else {
          pk[k] = w / (int)g.n;
          jk[k] = w - pk[k] * (int)g.n;
        }
        const ix b = bk[k];
        if (b >= g.batch) continue;
        const int r0 = 4 * pk[k], rows = min(4, (int)g.m - r0), j = jk[k];
        if (MODE == 0) {
          const double *x = g.X + b * g.x_stride + (ix)r0 * g.x_row + (ix)j * g.x_col;
          if (rows == 4 && dense_vec) {
            const double2 a = *reinterpret_cast<const double2 *>(x), c2 = *reinterpret_cast<const double2 *>(x + 2);
            v[k][0] = a.x, v[k][1] = a.y, v[k][2] = c2.x, v[k][3] = c2.y;
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r) v[k][r] = r < rows ? x[(ix)r * g.x_row] : 0.0;
          }
        } else {
          const double *ps = g.S.item(b) + eo(g.si + r0, g.sj + j, g.S.cn);
          const double2 a = *reinterpret_cast<const double2 *>(ps), c2 = *reinterpret_cast<const double2 *>(ps + 2);
          v[k][0] = a.x, v[k][1] = a.y, v[k][2] = c2.x, v[k][3] = c2.y;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const ix b = bk[k];
        if (b >= g.batch) continue;
        const int r0 = 4 * pk[k], rows = min(4, (int)g.m - r0), j = jk[k];
        if (MODE == 1) {
          double *x = g.Xw + b * g.x_stride + (ix)r0 * g.x_row + (ix)j * g.x_col;
          if (rows == 4 && dense_vec) {
            *reinterpret_cast<double2 *>(x) = make_double2(v[k][0], v[k][1]);
            *reinterpret_cast<double2 *>(x + 2) = make_double2(v[k][2], v[k][3]);
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r)
              if (r < rows) x[(ix)r * g.x_row] = v[k][r];
          }
        } else {
          double *pd = g.D.item(b) + eo(g.di + r0, g.dj + j, g.D.cn);
          if (rows == 4) {
            *reinterpret_cast<double2 *>(pd) = make_double2(v[k][0], v[k][1]);
            *reinterpret_cast<double2 *>(pd + 2) = make_double2(v[k][2], v[k][3]);
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r)
              if (r < rows) pd[r] = v[k][r];
          }
        }
      }
    }
  }
}

static bool panel16(const Mat &M, ix i0) {
  return (i0 & 3) == 0 && ((uintptr_t)M.p & 15) == 0 && (M.stride & 1) == 0;
}

template <int MODE>
static cudaError_t launch_chunks(const CopyArgs &g, cudaStream_t st) {
  const int np = (int)((g.m + 3) / 4);
  const ix cpi64 = (ix)np * g.n;
  if (cpi64 > (1 << 30)) return cudaErrorInvalidValue;
  const int cpi = (int)cpi64;
  const int ipb = cpi >= 1024 ? 1 : 1024 / cpi;  // >= 4 chunks per thread per pass
  int dense_vec = 0;
  if (MODE == 0) dense_vec = g.x_row == 1 && ((uintptr_t)g.X & 15) == 0 && (g.x_col & 1) == 0 && (g.x_stride & 1) == 0;
  if (MODE == 1) dense_vec = g.x_row == 1 && ((uintptr_t)g.Xw & 15) == 0 && (g.x_col & 1) == 0 && (g.x_stride & 1) == 0;
  ix blocks = (g.batch + ipb - 1) / ipb;
  const ix cap = (ix)num_sms() * 8;  // 8 x 256 threads per SM, grid-stride over items
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  panel_chunk_kernel<MODE><<<(unsigned)blocks, 256, 0, st>>>(g, np, cpi, ipb, dense_vec);
  note_launch();
  return cudaGetLastError();
}

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
  if (panel16(g.D, g.di)) return launch_chunks<0>(g, st);
  const bool ifast = !(g.x_col == 1 && g.x_row != 1);
  dense_panel_kernel<true><<<copy_grid(total), 256, 0, st>>>(g, ifast);
  note_launch();
  return cudaGetLastError();
}

cudaError_t run_unpack(const CopyArgs &g, cudaStream_t st) {
  const ix total = g.m * g.n * g.batch;
  if (total == 0) return cudaSuccess;
  if (panel16(g.S, g.si)) return launch_chunks<1>(g, st);
  const bool ifast = !(g.x_col == 1 && g.x_row != 1);
  dense_panel_kernel<false><<<copy_grid(total), 256, 0, st>>>(g, ifast);
  note_launch();
  return cudaGetLastError();
}

cudaError_t run_gecp(const CopyArgs &g, cudaStream_t st) {
  const ix total = g.m * g.n * g.batch;
  if (total == 0) return cudaSuccess;
  if (panel16(g.S, g.si) && panel16(g.D, g.di)) return launch_chunks<2>(g, st);
  gecp_kernel<<<copy_grid(total), 256, 0, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pb
