// Batched getrf (LU with / without partial pivoting) on panel-major FP64
// items, bit-exact with the reference (sm_100a).  SURVEY.md §8f row 4.
//
// Reference: level3._getrf / _getrf_inplace (level3.py:405-498) over the
// core's gemm_nn_drv (ccore.pyx:774-801), kgetrf_panel (:563-650),
// krowswap (:661-670) and lu_rowsolve_drv (:488-500 -> _ktrsm_llnu_core
// :453-477).  Pivot choice is discrete, so parity must be exact: the
// kernel evaluates every element with the reference's operation sequence
// (sums from 0.0 over l ascending, v = -1*acc + 1*C, IEEE division, no FMA)
// and only parallelises across independent elements.
//
// One warp per CTA (converged control flow), one item at a time: the m x n
// window is staged into shared memory (column-major, odd leading
// dimension), factored in place panel by panel, and written back:
//  * panel downdate / U12 downdate: one element per lane-iteration;
//  * pivot search: per-lane scan of its rows in ascending order, then a
//    warp arg-max reduction that keeps the reference's semantics (first
//    index wins ties, NaN candidates never win, a NaN diagonal keeps c);
//  * row swaps, column scaling, rank-1 updates, row solves: one row /
//    column per lane-iteration, __syncwarp between dependent phases.
// Failure (zero pivot) stops the item exactly where the reference raises:
// completed panels' ipiv, completed columns' diag_inv, and -- for a
// panel-aligned destination -- the partially factored window are written;
// an unaligned destination stays untouched (the reference factors in a
// scratch matrix and raises before copying it back, level3.py:437-442).
#include "pb_gemm.cuh"

namespace pb {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

struct GetrfArgs {
  int m, n, pivot;
  Mat C, D;
  ix ci, cj, di, dj;
  int64_t *ipiv;
  ix ipiv_stride;
  int32_t *info;
  ix batch;
  int ld;
};

__global__ void __launch_bounds__(32) getrf_kernel(GetrfArgs g) {
  extern __shared__ __align__(16) double S[];
  const int lane = threadIdx.x;
  const int m = g.m, n = g.n, ld = g.ld;
  const int mn = m < n ? m : n;
#define A(i, j) S[(j) * ld + (i)]
  for (ix b = blockIdx.x; b < g.batch; b += gridDim.x) {
    const double *Cb = g.C.p + b * g.C.stride;
    for (int e = lane; e < m * n; e += 32) {
      const int j = e / m, i = e - j * m;
      A(i, j) = Cb[eo(g.ci + i, g.cj + j, g.C.cn)];
    }
    __syncwarp();
    double *dA = g.D.d + b * g.D.dstride + g.dj;
    int64_t *ip = g.ipiv ? g.ipiv + b * g.ipiv_stride : nullptr;
    int fail = -1;
    for (int j0 = 0; j0 < mn && fail < 0; j0 += 4) {
      const int jb = mn - j0 < 4 ? mn - j0 : 4;
      // (a) panel downdate: A[j0:, j0:j0+jb] = -1 * (A[j0:, :j0] A[:j0, j0:j0+jb]) + 1 * A
      if (j0 > 0) {
        const int rows = m - j0;
        for (int e = lane; e < rows * jb; e += 32) {
          const int j = j0 + e / rows, i = j0 + e % rows;
          double acc = 0.0;
          for (int l = 0; l < j0; ++l) acc = dadd(acc, dmul(A(i, l), A(l, j)));
          A(i, j) = dadd(dmul(-1.0, acc), dmul(1.0, A(i, j)));
        }
        __syncwarp();
      }
      // (b) panel factor (kgetrf_panel)
      int piv[4] = {0, 0, 0, 0};
      for (int c = 0; c < jb; ++c) {
        const int gc = j0 + c;
        if (g.pivot) {
          // lane-local scan of rows gc+1+lane, +32, ... ascending; NaN never wins
          double bv = -1.0;
          int best = -1;
          for (int r = gc + 1 + lane; r < m; r += 32) {
            const double v = fabs(A(r, gc));
            if (v > bv) bv = v, best = r;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(FULL, bv, o);
            const int ob = __shfl_xor_sync(FULL, best, o);
            if (ov > bv || (ov == bv && ob >= 0 && (best < 0 || ob < best))) bv = ov, best = ob;
          }
          const double d0 = fabs(A(gc, gc));
          // sequential rule: start at the diagonal, replace only on a strictly larger value
          if (d0 != d0 || best < 0 || !(bv > d0)) bv = d0, best = gc;
          if (bv == 0.0) {
            fail = gc;
            break;
          }
          piv[c] = best - j0;
          if (best != gc) {
            if (lane < jb) {
              const double t = A(gc, j0 + lane);
              A(gc, j0 + lane) = A(best, j0 + lane);
              A(best, j0 + lane) = t;
            }
            __syncwarp();
          }
        } else if (A(gc, gc) == 0.0) {
          fail = gc;
          break;
        }
        const double inv = __ddiv_rn(1.0, A(gc, gc));
        if (lane == 0) dA[gc] = inv;
        for (int r = gc + 1 + lane; r < m; r += 32) A(r, gc) = dmul(A(r, gc), inv);
        __syncwarp();
        for (int cc = c + 1; cc < jb; ++cc) {
          const double ucc = A(gc, j0 + cc);
          if (ucc != 0.0)
            for (int r = gc + 1 + lane; r < m; r += 32) A(r, j0 + cc) = dsub(A(r, j0 + cc), dmul(A(r, gc), ucc));
        }
        __syncwarp();
      }
      if (fail >= 0) break;
      // (c) deferred row swaps outside the panel, in panel-column order
      if (g.pivot) {
        for (int cc = 0; cc < jb; ++cc) {
          const int r = piv[cc];
          if (lane == 0 && ip) ip[j0 + cc] = j0 + r;
          if (r != cc) {
            for (int j = lane; j < n; j += 32) {
              if (j >= j0 && j < j0 + jb) continue;
              const double t = A(j0 + cc, j);
              A(j0 + cc, j) = A(j0 + r, j);
              A(j0 + r, j) = t;
            }
            __syncwarp();
          }
        }
      }
      // (d) U12: downdate of the panel's rows right of it, then the unit-lower row solve
      if (j0 + jb < n) {
        const int cols = n - j0 - jb;
        if (j0 > 0) {
          for (int e = lane; e < jb * cols; e += 32) {
            const int j = j0 + jb + e / jb, i = j0 + e % jb;
            double acc = 0.0;
            for (int l = 0; l < j0; ++l) acc = dadd(acc, dmul(A(i, l), A(l, j)));
            A(i, j) = dadd(dmul(-1.0, acc), dmul(1.0, A(i, j)));
          }
          __syncwarp();
        }
        for (int j = j0 + jb + lane; j < n; j += 32) {
          double acc[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (i < jb) acc[i] = dadd(0.0, dmul(1.0, A(j0 + i, j)));
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (i < jb) {
              const double x = acc[i];
#pragma unroll
              for (int t = 0; t < 4; ++t)
                if (t > i && t < jb) acc[t] = dsub(acc[t], dmul(A(j0 + t, j0 + i), x));
            }
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (i < jb) A(j0 + i, j) = acc[i];
        }
        __syncwarp();
      }
    }
    if (lane == 0 && g.info) g.info[b] = fail;
    // write back: the whole window, unless a failing item has an unaligned destination
    if (fail < 0 || (g.di & 3) == 0) {
      double *Db = g.D.p + b * g.D.stride;
      for (int e = lane; e < m * n; e += 32) {
        const int j = e / m, i = e - j * m;
        Db[eo(g.di + i, g.dj + j, g.D.cn)] = A(i, j);
      }
    }
    __syncwarp();
  }
#undef A
}

}  // namespace

size_t getrf_smem(int m, int n) { return sizeof(double) * (size_t)(m | 1) * (size_t)n; }

cudaError_t run_getrf(int m, int n, int pivot, const Mat &C, ix ci, ix cj, const Mat &D, ix di, ix dj, int64_t *ipiv,
                      ix ipiv_stride, int32_t *info, ix batch, cudaStream_t st) {
  GetrfArgs g;
  g.m = m, g.n = n, g.pivot = pivot;
  g.C = C, g.D = D;
  g.ci = ci, g.cj = cj, g.di = di, g.dj = dj;
  g.ipiv = ipiv, g.ipiv_stride = ipiv_stride;
  g.info = info;
  g.batch = batch;
  g.ld = m | 1;
  const size_t smem = getrf_smem(m, n);
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  static LaunchCache cache;
  const int occ = cache.occupancy((const void *)getrf_kernel, 32, smem);
  ix grid = (ix)num_sms() * occ;
  if (grid > batch) grid = batch;
  if (grid < 1) grid = 1;
  getrf_kernel<<<(unsigned)grid, 32, smem, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pb
