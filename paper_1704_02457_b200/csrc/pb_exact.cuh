// The reference's own potrf operation order for ONE item, run by one warp
// straight on global memory: potrf_drv (ccore.pyx:877-905) over 4x4 blocks,
// block row by block row, with _kpotrf_core (:404-438) on the diagonal and
// _trsm_rltn_core (:358-388) left of it; per element the downdate sum starts
// at 0.0 and adds D[i][l] * (-D[j][l]) for l ascending, then C, then the
// in-block updates; IEEE sqrt and division, no FMA.  The 16 dot products of
// a block run on 16 lanes, the in-block chain on lane 0.
//
// The register-tile kernel (pb_potrf_reg.cu) marks items whose write set
// came out non-finite (a NaN / Inf input, or overflow) with PB_INFO_EXACT
// and leaves them untouched: its reordered arithmetic (masked multipliers)
// may spread a non-finite input over more entries of its row than the
// reference does.  potrf_exact_kernel (pb_exact.cu), launched right after,
// redoes exactly those items here.  Finite items never take this path.
#pragma once
#include "pb_common.cuh"

namespace pb {

// info value of an item left for the reference-order pass (internal: never
// visible after a call returns)
constexpr int32_t PB_INFO_EXACT = -7;

__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }

// Returns -1 or the first failing pivot (window-relative).  D is written as
// far as the reference writes it; dA[c] = 1/L[c][c] for completed columns.
__device__ __forceinline__ int potrf_exact_warp(const double *C, ix ci, ix cj, ix ccn, double *D, ix di, ix dj, ix dcn,
                                             double *dA, int n) {
  const int lane = threadIdx.x & 31;
  const unsigned FULLM = 0xffffffffu;
  int fail = -1;
  for (int ii = 0; ii < n && fail < 0; ii += 4) {
    const int ms = min(4, n - ii);
    for (int jj = 0; jj <= ii && fail < 0; jj += 4) {
      const int ns = min(4, n - jj);
      // lane t < 16: element (i, j) = (t & 3, t >> 2) of the block
      const int i = lane & 3, j = lane >> 2;
      double a = 0.0;
      if (lane < 16 && i < ms && j < ns) {
        for (int l = 0; l < jj; ++l)
          a = xadd(a, xmul(D[eo(di + ii + i, dj + l, dcn)], -D[eo(di + jj + j, dj + l, dcn)]));
      }
      double acc[4][4];
#pragma unroll
      for (int t = 0; t < 16; ++t) acc[t >> 2][t & 3] = __shfl_sync(FULLM, a, t);  // acc[j][i]
      __syncwarp();
      if (lane == 0) {
        for (int c = 0; c < ns; ++c)
          for (int r = 0; r < ms; ++r) acc[c][r] = xadd(acc[c][r], C[eo(ci + ii + r, cj + jj + c, ccn)]);
        if (jj == ii) {
          int f = -1;
          for (int c = 0; c < ns && f < 0; ++c) {
            const double d = acc[c][c];
            if (d <= 0.0) {  // ccore.pyx:423 (NaN passes)
              f = c;
              break;
            }
            const double ljj = __dsqrt_rn(d);
            const double inv = __ddiv_rn(1.0, ljj);
            acc[c][c] = ljj;
            dA[jj + c] = inv;
            for (int r = c + 1; r < ms; ++r) acc[c][r] = xmul(acc[c][r], inv);
            for (int c2 = c + 1; c2 < ns; ++c2) {
              const double lcj = acc[c][c2];
              for (int r = c2; r < ms; ++r) acc[c2][r] = xsub(acc[c2][r], xmul(acc[c][r], lcj));
            }
          }
          if (f >= 0) {
            fail = jj + f;  // the reference returns before storing this block
          } else {
            for (int c = 0; c < ns; ++c)
              for (int r = c; r < ms; ++r) D[eo(di + ii + r, dj + jj + c, dcn)] = acc[c][r];
          }
        } else {
          for (int c = 0; c < ns; ++c) {
            for (int t = 0; t < c; ++t) {
              const double e = D[eo(di + jj + c, dj + jj + t, dcn)];
              for (int r = 0; r < ms; ++r) acc[c][r] = xsub(acc[c][r], xmul(acc[t][r], e));
            }
            const double inv = dA[jj + c];
            for (int r = 0; r < ms; ++r) {
              acc[c][r] = xmul(acc[c][r], inv);
              D[eo(di + ii + r, dj + jj + c, dcn)] = acc[c][r];
            }
          }
        }
      }
      fail = __shfl_sync(FULLM, fail, 0);
      __syncwarp();
    }
  }
  return fail;
}

}  // namespace pb
