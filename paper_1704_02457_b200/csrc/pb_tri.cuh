// Device building blocks shared by the factorization kernels (pb_factor.cu)
// and the fused Riccati chain (pb_chain.cu): the compact tri-panel shared
// memory layout, 8x8 tile fragments, the in-register diagonal Cholesky
// factor and the DMMA triangular solve through inverted diagonal blocks.
#pragma once
#include "pb_gemm.cuh"

namespace pb {

// ---- compact tri-panel layout ---------------------------------------------
// Row group g (rows 8g..8g+7, panels 2g and 2g+1) stores columns
// [0, w_g), w_g = min(8g+8, cn8), cn8 = round_up(n, 8).
struct Tri {
  int gn;   // column groups = cn8 / 8
  int cn8;
  __device__ __forceinline__ int width(int g) const { return g < gn ? 8 * g + 8 : cn8; }
  __device__ __forceinline__ int group_off(int g) const {
    return g < gn ? 32 * g * (g + 1) : 32 * gn * (gn + 1) + 8 * (g - gn) * cn8;
  }
  // element (r, c) with c < width(r/8)
  __device__ __forceinline__ int off(int r, int c) const {
    const int g = r >> 3;
    return group_off(g) + ((r >> 2) & 1) * 4 * width(g) + 4 * c + (r & 3);
  }
  static __host__ __device__ ix size(ix m, ix n) {
    const ix cn8 = (n + 7) / 8 * 8, gn = cn8 / 8, gm = (m + 7) / 8;
    return gm <= gn ? 32 * gm * (gm + 1) : 32 * gn * (gn + 1) + 8 * (gm - gn) * cn8;
  }
};

// Fragment offset of (row group g, k-step kk) for lane: rows 8g+(lane>>2),
// col 4kk+(lane&3).
__device__ __forceinline__ int tri_frag(const Tri &t, int g, int kk, int lane) {
  return t.group_off(g) + (lane >> 4) * 4 * t.width(g) + 16 * kk + 4 * (lane & 3) + ((lane >> 2) & 3);
}

// 1/sqrt(d) to ~1 ulp: MUFU seed + two Newton steps, branch-free (the
// library rsqrt() carries special-case paths that break warp convergence).
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double h = 0.5 * d;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// 1/d to ~1 ulp: MUFU seed (rel. error 2^-23) + one cubic step, three dependent FMAs.
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fma(-d, r, 1.0);
  const double p = fma(e, e, e);
  return fma(r, p, r);
}

// Cholesky factor AND inverse of the 8x8 diagonal tile in one column sweep
// (fragment layout: lane holds row lane>>2, cols 2(lane&3)+e).  Returns the
// first failing column (d <= 0, NaN passes) or -1; the tile holds L for the
// columns left of it; dinv_out[c] = 1/L[c,c]; w = W = L^{-1} (rows/cols past
// ncol unused).  The pivot chain of the n > 64 factorization is latency-bound
// on exactly this sweep, so its dependency chain is kept short: the
// columns stay UNSCALED while they are live (u = L * sqrt(d)): the rank-1
// update uses the multiplier u[r][c] / d_c, so column c's shuffles do not
// wait for its pivot's rsqrt and the chain per column is shuffle -> 1/d ->
// multiplier -> FMA (tools/factor_lat.cu: 1140 cycles per tile alone on an SM).  Column c of L and row c of
// W = L^{-1} take their 1/sqrt(d_c) factor when they become final (V is the
// unit-triangular inverse of U D^{-1}, forward-substituted with the same
// multipliers).
__device__ __forceinline__ int factor_inv_tile_u(double (&x)[2], double (&v)[2], int ncol, double *dinv_out, int lane) {
  const int fr = lane >> 2, fc = lane & 3;
  int fail = -1;
  v[0] = (fr == 2 * fc) ? 1.0 : 0.0;
  v[1] = (fr == 2 * fc + 1) ? 1.0 : 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int h = c >> 1, e = c & 1;
    const double d = __shfl_sync(0xffffffffu, x[e], 4 * c + h);
    const double ur = __shfl_sync(0xffffffffu, x[e], 4 * fr + h);
    const double u0 = __shfl_sync(0xffffffffu, x[e], 8 * fc + h);
    const double u1 = __shfl_sync(0xffffffffu, x[e], 8 * fc + 4 + h);
    const double v0 = __shfl_sync(0xffffffffu, v[0], 4 * c + fc);
    const double v1 = __shfl_sync(0xffffffffu, v[1], 4 * c + fc);
    const bool live = c < ncol && fail < 0;
    if (live && d <= 0.0) fail = c;  // NaN passes, as in the reference (ccore.pyx:423)
    const double rc = rcp_nr(d);
    const double rs = rsqrt_nr(d);
    if (lane == 0 && live && fail < 0) dinv_out[c] = rs;
    const double m = ur * rc;
    // column c of L and row c of W are final: scale them (predicated, no selects)
    if (fc == h) x[e] *= rs;
    if (fr == c) v[0] *= rs, v[1] *= rs;
    // trailing updates
    if (2 * fc > c) x[0] = fma(-m, u0, x[0]);
    if (2 * fc + 1 > c) x[1] = fma(-m, u1, x[1]);
    if (fr > c) v[0] = fma(-m, v0, v[0]), v[1] = fma(-m, v1, v[1]);
  }
  return fail;
}

// Store W (accumulator layout, from factor_inv_tile_u / inv_tile_regs) as the B operand of
// apply_inv_block: panel layout, element (n, k) at (n>>2)*32 + 4k + (n&3), read back as the B
// fragment of an m8n8k4 MMA:  X * L_jj^{-T} = X * W^T.
__device__ __forceinline__ void store_inv_block(const double (&w)[2], double *Wp, int lane) {
  const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
  for (int e = 0; e < 2; ++e) Wp[(fr >> 2) * 32 + 4 * (2 * fc + e) + (fr & 3)] = w[e];
}

// W = L_jj^{-1} of an already factored 8x8 diagonal block held in REGISTERS (x: accumulator layout, lane
// (fr, fc) holds L[fr][2fc + e]; dv = 1/L[c][c] for this lane's columns is read from dinv8[0..7]).  Same
// forward substitution as factor_inv_tile_u's inverse part, but every multiplier L[r][c] / L[c][c] is known
// up front, so the chain per column is one shuffle + one FMA (~35 cycles) instead of the shared-memory
// substitution sweep it replaces (~150).  w: W in accumulator layout; rows/columns >= ncol stay identity.
__device__ __forceinline__ void inv_tile_regs(const double (&x)[2], const double *dinv8, int ncol, double (&w)[2], int lane) {
  const int fr = lane >> 2, fc = lane & 3;
  w[0] = (fr == 2 * fc) ? 1.0 : 0.0;
  w[1] = (fr == 2 * fc + 1) ? 1.0 : 0.0;
  const double dr = fr < ncol ? dinv8[fr] : 1.0;  // this lane's row scale
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double lr = __shfl_sync(0xffffffffu, x[c & 1], 4 * fr + (c >> 1));  // L[fr][c]
    const double v0 = __shfl_sync(0xffffffffu, w[0], 4 * c + fc);
    const double v1 = __shfl_sync(0xffffffffu, w[1], 4 * c + fc);
    if (c < ncol && fr > c && fr < ncol) {
      const double m = lr * dinv8[c];
      w[0] = fma(-m, v0, w[0]);
      w[1] = fma(-m, v1, w[1]);
    }
  }
  w[0] *= dr, w[1] *= dr;
}

// acc := X * W^T for an 8x8 tile X held in shared memory (tri layout, rows
// 8g.., cols 8j..) and W from store_inv_block.
__device__ __forceinline__ void apply_inv_block(double (&acc)[2], const double *S, const Tri &t, int g, int j,
                                                const double *Wp, int lane) {
  const int fr = lane >> 2, fc = lane & 3;
  const int fa = tri_frag(t, g, 0, lane) + 32 * j;  // column block j starts at 4*8j
  const int fb = (lane >> 4) * 32 + 4 * fc + (fr & 3);
  acc[0] = acc[1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) dmma(acc, S[fa + 16 * kk], Wp[fb + 16 * kk]);
}


// Bulk-copy staging of an item into the tri layout for panel-aligned, 16-byte aligned items:
// every (row group, half) of the tri layout is ONE contiguous run of the
// item's panel (4 rows x min(width, n) columns), so thread 0 issues one
// cp.async.bulk per run (completion on the team's mbarrier) and the other
// threads only zero the padding columns [n, width) and the rows past m.
// Rows of a partial last panel are read as stored (they only ever feed
// their own rows and are never written back).
__device__ __forceinline__ void tri_load_bulk(double *S, const Tri &t, const double *C, ix cn, ix ci, ix cj, int m,
                                              int n, int gm, uint64_t *tbar, int ttid, int tthreads) {
  if (ttid == 0) {
    unsigned bytes = 0;
    for (int gg = 0; gg < gm; ++gg)
      for (int h = 0; h < 2; ++h)
        if (8 * gg + 4 * h < m) bytes += 32u * (unsigned)min(t.width(gg), n);
    mbar_arrive_expect_tx(tbar, bytes);
    for (int gg = 0; gg < gm; ++gg) {
      const int w = t.width(gg), base = t.group_off(gg);
      for (int h = 0; h < 2; ++h) {
        const int r0 = 8 * gg + 4 * h;
        if (r0 < m) tma_load_1d(S + base + h * 4 * w, C + eo(ci + r0, cj, cn), 32u * (unsigned)min(w, n), tbar);
      }
    }
  }
  for (int gg = 0; gg < gm; ++gg) {
    const int w = t.width(gg), base = t.group_off(gg);
    for (int h = 0; h < 2; ++h) {
      const int r0 = 8 * gg + 4 * h;
      const int c0 = r0 < m ? min(w, n) : 0;
      for (int q = ttid; q < 4 * (w - c0); q += tthreads) S[base + h * 4 * w + 4 * c0 + q] = 0.0;
    }
  }
}


}  // namespace pb
