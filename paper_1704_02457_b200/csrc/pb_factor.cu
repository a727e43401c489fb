// Batched dpotrf_l and dtrsm_rltn on panel-major FP64 storage (sm_100a).
//
// Reference semantics: potrf_drv ccore.pyx:877-905 (+ _kpotrf_core
// :404-438, _trsm_rltn_core :358-388), trsm_rltn_drv ccore.pyx:855-874,
// reciprocal selection level3._recip_diag level3.py:160-177.
//
// Design (B200-first, not the reference's 4x4 CPU blocking):
//  * a "team" of TW warps owns one item at a time; the item's lower
//    trapezoid lives in shared memory in a compact tri-panel layout (panel
//    pair g holds only columns [0, 8g+8)), so n <= 232 fits one CTA;
//  * left-looking over 8-column blocks: every 8x8 output tile is one
//    m8n8k4 accumulator; the downdate  tile -= L[g,:j] L[j,:j]^T  runs on
//    DMMA straight from shared memory (fragments = two 128-byte runs);
//  * the 8x8 diagonal factor and the 8-column triangular solves run in
//    registers with warp shuffles (sqrt and one reciprocal per column, then
//    multiplies, like the reference's dinv convention ccore.pyx:426-428);
//  * several teams per CTA, and many CTAs per SM for small n, hide the
//    serial sqrt/reciprocal chain.
// Bad pivots: the first index with d <= 0 (NaN passes, ccore.pyx:423) goes
// to info[b]; the write-back then stores exactly the part of D the
// reference would have stored before returning, and dinv[0, index).
#include <cstdlib>

#include "pb_tri.cuh"

namespace pb {

// ---------------------------------------------------------------------------
// potrf team kernel

// Stage item b's lower trapezoid of C into the tri layout.  vec: 16-byte
// cp.async pieces (panel-aligned window, asynchronous); else 8-byte loads.
// Columns >= n and panels past m are zero-filled; upper elements inside a
// diagonal tile are loaded as-is (never used for the lower factor).
__device__ __forceinline__ void tri_load(double *S, const Tri &t, const double *C, ix cn, ix ci, ix cj, int m, int n,
                                         int gm, bool vec, int ttid, int tthreads) {
  for (int gg = 0; gg < gm; ++gg) {
    const int w = t.width(gg), base = t.group_off(gg);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int r0 = 8 * gg + 4 * half;
      if (vec) {
        for (int q = ttid; q < 2 * w; q += tthreads) {
          const int c = q >> 1, h2 = q & 1;
          const bool ok = r0 < m && c < n;
          const double *src = ok ? C + eo(ci + r0, cj + c, cn) + 2 * h2 : C;
          cp_async16(S + base + half * 4 * w + 4 * c + 2 * h2, src, ok ? 16 : 0);
        }
      } else {
        for (int q = ttid; q < 4 * w; q += tthreads) {
          const int c = q >> 2, r = r0 + (q & 3);
          S[base + half * 4 * w + q] = (r < m && c < n && c <= r) ? C[eo(ci + r, cj + c, cn)] : 0.0;
        }
      }
    }
  }
}

// Stage a rows x k window (rows padded to rpad with zeros, columns to kp)
// into a plain panel-major buffer of panel length kp.
__device__ __forceinline__ void panel_load(double *S, int kp, const double *X, ix cn, ix xi, ix xj, int rows, int rpad,
                                           int k, int ttid, int tthreads) {
  const bool vec = (xi & 3) == 0 && ((uintptr_t)X & 15) == 0;
  if (vec) {
    for (int q = ttid; q < (rpad / 4) * kp * 2; q += tthreads) {
      const int p = q / (2 * kp), w = q % (2 * kp), l = w >> 1, h = w & 1;
      const int r = 4 * p + 2 * h;
      const bool ok = r < rows && l < k;  // rows come in pairs: rows, k are whole-panel padded below
      const double *src = ok ? X + eo(xi + r, xj + l, cn) : X;
      cp_async16(S + p * 4 * kp + 4 * l + 2 * h, src, ok ? 16 : 0);
    }
  } else {
    for (int q = ttid; q < rpad * kp; q += tthreads) {
      const int p = q / (4 * kp), w = q % (4 * kp), l = w >> 2, rr = w & 3;
      const int r = 4 * p + rr;
      S[q] = (r < rows && l < k) ? X[eo(xi + r, xj + l, cn)] : 0.0;
    }
  }
}

// ---- look-ahead downdate helpers (row-cyclic tile ownership) ------------
// A warp owns row groups gg = tw + i*TW (slot i).  The active slots of a
// column step are always a suffix [i0, MAXT); they are processed by fully
// unrolled, branch-free slot loops (rows past gm are clamped to a valid row
// and their results discarded), so every DMMA issues from converged code.

template <int MAXT, int TW>
__device__ __forceinline__ int first_slot(int tw, int lo) {
  const int d = lo - tw;
  return d <= 0 ? 0 : (d + TW - 1) / TW;
}

// a[i] = C(gg_i, cb) [+ A_gg B_cb^T] - sum_{k < kend blocks} L(gg_i, k) L(cb, k)^T for i >= I0
template <int MAXT, int TW, int I0, bool SK>
__device__ __forceinline__ void dd_suffix(double (&a)[MAXT][2], const double *S, const Tri &t, const double *SA,
                                          const double *SB, int kp, int tw, int gm, int cb, int kend, int lane) {
  const int fr = lane >> 2, fc = lane & 3;
  int fa[MAXT];
#pragma unroll
  for (int i = I0; i < MAXT; ++i) {
    const int gg = min(tw + i * TW, gm - 1);
    a[i][0] = S[t.off(8 * gg + fr, 8 * cb + 2 * fc)];
    a[i][1] = S[t.off(8 * gg + fr, 8 * cb + 2 * fc + 1)];
    fa[i] = tri_frag(t, gg, 0, lane);
  }
  if (SK) {
    const int po = (lane >> 4) * 4 * kp + 4 * fc + (fr & 3);
    const int pb = 2 * cb * 4 * kp + po;
    for (int kk = 0; kk < kp / 4; ++kk) {
      const double bv = SB[pb + 16 * kk];
#pragma unroll
      for (int i = I0; i < MAXT; ++i) {
        const int gg = min(tw + i * TW, gm - 1);
        dmma(a[i], SA[2 * gg * 4 * kp + po + 16 * kk], bv);
      }
    }
  }
  const int fb = tri_frag(t, cb, 0, lane);
#pragma unroll 2
  for (int kk = 0; kk < 2 * kend; ++kk) {
    const double bv = S[fb + 16 * kk];
#pragma unroll
    for (int i = I0; i < MAXT; ++i) dmma(a[i], -S[fa[i] + 16 * kk], bv);
  }
}

template <int MAXT, int TW, bool SK>
__device__ __forceinline__ void downdate_tiles(double (&a)[MAXT][2], const double *S, const Tri &t, const double *SA,
                                               const double *SB, int kp, int tw, int gm, int lo, int cb, int kend,
                                               int lane) {
  const int i0 = first_slot<MAXT, TW>(tw, lo);
#define PB_DD(I_) \
  if (MAXT > I_ && i0 == I_) dd_suffix<MAXT, TW, (MAXT > I_ ? I_ : 0), SK>(a, S, t, SA, SB, kp, tw, gm, cb, kend, lane);
  PB_DD(0) PB_DD(1) PB_DD(2) PB_DD(3) PB_DD(4) PB_DD(5) PB_DD(6) PB_DD(7)
#undef PB_DD
}

// a[i] = p[i] - L(gg_i, kb) L(cb, kb)^T for i >= I0 (one column block)
template <int MAXT, int TW, int I0>
__device__ __forceinline__ void ab_suffix(double (&a)[MAXT][2], const double (&p)[MAXT][2], const double *S,
                                          const Tri &t, int tw, int gm, int cb, int kb, int lane) {
  const int fb = tri_frag(t, cb, 0, lane) + 32 * kb;
  const double b0 = S[fb], b1 = S[fb + 16];
#pragma unroll
  for (int i = I0; i < MAXT; ++i) {
    const int gg = min(tw + i * TW, gm - 1);
    const int fa = tri_frag(t, gg, 0, lane) + 32 * kb;
    a[i][0] = p[i][0], a[i][1] = p[i][1];
    dmma(a[i], -S[fa], b0);
    dmma(a[i], -S[fa + 16], b1);
  }
}

template <int MAXT, int TW>
__device__ __forceinline__ void add_block_tiles(double (&a)[MAXT][2], const double (&p)[MAXT][2], const double *S,
                                                const Tri &t, int tw, int gm, int lo, int cb, int kb, int lane) {
  const int i0 = first_slot<MAXT, TW>(tw, lo);
#define PB_AB(I_) \
  if (MAXT > I_ && i0 == I_) ab_suffix<MAXT, TW, (MAXT > I_ ? I_ : 0)>(a, p, S, t, tw, gm, cb, kb, lane);
  PB_AB(0) PB_AB(1) PB_AB(2) PB_AB(3) PB_AB(4) PB_AB(5) PB_AB(6) PB_AB(7)
#undef PB_AB
}

// GM/GN > 0 fix the row/column group counts at compile time (the common
// square sizes): every tile loop then unrolls and all tri-layout offsets
// fold to constants; GM = GN = 0 is the generic runtime-shaped kernel.
// SK: fused syrk_potrf -- the item's A (and B) windows sit next to the tri
// buffer and every tile's downdate also accumulates + A_g B_j^T, exactly
// the per-tile order of syrk_potrf_drv (ccore.pyx:908-941).
template <int TW, int MAXT, bool DB, int GM = 0, int GN = 0, bool SK = false, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) potrf_team_kernel(PotrfArgs g, int team_elems, int vec_in, int vec_out) {
  extern __shared__ __align__(128) double smem[];
  const int lane = threadIdx.x & 31, warp = warp_uniform();
  const int team = warp / TW, tw = warp % TW;
  const int teams_per_cta = (blockDim.x >> 5) / TW;
  const int tthreads = TW * 32, ttid = tw * 32 + lane;
  const int bar = 1 + team;
  const int m = (int)g.m, n = (int)g.n;
  Tri t;
  t.cn8 = GN > 0 ? 8 * GN : (n + 7) / 8 * 8;
  t.gn = GN > 0 ? GN : t.cn8 / 8;
  const int gm = GM > 0 ? GM : (m + 7) / 8;
  const int tri_elems = GM > 0 ? (int)Tri::size(8 * GM, 8 * GN) : (int)Tri::size(m, n);
  double *S0 = smem + (ix)team * team_elems;
  double *S1 = DB ? S0 + tri_elems : S0;
  double *dinv = S0 + (DB ? 2 : 1) * tri_elems;         // cn8 doubles
  volatile int *flag = (volatile int *)(dinv + t.cn8);  // failure index
  double *Wp = dinv + t.cn8 + 8;                        // inverted diagonal block (64)
  uint64_t *tbar = reinterpret_cast<uint64_t *>(dinv + t.cn8 + 1);  // bulk-load barrier
  // SK operands: A rows padded to 8*gm, B rows to 8*gn, panel length kp
  const int kp = SK ? (int)((g.k + 3) & ~(ix)3) : 0;
  double *SA = Wp + 64;
  double *SB = SK && !g.ab_same ? SA + 8 * gm * kp : SA;
  const int fr = lane >> 2, fc = lane & 3;
  const bool aligned_out = (g.di & 3) == 0;
  const bool vin = vec_in != 0;
  const ix stride = (ix)gridDim.x * teams_per_cta;
  // bulk (TMA) tri staging and write-back: single-buffered, aligned items
  const bool bulk_in = !DB && vin;
  const bool bulk_out = !DB && vec_out != 0;
  unsigned phase = 0;
  if (bulk_in) {
    if (ttid == 0) {
      mbar_init(tbar, 1);
      mbar_fence_init();
    }
    team_sync(bar, tthreads);
  }
  auto load_item = [&](ix bb) {
    if (bulk_in) tri_load_bulk(S0, t, g.C.item(bb), g.C.cn, g.ci, g.cj, m, n, gm, tbar, ttid, tthreads);
    else tri_load(S0, t, g.C.item(bb), g.C.cn, g.ci, g.cj, m, n, gm, vin, ttid, tthreads);
  };

  auto skip = [&](ix b) { return g.merge && g.info[b] >= 0; };
  ix b = (ix)blockIdx.x * teams_per_cta + team;
  while (b < g.batch && skip(b)) b += stride;
  auto stage_ab = [&](ix bb) {
    if (SK) {
      panel_load(SA, kp, g.A.item(bb), g.A.cn, g.ai, g.aj, m, 8 * gm, (int)g.k, ttid, tthreads);
      if (!g.ab_same) panel_load(SB, kp, g.B.item(bb), g.B.cn, g.bi, g.bj, n, 8 * t.gn, (int)g.k, ttid, tthreads);
    }
  };
  if (b < g.batch) {
    load_item(b);
    stage_ab(b);
  }
  cp_async_commit();
  int cur = 0;
  for (; b < g.batch;) {
    ix nb = b + stride;
    while (nb < g.batch && skip(nb)) nb += stride;
    double *S = cur ? S1 : S0;
    if (DB && vin) {
      if (nb < g.batch) tri_load(cur ? S0 : S1, t, g.C.item(nb), g.C.cn, g.ci, g.cj, m, n, gm, true, ttid, tthreads);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
      if (bulk_in) {
        mbar_wait(tbar, phase);
        phase ^= 1;
      }
    }
    if (ttid == 0) *flag = -1;
    team_sync(bar, tthreads);

    int fail = -1;
    // Look-ahead left-looking schedule.  Tile rows are owned row-cyclically
    // (row group gg by warp gg % TW, slot i = gg / TW), so the diagonal
    // tile of column block jb belongs to warp jb % TW.  While that warp runs
    // the serial 8x8 factor + inverse, every other warp completes its
    // column-jb tiles and already accumulates the downdate of column block
    // jb+1 over blocks 0..jb-1 (acc_nx); the next step then adds only block
    // jb's contribution (two DMMAs) before factoring.
    double acc_nx[MAXT][2];
    bool prep = false;  // acc_nx holds column block jb's partial (blocks < jb-1 applied)
#pragma unroll
    for (int i = 0; i < MAXT; ++i) acc_nx[i][0] = acc_nx[i][1] = 0.0;
#pragma unroll(GN > 0 ? GN : 1)
    for (int jb = 0; jb < (GN > 0 ? GN : 64); ++jb) {
      if (GN == 0 && jb >= t.gn) break;
      const int ncol = min(8, n - 8 * jb);
      const bool is_d = TW == 1 || tw == jb % TW;
      double acc[MAXT][2];
      if (is_d) {
        // ---- diagonal warp: complete the diagonal tile, factor, invert
        const int id = jb / TW;  // slot of row group jb
        double dg[2];
        if (prep) {
          const int fb = tri_frag(t, jb, 0, lane) + 32 * (jb - 1);
          dg[0] = dg[1] = 0.0;
#pragma unroll
          for (int i = 0; i < MAXT; ++i)
            if (i == id) dg[0] = acc_nx[i][0], dg[1] = acc_nx[i][1];  // static register indexing
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) dmma(dg, -S[fb + 16 * kk], S[fb + 16 * kk]);
        } else {
          dg[0] = S[t.off(8 * jb + fr, 8 * jb + 2 * fc)];
          dg[1] = S[t.off(8 * jb + fr, 8 * jb + 2 * fc + 1)];
          if (SK) {
            const int pb = (2 * jb + (lane >> 4)) * 4 * kp + 4 * fc + (fr & 3);
#pragma unroll 4
            for (int kk = 0; kk < kp / 4; ++kk) dmma(dg, SA[pb + 16 * kk], SB[pb + 16 * kk]);
          }
          const int fb = tri_frag(t, jb, 0, lane);
#pragma unroll 4
          for (int kk = 0; kk < 2 * jb; ++kk) dmma(dg, -S[fb + 16 * kk], S[fb + 16 * kk]);
        }
        double wi[2];
        const int f = factor_inv_tile_u(dg, wi, ncol, dinv + 8 * jb, lane);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 2 * fc + e;
          if (c < ncol && (f < 0 || c < f)) S[t.off(8 * jb + fr, 8 * jb + c)] = dg[e];
        }
        if (f >= 0 && lane == 0) *flag = 8 * jb + f;
        if (f < 0 && jb + 1 < gm) store_inv_block(wi, Wp, lane);
        // then this warp's other column-jb tiles
        if (prep) add_block_tiles<MAXT, TW>(acc, acc_nx, S, t, tw, gm, jb + 1, jb, jb - 1, lane);
        else downdate_tiles<MAXT, TW, SK>(acc, S, t, SA, SB, kp, tw, gm, jb + 1, jb, jb, lane);
      } else {
        // ---- other warps: column-jb tiles now, column-(jb+1) partials next
        if (prep) add_block_tiles<MAXT, TW>(acc, acc_nx, S, t, tw, gm, jb + 1, jb, jb - 1, lane);
        else downdate_tiles<MAXT, TW, SK>(acc, S, t, SA, SB, kp, tw, gm, jb + 1, jb, jb, lane);
      }
      // park the column-jb tiles below the diagonal (A operand of the solve)
#pragma unroll
      for (int i = 0; i < MAXT; ++i) {
        const int gg = tw + i * TW;
        if (gg > jb && gg < gm) {
#pragma unroll
          for (int e = 0; e < 2; ++e) S[t.off(8 * gg + fr, 8 * jb + 2 * fc + e)] = acc[i][e];
        }
      }
      const bool look = TW > 1 && !is_d && jb + 1 < t.gn;
      if (look) downdate_tiles<MAXT, TW, SK>(acc_nx, S, t, SA, SB, kp, tw, gm, jb + 1, jb + 1, jb, lane);
      team_sync(bar, tthreads);
      fail = *flag;
      if (fail >= 0) break;
      // solve the tiles below the diagonal: X := X * L_jj^{-T} on DMMA
#pragma unroll
      for (int i = 0; i < MAXT; ++i) {
        const int gg = tw + i * TW;
        if (gg > jb && gg < gm) {
          apply_inv_block(acc[i], S, t, gg, jb, Wp, lane);
          __syncwarp();
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 2 * fc + e;
            if (c < ncol) S[t.off(8 * gg + fr, 8 * jb + c)] = acc[i][e];
          }
        }
      }
      prep = look;
      team_sync(bar, tthreads);
    }

    // write back the lower trapezoid (or, on failure, exactly what the
    // reference's block-row order would have stored, ccore.pyx:884-899)
    double *D = g.D.item(b);
    const int iif = fail >= 0 ? (fail & ~3) : 0;
    if (fail < 0 && bulk_out) {
      // whole 4-row panels strictly below the diagonal: one bulk store
      // each (thread 0); the 4x4 diagonal pieces and a partial last panel
      // element-wise.  The loop's last team_sync ordered every thread's
      // shared stores; the fence hands them to the async proxy.
      fence_proxy_async();
      team_sync(bar, tthreads);
      for (int gg = 0; gg < gm; ++gg) {
        const int w = t.width(gg), base = t.group_off(gg);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r0 = 8 * gg + 4 * h;
          if (r0 >= m) continue;
          const double *src = S + base + h * 4 * w;
          const bool full = r0 + 4 <= m;
          const int cl = full ? min(r0, n) : 0;
          if (cl > 0 && ttid == 0) tma_store_1d(D + eo(g.di + r0, g.dj, g.D.cn), src, 32u * (unsigned)cl);
          const int ce = min(r0 + 4, n);
          for (int q = ttid; q < 4 * (ce - cl); q += tthreads) {
            const int c = cl + (q >> 2), r = r0 + (q & 3);
            if (r < m && c <= r) D[eo(g.di + r, g.dj + c, g.D.cn)] = src[4 * c + (q & 3)];
          }
        }
      }
      if (ttid == 0) bulk_commit();
    } else if (fail < 0 || aligned_out) {
      for (int gg = 0; gg < gm; ++gg) {
        const int w = t.width(gg), base = t.group_off(gg);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int rp = 8 * gg + 4 * half;
          if (rp >= m) continue;
          if (vec_out) {
            for (int q = ttid; q < 2 * w; q += tthreads) {
              const int c = q >> 1, r0 = rp + 2 * (q & 1);
              bool w0 = r0 < m && c < n && c <= r0, w1 = r0 + 1 < m && c < n && c <= r0 + 1;
              if (fail >= 0) {
                w0 = w0 && (r0 < iif || (r0 < iif + 4 && c < iif));
                w1 = w1 && (r0 + 1 < iif || (r0 + 1 < iif + 4 && c < iif));
              }
              const double *src = S + base + half * 4 * w + 4 * c + 2 * (q & 1);
              double *dst = D + eo(g.di + r0, g.dj + c, g.D.cn);
              if (w0 && w1) *reinterpret_cast<double2 *>(dst) = *reinterpret_cast<const double2 *>(src);
              else if (w0) dst[0] = src[0];
              else if (w1) dst[1] = src[1];
            }
          } else {
            for (int q = ttid; q < 4 * w; q += tthreads) {
              const int c = q >> 2, r = rp + (q & 3);
              bool st = r < m && c < n && c <= r;
              if (fail >= 0) st = st && (r < iif || (r < iif + 4 && c < iif));
              if (st) D[eo(g.di + r, g.dj + c, g.D.cn)] = S[base + half * 4 * w + q];
            }
          }
        }
      }
    }
    double *dA = g.D.ditem(b);
    const int nd = fail >= 0 ? fail : n;
    for (int c = ttid; c < nd; c += tthreads) dA[g.dj + c] = dinv[c];
    if (ttid == 0 && g.info) g.info[b] = fail >= 0 ? fail + g.info_offset : -1;
    if (bulk_out && ttid == 0) bulk_wait_read0();  // S is free once the stores have read it
    team_sync(bar, tthreads);
    b = nb;
    if (DB && vin) cur ^= 1;
    else if (b < g.batch) {
      load_item(b);
      stage_ab(b);
      cp_async_commit();
    }
  }
  cp_async_wait<0>();
  if (bulk_out && ttid == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------
// trsm_rltn team kernel: D * A^T = alpha * B

template <int TW>
__global__ void __launch_bounds__(256) trsm_team_kernel(TrsmArgs g, int team_elems, int vec_in) {
  extern __shared__ __align__(128) double smem[];
  const int lane = threadIdx.x & 31, warp = warp_uniform();
  const int team = warp / TW, tw = warp % TW;
  const int teams_per_cta = (blockDim.x >> 5) / TW;
  const int tthreads = TW * 32, ttid = tw * 32 + lane;
  // one team per CTA (launch_trsm): the team barrier is the CTA barrier -- a runtime named-barrier id would
  // reserve all 16 hardware barriers and cap the SM at 4 CTAs
  auto team_sync = [&](int, int) { __syncthreads(); };
  const int bar = 0;
  const int m = (int)g.m, n = (int)g.n;
  Tri t;
  t.cn8 = (n + 7) / 8 * 8;
  t.gn = t.cn8 / 8;
  const int tri_elems = (int)Tri::size(n, n);
  double *S = smem + (ix)team * team_elems;
  double *dinv = S + tri_elems;
  double *Wall = dinv + t.cn8 + 8;                      // gn inverted diagonal blocks
  double *strip = Wall + 64 * t.gn + tw * 8 * t.cn8;    // this warp's rows, 2 panels x cn8
  const int fr = lane >> 2, fc = lane & 3;
  const int gmr = (m + 7) / 8;
  const int fa = (lane >> 4) * 4 * t.cn8 + 4 * fc + ((lane >> 2) & 3);

  for (ix b = (ix)blockIdx.x * teams_per_cta + team; b < g.batch; b += (ix)gridDim.x * teams_per_cta) {
    if (g.skip && g.skip[b] >= 0) continue;
    tri_load(S, t, g.A.item(b), g.A.cn, g.ai, g.aj, n, n, t.gn, vec_in != 0, ttid, tthreads);
    cp_async_commit();
    cp_async_wait<0>();
    team_sync(bar, tthreads);
    // reciprocals: reuse the factorization's, or compute (zero -> info);
    // use_dA == 2 decides per item: reuse where the factorization succeeded
    // (info on entry < 0), compute where it failed (its diag_inv is invalid,
    // level3.py:346-349)
    const bool reuse = g.use_dA == 1 || (g.use_dA == 2 && g.info[b] < 0);
    if (reuse) {
      const double *dA = g.A.ditem(b);
      for (int c = ttid; c < n; c += tthreads) dinv[c] = dA[g.aj + c];
    } else {
      for (int c = ttid; c < n; c += tthreads) dinv[c] = 1.0 / S[t.off(c, c)];
    }
    team_sync(bar, tthreads);
    // first zero pivot (level3.py:171-175): the item is then left untouched
    int fail = -1;
    if (!reuse) {
      for (int c = 0; c < n; ++c)
        if (S[t.off(c, c)] == 0.0) { fail = c; break; }
    }
    if (fail < 0) {
      // inverse of every 8x8 diagonal block, spread over the team's warps
      for (int jb = tw; jb < t.gn; jb += TW) {
        double xl[2], wv[2];
        xl[0] = S[t.off(8 * jb + fr, 8 * jb + 2 * fc)];
        xl[1] = S[t.off(8 * jb + fr, 8 * jb + 2 * fc + 1)];
        inv_tile_regs(xl, dinv + 8 * jb, min(8, n - 8 * jb), wv, lane);
        store_inv_block(wv, Wall + 64 * jb, lane);
      }
      team_sync(bar, tthreads);
      const double *B = g.B.item(b);
      double *D = g.D.item(b);
      for (int gg = tw; gg < gmr; gg += TW) {
        const int r = 8 * gg + fr;
        for (int jb = 0; jb < t.gn; ++jb) {
          double x[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 8 * jb + 2 * fc + e;
            x[e] = (r < m && c < n) ? __dmul_rn(g.alpha, B[eo(g.bi + r, g.bj + c, g.B.cn)]) : 0.0;
          }
          const int fb = tri_frag(t, jb, 0, lane);
#pragma unroll 4
          for (int kk = 0; kk < 2 * jb; ++kk) dmma(x, -strip[fa + 16 * kk], S[fb + 16 * kk]);
          // x := x * L_jj^{-T} via the inverted block (two DMMAs)
#pragma unroll
          for (int e = 0; e < 2; ++e) strip[((fr >> 2) * 4 * t.cn8) + 4 * (8 * jb + 2 * fc + e) + (fr & 3)] = x[e];
          __syncwarp();
          const double *W = Wall + 64 * jb;
          const int fw = (lane >> 4) * 32 + 4 * fc + (fr & 3);
          x[0] = x[1] = 0.0;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) dmma(x, strip[fa + 32 * jb + 16 * kk], W[fw + 16 * kk]);
          __syncwarp();
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 8 * jb + 2 * fc + e;
            strip[((fr >> 2) * 4 * t.cn8) + 4 * c + (fr & 3)] = x[e];
            if (r < m && c < n) D[eo(g.di + r, g.dj + c, g.D.cn)] = x[e];
          }
          __syncwarp();
        }
      }
    }
    if (ttid == 0 && g.info) g.info[b] = fail;
    team_sync(bar, tthreads);
  }
}

// ---------------------------------------------------------------------------
// host dispatch

static int pick_teams(int tw, ix team_elems, int &threads, size_t &smem) {
  int teams = 8 / tw;
  if (teams < 1) teams = 1;
  const size_t cap = 200 * 1024;
  while (teams > 1 && (size_t)teams * team_elems * sizeof(double) > cap) --teams;
  threads = teams * tw * 32;
  smem = (size_t)teams * team_elems * sizeof(double);
  return teams;
}

static ix syrk_operand_elems(ix m, ix n, ix k, bool ab_same) {
  const ix kp = (k + 3) & ~(ix)3;
  return (m + 7) / 8 * 8 * kp + (ab_same ? 0 : (n + 7) / 8 * 8 * kp);
}

template <int TW, int MAXT, bool DB, int GM = 0, int GN = 0, bool SK = false, int MINB = 1>
static cudaError_t launch_potrf(const PotrfArgs &g, cudaStream_t st) {
  auto kern = potrf_team_kernel<TW, MAXT, DB, GM, GN, SK, MINB>;
  const ix cn8 = (g.n + 7) / 8 * 8;
  ix team_elems = Tri::size(g.m, g.n) * (DB ? 2 : 1) + cn8 + 8 + 64 +
                  (SK ? syrk_operand_elems(g.m, g.n, g.k, g.ab_same != 0) : 0);
  team_elems = (team_elems + 15) / 16 * 16;
  int threads;
  size_t smem;
  const int teams = pick_teams(TW, team_elems, threads, smem);
  static LaunchCache cache;
  const int occ = cache.occupancy((const void *)kern, threads, smem);
  ix grid = (g.batch + teams - 1) / teams;
  const ix cap = (ix)num_sms() * occ;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  const int vin = (g.ci & 3) == 0 && ((uintptr_t)g.C.p & 15) == 0 && (g.C.stride & 1) == 0;
  const int vout = (g.di & 3) == 0 && ((uintptr_t)g.D.p & 15) == 0 && (g.D.stride & 1) == 0;
  kern<<<(unsigned)grid, threads, smem, st>>>(g, (int)team_elems, vin, vout);
  note_launch();
  return cudaGetLastError();
}

bool potrf_fits(ix m, ix n) {
  const ix cn8 = (n + 7) / 8 * 8;
  const ix e = Tri::size(m, n) + cn8 + 8 + 64;
  const ix gm = (m + 7) / 8;
  return e * 8 <= 220 * 1024 && gm <= 8 * 8;
}

cudaError_t run_potrf_l(const PotrfArgs &g, cudaStream_t st) {
  if (potrf_small_ok(g)) return run_potrf_small(g, st);
  if (potrf_reg_ok(g)) return run_potrf_reg(g, st);
  if (potrf_chain_ok(g)) return run_potrf_chain(g, st);
  const ix gm = (g.m + 7) / 8;
  const bool db = Tri::size(g.m, g.n) * 8 <= 40 * 1024;  // double-buffer while it fits 2+ teams/SM
  const ix gn = (g.n + 7) / 8;
  // compile-time shaped instances for the common (benchmark) sizes
  // measured on B200 (profiles/r01_potrf_team_tuning.txt): more, smaller
  // teams without double buffering win where the diagonal chain dominates
  if (gm == 4 && gn == 4) return launch_potrf<1, 4, false, 4, 4, false, 4>(g, st);
  if (gm == 8 && gn == 8) return launch_potrf<2, 4, false, 8, 8, false, 3>(g, st);
  if (gm <= 2) return db ? launch_potrf<1, 2, true, 0, 0, false, 4>(g, st) : launch_potrf<1, 2, false, 0, 0, false, 4>(g, st);
  if (gm <= 4) return db ? launch_potrf<1, 4, true, 0, 0, false, 4>(g, st) : launch_potrf<1, 4, false, 0, 0, false, 4>(g, st);
  if (gm <= 8) return db ? launch_potrf<4, 2, true, 0, 0, false, 3>(g, st) : launch_potrf<4, 2, false, 0, 0, false, 3>(g, st);
  if (gm <= 16) return launch_potrf<8, 2, false, 0, 0, false, 3>(g, st);
  if (gm <= 32) return launch_potrf<8, 4, false, 0, 0, false, 2>(g, st);
  return launch_potrf<8, 8, false>(g, st);
}

bool syrk_potrf_fits(ix m, ix n, ix k, bool ab_same) {
  const ix cn8 = (n + 7) / 8 * 8;
  const ix e = Tri::size(m, n) + cn8 + 8 + 64 + syrk_operand_elems(m, n, k, ab_same);
  return e * 8 <= 220 * 1024 && (m + 7) / 8 <= 8 * 8;
}

// fused syrk + potrf: single-buffered generic team shapes
cudaError_t run_syrk_potrf(const PotrfArgs &g, cudaStream_t st) {
  if (potrf_reg_ok(g)) return run_potrf_reg(g, st);
  const ix gm = (g.m + 7) / 8;
  if (gm <= 2) return launch_potrf<1, 2, false, 0, 0, true, 4>(g, st);
  if (gm <= 4) return launch_potrf<1, 4, false, 0, 0, true, 4>(g, st);
  if (gm <= 8) return launch_potrf<4, 2, false, 0, 0, true, 3>(g, st);
  if (gm <= 16) return launch_potrf<8, 2, false, 0, 0, true, 3>(g, st);
  if (gm <= 32) return launch_potrf<8, 4, false, 0, 0, true, 2>(g, st);
  return launch_potrf<8, 8, false, 0, 0, true>(g, st);
}

bool trsm_fits(ix m, ix n) {
  (void)m;
  const ix cn8 = (n + 7) / 8 * 8;
  const ix e = Tri::size(n, n) + cn8 + 8 + 64 * (cn8 / 8) + 8 * 8 * cn8;
  return e * 8 <= 220 * 1024;
}

template <int TW>
static cudaError_t launch_trsm(const TrsmArgs &g, cudaStream_t st) {
  auto kern = trsm_team_kernel<TW>;
  const ix cn8 = (g.n + 7) / 8 * 8;
  ix team_elems = Tri::size(g.n, g.n) + cn8 + 8 + 64 * (cn8 / 8) + (ix)TW * 8 * cn8;
  team_elems = (team_elems + 15) / 16 * 16;
  const int teams = 1, threads = TW * 32;  // a CTA is one team (see the barrier note in the kernel)
  const size_t smem = (size_t)team_elems * sizeof(double);
  static LaunchCache cache;
  static bool carve = false;
  if (!carve) {  // small triangles: many CTAs per SM want the largest shared-memory carve-out
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    carve = true;
  }
  const int occ = cache.occupancy((const void *)kern, threads, smem);
  ix grid = (g.batch + teams - 1) / teams;
  const ix cap = (ix)num_sms() * occ;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  const int vin = (g.ai & 3) == 0 && ((uintptr_t)g.A.p & 15) == 0 && (g.A.stride & 1) == 0;
  kern<<<(unsigned)grid, threads, smem, st>>>(g, (int)team_elems, vin);
  note_launch();
  return cudaGetLastError();
}

// first zero on the diagonal of each item's n x n window (level3.py:171-175)
__global__ void diag_check_kernel(Mat A, ix ai, ix aj, ix n, ix batch, int32_t *info) {
  for (ix b = (ix)blockIdx.x * blockDim.x + threadIdx.x; b < batch; b += (ix)gridDim.x * blockDim.x) {
    const double *p = A.item(b);
    int f = -1;
    for (ix j = 0; j < n; ++j)
      if (p[eo(ai + j, aj + j, A.cn)] == 0.0) { f = (int)j; break; }
    info[b] = f;
  }
}

cudaError_t run_diag_check(const Mat &A, ix ai, ix aj, ix n, ix batch, int32_t *info, cudaStream_t st) {
  ix blocks = (batch + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  diag_check_kernel<<<(unsigned)blocks, 256, 0, st>>>(A, ai, aj, n, batch, info);
  note_launch();
  return cudaGetLastError();
}

cudaError_t run_trsm_rltn(const TrsmArgs &g, cudaStream_t st) {
  if (trsm_wide_ok(g)) return run_trsm_wide(g, st);  // register-resident strips (pb_trsm_wide.cu)
  // team width: the warps of a team take the item's 8-row strips round-robin
  // and meet at a barrier per item, so pick the width with the best strip
  // utilisation gmr / (TW * rounds) (ties -> wider team, fewer rounds): e.g.
  // C4's m = 72 (9 strips) runs 3 rounds on 3 warps instead of 2 on 8
  const ix gmr = (g.m + 7) / 8;
  static const int widths[6] = {8, 6, 4, 3, 2, 1};
  int best = 1;
  double bu = -1.0;
  for (int w : widths) {
    const ix rounds = (gmr + w - 1) / w;
    const double u = (double)gmr / (double)(w * rounds);
    if (u > bu + 1e-9) bu = u, best = w;
  }
  switch (best) {
    case 8: return launch_trsm<8>(g, st);
    case 6: return launch_trsm<6>(g, st);
    case 4: return launch_trsm<4>(g, st);
    case 3: return launch_trsm<3>(g, st);
    case 2: return launch_trsm<2>(g, st);
    default: return launch_trsm<1>(g, st);
  }
}

}  // namespace pb
