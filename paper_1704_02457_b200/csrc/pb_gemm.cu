// Batched dgemm_nt / dsyrk_ln on panel-major FP64 storage (sm_100a).
//
// Reference semantics: gemm_nt_drv ccore.pyx:746-771 (+ _store_block
// :26-42), syrk_ln_drv ccore.pyx:804-831 (+ _ksyrk_core :275-293).
//
// Two kernel families, both on the FP64 tensor path (mma.sync m8n8k4 f64,
// SASS DMMA.8x8x4; on B200 DMMA and DFMA share the same 37 TF/s peak, see
// profiles/r01_fp64_peak.log, but DMMA needs 1/8 of the issue slots and
// shares each fragment across an 8x8 tile instead of re-reading it):
//
//  * gemm_direct: one warp per item for tiny items (m, n <= 24).  The
//    panel-major layout makes every A/B fragment two contiguous 128-byte
//    runs, so fragments are read straight from HBM, fully coalesced, with
//    no shared-memory staging at all.
//  * gemm_tiled: persistent CTAs stream (item, tile, k-chunk) steps
//    through a cp.async multi-stage shared-memory pipeline that crosses
//    item boundaries, so the next item's operands are in flight while the
//    current item's epilogue drains.
//
// Both honour the reference's discrete semantics exactly: alpha == 0
// never touches A/B (NaN-safe), beta == 0 never reads C, writes stay in
// the m x n window (syrk: lower triangle only), unaligned row origins are
// gathered in-kernel instead of the reference's host repack
// (level3.py:56-62).
#include <cstdlib>
#include <string>

#include "pb_gemm.cuh"

namespace pb {

// _store_block rule (ccore.pyx:26-42); no contraction so alpha=1/beta=0
// and the special cases are exact.
__device__ __forceinline__ double store_rule(double alpha, double acc, double beta, double c) {
  if (alpha != 0.0) {
    double v = __dmul_rn(alpha, acc);
    if (beta != 0.0) v = __dadd_rn(v, __dmul_rn(beta, c));
    return v;
  }
  return beta != 0.0 ? __dmul_rn(beta, c) : 0.0;
}
// _ksyrk_core diagonal-tile rule (ccore.pyx:288-292).
__device__ __forceinline__ double syrk_diag_rule(double alpha, double acc, double beta, double c) {
  double v = beta != 0.0 ? __dmul_rn(beta, c) : 0.0;
  if (alpha != 0.0) v = __dadd_rn(__dmul_rn(alpha, acc), v);
  return v;
}

template <bool SYRK>
__device__ __forceinline__ bool in_store(ix r, ix c, ix m, ix n) {
  return r < m && c < n && (!SYRK || r >= c);
}

template <bool SYRK>
__device__ __forceinline__ double epilogue_value(const GemmArgs &g, ix r, ix c, double acc, double cv) {
  if (SYRK && ((r >> 2) == (c >> 2))) return syrk_diag_rule(g.alpha, acc, g.beta, cv);
  return store_rule(g.alpha, acc, g.beta, cv);
}

// unit -> (item, tile row, tile column).  Every warp of a CTA calls this once per unit, and a 64-bit division is an
// out-of-line ~80-instruction routine (two of them were as many instructions as a warp's share of a 32 x 32 x 36
// tile): one tile per item needs no division at all, and unit indices below 2^32 divide in 32 bits.
__device__ __forceinline__ void unit_coords(ix u, ix tiles_m, ix tiles_n, bool syrk, ix &b, ix &tm, ix &tn) {
  const ix per = syrk ? tiles_m * (tiles_m + 1) / 2 : tiles_m * tiles_n;
  if (per == 1) {
    b = u, tm = 0, tn = 0;
    return;
  }
  unsigned t;
  if (((unsigned long long)u >> 32) == 0 && ((unsigned long long)per >> 32) == 0) {
    const unsigned uu = (unsigned)u, pp = (unsigned)per, q = uu / pp;
    b = q, t = uu - q * pp;
  } else {
    b = u / per;
    t = (unsigned)(u - b * per);  // tiles per item fit 32 bits (m, n < 2^31 / tile)
  }
  if (!syrk) {
    const unsigned tnn = (unsigned)tiles_n, q = t / tnn;
    tm = q, tn = t - q * tnn;
  } else {
    // lower-triangular tile index -> (tm, tn), tn <= tm
    unsigned r = (unsigned)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
    while (r * (r + 1) / 2 > t) --r;
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    tm = r;
    tn = t - r * (r + 1) / 2;
  }
}

// B-operand modes.  BOP_NT: B is n x k, fragments read along B's rows
// (gemm_nt / syrk).  BOP_NN: B is k x n read down its columns across
// panels (gemm_nn_drv ccore.pyx:774-801).  BOP_TRI: BOP_NN with B an n x n
// lower-triangular right factor, entries above its diagonal read as 0 and
// D = alpha*acc with no C term (trmm_rlnn_drv ccore.pyx:834-852,
// _ktrmm_core :305-349).
enum { BOP_NT = 0, BOP_NN = 1, BOP_TRI = 2 };

// ---------------------------------------------------------------------------
// gemm_direct: one warp per (item, 8MT x 8NT output tile), fragments
// straight from global memory.  Used for tiny items (one tile per item)
// and as the any-alignment fallback of the NN modes.

// ONE: the tile is the whole item (every window the tiny-item dispatch sends here): unit = item, and the
// per-lane fragment / accumulator offsets are hoisted out of the unit loop (no 64-bit divisions, no eo()
// products per fragment -- ~300 -> ~80 instructions per 8 x 8 x 8 item).
template <int MT, int NT, bool SYRK, int BOP = BOP_NT, int MINB = 1, bool ONE = false>
__global__ void __launch_bounds__(256, MINB) gemm_direct_kernel(GemmArgs g, ix tiles_m, ix tiles_n, ix nunits) {
  const int lane = threadIdx.x & 31;
  const ix warp = (ix)blockIdx.x * (blockDim.x >> 5) + warp_uniform();
  const ix nwarps = (ix)gridDim.x * (blockDim.x >> 5);
  const int fr = lane >> 2, fc = lane & 3;  // fragment row / k-col
  const ix ncols = SYRK ? g.m : g.n;
  ix hA[MT], hB[NT], hC[MT], hD[MT];
  if constexpr (ONE) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      hA[i] = eo(g.ai + 8 * i + fr, g.aj + fc, g.A.cn);
      hC[i] = eo(g.ci + 8 * i + fr, g.cj + 2 * fc, g.C.cn);
      hD[i] = eo(g.di + 8 * i + fr, g.dj + 2 * fc, g.D.cn);
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) hB[j] = eo(g.bi + 8 * j + fr, g.bj + fc, g.B.cn);
  }
  for (ix u = warp; u < nunits; u += nwarps) {
    ix b, tm, tn;
    if constexpr (ONE) b = u, tm = 0, tn = 0;
    else unit_coords(u, tiles_m, tiles_n, SYRK, b, tm, tn);
    if (g.skip && g.skip[b] >= 0) continue;
    const ix rbase = tm * (8 * MT), cbase = tn * (8 * NT);
    const double *A = g.A.item(b);
    const double *B = g.B.item(b);
    const double *C = g.C.item(b);
    double *D = g.D.item(b);
    double cv[MT][NT][2];
    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          acc[i][j][e] = 0.0;
          cv[i][j][e] = 0.0;
          const ix r = rbase + 8 * i + fr, c = cbase + 8 * j + 2 * fc + e;
          if (BOP != BOP_TRI && g.beta != 0.0 && in_store<SYRK>(r, c, g.m, g.n))
            cv[i][j][e] = ONE ? C[hC[i] + 4 * (8 * j + e)] : C[eo(g.ci + r, g.cj + c, g.C.cn)];
        }
    if (g.alpha != 0.0 || BOP == BOP_TRI) {
      // triangular B: rows above this tile's first column are all zero
      const ix kstart = BOP == BOP_TRI ? (cbase & ~(ix)3) : 0;
      // KU k-steps of fragments are loaded before their DMMAs, so a unit
      // exposes one global-load latency per 4*KU columns, not one per 4
      // (measured on the C3 sweep: KU = 4 up to 2x2 tiles, KU = 2 for the
      // 3x3-tile units, faster even with the few spills it costs at the
      // 85-register cap)
      constexpr int KU = MT * NT <= 4 ? 4 : 2;
      for (ix k0 = kstart; k0 < g.k; k0 += 4 * KU) {
        double a[KU][MT], bb[KU][NT];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          const ix l = k0 + 4 * u + fc;
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const ix r = rbase + 8 * i + fr;
            a[u][i] = (r < g.m && l < g.k) ? ldg_nc(ONE ? A + hA[i] + 4 * (l - fc) : A + eo(g.ai + r, g.aj + l, g.A.cn)) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const ix r = cbase + 8 * j + fr;
            if (BOP == BOP_NT)
              bb[u][j] = (r < ncols && l < g.k) ? ldg_nc(ONE ? B + hB[j] + 4 * (l - fc) : B + eo(g.bi + r, g.bj + l, g.B.cn)) : 0.0;
            else
              bb[u][j] = (r < ncols && l < g.k && (BOP != BOP_TRI || l >= r))
                             ? ldg_nc(B + eo(g.bi + l, g.bj + r, g.B.cn))
                             : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          if (k0 + 4 * u < g.k) {  // no zero-fragment steps past k (keeps -0.0 results exact)
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
              for (int j = 0; j < NT; ++j)
                if (!SYRK || j <= i) dmma(acc[i][j], a[u][i], bb[u][j]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const ix r = rbase + 8 * i + fr, c = cbase + 8 * j + 2 * fc + e;
          if (in_store<SYRK>(r, c, g.m, g.n))
            D[ONE ? hD[i] + 4 * (8 * j + e) : eo(g.di + r, g.dj + c, g.D.cn)] = BOP == BOP_TRI ? __dmul_rn(g.alpha, acc[i][j][e])
                                                               : epilogue_value<SYRK>(g, r, c, acc[i][j][e], cv[i][j][e]);
        }
  }
}

// ---------------------------------------------------------------------------
// gemm_tiled: persistent, cp.async multi-stage pipeline over
// (unit = item x output tile, k-chunk) steps.

template <int BM, int BN, int WM, int WN, int KC, int STAGES>
struct TiledCfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NWARPS = WARPS_M * WARPS_N;
  static constexpr int NTHREADS = 32 * NWARPS;
  static constexpr int MT = WM / 8, NT = WN / 8;
  static constexpr int A_ELEMS = BM * KC, B_ELEMS = BN * KC;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = sizeof(double) * STAGE_ELEMS * STAGES;
};

// Load a (ROWS x KC) panel tile of window rows [r0, r0+ROWS), cols
// [l0, l0+KC) into shared memory (panel-major, panel length KC).
// Rows >= rows_valid and cols >= k are zero-filled without reading.
template <int ROWS, int KC, int NTHREADS>
__device__ __forceinline__ void load_panel_tile(double *s, const double *G, ix cn, ix gi, ix gj, ix r0, ix l0,
                                                ix rows_valid, ix k, bool vec16) {
  if (vec16) {
    // 16-byte pieces: (panel p, col l, half h) -> rows 4p+2h, 4p+2h+1.
    constexpr int PIECES = (ROWS / 4) * KC * 2;
#pragma unroll 4
    for (int q = threadIdx.x; q < PIECES; q += NTHREADS) {
      const int p = q / (2 * KC), w = q % (2 * KC), l = w >> 1, h = w & 1;
      const ix R = r0 + 4 * p + 2 * h, L = l0 + l;
      const bool ok = R < rows_valid && L < k;
      const double *src = ok ? G + eo(gi + R, gj + L, cn) : G;
      cp_async16(s + p * 4 * KC + 4 * l + 2 * h, src, ok ? 16 : 0);
    }
  } else {
    constexpr int ELEMS = ROWS * KC;
#pragma unroll 4
    for (int q = threadIdx.x; q < ELEMS; q += NTHREADS) {
      const int p = q / (4 * KC), w = q % (4 * KC), l = w >> 2, rr = w & 3;
      const ix R = r0 + 4 * p + rr, L = l0 + l;
      const bool ok = R < rows_valid && L < k;
      const double *src = ok ? G + eo(gi + R, gj + L, cn) : G;
      cp_async8(s + p * 4 * KC + 4 * l + rr, src, ok ? 8 : 0);
    }
  }
}

template <int BM, int BN, int WM, int WN, int KC, int STAGES, bool SYRK>
__global__ void __launch_bounds__(TiledCfg<BM, BN, WM, WN, KC, STAGES>::NTHREADS)
    gemm_tiled_kernel(GemmArgs g, ix tiles_m, ix tiles_n, ix nunits) {
  using Cfg = TiledCfg<BM, BN, WM, WN, KC, STAGES>;
  constexpr int MT = Cfg::MT, NT = Cfg::NT;
  extern __shared__ __align__(128) double smem[];
  const int lane = threadIdx.x & 31, warp = warp_uniform();
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  const int fr = lane >> 2, fc = lane & 3;

  const ix nk = g.alpha != 0.0 ? (g.k + KC - 1) / KC : 0;
  const ix steps_per_unit = nk > 0 ? nk : 1;
  const ix my_units = blockIdx.x < nunits ? (nunits - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const ix nsteps = my_units * steps_per_unit;
  const bool vecA = g.vecA, vecB = g.vecB;

  auto issue = [&](ix s) {
    const ix u = blockIdx.x + (s / steps_per_unit) * gridDim.x;
    const ix ch = s % steps_per_unit;
    ix b, tm, tn;
    unit_coords(u, tiles_m, tiles_n, SYRK, b, tm, tn);
    double *st = smem + (s % STAGES) * Cfg::STAGE_ELEMS;
    load_panel_tile<BM, KC, Cfg::NTHREADS>(st, g.A.item(b), g.A.cn, g.ai, g.aj, tm * BM, ch * KC, g.m, g.k, vecA);
    load_panel_tile<BN, KC, Cfg::NTHREADS>(st + Cfg::A_ELEMS, g.B.item(b), g.B.cn, g.bi, g.bj, tn * BN, ch * KC,
                                           SYRK ? g.m : g.n, g.k, vecB);
  };

  if (nk > 0) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nsteps) issue(s);
      cp_async_commit();
    }
  }

  double acc[MT][NT][2];
  double cv[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (ix s = 0; s < nsteps; ++s) {
    const ix u = blockIdx.x + (s / steps_per_unit) * gridDim.x;
    const ix ch = s % steps_per_unit;
    ix b, tm, tn;
    unit_coords(u, tiles_m, tiles_n, SYRK, b, tm, tn);
    const ix rbase = tm * BM + wm * WM, cbase = tn * BN + wn * WN;
    if (ch == 0 && g.beta != 0.0) {
      // prefetch this unit's C fragments; consumed in the epilogue
      const double *C = g.C.item(b);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const ix r = rbase + 8 * i + fr, c = cbase + 8 * j + 2 * fc + e;
            cv[i][j][e] = in_store<SYRK>(r, c, g.m, g.n) ? ldg_nc(C + eo(g.ci + r, g.cj + c, g.C.cn)) : 0.0;
          }
    }
    if (nk > 0) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      if (s + STAGES - 1 < nsteps) issue(s + STAGES - 1);
      cp_async_commit();
      const double *sa = smem + (s % STAGES) * Cfg::STAGE_ELEMS + (wm * WM / 4) * 4 * KC;
      const double *sb = smem + (s % STAGES) * Cfg::STAGE_ELEMS + Cfg::A_ELEMS + (wn * WN / 4) * 4 * KC;
      const bool active = !SYRK || (cbase <= rbase + WM - 1);
      if (active) {
        const int foff = (lane >> 4) * 4 * KC + 4 * fc + (fr & 3);
#pragma unroll
        for (int kk = 0; kk < KC / 4; ++kk) {
          double a[MT], bb[NT];
#pragma unroll
          for (int i = 0; i < MT; ++i) a[i] = sa[i * 8 * KC + 16 * kk + foff];
#pragma unroll
          for (int j = 0; j < NT; ++j) bb[j] = sb[j * 8 * KC + 16 * kk + foff];
#pragma unroll
          for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma(acc[i][j], a[i], bb[j]);
        }
      }
    }
    if (ch == steps_per_unit - 1) {
      double *D = g.D.item(b);
      const bool skip = g.skip && g.skip[b] >= 0;
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const ix r = rbase + 8 * i + fr, c = cbase + 8 * j + 2 * fc + e;
            if (!skip && in_store<SYRK>(r, c, g.m, g.n))
              D[eo(g.di + r, g.dj + c, g.D.cn)] =
                  epilogue_value<SYRK>(g, r, c, acc[i][j][e], g.beta != 0.0 ? cv[i][j][e] : 0.0);
            acc[i][j][e] = 0.0;
          }
    }
  }
  if (nk > 0) cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// gemm_tma: persistent CTAs, TMA bulk-copy pipeline.  In panel-major every
// (4-row panel x KC-column chunk) of an operand tile is ONE contiguous run
// of 32*KC bytes, so a stage is a handful of cp.async.bulk copies issued by
// one warp and tracked by an mbarrier -- no per-element address math.
// Window rows that do not start on a panel boundary (ai % 4 != 0) copy one
// extra panel and index fragments with the constant row shift ai % 4, so
// unaligned stream operands need no repack (level3.py:56-62).

template <int BM, int BN, int WM, int WN, int KC, int STAGES, int CB, int BOP = BOP_NT>
struct TmaCfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NWARPS = WARPS_M * WARPS_N;      // consumer (MMA) warps
  static constexpr int NTHREADS = 32 * (NWARPS + 1);    // + one producer (TMA) warp
  static constexpr int MT = WM / 8, NT = WN / 8;
  static constexpr int PA = BM / 4 + 1;                  // panels per A tile
  // B tile: NT -> BN/4+1 panels x KC columns; NN -> KC/4+1 panels x BN columns
  static constexpr int B_PANEL = BOP == BOP_NT ? KC : BN;
  static constexpr int PB = BOP == BOP_NT ? BN / 4 + 1 : KC / 4 + 1;
  static constexpr int A_ELEMS = PA * 4 * KC, B_ELEMS = PB * 4 * B_PANEL;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr int C_ELEMS = PA * 4 * BN;            // one C tile (panels x BN columns)
  static constexpr size_t SMEM = sizeof(double) * (STAGE_ELEMS * STAGES + C_ELEMS * CB) + 16 * (STAGES + CB);
};

// First k-chunk a unit needs: a lower-triangular B has no nonzero rows
// above the tile's first column.
template <int BN, int KC, int BOP>
__device__ __forceinline__ ix first_chunk(ix tn) {
  return BOP == BOP_TRI ? (tn * BN) / KC : 0;
}

// Warp-specialised: warp NWARPS is the producer (bulk copies gated by
// per-stage "empty" mbarriers), warps 0..NWARPS-1 consume stages gated by
// "full" mbarriers -- no CTA-wide barrier in the main loop.  With CB > 0
// the producer also streams each unit's C tile into one of CB shared
// buffers, so the epilogue reads C from shared memory instead of waiting
// on global loads.  Both sides walk the same (unit, k-chunk) sequence; the
// running stage counter s selects the ring slot and its phase.
template <int BM, int BN, int WM, int WN, int KC, int STAGES, bool SYRK, int CB, int BOP>
__global__ void __launch_bounds__(TmaCfg<BM, BN, WM, WN, KC, STAGES, CB, BOP>::NTHREADS, (CB >= 2 ? 1 : 2))
    gemm_tma_kernel(GemmArgs g, ix tiles_m, ix tiles_n, ix nunits) {
  using Cfg = TmaCfg<BM, BN, WM, WN, KC, STAGES, CB, BOP>;
  constexpr int MT = Cfg::MT, NT = Cfg::NT;
  constexpr int BSTEP = BOP == BOP_NT ? 16 : 4 * BN;  // B fragment advance per k-step of 4
  extern __shared__ __align__(128) double smem[];
  double *cbuf = smem + Cfg::STAGE_ELEMS * STAGES;
  uint64_t *full = reinterpret_cast<uint64_t *>(cbuf + Cfg::C_ELEMS * CB);
  uint64_t *empty = full + STAGES;
  uint64_t *cfull = empty + STAGES;
  uint64_t *cempty = cfull + CB;
  const int lane = threadIdx.x & 31, warp = warp_uniform();
  const ix ncols = SYRK ? g.m : g.n;
  const bool cin = CB > 0 && BOP != BOP_TRI && g.beta != 0.0 && g.tmaC;  // C through shared memory
  const bool domma = g.alpha != 0.0 || BOP == BOP_TRI;

  const ix nk = domma ? (g.k + KC - 1) / KC : 0;
  const ix my_units = blockIdx.x < nunits ? (nunits - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::NWARPS);
    }
#pragma unroll
    for (int s = 0; s < CB; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], Cfg::NWARPS);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == Cfg::NWARPS) {
    // ===== producer =====
    if (nk == 0 && !cin) return;
    ix s = 0;
    for (ix ul = 0; ul < my_units; ++ul) {
      const ix u = blockIdx.x + ul * gridDim.x;
      ix b, tm, tn;
      unit_coords(u, tiles_m, tiles_n, SYRK, b, tm, tn);
      for (ix ch = first_chunk<BN, KC, BOP>(tn); ch < nk; ++ch, ++s) {
        const int st = (int)(s % STAGES);
        if (s >= STAGES) mbar_wait(&empty[st], (unsigned)(((s / STAGES) - 1) & 1));
        double *sa = smem + st * Cfg::STAGE_ELEMS;
        double *sb = sa + Cfg::A_ELEMS;
        const ix l0 = ch * KC;
        const int kc = (int)min((ix)KC, g.k - l0);
        const ix ra = g.ai + tm * BM;
        const ix rowsa = min((ix)BM, g.m - tm * BM);
        const int npa = (int)(((ra + rowsa - 1) >> 2) - (ra >> 2) + 1);
        const unsigned bytesa = 32u * kc;
        const double *A = g.A.item(b) + (ra >> 2) * 4 * g.A.cn + 4 * (g.aj + l0);
        if (BOP == BOP_NT) {
          const ix rb = g.bi + tn * BN;
          const ix rowsb = min((ix)BN, ncols - tn * BN);
          const int npb = (int)(((rb + rowsb - 1) >> 2) - (rb >> 2) + 1);
          if (lane == 0) mbar_arrive_expect_tx(&full[st], bytesa * (npa + npb));
          __syncwarp();
          const double *B = g.B.item(b) + (rb >> 2) * 4 * g.B.cn + 4 * (g.bj + l0);
          for (int p = lane; p < npa + npb; p += 32) {
            if (p < npa) tma_load_1d(sa + p * 4 * KC, A + (ix)p * 4 * g.A.cn, bytesa, &full[st]);
            else tma_load_1d(sb + (p - npa) * 4 * KC, B + (ix)(p - npa) * 4 * g.B.cn, bytesa, &full[st]);
          }
        } else {
          // B rows [bi + l0, bi + l0 + kc) x columns [tn*BN, +cols): one run per panel
          const ix rb = g.bi + l0;
          const int npb = (int)(((rb + kc - 1) >> 2) - (rb >> 2) + 1);
          const unsigned bytesb = 32u * (unsigned)min((ix)BN, ncols - tn * BN);
          if (lane == 0) mbar_arrive_expect_tx(&full[st], bytesa * npa + bytesb * npb);
          __syncwarp();
          const double *B = g.B.item(b) + (rb >> 2) * 4 * g.B.cn + 4 * (g.bj + tn * BN);
          for (int p = lane; p < npa + npb; p += 32) {
            if (p < npa) tma_load_1d(sa + p * 4 * KC, A + (ix)p * 4 * g.A.cn, bytesa, &full[st]);
            else tma_load_1d(sb + (p - npa) * 4 * BN, B + (ix)(p - npa) * 4 * g.B.cn, bytesb, &full[st]);
          }
        }
      }
      // the unit's C tile after its A/B chunks: with one C buffer its
      // issue waits for the previous unit's epilogue, which must not hold
      // back this unit's operand loads
      if (CB > 0 && cin) {
        const int cb = (int)(ul % (CB > 0 ? CB : 1));
        if (ul >= CB) mbar_wait(&cempty[cb], (unsigned)(((ul / (CB > 0 ? CB : 1)) - 1) & 1));
        const ix rc = g.ci + tm * BM;
        // C columns clip at g.n, not at the syrk tile range: a lower trapezoid
        // (g.n < g.m, the blocked potrf's trailing update) must not read past
        // C's window (the consumers read only in-store elements of the tile)
        const ix rows = min((ix)BM, g.m - tm * BM), cols = max((ix)0, min((ix)BN, g.n - tn * BN));
        const int npc = cols > 0 ? (int)(((rc + rows - 1) >> 2) - (rc >> 2) + 1) : 0;
        const unsigned bytes = 32u * (unsigned)cols;
        if (lane == 0) mbar_arrive_expect_tx(&cfull[cb], bytes * npc);
        __syncwarp();
        const double *C = g.C.item(b) + (rc >> 2) * 4 * g.C.cn + 4 * (g.cj + tn * BN);
        for (int p = lane; p < npc; p += 32)
          tma_load_1d(cbuf + cb * Cfg::C_ELEMS + p * 4 * BN, C + (ix)p * 4 * g.C.cn, bytes, &cfull[cb]);
      }
    }
    return;
  }

  // ===== consumers =====
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  const int fr = lane >> 2, fc = lane & 3;
  const int aira = (int)(g.ai & 3), airb = (int)(g.bi & 3), airc = (int)(g.ci & 3);
  int offa[MT], offb[NT], offc[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int r = aira + wm * WM + 8 * i + fr;
    offa[i] = (r >> 2) * 4 * KC + (r & 3) + 4 * fc;
    const int rc = airc + wm * WM + 8 * i + fr;
    offc[i] = (rc >> 2) * 4 * BN + (rc & 3) + 4 * (wn * WN + 2 * fc);
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (BOP == BOP_NT) {
      const int r = airb + wn * WN + 8 * j + fr;
      offb[j] = (r >> 2) * 4 * KC + (r & 3) + 4 * fc;
    } else {
      const int r = airb + fc;  // k row within the chunk
      offb[j] = (r >> 2) * 4 * BN + (r & 3) + 4 * (wn * WN + 8 * j + fr);
    }
  }

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  ix s = 0;
  for (ix ul = 0; ul < my_units; ++ul) {
    ix b, tm, tn;
    unit_coords(blockIdx.x + ul * gridDim.x, tiles_m, tiles_n, SYRK, b, tm, tn);
    const ix rbase = tm * BM + wm * WM, cbase = tn * BN + wn * WN;
    const bool active = !SYRK || (cbase <= rbase + WM - 1);
    for (ix ch = first_chunk<BN, KC, BOP>(tn); ch < nk; ++ch, ++s) {
      const int st = (int)(s % STAGES);
      mbar_wait(&full[st], (unsigned)((s / STAGES) & 1));
      const double *sa = smem + st * Cfg::STAGE_ELEMS;
      const double *sb = sa + Cfg::A_ELEMS;
      const int kc = (int)min((ix)KC, g.k - ch * KC);
      // triangular B: this chunk crosses the diagonal of the warp's columns
      const bool tri = BOP == BOP_TRI && ch * KC < cbase + WN;
      if (active) {
        if (kc == KC && !tri) {
#pragma unroll
          for (int kk = 0; kk < KC / 4; ++kk) {
            double a[MT], bb[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i) a[i] = sa[offa[i] + 16 * kk];
#pragma unroll
            for (int j = 0; j < NT; ++j) bb[j] = sb[offb[j] + BSTEP * kk];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
              for (int j = 0; j < NT; ++j) dmma(acc[i][j], a[i], bb[j]);
          }
        } else {
          for (int kk = 0; 4 * kk < kc; ++kk) {
            const int lk = 4 * kk + fc;
            const bool okc = lk < kc;
            double a[MT], bb[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i) a[i] = okc ? sa[offa[i] + 16 * kk] : 0.0;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              const bool okt = BOP != BOP_TRI || ch * KC + lk >= cbase + 8 * j + fr;
              bb[j] = (okc && okt) ? sb[offb[j] + BSTEP * kk] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
              for (int j = 0; j < NT; ++j) dmma(acc[i][j], a[i], bb[j]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    {
      double *D = g.D.item(b);
      const double *C = g.C.item(b);
      const bool skip = g.skip && g.skip[b] >= 0;
      double cv[MT][NT][2];
      const int cb = CB > 0 ? (int)(ul % (CB > 0 ? CB : 1)) : 0;
      if (cin) {
        mbar_wait(&cfull[cb], (unsigned)((ul / (CB > 0 ? CB : 1)) & 1));
        const double *cs = cbuf + cb * Cfg::C_ELEMS;
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) cv[i][j][e] = cs[offc[i] + 4 * (8 * j + e)];
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty[cb]);
      } else {
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const ix r = rbase + 8 * i + fr, c = cbase + 8 * j + 2 * fc + e;
              cv[i][j][e] = (BOP != BOP_TRI && g.beta != 0.0 && in_store<SYRK>(r, c, g.m, g.n))
                                ? ldg_nc(C + eo(g.ci + r, g.cj + c, g.C.cn))
                                : 0.0;
            }
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const ix r = rbase + 8 * i + fr, c = cbase + 8 * j + 2 * fc + e;
            if (!skip && in_store<SYRK>(r, c, g.m, g.n))
              D[eo(g.di + r, g.dj + c, g.D.cn)] = BOP == BOP_TRI
                                                      ? __dmul_rn(g.alpha, acc[i][j][e])
                                                      : epilogue_value<SYRK>(g, r, c, acc[i][j][e], cv[i][j][e]);
            acc[i][j][e] = 0.0;
          }
    }
  }
}

// ---------------------------------------------------------------------------
// gemm_item: one THREAD per item for m, n <= 4 (one panel), k <= 16 -- the
// smallest C3 points are pure HBM streaming, so the kernel mirrors the
// tiny-potrf design: persistent CTAs, a 2-stage cp.async ring of the
// items' A/B(/C) panel runs (16-byte pieces, coalesced across the warp),
// the product in registers (FMA), coalesced 16-byte stores of D's window.

template <int KMAX, int STG = 1>
struct ItemCfg {
  static constexpr int NTH = 128, ITEMS = NTH;
  static constexpr int STRIDE = 3 * 4 * KMAX + 2;  // A, B (4 x KMAX each) + C (4 x 4 <= 4 x KMAX), padded
  static constexpr int STAGES = STG;
  static constexpr size_t SMEM = sizeof(double) * STG * ITEMS * STRIDE;
};

// STG = 1 (single stage, 4 CTAs / 16 warps per SM) measured faster than the
// 2-stage ring (2 CTAs / 8 warps) at C3 n = 4: more rounds in flight per SM.
template <int KMAX, bool SYRK, int STG = 1>
__global__ void __launch_bounds__(128) gemm_item_kernel(GemmArgs g) {
  using Cfg = ItemCfg<KMAX, STG>;
  constexpr int ITEMS = Cfg::ITEMS, NTH = Cfg::NTH, STRIDE = Cfg::STRIDE;
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x;
  const int m = (int)g.m, n = (int)g.n, k = (int)g.k;
  const ix nrounds = (g.batch + ITEMS - 1) / ITEMS;
  const bool rc = g.beta != 0.0, ab = g.alpha != 0.0;
  // pieces per item: A 2k, B 2k, C 2n (16 bytes each)
  const int pa = ab ? 2 * k : 0, pbb = ab ? 2 * k : 0, pc = rc ? 2 * n : 0;
  const int pieces = pa + pbb + pc;

  auto issue = [&](ix rd, int buf) {
    double *S = smem + buf * ITEMS * STRIDE;
    const ix b0 = rd * ITEMS;
    for (int q = tid; q < ITEMS * pieces; q += NTH) {
      const int it = q / pieces, w = q - it * pieces;
      const ix b = b0 + it;
      const bool ok = b < g.batch;
      const double *src;
      int dst;
      if (w < pa) {
        src = g.A.item(b) + eo(g.ai, g.aj + (w >> 1), g.A.cn) + 2 * (w & 1);
        dst = 2 * w;
      } else if (w < pa + pbb) {
        const int v = w - pa;
        src = g.B.item(b) + eo(g.bi, g.bj + (v >> 1), g.B.cn) + 2 * (v & 1);
        dst = 4 * KMAX + 2 * v;
      } else {
        const int v = w - pa - pbb;
        src = g.C.item(b) + eo(g.ci, g.cj + (v >> 1), g.C.cn) + 2 * (v & 1);
        dst = 8 * KMAX + 2 * v;
      }
      cp_async16(S + it * STRIDE + dst, ok ? src : g.D.p, ok ? 16 : 0);
    }
  };

  if (STG == 2 && blockIdx.x < nrounds) issue(blockIdx.x, 0);
  cp_async_commit();
  int buf = 0;
  for (ix rd = blockIdx.x; rd < nrounds; rd += gridDim.x, buf ^= (STG - 1)) {
    if (STG == 2) {
      if (rd + gridDim.x < nrounds) issue(rd + gridDim.x, buf ^ 1);
    } else {
      issue(rd, 0);
    }
    cp_async_commit();
    if (STG == 2) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    double *S = smem + buf * ITEMS * STRIDE + tid * STRIDE;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    if (ab) {
#pragma unroll
      for (int l = 0; l < KMAX; ++l) {
        if (l < k) {
          const double2 a01 = *reinterpret_cast<const double2 *>(S + 4 * l);
          const double2 a23 = *reinterpret_cast<const double2 *>(S + 4 * l + 2);
          const double2 b01 = *reinterpret_cast<const double2 *>(S + 4 * KMAX + 4 * l);
          const double2 b23 = *reinterpret_cast<const double2 *>(S + 4 * KMAX + 4 * l + 2);
          const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
      }
    }
    // epilogue into the same slot (A's area), then coalesced stores
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double cv = rc ? S[8 * KMAX + 4 * j + i] : 0.0;
        S[4 * j + i] = (SYRK && (i >> 2) == (j >> 2)) ? syrk_diag_rule(g.alpha, acc[i][j], g.beta, cv)
                                                       : store_rule(g.alpha, acc[i][j], g.beta, cv);
      }
    __syncthreads();
    const ix b0 = rd * ITEMS;
    for (int q = tid; q < ITEMS * 2 * n; q += NTH) {
      const int it = q / (2 * n), w = q - it * 2 * n;
      const ix bb = b0 + it;
      if (bb >= g.batch || (g.skip && g.skip[bb] >= 0)) continue;
      const int col = w >> 1, h = w & 1;
      const double *src = smem + buf * ITEMS * STRIDE + it * STRIDE + 4 * col + 2 * h;
      double *dst = g.D.item(bb) + eo(g.di, g.dj + col, g.D.cn) + 2 * h;
      const int r0 = 2 * h;
      const bool w0 = r0 < m && (!SYRK || r0 >= col), w1 = r0 + 1 < m && (!SYRK || r0 + 1 >= col);
      if (w0 && w1) *reinterpret_cast<double2 *>(dst) = *reinterpret_cast<const double2 *>(src);
      else if (w0) dst[0] = src[0];
      else if (w1) dst[1] = src[1];
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

template <int KMAX, bool SYRK, int STG = 1>
static cudaError_t launch_item(const GemmArgs &g, cudaStream_t st) {
  using Cfg = ItemCfg<KMAX, STG>;
  auto kern = gemm_item_kernel<KMAX, SYRK, STG>;
  static LaunchCache cache;
  const int occ = cache.occupancy((const void *)kern, Cfg::NTH, Cfg::SMEM);
  const ix rounds = (g.batch + Cfg::ITEMS - 1) / Cfg::ITEMS;
  ix grid = (ix)num_sms() * occ;
  if (grid > rounds) grid = rounds;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, Cfg::NTH, Cfg::SMEM, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

// gemm_item_reg: the same one-thread-per-item product with no shared-memory
// staging: every thread loads its item's A/B(/C) panel runs straight into
// registers with 16-byte loads (all of an item's bytes are used by the one
// thread, so every fetched sector is consumed), computes, and stores its own
// window.  With no round barrier every warp keeps ~8 KB of loads in flight,
// which the staged kernel's load / compute / store rounds could not.
template <bool SYRK, int MINB = 1>
__global__ void __launch_bounds__(128, MINB) gemm_item_reg_kernel(GemmArgs g) {
  const int m = (int)g.m, n = (int)g.n, k = (int)g.k;
  const bool rc = g.beta != 0.0, ab = g.alpha != 0.0;
  for (ix b = (ix)blockIdx.x * blockDim.x + threadIdx.x; b < g.batch; b += (ix)gridDim.x * blockDim.x) {
    double av[4][4], bv[4][4], cv[4][4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const bool ok = ab && l < k;
      double2 a01 = make_double2(0.0, 0.0), a23 = a01, b01 = a01, b23 = a01;
      if (ok) {
        const double *A = g.A.item(b) + eo(g.ai, g.aj + l, g.A.cn);
        const double *B = g.B.item(b) + eo(g.bi, g.bj + l, g.B.cn);
        a01 = ldg_nc2(A), a23 = ldg_nc2(A + 2);
        b01 = ldg_nc2(B), b23 = ldg_nc2(B + 2);
      }
      av[l][0] = a01.x, av[l][1] = a01.y, av[l][2] = a23.x, av[l][3] = a23.y;
      bv[l][0] = b01.x, bv[l][1] = b01.y, bv[l][2] = b23.x, bv[l][3] = b23.y;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double2 c01 = make_double2(0.0, 0.0), c23 = c01;
      if (rc && j < n) {
        const double *C = g.C.item(b) + eo(g.ci, g.cj + j, g.C.cn);
        c01 = ldg_nc2(C), c23 = ldg_nc2(C + 2);
      }
      cv[0][j] = c01.x, cv[1][j] = c01.y, cv[2][j] = c23.x, cv[3][j] = c23.y;
    }
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
#pragma unroll
    for (int l = 0; l < 4; ++l)
      if (ab && l < k) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[l][i], bv[l][j], acc[i][j]);
      }
    if (g.skip && g.skip[b] >= 0) continue;
    double *D = g.D.item(b);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j < n) {
      double v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        v[i] = (SYRK && (i >> 2) == (j >> 2)) ? syrk_diag_rule(g.alpha, acc[i][j], g.beta, cv[i][j])
                                               : store_rule(g.alpha, acc[i][j], g.beta, cv[i][j]);
      double *dst = D + eo(g.di, g.dj + j, g.D.cn);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r0 = 2 * h;
        const bool w0 = r0 < m && (!SYRK || r0 >= j), w1 = r0 + 1 < m && (!SYRK || r0 + 1 >= j);
        if (w0 && w1) *reinterpret_cast<double2 *>(dst + r0) = make_double2(v[r0], v[r0 + 1]);
        else if (w0) dst[r0] = v[r0];
        else if (w1) dst[r0 + 1] = v[r0 + 1];
      }
      }
    }
  }
}

// gemm_nt, m = n = k = 4 exactly, one-panel windows (the C3 sweep's first point: 128-byte items, pure HBM
// streaming).  The thread-per-item register kernel reads each item with eight 16-byte loads at a 128-byte
// lane stride and reached 0.68 of HBM.  Here a CTA stages a round of 128 items cooperatively -- thread t
// keeps ONE piece position (t % 8) and item lane (t / 8), so consecutive lanes move consecutive 16-byte
// pieces (coalesced both ways) and every address is a base plus a per-trip item stride -- then each thread
// multiplies its own item out of its (conflict-free, 18-double) shared-memory slot and leaves D there for
// the coalesced store.  Same _store_block rules (alpha = 0 never reads A / B, beta = 0 never reads C).
template <int NTH>
__global__ void __launch_bounds__(NTH) gemm4_staged_kernel(GemmArgs g) {
  constexpr int ITEMS = NTH, STR = 18, STEP = NTH / 8, TRIPS = ITEMS / STEP;
  extern __shared__ __align__(16) double sm4[];
  double *sA = sm4, *sB = sA + ITEMS * STR, *sC = sB + ITEMS * STR;
  const int tid = threadIdx.x, w = tid & 7, it0 = tid >> 3;
  const bool ab = g.alpha != 0.0, rc = g.beta != 0.0;
  const ix offA = eo(g.ai, g.aj, g.A.cn) + 2 * w, offB = eo(g.bi, g.bj, g.B.cn) + 2 * w;
  const ix offC = eo(g.ci, g.cj, g.C.cn) + 2 * w, offD = eo(g.di, g.dj, g.D.cn) + 2 * w;
  const ix nrounds = (g.batch + ITEMS - 1) / ITEMS;
  for (ix rd = blockIdx.x; rd < nrounds; rd += gridDim.x) {
    const ix b0 = rd * ITEMS;
    {
      const double *pa = g.A.p + (b0 + it0) * g.A.stride + offA, *pb_ = g.B.p + (b0 + it0) * g.B.stride + offB;
      const double *pc = g.C.p + (b0 + it0) * g.C.stride + offC;
      const int so = it0 * STR + 2 * w;
#pragma unroll
      for (int k = 0; k < TRIPS; ++k) {
        const bool ok = b0 + it0 + k * STEP < g.batch;
        if (ab) {
          cp_async16(sA + so + k * STEP * STR, ok ? pa + (ix)k * STEP * g.A.stride : g.A.p, ok ? 16 : 0);
          cp_async16(sB + so + k * STEP * STR, ok ? pb_ + (ix)k * STEP * g.B.stride : g.B.p, ok ? 16 : 0);
        }
        if (rc) cp_async16(sC + so + k * STEP * STR, ok ? pc + (ix)k * STEP * g.C.stride : g.C.p, ok ? 16 : 0);
      }
      cp_async_commit();
      cp_async_wait<0>();
    }
    __syncthreads();
    {
      // this thread's item: column l of A / B at slot + 4 l (rows 0..3 contiguous)
      double *mA = sA + tid * STR;
      const double *mB = sB + tid * STR, *mC = sC + tid * STR;
      double acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
      if (ab) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          const double2 a01 = *reinterpret_cast<const double2 *>(mA + 4 * l), a23 = *reinterpret_cast<const double2 *>(mA + 4 * l + 2);
          const double2 b01 = *reinterpret_cast<const double2 *>(mB + 4 * l), b23 = *reinterpret_cast<const double2 *>(mB + 4 * l + 2);
          const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double2 c01 = make_double2(0.0, 0.0), c23 = c01;
        if (rc) c01 = *reinterpret_cast<const double2 *>(mC + 4 * j), c23 = *reinterpret_cast<const double2 *>(mC + 4 * j + 2);
        const double cv[4] = {c01.x, c01.y, c23.x, c23.y};
        double v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = store_rule(g.alpha, acc[i][j], g.beta, cv[i]);
        *reinterpret_cast<double2 *>(mA + 4 * j) = make_double2(v[0], v[1]);
        *reinterpret_cast<double2 *>(mA + 4 * j + 2) = make_double2(v[2], v[3]);
      }
    }
    __syncthreads();
    {
      double *pd = g.D.p + (b0 + it0) * g.D.stride + offD;
      const int so = it0 * STR + 2 * w;
#pragma unroll
      for (int k = 0; k < TRIPS; ++k) {
        const ix b = b0 + it0 + k * STEP;
        if (b < g.batch && !(g.skip && g.skip[b] >= 0))
          *reinterpret_cast<double2 *>(pd + (ix)k * STEP * g.D.stride) = *reinterpret_cast<const double2 *>(sA + so + k * STEP * STR);
      }
    }
    __syncthreads();
  }
}

static cudaError_t launch_gemm4_staged(const GemmArgs &g, cudaStream_t st) {
  constexpr int NTH = 128;
  auto kern = gemm4_staged_kernel<NTH>;
  const size_t smem = sizeof(double) * NTH * 18 * (g.beta != 0.0 ? 3 : 2);
  static LaunchCache cache;
  static bool carve = false;
  if (!carve) {
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    carve = true;
  }
  const int occ = cache.occupancy((const void *)kern, NTH, smem);
  const ix rounds = (g.batch + NTH - 1) / NTH;
  ix grid = (ix)num_sms() * occ;
  if (grid > rounds) grid = rounds;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, NTH, smem, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

template <bool SYRK, int MINB = 1>
static cudaError_t launch_item_reg(const GemmArgs &g, cudaStream_t st) {
  auto kern = gemm_item_reg_kernel<SYRK, MINB>;
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0);
    if (occ < 1) occ = 1;
  }
  ix grid = (ix)num_sms() * occ;
  const ix need = (g.batch + 127) / 128;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, 128, 0, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host dispatch

static int g_num_sms[64] = {0};
int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!g_num_sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms[dev] = v > 0 ? v : 148;
  }
  return g_num_sms[dev];
}

template <int MT, int NT, bool SYRK, int BOP = BOP_NT>
static cudaError_t launch_direct(const GemmArgs &g, cudaStream_t st) {
  const int threads = 256;
  const ix tiles_m = (g.m + 8 * MT - 1) / (8 * MT);
  const ix tiles_n = SYRK ? tiles_m : (g.n + 8 * NT - 1) / (8 * NT);
  const ix per = SYRK ? tiles_m * (tiles_m + 1) / 2 : tiles_m * tiles_n;
  const ix nunits = per * g.batch;
  ix blocks = (nunits + 7) / 8;
  const ix cap = (ix)num_sms() * 8 * 8;  // ~8 resident CTAs of 8 warps per SM, a few waves
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  // min 3 CTAs/SM (<= 85 registers): C3 n = 8..24 6.25 -> 4.63 ms summed (n = 16 alone 9 % slower).
  // One-tile items (m, n <= 8) are latency-bound, not register-bound: 8 CTAs/SM (32 registers, 64 resident
  // warps) took C3 n = 8 from 22.4 to 16.5 ms (0.71 -> 0.97 of HBM); 2x2 tiles lose at anything above 3
  // (n = 12: 14.2 / 15.1 / 21.0 ms at 3 / 4 / 5).  The hoisted one-tile-per-item path (ONE) pays for items of
  // up to 2x2 tiles (n = 12 15.3 -> 14.1 ms) and costs spills at 3x3 (n = 20 9.0 -> 9.4 ms).
  if constexpr (BOP == BOP_NT && MT * NT <= 4) {
    if (per == 1) {
      gemm_direct_kernel<MT, NT, SYRK, BOP, (MT * NT == 1 ? 8 : 3), true>
          <<<(unsigned)blocks, threads, 0, st>>>(g, tiles_m, tiles_n, nunits);
      note_launch();
      return cudaGetLastError();
    }
  }
  gemm_direct_kernel<MT, NT, SYRK, BOP, 3><<<(unsigned)blocks, threads, 0, st>>>(g, tiles_m, tiles_n, nunits);
  note_launch();
  return cudaGetLastError();
}

template <bool SYRK, int BOP = BOP_NT>
static cudaError_t dispatch_direct(const GemmArgs &g, cudaStream_t st) {
  const int mt = (int)((g.m + 7) / 8), nt = (int)(((SYRK ? g.m : g.n) + 7) / 8);
#define PB_DIRECT(M_, N_) \
  if (mt == M_ && nt == N_) return launch_direct<M_, N_, SYRK, BOP>(g, st);
  PB_DIRECT(1, 1) PB_DIRECT(1, 2) PB_DIRECT(1, 3) PB_DIRECT(2, 1) PB_DIRECT(2, 2) PB_DIRECT(2, 3)
  PB_DIRECT(3, 1) PB_DIRECT(3, 2) PB_DIRECT(3, 3)
#undef PB_DIRECT
  return cudaErrorInvalidValue;
}

template <int BM, int BN, int WM, int WN, int KC, int STAGES, bool SYRK>
static cudaError_t launch_tiled(const GemmArgs &g, cudaStream_t st) {
  using Cfg = TiledCfg<BM, BN, WM, WN, KC, STAGES>;
  auto kern = gemm_tiled_kernel<BM, BN, WM, WN, KC, STAGES, SYRK>;
  static LaunchCache cache;
  const int occ = cache.occupancy((const void *)kern, Cfg::NTHREADS, Cfg::SMEM);
  const ix tiles_m = (g.m + BM - 1) / BM;
  const ix tiles_n = SYRK ? tiles_m : (g.n + BN - 1) / BN;
  const ix per = SYRK ? tiles_m * (tiles_m + 1) / 2 : tiles_m * tiles_n;
  const ix nunits = per * g.batch;
  ix grid = (ix)num_sms() * occ;
  if (grid > nunits) grid = nunits;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, Cfg::NTHREADS, Cfg::SMEM, st>>>(g, tiles_m, tiles_n, nunits);
  note_launch();
  return cudaGetLastError();
}

template <int BM, int BN, int WM, int WN, int KC, int STAGES, bool SYRK, int CB = 0, int BOP = BOP_NT>
static cudaError_t launch_tma(const GemmArgs &g, cudaStream_t st) {
  using Cfg = TmaCfg<BM, BN, WM, WN, KC, STAGES, CB, BOP>;
  auto kern = gemm_tma_kernel<BM, BN, WM, WN, KC, STAGES, SYRK, CB, BOP>;
  static LaunchCache cache;
  const int occ = cache.occupancy((const void *)kern, Cfg::NTHREADS, Cfg::SMEM);
  const ix tiles_m = (g.m + BM - 1) / BM;
  const ix tiles_n = SYRK ? tiles_m : (g.n + BN - 1) / BN;
  const ix per = SYRK ? tiles_m * (tiles_m + 1) / 2 : tiles_m * tiles_n;
  const ix nunits = per * g.batch;
  ix grid = (ix)num_sms() * occ;
  if (grid > nunits) grid = nunits;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, Cfg::NTHREADS, Cfg::SMEM, st>>>(g, tiles_m, tiles_n, nunits);
  note_launch();
  return cudaGetLastError();
}

template <bool SYRK>
static cudaError_t dispatch_gemm(GemmArgs g, cudaStream_t st) {
  const ix ncols = SYRK ? g.m : g.n;
  const ix big = g.m > ncols ? g.m : ncols;
  // one thread per item: one-panel windows (rows in a single aligned panel)
  // with 16-byte aligned item storage
  const bool one_panel = (g.ai & 3) == 0 && (g.bi & 3) == 0 && (g.ci & 3) == 0 && (g.di & 3) == 0 && g.tma && g.tmaC &&
                         ((uintptr_t)g.D.p & 15) == 0 && (g.D.stride & 1) == 0;
  if (big <= 4 && one_panel) {
    // (k <= 4 only: the per-thread staging of larger k does not fit shared memory)
    // register-direct kernel (C3 n = 4: 3.40 -> 3.01 ms over the staged one;
    // capping it at 4-6 CTAs/SM spills and is slower)
    // the full 4 x 4 x 4 product (the C3 sweep's first point): cooperative staging, coalesced both ways
    if (!SYRK && g.m == 4 && g.n == 4 && g.k == 4 && (g.A.stride & 1) == 0 && (g.B.stride & 1) == 0 &&
        (g.C.stride & 1) == 0)
      return launch_gemm4_staged(g, st);
    if (g.k <= 4) return launch_item_reg<SYRK>(g, st);
  }
  if (big <= 24) return dispatch_direct<SYRK>(g, st);
  const ix small = g.m < ncols ? g.m : ncols;
  if (g.tma) {
    // square output tile T in {32, 48, 64} minimising the padded tile area
    // (ties -> larger T); k-chunk 40 when it covers k in one chunk.
    // Measured on B200: profiles/r01_gemm_tuning.txt
    // square output tile T minimising padded tile area x measured cost per
    // unit area of that tile shape (fitted over the C3 sweep n = 28..300 on
    // B200, profiles/r01_gemm_tile_sweep.txt: within 0.1 % of the per-size best)
    // (round 2: tiles 80 / 88 added and tiles >= 72 on a 2-stage ring, so
    // two CTAs fit an SM; weights refitted on the full C3 sweep per tile,
    // profiles/r02_gemm_c3_tile_refit.txt: n >= 64 min 0.44 -> 0.51)
    int T = 64;
    double best = 1e30;
    const int tiles[8] = {64, 32, 56, 48, 72, 40, 80, 88};
    const double wcost[8] = {1.000, 1.081, 1.056, 1.241, 1.107, 1.422, 1.350, 1.182};
    for (int i = 0; i < 8; ++i) {
      const int t = tiles[i];
      const ix tmr = (g.m + t - 1) / t, tnc = (ncols + t - 1) / t;
      // syrk runs the lower tiles only: tmr (tmr + 1) / 2 of them
      const double area = (SYRK ? 0.5 * (double)(tmr * (tmr + 1)) : (double)(tmr * tnc)) * (double)t * (double)t * wcost[i];
      if (area < best * 0.999) best = area, T = t;
    }
    const bool k40 = g.k > 32 && g.k <= 40;
    const bool cs = g.beta != 0.0 && g.tmaC;  // C tile through shared memory
#define PB_TMA(T_, WM_, WN_, K_)                                                    \
  if (T == T_ && (K_ == 40) == k40) {                                                \
    if (cs) return launch_tma<T_, T_, WM_, WN_, K_, 2, SYRK, 1>(g, st);              \
    if (T_ >= 72) return launch_tma<T_, T_, WM_, WN_, K_, 2, SYRK, 0>(g, st); /* 2 CTAs/SM */ \
    return launch_tma<T_, T_, WM_, WN_, K_, 3, SYRK, 0>(g, st);                      \
  }
    PB_TMA(64, 32, 16, 32) PB_TMA(64, 32, 16, 40) PB_TMA(48, 24, 16, 32) PB_TMA(48, 24, 16, 40)
    PB_TMA(32, 16, 16, 32) PB_TMA(32, 16, 16, 40) PB_TMA(72, 24, 24, 32) PB_TMA(72, 24, 24, 40)
    PB_TMA(56, 56, 8, 32) PB_TMA(56, 56, 8, 40) PB_TMA(40, 40, 8, 32) PB_TMA(40, 40, 8, 40)
    PB_TMA(80, 40, 16, 32) PB_TMA(80, 40, 16, 40) PB_TMA(88, 88, 8, 32) PB_TMA(88, 88, 8, 40)
#undef PB_TMA
  }
  if (small <= 40) return launch_tiled<32, 32, 16, 16, 32, 3, SYRK>(g, st);
  return launch_tiled<64, 64, 32, 32, 32, 2, SYRK>(g, st);
}

// gemm_nn / trmm_rlnn: B read down its columns (BOP_NN / BOP_TRI).
template <int BOP>
static cudaError_t dispatch_nn(const GemmArgs &g, cudaStream_t st) {
  const ix big = g.m > g.n ? g.m : g.n;
  if (big <= 24) return dispatch_direct<false, BOP>(g, st);
  if (!g.tma) return launch_direct<3, 3, false, BOP>(g, st);  // any alignment
  int T = 64;
  double best = 1e30;
  for (int t : {64, 48, 32}) {
    const double area = (double)((g.m + t - 1) / t * t) * (double)((g.n + t - 1) / t * t);
    if (area < best * 0.999) best = area, T = t;
  }
  const bool cs = BOP == BOP_NN && g.beta != 0.0 && g.tmaC;
#define PB_TMA_NN(T_, WM_)                                                                     \
  if (T == T_) {                                                                               \
    if (cs) return launch_tma<T_, T_, WM_, 16, 32, 2, false, (BOP == BOP_NN ? 1 : 0), BOP>(g, st); \
    return launch_tma<T_, T_, WM_, 16, 32, 3, false, 0, BOP>(g, st);                             \
  }
  PB_TMA_NN(64, 32) PB_TMA_NN(48, 24) PB_TMA_NN(32, 16)
#undef PB_TMA_NN
  return cudaErrorInvalidValue;
}

cudaError_t run_gemm_nt(const GemmArgs &g, cudaStream_t st) { return dispatch_gemm<false>(g, st); }
cudaError_t run_gemm_nn(const GemmArgs &g, cudaStream_t st) { return dispatch_nn<BOP_NN>(g, st); }
cudaError_t run_trmm_rlnn(const GemmArgs &g, cudaStream_t st) { return dispatch_nn<BOP_TRI>(g, st); }
cudaError_t run_syrk_ln(const GemmArgs &g, cudaStream_t st) { return dispatch_gemm<true>(g, st); }

}  // namespace pb
