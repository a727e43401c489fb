// Batched dpotrf_l for 17 <= n <= 64: one warp per item, the whole lower
// triangle register-resident as 8x8 DMMA accumulator tiles (sm_100a).
//
// Reference semantics: potrf_drv ccore.pyx:877-905 (+ _kpotrf_core
// :404-438): lower Cholesky of lower(C), sqrt then one reciprocal per
// column (dinv[j] = 1/L[j][j], column scaled by it), first pivot with
// d <= 0 (NaN passes) -> info, failing items written exactly as far as the
// reference writes them.  Floating-point order differs from the reference
// (right-looking, FMA, DMMA): parity is the 50*n*eps Frobenius tolerance.
//
// Why this shape: the C2 points n = 32 / 64 are HBM-bound (AI 1.3 / 2.6
// flop/B).  The shared-memory team kernel spent ~3.7K / 9.6K warp
// instructions per item on staging, index math and barriers
// (profiles/r01_c2_kernels_ncu.txt).  Here an item costs one pass of loads,
// register math and one pass of stores:
//  * tile (i, j), i >= j, of 8x8 elements is one m8n8k4 accumulator: lane
//    (r = lane/4, q = lane%4) holds (8i + r, 8j + 2q + {0,1}); a warp-wide
//    8-byte load/store of one element slot covers 8 whole 32-byte sectors
//    of the panel-major item (two panels x four columns);
//  * right-looking over 8-column panels: the panel is factored column by
//    column with warp shuffles (pivot broadcast, sqrt, one reciprocal,
//    column scale, rank-1 update of the panel's remaining columns), then
//    the trailing lower tiles take  T(i,j) -= P(i) P(j)^T  on DMMA; a panel
//    tile's accumulator registers are used directly as the A fragment and,
//    for its transpose, the B fragment (k-step e contracts over columns
//    2q + e), so the update needs no shuffles;
//  * no shared memory and no barriers: occupancy is set by registers only,
//    and other warps hide each item's load latency and pivot chain; the
//    next item's rows are prefetched into L2 by one bulk prefetch.
#include "pb_exact.cuh"
#include "pb_gemm.cuh"

namespace pb {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__host__ __device__ constexpr int ti(int i, int j) { return i * (i + 1) / 2 + j; }

// 1/sqrt(d) for the pivot: MUFU seed (rel. error 2^-22) + ONE cubic step
// y (1 + e/2 + 3e^2/8), e = 1 - d y^2: five FP64 instructions instead of the
// seven of two Newton steps, branch-free (the kernel is bound by its FP64 /
// issue slots, not by this chain; __dsqrt_rn + __ddiv_rn cost two slow-path
// call sequences per column).  d > 0 here (d <= 0 failed before); NaN propagates.
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-(d * y), y, 1.0);
  const double p = fma(0.375, e, 0.5);
  return fma(y, e * p, y);
}

__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

template <int GM, bool SYRK>
__global__ void __launch_bounds__(32, (GM <= 2 ? 32 : (GM <= 4 ? 16 : (GM <= 6 ? 12 : 8)))) potrf_reg_kernel(PotrfArgs g, int pf_ok) {
  constexpr int NT = GM * (GM + 1) / 2;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int n = (int)g.n;
  // one warp per CTA: the item index is CTA-uniform, so the compiler sees
  // converged control flow around every shuffle and DMMA
  const ix nw = (ix)gridDim.x;
  // L2 prefetch of the next item (PB_REG_PF): 1 = one bulk prefetch of its
  // whole panels (default, measured best), 2 = only each panel's lower
  // prefix, one prefetch per lane (fewer bytes, measured 2-3 % slower),
  // 0 = none (10-20 % slower); prefetching D too was 25 % slower
  const int np4 = (n + 3) / 4;
  const unsigned pf_bytes = 32u * (unsigned)min(4 * lane + 4, n);
  // per-lane row offsets of the window rows 8i + r (panel carry included),
  // so an element address is one add of a compile-time column offset
  ix offC[GM], offD[GM];
#pragma unroll
  for (int i = 0; i < GM; ++i) {
    offC[i] = eo(g.ci + 8 * i + r, g.cj + 2 * q, g.C.cn);
    offD[i] = eo(g.di + 8 * i + r, g.dj + 2 * q, g.D.cn);
  }
  for (ix b = (ix)blockIdx.x; b < g.batch; b += nw) {
    if (g.merge && g.info[b] >= 0) continue;  // blocked driver: item failed in an earlier panel
    const double *Cb = g.C.p + b * g.C.stride;
    if (pf_ok == 2 && lane < np4 && b + nw < g.batch)
      prefetch_l2(g.C.p + (b + nw) * g.C.stride + eo(g.ci + 4 * lane, g.cj, g.C.cn), pf_bytes);
    if (pf_ok == 1 && lane == 0 && b + nw < g.batch)
      prefetch_l2(g.C.p + (b + nw) * g.C.stride + eo(g.ci, 0, g.C.cn), 32u * (unsigned)g.C.cn * (unsigned)np4);
    double T[NT][2];
#pragma unroll
    for (int i = 0; i < GM; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int R = 8 * i + r, Cc = 8 * j + 2 * q + e;
          // lower(C) inside the window; outside: identity padding, so the
          // padded columns factor trivially and never couple to real rows
          T[ti(i, j)][e] = (R < n && Cc <= R) ? Cb[offC[i] + 4 * (8 * j + e)] : (R == Cc ? 1.0 : 0.0);
        }
    if constexpr (SYRK) {  // fused syrk_potrf_ln (ccore.pyx:908-941): factor lower(C + A B^T)
      const double *Ab = g.A.p + b * g.A.stride, *Bb = g.B.p + b * g.B.stride;
      const int k = (int)g.k;
      for (int s = 0; s < (k + 3) / 4; ++s) {
        const int kk = 4 * s + q;  // A fragment (8x4 row-major) == B fragment of the transpose
        double fa[GM], fb[GM];
#pragma unroll
        for (int i = 0; i < GM; ++i) {
          const int R = 8 * i + r;
          const bool ok = R < n && kk < k;
          fa[i] = ok ? Ab[eo(g.ai + R, g.aj + kk, g.A.cn)] : 0.0;
          fb[i] = g.ab_same ? fa[i] : (ok ? Bb[eo(g.bi + R, g.bj + kk, g.B.cn)] : 0.0);
        }
#pragma unroll
        for (int i = 0; i < GM; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) dmma(T[ti(i, j)], fa[i], fb[j]);
      }
    }
    int fail = -1;
    double *dA = g.D.d + b * g.D.dstride + g.dj;
    double dkeep[GM];
#pragma unroll
    for (int k = 0; k < GM; ++k) dkeep[k] = 0.0;
    // Control flow stays warp-uniform and branch-free: a failing pivot only
    // records its index and zeroes its reciprocal (the columns left of it
    // are final in a right-looking sweep and are never touched again; the
    // rest is garbage that the write mask drops).
    //
    // Within a panel the columns stay UNSCALED (u = L * sqrt(d)): the rank-1
    // update uses  u[r][j] * u[c][j] / d_j  and the whole panel is scaled by
    // its reciprocals once at the end (the diagonal u[c][c] is d_c itself, so
    // u * (1/sqrt d) gives L[c][c] = sqrt(d_c) by the same rule).  The
    // shuffles of column j then do not wait for its pivot's rsqrt.
#pragma unroll
    for (int k = 0; k < GM; ++k) {
      double myinv = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        constexpr int dummy = 0;
        (void)dummy;
        const int h = j >> 1, ej = j & 1;
        const double d = __shfl_sync(FULL, T[ti(k, k)][ej], 4 * j + h);
        const bool bad = d <= 0.0;  // ccore.pyx:423 (NaN passes); warp-uniform
        if (bad && fail < 0) fail = 8 * k + j;
        const double inv = bad ? 0.0 : rsqrt_nr(d);
        if (lane == j) myinv = inv;
        if (j < 7) {
          // rank-1 update of the panel's columns c > j; the multiplier is
          // zeroed in lanes whose column c <= j, so every update is one
          // unconditional FMA (the diagonal tile's strict upper is scratch)
          const double lc0 = __shfl_sync(FULL, T[ti(k, k)][ej], 8 * q + h);
          const double lc1 = __shfl_sync(FULL, T[ti(k, k)][ej], 8 * q + 4 + h);
          const double inv2 = inv * inv;
          const double m0 = 2 * q > j ? -(lc0 * inv2) : 0.0, m1 = 2 * q + 1 > j ? -(lc1 * inv2) : 0.0;
#pragma unroll
          for (int i = k; i < GM; ++i) {
            const double prj = __shfl_sync(FULL, T[ti(i, k)][ej], 4 * r + h);  // u(i)[r][j]
            T[ti(i, k)][0] = fma(prj, m0, T[ti(i, k)][0]);
            T[ti(i, k)][1] = fma(prj, m1, T[ti(i, k)][1]);
          }
        }
      }
      // scale the panel: column c = 2q + e by its reciprocal
      {
        const double s0 = __shfl_sync(FULL, myinv, 2 * q), s1 = __shfl_sync(FULL, myinv, 2 * q + 1);
#pragma unroll
        for (int i = k; i < GM; ++i) {
          T[ti(i, k)][0] *= s0;
          T[ti(i, k)][1] *= s1;
        }
      }
      dkeep[k] = myinv;  // lane j < 8: 1/L[8k+j][8k+j], written after the finiteness check
      // trailing update  T(i,jj) -= P(i) P(jj)^T,  k < jj <= i
      // (an accumulator tile IS an m8n8k4 operand when k-step e of a pair
      // contracts over columns 2q + e: lane (r, q) holds P[r][2q + e] -- the A
      // element of row r and, for P^T, the B element of column r -- so the
      // panel tiles feed the DMMAs straight from their registers, no shuffles)
      if (k + 1 < GM) {
#pragma unroll
        for (int i = k + 1; i < GM; ++i) {
          const double na0 = -T[ti(i, k)][0], na1 = -T[ti(i, k)][1];
#pragma unroll
          for (int jj = k + 1; jj <= i; ++jj) {
            dmma(T[ti(i, jj)], na0, T[ti(jj, k)][0]);
            dmma(T[ti(i, jj)], na1, T[ti(jj, k)][1]);
          }
        }
      }
    }
    // write set: lower triangle of the window; a failing item only rows
    // < iif plus block row iif left of iif (iif = fail & ~3), as the
    // reference stores before returning (ccore.pyx:884-899), and nothing of
    // an unaligned window (level3.py:338-344 factors into scratch)
    const int iif = fail >= 0 ? (fail & ~3) : 0;
    const bool none = fail >= 0 && (g.di & 3) != 0;
    // A NaN / Inf among the results (a non-finite input, or overflow): the
    // masked-multiplier updates may have spread it over more entries of its
    // row than the reference does.  The item is left untouched here and
    // marked (info = PB_INFO_EXACT); potrf_exact_kernel redoes it in the
    // reference's own operation order right after this launch (pb_exact.cu).
    // Detection is one FMA per register (x * 0 is NaN only for NaN / Inf x);
    // a failing item's unused trailing entries count too (rare, still exact).
    double chk = 0.0;
#pragma unroll
    for (int k = 0; k < GM; ++k) chk = fma(dkeep[k], 0.0, chk);
#pragma unroll
    for (int t = 0; t < NT; ++t) chk = fma(T[t][1], 0.0, fma(T[t][0], 0.0, chk));
    const bool nonfinite = !isfinite(chk);
    if (!SYRK && __any_sync(FULL, nonfinite)) {
      if (lane == 0) g.info[b] = PB_INFO_EXACT;
      continue;
    }
    if (lane == 0 && g.info) g.info[b] = fail >= 0 ? fail + g.info_offset : -1;
#pragma unroll
    for (int k = 0; k < GM; ++k) {
      const int c = 8 * k + lane;
      if (lane < 8 && c < n && (fail < 0 || c < fail)) dA[c] = dkeep[k];
    }
    double *Db = g.D.p + b * g.D.stride;
#pragma unroll
    for (int i = 0; i < GM; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int R = 8 * i + r, Cc = 8 * j + 2 * q + e;
          bool w = R < n && Cc <= R && !none;
          if (fail >= 0) w = w && (R < iif || (R < iif + 4 && Cc < iif));
          if (w) Db[offD[i] + 4 * (8 * j + e)] = T[ti(i, j)][e];
        }
  }
}

template <int GM, bool SYRK>
cudaError_t launch_reg(const PotrfArgs &g, cudaStream_t st) {
  auto kern = potrf_reg_kernel<GM, SYRK>;
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32, 0);
    if (occ < 1) occ = 1;
  }
  const ix ctas = g.batch;
  ix grid = (ix)num_sms() * occ;
  if (grid > ctas) grid = ctas;
  if (grid < 1) grid = 1;
  // next-item L2 prefetch of whole panels (measured best; profiles/r01_c2_kernels_ncu.txt)
  const int pf_ok = ((g.ci & 3) == 0 && ((uintptr_t)g.C.p & 15) == 0 && (g.C.stride & 1) == 0) ? 1 : 0;
  kern<<<(unsigned)grid, 32, 0, st>>>(g, pf_ok);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

// 9 <= n <= 16 stays on the bit-exact quad kernel (aligned windows)
bool potrf_reg_ok(const PotrfArgs &g) { return g.m == g.n && g.n >= 17 && g.n <= 64; }

static cudaError_t run_potrf_reg_only(const PotrfArgs &g, cudaStream_t st) {
  const int gm = (int)((g.n + 7) / 8);
  if (g.syrk) {
    switch (gm) {
      case 2: return launch_reg<2, true>(g, st);
      case 3: return launch_reg<3, true>(g, st);
      case 4: return launch_reg<4, true>(g, st);
      case 5: return launch_reg<5, true>(g, st);
      case 6: return launch_reg<6, true>(g, st);
      case 7: return launch_reg<7, true>(g, st);
      case 8: return launch_reg<8, true>(g, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (gm) {
    case 2: return launch_reg<2, false>(g, st);
    case 3: return launch_reg<3, false>(g, st);
    case 4: return launch_reg<4, false>(g, st);
    case 5: return launch_reg<5, false>(g, st);
    case 6: return launch_reg<6, false>(g, st);
    case 7: return launch_reg<7, false>(g, st);
    case 8: return launch_reg<8, false>(g, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t run_potrf_reg(const PotrfArgs &g, cudaStream_t st) {
  const cudaError_t e = run_potrf_reg_only(g, st);
  if (e != cudaSuccess || g.syrk) return e;
  return run_potrf_exact_fixup(g, st);  // items marked PB_INFO_EXACT (non-finite), if any
}

}  // namespace pb
