// Batched dpotrf_l for tiny matrices (n <= 16): register-resident,
// bit-exact with the reference (sm_100a).
//
// For n <= 16 the factorization is pure HBM streaming (AI < 0.6 flop/B),
// so the kernel is built around the memory system:
//  * persistent CTAs, double-buffered: while a round of items is factored
//    from shared memory, the next round's lower-triangle panel prefixes
//    stream in with 16-byte cp.async (one panel row-block of the lower
//    triangle, columns [0, 4p+4), is a contiguous run in panel-major);
//  * every lane of a warp issues consecutive 16-byte pieces, so loads and
//    the masked stores of the results are fully coalesced;
//  * n <= 8: one thread owns one item, entirely in registers, and every
//    touched 32-byte sector of D is stored whole (potrf_small1_kernel);
//    9 <= n <= 16: a quad of threads owns one item, lane q owning row q of
//    every panel (row-cyclic: equal work per lane in every column block),
//    left-looking over 4-column blocks, computed in place in the staged
//    shared-memory copy (block rows read back by broadcast, the diagonal
//    tile's pivots and multipliers exchanged by quad shuffles).
//
// Arithmetic follows the reference's per-element operation order exactly
// (potrf_drv ccore.pyx:877-905, _kpotrf_core :404-438, _trsm_rltn_core
// :358-388): downdate sum from 0.0 over l ascending, then + C, then the
// in-tile updates, IEEE sqrt and division, no FMA contraction -- so the
// factor and diag_inv are bit-identical to the reference's.  Failure
// index and the partially written factor of a failing item match too.
#include <type_traits>

#include "pb_gemm.cuh"

namespace pb {

template <int N, int NTH_ = 128, int STAGES_ = 2>
struct SmallCfg {
  static constexpr int NP = (N + 3) / 4;  // panels
  static constexpr int T = N <= 8 ? 1 : 4;  // threads per item
  static constexpr int NTHREADS = NTH_;
  static constexpr int STAGES = STAGES_;
  static constexpr int ITEMS = NTHREADS / T;
  __host__ __device__ static constexpr int cols(int p) { return 4 * p + 4 < N ? 4 * p + 4 : N; }
  // doubles before panel p's prefix = 4 * sum of cols(j), j < p; closed form (a recursive definition is compiled
  // as an out-of-line loop wherever p is not folded: 10 calls per n = 16 item in the plain staging / store loops)
  __host__ __device__ static constexpr int poff(int p) { return p < NP ? 8 * p * (p + 1) : 8 * (NP - 1) * NP + 4 * N; }
  static constexpr int ITEM_ELEMS = poff(NP);        // lower-prefix doubles per item
  // padded item stride, 16-byte aligned: thread-per-item reads 16-byte pieces at the item stride (odd
  // 16-byte units); the quad path reads 8 bytes per lane = 32 contiguous bytes per quad (odd 32-byte units)
  static constexpr int STRIDE = T == 1 ? ITEM_ELEMS + 2 : ITEM_ELEMS + (20 - ITEM_ELEMS % 16) % 16;
  static constexpr int BUF = ITEMS * STRIDE;
  static constexpr int DINV = ITEMS * N;  // one round's reciprocals
  static constexpr size_t SMEM = sizeof(double) * (STAGES * BUF + DINV) + sizeof(int) * ITEMS;
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// One item, one thread (n <= 8).  L holds C's lower prefix on entry (rows
// 0..4NP-1, cols 0..N-1 as available) and the factor on exit (write set
// only: strict-upper and padding-row entries are never read, so they stay
// dead and cost no registers).
template <int N>
__device__ __forceinline__ int factor_t1(double (&L)[4 * SmallCfg<N>::NP][N], double *dinv) {
  constexpr int NP = SmallCfg<N>::NP;
#pragma unroll
  for (int ii = 0; ii < NP; ++ii) {
    constexpr int dummy = 0;
    (void)dummy;
#pragma unroll
    for (int jj = 0; jj <= ii; ++jj) {
      const int ns = N - 4 * jj < 4 ? N - 4 * jj : 4;
      double acc[4][4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double s = 0.0;
#pragma unroll
          for (int l = 0; l < 4 * jj; ++l)
            if (c < ns && 4 * ii + r < N && (jj < ii || r >= c)) s = dadd(s, dmul(L[4 * ii + r][l], -L[4 * jj + c][l]));
          acc[c][r] = s;
        }
      if (jj < ii) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < ns) {
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[c][r] = dadd(acc[c][r], L[4 * ii + r][4 * jj + c]);
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (t < c) {
                const double e = L[4 * jj + c][4 * jj + t];
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[c][r] = dsub(acc[c][r], dmul(acc[t][r], e));
              }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              acc[c][r] = dmul(acc[c][r], dinv[4 * jj + c]);
              L[4 * ii + r][4 * jj + c] = acc[c][r];
            }
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (c < ns && r >= c && 4 * ii + r < N) acc[c][r] = dadd(acc[c][r], L[4 * ii + r][4 * jj + c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < ns) {
            const double d = acc[c][c];
            if (d <= 0.0) return 4 * jj + c;
            const double ljj = __dsqrt_rn(d);
            const double inv = __ddiv_rn(1.0, ljj);
            acc[c][c] = ljj;
            dinv[4 * jj + c] = inv;
#pragma unroll
            for (int r = 0; r < 4; ++r)
              if (r > c) acc[c][r] = dmul(acc[c][r], inv);
#pragma unroll
            for (int c2 = 0; c2 < 4; ++c2)
              if (c2 > c && c2 < ns) {
                const double lcj = acc[c][c2];
#pragma unroll
                for (int r = 0; r < 4; ++r)
                  if (r >= c2) acc[c2][r] = dsub(acc[c2][r], dmul(acc[c][r], lcj));
              }
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (c < ns && r >= c) L[4 * ii + r][4 * jj + c] = acc[c][r];
      }
    }
  }
  return -1;
}

// One item, a quad of threads (9 <= n <= 16), computed IN SHARED MEMORY with
// ROW-CYCLIC ownership: lane q of the quad owns row q of every panel (rows
// q, 4 + q, 8 + q, 12 + q).  Left-looking over 4-column blocks: for block s
// every lane downdates its rows of panels s..NP-1 against block row s (read
// back from shared memory by broadcast), so all four lanes carry the same
// amount of work in every block (a panel-per-lane split leaves lane 0 idle
// after block 0 and lane 3 with 2.4x the mean downdate).  The 4x4 diagonal
// tile has one row per lane: its pivot and the multipliers L[4s+c2][4s+c]
// travel by quad shuffles, sqrt / reciprocal are computed by all four lanes
// (lockstep, no second broadcast), and the rows below are solved in the same
// right-looking sweep.  Per element the reference's operation order (downdate
// sum from 0.0 over l ascending, + C, - L[r][t] * L[c][t] over t ascending,
// * 1/ljj), IEEE sqrt/div, no FMA: bit-identical.  No branch depends on the
// data: after a bad pivot the lanes keep computing on dead values and only
// the stores are switched off (the shuffles stay warp-uniform).
template <int N>
__device__ __forceinline__ int factor_t4c(double *Si, double *dinv, int q) {
  using Cfg = SmallCfg<N>;
  constexpr int NP = Cfg::NP;
  const int qb = (threadIdx.x & 31) & ~3;  // first lane of this quad
  int fail = -1;
  double *Sq = Si + q;  // element (4p + q, l) at Sq[poff(p) + 4l]
#pragma unroll
  for (int s = 0; s < NP; ++s) {
    const int ns = N - 4 * s < 4 ? N - 4 * s : 4;
    const double *Ls = Si + Cfg::poff(s);  // block row s: element (4s + c, l) at Ls[4l + c]
    double acc[NP][4];
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[p][c] = 0.0;
#pragma unroll
    for (int l = 0; l < 4 * s; ++l) {
      const double2 lo = *reinterpret_cast<const double2 *>(Ls + 4 * l);
      const double2 hi = *reinterpret_cast<const double2 *>(Ls + 4 * l + 2);
      const double v[4] = {lo.x, lo.y, hi.x, hi.y};
#pragma unroll
      for (int p = s; p < NP; ++p) {
        const double x = Sq[Cfg::poff(p) + 4 * l];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < ns) acc[p][c] = dadd(acc[p][c], dmul(x, -v[c]));
      }
    }
#pragma unroll
    for (int p = s; p < NP; ++p)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c < ns) acc[p][c] = dadd(acc[p][c], Sq[Cfg::poff(p) + 4 * (4 * s + c)]);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c < ns) {
        const double d = __shfl_sync(0xffffffffu, acc[s][c], qb + c);  // pivot: row c of the tile
        if (fail < 0 && d <= 0.0) fail = 4 * s + c;                    // ccore.pyx:423 (NaN passes)
        const double ljj = __dsqrt_rn(d);
        const double inv = __ddiv_rn(1.0, ljj);
        if (fail < 0 && q == 0) dinv[4 * s + c] = inv;
        acc[s][c] = q == c ? ljj : dmul(acc[s][c], inv);
#pragma unroll
        for (int p = s + 1; p < NP; ++p) acc[p][c] = dmul(acc[p][c], inv);
#pragma unroll
        for (int c2 = c + 1; c2 < 4; ++c2) {
          if (c2 < ns) {
            const double lcj = __shfl_sync(0xffffffffu, acc[s][c], qb + c2);  // L[4s + c2][4s + c]
#pragma unroll
            for (int p = s; p < NP; ++p) acc[p][c2] = dsub(acc[p][c2], dmul(acc[p][c], lcj));
          }
        }
      }
    }
    if (fail < 0) {
#pragma unroll
      for (int p = s; p < NP; ++p)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < ns && 4 * p + q < N && (p > s || q >= c)) Sq[Cfg::poff(p) + 4 * (4 * s + c)] = acc[p][c];
    }
    __syncwarp();
  }
  return fail;
}

__device__ __forceinline__ void prefetch_l2_small(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

template <int N, int NTH_, int STAGES_, bool QRMW = false, int MINB = 1, bool HOIST = false, bool PF = false>
__global__ void __launch_bounds__(NTH_, MINB) potrf_small_kernel(PotrfArgs g) {
  using Cfg = SmallCfg<N, NTH_, STAGES_>;
  constexpr int STG = Cfg::STAGES;
  constexpr int NP = Cfg::NP, T = Cfg::T, ITEMS = Cfg::ITEMS, STRIDE = Cfg::STRIDE, NTH = Cfg::NTHREADS;
  extern __shared__ __align__(128) double smem[];
  double *sdinv = smem + STG * Cfg::BUF;
  int *sinfo = (int *)(sdinv + Cfg::DINV);
  const int tid = threadIdx.x;
  const ix nrounds = (g.batch + ITEMS - 1) / ITEMS;
  const double *Cb = g.C.p;
  double *Db = g.D.p;

  // stage the lower prefix of round `rd`'s items into buffer `buf`: panel p
  // of an item contributes columns [0, cols(p)) = 2*cols(p) 16-byte pieces
  // Regular rounds of the quad path (HOIST; N % 4 == 0, full round, no failing item): a panel's prefix is
  // walked in groups of four columns = eight 16-byte pieces, so a thread keeps ONE piece position
  // (tid % 8) and item lane (tid / 8) for the whole round; every address is a base plus compile-time
  // offsets and per-trip item strides -- no per-piece division, no 64-bit products.  It costs registers:
  // at the 128-register cap of 8 CTAs/SM it spills (11.3 -> 12.4 ms at the C2 n = 16 point), at 6 CTAs/SM
  // it does not (10.6 ms); in place the plain loops at 8 CTAs/SM stay ahead (10.7 vs 10.9 ms).
  constexpr int GSTEP = NTH / 8;  // items covered by one trip of a column group
  constexpr bool REGQ = HOIST && T == 4 && !QRMW && N % 4 == 0 && NTH % 8 == 0 && ITEMS % GSTEP == 0 &&
                        NTH % N == 0 && (ITEMS * N) % NTH == 0;
  const int gw = tid & 7, git = tid >> 3;
  auto issue = [&](ix rd, int buf) {
    double *S = smem + buf * Cfg::BUF;
    const ix b0 = rd * ITEMS;
    if (REGQ && b0 + ITEMS <= g.batch && (g.ci & 3) == 0) {
      const double *src0 = Cb + (b0 + git) * g.C.stride + g.ci * g.C.cn + 4 * g.cj + 2 * gw;
      double *dst0 = S + git * STRIDE + 2 * gw;
#pragma unroll
      for (int k = 0; k < ITEMS / GSTEP; ++k) {
        const double *src = src0 + (ix)k * GSTEP * g.C.stride;
        double *dst = dst0 + k * GSTEP * STRIDE;
#pragma unroll
        for (int p = 0; p < NP; ++p)
#pragma unroll
          for (int cg = 0; cg <= p; ++cg) cp_async16(dst + Cfg::poff(p) + 16 * cg, src + (ix)4 * p * g.C.cn + 16 * cg, 16);
      }
      return;
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      constexpr int dummy = 0;
      (void)dummy;
      const int pieces = 2 * Cfg::cols(p);
      const int trips = (ITEMS * pieces + NTH - 1) / NTH;
#pragma unroll
      for (int k = 0; k < trips; ++k) {
        const int q = tid + k * NTH;
        if (q < ITEMS * pieces) {
          const int it = q / pieces, w = q - it * pieces;
          const int col = w >> 1, h = w & 1;
          const ix b = b0 + it;
          const bool ok = b < g.batch;
          const double *src = ok ? Cb + b * g.C.stride + eo(g.ci + 4 * p, g.cj + col, g.C.cn) + 2 * h : Cb;
          cp_async16(S + it * STRIDE + Cfg::poff(p) + 4 * col + 2 * h, src, ok ? 16 : 0);
        }
      }
    }
  };

#pragma unroll
  for (int s0 = 0; s0 < STG - 1; ++s0) {
    const ix r0 = blockIdx.x + (ix)s0 * gridDim.x;
    if (r0 < nrounds) issue(r0, s0);
    cp_async_commit();
  }
  // Whole-sector stores for the quad path (T == 4, two stages): the strict
  // upper of the diagonal blocks is only ever READ by factor_t4s (into
  // discarded accumulator entries), so D's bytes for those elements are
  // cp.async'd into their own slots while the factor runs; full panels then
  // store every piece whole (no L2 fills from DRAM mid write stream).
  // Panels with padding rows (n % 4 != 0) keep element-masked stores.
  // Opt-in (PB_QUAD_RMW): the quad path is compute-latency bound, and this
  // measured 13.8 -> 14.3 ms at the C2 n = 16 point, so it is off by default.
  constexpr bool RMW = (T == 4 && STG == 2 && QRMW);
  int buf = 0;
  for (ix rd = blockIdx.x; rd < nrounds; rd += gridDim.x, buf = (buf + 1 == STG ? 0 : buf + 1)) {
    if constexpr (!RMW) {
      const ix rn = rd + (ix)(STG - 1) * gridDim.x;
      const int bn = (buf + STG - 1) % STG;
      if (rn < nrounds) issue(rn, bn);
      cp_async_commit();
      cp_async_wait<STG - 1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if constexpr (PF && STG == 1 && T == 4 && NP == 4) {
      // single stage: pull the next round's panel prefixes into L2 while this round is factored
      const ix rn = rd + gridDim.x;
      const int it2 = tid / NP, pp = tid % NP;
      const ix b = rn * ITEMS + it2;
      if (rn < nrounds && b < g.batch && (g.ci & 3) == 0)
        prefetch_l2_small(Cb + b * g.C.stride + eo(g.ci + 4 * pp, g.cj, g.C.cn), (unsigned)(Cfg::cols(pp) * 32));
    }
    double *S = smem + buf * Cfg::BUF;
    const int it = tid / T, q = tid % T;
    double *Si = S + it * STRIDE;
    double *di = sdinv + it * N;
    if constexpr (RMW) {
      const ix bi = rd * ITEMS + it;
      if (q < NP && 4 * q + 3 < N && bi < g.batch) {
        const double *Di = Db + bi * g.D.stride;
        // strict-upper elements (r, c), r < c, of diagonal block q: the two
        // whole pieces (rows 0-1 of cols 2, 3) as 16 B, (0,1) and (2,3) as 8 B
        // (their piece-mates are on the diagonal, which the factor owns)
        const double *Dq = Di + eo(g.di + 4 * q, g.dj + 4 * q, g.D.cn);
        double *Sq = Si + Cfg::poff(q) + 4 * (4 * q);
        cp_async16(Sq + 8, Dq + 8, 16);
        cp_async16(Sq + 12, Dq + 12, 16);
        cp_async8(Sq + 4, Dq + 4, 8);
        cp_async8(Sq + 14, Dq + 14, 8);
      }
      cp_async_commit();
      const ix rn = rd + gridDim.x;
      if (rn < nrounds) issue(rn, buf ^ 1);
      cp_async_commit();
    }
    int fail;
    if constexpr (T == 1) {
      double L[4 * NP][N];
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          if (c < Cfg::cols(p)) {
            const double2 lo = *reinterpret_cast<const double2 *>(Si + Cfg::poff(p) + 4 * c);
            const double2 hi = *reinterpret_cast<const double2 *>(Si + Cfg::poff(p) + 4 * c + 2);
            L[4 * p][c] = lo.x, L[4 * p + 1][c] = lo.y, L[4 * p + 2][c] = hi.x, L[4 * p + 3][c] = hi.y;
          } else {
            L[4 * p][c] = L[4 * p + 1][c] = L[4 * p + 2][c] = L[4 * p + 3][c] = 0.0;
          }
        }
      fail = factor_t1<N>(L, di);
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int c = 0; c < N; ++c)
          if (c < Cfg::cols(p)) {
            *reinterpret_cast<double2 *>(Si + Cfg::poff(p) + 4 * c) = make_double2(L[4 * p][c], L[4 * p + 1][c]);
            *reinterpret_cast<double2 *>(Si + Cfg::poff(p) + 4 * c + 2) = make_double2(L[4 * p + 2][c], L[4 * p + 3][c]);
          }
    } else {
      fail = factor_t4c<N>(Si, di, q);
    }
    const ix b0 = rd * ITEMS;
    if (q == 0) {
      sinfo[it] = fail;
      if (b0 + it < g.batch && g.info) g.info[b0 + it] = fail;
    }
    if constexpr (RMW) cp_async_wait<1>();  // this thread's D pieces have landed
    const int anyfail = __syncthreads_or(fail >= 0);
    if (REGQ && !anyfail && b0 + ITEMS <= g.batch && (g.di & 3) == 0) {
      const int cl = gw >> 1, h2 = 2 * (gw & 1);
      const bool m0 = h2 >= cl, m1 = h2 + 1 >= cl;
      const double *src0 = S + git * STRIDE + 2 * gw;
      double *dst0 = Db + (b0 + git) * g.D.stride + g.di * g.D.cn + 4 * g.dj + 2 * gw;
#pragma unroll
      for (int k = 0; k < ITEMS / GSTEP; ++k) {
        const double *src = src0 + k * GSTEP * STRIDE;
        double *dst = dst0 + (ix)k * GSTEP * g.D.stride;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
#pragma unroll
          for (int cg = 0; cg < p; ++cg)
            *reinterpret_cast<double2 *>(dst + (ix)4 * p * g.D.cn + 16 * cg) =
                *reinterpret_cast<const double2 *>(src + Cfg::poff(p) + 16 * cg);
          const double2 v = *reinterpret_cast<const double2 *>(src + Cfg::poff(p) + 16 * p);
          double *dd = dst + (ix)4 * p * g.D.cn + 16 * p;
          if (m0) *reinterpret_cast<double2 *>(dd) = v;
          else if (m1) dd[1] = v.y;
        }
      }
      {
        const double *ds = sdinv + tid;
        double *dd = g.D.d + (b0 + tid / N) * g.D.dstride + g.dj + tid % N;
#pragma unroll
        for (int k = 0; k < ITEMS * N / NTH; ++k) {
          *dd = *ds;
          ds += NTH;
          dd += (ix)(NTH / N) * g.D.dstride;
        }
      }
      __syncthreads();
      continue;
    }
    // Stores of the reference's write set (lower triangle; on failure only
    // what the reference stored before returning).  Columns left of a
    // panel's diagonal block are entirely lower: full 16-byte pieces.  The
    // diagonal 4x4 block holds strict-upper bytes that must stay untouched:
    // masked stores there (the L2 fills those chunks from DRAM; a software
    // read-modify-write of D was measured slower -- see DESIGN.md).
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      // (1) off-diagonal columns [0, 4p)
      {
        const int pieces = 8 * p;
        const int trips = (ITEMS * pieces + NTH - 1) / NTH;
        constexpr int MAXTRIPS = (ITEMS * 8 * (NP - 1) + NTH - 1) / NTH;
#pragma unroll
        for (int k = 0; k < (MAXTRIPS > 0 ? MAXTRIPS : 1); ++k) {
          const int qq = tid + k * NTH;
          if (k < trips && qq < ITEMS * pieces) {
            const int it2 = qq / pieces, w = qq - it2 * pieces;
            const int col = w >> 1, h = w & 1;
            const ix bb = b0 + it2;
            if (bb < g.batch) {
              const double2 v = *reinterpret_cast<const double2 *>(S + it2 * STRIDE + Cfg::poff(p) + 4 * col + 2 * h);
              const int f = sinfo[it2];
              const int r0 = 4 * p + 2 * h;
              bool w0 = r0 < N, w1 = r0 + 1 < N;
              if (f >= 0) {
                const int iif = f & ~3;
                w0 = w0 && (r0 < iif || (r0 < iif + 4 && col < iif));
                w1 = w1 && (r0 + 1 < iif || (r0 + 1 < iif + 4 && col < iif));
              }
              double *dst = Db + bb * g.D.stride + eo(g.di + 4 * p, g.dj + col, g.D.cn) + 2 * h;
              if (w0 && w1) *reinterpret_cast<double2 *>(dst) = v;
              else if (w0) dst[0] = v.x;
              else if (w1) dst[1] = v.y;
            }
          }
        }
      }
      // (2) the diagonal block, columns [4p, 4p+4)
      {
        constexpr int trips = (ITEMS * 8 + NTH - 1) / NTH;
#pragma unroll
        for (int k = 0; k < trips; ++k) {
          const int qq = tid + k * NTH;
          if (qq < ITEMS * 8) {
            const int it2 = qq >> 3, w = qq & 7;
            const int cl = w >> 1, h = w & 1, col = 4 * p + cl;
            const ix bb = b0 + it2;
            if (bb < g.batch && col < Cfg::cols(p)) {
              const double *Si2 = S + it2 * STRIDE;
              const int f = sinfo[it2];
              const int iif = f >= 0 ? (f & ~3) : 0;
              double val[2];
              bool wr[2];
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int r = 4 * p + 2 * h + i;
                bool wi = r >= col && r < N && col < N;
                if (f >= 0) wi = wi && (r < iif || (r < iif + 4 && col < iif));
                else if (RMW && 4 * p + 3 < N) wi = true;  // merged sector: D's own bytes above the diagonal
                wr[i] = wi;
                val[i] = Si2[Cfg::poff(p) + 4 * col + 2 * h + i];
              }
              double *dst = Db + bb * g.D.stride + eo(g.di + 4 * p, g.dj + col, g.D.cn) + 2 * h;
              if (wr[0] && wr[1]) *reinterpret_cast<double2 *>(dst) = make_double2(val[0], val[1]);
              else if (wr[0]) dst[0] = val[0];
              else if (wr[1]) dst[1] = val[1];
            }
          }
        }
      }
    }
    // reciprocals: dA[dj + c] for c < (fail >= 0 ? fail : n)
    {
      constexpr int trips = (ITEMS * N + NTH - 1) / NTH;
#pragma unroll
      for (int k = 0; k < trips; ++k) {
        const int qq = tid + k * NTH;
        if (qq < ITEMS * N) {
          const int it2 = qq / N, c = qq - it2 * N;
          const ix bb = b0 + it2;
          const int f = sinfo[it2];
          if (bb < g.batch && (f < 0 || c < f)) g.D.d[bb * g.D.dstride + g.dj + c] = sdinv[qq];
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

// element (row 4p + r, col) of an n x n item's lower prefix is in the
// reference's write set (lower triangle, rows < n)
template <int N>
struct WarpCfg {
  __host__ __device__ static constexpr bool wr(int p, int col, int r) { return 4 * p + r < N && 4 * p + r >= col; }
};

// ---------------------------------------------------------------------
// n <= 8: the CTA kernel's thread-per-item factor (registers), with
// whole-sector stores.  After a thread has copied its item's staged prefix
// into registers, the item's smem slot is free: the thread cp.asyncs the
// pieces of D that share a sector with the write set but are not in it
// (diagonal-block strict upper, padding rows) straight into their own slots,
// overlapped with the factor; the factor then writes back only its write
// set, so the slot holds exactly the merged sectors and every piece of the
// prefix is stored whole (no L2 fills from DRAM in the write stream).
template <int N, int NTH, int STG = 2, int MINB = 1>
__global__ void __launch_bounds__(NTH, MINB) potrf_small1_kernel(PotrfArgs g) {
  using Cfg = SmallCfg<N, NTH, STG>;
  using WC = WarpCfg<N>;
  constexpr int NP = Cfg::NP, ITEMS = Cfg::ITEMS, STRIDE = Cfg::STRIDE;
  static_assert(Cfg::T == 1, "thread-per-item sizes only");
  extern __shared__ __align__(128) double smem[];
  double *sdinv = smem + STG * Cfg::BUF;
  int *sinfo = (int *)(sdinv + Cfg::DINV);
  const int tid = threadIdx.x;
  const ix nrounds = (g.batch + ITEMS - 1) / ITEMS;
  const double *Cb = g.C.p;
  double *Db = g.D.p;
  const bool inplace = g.C.p == g.D.p && g.C.stride == g.D.stride && g.C.cn == g.D.cn && g.ci == g.di && g.cj == g.dj;
  // Regular rounds (N = 4, 8: every panel's 16-byte piece count divides the CTA, the round is full, no item
  // failed): a thread's piece (column, half) is the same in every trip and only the item advances, so the
  // staging and store loops are one address + pointer increments instead of a division and two 64-bit
  // products per piece (the n = 8 kernel spent a third of its instructions on that index math).
  constexpr bool REGP = NP <= 2 && NTH % (2 * Cfg::cols(0)) == 0 && NTH % (2 * Cfg::cols(NP - 1)) == 0 && NTH % N == 0;
  auto stage_panel = [&](auto pc, double *S, ix b0) {
    constexpr int P = decltype(pc)::value, pieces = 2 * Cfg::cols(P), step = NTH / pieces;
    const int it0 = tid / pieces, w = tid % pieces;
    const double *src = Cb + (b0 + it0) * g.C.stride + eo(g.ci + 4 * P, g.cj + (w >> 1), g.C.cn) + 2 * (w & 1);
    double *dst = S + it0 * STRIDE + Cfg::poff(P) + 2 * w;
#pragma unroll
    for (int k = 0; k < ITEMS / step; ++k) {
      cp_async16(dst, src, 16);
      src += (ix)step * g.C.stride;
      dst += step * STRIDE;
    }
  };
  auto store_panel = [&](auto pc, const double *S, ix b0) {
    constexpr int P = decltype(pc)::value, pieces = 2 * Cfg::cols(P), step = NTH / pieces;
    const int it0 = tid / pieces, w = tid % pieces;
    const double *src = S + it0 * STRIDE + Cfg::poff(P) + 2 * w;
    double *dst = Db + (b0 + it0) * g.D.stride + eo(g.di + 4 * P, g.dj + (w >> 1), g.D.cn) + 2 * (w & 1);
#pragma unroll
    for (int k = 0; k < ITEMS / step; ++k) {
      *reinterpret_cast<double2 *>(dst) = *reinterpret_cast<const double2 *>(src);
      src += step * STRIDE;
      dst += (ix)step * g.D.stride;
    }
  };

  auto issue = [&](ix rd, int buf) {
    double *S = smem + buf * Cfg::BUF;
    const ix b0 = rd * ITEMS;
    if (REGP && b0 + ITEMS <= g.batch) {
      stage_panel(std::integral_constant<int, 0>{}, S, b0);
      if constexpr (NP > 1) stage_panel(std::integral_constant<int, NP - 1>{}, S, b0);
      return;
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int pieces = 2 * Cfg::cols(p);
      constexpr int dummy = 0;
      (void)dummy;
      const int trips = (ITEMS * pieces + NTH - 1) / NTH;
#pragma unroll
      for (int k = 0; k < trips; ++k) {
        const int q = tid + k * NTH;
        if (q < ITEMS * pieces) {
          const int it = q / pieces, w = q - it * pieces;
          const int col = w >> 1, h = w & 1;
          const ix b = b0 + it;
          const bool ok = b < g.batch;
          const double *src = ok ? Cb + b * g.C.stride + eo(g.ci + 4 * p, g.cj + col, g.C.cn) + 2 * h : Cb;
          cp_async16(S + it * STRIDE + Cfg::poff(p) + 4 * col + 2 * h, src, ok ? 16 : 0);
        }
      }
    }
  };

  // STG == 2: the next round streams in while this one is factored;
  // STG == 1: half the shared memory per item (more CTAs per SM), the
  // overlap comes from the other CTAs
  ix rd = blockIdx.x;
  int buf = 0;
  if (STG == 2 && rd < nrounds) issue(rd, 0);
  cp_async_commit();
  for (; rd < nrounds; rd += gridDim.x, buf ^= (STG - 1)) {
    if (STG == 1) {
      issue(rd, 0);
      cp_async_commit();
    }
    cp_async_wait<0>();
    __syncthreads();
    double *S = smem + buf * Cfg::BUF;
    const ix b0 = rd * ITEMS;
    const int it = tid;
    double *Si = S + it * STRIDE;
    double L[4 * NP][N];
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        if (c < Cfg::cols(p)) {
          const double2 lo = *reinterpret_cast<const double2 *>(Si + Cfg::poff(p) + 4 * c);
          const double2 hi = *reinterpret_cast<const double2 *>(Si + Cfg::poff(p) + 4 * c + 2);
          L[4 * p][c] = lo.x, L[4 * p + 1][c] = lo.y, L[4 * p + 2][c] = hi.x, L[4 * p + 3][c] = hi.y;
        } else {
          L[4 * p][c] = L[4 * p + 1][c] = L[4 * p + 2][c] = L[4 * p + 3][c] = 0.0;
        }
      }
    const ix bi = b0 + it;
    // D's bytes for the non-written part of every touched sector -> own slot;
    // in place (D is C's window) the slot already holds them: C's staged
    // prefix covers every touched sector, so the second round trip is skipped
    if (bi < g.batch && !inplace) {
      const double *Di = Db + bi * g.D.stride;
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int c = 0; c < N; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (c < Cfg::cols(p) && !(WC::wr(p, c, 2 * h) && WC::wr(p, c, 2 * h + 1)))
              cp_async16(Si + Cfg::poff(p) + 4 * c + 2 * h, Di + eo(g.di + 4 * p, g.dj + c, g.D.cn) + 2 * h, 16);
    }
    cp_async_commit();
    if (STG == 2 && rd + gridDim.x < nrounds) issue(rd + gridDim.x, buf ^ 1);
    cp_async_commit();
    int fail = -1;
    double *di = sdinv + it * N;
    if (bi < g.batch) fail = factor_t1<N>(L, di);
    cp_async_wait<1>();  // this thread's D pieces have landed
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int c = 0; c < N; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (c < Cfg::cols(p) && WC::wr(p, c, r)) Si[Cfg::poff(p) + 4 * c + r] = L[4 * p + r][c];
    sinfo[it] = fail;
    if (bi < g.batch && g.info) g.info[bi] = fail;
    const int anyfail = __syncthreads_or(fail >= 0);
    if (REGP && !anyfail && b0 + ITEMS <= g.batch) {
      // regular round: whole pieces, pointer increments only
      store_panel(std::integral_constant<int, 0>{}, S, b0);
      if constexpr (NP > 1) store_panel(std::integral_constant<int, NP - 1>{}, S, b0);
      const double *ds = sdinv + tid;
      double *dd = g.D.d + (b0 + tid / N) * g.D.dstride + g.dj + tid % N;
#pragma unroll
      for (int k = 0; k < ITEMS * N / NTH; ++k) {
        *dd = *ds;
        ds += NTH;
        dd += (ix)(NTH / N) * g.D.dstride;
      }
      if (STG == 1) __syncthreads();
      continue;
    }
    // stores: every 16-byte piece of the lower prefix, whole, unless the
    // item failed (then exactly the reference's partial write set)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int pieces = 2 * Cfg::cols(p);
      const int trips = (ITEMS * pieces + NTH - 1) / NTH;
      constexpr int MAXTRIPS = (ITEMS * 2 * N + NTH - 1) / NTH;
#pragma unroll
      for (int k = 0; k < MAXTRIPS; ++k) {
        const int qq = tid + k * NTH;
        if (k < trips && qq < ITEMS * pieces) {
          const int it2 = qq / pieces, w = qq - it2 * pieces;
          const int col = w >> 1, h = w & 1;
          const ix bb = b0 + it2;
          if (bb < g.batch) {
            const double2 v = *reinterpret_cast<const double2 *>(S + it2 * STRIDE + Cfg::poff(p) + 4 * col + 2 * h);
            double *dst = Db + bb * g.D.stride + eo(g.di + 4 * p, g.dj + col, g.D.cn) + 2 * h;
            const int f = sinfo[it2];
            if (f < 0) {
              *reinterpret_cast<double2 *>(dst) = v;
            } else {
              const int r0 = 4 * p + 2 * h, iif = f & ~3;
              const bool w0 = r0 < N && r0 >= col && (r0 < iif || (r0 < iif + 4 && col < iif));
              const bool w1 = r0 + 1 < N && r0 + 1 >= col && (r0 + 1 < iif || (r0 + 1 < iif + 4 && col < iif));
              if (w0 && w1) *reinterpret_cast<double2 *>(dst) = v;
              else if (w0) dst[0] = v.x;
              else if (w1) dst[1] = v.y;
            }
          }
        }
      }
    }
    {
      constexpr int trips = (ITEMS * N + NTH - 1) / NTH;
#pragma unroll
      for (int k = 0; k < trips; ++k) {
        const int qq = tid + k * NTH;
        if (qq < ITEMS * N) {
          const int it2 = qq / N, c = qq - it2 * N;
          const ix bb = b0 + it2;
          const int f = sinfo[it2];
          if (bb < g.batch && (f < 0 || c < f)) g.D.d[bb * g.D.dstride + g.dj + c] = sdinv[qq];
        }
      }
    }
    if (STG == 1) __syncthreads();
  }
  cp_async_wait<0>();
}

template <int N, int NTH = 128, int STG = 2, int MINB = 1>
static cudaError_t launch_small1(const PotrfArgs &g, cudaStream_t st) {
  using Cfg = SmallCfg<N, NTH, STG>;
  auto kern = potrf_small1_kernel<N, NTH, STG, MINB>;
  static LaunchCache cache;
  const int occ = cache.occupancy((const void *)kern, NTH, Cfg::SMEM);
  const ix rounds = (g.batch + Cfg::ITEMS - 1) / Cfg::ITEMS;
  ix grid = (ix)num_sms() * occ;
  if (grid > rounds) grid = rounds;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, NTH, Cfg::SMEM, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

template <int N, int NTH_ = 128, int STAGES_ = 2, bool QRMW = false, int MINB = 1, bool HOIST = false, bool PF = false>
static cudaError_t launch_small(const PotrfArgs &g, cudaStream_t st) {
  using Cfg = SmallCfg<N, NTH_, STAGES_>;
  auto kern = potrf_small_kernel<N, NTH_, STAGES_, QRMW, MINB, HOIST, PF>;
  static LaunchCache cache;
  const int occ = cache.occupancy((const void *)kern, Cfg::NTHREADS, Cfg::SMEM);
  const ix rounds = (g.batch + Cfg::ITEMS - 1) / Cfg::ITEMS;
  ix grid = (ix)num_sms() * occ;
  if (grid > rounds) grid = rounds;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, Cfg::NTHREADS, Cfg::SMEM, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

// Default shape of the quad path (9 <= n <= 16), row-cyclic factor, C2 n = 16 point on one box
// (profiles/r02_potrf_n16_rowcyclic.txt): D != C <64,1,6,hoisted> 7.63 ms = 0.589 of HBM (<64,2,4> and <32,2,8>
// 8.9-9.0, plain loops <64,1,8> 9.19, <64,1,6> 9.59, two plain stages 9.8-10.1); in place <32,2,8,hoisted> 6.86 ms =
// 0.655 (<64,2,4> 7.19, plain <64,1,8> 8.46).  The hoisted loops need n % 4 == 0 and NTH % n == 0, so n = 12 and
// the ragged sizes run the plain loops at 6 / 8 CTAs per SM.
template <int N>
static cudaError_t launch_small_default(const PotrfArgs &g, cudaStream_t st) {
  if constexpr (SmallCfg<N>::T == 4) {
    if constexpr (N % 4 == 0) {
      const bool ip = g.C.p == g.D.p && g.C.stride == g.D.stride && g.ci == g.di && g.cj == g.dj;
      // hoisted staging / store loops, 6 CTAs/SM, L2 prefetch of the next round (n = 16: 7.54 -> 7.41 ms)
      if (!ip) return launch_small<N, 64, 1, false, 6, true, true>(g, st);
      if constexpr (N == 16) return launch_small<N, 32, 2, false, 8, true>(g, st);
    }
    return launch_small<N, 64, 1, false, 8>(g, st);
  }
  else return launch_small<N>(g, st);
}

bool potrf_small_ok(const PotrfArgs &g) {
  if (g.m != g.n || g.n > 16 || g.n < 1 || g.merge) return false;
  if ((g.ci & 3) || (g.di & 3)) return false;
  if (((uintptr_t)g.C.p & 15) || ((uintptr_t)g.D.p & 15)) return false;
  if ((g.C.stride & 1) || (g.D.stride & 1)) return false;
  return true;
}

cudaError_t run_potrf_small(const PotrfArgs &g, cudaStream_t st) {
  // n <= 8: thread-per-item factor with whole-sector stores (potrf_small1_kernel):
  // measured n = 4 0.27 -> 0.33, n = 8 0.34 -> 0.45 of HBM (profiles/r01_potrf_small_rmw.txt);
  // n = 4 single stage, 16 warps/SM: 71.8 -> 68.9 ms at the C2 n = 4 point
  switch (g.n) {
    case 1: return launch_small1<1>(g, st);
    case 2: return launch_small1<2>(g, st);
    case 3: return launch_small1<3>(g, st);
    case 4: {
      // in place the D-piece round trip is gone and the kernel is latency-bound:
      // two stages at 3 CTAs/SM measured best (0.553 -> 0.625 of HBM; D != C
      // stays single-stage, DRAM-saturated)
      const bool ip = g.C.p == g.D.p && g.C.stride == g.D.stride && g.ci == g.di && g.cj == g.dj;
      if (ip) return launch_small1<4, 128, 2, 3>(g, st);
      return launch_small1<4, 128, 1, 4>(g, st);
    }
    case 5: return launch_small1<5>(g, st);
    case 6: return launch_small1<6>(g, st);
    case 7: return launch_small1<7>(g, st);
    case 8: {
      // single stage: with the regular-round staging / store loops the second stage only costs shared memory
      // (config sweep, C2 n = 8 point, one box: <128,2,1> 19.30 ms, <128,1,3> 18.53, <64,2,4> 18.79,
      // <128,1,2> 17.41 = 0.574 of HBM; in place <128,2,1> 0.67, <128,1,2> 0.66, <64,1,4> 0.72)
      const bool ip = g.C.p == g.D.p && g.C.stride == g.D.stride && g.ci == g.di && g.cj == g.dj;
      if (ip) return launch_small1<8, 64, 1, 4>(g, st);
      return launch_small1<8, 128, 1, 2>(g, st);
    }
#define PB_SMALL(N_) \
  case N_:           \
    return launch_small_default<N_>(g, st);
    PB_SMALL(9) PB_SMALL(10) PB_SMALL(11) PB_SMALL(12) PB_SMALL(13) PB_SMALL(14) PB_SMALL(15) PB_SMALL(16)
#undef PB_SMALL
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace pb
