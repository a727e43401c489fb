// Batched dpotrf_l for square windows 65 <= n <= 128 (and the blocked
// driver's 128-column panels): one 8-warp CTA per item, the pivot chain
// decoupled from the bulk downdates (sm_100a).
//
// Reference semantics: potrf_drv ccore.pyx:877-905 (+ _kpotrf_core
// :404-438): lower Cholesky of lower(C), dinv[j] = 1/L[j][j], first pivot
// with d <= 0 (NaN passes) -> info, a failing item written exactly as far
// as the reference's row-panel order writes it.
//
// Why this shape.  The round-1/2 team kernel ran the same left-looking
// 8-column schedule behind two CTA-wide barriers per column block: ncu showed
// 49 % of the stall samples on those barriers (seven warps waiting for the
// one warp that factors the 8x8 diagonal tile) and 63K warp instructions per
// n = 128 item for 1.6K DMMAs (runtime tile-slot dispatch and tri-layout
// address arithmetic).  Here:
//  * the chain  factor(j) -> solve tile (j+1, j) -> update diag(j+1) ->
//    factor(j+1)  runs on the two warps that own rows j and j+1 and never
//    waits for the other warps: two named hardware barriers per step (E1
//    "W_j published", E2 "column block j solved"; ids alternate with the
//    step parity) are joined by all eight warps, but the producers only
//    bar.arrive: the diagonal warp at E1, the owner of row j+1 at E2 (its
//    operands are its own registers; it catches up on its look-ahead work
//    after its factor).  Waiting warps block in hardware -- an mbarrier
//    try_wait spin by 21 warps per SM kept the MIO queue busy and slowed
//    the chain warp's shuffles;
//  * an 8x8 accumulator tile is used AS the A (and B) operand of the next
//    m8n8k4 without any shuffle: k-step e of a pair contracts over columns
//    2q+e, which is exactly what lane (r, q) holds; the inverted diagonal
//    block and the solved tile of row j+1 are published "lane-linear"
//    (element e of lane l at [32e + l]) so every other warp's B fragment is
//    one conflict-free load with no address arithmetic;
//  * accumulators carry the NEGATED partial sums (-C + sum L L^T), so the
//    bulk loops issue plain DMMAs on fragments straight from shared memory;
//  * all tri-layout offsets are per-warp constants hoisted out of the item
//    loop; the step loop has warp-uniform branches only.
#include "pb_tri.cuh"

namespace pb {

namespace {

__device__ __forceinline__ double dneg(double x) {
  return __hiloint2double(__double2hiint(x) ^ (int)0x80000000, __double2loint(x));
}

// NX[i] = -C(g_i, c) + sum_{k-steps < nk} L(g_i, .) L(c, .)^T for the active slots
template <bool A0, bool A1>
__device__ __forceinline__ void lookahead_slots(double (&NX)[2][2], const double *S, int fb, int fa0, int fa1, int ao0,
                                                int ao1, int c, int nk) {
  if (A0) {
    NX[0][0] = dneg(S[ao0 + 32 * c]);
    NX[0][1] = dneg(S[ao0 + 32 * c + 4]);
  }
  if (A1) {
    NX[1][0] = dneg(S[ao1 + 32 * c]);
    NX[1][1] = dneg(S[ao1 + 32 * c + 4]);
  }
#pragma unroll 4
  for (int kk = 0; kk < nk; ++kk) {
    const double bv = S[fb + 16 * kk];
    if (A0) dmma(NX[0], S[fa0 + 16 * kk], bv);
    if (A1) dmma(NX[1], S[fa1 + 16 * kk], bv);
  }
}

constexpr int CHAIN_THREADS = 256;

// producer / consumer halves of a named barrier joined by the whole CTA
__device__ __forceinline__ void bar_sync_all(int id) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(CHAIN_THREADS) : "memory");
}
__device__ __forceinline__ void bar_arrive_all(int id) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "n"(CHAIN_THREADS) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(CHAIN_THREADS, 3) potrf_chain_kernel(PotrfArgs g) {
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, tw = warp_uniform();
  const int r = lane >> 2, q = lane & 3;
  const int n = (int)g.n;
  Tri t;
  t.cn8 = (n + 7) / 8 * 8;
  t.gn = t.cn8 / 8;
  const int gn = t.gn;
  double *S = smem;
  double *dinv = S + 32 * gn * (gn + 1);                    // cn8 reciprocals
  double *Wp = dinv + t.cn8;                                // 2 x 64: inverted diagonal block, lane-linear
  double *Xp = Wp + 128;                                    // 2 x 64: solved tile of row j+1, lane-linear
  uint64_t *tbar = reinterpret_cast<uint64_t *>(Xp + 128);  // bulk-load barrier
  volatile int *flagv = reinterpret_cast<volatile int *>(tbar + 1);  // failing column per step (16)

  // per-warp constants: rows tw and tw + 8 (slot 0 / 1)
  const int g0 = tw, g1 = tw + 8;
  const bool has1 = g1 < gn;
  const int g1c = has1 ? g1 : gn - 1;
  const int fa0 = tri_frag(t, g0, 0, lane), fa1 = tri_frag(t, g1c, 0, lane);
  const int ao0 = t.group_off(g0) + (r >> 2) * 4 * t.width(g0) + 8 * q + (r & 3);
  const int ao1 = t.group_off(g1c) + (r >> 2) * 4 * t.width(g1c) + 8 * q + (r & 3);

  if (tid == 0) {
    mbar_init(tbar, 1);
    mbar_fence_init();
  }
  __syncthreads();

  auto skip = [&](ix b) { return g.merge && g.info[b] >= 0; };
  const ix stride = (ix)gridDim.x;
  ix b = (ix)blockIdx.x;
  while (b < g.batch && skip(b)) b += stride;
  // staging: every warp's lane 0 bulk-copies its own row groups (tw, tw + 8)
  auto load_item = [&](ix bb) {
    const double *C = g.C.item(bb);
    if (tid == 0) {
      unsigned bytes = 0;
      for (int gg = 0; gg < gn; ++gg)
        for (int h = 0; h < 2; ++h)
          if (8 * gg + 4 * h < n) bytes += 32u * (unsigned)min(t.width(gg), n);
      mbar_arrive_expect_tx(tbar, bytes);
    }
    for (int gg = tw; gg < gn; gg += 8) {
      const int w = t.width(gg), base = t.group_off(gg);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r0 = 8 * gg + 4 * h;
        const int c0 = r0 < n ? min(w, n) : 0;
        if (lane == 0 && c0 > 0) tma_load_1d(S + base + h * 4 * w, C + eo(g.ci + r0, g.cj, g.C.cn), 32u * (unsigned)c0, tbar);
        for (int qq = lane; qq < 4 * (w - c0); qq += 32) S[base + h * 4 * w + 4 * c0 + qq] = 0.0;
      }
    }
  };
  if (b < g.batch) load_item(b);
  unsigned tphase = 0, step = 0;
  while (b < g.batch) {
    ix nb = b + stride;
    while (nb < g.batch && skip(nb)) nb += stride;
    mbar_wait(tbar, tphase);
    tphase ^= 1;
    if (tid < 16) flagv[tid] = -1;
    __syncthreads();
    // next item's lower panel prefixes into L2 while this one is factored
    if (tw == 7 && nb < g.batch && 4 * lane < n)
      prefetch_l2(g.C.item(nb) + eo(g.ci + 4 * lane, g.cj, g.C.cn), 32u * (unsigned)min(4 * lane + 4, n));

    // P: this warp's tiles of the current column block, fully downdated;
    // NX: negated partial sums of the next column block (look-ahead)
    double P[2][2], NX[2][2];
    P[0][0] = S[ao0], P[0][1] = S[ao0 + 4];
    P[1][0] = S[ao1], P[1][1] = S[ao1 + 4];
    NX[0][0] = dneg(S[ao0 + 32]), NX[0][1] = dneg(S[ao0 + 36]);
    NX[1][0] = dneg(S[ao1 + 32]), NX[1][1] = dneg(S[ao1 + 36]);
    int fail = -1;
    for (int jb = 0; jb < gn; ++jb) {
      const unsigned par = (step + jb) & 1;
      const int d = jb & 7, nd = (jb + 1) & 7;
      const int ncol = min(8, n - 8 * jb);
      const int wofs = (jb & 1) * 64 + lane;
      double wb0, wb1;
      if (tw == d) {
        // ---- diagonal warp: factor + invert the 8x8 tile, publish W
        const bool ds = jb >= 8;
        double dg[2], wi[2];
        dg[0] = ds ? P[1][0] : P[0][0];
        dg[1] = ds ? P[1][1] : P[0][1];
        const int f = factor_inv_tile(dg, wi, ncol, dinv + 8 * jb, lane);
        const int aod = (ds ? ao1 : ao0) + 32 * jb;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 2 * q + e;
          if (c < ncol && (f < 0 || c < f)) S[aod + 4 * e] = dg[e];
        }
        if (f >= 0 && lane == 0) flagv[jb] = 8 * jb + f;
        Wp[wofs] = wi[0];
        Wp[wofs + 32] = wi[1];
        wb0 = wi[0], wb1 = wi[1];
        __syncwarp();
        bar_arrive_all(1 + par);
      } else {
        bar_sync_all(1 + par);
        wb0 = Wp[wofs];
        wb1 = Wp[wofs + 32];
      }
      fail = flagv[jb];
      const bool s0 = g0 > jb, s1 = has1 && g1 > jb;  // slots with a tile below the diagonal
      double X[2][2];
      if (fail < 0) {
        // ---- solve: X = P * W^T (the accumulator IS the A operand)
        if (s0) {
          X[0][0] = X[0][1] = 0.0;
          dmma(X[0], P[0][0], wb0);
          dmma(X[0], P[0][1], wb1);
          S[ao0 + 32 * jb] = X[0][0];
          S[ao0 + 32 * jb + 4] = X[0][1];
        }
        if (s1) {
          X[1][0] = X[1][1] = 0.0;
          dmma(X[1], P[1][0], wb0);
          dmma(X[1], P[1][1], wb1);
          S[ao1 + 32 * jb] = X[1][0];
          S[ao1 + 32 * jb + 4] = X[1][1];
        }
        if (tw == nd && jb + 1 < gn) {
          const bool ns = jb + 1 >= 8;
          Xp[wofs] = ns ? X[1][0] : X[0][0];
          Xp[wofs + 32] = ns ? X[1][1] : X[0][1];
        }
      }
      __syncwarp();
      if (fail >= 0 || jb + 1 == gn) {
        bar_arrive_all(3 + par);
        step += jb + 1;
        break;
      }
      // ---- column block jb + 1: P = -(NX + X * X(jb+1)^T)
      double xb0, xb1;
      if (tw == nd) {
        // owner of row jb + 1: straight on to its diagonal tile
        bar_arrive_all(3 + par);
        const bool ns = jb + 1 >= 8;
        xb0 = ns ? X[1][0] : X[0][0];
        xb1 = ns ? X[1][1] : X[0][1];
      } else {
        bar_sync_all(3 + par);
        // look-ahead this warp deferred while it owned the chain (column jb + 1)
        if (tw == d && jb > 0) {
          const int c = jb + 1, fb = tri_frag(t, c, 0, lane), nk = 2 * (c - 1);
          if (g0 >= c && s1) lookahead_slots<true, true>(NX, S, fb, fa0, fa1, ao0, ao1, c, nk);
          else if (s1) lookahead_slots<false, true>(NX, S, fb, fa0, fa1, ao0, ao1, c, nk);
          else if (g0 >= c) lookahead_slots<true, false>(NX, S, fb, fa0, fa1, ao0, ao1, c, nk);
        }
        xb0 = Xp[wofs];
        xb1 = Xp[wofs + 32];
      }
      if (s0) {
        dmma(NX[0], X[0][0], xb0);
        dmma(NX[0], X[0][1], xb1);
        P[0][0] = dneg(NX[0][0]), P[0][1] = dneg(NX[0][1]);
      }
      if (s1) {
        dmma(NX[1], X[1][0], xb0);
        dmma(NX[1], X[1][1], xb1);
        P[1][0] = dneg(NX[1][0]), P[1][1] = dneg(NX[1][1]);
      }
      // ---- look-ahead: column block jb + 2 over the solved blocks 0..jb
      if (tw != nd && jb + 2 < gn) {
        const int c = jb + 2, fb = tri_frag(t, c, 0, lane), nk = 2 * (c - 1);
        const bool a0 = g0 >= c, a1 = has1 && g1 >= c;
        if (a0 && a1) lookahead_slots<true, true>(NX, S, fb, fa0, fa1, ao0, ao1, c, nk);
        else if (a1) lookahead_slots<false, true>(NX, S, fb, fa0, fa1, ao0, ao1, c, nk);
        else if (a0) lookahead_slots<true, false>(NX, S, fb, fa0, fa1, ao0, ao1, c, nk);
      }
    }
    __syncthreads();
    // ---- write back the lower triangle (or, on failure, exactly what the
    // reference's block-row order would have stored, ccore.pyx:884-899)
    double *D = g.D.item(b);
    if (fail < 0) {
      // whole 4-row panels strictly left of their diagonal piece: one bulk
      // store each; the 4x4 diagonal pieces and a partial last panel
      // element-wise
      fence_proxy_async();
      __syncthreads();
      for (int gg = tw; gg < gn; gg += 8) {
        const int w = t.width(gg), base = t.group_off(gg);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r0 = 8 * gg + 4 * h;
          if (r0 >= n) continue;
          const double *src = S + base + h * 4 * w;
          const bool full = r0 + 4 <= n;
          const int cl = full ? min(r0, n) : 0;
          if (cl > 0 && lane == 0) tma_store_1d(D + eo(g.di + r0, g.dj, g.D.cn), src, 32u * (unsigned)cl);
          const int ce = min(r0 + 4, n);
          for (int qq = lane; qq < 4 * (ce - cl); qq += 32) {
            const int c = cl + (qq >> 2), rr = r0 + (qq & 3);
            if (rr < n && c <= rr) D[eo(g.di + rr, g.dj + c, g.D.cn)] = src[4 * c + (qq & 3)];
          }
        }
      }
      if (lane == 0) bulk_commit();
    } else {
      const int iif = fail & ~3;
      for (int gg = 0; gg < gn; ++gg) {
        const int w = t.width(gg), base = t.group_off(gg);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int rp = 8 * gg + 4 * h;
          if (rp >= n || rp > iif) continue;
          for (int qq = tid; qq < 4 * w; qq += CHAIN_THREADS) {
            const int c = qq >> 2, rr = rp + (qq & 3);
            const bool st = rr < n && c < n && c <= rr && (rr < iif || (rr < iif + 4 && c < iif));
            if (st) D[eo(g.di + rr, g.dj + c, g.D.cn)] = S[base + h * 4 * w + qq];
          }
        }
      }
    }
    double *dA = g.D.ditem(b);
    const int nd_ = fail >= 0 ? fail : n;
    for (int c = tid; c < nd_; c += CHAIN_THREADS) dA[g.dj + c] = dinv[c];
    if (tid == 0 && g.info) g.info[b] = fail >= 0 ? fail + g.info_offset : -1;
    if (lane == 0) bulk_wait_read0();  // S is free once the stores have read it
    __syncthreads();
    b = nb;
    if (b < g.batch) load_item(b);
  }
  if (lane == 0) bulk_wait0();
}

}  // namespace

// square, panel-aligned, 16-byte aligned items in and out
bool potrf_chain_ok(const PotrfArgs &g) {
  return g.m == g.n && g.n > 64 && g.n <= 128 && !g.syrk && (g.ci & 3) == 0 && (g.di & 3) == 0 &&
         ((uintptr_t)g.C.p & 15) == 0 && (g.C.stride & 1) == 0 && ((uintptr_t)g.D.p & 15) == 0 &&
         (g.D.stride & 1) == 0;
}

cudaError_t run_potrf_chain(const PotrfArgs &g, cudaStream_t st) {
  const ix gn = (g.n + 7) / 8;
  const size_t smem = sizeof(double) * (32 * gn * (gn + 1) + 8 * gn + 128 + 128) + sizeof(uint64_t) + 16 * sizeof(int);
  static LaunchCache cache;
  const int occ = cache.occupancy((const void *)potrf_chain_kernel, CHAIN_THREADS, smem);
  ix grid = (ix)num_sms() * occ;
  if (grid > g.batch) grid = g.batch;
  if (grid < 1) grid = 1;
  potrf_chain_kernel<<<(unsigned)grid, CHAIN_THREADS, smem, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pb
