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

// NX[s] = -C(g_s, c) + sum_{k-steps < nk} L(g_s, .) L(c, .)^T for slots F..E-1
// (nk is even).  A single slot runs two partial accumulators so that its
// dependent-DMMA latency (26 cycles) stays below the pipe's issue interval.
template <int F, int E>
__device__ __forceinline__ void lookahead_slots(double (&NX)[3][2], const double *S, int fb, const int (&fa)[3],
                                                const int (&ao)[3], int c, int nk) {
#pragma unroll
  for (int s = F; s < E; ++s) {
    NX[s][0] = dneg(S[ao[s] + 32 * c]);
    NX[s][1] = dneg(S[ao[s] + 32 * c + 4]);
  }
  if (E - F == 1) {
    double a1[2] = {0.0, 0.0};
#pragma unroll 2
    for (int kk = 0; kk < nk; kk += 2) {
      dmma(NX[F], S[fa[F] + 16 * kk], S[fb + 16 * kk]);
      dmma(a1, S[fa[F] + 16 * kk + 16], S[fb + 16 * kk + 16]);
    }
    NX[F][0] += a1[0], NX[F][1] += a1[1];
  } else {
#pragma unroll 4
    for (int kk = 0; kk < nk; ++kk) {
      const double bv = S[fb + 16 * kk];
#pragma unroll
      for (int s = F; s < E; ++s) dmma(NX[s], S[fa[s] + 16 * kk], bv);
    }
  }
}

// runtime slot range [f, e) -> the unrolled instance
__device__ __forceinline__ void lookahead_range(int f, int e, double (&NX)[3][2], const double *S, int fb,
                                                const int (&fa)[3], const int (&ao)[3], int c, int nk) {
  if (f == 0) {
    if (e == 3) lookahead_slots<0, 3>(NX, S, fb, fa, ao, c, nk);
    else if (e == 2) lookahead_slots<0, 2>(NX, S, fb, fa, ao, c, nk);
    else if (e == 1) lookahead_slots<0, 1>(NX, S, fb, fa, ao, c, nk);
  } else if (f == 1) {
    if (e == 3) lookahead_slots<1, 3>(NX, S, fb, fa, ao, c, nk);
    else if (e == 2) lookahead_slots<1, 2>(NX, S, fb, fa, ao, c, nk);
  } else if (f == 2 && e == 3) {
    lookahead_slots<2, 3>(NX, S, fb, fa, ao, c, nk);
  }
}

constexpr int CHAIN_THREADS = 256;
constexpr int STEP_THREADS = 7 * 32;  // chain warp + six bulk warps meet at the step barriers

template <int N>
__device__ __forceinline__ void bar_sync_n(int id) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bar_arrive_n(int id) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "n"(N) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Blocked driver: the rows below the previous panel (solved into the aligned workspace matrix cS) go to
// D once item b's fate is known: rows [0, rmax), rmax = c_rows for a healthy item, (f & ~3) + 4 for one
// failing at local pivot f (the reference's row-panel write set).  Whole 4-row panels are contiguous runs
// of 32 c_cols bytes on both sides.  Kept out of line: the kernel is at its register cap.
__device__ __noinline__ void commit_rows(const double *cs, double *cd, int scn, int dcn, int c_di, int c_dj, int c_cols,
                                        int rmax, int tid) {
  const int vpp = 2 * c_cols, nv = (rmax >> 2) * vpp;
  for (int v0 = tid; v0 < nv; v0 += 8 * CHAIN_THREADS) {
    double2 tmp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int v = v0 + u * CHAIN_THREADS;
      if (v < nv) {
        const int p = v / vpp, o = v - p * vpp;
        tmp[u] = reinterpret_cast<const double2 *>(cs + (ix)4 * p * scn)[o];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int v = v0 + u * CHAIN_THREADS;
      if (v < nv) {
        const int p = v / vpp, o = v - p * vpp;
        reinterpret_cast<double2 *>(cd + eo(c_di + 4 * p, c_dj, dcn))[o] = tmp[u];
      }
    }
  }
  const int rem = rmax & 3;  // a partial last panel, element-wise
  for (int e = tid; e < rem * c_cols; e += CHAIN_THREADS) {
    const int rr = (rmax & ~3) + e % rem, c = e / rem;
    cd[eo(c_di + rr, c_dj + c, dcn)] = cs[eo(rr, c, scn)];
  }
}

template <bool COMMIT>
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
  double *Xp = Wp + 128;                                    // 2 x 64: solved tile (j+1, j), lane-linear
  double *Yp = Xp + 128;                                    // 2 x 64: solved tile (j+2, j), lane-linear
  double *Mb = Yp + 128;                                    // 2 x 128: hand-off of row j+1's two chain tiles
  uint64_t *tbar = reinterpret_cast<uint64_t *>(Mb + 256);  // bulk-load barrier
  volatile int *flagv = reinterpret_cast<volatile int *>(tbar + 1);  // failing column per step (16) + item (1)

  // Roles by hardware scheduler.  The chain's ~20 dependent FP64 instructions
  // per column queue behind every DMMA issued on the same sub-partition (one
  // m8n8k4 holds its FP64 pipe for 16 cycles), so the chain warps of all CTAs
  // on an SM are put on sub-partition 0 and no bulk work runs there.  The
  // hardware rotates a CTA's warps over the sub-partitions per resident CTA
  // (tools/warp_slots.cu: slots 0-7, 9 10 11 8 13 ..., 18 19 16 17 ...), so the
  // roles come from %warpid, not from the warp index: the two warps whose
  // slot % 4 == 0 are the chain warp and an idle stager, the other six own
  // the row groups cyclically (bw, bw + 6, bw + 12).  (Performance only: any
  // assignment is correct.)
  int *role = reinterpret_cast<int *>(tbar + 1) + 20;
  {
    unsigned slot;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(slot));
    if (lane == 0) role[tw] = (int)(slot & 3);
  }
  __syncthreads();
  int chain_w = -1, stage_w = -1;
#pragma unroll
  for (int w = 0; w < 8; ++w)
    if (role[w] == 0) {
      if (chain_w < 0) chain_w = w;
      else if (stage_w < 0) stage_w = w;
    }
  if (chain_w < 0) chain_w = 0;
  if (stage_w < 0) stage_w = (chain_w + 4) & 7;
  const bool is_chain = tw == chain_w, is_bulk = tw != chain_w && tw != stage_w;
  const int bw = tw - (tw > chain_w) - (tw > stage_w);
  const int ro = (r >> 2) * 4, lo = 8 * q + (r & 3);  // accumulator-layout offsets inside a tile row
  int fa[3], ao[3], gs[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    gs[s] = bw + 6 * s;
    const int gc = min(max(gs[s], 0), gn - 1);
    fa[s] = tri_frag(t, gc, 0, lane);
    ao[s] = t.group_off(gc) + ro * t.width(gc) + lo;
  }
  const int ns = !is_bulk ? 0 : (gs[2] < gn ? 3 : (gs[1] < gn ? 2 : 1));

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
    if (tid < 17) flagv[tid] = -1;
    __syncthreads();
    if (is_chain) {
      // ---- the pivot chain: factor(jb) -> solve tile (jb+1, jb) -> diag(jb+1)
      double dg[2];
      dg[0] = S[ro * 8 + lo], dg[1] = S[ro * 8 + lo + 4];
      for (int jb = 0; jb < gn; ++jb) {
        const int par = (step + jb) & 1;
        const int ncol = min(8, n - 8 * jb);
        const int wofs = (jb & 1) * 64 + lane;
        double wi[2];
        const int f = factor_inv_tile_u(dg, wi, ncol, dinv + 8 * jb, lane);
        const int aod = t.group_off(jb) + ro * t.width(jb) + lo + 32 * jb;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 2 * q + e;
          if (c < ncol && (f < 0 || c < f)) S[aod + 4 * e] = dg[e];
        }
        if (f >= 0 && lane == 0) flagv[jb] = flagv[16] = 8 * jb + f;
        Wp[wofs] = wi[0];
        Wp[wofs + 32] = wi[1];
        __syncwarp();
        bar_arrive_n<STEP_THREADS>(1 + par);
        const bool last = jb + 1 == gn;
        double ps[2], nx[2];
        if (!last) {
          // row jb+1's tiles (jb+1, jb) and -(jb+1, jb+1), downdated over blocks < jb by their owner
          bar_sync_n<64>(5 + par);
          const int mo = (jb & 1) * 128 + lane;
          ps[0] = Mb[mo], ps[1] = Mb[mo + 32];
          nx[0] = Mb[mo + 64], nx[1] = Mb[mo + 96];
        }
        if (f >= 0 || last) break;
        double X[2] = {0.0, 0.0};
        dmma(X, ps[0], wi[0]);
        dmma(X, ps[1], wi[1]);
        const int aox = t.group_off(jb + 1) + ro * t.width(jb + 1) + lo + 32 * jb;
        S[aox] = X[0];
        S[aox + 4] = X[1];
        Xp[wofs] = X[0];
        Xp[wofs + 32] = X[1];
        __syncwarp();
        bar_arrive_n<STEP_THREADS>(3 + par);
        dmma(nx, X[0], X[0]);
        dmma(nx, X[1], X[1]);
        dg[0] = dneg(nx[0]), dg[1] = dneg(nx[1]);
      }
    } else if (is_bulk) {
      // next item's lower panel prefixes into L2 while this one is factored
      if (bw == 5 && nb < g.batch && 4 * lane < n)
        prefetch_l2(g.C.item(nb) + eo(g.ci + 4 * lane, g.cj, g.C.cn), 32u * (unsigned)min(4 * lane + 4, n));
      // Per row slot: P = tile (g, jb), complete; NA = negated partial sum of
      // (g, jb+1) and NB of (g, jb+2), both over the column blocks < jb.  Two
      // columns of look-ahead: what the chain needs next (row jb+2's tiles)
      // is two 2-DMMA increments away from the step barrier, and the long
      // downdate loop (column jb+3) has a whole step of slack.
      double P[3][2], NA[3][2], NB[3][2], X[3][2];
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        P[s][0] = S[ao[s]], P[s][1] = S[ao[s] + 4];
        NA[s][0] = dneg(S[ao[s] + 32]), NA[s][1] = dneg(S[ao[s] + 36]);
        NB[s][0] = dneg(S[ao[s] + 64]), NB[s][1] = dneg(S[ao[s] + 68]);
      }
      if (bw == 1 && gn > 1) {  // hand row 1's tiles to the chain
        Mb[lane] = P[0][0], Mb[lane + 32] = P[0][1];
        Mb[lane + 64] = NA[0][0], Mb[lane + 96] = NA[0][1];
        __syncwarp();
        bar_arrive_n<64>(5 + (step & 1));
      }
      for (int jb = 0; jb < gn; ++jb) {
        const int par = (step + jb) & 1;
        const int wofs = (jb & 1) * 64 + lane;
        bar_sync_n<STEP_THREADS>(1 + par);
        if (flagv[jb] >= 0 || jb + 1 == gn) break;
        const double wb0 = Wp[wofs], wb1 = Wp[wofs + 32];
        // ---- solve X = P * W^T for rows >= jb + 2 (the accumulator IS the A operand)
        const int c = jb + 2;
        const int f0 = gs[0] >= c ? 0 : (gs[1] >= c ? 1 : (gs[2] >= c ? 2 : 3));  // first active slot (rows ascend)
        const bool own = bw == c % 6 && c < gn;                                   // this warp owns row jb + 2 (slot f0)
#pragma unroll
        for (int s = 0; s < 3; ++s)
          if (s < ns && gs[s] >= c) {
            X[s][0] = X[s][1] = 0.0;
            dmma(X[s], P[s][0], wb0);
            dmma(X[s], P[s][1], wb1);
            S[ao[s] + 32 * jb] = X[s][0];
            S[ao[s] + 32 * jb + 4] = X[s][1];
          }
        if (own) {  // tile (jb+2, jb), lane-linear: everyone's B operand for column block jb + 2
          Yp[wofs] = f0 == 0 ? X[0][0] : (f0 == 1 ? X[1][0] : X[2][0]);
          Yp[wofs + 32] = f0 == 0 ? X[0][1] : (f0 == 1 ? X[1][1] : X[2][1]);
        }
        bar_sync_n<STEP_THREADS>(3 + par);
        if (c >= gn) continue;  // nothing below row jb + 1
        // ---- block jb into column blocks jb + 1 (complete: P) and jb + 2
        const double xb0 = Xp[wofs], xb1 = Xp[wofs + 32];
        const double yb0 = Yp[wofs], yb1 = Yp[wofs + 32];
#pragma unroll
        for (int s = 0; s < 3; ++s)
          if (s < ns && gs[s] >= c) {
            dmma(NA[s], X[s][0], xb0);
            dmma(NA[s], X[s][1], xb1);
            dmma(NB[s], X[s][0], yb0);
            dmma(NB[s], X[s][1], yb1);
            P[s][0] = dneg(NA[s][0]), P[s][1] = dneg(NA[s][1]);
            NA[s][0] = NB[s][0], NA[s][1] = NB[s][1];
          }
        // ---- hand row jb + 2's tiles (jb+2, jb+1) and -(jb+2, jb+2) to the chain
        if (own) {
          const int mo = ((jb + 1) & 1) * 128 + lane;
          Mb[mo] = f0 == 0 ? P[0][0] : (f0 == 1 ? P[1][0] : P[2][0]);
          Mb[mo + 32] = f0 == 0 ? P[0][1] : (f0 == 1 ? P[1][1] : P[2][1]);
          Mb[mo + 64] = f0 == 0 ? NA[0][0] : (f0 == 1 ? NA[1][0] : NA[2][0]);
          Mb[mo + 96] = f0 == 0 ? NA[0][1] : (f0 == 1 ? NA[1][1] : NA[2][1]);
          __syncwarp();
          bar_arrive_n<64>(5 + (par ^ 1));
        }
        // ---- long look-ahead: column block jb + 3 over the solved blocks 0..jb
        const int c3 = jb + 3;
        if (c3 < gn) {
          const int f3 = gs[0] >= c3 ? 0 : (gs[1] >= c3 ? 1 : (gs[2] >= c3 ? 2 : 3));
          if (f3 < ns) lookahead_range(f3, ns, NB, S, tri_frag(t, c3, 0, lane), fa, ao, c3, 2 * (jb + 1));
        }
      }
    }
    __syncthreads();
    const int fail = flagv[16];
    step += flagv[16] >= 0 ? (unsigned)(flagv[16] / 8 + 1) : (unsigned)gn;
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
    const ix bdone = b;
    b = nb;
    if (b < g.batch) load_item(b);
    if (COMMIT)  // overlaps the next item's staging
      commit_rows(g.cS.item(bdone), g.D.item(bdone), (int)g.cS.cn, (int)g.D.cn, (int)g.c_di, (int)g.c_dj, (int)g.c_cols,
                  fail < 0 ? (int)g.c_rows : min((int)g.c_rows, (fail & ~3) + 4), tid);
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
  const size_t smem = sizeof(double) * (32 * gn * (gn + 1) + 8 * gn + 128 + 128 + 128 + 256) + sizeof(uint64_t) + 28 * sizeof(int);
  // two instances: the fused commit costs the plain factorization registers (it is at its cap)
  static LaunchCache cache[2];
  const void *kern = g.commit ? (const void *)potrf_chain_kernel<true> : (const void *)potrf_chain_kernel<false>;
  const int occ = cache[g.commit ? 1 : 0].occupancy(kern, CHAIN_THREADS, smem);
  ix grid = (ix)num_sms() * occ;
  if (grid > g.batch) grid = g.batch;
  if (grid < 1) grid = 1;
  if (g.commit) potrf_chain_kernel<true><<<(unsigned)grid, CHAIN_THREADS, smem, st>>>(g);
  else potrf_chain_kernel<false><<<(unsigned)grid, CHAIN_THREADS, smem, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pb
