// Fused Config-5 chain: N stages of
//   W = BAt P^T ; lower(M) = W BAt^T + RQ ; F = chol(M) ; K = -F21 F11^{-T} ;
//   P = F22 F22^T
// for every problem, in ONE persistent kernel (SURVEY.md §8a row 19, §8f:
// composite consumers of the four hot-path routines are the natural
// persistent-kernel fusion targets).
//
// A team of TW warps owns one problem at a time; all of the problem's
// matrices stay in shared memory for all N stages (~47 KB for nx=32,
// nu=8), so HBM is touched only to load BAt, RQ, P_N and store P_0, K.
// Every stage is the same arithmetic as the five batched routines: DMMA
// m8n8k4 tiles for the products, the register 8x8 Cholesky + inverted
// diagonal blocks (pb_tri.cuh) for the factorization and the solve.
// Restrictions (else the per-stage batched path in chain.py is used):
// nx, nu multiples of 8, nu == 8 (one 8x8 Lambda block).
#include <cstdlib>

#include "pb_tri.cuh"

namespace pb {

struct ChainArgs {
  Mat BAt, RQ, P, K;  // BAt: ns x nx, RQ: ns x ns (lower used), P: nx x nx (in: P_N, out: P_0), K: nx x nu
  int32_t *info;      // -1 ok, else stage * 1000 + failing pivot
  ix batch;
  int stages;
};

template <int NXB, int TW>
struct ChainCfg {
  static constexpr int NUB = 1;
  static constexpr int NB = NXB + NUB;  // 8-row groups of ns
  static constexpr int NS = 8 * NB, NX = 8 * NXB, NU = 8 * NUB;
  static constexpr int TRI = 32 * NB * (NB + 1);  // Tri::size(ns, ns)
  static constexpr int OFF_BAT = 0;                // full panel layout ns x nx
  static constexpr int OFF_RQ = OFF_BAT + NS * NX;  // tri
  // P (full nx x nx), W (full ns x nx) and F (tri) are never live together once every step accumulates its
  // tiles in registers and stores them behind a team barrier: ONE buffer holds whichever is current.  31 KB
  // per problem instead of 47 (nx = 32): seven problems per SM, so Config 5's 1024 problems run in one wave.
  static constexpr int XSZ = NS * NX > TRI ? NS * NX : TRI;
  static constexpr int OFF_P = OFF_RQ + TRI;
  static constexpr int OFF_W = OFF_P;
  static constexpr int OFF_F = OFF_P;
  static constexpr int OFF_DINV = OFF_P + XSZ;      // ns
  static constexpr int OFF_WP = OFF_DINV + NS;      // NB inverted diagonal blocks
  static constexpr int OFF_FLAG = OFF_WP + 64 * NB;
  static constexpr int TEAM = (OFF_FLAG + 8 + 15) / 16 * 16;
};

// fragment offset of row group g, k-step kk in a full panel-major block
// with panel length cn
__device__ __forceinline__ int full_frag(int g, int kk, int cn, int lane) {
  return (2 * g + (lane >> 4)) * 4 * cn + 16 * kk + 4 * (lane & 3) + ((lane >> 2) & 3);
}
__device__ __forceinline__ int full_off(int r, int c, int cn) { return (r >> 2) * 4 * cn + 4 * c + (r & 3); }

template <int NXB, int TW>
__global__ void __launch_bounds__(128, (NXB == 4 && TW == 4) ? 7 : 1) chain_kernel(ChainArgs g) {
  using Cfg = ChainCfg<NXB, TW>;
  constexpr int NB = Cfg::NB, NS = Cfg::NS, NX = Cfg::NX;
  extern __shared__ __align__(128) double smem[];
  const int lane = threadIdx.x & 31, warp = warp_uniform();
  const int team = warp / TW, tw = warp % TW;
  const int teams_per_cta = (blockDim.x >> 5) / TW;
  const int tthreads = TW * 32, ttid = tw * 32 + lane;
  const int bar = 1 + team;
  const int fr = lane >> 2, fc = lane & 3;
  double *T = smem + (ix)team * Cfg::TEAM;
  // One team per CTA (launch_chain): the team barrier is the CTA barrier.  A runtime named-barrier id makes
  // ptxas reserve all 16 hardware barriers for the CTA, which alone caps the SM at 4 CTAs (ncu:
  // launch__occupancy_limit_barriers).
  auto team_sync = [&](int, int) { __syncthreads(); };
  double *sBAt = T + Cfg::OFF_BAT, *sRQ = T + Cfg::OFF_RQ, *sP = T + Cfg::OFF_P, *sW = T + Cfg::OFF_W;
  double *sF = T + Cfg::OFF_F, *dinv = T + Cfg::OFF_DINV, *Wp = T + Cfg::OFF_WP;
  volatile int *flag = (volatile int *)(T + Cfg::OFF_FLAG);
  Tri t;
  t.gn = NB;
  t.cn8 = NS;

  for (ix b = (ix)blockIdx.x * teams_per_cta + team; b < g.batch; b += (ix)gridDim.x * teams_per_cta) {
    // ---- load BAt, lower(RQ), P_N (16-byte cp.async, panel rows contiguous)
    {
      const double *gB = g.BAt.item(b);
      for (int q = ttid; q < NS * NX / 2; q += tthreads) {
        const int p = q / (2 * NX), w = q - p * 2 * NX;
        cp_async16(sBAt + p * 4 * NX + 2 * w, gB + p * 4 * g.BAt.cn + 2 * w, 16);
      }
      const double *gP = g.P.item(b);
      for (int q = ttid; q < NX * NX / 2; q += tthreads) {
        const int p = q / (2 * NX), w = q - p * 2 * NX;
        cp_async16(sP + p * 4 * NX + 2 * w, gP + p * 4 * g.P.cn + 2 * w, 16);
      }
      const double *gR = g.RQ.item(b);
      for (int gg = 0; gg < NB; ++gg) {
        const int w = t.width(gg), base = t.group_off(gg);
        for (int q = ttid; q < 4 * w; q += tthreads) {
          const int half = q / (2 * w), rem = q - half * 2 * w;
          const int c = rem >> 1, h2 = rem & 1;
          cp_async16(sRQ + base + half * 4 * w + 4 * c + 2 * h2, gR + (2 * gg + half) * 4 * g.RQ.cn + 4 * c + 2 * h2,
                     16);
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
      if (ttid == 0) *flag = -1;
      team_sync(bar, tthreads);
    }
    int info = -1;
    for (int stage = 0; stage < g.stages; ++stage) {
      // (1) W = BAt * P^T   (NB x NXB tiles, k = nx); a warp's tiles are
      // unrolled so their DMMA chains interleave
      {
        constexpr int NT1 = (NB * NXB + TW - 1) / TW;
        double acc[NT1][2];
#pragma unroll
        for (int q = 0; q < NT1; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < NX / 4; ++kk) {
#pragma unroll
          for (int q = 0; q < NT1; ++q) {
            const int tile = tw + q * TW;
            if (tile < NB * NXB) {
              const int i = tile / NXB, j = tile % NXB;
              dmma(acc[q], sBAt[full_frag(i, kk, NX, lane)], sP[full_frag(j, kk, NX, lane)]);
            }
          }
        }
        team_sync(bar, tthreads);  // W replaces P in the shared buffer: every warp is done reading P
#pragma unroll
        for (int q = 0; q < NT1; ++q) {
          const int tile = tw + q * TW;
          if (tile < NB * NXB) {
            const int i = tile / NXB, j = tile % NXB;
#pragma unroll
            for (int e = 0; e < 2; ++e) sW[full_off(8 * i + fr, 8 * j + 2 * fc + e, NX)] = acc[q][e];
          }
        }
      }
      team_sync(bar, tthreads);
      // (2) lower(M) = W * BAt^T + RQ   (lower tiles, k = nx) into F (tri)
      {
        constexpr int NL = NB * (NB + 1) / 2, NT2 = (NL + TW - 1) / TW;
        double acc[NT2][2];
        int ti[NT2], tj[NT2];
#pragma unroll
        for (int q = 0; q < NT2; ++q) {
          const int tile = tw + q * TW;
          int i = 0;
          while ((i + 1) * (i + 2) / 2 <= tile) ++i;
          ti[q] = i;
          tj[q] = tile - i * (i + 1) / 2;
          if (tile < NL) {
#pragma unroll
            for (int e = 0; e < 2; ++e) acc[q][e] = sRQ[t.off(8 * ti[q] + fr, 8 * tj[q] + 2 * fc + e)];
          }
        }
#pragma unroll
        for (int kk = 0; kk < NX / 4; ++kk) {
#pragma unroll
          for (int q = 0; q < NT2; ++q)
            if (tw + q * TW < NL) dmma(acc[q], sW[full_frag(ti[q], kk, NX, lane)], sBAt[full_frag(tj[q], kk, NX, lane)]);
        }
        team_sync(bar, tthreads);  // F replaces W in the shared buffer
#pragma unroll
        for (int q = 0; q < NT2; ++q)
          if (tw + q * TW < NL) {
#pragma unroll
            for (int e = 0; e < 2; ++e) sF[t.off(8 * ti[q] + fr, 8 * tj[q] + 2 * fc + e)] = acc[q][e];
          }
      }
      team_sync(bar, tthreads);
      // (3) F = chol(M), left-looking over 8-column blocks (as potrf_team_kernel)
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        constexpr int MAXT = (NB + TW - 1) / TW;
        double acc[MAXT][2];
#pragma unroll
        for (int u = 0; u < MAXT; ++u) {
          const int gg = jb + tw + u * TW;
          if (gg < NB) {
            acc[u][0] = sF[t.off(8 * gg + fr, 8 * jb + 2 * fc)];
            acc[u][1] = sF[t.off(8 * gg + fr, 8 * jb + 2 * fc + 1)];
            const int fa = tri_frag(t, gg, 0, lane), fb = tri_frag(t, jb, 0, lane);
#pragma unroll
            for (int kk = 0; kk < 2 * jb; ++kk) dmma(acc[u], -sF[fa + 16 * kk], sF[fb + 16 * kk]);
          }
        }
        if (tw == 0) {
          // factor and inverse of the diagonal tile in ONE unscaled column sweep (pb_tri.cuh), instead of
          // a factor sweep followed by a substitution sweep on the stored tile
          double wi[2];
          const int f = factor_inv_tile_u(acc[0], wi, 8, dinv + 8 * jb, lane);
#pragma unroll
          for (int e = 0; e < 2; ++e) sF[t.off(8 * jb + fr, 8 * jb + 2 * fc + e)] = acc[0][e];
          if (f >= 0 && lane == 0 && *flag < 0) *flag = stage * 1000 + 8 * jb + f;
          store_inv_block(wi, Wp + 64 * jb, lane);
        }
#pragma unroll
        for (int u = 0; u < MAXT; ++u) {
          const int gg = jb + tw + u * TW;
          if (gg < NB && gg > jb) {
#pragma unroll
            for (int e = 0; e < 2; ++e) sF[t.off(8 * gg + fr, 8 * jb + 2 * fc + e)] = acc[u][e];
          }
        }
        team_sync(bar, tthreads);
#pragma unroll
        for (int u = 0; u < MAXT; ++u) {
          const int gg = jb + tw + u * TW;
          if (gg < NB && gg > jb) {
            apply_inv_block(acc[u], sF, t, gg, jb, Wp + 64 * jb, lane);
            __syncwarp();
#pragma unroll
            for (int e = 0; e < 2; ++e) sF[t.off(8 * gg + fr, 8 * jb + 2 * fc + e)] = acc[u][e];
          }
        }
        team_sync(bar, tthreads);
      }
      // (4) K = -L * Lambda^{-T} (only the last stage's K is returned)
      if (stage == g.stages - 1) {
        double *gK = g.K.item(b);
        for (int i = tw; i < NXB; i += TW) {
          double acc[2];
          apply_inv_block(acc, sF, t, 1 + i, 0, Wp, lane);
#pragma unroll
          for (int e = 0; e < 2; ++e) gK[eo(8 * i + fr, 2 * fc + e, g.K.cn)] = -acc[e];
        }
      }
      // (5) P = Lcal * Lcal^T, Lcal = F[nu:, nu:] (strict upper of its diagonal tiles masked); the warp's tiles
      // stay in registers until every warp is done reading F, then P replaces it in the shared buffer
      {
        constexpr int NT5 = (NXB * NXB + TW - 1) / TW;
        double acc[NT5][2];
#pragma unroll
        for (int q = 0; q < NT5; ++q) {
          const int tile = tw + q * TW;
          acc[q][0] = acc[q][1] = 0.0;
          if (tile < NXB * NXB) {
            const int i = tile / NXB, j = tile % NXB;
            const int kbmax = i < j ? i : j;
            for (int kb = 0; kb <= kbmax; ++kb) {
              const int fa = tri_frag(t, 1 + i, 0, lane) + 32 * (1 + kb), fb = tri_frag(t, 1 + j, 0, lane) + 32 * (1 + kb);
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) {
                const int col = 4 * kk + fc;
                double a = sF[fa + 16 * kk], bv = sF[fb + 16 * kk];
                if (kb == i && col > fr) a = 0.0;
                if (kb == j && col > fr) bv = 0.0;
                dmma(acc[q], a, bv);
              }
            }
          }
        }
        team_sync(bar, tthreads);
#pragma unroll
        for (int q = 0; q < NT5; ++q) {
          const int tile = tw + q * TW;
          if (tile < NXB * NXB) {
            const int i = tile / NXB, j = tile % NXB;
#pragma unroll
            for (int e = 0; e < 2; ++e) sP[full_off(8 * i + fr, 8 * j + 2 * fc + e, NX)] = acc[q][e];
          }
        }
      }
      team_sync(bar, tthreads);
    }
    // ---- store P_0
    {
      double *gP = g.P.item(b);
      for (int q = ttid; q < NX * NX / 2; q += tthreads) {
        const int p = q / (2 * NX), w = q - p * 2 * NX;
        *reinterpret_cast<double2 *>(gP + p * 4 * g.P.cn + 2 * w) = *reinterpret_cast<const double2 *>(sP + p * 4 * NX + 2 * w);
      }
      info = *flag;
      if (ttid == 0 && g.info) g.info[b] = info;
      team_sync(bar, tthreads);
    }
  }
}

template <int NXB, int TW>
static cudaError_t launch_chain(const ChainArgs &g, cudaStream_t st) {
  using Cfg = ChainCfg<NXB, TW>;
  auto kern = chain_kernel<NXB, TW>;
  const int teams = 1, threads = 32 * TW;  // a CTA is one team (see the barrier note in the kernel)
  const size_t smem = sizeof(double) * Cfg::TEAM * teams;
  static LaunchCache cache;
  static bool carve = false;
  if (!carve) {  // seven 31 KB problems per SM need the largest shared-memory carve-out
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    carve = true;
  }
  const int occ = cache.occupancy((const void *)kern, threads, smem);
  ix grid = (g.batch + teams - 1) / teams;
  const ix cap = (ix)num_sms() * occ;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, threads, smem, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

cudaError_t run_chain_riccati(const ChainArgs &g, int nx, int nu, cudaStream_t st) {
  if (nu != 8) return cudaErrorInvalidValue;
  switch (nx) {
    case 8: return launch_chain<1, 2>(g, st);
    case 16: return launch_chain<2, 2>(g, st);
    case 24: return launch_chain<3, 2>(g, st);
    case 32: return launch_chain<4, 4>(g, st);  // 4 warps per problem measured best (1.405 -> 1.321 ms at C5)
    case 48: return launch_chain<6, 4>(g, st);
    case 64: return launch_chain<8, 4>(g, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pb

using namespace pb;

extern "C" int pb_driccati_chain(int nx, int nu, int stages, const pb_dmat_batch *sBAt, const pb_dmat_batch *sRQ,
                                 const pb_dmat_batch *sP, const pb_dmat_batch *sK, int32_t *info, void *stream) {
  // positions: nx1 nu2 stages3 BAt4 RQ5 P6 K7 info8
  if (nx <= 0 || nx % 8 || nx > 64) return -1;
  if (nu != 8) return -2;
  if (stages < 0) return -3;
  const int ns = nx + nu;
  const pb_dmat_batch *ds[4] = {sBAt, sRQ, sP, sK};
  const int rows[4] = {ns, ns, nx, nx}, cols[4] = {nx, ns, nx, nu};
  for (int i = 0; i < 4; ++i) {
    const pb_dmat_batch *d = ds[i];
    if (!d || d->m != rows[i] || d->n != cols[i] || d->cn != ((cols[i] + 3) & ~3) || !d->pA) return -(4 + i);
    if (d->batch != sP->batch || (d->stride != 0 && d->stride < 1) || ((uintptr_t)d->pA & 15) || (d->stride & 1))
      return -(4 + i);
  }
  if (sP->batch == 0 || stages == 0) return 0;
  ChainArgs g;
  g.BAt = {sBAt->pA, sBAt->stride, sBAt->cn, nullptr, 0};
  g.RQ = {sRQ->pA, sRQ->stride, sRQ->cn, nullptr, 0};
  g.P = {sP->pA, sP->stride, sP->cn, nullptr, 0};
  g.K = {sK->pA, sK->stride, sK->cn, nullptr, 0};
  g.info = info;
  g.batch = sP->batch;
  g.stages = stages;
  const cudaError_t e = run_chain_riccati(g, nx, nu, (cudaStream_t)stream);
  return e == cudaSuccess ? 0 : PB_ERR_CUDA;
}
