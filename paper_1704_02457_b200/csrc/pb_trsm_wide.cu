// Batched dtrsm_rltn  D * A^T = alpha * B  for triangles up to 128 columns,
// register-resident row strips (sm_100a).
//
// Reference semantics: trsm_rltn_drv ccore.pyx:855-874 (+ _trsm_rltn_core
// :358-388), reciprocal selection level3._recip_diag level3.py:160-177:
// dinv = 1/A[j,j] multiplied, not divided; a zero pivot (when reciprocals are
// computed) -> info, item untouched; D may alias B.
//
// Why this shape.  The team kernel keeps each warp's 8-row strip of X in
// shared memory and re-reads it as the A operand of every later column block
// (two loads per DMMA, a __syncwarp + store + reload per block): the blocked
// n = 256 factorization spent 0.94 of its 2.0 ms in its 128 x 128 solve
// (6.9 TF/s).  Here a warp keeps its whole strip in REGISTERS: an 8x8
// accumulator tile is an m8n8k4 A operand as it stands when k-step e of a
// pair contracts over columns 2q + e (lane (r, q) holds X[r][2q + e]), so
//    acc = alpha * B_j - sum_{k<j} X_k L_jk^T ;   X_j = acc * W_jj^T
// costs one shared-memory load (the L_jk fragment, read with the same
// permuted k mapping) per DMMA and nothing else; the negated X_k stay in
// registers for the later column blocks (in the slots that held the strip's
// alpha * B tiles, all requested before the triangle is even staged), X_j
// goes straight to D.  W_jj =
// L_jj^{-1} (all diagonal blocks, built once per item by the CTA's warps) is
// stored lane-linear so its fragment is one conflict-free load.  The strips
// of an item are independent: 8 warps x 2 CTAs per SM keep 16 accumulator
// chains in flight, enough to cover the 26-cycle dependent-DMMA latency.
#include "pb_tri.cuh"

namespace pb {

namespace {

constexpr int WT = 256;     // threads per CTA (8 warps, one 8-row strip each at a time)
constexpr int GNMAX = 16;   // column blocks (n <= 128)

__device__ __forceinline__ double dneg(double x) {
  return __hiloint2double(__double2hiint(x) ^ (int)0x80000000, __double2loint(x));
}

// bytes need not be a multiple of 16 here: round down, the tail comes with the first demand load
__device__ __forceinline__ void prefetch_l2_range(const void *p, int bytes) {
  const unsigned b16 = (unsigned)bytes & ~15u;
  if (b16 && ((uintptr_t)p & 15) == 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(b16) : "memory");
}

__global__ void __launch_bounds__(WT, 2) trsm_wide_kernel(TrsmArgs g) {
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, tw = warp_uniform();
  const int r = lane >> 2, q = lane & 3;
  const int m = (int)g.m, n = (int)g.n;
  Tri t;
  t.cn8 = (n + 7) / 8 * 8;
  t.gn = t.cn8 / 8;
  const int gn = t.gn, gmr = (m + 7) / 8;
  double *S = smem;
  double *dinv = S + 32 * gn * (gn + 1);  // cn8 reciprocals
  double *Wall = dinv + t.cn8;            // gn x 64: inverted diagonal blocks, lane-linear
  uint64_t *tbar = reinterpret_cast<uint64_t *>(Wall + 64 * gn);
  int *flag = reinterpret_cast<int *>(tbar + 1);
  if (tid == 0) {
    mbar_init(tbar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  unsigned tphase = 0;
  // B-operand base of row group j for this lane (k-step e contracts over columns 2q + e):
  // lane (q, nn = lane >> 2) reads L[8j + nn][8k + 2q + e] at lb_j + 32 k + 4 e
  const int hi = lane >> 4, lbl = 8 * q + (r & 3);
  for (ix b = (ix)blockIdx.x; b < g.batch; b += (ix)gridDim.x) {
    if (g.skip && g.skip[b] >= 0) continue;
    tri_load_bulk(S, t, g.A.item(b), g.A.cn, g.ai, g.aj, n, n, gn, tbar, tid, WT);
    // R: the strip's register file -- tile k holds alpha * B_k until column block k is solved, then -X_k (the A
    // operand of the later blocks).  The first strip's B tiles are requested now, before the triangle is staged
    // and its diagonal blocks inverted, so their HBM latency is hidden; later strips are pulled into L2.
    const double *Bb = g.B.item(b);
    double *Db = g.D.item(b);
    double R[GNMAX][2];
    auto load_strip = [&](int gg) {
      const int row = 8 * gg + r;
      const ix offB = eo(g.bi + row, g.bj + 2 * q, g.B.cn);
#pragma unroll
      for (int j = 0; j < GNMAX; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          R[j][e] = (j < gn && row < m && 8 * j + 2 * q + e < n) ? Bb[offB + 4 * (8 * j + e)] : 0.0;
    };
    if (tw < gmr) load_strip(tw);
    for (int gg = tw + WT / 32; gg < gmr; gg += WT / 32)
      if (lane < 2 && 8 * gg + 4 * lane < m)  // the strip's two 4-row panels: contiguous runs of 32 n bytes
        prefetch_l2_range(Bb + eo(g.bi + 8 * gg + 4 * lane, g.bj, g.B.cn), 32 * n);
    const bool reuse = g.use_dA == 1 || (g.use_dA == 2 && g.info[b] < 0);
    if (tid == 0) *flag = 0x7fffffff;
    mbar_wait(tbar, tphase);
    tphase ^= 1;
    __syncthreads();
    // reciprocals: reuse the factorization's, or compute (zero -> info, item untouched; level3.py:171-175)
    if (reuse) {
      const double *dA = g.A.ditem(b);
      for (int c = tid; c < n; c += WT) dinv[c] = dA[g.aj + c];
    } else {
      for (int c = tid; c < n; c += WT) {
        const double d = S[t.off(c, c)];
        dinv[c] = 1.0 / d;
        if (d == 0.0) atomicMin(flag, c);
      }
    }
    __syncthreads();
    const int fail = reuse || *flag == 0x7fffffff ? -1 : *flag;
    if (fail < 0) {
      // inverse of every 8x8 diagonal block, spread over the warps (register sweep, pb_tri.cuh); lane
      // (nn, q) holds W[nn][2q + e] -- exactly the B fragment of k-step e, so it is stored lane-linear
      for (int jb = tw; jb < gn; jb += WT / 32) {
        double x[2], wv[2];
        x[0] = S[t.off(8 * jb + r, 8 * jb + 2 * q)];
        x[1] = S[t.off(8 * jb + r, 8 * jb + 2 * q + 1)];
        inv_tile_regs(x, dinv + 8 * jb, min(8, n - 8 * jb), wv, lane);
        Wall[64 * jb + lane] = wv[0];
        Wall[64 * jb + 32 + lane] = wv[1];
      }
      __syncthreads();
      for (int gg = tw; gg < gmr; gg += WT / 32) {
        if (gg != tw) load_strip(gg);
        const int row = 8 * gg + r;
        const bool rok = row < m;
        const ix offD = eo(g.di + row, g.dj + 2 * q, g.D.cn);
#pragma unroll
        for (int j = 0; j < GNMAX; ++j) {
          if (j < gn) {
            double acc[2];
            acc[0] = __dmul_rn(g.alpha, R[j][0]);
            acc[1] = __dmul_rn(g.alpha, R[j][1]);
            const int lb = 32 * j * (j + 1) + hi * (32 * j + 32) + lbl;
#pragma unroll
            for (int k = 0; k < j; ++k) {
              dmma(acc, R[k][0], S[lb + 32 * k]);
              dmma(acc, R[k][1], S[lb + 32 * k + 4]);
            }
            double X[2] = {0.0, 0.0};
            dmma(X, acc[0], Wall[64 * j + lane]);
            dmma(X, acc[1], Wall[64 * j + 32 + lane]);
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (rok && 8 * j + 2 * q + e < n) Db[offD + 4 * (8 * j + e)] = X[e];
            R[j][0] = dneg(X[0]), R[j][1] = dneg(X[1]);
          }
        }
      }
    }
    if (tid == 0 && g.info) g.info[b] = fail;
    __syncthreads();  // S, dinv, Wall are reused by the next item
  }
}

}  // namespace

bool trsm_wide_ok(const TrsmArgs &g) {
  return g.n >= 64 && g.n <= 8 * GNMAX && g.m >= 64 && (g.ai & 3) == 0 && ((uintptr_t)g.A.p & 15) == 0 &&
         (g.A.stride & 1) == 0;
}

cudaError_t run_trsm_wide(const TrsmArgs &g, cudaStream_t st) {
  const ix gn = (g.n + 7) / 8;
  const size_t smem = sizeof(double) * (32 * gn * (gn + 1) + 8 * gn + 64 * gn) + sizeof(uint64_t) + 2 * sizeof(int);
  static LaunchCache cache;
  const int occ = cache.occupancy((const void *)trsm_wide_kernel, WT, smem);
  ix grid = (ix)num_sms() * occ;
  if (grid > g.batch) grid = g.batch;
  if (grid < 1) grid = 1;
  trsm_wide_kernel<<<(unsigned)grid, WT, smem, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pb
