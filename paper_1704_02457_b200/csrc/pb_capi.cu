// extern "C" entry points of libpb_b200.so (declared in include/pb_b200.h).
//
// Validation mirrors the reference's L3 checks (level3.py:47-53,
// pack.py:36-42): negative sizes and windows leaving the matrix are
// rejected before anything is launched (return -argument_position); the
// Python layer turns those into DimensionError with the reference's text.
// Sizes that do not fit one CTA's shared memory are handled by a blocked
// driver built from the same kernels (potrf: tall panel factor + syrk
// downdate + recursive trailing factor; trsm: column-block solve + gemm
// downdate), so every size the reference accepts runs on the GPU.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "pb_gemm.cuh"

namespace pb {

static thread_local std::string t_err;
static thread_local int64_t t_launches = 0;
void note_launch() { ++t_launches; }

static int fail_arg(int pos, const char *what) {
  char buf[256];
  snprintf(buf, sizeof buf, "argument %d: %s", pos, what);
  t_err = buf;
  return -pos;
}

static int cuda_fail(cudaError_t e) {
  t_err = std::string("CUDA: ") + cudaGetErrorString(e);
  return PB_ERR_CUDA;
}

static Mat to_mat(const pb_dmat_batch *x) {
  Mat r;
  r.p = x->pA;
  r.stride = x->stride;
  r.cn = x->cn;
  r.d = x->dA;
  r.dstride = x->dA_stride;
  return r;
}

// Check one operand: descriptor sanity and window (i0, j0, rows, cols).
static int check_mat(const pb_dmat_batch *x, int pos_mat, int i0, int j0, int64_t rows, int64_t cols, int batch,
                     bool is_output) {
  if (!x) return fail_arg(pos_mat, "null matrix descriptor");
  if (x->m < 0 || x->n < 0) return fail_arg(pos_mat, "negative matrix size");
  if (x->cn < ((x->n + 3) & ~3) || (x->cn & 3)) return fail_arg(pos_mat, "panel length must be round_up(n,4)");
  if (i0 < 0 || j0 < 0) return fail_arg(pos_mat + 1, "negative sub-matrix origin");
  if (i0 + rows > x->m || j0 + cols > x->n) return fail_arg(pos_mat, "window exceeds matrix");
  if (rows > 0 && cols > 0 && !x->pA) return fail_arg(pos_mat, "null data pointer");
  if (is_output) {
    if (x->stride <= 0 && batch > 1) return fail_arg(pos_mat, "output needs a positive item stride");
  } else if (x->stride != 0 && x->batch != batch) {
    return fail_arg(pos_mat, "batch size differs from the output's");
  }
  if (x->stride < 0) return fail_arg(pos_mat, "negative item stride");
  return 0;
}

static bool vec16_ok(const pb_dmat_batch *x, int i0) {
  return (i0 & 3) == 0 && ((uintptr_t)x->pA & 15) == 0 && (x->stride & 1) == 0;
}
static bool tma_ok(const pb_dmat_batch *x) { return ((uintptr_t)x->pA & 15) == 0 && (x->stride & 1) == 0; }

static int finish(cudaError_t e) { return e == cudaSuccess ? 0 : cuda_fail(e); }

static int work_fail() {
  t_err = "workspace smaller than the worksize query reported";
  return PB_ERR_WORKSPACE;
}

static size_t ws_round(size_t b) { return (b + 255) & ~(size_t)255; }
static size_t panel_bytes(int64_t rows, int64_t cols) {
  return ws_round(sizeof(double) * (size_t)((rows + 3) & ~3) * (size_t)((cols + 3) & ~3));
}

// caller-owned workspace, carved by a bump pointer in call order
struct Work {
  char *base = nullptr;
  size_t cap = 0, used = 0;
  double *take(size_t bytes) {
    const size_t a = ws_round(used);
    if (a + bytes > cap) return nullptr;
    used = a + bytes;
    return (double *)(base + a);
  }
};

static pb_dmat_batch panel_desc(double *p, int rows, int cols, int batch, double *dA = nullptr,
                                int64_t dA_stride = 0) {
  pb_dmat_batch w;
  memset(&w, 0, sizeof w);
  w.pA = p, w.dA = dA, w.m = rows, w.n = cols, w.cn = (cols + 3) & ~3, w.batch = batch;
  w.stride = (int64_t)((rows + 3) & ~3) * w.cn, w.dA_stride = dA_stride;
  return w;
}

}  // namespace pb

using namespace pb;

extern "C" {

int pb_version(void) { return 2; }
const char *pb_last_error(void) { return t_err.c_str(); }
// diag_inv of an output holds min(m, n) reciprocals of its matrix; a factor
// of width w written at column dj needs dj + w of them.  The reference core
// would write past the end of the diag_inv view (no bounds check,
// ccore.pyx:1); here it is an argument error.
static int check_dinv(const pb_dmat_batch *d, int pos, int dj, int w) {
  const int cap = d->m < d->n ? d->m : d->n;
  if (dj + w > cap) return fail_arg(pos, "diag_inv too short: dj + n exceeds min(rows, cols) of D");
  return 0;
}

int pb_dgetrf(int m, int n, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di, int dj,
              int pivot, int64_t *ipiv, int64_t ipiv_stride, int32_t *info, void *stream) {
  // positions: m1 n2 C3 ci4 cj5 D6 di7 dj8 pivot9 ipiv10 ipiv_stride11 info12 (level3.py:405-446)
  if (m < 0) return fail_arg(1, "negative size");
  if (n < 0) return fail_arg(2, "negative size");
  if (!sD) return fail_arg(6, "null matrix descriptor");
  const int batch = sD->batch;
  int r;
  if ((r = check_mat(sC, 3, ci, cj, m, n, batch, false))) return r;
  if ((r = check_mat(sD, 6, di, dj, m, n, batch, true))) return r;
  const int mn = m < n ? m : n;
  if (mn == 0 || batch == 0) return 0;  // level3.py:435-436
  if (!sD->dA) return fail_arg(6, "output needs diag_inv storage");
  if ((r = check_dinv(sD, 6, dj, mn))) return r;
  if (pivot && !ipiv) return fail_arg(10, "ipiv is required with pivoting");
  if (pivot && ipiv_stride < mn) return fail_arg(11, "ipiv stride below min(m, n)");
  if (!info) return fail_arg(12, "info is required");
  if (getrf_smem(m, n) > 220 * 1024) return fail_arg(1, "window too large for the shared-memory LU (m*n*8 > 220 KB)");
  return finish(run_getrf(m, n, pivot ? 1 : 0, to_mat(sC), ci, cj, to_mat(sD), di, dj, ipiv, ipiv_stride, info, batch,
                          (cudaStream_t)stream));
}

int64_t pb_launch_count(int reset) {
  const int64_t v = t_launches;
  if (reset) t_launches = 0;
  return v;
}

static int gemm_common(int op, int m, int n, int k, double alpha, const pb_dmat_batch *sA, int ai, int aj,
                       const pb_dmat_batch *sB, int bi, int bj, double beta, const pb_dmat_batch *sC, int ci,
                       int cj, const pb_dmat_batch *sD, int di, int dj, void *stream, const int32_t *skip) {
  // positions: gemm (m1 n2 k3 alpha4 A5 ai6 aj7 B8 bi9 bj10 beta11 C12 ci13 cj14 D15 di16 dj17)
  //            syrk (m1 k2 alpha3 A4 ai5 aj6 B7 bi8 bj9 beta10 C11 ci12 cj13 D14 di15 dj16)
  //            gemm_nn (as gemm_nt, B is k x n)
  const bool syrk = op == 1, nn_b = op == 2;
  const int o = syrk ? -1 : 0;
  if (m < 0) return fail_arg(1, "negative size");
  if (!syrk && n < 0) return fail_arg(2, "negative size");
  if (k < 0) return fail_arg(3 + o, "negative size");
  if (!sD) return fail_arg(15 + o, "null matrix descriptor");
  const int batch = sD->batch;
  if (batch < 0) return fail_arg(15 + o, "negative batch");
  const int64_t nn = syrk ? m : n;
  int r;
  if ((r = check_mat(sA, 5 + o, ai, aj, m, k, batch, false))) return r;
  if ((r = check_mat(sB, 8 + o, bi, bj, nn_b ? k : nn, nn_b ? nn : k, batch, false))) return r;
  if ((r = check_mat(sC, 12 + o, ci, cj, m, nn, batch, false))) return r;
  if ((r = check_mat(sD, 15 + o, di, dj, m, nn, batch, true))) return r;
  if (m == 0 || nn == 0 || batch == 0) return 0;  // level3.py:91-92, 130-131
  GemmArgs g;
  g.m = m;
  g.n = nn;
  g.k = k;
  g.alpha = alpha;
  g.beta = beta;
  g.A = to_mat(sA);
  g.B = to_mat(sB);
  g.C = to_mat(sC);
  g.D = to_mat(sD);
  g.ai = ai, g.aj = aj, g.bi = bi, g.bj = bj, g.ci = ci, g.cj = cj, g.di = di, g.dj = dj;
  g.batch = batch;
  g.vecA = vec16_ok(sA, ai);
  g.vecB = vec16_ok(sB, bi);
  g.tma = tma_ok(sA) && tma_ok(sB);
  g.tmaC = tma_ok(sC);
  g.skip = skip;
  cudaStream_t st = (cudaStream_t)stream;
  return finish(syrk ? run_syrk_ln(g, st) : nn_b ? run_gemm_nn(g, st) : run_gemm_nt(g, st));
}

int pb_dgemm_nt(int m, int n, int k, double alpha, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB,
                int bi, int bj, double beta, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di,
                int dj, void *stream) {
  return gemm_common(0, m, n, k, alpha, sA, ai, aj, sB, bi, bj, beta, sC, ci, cj, sD, di, dj, stream, nullptr);
}

int pb_dgemm_nn(int m, int n, int k, double alpha, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB,
                int bi, int bj, double beta, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di,
                int dj, void *stream) {
  return gemm_common(2, m, n, k, alpha, sA, ai, aj, sB, bi, bj, beta, sC, ci, cj, sD, di, dj, stream, nullptr);
}

static int trmm_check(int m, int n, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB, int bi, int bj,
                      const pb_dmat_batch *sD, int di, int dj) {
  // positions: m1 n2 alpha3 A4 ai5 aj6 B7 bi8 bj9 D10 di11 dj12 (level3.py:140-153)
  if (m < 0) return fail_arg(1, "negative size");
  if (n < 0) return fail_arg(2, "negative size");
  if (!sD) return fail_arg(10, "null matrix descriptor");
  const int batch = sD->batch;
  int r;
  if ((r = check_mat(sA, 4, ai, aj, n, n, batch, false))) return r;
  if ((r = check_mat(sB, 7, bi, bj, m, n, batch, false))) return r;
  return check_mat(sD, 10, di, dj, m, n, batch, true);
}

// In place (D on B's storage, test_level3.py:190-195): tiles of D would
// overwrite columns of B other column tiles still read once n spans several
// tiles, so B's window is first copied to workspace (one warp-tile spans all
// n <= 24 columns: no copy needed).
static size_t trmm_ws(int m, int n, const pb_dmat_batch *sB, const pb_dmat_batch *sD) {
  return (sD->pA == sB->pA && n > 24) ? panel_bytes(m, n) * sD->batch : 0;
}

int64_t pb_dtrmm_rlnn_worksize(int m, int n, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB, int bi,
                               int bj, const pb_dmat_batch *sD, int di, int dj) {
  const int r = trmm_check(m, n, sA, ai, aj, sB, bi, bj, sD, di, dj);
  if (r) return r;
  if (m == 0 || n == 0 || sD->batch == 0) return 0;
  return (int64_t)trmm_ws(m, n, sB, sD);
}

int pb_dtrmm_rlnn(int m, int n, double alpha, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB, int bi,
                  int bj, const pb_dmat_batch *sD, int di, int dj, void *work, int64_t work_bytes, void *stream) {
  // positions: m1 n2 alpha3 A4 ai5 aj6 B7 bi8 bj9 D10 di11 dj12 work13 work_bytes14
  int r;
  if ((r = trmm_check(m, n, sA, ai, aj, sB, bi, bj, sD, di, dj))) return r;
  const int batch = sD->batch;
  if (m == 0 || n == 0 || batch == 0) return 0;  // level3.py:148-149
  const size_t need = trmm_ws(m, n, sB, sD);
  if (need && (!work || work_bytes < (int64_t)need)) return fail_arg(13, "workspace too small (see pb_dtrmm_rlnn_worksize)");
  // D = alpha * X * T as an NN product: the streamed operand X (= B) is the
  // kernel's A, the triangular factor T (= A) its B
  cudaStream_t st = (cudaStream_t)stream;
  pb_dmat_batch w;
  const pb_dmat_batch *sX = sB;
  int xi = bi, xj = bj;
  if (need) {
    w = panel_desc((double *)work, m, n, batch);
    CopyArgs c;
    memset(&c, 0, sizeof c);
    c.m = m, c.n = n;
    c.S = to_mat(sB), c.D = to_mat(&w);
    c.si = bi, c.sj = bj;
    c.batch = batch;
    if ((r = finish(run_gecp(c, st)))) return r;
    sX = &w, xi = 0, xj = 0;
  }
  GemmArgs g;
  g.m = m, g.n = n, g.k = n;
  g.alpha = alpha, g.beta = 0.0;
  g.A = to_mat(sX), g.B = to_mat(sA), g.C = to_mat(sD), g.D = to_mat(sD);
  g.ai = xi, g.aj = xj, g.bi = ai, g.bj = aj, g.ci = di, g.cj = dj, g.di = di, g.dj = dj;
  g.batch = batch;
  g.vecA = vec16_ok(sX, xi);
  g.vecB = vec16_ok(sA, ai);
  g.tma = tma_ok(sA) && tma_ok(sX);
  g.tmaC = false;
  g.skip = nullptr;
  return finish(run_trmm_rlnn(g, st));
}

int pb_dsyrk_ln(int m, int k, double alpha, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB, int bi,
                int bj, double beta, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di, int dj,
                void *stream) {
  return gemm_common(1, m, 0, k, alpha, sA, ai, aj, sB, bi, bj, beta, sC, ci, cj, sD, di, dj, stream, nullptr);
}

// ---- trsm_rltn ----------------------------------------------------------

static int trsm_run(int m, int n, double alpha, const pb_dmat_batch *sA, int ai, int aj, int use_dA,
                    const pb_dmat_batch *sB, int bi, int bj, const pb_dmat_batch *sD, int di, int dj, int32_t *info,
                    const int32_t *skip, cudaStream_t st) {
  if (trsm_fits(m, n)) {
    TrsmArgs g;
    g.m = m, g.n = n, g.alpha = alpha;
    g.A = to_mat(sA), g.B = to_mat(sB), g.D = to_mat(sD);
    g.ai = ai, g.aj = aj, g.bi = bi, g.bj = bj, g.di = di, g.dj = dj;
    g.use_dA = use_dA;
    g.info = info;
    g.batch = sD->batch;
    g.skip = skip;
    return finish(run_trsm_rltn(g, st));
  }
  // blocked: D1 = solve(B1, A11); D2 = alpha*B2 - D1*A21^T; D2 = solve(D2, A22)
  int n1 = 8;
  while (n1 + 8 < n && trsm_fits(m, n1 + 8)) n1 += 8;
  int r;
  if ((r = trsm_run(m, n1, alpha, sA, ai, aj, use_dA, sB, bi, bj, sD, di, dj, nullptr, skip, st))) return r;
  GemmArgs g;
  g.m = m, g.n = n - n1, g.k = n1, g.alpha = -1.0, g.beta = alpha;
  g.A = to_mat(sD), g.B = to_mat(sA), g.C = to_mat(sB), g.D = to_mat(sD);
  g.ai = di, g.aj = dj, g.bi = ai + n1, g.bj = aj, g.ci = bi, g.cj = bj + n1, g.di = di, g.dj = dj + n1;
  g.batch = sD->batch;
  g.vecA = vec16_ok(sD, di);
  g.vecB = vec16_ok(sA, ai + n1);
  g.tma = tma_ok(sD) && tma_ok(sA);
  g.tmaC = tma_ok(sB);
  g.skip = skip;
  if ((r = finish(run_gemm_nt(g, st)))) return r;
  return trsm_run(m, n - n1, 1.0, sA, ai + n1, aj + n1, use_dA, sD, di, dj + n1, sD, di, dj + n1, nullptr, skip, st);
}

int pb_dtrsm_rltn(int m, int n, double alpha, const pb_dmat_batch *sA, int ai, int aj, int use_dA,
                  const pb_dmat_batch *sB, int bi, int bj, const pb_dmat_batch *sD, int di, int dj, int32_t *info,
                  void *stream) {
  // positions: m1 n2 alpha3 A4 ai5 aj6 use_dA7 B8 bi9 bj10 D11 di12 dj13 info14
  if (m < 0) return fail_arg(1, "negative size");
  if (n < 0) return fail_arg(2, "negative size");
  if (!sD) return fail_arg(11, "null matrix descriptor");
  const int batch = sD->batch;
  int r;
  if ((r = check_mat(sA, 4, ai, aj, n, n, batch, false))) return r;
  if ((r = check_mat(sB, 8, bi, bj, m, n, batch, false))) return r;
  if ((r = check_mat(sD, 11, di, dj, m, n, batch, true))) return r;
  if (use_dA < 0 || use_dA > 2) return fail_arg(7, "use_dA must be 0, 1 or 2");
  if (use_dA && n > 0 && !sA->dA) return fail_arg(4, "use_dA set but the factor has no diag_inv");
  if (use_dA != 1 && !info) return fail_arg(14, "info is required when reciprocals may be computed");
  if (m == 0 || n == 0 || batch == 0) return 0;  // level3.py:200-201
  cudaStream_t st = (cudaStream_t)stream;
  if (trsm_fits(m, n)) return trsm_run(m, n, alpha, sA, ai, aj, use_dA, sB, bi, bj, sD, di, dj, info, nullptr, st);
  // blocked windows decide once for the whole batch: use_dA == 2 computes
  // every item's reciprocals (equal to the factorization's up to rounding)
  if (use_dA == 2) use_dA = 0;
  // blocked path: the zero-pivot check covers the whole diagonal first, so a
  // singular item is left completely untouched (level3.py:171-177)
  if (info) {
    if (!use_dA) {
      if ((r = finish(run_diag_check(to_mat(sA), ai, aj, n, batch, info, st)))) return r;
    } else if ((r = finish(cudaMemsetAsync(info, 0xff, sizeof(int32_t) * batch, st)))) {
      return r;
    }
  }
  return trsm_run(m, n, alpha, sA, ai, aj, use_dA, sB, bi, bj, sD, di, dj, nullptr, info, st);
}

// ---- potrf_l ------------------------------------------------------------
//
// Direct kernels: square n <= 16 (register / quad, bit-exact), 17..64 (one
// warp per item), 65..128 (one CTA per item, register tiles), tall windows
// that fit one team's shared memory (team kernel).  Everything else runs the
// blocked driver below, on caller-owned workspace (the library never
// allocates):
//   1. square factor of the first n1 <= 128 columns into D (direct kernel);
//   2. rows [n1, m):  W = C21 L11^{-T}   (trsm, reciprocals reused) -> workspace;
//   3. trailing:      T = C22 - W W^T     (syrk, lower trapezoid)   -> workspace;
//      potrf of T into D22 (recursive, failing items skipped, global index);
//   4. commit W -> D21: all rows of a healthy item; for an item failing at
//      pivot f >= n1 the rows above f's row panel and the panel itself
//      (rows < (f & ~3) + 4), which is exactly what the reference's row-panel
//      order (ccore.pyx:877-905) has written when it stops; nothing for f < n1.
// An unaligned D window (di % 4 != 0) factors into an aligned workspace copy
// and commits the lower trapezoid of healthy items only: level3.potrf_l
// factors into scratch and copies on success (level3.py:338-344), while the
// core writes diag_inv directly (so does this path).

static bool potrf_direct(int m, int n) {
  if (m == n) return n <= 128;
  // tall windows from 17 columns up: square factor (register-tile / chain kernel) + solve of the rows below
  // (blocked driver, no workspace while n <= 128) -- 1.7-2.3x the one-CTA team kernel (tools/prof_tall.py)
  if (n >= 17) return false;
  return potrf_fits(m, n);
}
static int potrf_split(int n) {  // first panel width of the blocked driver
  int n1 = ((n / 2) + 7) / 8 * 8;
  return n1 > 128 ? 128 : (n1 < 8 ? 8 : n1);
}

static size_t potrf_ws(int m, int n, int di, int batch) {
  if (potrf_direct(m, n)) return 0;
  if (di & 3) return panel_bytes(m, n) * batch + potrf_ws(m, n, 0, batch);
  const int n1 = m == n || n > 128 ? potrf_split(n) : n;
  // step 1's own scratch (if its square is blocked too) is released before
  // steps 2-4 take theirs (potrf_run resets the arena mark)
  const size_t w1 = potrf_ws(n1, n1, 0, batch);
  size_t w = 0;
  if (n > n1) w += panel_bytes(m - n1, n1) * batch + panel_bytes(m - n1, n - n1) * batch + potrf_ws(m - n1, n - n1, 0, batch);
  return w1 > w ? w1 : w;
}

// rows of W (relative rows [0, rows)) item b may commit into D, see step 4
__global__ void potrf_commit_kernel(Mat S, Mat D, ix di, ix dj, ix rows, ix cols, const int32_t *info, int off,
                                    int n1, int lower) {
  const ix b = blockIdx.y;
  const int f = info[b];
  ix rmax;
  if (lower) {
    rmax = f < 0 ? rows : 0;  // unaligned window: healthy items only
  } else if (f < 0) {
    rmax = rows;
  } else {
    const ix fr = (ix)f - off;  // window-relative failing pivot
    rmax = fr >= n1 ? ((fr & ~(ix)3) + 4) - n1 : 0;
    if (rmax > rows) rmax = rows;
  }
  if (rmax <= 0) return;
  const double *s = S.p + b * S.stride;
  double *d = D.p + b * D.stride;
  // whole 4-row panels of an aligned window are contiguous runs of 32 * cols bytes on both sides: 16-byte copies
  ix r0 = 0;
  if (!lower && (di & 3) == 0 && (((uintptr_t)s | (uintptr_t)d) & 15) == 0 && ((S.stride | D.stride) & 1) == 0) {
    const int nfull = (int)(rmax >> 2), vpp = 2 * (int)cols, nv = nfull * vpp;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
      const int p = v / vpp, o = v - p * vpp;
      reinterpret_cast<double2 *>(d + eo(di + 4 * p, dj, D.cn))[o] = reinterpret_cast<const double2 *>(s + (ix)4 * p * S.cn)[o];
    }
    r0 = (ix)4 * nfull;
  }
  // the rest (a partial last panel, unaligned or lower-only windows) element-wise, in the source's panel-major order
  const ix nq = (rmax - r0 + 3) / 4, per = nq * cols * 4;
  for (ix e = (ix)blockIdx.x * blockDim.x + threadIdx.x; e < per; e += (ix)gridDim.x * blockDim.x) {
    const ix r = r0 + (e / (4 * cols)) * 4 + (e & 3), c = (e >> 2) % cols;
    if (r >= rmax || (lower && c > r)) continue;
    d[eo(di + r, dj + c, D.cn)] = s[eo(r, c, S.cn)];
  }
}

// Tall window whose square part has n % 4 != 0 columns: the row panel in which a failing item stops
// (rows iif .. iif + 3, iif = f & ~3) can reach past the square into the rows below it, and the reference's
// row-panel order has then solved those rows against the columns < iif (ccore.pyx:884-899).  The batched
// solve skips failing items, so their (at most three) rows are done here: one thread per row, forward
// substitution with the reciprocals the factorization stored.
__global__ void potrf_tail_rows_kernel(Mat C, Mat D, ix ci, ix cj, ix di, ix dj, ix m, ix n, const int32_t *info,
                                       int off, ix batch) {
  const ix b = (ix)blockIdx.x * (blockDim.x >> 2) + (threadIdx.x >> 2);
  if (b >= batch) return;
  const int f = info[b] - off;
  if (f < 0 || f >= (int)n) return;
  const ix iif = f & ~3;
  const ix r = n + (threadIdx.x & 3);
  if (r >= m || r >= iif + 4) return;
  const double *c = C.item(b), *dinv = D.ditem(b) + dj;
  double *d = D.item(b);
  for (ix j = 0; j < iif; ++j) {
    double s = c[eo(ci + r, cj + j, C.cn)];
    for (ix k = 0; k < j; ++k) s -= d[eo(di + r, dj + k, D.cn)] * d[eo(di + j, dj + k, D.cn)];
    d[eo(di + r, dj + j, D.cn)] = s * dinv[j];
  }
}

static int potrf_commit(const pb_dmat_batch &W, const pb_dmat_batch *sD, int di, int dj, int rows, int cols,
                        int32_t *info, int off, int n1, int lower, cudaStream_t st) {
  const int batch = sD->batch;
  ix per = (ix)((rows + 3) / 4) * cols * 4;
  unsigned gx = (unsigned)((per + 255) / 256);
  if (gx > 64) gx = 64;
  if (gx < 1) gx = 1;
  for (int b0 = 0; b0 < batch; b0 += 65535) {  // gridDim.y limit
    const int nb = batch - b0 < 65535 ? batch - b0 : 65535;
    Mat S = to_mat(&W), D = to_mat(sD);
    S.p += (ix)b0 * S.stride;
    D.p += (ix)b0 * D.stride;
    potrf_commit_kernel<<<dim3(gx, (unsigned)nb), 256, 0, st>>>(S, D, di, dj, rows, cols, info + b0, off, n1, lower);
    note_launch();
  }
  return finish(cudaGetLastError());
}

static int potrf_run(int m, int n, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di, int dj,
                     int32_t *info, int merge, int off, Work &w, cudaStream_t st) {
  const int batch = sD->batch;
  if (potrf_direct(m, n)) {
    PotrfArgs g;
    g.m = m, g.n = n;
    g.C = to_mat(sC), g.D = to_mat(sD);
    g.ci = ci, g.cj = cj, g.di = di, g.dj = dj;
    g.info = info;
    g.batch = batch;
    g.merge = merge;
    g.info_offset = off;
    return finish(run_potrf_l(g, st));
  }
  int r;
  if (di & 3) {
    // aligned workspace copy of the window; diag_inv straight into D's
    double *p = w.take(panel_bytes(m, n) * batch);
    if (!p) return work_fail();
    pb_dmat_batch X = panel_desc(p, m, n, batch, sD->dA ? sD->dA + dj : nullptr, sD->dA_stride);
    if ((r = potrf_run(m, n, sC, ci, cj, &X, 0, 0, info, merge, off, w, st))) return r;
    return potrf_commit(X, sD, di, dj, m, n, info, off, 0, 1, st);
  }
  const int n1 = m == n || n > 128 ? potrf_split(n) : n;
  // 1. square factor of the first n1 columns (its scratch, if any, is free again afterwards)
  const size_t mark = w.used;
  if ((r = potrf_run(n1, n1, sC, ci, cj, sD, di, dj, info, merge, off, w, st))) return r;
  w.used = mark;
  if (m == n1) return 0;
  if (n == n1) {
    // no trailing columns: nothing can fail after this solve, so the rows below go straight to D
    // (items that failed in the square are skipped and keep D's rows, like the reference's row-panel
    // order, which never reaches them)
    TrsmArgs g;
    g.m = m - n1, g.n = n1, g.alpha = 1.0;
    g.A = to_mat(sD), g.B = to_mat(sC), g.D = to_mat(sD);
    g.ai = di, g.aj = dj, g.bi = ci + n1, g.bj = cj, g.di = di + n1, g.dj = dj;
    g.use_dA = 1;
    g.info = nullptr;
    g.batch = batch;
    g.skip = info;
    if ((r = trsm_fits(m - n1, n1) ? finish(run_trsm_rltn(g, st)) : fail_arg(2, "panel too wide"))) return r;
    if (n1 & 3) {  // a failing item's last row panel may straddle the end of the square
      potrf_tail_rows_kernel<<<(unsigned)((batch + 31) / 32), 128, 0, st>>>(to_mat(sC), to_mat(sD), ci, cj, di, dj, m,
                                                                              n1, info, off, batch);
      note_launch();
      return finish(cudaGetLastError());
    }
    return 0;
  }
  // 2. rows below against it, into workspace
  double *pw = w.take(panel_bytes(m - n1, n1) * batch);
  if (!pw) return work_fail();
  pb_dmat_batch W = panel_desc(pw, m - n1, n1, batch);
  {
    TrsmArgs g;
    g.m = m - n1, g.n = n1, g.alpha = 1.0;
    g.A = to_mat(sD), g.B = to_mat(sC), g.D = to_mat(&W);
    g.ai = di, g.aj = dj, g.bi = ci + n1, g.bj = cj, g.di = 0, g.dj = 0;
    g.use_dA = 1;
    g.info = nullptr;
    g.batch = batch;
    g.skip = info;
    if ((r = trsm_fits(m - n1, n1) ? finish(run_trsm_rltn(g, st)) : fail_arg(2, "panel too wide"))) return r;
  }
  // 3. trailing block: T = C22 - W W^T, factored into D22
  if (n > n1) {
    double *pt = w.take(panel_bytes(m - n1, n - n1) * batch);
    if (!pt) return work_fail();
    pb_dmat_batch T = panel_desc(pt, m - n1, n - n1, batch);
    GemmArgs g;
    // lower trapezoid: m - n1 rows, n - n1 columns (syrk tiles cover m - n1 columns, stores clip to g.n)
    g.m = m - n1, g.n = n - n1, g.k = n1, g.alpha = -1.0, g.beta = 1.0;
    g.A = to_mat(&W), g.B = to_mat(&W), g.C = to_mat(sC), g.D = to_mat(&T);
    g.ai = 0, g.aj = 0, g.bi = 0, g.bj = 0, g.ci = ci + n1, g.cj = cj + n1, g.di = 0, g.dj = 0;
    g.batch = batch;
    g.vecA = g.vecB = true;
    g.tma = true;
    g.tmaC = tma_ok(sC);
    g.skip = info;
    if ((r = finish(run_syrk_ln(g, st)))) return r;
    // a square trailing block the chain kernel factors in one launch also commits the rows below the
    // first panel (step 4) per item, right after the item's factorization
    if (m == n && potrf_direct(m - n1, n - n1)) {
      PotrfArgs p;
      p.m = m - n1, p.n = n - n1;
      p.C = to_mat(&T), p.D = to_mat(sD);
      p.ci = 0, p.cj = 0, p.di = di + n1, p.dj = dj + n1;
      p.info = info;
      p.batch = batch;
      p.merge = 1;
      p.info_offset = off + n1;
      if (potrf_chain_ok(p) && (W.stride & 1) == 0) {
        p.commit = 1;
        p.cS = to_mat(&W);
        p.c_rows = m - n1, p.c_cols = n1, p.c_di = di + n1, p.c_dj = dj;
        return finish(run_potrf_chain(p, st));
      }
    }
    if ((r = potrf_run(m - n1, n - n1, &T, 0, 0, sD, di + n1, dj + n1, info, 1, off + n1, w, st))) return r;
  }
  // 4. commit the rows below the first panel
  return potrf_commit(W, sD, di + n1, dj, m - n1, n1, info, off, n1, 0, st);
}

static int potrf_check(int m, int n, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di,
                       int dj, int pc, int pd) {
  if (m < 0) return fail_arg(1, "negative size");
  if (n < 0 || n > m) return fail_arg(2, "potrf_l needs 0 <= n <= m");
  if (!sD) return fail_arg(pd, "null matrix descriptor");
  int r;
  if ((r = check_mat(sC, pc, ci, cj, m, n, sD->batch, false))) return r;
  if ((r = check_mat(sD, pd, di, dj, m, n, sD->batch, true))) return r;
  if (n == 0 || sD->batch == 0) return 0;
  if (!sD->dA) return fail_arg(pd, "output needs diag_inv storage");
  return check_dinv(sD, pd, dj, n);
}

int64_t pb_dpotrf_l_worksize(int m, int n, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di,
                             int dj) {
  const int r = potrf_check(m, n, sC, ci, cj, sD, di, dj, 3, 6);
  if (r) return r;
  if (n == 0 || sD->batch == 0) return 0;
  return (int64_t)potrf_ws(m, n, di, sD->batch);
}

int pb_dpotrf_l(int m, int n, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di, int dj,
                int32_t *info, void *work, int64_t work_bytes, void *stream) {
  // positions: m1 n2 C3 ci4 cj5 D6 di7 dj8 info9 work10 work_bytes11
  int r;
  if ((r = potrf_check(m, n, sC, ci, cj, sD, di, dj, 3, 6))) return r;
  if (n == 0 || sD->batch == 0) return 0;  // level3.py:335-336
  if (!info) return fail_arg(9, "info is required");
  const size_t need = potrf_ws(m, n, di, sD->batch);
  if (need && (!work || work_bytes < (int64_t)need)) return fail_arg(10, "workspace too small (see pb_dpotrf_l_worksize)");
  Work w;
  w.base = (char *)work, w.cap = (size_t)(work ? work_bytes : 0);
  return potrf_run(m, n, sC, ci, cj, sD, di, dj, info, 0, 0, w, (cudaStream_t)stream);
}

// ---- syrk_potrf_ln --------------------------------------------------------

static bool syrk_potrf_fused(int m, int n, int k, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB,
                             int bi, int bj, const pb_dmat_batch *sD, int di, bool &ab_same) {
  ab_same = sA->pA == sB->pA && sA->stride == sB->stride && sA->cn == sB->cn && ai == bi && aj == bj;
  // squares the register-resident small potrf covers keep its rounding
  // (zero factors then reproduce potrf_l bit for bit, test_level3.py:632-641)
  const bool small = m == n && n <= 16 && (di & 3) == 0 && tma_ok(sD);
  // one kernel for the register-tile squares (17..64) and for windows below 17 columns; wider or tall
  // windows go syrk -> workspace -> potrf_l (chain kernel / square factor + solve): 2-3x the fused
  // one-CTA team kernel from 65 columns up (tools/prof_syrk_potrf.py)
  const bool one_kernel = n <= 16 || (m == n && n <= 64);
  return !small && one_kernel && syrk_potrf_fits(m, n, k, ab_same);
}

static int syrk_potrf_check(int m, int n, int k, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB,
                            int bi, int bj, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di,
                            int dj) {
  if (m < 0) return fail_arg(1, "negative size");
  if (n < 0 || n > m) return fail_arg(2, "syrk_potrf_ln needs 0 <= n <= m");
  if (k < 0) return fail_arg(3, "negative size");
  if (!sD) return fail_arg(13, "null matrix descriptor");
  const int batch = sD->batch;
  int r;
  if ((r = check_mat(sA, 4, ai, aj, m, k, batch, false))) return r;
  if ((r = check_mat(sB, 7, bi, bj, n, k, batch, false))) return r;
  if ((r = check_mat(sC, 10, ci, cj, m, n, batch, false))) return r;
  if ((r = check_mat(sD, 13, di, dj, m, n, batch, true))) return r;
  if (n == 0 || batch == 0) return 0;
  if (!sD->dA) return fail_arg(13, "output needs diag_inv storage");
  return check_dinv(sD, 13, dj, n);
}

static size_t syrk_potrf_ws(int m, int n, int k, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB,
                            int bi, int bj, const pb_dmat_batch *sD, int di) {
  const int batch = sD->batch;
  if (k == 0) return potrf_ws(m, n, di, batch);
  bool ab_same;
  if (syrk_potrf_fused(m, n, k, sA, ai, aj, sB, bi, bj, sD, di, ab_same)) return 0;
  return panel_bytes(m, n) * batch + potrf_ws(m, n, di, batch);
}

int64_t pb_dsyrk_potrf_ln_worksize(int m, int n, int k, const pb_dmat_batch *sA, int ai, int aj,
                                   const pb_dmat_batch *sB, int bi, int bj, const pb_dmat_batch *sC, int ci, int cj,
                                   const pb_dmat_batch *sD, int di, int dj) {
  const int r = syrk_potrf_check(m, n, k, sA, ai, aj, sB, bi, bj, sC, ci, cj, sD, di, dj);
  if (r) return r;
  if (n == 0 || sD->batch == 0) return 0;
  return (int64_t)syrk_potrf_ws(m, n, k, sA, ai, aj, sB, bi, bj, sD, di);
}

int pb_dsyrk_potrf_ln(int m, int n, int k, const pb_dmat_batch *sA, int ai, int aj, const pb_dmat_batch *sB, int bi,
                      int bj, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di, int dj,
                      int32_t *info, void *work, int64_t work_bytes, void *stream) {
  // positions: m1 n2 k3 A4 ai5 aj6 B7 bi8 bj9 C10 ci11 cj12 D13 di14 dj15 info16 work17 work_bytes18
  // (level3.py:353-391)
  int r;
  if ((r = syrk_potrf_check(m, n, k, sA, ai, aj, sB, bi, bj, sC, ci, cj, sD, di, dj))) return r;
  const int batch = sD->batch;
  if (n == 0 || batch == 0) return 0;  // level3.py:370-371
  if (!info) return fail_arg(16, "info is required");
  const size_t need = syrk_potrf_ws(m, n, k, sA, ai, aj, sB, bi, bj, sD, di);
  if (need && (!work || work_bytes < (int64_t)need))
    return fail_arg(17, "workspace too small (see pb_dsyrk_potrf_ln_worksize)");
  Work w;
  w.base = (char *)work, w.cap = (size_t)(work ? work_bytes : 0);
  cudaStream_t st = (cudaStream_t)stream;
  // k == 0: exactly potrf_l of C (test_level3.py:343-353)
  if (k == 0) return potrf_run(m, n, sC, ci, cj, sD, di, dj, info, 0, 0, w, st);
  bool ab_same;
  if (syrk_potrf_fused(m, n, k, sA, ai, aj, sB, bi, bj, sD, di, ab_same)) {
    // one fused kernel: the item's C tri, A and B windows in shared memory
    PotrfArgs g;
    g.m = m, g.n = n;
    g.C = to_mat(sC), g.D = to_mat(sD);
    g.ci = ci, g.cj = cj, g.di = di, g.dj = dj;
    g.info = info;
    g.batch = batch;
    g.merge = 0;
    g.info_offset = 0;
    g.syrk = 1;
    g.ab_same = ab_same;
    g.A = to_mat(sA), g.B = to_mat(sB);
    g.ai = ai, g.aj = aj, g.bi = bi, g.bj = bj, g.k = k;
    return finish(run_syrk_potrf(g, st));
  }
  // W = lower trapezoid of C + A*B^T in workspace, then potrf_l(W -> D).
  // syrk_potrf_drv (ccore.pyx:908-941) walks the same block rows as
  // potrf_drv with the tile input C + A*B^T, so D's contents on a failed
  // pivot follow potrf_l's rule on W.
  double *wp = w.take(panel_bytes(m, n) * batch);
  if (!wp) return work_fail();
  pb_dmat_batch W = panel_desc(wp, m, n, batch);
  GemmArgs g;
  g.n = n, g.k = k, g.alpha = 1.0, g.beta = 1.0;
  g.A = to_mat(sA), g.B = to_mat(sB), g.C = to_mat(sC), g.D = to_mat(&W);
  g.batch = batch;
  g.tma = tma_ok(sA) && tma_ok(sB);
  g.tmaC = tma_ok(sC);
  g.skip = nullptr;
  // top n x n block: lower triangle only
  g.m = n;
  g.ai = ai, g.aj = aj, g.bi = bi, g.bj = bj, g.ci = ci, g.cj = cj, g.di = 0, g.dj = 0;
  g.vecA = vec16_ok(sA, ai), g.vecB = vec16_ok(sB, bi);
  r = finish(run_syrk_ln(g, st));
  if (!r && m > n) {  // trailing (m - n) x n rows: full product
    g.m = m - n;
    g.ai = ai + n, g.ci = ci + n, g.di = n;
    g.vecA = vec16_ok(sA, ai + n);
    r = finish(run_gemm_nt(g, st));
  }
  if (!r) r = potrf_run(m, n, &W, 0, 0, sD, di, dj, info, 0, 0, w, st);
  return r;
}

// ---- pack / unpack / gecp ------------------------------------------------

int pb_dpack(int m, int n, const double *S, int64_t s_row, int64_t s_col, int64_t s_stride, const pb_dmat_batch *sD,
             int di, int dj, void *stream) {
  if (m < 0) return fail_arg(1, "negative size");
  if (n < 0) return fail_arg(2, "negative size");
  if (!sD) return fail_arg(7, "null matrix descriptor");
  int r;
  if ((r = check_mat(sD, 7, di, dj, m, n, sD->batch, true))) return r;
  if (m == 0 || n == 0 || sD->batch == 0) return 0;
  if (!S) return fail_arg(3, "null source");
  CopyArgs g;
  memset(&g, 0, sizeof g);
  g.m = m, g.n = n;
  g.X = S;
  g.x_row = s_row, g.x_col = s_col, g.x_stride = s_stride;
  g.D = to_mat(sD);
  g.di = di, g.dj = dj;
  g.batch = sD->batch;
  return finish(run_pack(g, (cudaStream_t)stream));
}

int pb_dpack_cm(int m, int n, const double *S, int64_t lds, int64_t s_stride, const pb_dmat_batch *sD, int di, int dj,
                void *stream) {
  if (lds < (m > 1 ? m : 1)) return fail_arg(4, "lds < rows");
  const int r = pb_dpack(m, n, S, 1, lds, s_stride, sD, di, dj, stream);
  return r == -7 ? -6 : r;
}

int pb_dunpack(int m, int n, const pb_dmat_batch *sS, int si, int sj, double *X, int64_t x_row, int64_t x_col,
               int64_t x_stride, void *stream) {
  if (m < 0) return fail_arg(1, "negative size");
  if (n < 0) return fail_arg(2, "negative size");
  if (!sS) return fail_arg(3, "null matrix descriptor");
  int r;
  if ((r = check_mat(sS, 3, si, sj, m, n, sS->batch, false))) return r;
  if (m == 0 || n == 0 || sS->batch == 0) return 0;
  if (!X) return fail_arg(6, "null destination");
  CopyArgs g;
  memset(&g, 0, sizeof g);
  g.m = m, g.n = n;
  g.Xw = X;
  g.x_row = x_row, g.x_col = x_col, g.x_stride = x_stride;
  g.S = to_mat(sS);
  g.si = si, g.sj = sj;
  g.batch = sS->batch;
  return finish(run_unpack(g, (cudaStream_t)stream));
}

int pb_dunpack_cm(int m, int n, const pb_dmat_batch *sS, int si, int sj, double *Dcm, int64_t ldd, int64_t d_stride,
                  void *stream) {
  if (ldd < (m > 1 ? m : 1)) return fail_arg(7, "ldd < rows");
  return pb_dunpack(m, n, sS, si, sj, Dcm, 1, ldd, d_stride, stream);
}

int pb_dgecp(int m, int n, const pb_dmat_batch *sS, int si, int sj, const pb_dmat_batch *sD, int di, int dj,
             void *stream) {
  if (m < 0) return fail_arg(1, "negative size");
  if (n < 0) return fail_arg(2, "negative size");
  if (!sD) return fail_arg(6, "null matrix descriptor");
  int r;
  if ((r = check_mat(sS, 3, si, sj, m, n, sD->batch, false))) return r;
  if ((r = check_mat(sD, 6, di, dj, m, n, sD->batch, true))) return r;
  if (m == 0 || n == 0 || sD->batch == 0) return 0;
  CopyArgs g;
  memset(&g, 0, sizeof g);
  g.m = m, g.n = n;
  g.S = to_mat(sS);
  g.D = to_mat(sD);
  g.si = si, g.sj = sj, g.di = di, g.dj = dj;
  g.batch = sD->batch;
  return finish(run_gecp(g, (cudaStream_t)stream));
}

}  // extern "C"
