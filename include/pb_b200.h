/*
 * pb_b200.h -- C ABI of the B200-native batched panel-major FP64 engine.
 *
 * This is the drop-in boundary for the reference's compute-core surface
 * (panelblas `_backend` core module, selected in
 * /root/reference/pkg/src/panelblas/_backend/__init__.py:12-44 and bound
 * by level3.py:31 / pack.py:15).  Each entry point replaces one core
 * function, extended with a leading batch dimension:
 *
 *   pb_dgemm_nt    <- ccore.gemm_nt_drv   (ccore.pyx:746-771)
 *   pb_dsyrk_ln    <- ccore.syrk_ln_drv   (ccore.pyx:804-831)
 *   pb_dtrsm_rltn  <- ccore.trsm_rltn_drv (ccore.pyx:855-874) + the
 *                     reciprocal selection of level3._recip_diag (level3.py:160-177)
 *   pb_dpotrf_l    <- ccore.potrf_drv     (ccore.pyx:877-905)
 *   pb_dpack_cm    <- ccore.kpack_cm      (ccore.pyx:718-723)
 *   pb_dunpack_cm  <- ccore.kunpack_cm    (ccore.pyx:734-739)
 *   pb_dgecp       <- ccore.kgecp         (ccore.pyx:677-682)
 * and, for the next tier of callers:
 *   pb_dgemm_nn       <- ccore.gemm_nn_drv    (ccore.pyx:774-801)
 *   pb_dtrmm_rlnn     <- ccore.trmm_rlnn_drv  (ccore.pyx:834-852)
 *   pb_dsyrk_potrf_ln <- ccore.syrk_potrf_drv (ccore.pyx:908-941)
 *   pb_dgetrf         <- level3._getrf / _getrf_inplace (level3.py:405-498) over
 *                        kgetrf_panel, krowswap, lu_rowsolve_drv, gemm_nn_drv
 *
 * Conventions (mirroring the reference core):
 *   - caller owns every buffer; nothing here allocates device memory.  The
 *     calls whose reference counterpart needs scratch (level3.py:59, 236,
 *     338: unaligned windows, in-place trmm, the blocked factorization of
 *     large windows) take a caller-owned device workspace `work` of
 *     `work_bytes` bytes (256-byte aligned), sized by the matching
 *     pb_*_worksize query on the same arguments (0 = none needed, NULL ok);
 *     the library keeps no global state besides per-kernel launch
 *     attributes, and never changes the device's memory pools;
 *   - all pointers are DEVICE pointers; work is enqueued on `stream`
 *     (a cudaStream_t, NULL = legacy default stream) and is asynchronous;
 *   - panel size ps = 4; element (i, j) of an item lives at
 *       (i - i%4)*cn + 4*j + i%4      (matstore.py:37-45)
 *   - windows may start anywhere (ai%4 != 0 included); results never leave
 *     the m_store x n_store window (syrk/potrf: lower triangle only): every
 *     byte outside it reads back unchanged after the call.  Stream contract:
 *     the streaming kernels store whole 32-byte sectors, re-storing the
 *     bytes of a sector that lie outside the window with the values they
 *     read in the same kernel (strict upper of a diagonal 4x4 block, padding
 *     rows of the last panel).  So, as for partial overlap below, another
 *     stream must not write those sectors of the SAME item while the call
 *     runs; disjoint items, and windows sharing no 32-byte sector, may be
 *     processed concurrently on any streams;
 *   - D == C (gemm, syrk, potrf) and D == B (trsm) aliasing is supported;
 *     partial overlap is undefined (level3.py:14-15);
 *   - return 0 on success, -i if argument i (1-based) is invalid,
 *     PB_ERR_CUDA if a launch failed.  Bad pivots are not errors of the
 *     call: they are reported per item in `info` (-1 = ok, else the first
 *     failing pivot index, like the core's integer status), so one bad
 *     item never blocks the others.
 */
#ifndef PB_B200_H
#define PB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PB_PS 4
#define PB_ERR_CUDA (-1000)
#define PB_ERR_WORKSPACE (-1001) /* work smaller than the worksize query said */

/* A batch of equally-shaped panel-major matrices: blasfeo_dmat
 * / panelblas PanelMatrix (matstore.py:68-115) with
 * a leading batch axis.  Item b's data starts at pA + b*stride and its
 * diag_inv at dA + b*dA_stride.  stride == 0 broadcasts one matrix to all
 * items (inputs only). */
typedef struct pb_dmat_batch {
  double *pA;        /* panel-major data of item 0                       */
  double *dA;        /* diag_inv of item 0 (may be NULL if unused)        */
  int32_t m, n;      /* rows, cols of every item                          */
  int32_t cn;        /* panel length (blasfeo sda) = round_up(n, 4)       */
  int32_t batch;     /* number of items                                   */
  int64_t stride;    /* doubles between consecutive items' pA             */
  int64_t dA_stride; /* doubles between consecutive items' dA             */
} pb_dmat_batch;

/* ABI version (bumped on any signature change): 2 = caller-owned workspace. */
int pb_version(void);
/* Human-readable text of the last error raised on this thread. */
const char *pb_last_error(void);

/* D = alpha*A*B^T + beta*C (blasfeo_dgemm_nt).
 * A: m x k at (ai,aj); B: n x k at (bi,bj); C, D: m x n.
 * alpha == 0 ignores A and B (NaN-safe); beta == 0 never reads C. */
int pb_dgemm_nt(int m, int n, int k, double alpha,
                const pb_dmat_batch *sA, int ai, int aj,
                const pb_dmat_batch *sB, int bi, int bj, double beta,
                const pb_dmat_batch *sC, int ci, int cj,
                const pb_dmat_batch *sD, int di, int dj, void *stream);

/* lower(D) = alpha*A*B^T + beta*C, m x m, A and B m x k (blasfeo_dsyrk_ln).
 * The strict upper triangle of D is never written. */
int pb_dsyrk_ln(int m, int k, double alpha,
                const pb_dmat_batch *sA, int ai, int aj,
                const pb_dmat_batch *sB, int bi, int bj, double beta,
                const pb_dmat_batch *sC, int ci, int cj,
                const pb_dmat_batch *sD, int di, int dj, void *stream);

/* D = alpha*A*B + beta*C; A m x k, B k x n (level3.py:101-117,
 * gemm_nn_drv ccore.pyx:774-801).  Same special cases as pb_dgemm_nt. */
int pb_dgemm_nn(int m, int n, int k, double alpha,
                const pb_dmat_batch *sA, int ai, int aj,
                const pb_dmat_batch *sB, int bi, int bj, double beta,
                const pb_dmat_batch *sC, int ci, int cj,
                const pb_dmat_batch *sD, int di, int dj, void *stream);

/* D = alpha*B*A, A an n x n lower-triangular right factor (entries above
 * its diagonal are never read), B and D m x n (level3.py:140-153,
 * trmm_rlnn_drv ccore.pyx:834-852).  D = alpha*acc for every alpha.
 * Workspace: in place (D on B's storage) with n > 24. */
int64_t pb_dtrmm_rlnn_worksize(int m, int n, const pb_dmat_batch *sA, int ai, int aj,
                               const pb_dmat_batch *sB, int bi, int bj,
                               const pb_dmat_batch *sD, int di, int dj);
int pb_dtrmm_rlnn(int m, int n, double alpha,
                  const pb_dmat_batch *sA, int ai, int aj,
                  const pb_dmat_batch *sB, int bi, int bj,
                  const pb_dmat_batch *sD, int di, int dj,
                  void *work, int64_t work_bytes, void *stream);

/* D * A^T = alpha*B, A n x n lower non-unit, B and D m x n
 * (blasfeo_dtrsm_rltn).  Reciprocals of A's diagonal: use_dA == 1 reuses
 * sA->dA[aj .. aj+n) written by a factorization (level3.py:169-170);
 * use_dA == 0 computes 1/A[j,j] in-kernel, and an item with a zero
 * diagonal gets info[b] = j and is left untouched (level3.py:171-177);
 * use_dA == 2 decides per item from info ON ENTRY (the factorization's
 * per-item status): reuse where info[b] < 0, compute (with the zero-pivot
 * rule) where the factorization failed and its diag_inv is therefore
 * invalid (level3.py:346-349).  info may be NULL only when use_dA == 1. */
int pb_dtrsm_rltn(int m, int n, double alpha,
                  const pb_dmat_batch *sA, int ai, int aj, int use_dA,
                  const pb_dmat_batch *sB, int bi, int bj,
                  const pb_dmat_batch *sD, int di, int dj,
                  int32_t *info, void *stream);

/* Lower Cholesky factor of lower(C) into D (blasfeo_dpotrf_l), m x n with
 * n <= m (n < m: trailing rows solved against the factor, the reference's
 * non-squared variant).  Writes sD->dA[dj .. dj+n) = 1/L[j,j].
 * info[b] = -1, or the first pivot index with d <= 0 (NaN passes, as in
 * ccore.pyx:423); a failing item is written exactly as far as the
 * reference would have written it before returning (an unaligned D window,
 * di % 4 != 0, of a failing item is left untouched, level3.py:338-344).
 * Workspace: windows not factored by one kernel (n > 128, or tall windows
 * that do not fit one CTA) and unaligned D windows of those. */
int64_t pb_dpotrf_l_worksize(int m, int n,
                             const pb_dmat_batch *sC, int ci, int cj,
                             const pb_dmat_batch *sD, int di, int dj);
int pb_dpotrf_l(int m, int n,
                const pb_dmat_batch *sC, int ci, int cj,
                const pb_dmat_batch *sD, int di, int dj,
                int32_t *info, void *work, int64_t work_bytes, void *stream);

/* D = chol(lower(C + A*B^T)), m x n with n <= m, A m x k, B n x k
 * (level3.py:353-391, syrk_potrf_drv ccore.pyx:908-941): fused in one
 * kernel when the item fits one CTA, else the product goes to workspace
 * and pb_dpotrf_l's rules apply to it (info, diag_inv, partial writes of a
 * failed item). */
int64_t pb_dsyrk_potrf_ln_worksize(int m, int n, int k,
                                   const pb_dmat_batch *sA, int ai, int aj,
                                   const pb_dmat_batch *sB, int bi, int bj,
                                   const pb_dmat_batch *sC, int ci, int cj,
                                   const pb_dmat_batch *sD, int di, int dj);
int pb_dsyrk_potrf_ln(int m, int n, int k,
                      const pb_dmat_batch *sA, int ai, int aj,
                      const pb_dmat_batch *sB, int bi, int bj,
                      const pb_dmat_batch *sC, int ci, int cj,
                      const pb_dmat_batch *sD, int di, int dj,
                      int32_t *info, void *work, int64_t work_bytes, void *stream);

/* LU of the m x n window of C into D (level3.getrf_pivot / getrf_nopivot,
 * level3.py:405-498): D holds unit-L below the diagonal and U on/above,
 * diag_inv of D gets 1/U[j][j].  pivot != 0: partial pivoting, first
 * largest |value| wins, ipiv[b*ipiv_stride + j] = row exchanged with j
 * (completed 4-column panels only).  Bit-identical to the reference.
 * info[b] = -1, or the first zero pivot; then D holds the partially
 * factored window (panel-aligned di) or is untouched (di % 4 != 0), as the
 * reference leaves it when it raises SingularMatrixError.
 * Needs (m|1)*n*8 <= 220 KB (one item factored in shared memory). */
int pb_dgetrf(int m, int n, const pb_dmat_batch *sC, int ci, int cj, const pb_dmat_batch *sD, int di, int dj,
              int pivot, int64_t *ipiv, int64_t ipiv_stride, int32_t *info, void *stream);

/* Column-major -> panel-major copy (kpack_cm): item b's source element
 * (i, j) is S[b*s_stride + i + j*lds]. */
int pb_dpack_cm(int m, int n, const double *S, int64_t lds, int64_t s_stride,
                const pb_dmat_batch *sD, int di, int dj, void *stream);

/* Panel-major -> column-major copy (kunpack_cm): Dcm[b*d_stride + i + j*ldd]. */
int pb_dunpack_cm(int m, int n, const pb_dmat_batch *sS, int si, int sj,
                  double *Dcm, int64_t ldd, int64_t d_stride, void *stream);

/* Strided variants of pack/unpack for row-major host arrays
 * (pack.panel_from_array / panel_to_array, pack.py:215-237): element (i, j)
 * of item b at X[b*x_stride + i*x_row + j*x_col]. */
int pb_dpack(int m, int n, const double *S, int64_t s_row, int64_t s_col, int64_t s_stride,
             const pb_dmat_batch *sD, int di, int dj, void *stream);
int pb_dunpack(int m, int n, const pb_dmat_batch *sS, int si, int sj,
               double *X, int64_t x_row, int64_t x_col, int64_t x_stride, void *stream);

/* Panel -> panel window copy (kgecp), arbitrary origins on both sides. */
int pb_dgecp(int m, int n, const pb_dmat_batch *sS, int si, int sj,
             const pb_dmat_batch *sD, int di, int dj, void *stream);

/* Fused Config-5 chain: for every problem run
 * `stages` times  W = BAt P^T; lower(M) = W BAt^T + RQ; F = chol(M);
 * K = -F21 F11^{-T}; P = F22 F22^T  -- the composition of pb_dgemm_nt,
 * pb_dsyrk_ln, pb_dpotrf_l, pb_dtrsm_rltn, pb_dgemm_nt -- in one persistent
 * kernel with each problem resident in shared memory.  BAt: (nx+nu) x nx,
 * RQ: (nx+nu) x (nx+nu) (lower read), P: nx x nx (in: P_N, out: P_0),
 * K: nx x nu (last stage).  nx in {8,16,24,32,48,64}, nu == 8.
 * info[b] = -1, or stage*1000 + first bad pivot. */
int pb_driccati_chain(int nx, int nu, int stages, const pb_dmat_batch *sBAt, const pb_dmat_batch *sRQ,
                      const pb_dmat_batch *sP, const pb_dmat_batch *sK, int32_t *info, void *stream);

/* Number of kernels this thread has launched through the ABI since the
 * last reset (bench.py's gpu_launches evidence). */
int64_t pb_launch_count(int reset);

#ifdef __cplusplus
}
#endif

#endif /* PB_B200_H */
