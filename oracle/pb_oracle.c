/*
 * TEST INFRASTRUCTURE ONLY -- NOT PART OF THE PRODUCT PATH.
 *
 * CPU restatement of the reference's hot-path arithmetic (panelblas
 * `_backend/ccore.pyx`), used by tests/, __graft_entry__.smoke() and the
 * bench.py cpu_baseline / --impl reference legs as the parity checker.
 * The product (paper_1704_02457_b200/) never links, loads or calls this.
 *
 * Every function works on ONE panel-major item (plain double arrays plus
 * element offsets, exactly like the reference core) and has a `_batch`
 * twin that loops over items with explicit item strides.
 *
 * Bit-exactness: compiled with -ffp-contract=off (no FMA) and evaluates
 * each output element with the same operation sequence as the reference
 * core, so results are bit-identical to the compiled reference (pinned in
 * tests/test_oracle.py against tests/golden/ and oracle/_ref).
 *
 * Why per-element evaluation is the same sequence as the reference's
 * register-blocked kernels: `_acc_nt` (ccore.pyx:45-127) keeps one
 * independent accumulator per output element, starts it at 0.0 and adds
 * A[i,l]*(sign*B[j,l]) for l ascending; the mr=4/8 blocking only changes
 * which elements share a loop, never the order of one element's sum.
 */
#include <math.h>
#include <stdint.h>

typedef int64_t ix;

/* element_offset: matstore.py:37-45, ccore.pyx:16-18 (ps = 4). */
static inline ix eo(ix i, ix j, ix sd) { return (i & ~(ix)3) * sd + 4 * j + (i & 3); }

ix po_element_offset(ix i, ix j, ix sd) { return eo(i, j, sd); }

/* memsize_panel_matrix: matstore.py:208-218. */
static ix ru(ix x, ix to) { return (x + to - 1) / to * to; }
ix po_memsize(ix m, ix n) {
  ix mn = m < n ? m : n;
  return ru(ru(m, 4) * ru(n, 4) * 8, 64) + ru(mn * 8, 64);
}

/* _store_block scalar rule, ccore.pyx:26-42: alpha==0 ignores acc,
 * beta==0 never reads C. */
static inline double store_rule(double alpha, double acc, double beta, const double *c) {
  if (alpha != 0.0) {
    double v = alpha * acc;
    if (beta != 0.0) v += beta * (*c);
    return v;
  }
  if (beta != 0.0) return beta * (*c);
  return 0.0;
}

/* _ksyrk_core diagonal-tile rule, ccore.pyx:288-292. */
static inline double syrk_diag_rule(double alpha, double acc, double beta, const double *c) {
  double v = (beta != 0.0) ? beta * (*c) : 0.0;
  if (alpha != 0.0) v = alpha * acc + v;
  return v;
}

/* ---- pack / unpack / gecp: ccore.pyx:677-682, 718-723, 734-739 ---- */

void po_pack_cm(ix m, ix n, const double *S, ix so, ix lds, double *D, ix di, ix dj, ix sdd) {
  for (ix j = 0; j < n; ++j)
    for (ix i = 0; i < m; ++i) D[eo(di + i, dj + j, sdd)] = S[so + i + j * lds];
}

void po_unpack_cm(ix m, ix n, const double *S, ix si, ix sj, ix sds, double *D, ix dofs, ix ldd) {
  for (ix j = 0; j < n; ++j)
    for (ix i = 0; i < m; ++i) D[dofs + i + j * ldd] = S[eo(si + i, sj + j, sds)];
}

void po_gecp(ix m, ix n, const double *S, ix si, ix sj, ix sds, double *D, ix di, ix dj, ix sdd) {
  for (ix j = 0; j < n; ++j)
    for (ix i = 0; i < m; ++i) D[eo(di + i, dj + j, sdd)] = S[eo(si + i, sj + j, sds)];
}

/* ---- gemm_nt: level3.py:81-98 + gemm_nt_drv ccore.pyx:746-771 ----
 * D = alpha*A*B^T + beta*C.  Unaligned stream windows are read in place
 * (the reference's _aligned_stream repack is a bit-exact copy). */
void po_gemm_nt(ix m, ix n, ix k, double alpha,
                const double *A, ix ai, ix aj, ix sda,
                const double *B, ix bi, ix bj, ix sdb, double beta,
                const double *C, ix ci, ix cj, ix sdc,
                double *D, ix di, ix dj, ix sdd) {
  for (ix j = 0; j < n; ++j)
    for (ix i = 0; i < m; ++i) {
      double s = 0.0;
      for (ix l = 0; l < k; ++l) s += A[eo(ai + i, aj + l, sda)] * B[eo(bi + j, bj + l, sdb)];
      D[eo(di + i, dj + j, sdd)] = store_rule(alpha, s, beta, &C[eo(ci + i, cj + j, sdc)]);
    }
}

/* ---- syrk_ln: level3.py:120-137 + syrk_ln_drv ccore.pyx:804-831 ----
 * Lower triangle only; elements inside a diagonal 4x4 tile use the
 * _ksyrk_core rule, the rest the _store_block rule. */
void po_syrk_ln(ix m, ix k, double alpha,
                const double *A, ix ai, ix aj, ix sda,
                const double *B, ix bi, ix bj, ix sdb, double beta,
                const double *C, ix ci, ix cj, ix sdc,
                double *D, ix di, ix dj, ix sdd) {
  for (ix j = 0; j < m; ++j)
    for (ix i = j; i < m; ++i) {
      double s = 0.0;
      for (ix l = 0; l < k; ++l) s += A[eo(ai + i, aj + l, sda)] * B[eo(bi + j, bj + l, sdb)];
      const double *c = &C[eo(ci + i, cj + j, sdc)];
      D[eo(di + i, dj + j, sdd)] =
          ((i >> 2) == (j >> 2)) ? syrk_diag_rule(alpha, s, beta, c) : store_rule(alpha, s, beta, c);
    }
}

/* One 4-wide column block of a right-transposed lower solve, shared by
 * trsm_rltn and the off-diagonal tiles of potrf (_trsm_rltn_core,
 * ccore.pyx:358-388 with kp = 0):
 *   acc = -sum_{l<jj} X[r,l]*T[jj+c,l]   (l ascending, from 0.0)
 *   acc += alpha*Bv[r,c]
 *   acc -= X[r,jj+t]*T[jj+c,jj+t]        (t < c ascending, solved values)
 *   acc *= dinv[jj+c]                     (unless unit)
 * X is the output (already-solved columns), T the triangular factor.
 * Stores column by column into X, like the reference. */
static void rltn_block(ix rows, ix jj, ix ns, double alpha,
                       const double *T, ix ti, ix tj, ix sdt, int unit,
                       const double *Bv, ix bi, ix bj, ix sdb,
                       double *X, ix xi, ix xj, ix sdx,
                       const double *dinv, ix dio) {
  /* all downdates first, then the reference's column-outer loop, so that
   * in-place X == Bv reads B before the column is overwritten */
  double acc[4][4];
  for (ix r = 0; r < rows; ++r)
    for (ix c = 0; c < ns; ++c) {
      double s = 0.0;
      for (ix l = 0; l < jj; ++l) s += X[eo(xi + r, xj + l, sdx)] * (-T[eo(ti + jj + c, tj + l, sdt)]);
      acc[c][r] = s;
    }
  for (ix c = 0; c < ns; ++c) {
    for (ix r = 0; r < rows; ++r) acc[c][r] += alpha * Bv[eo(bi + r, bj + jj + c, sdb)];
    for (ix t = 0; t < c; ++t) {
      double e = T[eo(ti + jj + c, tj + jj + t, sdt)];
      for (ix r = 0; r < rows; ++r) acc[c][r] -= acc[t][r] * e;
    }
    if (!unit) {
      double inv = dinv[dio + jj + c];
      for (ix r = 0; r < rows; ++r) acc[c][r] *= inv;
    }
    for (ix r = 0; r < rows; ++r) X[eo(xi + r, xj + jj + c, sdx)] = acc[c][r];
  }
}

/* ---- trsm_rltn: trsm_rltn_drv ccore.pyx:855-874 ----
 * D*A^T = alpha*B, A lower (non-unit unless `unit`); reciprocals come from
 * dinv[dio + j] (level3.py:160-177 decides where they come from). */
void po_trsm_rltn(ix m, ix n, double alpha,
                  const double *A, ix ai, ix aj, ix sda, int unit,
                  const double *B, ix bi, ix bj, ix sdb,
                  double *D, ix di, ix dj, ix sdd,
                  const double *dinv, ix dio) {
  for (ix ii = 0; ii < m; ii += 4) {
    ix ms = m - ii < 4 ? m - ii : 4;
    for (ix jj = 0; jj < n; jj += 4) {
      ix ns = n - jj < 4 ? n - jj : 4;
      rltn_block(ms, jj, ns, alpha, A, ai, aj, sda, unit, B, bi + ii, bj, sdb, D, di + ii, dj, sdd, dinv, dio);
    }
  }
}

/* ---- potrf_l: potrf_drv ccore.pyx:877-905, _kpotrf_core :404-438 ----
 * Block-row ("up-looking") order; returns -1 or the first failing pivot
 * index.  On failure the failing diagonal tile is not stored, earlier
 * tiles and dinv[dio .. dio+index) are, exactly like the reference.
 * n < m: the trailing m-n rows are solved against the factor (tall). */
int po_potrf_l(ix m, ix n, const double *C, ix ci, ix cj, ix sdc,
               double *D, ix di, ix dj, ix sdd, double *dinv, ix dio) {
  for (ix ii = 0; ii < m; ii += 4) {
    ix ms = m - ii < 4 ? m - ii : 4;
    ix jmax = ii + 4 < n ? ii + 4 : n;
    for (ix jj = 0; jj < jmax; jj += 4) {
      ix ns = n - jj < 4 ? n - jj : 4;
      if (jj < ii) {
        rltn_block(ms, jj, ns, 1.0, D, di, dj, sdd, 0, C, ci + ii, cj, sdc, D, di + ii, dj, sdd, dinv, dio);
        continue;
      }
      /* diagonal tile: downdate, add C, in-register right-looking factor */
      double acc[4][4];
      for (ix c = 0; c < ns; ++c)
        for (ix r = 0; r < ms; ++r) {
          double s = 0.0;
          for (ix l = 0; l < jj; ++l)
            s += D[eo(di + ii + r, dj + l, sdd)] * (-D[eo(di + jj + c, dj + l, sdd)]);
          acc[c][r] = s;
        }
      for (ix c = 0; c < ns; ++c)
        for (ix r = 0; r < ms; ++r) acc[c][r] += C[eo(ci + ii + r, cj + jj + c, sdc)];
      for (ix c = 0; c < ns; ++c) {
        double d = acc[c][c];
        if (d <= 0.0) return (int)(jj + c); /* NaN passes, as in the reference */
        double ljj = sqrt(d);
        double inv = 1.0 / ljj;
        acc[c][c] = ljj;
        dinv[dio + jj + c] = inv;
        for (ix r = c + 1; r < ms; ++r) acc[c][r] *= inv;
        for (ix c2 = c + 1; c2 < ns; ++c2) {
          double lcj = acc[c][c2];
          for (ix r = c2; r < ms; ++r) acc[c2][r] -= acc[c][r] * lcj;
        }
      }
      for (ix c = 0; c < ns; ++c)
        for (ix r = c; r < ms; ++r) D[eo(di + ii + r, dj + jj + c, sdd)] = acc[c][r];
    }
  }
  return -1;
}


/* ---- §8f next tier: gemm_nn, trmm_rlnn, syrk_potrf_ln ---------------- */

/* gemm_nn: level3.py:101-117 + gemm_nn_drv ccore.pyx:774-801 (_acc_nn
 * :130-245): D = alpha*A*B + beta*C, B read across panels; per element the
 * sum starts at 0.0 and adds A[i,l]*B[l,j] for l ascending. */
void po_gemm_nn(ix m, ix n, ix k, double alpha,
                const double *A, ix ai, ix aj, ix sda,
                const double *B, ix bi, ix bj, ix sdb, double beta,
                const double *C, ix ci, ix cj, ix sdc,
                double *D, ix di, ix dj, ix sdd) {
  for (ix j = 0; j < n; ++j)
    for (ix i = 0; i < m; ++i) {
      double s = 0.0;
      for (ix l = 0; l < k; ++l) s += A[eo(ai + i, aj + l, sda)] * B[eo(bi + l, bj + j, sdb)];
      D[eo(di + i, dj + j, sdd)] = store_rule(alpha, s, beta, &C[eo(ci + i, cj + j, sdc)]);
    }
}

/* trmm_rlnn: level3.py:140-153 + trmm_rlnn_drv ccore.pyx:834-852
 * (_ktrmm_core :305-348): D = alpha*X*T, T n x n lower.  Column c of block
 * jj = c & ~3 sums l = jj .. n-1 ascending; the triangle head uses 0.0 for
 * T's strict upper (never read). */
void po_trmm_rlnn(ix m, ix n, double alpha,
                  const double *T, ix ti, ix tj, ix sdt,
                  const double *X, ix xi, ix xj, ix sdx,
                  double *D, ix di, ix dj, ix sdd) {
  for (ix c = 0; c < n; ++c) {
    const ix jj = c & ~(ix)3;
    for (ix i = 0; i < m; ++i) {
      double s = 0.0;
      for (ix l = jj; l < n; ++l) s += X[eo(xi + i, xj + l, sdx)] * (l >= c ? T[eo(ti + l, tj + c, sdt)] : 0.0);
      D[eo(di + i, dj + c, sdd)] = alpha * s;
    }
  }
}

/* syrk_potrf_ln: level3.py:353-391 + syrk_potrf_drv ccore.pyx:908-941:
 * fused D = chol(lower(C + A*B^T)); per element the accumulator first adds
 * A[i,l]*B[c,l] (l < k), then -L[i,l]*L[c,l] (l < jj), then C, then the
 * in-tile updates.  n < m solves the trailing rows (tall variant). */
int po_syrk_potrf_ln(ix m, ix n, ix k,
                     const double *A, ix ai, ix aj, ix sda,
                     const double *B, ix bi, ix bj, ix sdb,
                     const double *C, ix ci, ix cj, ix sdc,
                     double *D, ix di, ix dj, ix sdd, double *dinv, ix dio) {
  for (ix ii = 0; ii < m; ii += 4) {
    ix ms = m - ii < 4 ? m - ii : 4;
    ix jmax = ii + 4 < n ? ii + 4 : n;
    for (ix jj = 0; jj < jmax; jj += 4) {
      ix ns = n - jj < 4 ? n - jj : 4;
      double acc[4][4];
      for (ix c = 0; c < ns; ++c)
        for (ix r = 0; r < ms; ++r) {
          double s = 0.0;
          for (ix l = 0; l < k; ++l) s += A[eo(ai + ii + r, aj + l, sda)] * B[eo(bi + jj + c, bj + l, sdb)];
          for (ix l = 0; l < jj; ++l)
            s += D[eo(di + ii + r, dj + l, sdd)] * (-D[eo(di + jj + c, dj + l, sdd)]);
          acc[c][r] = s;
        }
      if (jj < ii) {
        for (ix c = 0; c < ns; ++c) {
          for (ix r = 0; r < ms; ++r) acc[c][r] += 1.0 * C[eo(ci + ii + r, cj + jj + c, sdc)];
          for (ix t = 0; t < c; ++t) {
            double e = D[eo(di + jj + c, dj + jj + t, sdd)];
            for (ix r = 0; r < ms; ++r) acc[c][r] -= acc[t][r] * e;
          }
          double inv = dinv[dio + jj + c];
          for (ix r = 0; r < ms; ++r) {
            acc[c][r] *= inv;
            D[eo(di + ii + r, dj + jj + c, sdd)] = acc[c][r];
          }
        }
        continue;
      }
      for (ix c = 0; c < ns; ++c)
        for (ix r = 0; r < ms; ++r) acc[c][r] += C[eo(ci + ii + r, cj + jj + c, sdc)];
      for (ix c = 0; c < ns; ++c) {
        double d = acc[c][c];
        if (d <= 0.0) return (int)(jj + c);
        double ljj = sqrt(d);
        double inv = 1.0 / ljj;
        acc[c][c] = ljj;
        dinv[dio + jj + c] = inv;
        for (ix r = c + 1; r < ms; ++r) acc[c][r] *= inv;
        for (ix c2 = c + 1; c2 < ns; ++c2) {
          double lcj = acc[c][c2];
          for (ix r = c2; r < ms; ++r) acc[c2][r] -= acc[c][r] * lcj;
        }
      }
      for (ix c = 0; c < ns; ++c)
        for (ix r = c; r < ms; ++r) D[eo(di + ii + r, dj + jj + c, sdd)] = acc[c][r];
    }
  }
  return -1;
}

/* ---- §8f row 4: getrf (LU, with / without partial pivoting) ----------
 * In place on D (the caller has copied C's window there), exactly
 * level3._getrf_inplace (level3.py:448-498): left-looking 4-column panels;
 * per panel the gemm_nn_drv downdate (ccore.pyx:774-801, store rule
 * v = -1*acc + 1*C), kgetrf_panel (:563-650: pivot = first largest |.|,
 * strict >, bv == 0 -> singular; row swap inside the panel's columns;
 * inv = 1/u; column scaled by inv; rank-1 update skipped where u_cc == 0),
 * then the deferred row swaps left/right of the panel (krowswap :661-670)
 * and the U12 row solve (gemm_nn_drv + lu_rowsolve_drv :488-500 =
 * _ktrsm_llnu_core :453-477 with km = 0: acc = 0.0 + 1.0*C, forward
 * substitution with the unit-lower panel).  Returns -1 or the first zero
 * pivot (global index); ipiv[j0 + c] = j0 + r only for completed panels;
 * dinv[dio + c] for completed columns. */
int po_getrf(ix m, ix n, int pivot, double *D, ix di, ix dj, ix sdd, double *dinv, ix dio, int64_t *ipiv) {
  const ix mn = m < n ? m : n;
#define E(i, j) D[eo(di + (i), dj + (j), sdd)]
  for (ix j0 = 0; j0 < mn; j0 += 4) {
    const ix jb = mn - j0 < 4 ? mn - j0 : 4;
    if (j0 > 0)
      po_gemm_nn(m - j0, jb, j0, -1.0, D, di + j0, dj, sdd, D, di, dj + j0, sdd, 1.0, D, di + j0, dj + j0, sdd, D,
                 di + j0, dj + j0, sdd);
    ix piv[4] = {0, 0, 0, 0};
    for (ix c = 0; c < jb; ++c) {
      const ix gc = j0 + c;
      if (pivot) {
        ix best = c;
        double bv = fabs(E(gc, gc));
        for (ix r = c + 1; r < m - j0; ++r) {
          const double v = fabs(E(j0 + r, gc));
          if (v > bv) bv = v, best = r;
        }
        if (bv == 0.0) return (int)gc;
        piv[c] = best;
        if (best != c)
          for (ix cc = 0; cc < jb; ++cc) {
            const double t = E(gc, j0 + cc);
            E(gc, j0 + cc) = E(j0 + best, j0 + cc);
            E(j0 + best, j0 + cc) = t;
          }
      } else if (E(gc, gc) == 0.0) {
        return (int)gc;
      }
      const double u = E(gc, gc);
      const double inv = 1.0 / u;
      dinv[dio + gc] = inv;
      for (ix r = gc + 1; r < m; ++r) E(r, gc) *= inv;
      for (ix cc = c + 1; cc < jb; ++cc) {
        const double ucc = E(gc, j0 + cc);
        if (ucc != 0.0)
          for (ix r = gc + 1; r < m; ++r) E(r, j0 + cc) -= E(r, gc) * ucc;
      }
    }
    if (pivot)
      for (ix cc = 0; cc < jb; ++cc) {
        const ix r = piv[cc];
        ipiv[j0 + cc] = j0 + r;
        if (r != cc) {
          for (ix j = 0; j < j0; ++j) {
            const double t = E(j0 + cc, j);
            E(j0 + cc, j) = E(j0 + r, j);
            E(j0 + r, j) = t;
          }
          for (ix j = j0 + jb; j < n; ++j) {
            const double t = E(j0 + cc, j);
            E(j0 + cc, j) = E(j0 + r, j);
            E(j0 + r, j) = t;
          }
        }
      }
    if (j0 + jb < n) {
      if (j0 > 0)
        po_gemm_nn(jb, n - j0 - jb, j0, -1.0, D, di + j0, dj, sdd, D, di, dj + j0 + jb, sdd, 1.0, D, di + j0,
                   dj + j0 + jb, sdd, D, di + j0, dj + j0 + jb, sdd);
      for (ix j = j0 + jb; j < n; ++j) {
        double acc[4];
        for (ix i = 0; i < jb; ++i) acc[i] = 0.0 + 1.0 * E(j0 + i, j);
        for (ix i = 0; i < jb; ++i) {
          const double x = acc[i];
          for (ix t = i + 1; t < jb; ++t) acc[t] -= E(j0 + t, j0 + i) * x;
        }
        for (ix i = 0; i < jb; ++i) E(j0 + i, j) = acc[i];
      }
    }
  }
#undef E
  return -1;
}

/* ---- naive column-major oracles: ccore.pyx:1109-1223 (o_*) ----
 * Independent of the panel machinery; used to cross-check the above. */
void po_naive_potrf(ix m, const double *C, ix ldc, double *L, ix ldl) {
  for (ix j = 0; j < m; ++j) {
    double s = C[j + j * ldc];
    for (ix t = 0; t < j; ++t) s -= L[j + t * ldl] * L[j + t * ldl];
    double ljj = sqrt(s);
    L[j + j * ldl] = ljj;
    for (ix i = j + 1; i < m; ++i) {
      double v = C[i + j * ldc];
      for (ix t = 0; t < j; ++t) v -= L[i + t * ldl] * L[j + t * ldl];
      L[i + j * ldl] = v / ljj;
    }
  }
}

/* ---- batch loops (item strides in doubles; stride 0 broadcasts) ---- */

void po_pack_cm_batch(ix nb, ix m, ix n, const double *S, ix lds, ix s_stride,
                      double *D, ix di, ix dj, ix sdd, ix d_stride) {
  for (ix b = 0; b < nb; ++b) po_pack_cm(m, n, S + b * s_stride, 0, lds, D + b * d_stride, di, dj, sdd);
}

void po_unpack_cm_batch(ix nb, ix m, ix n, const double *S, ix si, ix sj, ix sds, ix s_stride,
                        double *D, ix ldd, ix d_stride) {
  for (ix b = 0; b < nb; ++b) po_unpack_cm(m, n, S + b * s_stride, si, sj, sds, D + b * d_stride, 0, ldd);
}

void po_gecp_batch(ix nb, ix m, ix n, const double *S, ix si, ix sj, ix sds, ix s_stride,
                   double *D, ix di, ix dj, ix sdd, ix d_stride) {
  for (ix b = 0; b < nb; ++b) po_gecp(m, n, S + b * s_stride, si, sj, sds, D + b * d_stride, di, dj, sdd);
}

void po_gemm_nt_batch(ix nb, ix m, ix n, ix k, double alpha,
                      const double *A, ix ai, ix aj, ix sda, ix as,
                      const double *B, ix bi, ix bj, ix sdb, ix bs, double beta,
                      const double *C, ix ci, ix cj, ix sdc, ix cs,
                      double *D, ix di, ix dj, ix sdd, ix ds) {
  for (ix b = 0; b < nb; ++b)
    po_gemm_nt(m, n, k, alpha, A + b * as, ai, aj, sda, B + b * bs, bi, bj, sdb, beta,
               C + b * cs, ci, cj, sdc, D + b * ds, di, dj, sdd);
}

void po_syrk_ln_batch(ix nb, ix m, ix k, double alpha,
                      const double *A, ix ai, ix aj, ix sda, ix as,
                      const double *B, ix bi, ix bj, ix sdb, ix bs, double beta,
                      const double *C, ix ci, ix cj, ix sdc, ix cs,
                      double *D, ix di, ix dj, ix sdd, ix ds) {
  for (ix b = 0; b < nb; ++b)
    po_syrk_ln(m, k, alpha, A + b * as, ai, aj, sda, B + b * bs, bi, bj, sdb, beta,
               C + b * cs, ci, cj, sdc, D + b * ds, di, dj, sdd);
}

void po_trsm_rltn_batch(ix nb, ix m, ix n, double alpha,
                        const double *A, ix ai, ix aj, ix sda, ix as, int unit,
                        const double *B, ix bi, ix bj, ix sdb, ix bs,
                        double *D, ix di, ix dj, ix sdd, ix ds,
                        const double *dinv, ix dio, ix dinv_stride) {
  for (ix b = 0; b < nb; ++b)
    po_trsm_rltn(m, n, alpha, A + b * as, ai, aj, sda, unit, B + b * bs, bi, bj, sdb,
                 D + b * ds, di, dj, sdd, dinv + b * dinv_stride, dio);
}

void po_potrf_l_batch(ix nb, ix m, ix n, const double *C, ix ci, ix cj, ix sdc, ix cs,
                      double *D, ix di, ix dj, ix sdd, ix ds, double *dinv, ix dio, ix dinv_stride,
                      int32_t *info) {
  for (ix b = 0; b < nb; ++b)
    info[b] = po_potrf_l(m, n, C + b * cs, ci, cj, sdc, D + b * ds, di, dj, sdd, dinv + b * dinv_stride, dio);
}
