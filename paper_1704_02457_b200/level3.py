"""Batched level-3 routines on panel-major batches: the reference's
``level3`` API (level3.py:81-350) with every operand a batch.

Same names, argument order, bounds checks, error types and discrete
semantics as the reference:

* ``gemm_nt(m, n, k, alpha, A, B, beta, C, D)``      level3.py:81-98
* ``syrk_ln(m, k, alpha, A, B, beta, C, D)``         level3.py:120-137
* ``trsm_rltn(m, n, alpha, A, B, D)``                level3.py:220-221, 180-244
* ``potrf_l(m, C, D, n=None)``                       level3.py:319-350

Operands are :class:`PanelBatch` objects or :class:`SubRef` windows into
them; an operand with batch 1 broadcasts to D's batch.  All work is
enqueued on the current torch CUDA stream through the C ABI
(include/pb_b200.h); the only host synchronisation is the optional
pivot check of the factorizations (``check=True``, the reference's
raise-on-bad-pivot behaviour).  Per-item statuses are returned as an
int32 device tensor ``info`` (-1 ok, else first failing index), and a
failing item is handled exactly like an independent reference call:
the other items are still computed.
"""
from __future__ import annotations

import ctypes

import torch

from . import _native
from .errors import DimensionError, NotPositiveDefiniteError, SingularMatrixError
from .matstore import PanelBatch, SubRef

TRSM_VARIANTS = ("llnu", "lunn", "rltn", "rltu", "rutn")


def _ref(x, name):
    if isinstance(x, PanelBatch):
        return x, 0, 0
    if isinstance(x, SubRef) and isinstance(x.mat, PanelBatch):
        return x.mat, x.ai, x.aj
    raise TypeError(f"{name} must be a PanelBatch or a panel SubRef")


def _check(mat, ai, aj, m, n, name):
    # level3.py:47-53
    if m < 0 or n < 0:
        raise DimensionError(f"negative size {m}x{n} for {name}")
    if ai + m > mat.rows or aj + n > mat.cols:
        raise DimensionError(
            f"{name} window ({ai}:{ai + m}, {aj}:{aj + n}) exceeds "
            f"{mat.rows}x{mat.cols} matrix")


def _batch_of(d, *inputs):
    nb = d.batch
    for x in inputs:
        if x.batch not in (nb, 1):
            raise DimensionError(f"operand batch {x.batch} does not match output batch {nb}")
        if x.device != d.device:
            raise DimensionError("operands live on different devices")
    if d.device.type != "cuda":
        raise RuntimeError("panel-major engine runs on CUDA devices only (no CPU fallback)")
    return nb


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _on(dev):
    """Run the native call with ``dev`` current: the library sizes grids and
    caches launch attributes for the current device."""
    return torch.cuda.device(dev)


def _mark_diag(mat, dj, n, diagonal, info=None):
    # level3.py:69-74; `info`: per-item status of an unchecked factorization
    # (failed items keep invalid reciprocals, level3.py:346-349)
    if diagonal:
        mat.diag_lo = dj
        mat.diag_hi = dj + n
    else:
        mat.diag_lo = mat.diag_hi = 0
    mat.diag_info = info if (diagonal and n > 0) else None


def _check_dinv(d, dj, w):
    # the output's diag_inv holds min(rows, cols) reciprocals (matstore.py:88-91);
    # the reference core would write past its end (unchecked), here it is an error
    if w > 0 and dj + w > min(d.rows, d.cols):
        raise DimensionError(f"D.diag_inv too short: dj + n = {dj + w} exceeds min(rows, cols) = {min(d.rows, d.cols)}")


def _first_failure(info):
    """(batch_index, index) of the first failing item, or None (host sync)."""
    bad = torch.nonzero(info >= 0)
    if bad.numel() == 0:
        return None
    b = int(bad[0, 0])
    return b, int(info[b])


# ---------------------------------------------------------------------------
# gemm / syrk


def gemm_nt(m, n, k, alpha, A, B, beta, C, D):
    """D = alpha*A*B' + beta*C with A m x k and B n x k, for every item."""
    a, ai, aj = _ref(A, "A")
    b, bi, bj = _ref(B, "B")
    c, ci, cj = _ref(C, "C")
    d, di, dj = _ref(D, "D")
    _check(a, ai, aj, m, k, "A")
    _check(b, bi, bj, n, k, "B")
    _check(c, ci, cj, m, n, "C")
    _check(d, di, dj, m, n, "D")
    nb = _batch_of(d, a, b, c)
    if m == 0 or n == 0 or nb == 0:
        return
    da, db, dc, dd = (x.descriptor(nb) for x in (a, b, c, d))
    with _on(d.device):
        _native.call("pb_dgemm_nt", m, n, k, float(alpha), ctypes.byref(da), ai, aj, ctypes.byref(db), bi, bj,
                     float(beta), ctypes.byref(dc), ci, cj, ctypes.byref(dd), di, dj, _stream(d.device))


def gemm_nn(m, n, k, alpha, A, B, beta, C, D):
    """D = alpha*A*B + beta*C with A m x k and B k x n, for every item
    (level3.py:101-117).  Unaligned A windows are read in place instead of
    the reference's repack (level3.py:113)."""
    a, ai, aj = _ref(A, "A")
    b, bi, bj = _ref(B, "B")
    c, ci, cj = _ref(C, "C")
    d, di, dj = _ref(D, "D")
    _check(a, ai, aj, m, k, "A")
    _check(b, bi, bj, k, n, "B")
    _check(c, ci, cj, m, n, "C")
    _check(d, di, dj, m, n, "D")
    nb = _batch_of(d, a, b, c)
    if m == 0 or n == 0 or nb == 0:
        return
    da, db, dc, dd = (x.descriptor(nb) for x in (a, b, c, d))
    with _on(d.device):
        _native.call("pb_dgemm_nn", m, n, k, float(alpha), ctypes.byref(da), ai, aj, ctypes.byref(db), bi, bj,
                     float(beta), ctypes.byref(dc), ci, cj, ctypes.byref(dd), di, dj, _stream(d.device))


def trmm_rlnn(m, n, alpha, A, B, D):
    """D = alpha*B*A with A an n x n lower-triangular right factor
    (level3.py:140-153); A's strict upper triangle is never read."""
    a, ai, aj = _ref(A, "A")
    b, bi, bj = _ref(B, "B")
    d, di, dj = _ref(D, "D")
    _check(a, ai, aj, n, n, "A")
    _check(b, bi, bj, m, n, "B")
    _check(d, di, dj, m, n, "D")
    nb = _batch_of(d, a, b)
    if m == 0 or n == 0 or nb == 0:
        return
    da, db, dd = (x.descriptor(nb) for x in (a, b, d))
    with _on(d.device):
        need = _native.worksize("pb_dtrmm_rlnn", m, n, ctypes.byref(da), ai, aj, ctypes.byref(db), bi, bj,
                                ctypes.byref(dd), di, dj)
        ws, wp, wb = _native.workspace(need, d.device)
        _native.call("pb_dtrmm_rlnn", m, n, float(alpha), ctypes.byref(da), ai, aj, ctypes.byref(db), bi, bj,
                     ctypes.byref(dd), di, dj, wp, wb, _stream(d.device))


def syrk_ln(m, k, alpha, A, B, beta, C, D):
    """Lower triangle of D = alpha*A*B' + beta*C (m x m); upper untouched."""
    a, ai, aj = _ref(A, "A")
    b, bi, bj = _ref(B, "B")
    c, ci, cj = _ref(C, "C")
    d, di, dj = _ref(D, "D")
    _check(a, ai, aj, m, k, "A")
    _check(b, bi, bj, m, k, "B")
    _check(c, ci, cj, m, m, "C")
    _check(d, di, dj, m, m, "D")
    nb = _batch_of(d, a, b, c)
    if m == 0 or nb == 0:
        return
    da, db, dc, dd = (x.descriptor(nb) for x in (a, b, c, d))
    with _on(d.device):
        _native.call("pb_dsyrk_ln", m, k, float(alpha), ctypes.byref(da), ai, aj, ctypes.byref(db), bi, bj,
                     float(beta), ctypes.byref(dc), ci, cj, ctypes.byref(dd), di, dj, _stream(d.device))


# ---------------------------------------------------------------------------
# triangular solve


def trsm(m, n, alpha, A, B, D, variant, check=True):
    """Variant dispatcher of the reference (level3.py:180-209); only the
    hot-path variant ``rltn`` is provided by this engine."""
    if variant not in TRSM_VARIANTS:
        raise ValueError(f"unknown trsm variant {variant!r}; one of {TRSM_VARIANTS}")
    if variant != "rltn":
        raise NotImplementedError(f"trsm variant {variant!r} is outside the batched hot path (rltn only)")
    return trsm_rltn(m, n, alpha, A, B, D, check=check)


def trsm_rltn(m, n, alpha, A, B, D, check=True):
    """Solve D*A' = alpha*B, A n x n lower non-unit, for every item.

    Reciprocals follow level3._recip_diag (level3.py:160-177): the
    factorization's diag_inv is reused when the A window sits on the
    diagonal of A's freshly factored range, otherwise 1/A[j,j] is computed
    in-kernel and an item with a zero pivot is left untouched.  Returns the
    per-item ``info`` tensor (or None when reciprocals were reused); with
    ``check`` a zero pivot raises SingularMatrixError like the reference.
    """
    a, ai, aj = _ref(A, "A")
    b, bi, bj = _ref(B, "B")
    d, di, dj = _ref(D, "D")
    _check(a, ai, aj, n, n, "A")
    _check(b, bi, bj, m, n, "B")
    _check(d, di, dj, m, n, "D")
    nb = _batch_of(d, a, b)
    if m == 0 or n == 0 or nb == 0:
        return None
    use_dA = 1 if (ai == aj and a.diag_inv_valid(aj, n)) else 0
    info = None
    if use_dA and a.diag_info is not None:
        # the factorization ran unchecked: reuse per item, recompute for the
        # items it failed on (their diag_inv is invalid, level3.py:346-349)
        use_dA = 2
        src = a.diag_info if a.batch == nb else a.diag_info.expand(nb)
        info = src.to(torch.int32).clone()
    elif not use_dA:
        info = torch.empty(nb, dtype=torch.int32, device=d.device)
    da, db, dd = (x.descriptor(nb) for x in (a, b, d))
    with _on(d.device):
        _native.call("pb_dtrsm_rltn", m, n, float(alpha), ctypes.byref(da), ai, aj, use_dA, ctypes.byref(db), bi,
                     bj, ctypes.byref(dd), di, dj, ctypes.c_void_p(info.data_ptr() if info is not None else 0),
                     _stream(d.device))
    if check and info is not None:
        f = _first_failure(info)
        if f is not None:
            raise SingularMatrixError(f"trsm_rlt: zero diagonal at column {f[1]} (batch item {f[0]})",
                                      f[1], batch_index=f[0], info=info)
    return info


# ---------------------------------------------------------------------------
# Cholesky


def potrf_l(m, C, D, n=None, check=True):
    """Lower Cholesky factor of every item's lower(C) into D (level3.py:319-350).

    n < m factors the top n x n block and solves the trailing rows against
    it.  Fills D.diag_inv[:, dj:dj+n].  Returns the per-item ``info``
    tensor; with ``check`` the first bad pivot raises
    NotPositiveDefiniteError (index relative to the window, plus
    batch_index) after all items have been processed.
    """
    if n is None:
        n = m
    if n > m:
        raise DimensionError(f"potrf_l needs n <= m, got m={m} n={n}")
    c, ci, cj = _ref(C, "C")
    d, di, dj = _ref(D, "D")
    _check(c, ci, cj, m, n, "C")
    _check(d, di, dj, m, n, "D")
    _check_dinv(d, dj, n)
    nb = _batch_of(d, c)
    if n == 0 or nb == 0:
        return None
    info = torch.empty(nb, dtype=torch.int32, device=d.device)
    dc, dd = c.descriptor(nb), d.descriptor(nb)
    with _on(d.device):
        need = _native.worksize("pb_dpotrf_l", m, n, ctypes.byref(dc), ci, cj, ctypes.byref(dd), di, dj)
        ws, wp, wb = _native.workspace(need, d.device)
        _native.call("pb_dpotrf_l", m, n, ctypes.byref(dc), ci, cj, ctypes.byref(dd), di, dj,
                     ctypes.c_void_p(info.data_ptr()), wp, wb, _stream(d.device))
    if check:
        f = _first_failure(info)
        if f is not None:
            _mark_diag(d, dj, 0, False)
            raise NotPositiveDefiniteError(
                f"potrf_l: non-positive pivot at index {f[1]} (batch item {f[0]})", f[1],
                batch_index=f[0], info=info)
    _mark_diag(d, dj, n, di == dj, None if check else info)
    return info


def syrk_potrf_ln(m, k, A, B, C, D, n=None, check=True):
    """D = chol(lower(C + A*B')) for every item (level3.py:353-391).

    A is m x k, B n x k, C and D m x n with n <= m.  Matches syrk_ln
    (alpha = beta = 1) followed by potrf_l up to rounding, as the
    reference's docstring states; info / diag_inv / failure rules are
    potrf_l's.
    """
    if n is None:
        n = m
    if n > m:
        raise DimensionError(f"syrk_potrf_ln needs n <= m, got m={m} n={n}")
    a, ai, aj = _ref(A, "A")
    b, bi, bj = _ref(B, "B")
    c, ci, cj = _ref(C, "C")
    d, di, dj = _ref(D, "D")
    _check(a, ai, aj, m, k, "A")
    _check(b, bi, bj, n, k, "B")
    _check(c, ci, cj, m, n, "C")
    _check(d, di, dj, m, n, "D")
    _check_dinv(d, dj, n)
    nb = _batch_of(d, a, b, c)
    if n == 0 or nb == 0:
        return None
    info = torch.empty(nb, dtype=torch.int32, device=d.device)
    da, db, dc, dd = (x.descriptor(nb) for x in (a, b, c, d))
    with _on(d.device):
        need = _native.worksize("pb_dsyrk_potrf_ln", m, n, k, ctypes.byref(da), ai, aj, ctypes.byref(db), bi, bj,
                                ctypes.byref(dc), ci, cj, ctypes.byref(dd), di, dj)
        ws, wp, wb = _native.workspace(need, d.device)
        _native.call("pb_dsyrk_potrf_ln", m, n, k, ctypes.byref(da), ai, aj, ctypes.byref(db), bi, bj,
                     ctypes.byref(dc), ci, cj, ctypes.byref(dd), di, dj, ctypes.c_void_p(info.data_ptr()),
                     wp, wb, _stream(d.device))
    if check:
        f = _first_failure(info)
        if f is not None:
            _mark_diag(d, dj, 0, False)
            raise NotPositiveDefiniteError(
                f"syrk_potrf_ln: non-positive pivot at index {f[1]} (batch item {f[0]})", f[1],
                batch_index=f[0], info=info)
    _mark_diag(d, dj, n, di == dj, None if check else info)
    return info


# ---------------------------------------------------------------------------
# LU


def _getrf(m, n, C, D, pivot, ipiv, check, name):
    # level3.py:431-446: bounds, min(m, n) == 0 no-op, D <- C window, in-place LU
    c, ci, cj = _ref(C, "C")
    d, di, dj = _ref(D, "D")
    _check(c, ci, cj, m, n, "C")
    _check(d, di, dj, m, n, "D")
    _check_dinv(d, dj, min(m, n))
    nb = _batch_of(d, c)
    mn = min(m, n)
    if mn == 0 or nb == 0:
        return None
    if pivot:
        if ipiv is None:
            ipiv = torch.zeros((nb, mn), dtype=torch.int64, device=d.device)
        elif ipiv.dim() != 2 or ipiv.shape[0] != nb or ipiv.shape[1] < mn or ipiv.dtype != torch.int64 \
                or ipiv.device != d.device or ipiv.stride(1) != 1:
            raise DimensionError(f"ipiv needs shape ({nb}, >= {mn}) int64 on {d.device}, unit column stride")
    info = torch.empty(nb, dtype=torch.int32, device=d.device)
    dc, dd = c.descriptor(nb), d.descriptor(nb)
    with _on(d.device):
        _native.call("pb_dgetrf", m, n, ctypes.byref(dc), ci, cj, ctypes.byref(dd), di, dj, 1 if pivot else 0,
                     ctypes.c_void_p(ipiv.data_ptr() if pivot else 0), ipiv.stride(0) if pivot else 0,
                     ctypes.c_void_p(info.data_ptr()), _stream(d.device))
    if check:
        f = _first_failure(info)
        if f is not None:
            _mark_diag(d, dj, 0, False)
            raise SingularMatrixError(f"{name}: zero pivot at index {f[1]} (batch item {f[0]})", f[1],
                                      batch_index=f[0], info=info)
    _mark_diag(d, dj, mn, di == dj, None if check else info)
    return ipiv if pivot else info


def getrf_nopivot(m, n, C, D, check=True):
    """LU without pivoting of every item (level3.py:405-411): D holds unit-L
    below the diagonal and U on/above, D.diag_inv the reciprocals of U's
    diagonal.  Bit-identical to the reference.  Returns ``info``; with
    ``check`` an exactly-zero pivot raises SingularMatrixError (index, and
    the batch_index of the first failing item)."""
    return _getrf(m, n, C, D, False, None, check, "getrf_nopivot")


def getrf_pivot(m, n, C, D, ipiv=None, check=True):
    """LU with partial pivoting, P*C = L*U, of every item (level3.py:414-428).

    ``ipiv`` is an int64 tensor (batch, >= min(m, n)) of transpositions:
    ipiv[b, j] = r means rows j and r (r >= j) were exchanged at step j;
    allocated when not supplied and returned either way.  The pivot is the
    largest magnitude, ties toward the lowest row (bit-identical to the
    reference, so ipiv matches exactly)."""
    return _getrf(m, n, C, D, True, ipiv, check, "getrf_pivot")

