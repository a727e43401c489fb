"""TEST INFRASTRUCTURE ONLY -- the CPU parity oracle.

Python side of the oracle: ctypes wrapper around ``libpb_oracle.so`` (the C
restatement in pb_oracle.c of the reference's hot path,
/root/reference/pkg/src/panelblas/_backend/ccore.pyx) plus the routine-level
semantics of the reference's level3 wrappers (level3.py:81-350):
bounds/no-op rules, _recip_diag reuse (level3.py:160-177), the unaligned
destination scratch path of potrf (level3.py:337-342) and bad-pivot
statuses.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may use this module, and only as the checker or the
timed CPU baseline -- never as the product path.

Host batches use the product's byte layout (matstore.PanelBatch): a
float64 array ``storage[batch, memsize/8]`` per operand, data first, then
diag_inv at a 64-byte boundary, exactly the reference's
create_panel_matrix layout (matstore.py:208-250).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libpb_oracle.so")
PS = 4
_lib = None


def build():
    """Compile the restatement (gcc, no FMA contraction)."""
    src = os.path.join(HERE, "pb_oracle.c")
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(src):
        return LIB
    subprocess.run(["make", "-s", "-C", HERE, "libpb_oracle.so"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB)
        _lib.po_element_offset.restype = ctypes.c_int64
        _lib.po_memsize.restype = ctypes.c_int64
        _lib.po_potrf_l.restype = ctypes.c_int
        _lib.po_syrk_potrf_ln.restype = ctypes.c_int
        _lib.po_getrf.restype = ctypes.c_int
    return _lib


def _ru(x, to):
    return -(-x // to) * to


def memsize(m, n):
    return _ru(_ru(m, 4) * _ru(n, 4) * 8, 64) + _ru(min(m, n) * 8, 64)


class HostBatch:
    """Host twin of PanelBatch: storage [batch, memsize/8] float64 (numpy)."""

    def __init__(self, batch, m, n, storage=None):
        self.batch, self.rows, self.cols = batch, m, n
        self.cn = _ru(n, 4)
        self.per = memsize(m, n) // 8
        self.diag_off = _ru(_ru(m, 4) * self.cn * 8, 64) // 8
        if storage is None:
            storage = np.zeros((batch, max(self.per, 1)), dtype=np.float64)
        assert storage.dtype == np.float64 and storage.shape[0] == batch
        self.storage = np.ascontiguousarray(storage)
        self.diag_lo = self.diag_hi = 0

    def copy(self):
        h = HostBatch(self.batch, self.rows, self.cols, self.storage.copy())
        h.diag_lo, h.diag_hi = self.diag_lo, self.diag_hi
        return h

    def diag_inv_valid(self, ai, n):
        return self.diag_lo <= ai and ai + n <= self.diag_hi

    def ptr(self, b=0):
        return ctypes.c_void_p(self.storage.ctypes.data + 8 * b * self.storage.shape[1])

    def dptr(self, b=0):
        return ctypes.c_void_p(self.storage.ctypes.data + 8 * (b * self.storage.shape[1] + self.diag_off))

    @property
    def stride(self):
        return self.storage.shape[1]

    def get(self, b, i, j):
        return self.storage[b, element_offset(i, j, self.cn)]

    def window(self, ai, aj, m, n):
        """-> [batch, m, n] dense copy of a window."""
        out = np.empty((self.batch, m, n))
        for i in range(m):
            for j in range(n):
                out[:, i, j] = self.storage[:, element_offset(ai + i, aj + j, self.cn)]
        return out

    def set_window(self, ai, aj, arr):
        arr = np.asarray(arr, dtype=np.float64)
        nb, m, n = arr.shape
        for i in range(m):
            for j in range(n):
                self.storage[:, element_offset(ai + i, aj + j, self.cn)] = arr[:, i, j]


def element_offset(i, j, cn):
    return (i - (i & 3)) * cn + 4 * j + (i & 3)


_L = ctypes.c_int64
_D = ctypes.c_double


def gemm_nt(m, n, k, alpha, A, ai, aj, B, bi, bj, beta, C, ci, cj, D, di, dj):
    """level3.gemm_nt semantics over a batch (level3.py:81-98)."""
    if m == 0 or n == 0:
        return
    lib().po_gemm_nt_batch(_L(D.batch), _L(m), _L(n), _L(k), _D(alpha),
                           A.ptr(), _L(ai), _L(aj), _L(A.cn), _L(A.stride if A.batch > 1 else 0),
                           B.ptr(), _L(bi), _L(bj), _L(B.cn), _L(B.stride if B.batch > 1 else 0), _D(beta),
                           C.ptr(), _L(ci), _L(cj), _L(C.cn), _L(C.stride if C.batch > 1 else 0),
                           D.ptr(), _L(di), _L(dj), _L(D.cn), _L(D.stride))


def syrk_ln(m, k, alpha, A, ai, aj, B, bi, bj, beta, C, ci, cj, D, di, dj):
    """level3.syrk_ln semantics over a batch (level3.py:120-137)."""
    if m == 0:
        return
    lib().po_syrk_ln_batch(_L(D.batch), _L(m), _L(k), _D(alpha),
                           A.ptr(), _L(ai), _L(aj), _L(A.cn), _L(A.stride if A.batch > 1 else 0),
                           B.ptr(), _L(bi), _L(bj), _L(B.cn), _L(B.stride if B.batch > 1 else 0), _D(beta),
                           C.ptr(), _L(ci), _L(cj), _L(C.cn), _L(C.stride if C.batch > 1 else 0),
                           D.ptr(), _L(di), _L(dj), _L(D.cn), _L(D.stride))


def trsm_rltn(m, n, alpha, A, ai, aj, B, bi, bj, D, di, dj):
    """level3.trsm_rltn semantics (level3.py:220-244) -> info[batch].

    Reciprocals per level3._recip_diag: reuse A's diag_inv if the window is
    on the freshly factored diagonal, else 1/A[j,j] with the first zero
    pivot reported in info and the item left untouched."""
    info = np.full(D.batch, -1, dtype=np.int32)
    if m == 0 or n == 0:
        return info
    A_stride = A.stride if A.batch > 1 else 0
    B_stride = B.stride if B.batch > 1 else 0
    if ai == aj and A.diag_inv_valid(aj, n):
        lib().po_trsm_rltn_batch(_L(D.batch), _L(m), _L(n), _D(alpha),
                                 A.ptr(), _L(ai), _L(aj), _L(A.cn), _L(A_stride), ctypes.c_int(0),
                                 B.ptr(), _L(bi), _L(bj), _L(B.cn), _L(B_stride),
                                 D.ptr(), _L(di), _L(dj), _L(D.cn), _L(D.stride),
                                 A.dptr(), _L(aj), _L(A_stride))
        return info
    for b in range(D.batch):
        ab = b if A.batch > 1 else 0
        bb = b if B.batch > 1 else 0
        diag = np.array([A.get(ab, ai + j, aj + j) for j in range(n)])
        zero = np.nonzero(diag == 0.0)[0]
        if zero.size:
            info[b] = int(zero[0])
            continue
        dinv = 1.0 / diag
        lib().po_trsm_rltn(_L(m), _L(n), _D(alpha), A.ptr(ab), _L(ai), _L(aj), _L(A.cn), ctypes.c_int(0),
                           B.ptr(bb), _L(bi), _L(bj), _L(B.cn), D.ptr(b), _L(di), _L(dj), _L(D.cn),
                           dinv.ctypes.data_as(ctypes.c_void_p), _L(0))
    return info


def potrf_l(m, C, ci, cj, D, di, dj, n=None):
    """level3.potrf_l semantics (level3.py:319-350) -> info[batch].

    Unaligned destinations (di % 4 != 0) factor into a scratch matrix and
    copy the lower trapezoid only on success, like the reference."""
    if n is None:
        n = m
    info = np.full(D.batch, -1, dtype=np.int32)
    if n == 0:
        return info
    C_stride = C.stride if C.batch > 1 else 0
    if di % 4 == 0:
        lib().po_potrf_l_batch(_L(D.batch), _L(m), _L(n), C.ptr(), _L(ci), _L(cj), _L(C.cn), _L(C_stride),
                               D.ptr(), _L(di), _L(dj), _L(D.cn), _L(D.stride), D.dptr(), _L(dj), _L(D.stride),
                               info.ctypes.data_as(ctypes.c_void_p))
    else:
        for b in range(D.batch):
            cb = b if C.batch > 1 else 0
            s = HostBatch(1, m, n)
            st = lib().po_potrf_l(_L(m), _L(n), C.ptr(cb), _L(ci), _L(cj), _L(C.cn), s.ptr(), _L(0), _L(0),
                                  _L(s.cn), D.dptr(b), _L(dj))
            info[b] = st
            if st < 0:
                for j in range(n):
                    for i in range(j, m):
                        D.storage[b, element_offset(di + i, dj + j, D.cn)] = s.get(0, i, j)
    ok = bool(np.all(info < 0))
    if ok and di == dj:
        D.diag_lo, D.diag_hi = dj, dj + n
    else:
        D.diag_lo = D.diag_hi = 0
    return info


def _item(X, b):
    return X.ptr(b if X.batch > 1 else 0)


def gemm_nn(m, n, k, alpha, A, ai, aj, B, bi, bj, beta, C, ci, cj, D, di, dj):
    """level3.gemm_nn semantics (level3.py:101-117) per item."""
    if m == 0 or n == 0:
        return
    for b in range(D.batch):
        lib().po_gemm_nn(_L(m), _L(n), _L(k), _D(alpha), _item(A, b), _L(ai), _L(aj), _L(A.cn),
                         _item(B, b), _L(bi), _L(bj), _L(B.cn), _D(beta), _item(C, b), _L(ci), _L(cj), _L(C.cn),
                         D.ptr(b), _L(di), _L(dj), _L(D.cn))


def trmm_rlnn(m, n, alpha, A, ai, aj, B, bi, bj, D, di, dj):
    """level3.trmm_rlnn (level3.py:140-153): D = alpha * B * A, A lower n x n."""
    if m == 0 or n == 0:
        return
    for b in range(D.batch):
        lib().po_trmm_rlnn(_L(m), _L(n), _D(alpha), _item(A, b), _L(ai), _L(aj), _L(A.cn),
                           _item(B, b), _L(bi), _L(bj), _L(B.cn), D.ptr(b), _L(di), _L(dj), _L(D.cn))


def syrk_potrf_ln(m, k, A, ai, aj, B, bi, bj, C, ci, cj, D, di, dj, n=None):
    """level3.syrk_potrf_ln (level3.py:353-391) -> info[batch]; unaligned
    destinations go through a scratch matrix copied only on success."""
    if n is None:
        n = m
    info = np.full(D.batch, -1, dtype=np.int32)
    if n == 0:
        return info
    for b in range(D.batch):
        args = (_L(m), _L(n), _L(k), _item(A, b), _L(ai), _L(aj), _L(A.cn), _item(B, b), _L(bi), _L(bj), _L(B.cn),
                _item(C, b), _L(ci), _L(cj), _L(C.cn))
        if di % 4 == 0:
            info[b] = lib().po_syrk_potrf_ln(*args, D.ptr(b), _L(di), _L(dj), _L(D.cn), D.dptr(b), _L(dj))
        else:
            s = HostBatch(1, m, n)
            st = lib().po_syrk_potrf_ln(*args, s.ptr(), _L(0), _L(0), _L(s.cn), D.dptr(b), _L(dj))
            info[b] = st
            if st < 0:
                for j in range(n):
                    for i in range(j, m):
                        D.storage[b, element_offset(di + i, dj + j, D.cn)] = s.get(0, i, j)
    ok = bool(np.all(info < 0))
    if ok and di == dj:
        D.diag_lo, D.diag_hi = dj, dj + n
    else:
        D.diag_lo = D.diag_hi = 0
    return info


def getrf(m, n, C, ci, cj, D, di, dj, pivot, ipiv=None):
    """level3._getrf semantics (level3.py:431-446) per item -> (info[batch], ipiv).

    D = copy of C's window (skipped when D is C at the same origin), then the
    in-place LU (po_getrf).  An unaligned destination (di % 4) is factored
    in a scratch matrix and copied only on success (the reference raises
    before its final gecp, so D stays untouched; diag_inv is written either
    way).  ipiv[b, j0 + c] is filled for completed panels only."""
    mn = min(m, n)
    info = np.full(D.batch, -1, dtype=np.int32)
    if ipiv is None:
        ipiv = np.zeros((D.batch, max(mn, 1)), dtype=np.int64)
    if mn == 0:
        return info, ipiv
    same = C is D and ci == di and cj == dj
    for b in range(D.batch):
        piv = np.ascontiguousarray(ipiv[b])
        if di % 4 == 0:
            if not same:
                lib().po_gecp(_L(m), _L(n), _item(C, b), _L(ci), _L(cj), _L(C.cn), D.ptr(b), _L(di), _L(dj), _L(D.cn))
            st = lib().po_getrf(_L(m), _L(n), ctypes.c_int(int(pivot)), D.ptr(b), _L(di), _L(dj), _L(D.cn),
                                D.dptr(b), _L(dj), piv.ctypes.data_as(ctypes.c_void_p))
        else:
            s = HostBatch(1, m, n)
            lib().po_gecp(_L(m), _L(n), _item(C, b), _L(ci), _L(cj), _L(C.cn), s.ptr(), _L(0), _L(0), _L(s.cn))
            st = lib().po_getrf(_L(m), _L(n), ctypes.c_int(int(pivot)), s.ptr(), _L(0), _L(0), _L(s.cn),
                                D.dptr(b), _L(dj), piv.ctypes.data_as(ctypes.c_void_p))
            if st < 0:
                lib().po_gecp(_L(m), _L(n), s.ptr(), _L(0), _L(0), _L(s.cn), D.ptr(b), _L(di), _L(dj), _L(D.cn))
        ipiv[b] = piv
        info[b] = st
    if bool(np.all(info < 0)) and di == dj:
        D.diag_lo, D.diag_hi = dj, dj + mn
    else:
        D.diag_lo = D.diag_hi = 0
    return info, ipiv


def pack_cm(m, n, S, lds, s_stride, D, di, dj):
    """kpack_cm over a batch: S is a flat float64 array."""
    lib().po_pack_cm_batch(_L(D.batch), _L(m), _L(n), S.ctypes.data_as(ctypes.c_void_p), _L(lds), _L(s_stride),
                           D.ptr(), _L(di), _L(dj), _L(D.cn), _L(D.stride))


def unpack_cm(m, n, S, si, sj, Dcm, ldd, d_stride):
    lib().po_unpack_cm_batch(_L(S.batch), _L(m), _L(n), S.ptr(), _L(si), _L(sj), _L(S.cn), _L(S.stride),
                             Dcm.ctypes.data_as(ctypes.c_void_p), _L(ldd), _L(d_stride))


def gecp(m, n, S, si, sj, D, di, dj):
    lib().po_gecp_batch(_L(D.batch), _L(m), _L(n), S.ptr(), _L(si), _L(sj), _L(S.cn),
                        _L(S.stride if S.batch > 1 else 0), D.ptr(), _L(di), _L(dj), _L(D.cn), _L(D.stride))


def rel_fro(got, want):
    """Relative Frobenius error ||got-want||_F / ||want||_F (north_star tolerance metric)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want)
    num = np.linalg.norm(got - want)
    return num / den if den > 0 else num


def tol(n):
    """North-star floating-point tolerance: 50 * n * eps_fp64."""
    return 50.0 * max(n, 1) * np.finfo(np.float64).eps
