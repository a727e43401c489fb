"""Batched conversions between dense and panel-major storage.

The reference's pack module (pack.py:45-82, 215-237) with a batch axis:

* ``pack_matrix(src, m, n, dst)``   column-major window -> panel window (kpack_cm)
* ``unpack_matrix(src, m, n, dst)`` panel window -> column-major window (kunpack_cm)
* ``gecp(m, n, A, B)``              panel -> panel window copy (kgecp)
* ``panel_from_array(arr)`` / ``panel_to_array(A, m, n)`` numpy/torch bridges

Column-major batches are :class:`ColBatch` (the ``ColMatrix`` analogue,
matstore.py:118-164): a float64 tensor ``[batch, lda*cols]`` where item
b's element (i, j) is ``data[b, i + j*lda]``.  All moves are bit-exact and
run as CUDA kernels through the C ABI.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .errors import DimensionError
from .matstore import PanelBatch, SubRef, allocate_panel_batch


class ColBatch:
    """``batch`` column-major m x n matrices with leading dimension lda."""

    __slots__ = ("batch", "rows", "cols", "lda", "data")

    def __init__(self, rows, cols, lda, data):
        if lda < rows:
            raise DimensionError(f"lda {lda} < rows {rows}")
        if data.dim() != 2 or data.shape[1] < lda * cols:
            raise DimensionError("column-major backing storage too small")
        if data.dtype != torch.float64 or data.stride(1) != 1:
            raise DimensionError("column-major storage must be float64 with unit inner stride")
        self.batch = data.shape[0]
        self.rows = rows
        self.cols = cols
        self.lda = lda
        self.data = data

    def __repr__(self):
        return f"ColBatch({self.batch} x {self.rows}x{self.cols}, lda={self.lda})"

    def ref(self, ai=0, aj=0):
        return SubRef(self, ai, aj)

    @property
    def device(self):
        return self.data.device

    @classmethod
    def from_array(cls, arr, device="cuda"):
        """[batch, m, n] array (numpy or torch) -> column-major batch."""
        t = torch.as_tensor(np.asarray(arr, dtype=np.float64) if not isinstance(arr, torch.Tensor) else arr,
                            dtype=torch.float64)
        if t.dim() != 3:
            raise DimensionError("expected a 3-d [batch, m, n] array")
        nb, m, n = t.shape
        lda = max(m, 1)
        data = t.transpose(1, 2).contiguous().reshape(nb, m * n).to(device)
        if m * n == 0:
            data = torch.zeros((nb, lda * n), dtype=torch.float64, device=device)
        return cls(m, n, lda, data)

    def to_array(self):
        """-> [batch, m, n] torch tensor (same device)."""
        nb = self.batch
        v = self.data[:, : self.lda * self.cols].reshape(nb, self.cols, self.lda)[:, :, : self.rows]
        return v.transpose(1, 2).contiguous()


def _panel_ref(x):
    if isinstance(x, PanelBatch):
        return x, 0, 0
    if isinstance(x, SubRef) and isinstance(x.mat, PanelBatch):
        return x.mat, x.ai, x.aj
    raise TypeError(f"expected a PanelBatch or a panel SubRef, got {type(x).__name__}")


def _col_ref(x):
    if isinstance(x, ColBatch):
        return x, 0, 0
    if isinstance(x, SubRef) and isinstance(x.mat, ColBatch):
        return x.mat, x.ai, x.aj
    raise TypeError(f"expected a ColBatch or a column-major SubRef, got {type(x).__name__}")


def _check_window(mat, ai, aj, m, n, what):
    # pack.py:36-42
    if m < 0 or n < 0:
        raise DimensionError(f"negative window size {m}x{n} for {what}")
    if ai + m > mat.rows or aj + n > mat.cols:
        raise DimensionError(
            f"{what} window ({ai}:{ai + m}, {aj}:{aj + n}) exceeds "
            f"{mat.rows}x{mat.cols} matrix")


def _dev_of(x):
    return x.device


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _same_batch(a, b):
    if a.batch != b.batch:
        raise DimensionError(f"batch sizes differ: {a.batch} vs {b.batch}")
    if a.device != b.device or a.device.type != "cuda":
        raise RuntimeError("pack/unpack run on one CUDA device (no CPU fallback)")


def pack_matrix(src, m, n, dst):
    """Copy every item's m x n column-major window into its panel window."""
    s, si, sj = _col_ref(src)
    d, di, dj = _panel_ref(dst)
    _check_window(s, si, sj, m, n, "pack source")
    _check_window(d, di, dj, m, n, "pack destination")
    _same_batch(s, d)
    if m == 0 or n == 0 or d.batch == 0:
        return
    dd = d.descriptor()
    base = s.data.data_ptr() + 8 * (si + sj * s.lda)
    with torch.cuda.device(_dev_of(d)):
        _native.call("pb_dpack_cm", m, n, ctypes.c_void_p(base), s.lda, s.data.stride(0), ctypes.byref(dd), di, dj,
                     _stream(d.device))


def unpack_matrix(src, m, n, dst):
    """Copy every item's m x n panel window into its column-major window."""
    s, si, sj = _panel_ref(src)
    d, di, dj = _col_ref(dst)
    _check_window(s, si, sj, m, n, "unpack source")
    _check_window(d, di, dj, m, n, "unpack destination")
    _same_batch(s, d)
    if m == 0 or n == 0 or s.batch == 0:
        return
    ds = s.descriptor()
    base = d.data.data_ptr() + 8 * (di + dj * d.lda)
    with torch.cuda.device(_dev_of(d)):
        _native.call("pb_dunpack_cm", m, n, ctypes.byref(ds), si, sj, ctypes.c_void_p(base), d.lda, d.data.stride(0),
                     _stream(s.device))


def gecp(m, n, A, B):
    """General panel-to-panel copy: B <- A over an m x n window, per item."""
    s, si, sj = _panel_ref(A)
    d, di, dj = _panel_ref(B)
    _check_window(s, si, sj, m, n, "copy source")
    _check_window(d, di, dj, m, n, "copy destination")
    if s.batch not in (d.batch, 1):
        raise DimensionError(f"batch sizes differ: {s.batch} vs {d.batch}")
    if m == 0 or n == 0 or d.batch == 0:
        return
    ds, dd = s.descriptor(d.batch), d.descriptor()
    with torch.cuda.device(_dev_of(d)):
        _native.call("pb_dgecp", m, n, ctypes.byref(ds), si, sj, ctypes.byref(dd), di, dj, _stream(d.device))


def pack_array_into(t, dst, di=0, dj=0):
    """Pack a device tensor t [batch, m, n] (any strides) into dst's window at (di, dj)."""
    d, di0, dj0 = _panel_ref(dst)
    di, dj = di + di0, dj + dj0
    nb, m, n = t.shape
    _check_window(d, di, dj, m, n, "pack destination")
    if nb != d.batch:
        raise DimensionError(f"batch sizes differ: {nb} vs {d.batch}")
    if m == 0 or n == 0 or nb == 0:
        return
    if t.dtype != torch.float64 or t.device != d.device:
        raise DimensionError("source must be a float64 tensor on the destination's device")
    dd = d.descriptor()
    with torch.cuda.device(_dev_of(d)):
        _native.call("pb_dpack", m, n, ctypes.c_void_p(t.data_ptr()), t.stride(1), t.stride(2), t.stride(0),
                     ctypes.byref(dd), di, dj, _stream(d.device))


def unpack_window(A, m, n, out=None):
    """Unpack every item's m x n window into a [batch, m, n] device tensor."""
    a, ai, aj = _panel_ref(A)
    _check_window(a, ai, aj, m, n, "unpack source")
    if out is None:
        out = torch.empty((a.batch, m, n), dtype=torch.float64, device=a.device)
    if m == 0 or n == 0 or a.batch == 0:
        return out
    da = a.descriptor()
    with torch.cuda.device(_dev_of(a)):
        _native.call("pb_dunpack", m, n, ctypes.byref(da), ai, aj, ctypes.c_void_p(out.data_ptr()), out.stride(1),
                     out.stride(2), out.stride(0), _stream(a.device))
    return out


def panel_from_array(arr, device="cuda"):
    """Pack a [batch, m, n] array (numpy or torch) into a fresh PanelBatch (pack.py:215-224)."""
    t = arr if isinstance(arr, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
    if t.dim() != 3:
        raise DimensionError("expected a 3-d [batch, m, n] array")
    t = t.to(device=device, dtype=torch.float64)
    nb, m, n = t.shape
    out = allocate_panel_batch(nb, m, n, device=t.device)
    pack_array_into(t, out)
    return out


def panel_to_array(A, m=None, n=None):
    """Unpack a panel window into a fresh [batch, m, n] tensor (pack.py:227-237)."""
    a, ai, aj = _panel_ref(A)
    if m is None:
        m = a.rows - ai
    if n is None:
        n = a.cols - aj
    return unpack_window(A, m, n)
