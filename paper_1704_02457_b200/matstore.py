"""Batched panel-major storage (device-resident, PyTorch-owned memory).

Mirrors the reference's storage layer (matstore.py:25-285) with a leading
batch axis:

* ``PS = 4`` rows per panel, ``ALIGN = 64`` bytes, and the same element
  offset ``(ai - ai%4)*cn + 4*aj + ai%4`` (matstore.py:37-45);
* an item's panel data is exactly the reference's: ``round_up(m,4) *
  round_up(n,4)`` doubles, panel p = rows 4p..4p+3, column j of a panel =
  32 contiguous bytes; ``diag_inv`` holds ``min(m,n)`` reciprocals;
* ``diag_lo/diag_hi`` record which diag_inv columns hold reciprocals from
  the latest diagonal-window factorization (matstore.py:88-91, 113-115),
  batch-uniformly.

Two batch layouts, both described by the same ABI descriptor
(``pb_dmat_batch``: ``pA``/``stride`` for the data, ``dA``/``dA_stride``
for the reciprocals, include/pb_b200.h):

``"split"`` (default, :func:`allocate_panel_batch`)
    a data plane ``data[batch, round_up(m,4)*cn]`` and a separate diag
    plane ``diag[batch, min(m,n)]``.  Consecutive items' panel data are
    back to back (an n = 4 item is exactly one 128-byte line), so the
    streaming kernels move no reciprocal slack with the data.
``"interleaved"`` (:func:`create_panel_batch` on one buffer)
    ``storage[batch, memsize/8]`` where item b is byte-for-byte the
    reference's ``create_panel_matrix`` region (data padded to 64 B, then
    diag_inv padded to 64 B, matstore.py:208-250), so a host copy of an
    item wraps zero-copy with the reference's own ``create_panel_matrix``.

:meth:`PanelBatch.item_storage` returns the reference byte layout for
either (a copy for ``split``).
"""
from __future__ import annotations

import torch

from ._native import DmatBatch
from .errors import DimensionError, MemoryLayoutError

PS = 4
ALIGN = 64
_ELEM = 8


def _round_up(x, to):
    return -(-x // to) * to


def element_offset(ai, aj, ps, sda):
    """Linear index of element (ai, aj) in a panel-major array (matstore.py:37-45)."""
    air = ai & (ps - 1)
    return (ai - air) * sda + aj * ps + air


def memsize_panel_matrix(m, n):
    """Bytes backing ONE m x n item in the reference layout: data + diag_inv,
    each 64-byte rounded (matstore.py:208-220)."""
    if m < 0 or n < 0:
        raise DimensionError(f"negative matrix size {m}x{n}")
    data_b = _round_up(m, PS) * _round_up(n, PS) * _ELEM
    diag_b = min(m, n) * _ELEM
    return _round_up(data_b, ALIGN) + _round_up(diag_b, ALIGN)


def memsize_panel_batch(batch, m, n):
    """Bytes of an interleaved batch (``batch`` reference-layout items)."""
    if batch < 0:
        raise DimensionError(f"negative batch {batch}")
    return batch * memsize_panel_matrix(m, n)


def panel_data_elems(m, n):
    """Doubles of one item's panel data (no padding): round_up(m,4)*round_up(n,4)."""
    if m < 0 or n < 0:
        raise DimensionError(f"negative matrix size {m}x{n}")
    return _round_up(m, PS) * _round_up(n, PS)


def memsize_split_batch(batch, m, n):
    """(data-plane bytes, diag-plane bytes) of a split batch."""
    if batch < 0:
        raise DimensionError(f"negative batch {batch}")
    return batch * panel_data_elems(m, n) * _ELEM, batch * min(m, n) * _ELEM


class SubRef:
    """A batch handle plus the (ai, aj) top-left corner of a window (matstore.py:48-65)."""

    __slots__ = ("mat", "ai", "aj")

    def __init__(self, mat, ai, aj):
        if ai < 0 or aj < 0:
            raise DimensionError(f"negative sub-matrix origin ({ai}, {aj})")
        self.mat = mat
        self.ai = ai
        self.aj = aj

    def __repr__(self):
        return f"SubRef({self.mat!r}, ai={self.ai}, aj={self.aj})"


class PanelBatch:
    """``batch`` independent m x n matrices in panel-major format.

    Build with :func:`allocate_panel_batch` or :func:`create_panel_batch`.
    ``storage`` is the interleaved buffer or, for a split batch, the data
    plane; ``diag_storage`` is the split batch's diag plane (None when
    interleaved).
    """

    __slots__ = ("batch", "rows", "cols", "panel_size", "panel_length", "storage", "diag_storage",
                 "memsize", "diag_lo", "diag_hi", "diag_info", "_diag_off", "_data_elems")

    def __init__(self, batch, rows, cols, storage, diag_storage=None):
        self.batch = batch
        self.rows = rows
        self.cols = cols
        self.panel_size = PS
        self.panel_length = _round_up(cols, PS)
        self.storage = storage
        self.diag_storage = diag_storage
        self.memsize = memsize_panel_matrix(rows, cols)
        self._data_elems = _round_up(rows, PS) * self.panel_length
        self._diag_off = _round_up(self._data_elems * _ELEM, ALIGN) // _ELEM
        self.diag_lo = 0
        self.diag_hi = 0
        # per-item status of that factorization when it ran unchecked
        # (check=False): items with diag_info[b] >= 0 failed, so their
        # reciprocals are not valid even inside [diag_lo, diag_hi)
        self.diag_info = None

    def __repr__(self):
        return (f"PanelBatch({self.batch} x {self.rows}x{self.cols}, cn={self.panel_length}, "
                f"layout={self.layout}, device={self.storage.device})")

    # views -----------------------------------------------------------------
    @property
    def layout(self):
        return "interleaved" if self.diag_storage is None else "split"

    @property
    def device(self):
        return self.storage.device

    @property
    def item_stride(self):
        """Doubles between consecutive items' panel data."""
        if self.batch > 1:
            return self.storage.stride(0)
        return self._data_elems if self.diag_storage is not None else self.memsize // _ELEM

    @property
    def diag_stride(self):
        """Doubles between consecutive items' diag_inv."""
        if self.diag_storage is None:
            return self.item_stride
        return self.diag_storage.stride(0) if self.batch > 1 else min(self.rows, self.cols)

    @property
    def data(self):
        """[batch, round_up(m,4)*cn] panel data (a view)."""
        return self.storage[:, : self._data_elems]

    @property
    def diag_inv(self):
        """[batch, min(m,n)] reciprocals written by factorizations (a view)."""
        dn = min(self.rows, self.cols)
        if self.diag_storage is not None:
            return self.diag_storage[:, :dn]
        return self.storage[:, self._diag_off: self._diag_off + dn]

    def diag_vector(self):
        """diag_inv as a :class:`DenseVectorBatch` view (the reference's
        diag_inv plays the blasfeo_dvec role)."""
        return DenseVectorBatch(self.batch, min(self.rows, self.cols), self.diag_inv)

    def panels(self):
        """[batch, pm, cn, 4] view: panel p, column j, row-in-panel r."""
        pm = _round_up(self.rows, PS) // PS
        return self.data.view(self.batch, pm, self.panel_length, PS)

    def ref(self, ai=0, aj=0):
        return SubRef(self, ai, aj)

    def diag_inv_valid(self, ai, n):
        """True if diag_inv covers columns [ai, ai+n) from a factorization
        (for every item whose ``diag_info`` does not say it failed)."""
        return self.diag_lo <= ai and ai + n <= self.diag_hi

    def _check_elem(self, b, ai, aj):
        if not (0 <= b < self.batch and 0 <= ai < self.rows and 0 <= aj < self.cols):
            raise DimensionError(
                f"element ({ai}, {aj}) of item {b} outside {self.batch} x {self.rows}x{self.cols} batch")

    def get(self, b, ai, aj):
        """Element (ai, aj) of item b (matstore.py:100-107; one host sync)."""
        self._check_elem(b, ai, aj)
        return float(self.storage[b, element_offset(ai, aj, PS, self.panel_length)])

    def set(self, b, ai, aj, v):
        """Write element (ai, aj) of item b (matstore.py:109-111)."""
        self._check_elem(b, ai, aj)
        self.storage[b, element_offset(ai, aj, PS, self.panel_length)] = v

    def item_storage(self):
        """[batch, memsize/8] float64 in the reference's per-item byte layout
        (the interleaved buffer itself, or an assembled copy of a split batch;
        padding slots of a copy are zero)."""
        if self.diag_storage is None:
            return self.storage
        out = torch.zeros((self.batch, self.memsize // _ELEM), dtype=torch.float64, device=self.device)
        out[:, : self._data_elems] = self.data
        dn = min(self.rows, self.cols)
        out[:, self._diag_off: self._diag_off + dn] = self.diag_inv
        return out

    def item_bytes(self, b):
        """Host copy of item b's storage in the reference byte layout (numpy uint8)."""
        return self.item_storage()[b].detach().cpu().numpy().view("uint8")

    def shard(self, lo, hi):
        """Items [lo, hi) as a PanelBatch view (no copy; diag validity kept)."""
        if not 0 <= lo <= hi <= self.batch:
            raise DimensionError(f"shard [{lo}, {hi}) outside batch {self.batch}")
        v = PanelBatch(hi - lo, self.rows, self.cols, self.storage[lo:hi],
                       None if self.diag_storage is None else self.diag_storage[lo:hi])
        v.diag_lo, v.diag_hi = self.diag_lo, self.diag_hi
        v.diag_info = None if self.diag_info is None else self.diag_info[lo:hi]
        return v

    # ABI descriptor ---------------------------------------------------------
    def descriptor(self, batch=None):
        """``pb_dmat_batch`` for this storage.  ``batch`` > self.batch == 1
        broadcasts this single matrix (stride 0) to a larger batch."""
        base = self.storage.data_ptr()
        if self.diag_storage is None:
            dbase = base + self._diag_off * _ELEM
        else:
            dbase = self.diag_storage.data_ptr() if min(self.rows, self.cols) > 0 else 0
        nb = self.batch if batch is None else batch
        stride, dstride = self.item_stride, self.diag_stride
        if nb != self.batch:
            if self.batch != 1:
                raise DimensionError(f"batch {self.batch} cannot broadcast to {nb}")
            stride = dstride = 0
        return DmatBatch(base, dbase, self.rows, self.cols, self.panel_length, nb, stride, dstride)


def _check_tensor(memory, need_bytes, what):
    if not isinstance(memory, torch.Tensor) or memory.dtype != torch.float64:
        raise MemoryLayoutError(f"{what} must be a float64 torch tensor")
    if not memory.is_contiguous():
        raise MemoryLayoutError(f"{what} must be contiguous")
    have = memory.numel() * _ELEM
    if have < need_bytes:
        raise MemoryLayoutError(f"{what} holds {have} bytes, {need_bytes} required")
    if need_bytes and memory.data_ptr() % ALIGN != 0:
        raise MemoryLayoutError(f"{what} must be {ALIGN}-byte aligned (address {memory.data_ptr():#x})")


def create_panel_batch(batch, m, n, memory, diag=None):
    """Wrap existing tensors as a PanelBatch without touching their contents.

    ``diag is None``: ``memory`` holds ``batch`` reference-layout items
    back to back (interleaved, ``memsize_panel_batch(batch, m, n)`` bytes,
    matstore.py:229-250).  Otherwise ``memory`` is the data plane
    (``batch * round_up(m,4)*round_up(n,4)`` doubles) and ``diag`` the
    diag plane (``batch * min(m,n)`` doubles): a split batch.  Float64,
    contiguous, 64-byte aligned.
    """
    if batch < 0:
        raise DimensionError(f"negative batch {batch}")
    if diag is None:
        need = memsize_panel_batch(batch, m, n)
        if isinstance(memory, torch.Tensor) and memory.dtype == torch.float64 and memory.is_contiguous() \
                and memory.numel() * _ELEM < need:
            raise MemoryLayoutError(
                f"memory region holds {memory.numel() * _ELEM} bytes, {need} required for "
                f"{batch} x {m}x{n} panel matrices")
        _check_tensor(memory, need, "memory region")
        per = memsize_panel_matrix(m, n) // _ELEM
        return PanelBatch(batch, m, n, memory.reshape(-1)[: batch * per].view(batch, per))
    dbytes, gbytes = memsize_split_batch(batch, m, n)
    _check_tensor(memory, dbytes, "data plane")
    _check_tensor(diag, gbytes, "diag plane")
    if memory.device != diag.device:
        raise MemoryLayoutError("data and diag planes live on different devices")
    per, dn = panel_data_elems(m, n), min(m, n)
    return PanelBatch(batch, m, n, memory.reshape(-1)[: batch * per].view(batch, per),
                      diag.reshape(-1)[: batch * dn].view(batch, dn))


def allocate_panel_batch(batch, m, n, device="cuda", zero=False, layout="split"):
    """Fresh storage (uninitialized unless ``zero``), like allocate_panel_matrix.
    ``layout`` is ``"split"`` (default) or ``"interleaved"`` (reference item layout)."""
    if batch < 0:
        raise DimensionError(f"negative batch {batch}")
    if m < 0 or n < 0:
        raise DimensionError(f"negative matrix size {m}x{n}")
    mk = torch.zeros if zero else torch.empty
    if layout == "interleaved":
        per = memsize_panel_matrix(m, n) // _ELEM
        storage = mk((batch, max(per, 1)), dtype=torch.float64, device=device)[:, :per]
        return PanelBatch(batch, m, n, storage)
    if layout != "split":
        raise ValueError(f"unknown layout {layout!r}")
    per, dn = panel_data_elems(m, n), min(m, n)
    data = mk((batch, max(per, 1)), dtype=torch.float64, device=device)[:, :per]
    diag = mk((batch, max(dn, 1)), dtype=torch.float64, device=device)[:, :dn]
    return PanelBatch(batch, m, n, data, diag)


# ---------------------------------------------------------------------------
# vectors (blasfeo_dvec / DenseVector, matstore.py:167-192, 261-285)


def memsize_vector(m):
    """Bytes backing one length-m vector: round_up(8m, 64) (matstore.py:261-264)."""
    if m < 0:
        raise DimensionError(f"negative vector length {m}")
    return _round_up(m * _ELEM, ALIGN)


class DenseVectorBatch:
    """``batch`` unit-stride float64 vectors of length ``len``: the
    reference's DenseVector (matstore.py:167-192) with a batch axis.
    ``data`` is ``[batch, >= len]`` with unit inner stride; item b's
    element i is ``data[b, i]``."""

    __slots__ = ("batch", "len", "data", "memsize")

    def __init__(self, batch, length, data):
        self.batch = batch
        self.len = length
        self.data = data
        self.memsize = memsize_vector(length)

    def __repr__(self):
        return f"DenseVectorBatch({self.batch} x len={self.len}, device={self.data.device})"

    @property
    def device(self):
        return self.data.device

    @property
    def stride(self):
        return self.data.stride(0) if self.batch > 1 else self.memsize // _ELEM

    def _check(self, b, i):
        if not (0 <= b < self.batch and 0 <= i < self.len):
            raise DimensionError(f"element {i} of item {b} outside {self.batch} x length-{self.len} vectors")

    def get(self, b, i):
        self._check(b, i)
        return float(self.data[b, i])

    def set(self, b, i, v):
        self._check(b, i)
        self.data[b, i] = v

    def to_array(self):
        """[batch, len] copy (matstore.py:191-192)."""
        return self.data[:, : self.len].clone()


def create_vector_batch(batch, m, memory):
    """Wrap ``memory`` (float64, contiguous, 64-byte aligned, at least
    ``batch * memsize_vector(m)`` bytes) as ``batch`` length-m vectors, one
    per ``memsize_vector(m)`` bytes, contents untouched (matstore.py:267-278)."""
    if batch < 0:
        raise DimensionError(f"negative batch {batch}")
    per = memsize_vector(m)
    _check_tensor(memory, batch * per, "memory region")
    return DenseVectorBatch(batch, m, memory.reshape(-1)[: batch * per // _ELEM].view(batch, per // _ELEM))


def allocate_vector_batch(batch, m, device="cuda", zero=False):
    """Fresh (uninitialized unless ``zero``) batch of length-m vectors (matstore.py:281-285)."""
    if batch < 0:
        raise DimensionError(f"negative batch {batch}")
    per = memsize_vector(m) // _ELEM
    mk = torch.zeros if zero else torch.empty
    return DenseVectorBatch(batch, m, mk((batch, max(per, 1)), dtype=torch.float64, device=device)[:, :per])
