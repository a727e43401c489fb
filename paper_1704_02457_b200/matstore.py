"""Batched panel-major storage (device-resident, PyTorch-owned memory).

Mirrors the reference's storage layer (matstore.py:25-258) with a leading
batch axis:

* ``PS = 4`` rows per panel, ``ALIGN = 64`` bytes, and the same element
  offset ``(ai - ai%4)*cn + 4*aj + ai%4`` (matstore.py:37-45);
* every batch item uses exactly the reference's ``create_panel_matrix``
  byte layout: ``round_up(m,4)*round_up(n,4)`` doubles of panel data,
  padded to 64 bytes, then ``min(m,n)`` doubles of ``diag_inv`` padded to
  64 bytes (matstore.py:208-250).  A host copy of item b can therefore be
  wrapped zero-copy by the reference's ``create_panel_matrix(m, n, buf)``;
* the batch is one ``torch.float64`` tensor ``storage[batch, memsize/8]``
  (``data``, ``diag_inv`` and ``panels()`` are views of it), so items are
  64-byte aligned and an item's row panel is one contiguous run;
* ``diag_lo/diag_hi`` record which diag_inv columns hold reciprocals from
  the latest diagonal-window factorization (matstore.py:88-91, 113-115),
  batch-uniformly.
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
    """Bytes backing ONE m x n item: data + diag_inv, each 64-byte rounded."""
    if m < 0 or n < 0:
        raise DimensionError(f"negative matrix size {m}x{n}")
    data_b = _round_up(m, PS) * _round_up(n, PS) * _ELEM
    diag_b = min(m, n) * _ELEM
    return _round_up(data_b, ALIGN) + _round_up(diag_b, ALIGN)


def memsize_panel_batch(batch, m, n):
    if batch < 0:
        raise DimensionError(f"negative batch {batch}")
    return batch * memsize_panel_matrix(m, n)


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
    """

    __slots__ = ("batch", "rows", "cols", "panel_size", "panel_length", "storage",
                 "memsize", "diag_lo", "diag_hi", "_diag_off")

    def __init__(self, batch, rows, cols, storage):
        self.batch = batch
        self.rows = rows
        self.cols = cols
        self.panel_size = PS
        self.panel_length = _round_up(cols, PS)
        self.storage = storage  # [batch, memsize/8] float64
        self.memsize = memsize_panel_matrix(rows, cols)
        self._diag_off = _round_up(_round_up(rows, PS) * self.panel_length * _ELEM, ALIGN) // _ELEM
        self.diag_lo = 0
        self.diag_hi = 0

    def __repr__(self):
        return (f"PanelBatch({self.batch} x {self.rows}x{self.cols}, cn={self.panel_length}, "
                f"device={self.storage.device})")

    # views -----------------------------------------------------------------
    @property
    def device(self):
        return self.storage.device

    @property
    def item_stride(self):
        return self.storage.stride(0) if self.batch > 1 else self.memsize // _ELEM

    @property
    def data(self):
        """[batch, round_up(m,4)*cn] panel data (a view)."""
        return self.storage[:, : _round_up(self.rows, PS) * self.panel_length]

    @property
    def diag_inv(self):
        """[batch, min(m,n)] reciprocals written by factorizations (a view)."""
        return self.storage[:, self._diag_off: self._diag_off + min(self.rows, self.cols)]

    def panels(self):
        """[batch, pm, cn, 4] view: panel p, column j, row-in-panel r."""
        pm = _round_up(self.rows, PS) // PS
        return self.data.view(self.batch, pm, self.panel_length, PS)

    def ref(self, ai=0, aj=0):
        return SubRef(self, ai, aj)

    def diag_inv_valid(self, ai, n):
        """True if diag_inv covers columns [ai, ai+n) from a factorization."""
        return self.diag_lo <= ai and ai + n <= self.diag_hi

    def item_bytes(self, b):
        """Host copy of item b's storage in the reference byte layout (numpy uint8)."""
        return self.storage[b].detach().cpu().numpy().view("uint8")

    # ABI descriptor ---------------------------------------------------------
    def descriptor(self, batch=None):
        """``pb_dmat_batch`` for this storage.  ``batch`` > self.batch == 1
        broadcasts this single matrix (stride 0) to a larger batch."""
        st = self.storage
        base = st.data_ptr()
        nb = self.batch if batch is None else batch
        stride = self.item_stride
        if nb != self.batch:
            if self.batch != 1:
                raise DimensionError(f"batch {self.batch} cannot broadcast to {nb}")
            stride = 0
        return DmatBatch(base, base + self._diag_off * _ELEM, self.rows, self.cols,
                         self.panel_length, nb, stride, self.item_stride if stride else 0)


def create_panel_batch(batch, m, n, memory):
    """Wrap an existing tensor as a PanelBatch without touching its contents.

    ``memory`` must be a float64 tensor (any shape, contiguous) holding at
    least ``memsize_panel_batch(batch, m, n)`` bytes, 64-byte aligned
    (matstore.py:229-250).
    """
    need = memsize_panel_batch(batch, m, n)
    if not isinstance(memory, torch.Tensor) or memory.dtype != torch.float64:
        raise MemoryLayoutError("memory must be a float64 torch tensor")
    if not memory.is_contiguous():
        raise MemoryLayoutError("memory must be contiguous")
    have = memory.numel() * _ELEM
    if have < need:
        raise MemoryLayoutError(
            f"memory region holds {have} bytes, {need} required for {batch} x {m}x{n} panel matrices")
    if need and memory.data_ptr() % ALIGN != 0:
        raise MemoryLayoutError(f"memory region must be {ALIGN}-byte aligned (address {memory.data_ptr():#x})")
    per = memsize_panel_matrix(m, n) // _ELEM
    storage = memory.reshape(-1)[: batch * per].view(batch, per)
    return PanelBatch(batch, m, n, storage)


def allocate_panel_batch(batch, m, n, device="cuda", zero=False):
    """Fresh storage (uninitialized unless ``zero``), like allocate_panel_matrix."""
    per = memsize_panel_matrix(m, n) // _ELEM
    if batch < 0:
        raise DimensionError(f"negative batch {batch}")
    mk = torch.zeros if zero else torch.empty
    storage = mk((batch, max(per, 1)), dtype=torch.float64, device=device)[:, :per]
    return PanelBatch(batch, m, n, storage)
