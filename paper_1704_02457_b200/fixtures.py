"""Plain-text fixture I/O: the reference's matrix and
optimal-control fixture formats, for batches.

* Matrix fixture (matstore.py:297-321): first line ``"m n"``, then m rows of
  n values printed with ``%.17g`` (so a round trip is bit-exact).
  ``write_fixture`` writes one item's window of a :class:`PanelBatch`,
  ``read_fixture`` returns a batch-1 :class:`PanelBatch` (the reference
  returns a ColMatrix; the values are the same).
* OCP fixture (apps.py:318-365): header ``"nx nu N"``, then per stage the
  arrays A, B, Q, R, S in the matrix format, then P_N.
* ``dump_failures`` writes the input window of every item whose ``info`` is
  a failing pivot -- the failing-item dumps SURVEY §5 suggests, readable by
  the reference's own ``read_fixture``.

Host-side text I/O only: device batches are copied to the host first.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from .errors import DimensionError
from .matstore import PS, PanelBatch, allocate_panel_batch


def _write_array(fh, arr):
    # apps.py:349-354 / matstore.py:301-307 (same layout)
    m, n = arr.shape
    fh.write(f"{m} {n}\n")
    for i in range(m):
        fh.write(" ".join(f"{float(arr[i, j]):.17g}" for j in range(n)))
        fh.write("\n")


def _read_array(fh):
    # apps.py:357-365 / matstore.py:310-321
    m, n = (int(t) for t in fh.readline().split())
    out = np.empty((m, n))
    for i in range(m):
        row = fh.readline().split()
        if len(row) != n:
            raise ValueError(f"fixture row {i} has {len(row)} values, expected {n}")
        out[i] = [float(t) for t in row]
    return out


def _offsets(ai, aj, m, n, cn):
    # element_offset (matstore.py:37-45) for every element of the window
    i = np.arange(ai, ai + m)[:, None]
    j = np.arange(aj, aj + n)[None, :]
    return (i - (i % PS)) * cn + PS * j + (i % PS)


def _window(mat, b, ai, aj, m, n):
    if not isinstance(mat, PanelBatch):
        raise TypeError("expected a PanelBatch")
    m = mat.rows - ai if m is None else m
    n = mat.cols - aj if n is None else n
    if ai < 0 or aj < 0 or ai + m > mat.rows or aj + n > mat.cols or not 0 <= b < mat.batch:
        raise DimensionError(f"fixture window ({ai}:{ai + m}, {aj}:{aj + n}) of item {b} out of bounds")
    row = mat.data[b].detach().cpu().numpy()
    return row[_offsets(ai, aj, m, n, mat.panel_length)]


def write_fixture(path, mat, b=0, ai=0, aj=0, m=None, n=None):
    """Write item ``b``'s window (default: the whole matrix) as a matrix fixture."""
    arr = _window(mat, b, ai, aj, m, n)
    with open(path, "w") as fh:
        _write_array(fh, arr)


def read_fixture(path, device="cuda"):
    """Read a matrix fixture into a batch-1 PanelBatch on ``device``."""
    with open(path) as fh:
        arr = _read_array(fh)
    m, n = arr.shape
    out = allocate_panel_batch(1, m, n, device="cpu", zero=True)
    row = out.data[0].numpy()
    row[_offsets(0, 0, m, n, out.panel_length)] = arr
    if device == "cpu":
        return out
    return PanelBatch(1, m, n, out.storage.to(device), out.diag_storage.to(device))


def write_ocp_fixture(path, nx, nu, stages, P):
    """stages: N tuples (A, B, Q, R, S) of arrays (nx x nx, nx x nu, nx x nx, nu x nu, nu x nx)."""
    with open(path, "w") as fh:
        fh.write(f"{nx} {nu} {len(stages)}\n")
        for st in stages:
            if len(st) != 5:
                raise DimensionError("a stage is (A, B, Q, R, S)")
            for arr in st:
                _write_array(fh, np.asarray(arr, dtype=np.float64))
        _write_array(fh, np.asarray(P, dtype=np.float64))


def read_ocp_fixture(path):
    """-> (nx, nu, stages [(A, B, Q, R, S)], P) as float64 arrays."""
    with open(path) as fh:
        nx, nu, N = (int(t) for t in fh.readline().split())
        stages = [tuple(_read_array(fh) for _ in range(5)) for _ in range(N)]
        P = _read_array(fh)
    return nx, nu, stages, P


def dump_failures(directory, C, info, ai=0, aj=0, m=None, n=None, prefix="item"):
    """Write the input window of every failing item (``info[b] >= 0``) as
    ``<directory>/<prefix>_<b>.txt``; returns the list of paths."""
    inf = info.detach().cpu().numpy() if isinstance(info, torch.Tensor) else np.asarray(info)
    os.makedirs(directory, exist_ok=True)
    paths = []
    for b in np.nonzero(inf >= 0)[0]:
        p = os.path.join(directory, f"{prefix}_{int(b)}.txt")
        write_fixture(p, C, int(b) if C.batch > 1 else 0, ai, aj, m, n)
        paths.append(p)
    return paths
