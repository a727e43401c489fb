"""Batched composite factorizations built ONLY from the four hot-path
routines: the reference's range-space KKT
factorization and block-tridiagonal Cholesky, applied to a batch of
independent problems.

* ``kkt_schur_factor(n, m, H, A)``  -- apps.py:46-59:
  L_H = chol(H); M = A L_H^{-T}; L_S = chol(M M^T)   (potrf -> trsm_rltn -> syrk_ln -> potrf)
* ``block_tridiag_chol_factor(N, diag, offdiag)`` -- apps.py:268-293:
  L_0 = chol(D_0); for i >= 1: O_{i-1} = E_{i-1} L_{i-1}^{-T};
  L_i = chol(D_i - O_{i-1} O_{i-1}^T)
* ``riccati_factorize(nx, nu, N, bat, rsq, P)`` -- apps.py:218-254 (the
  reference's own Riccati recursion):
  L_N = chol(P); per stage n = N-1..0: C = [B'; A'] L_{n+1} (trmm_rlnn),
  F_n = chol([R S; S' Q] + C C') (syrk_potrf_ln), L_n = F_n[nu:, nu:]

Pivot failures raise the reference's exception types (with ``index`` and,
for the block-tridiagonal factor, the reference's "block i:" message
prefix) for the first failing problem, after the whole batch ran.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import level3, pack
from .errors import DimensionError, FactorizationError
from .matstore import allocate_panel_batch


@dataclass
class KktSchurFactor:
    n: int
    m: int
    L_H: object
    M: object
    L_S: object


def kkt_schur_factor(n, m, H, A):
    """Factor the KKT systems [H A'; A 0] of every batch item (apps.py:46-59)."""
    h = H.mat if hasattr(H, "mat") else H
    nb, dev = h.batch, h.device
    lh = allocate_panel_batch(nb, n, n, device=dev, zero=True)
    mm = allocate_panel_batch(nb, m, n, device=dev, zero=True)
    ls = allocate_panel_batch(nb, m, m, device=dev, zero=True)
    sig = allocate_panel_batch(nb, m, m, device=dev, zero=True)
    level3.potrf_l(n, H, lh)
    level3.trsm_rltn(m, n, 1.0, lh, A, mm)
    level3.syrk_ln(m, n, 1.0, mm, mm, 0.0, sig, sig)
    level3.potrf_l(m, sig, ls)
    return KktSchurFactor(n, m, lh, mm, ls)


@dataclass
class BlockTridiagFactor:
    nx: int
    N: int
    diag: list
    offdiag: list


def block_tridiag_chol_factor(N, diag_blocks, offdiag_blocks):
    """Factor a batch of SPD block-tridiagonal matrices (apps.py:268-293).

    diag_blocks[i]: PanelBatch of nx x nx diagonal blocks (lower stored);
    offdiag_blocks[i]: sub-diagonal block coupling i+1 to i."""
    if len(diag_blocks) != N or len(offdiag_blocks) != N - 1:
        raise DimensionError(f"need {N} diagonal and {N - 1} off-diagonal blocks")
    d0 = diag_blocks[0]
    nx, nb, dev = d0.rows, d0.batch, d0.device
    ld = [allocate_panel_batch(nb, nx, nx, device=dev, zero=True) for _ in range(N)]
    lo = [allocate_panel_batch(nb, nx, nx, device=dev, zero=True) for _ in range(N - 1)]
    work = allocate_panel_batch(nb, nx, nx, device=dev, zero=True)
    try:
        level3.potrf_l(nx, diag_blocks[0], ld[0])
    except FactorizationError as e:
        raise type(e)(f"block 0: {e}", e.index, e.batch_index, e.info) from e
    for i in range(1, N):
        level3.trsm_rltn(nx, nx, 1.0, ld[i - 1], offdiag_blocks[i - 1], lo[i - 1])
        pack.gecp(nx, nx, diag_blocks[i], work.ref(0, 0))
        level3.syrk_ln(nx, nx, -1.0, lo[i - 1], lo[i - 1], 1.0, work, work)
        try:
            level3.potrf_l(nx, work, ld[i])
        except FactorizationError as e:
            raise type(e)(f"block {i}: {e}", e.index, e.batch_index, e.info) from e
    return BlockTridiagFactor(nx, N, ld, lo)


# ---------------------------------------------------------------------------
# backward Riccati recursion (apps.py:180-254)


class RiccatiBatchWorkspace:
    """Per-horizon buffers of apps.RiccatiWorkspace (apps.py:180-188) for a
    batch of problems: the C product, the N stage factors, the terminal
    factor."""

    def __init__(self, batch, nx, nu, N, device="cuda"):
        if nx < 1 or nu < 0 or N < 1:
            raise DimensionError(f"bad Riccati dims nx={nx} nu={nu} N={N}")
        ns = nx + nu
        self.batch, self.nx, self.nu, self.N = batch, nx, nu, N
        self.cbuf = allocate_panel_batch(batch, ns, nx, device=device, zero=True)
        self.factors = [allocate_panel_batch(batch, ns, ns, device=device, zero=True) for _ in range(N)]
        self.terminal = allocate_panel_batch(batch, nx, nx, device=device, zero=True)


def riccati_factor_step(nx, nu, bat, rsq, L_next, cbuf, out, check=True):
    """One backward step (apps.py:218-228): cbuf = [B'; A'] L_next,
    out = chol([R S; S' Q] + cbuf cbuf')."""
    ns = nx + nu
    level3.trmm_rlnn(ns, nx, 1.0, L_next, bat, cbuf)
    return level3.syrk_potrf_ln(ns, nx, cbuf, cbuf, rsq, out, check=check)


def riccati_factorize(nx, nu, N, bat, rsq, P, workspace=None, check=True):
    """Batched apps.riccati_factorize (apps.py:231-254).

    bat[n]: PanelBatch of (nu+nx) x nx stacks [B_n'; A_n'];
    rsq[n]: (nu+nx) square [R S; S' Q] (lower referenced); P: nx x nx
    terminal cost.  Returns the workspace; ``factors[n]`` holds
    [Lambda 0; L Lcal] of stage n for every problem.  A failed pivot raises
    the reference's exception with its "terminal cost:" / "stage n:" prefix
    once the step's whole batch has run.
    """
    if len(bat) != N or len(rsq) != N:
        raise DimensionError(f"expected {N} stages, got {len(bat)} / {len(rsq)}")
    p = P.mat if hasattr(P, "mat") else P
    ws = workspace or RiccatiBatchWorkspace(p.batch, nx, nu, N, device=p.device)
    try:
        level3.potrf_l(nx, P, ws.terminal, check=check)
    except FactorizationError as e:
        raise type(e)(f"terminal cost: {e}", e.index, e.batch_index, e.info) from e
    l_next = ws.terminal.ref(0, 0)
    for n in range(N - 1, -1, -1):
        try:
            riccati_factor_step(nx, nu, bat[n], rsq[n], l_next, ws.cbuf, ws.factors[n], check=check)
        except FactorizationError as e:
            raise type(e)(f"stage {n}: {e}", e.index, e.batch_index, e.info) from e
        l_next = ws.factors[n].ref(nu, nu)
    return ws
