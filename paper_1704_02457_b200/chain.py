"""Config-5 chain: a batched Riccati-recursion-style sweep built ONLY from the
four hot-path routines (BASELINE configs[4]).

Per stage, for every problem (S = 0, ns = nu + nx, P symmetric, F's strict
upper stays zero because potrf_l never writes it):

  1. gemm_nt(ns, nx, nx, 1, BAt, P, 0, W)            W   = [B A]^T P
  2. syrk_ln(ns, nx, 1, W, BAt, 1, RQ, M)            lower(M) = [B A]^T P [B A] + blkdiag(R, Q)
  3. potrf_l(ns, M, F)                               F   = [Lam 0; L Lcal]
  4. trsm_rltn(nx, nu, -1, F[0:nu,0:nu], F[nu:,0:nu], K)   K Lam^T = -L
  5. gemm_nt(nx, nx, nx, 1, Lcal, Lcal, 0, P)        P   = Lcal Lcal^T

This is the chain SURVEY §8a row 19 documents (its P_0 equals the
reference's riccati_factorize cost-to-go); the reference's own
apps.riccati_factor_step (trmm_rlnn + syrk_potrf_ln, apps.py:218-228) is a
different, out-of-scope composition.  Problems are time-invariant
(one A, B, Q, R per problem); the whole N-stage sweep of all problems is
5*N batched launches, optionally captured once into a CUDA graph.
"""
from __future__ import annotations

import ctypes

import torch

from . import _native, level3
from .matstore import allocate_panel_batch


class RiccatiChain:
    """Batched device state for `batch` problems of sizes (nx, nu)."""

    def __init__(self, batch, nx, nu, device="cuda"):
        self.batch, self.nx, self.nu = batch, nx, nu
        ns = nx + nu
        self.ns = ns
        mk = lambda m, n: allocate_panel_batch(batch, m, n, device=device, zero=True)  # noqa: E731
        self.BAt = mk(ns, nx)      # [B^T; A^T]
        self.RQ = mk(ns, ns)       # blkdiag(R, Q)
        self.P = mk(nx, nx)        # cost-to-go (full symmetric)
        self.W = mk(ns, nx)
        self.M = mk(ns, ns)
        self.F = mk(ns, ns)        # factor; strict upper stays zero
        self.K = mk(nx, nu)        # per-stage gain-like output (last stage kept)
        self.graph = None

    def stage(self):
        nx, nu, ns = self.nx, self.nu, self.ns
        level3.gemm_nt(ns, nx, nx, 1.0, self.BAt, self.P, 0.0, self.W, self.W)
        level3.syrk_ln(ns, nx, 1.0, self.W, self.BAt, 1.0, self.RQ, self.M)
        level3.potrf_l(ns, self.M, self.F, check=False)
        level3.trsm_rltn(nx, nu, -1.0, self.F.ref(0, 0), self.F.ref(nu, 0), self.K, check=False)
        level3.gemm_nt(nx, nx, nx, 1.0, self.F.ref(nu, nu), self.F.ref(nu, nu), 0.0, self.P, self.P)

    def run(self, stages):
        for _ in range(stages):
            self.stage()

    def capture(self, stages):
        """Record the whole sweep once into a CUDA graph (launch-overhead free replay)."""
        self.stage()  # initialise lazily configured kernels outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(stages)
        self.graph = g
        return g

    def replay(self):
        self.graph.replay()

    def fused_supported(self):
        return self.nu == 8 and self.nx in (8, 16, 24, 32, 48, 64)

    def run_fused(self, stages):
        """All `stages` in one persistent kernel (pb_driccati_chain): every
        problem stays resident in shared memory; P <- P_0, K <- last stage's K.
        Returns the per-problem info tensor (-1 ok, else stage*1000 + pivot)."""
        if not self.fused_supported():
            raise NotImplementedError("fused chain needs nu == 8 and nx in {8,16,24,32,48,64}")
        info = torch.empty(self.batch, dtype=torch.int32, device=self.P.device)
        d = [x.descriptor() for x in (self.BAt, self.RQ, self.P, self.K)]
        stream = ctypes.c_void_p(torch.cuda.current_stream(self.P.device).cuda_stream)
        _native.call("pb_driccati_chain", self.nx, self.nu, stages, *[ctypes.byref(x) for x in d],
                     ctypes.c_void_p(info.data_ptr()), stream)
        return info


def flops_per_stage(nx, nu):
    """Reference flop_count conventions (bench.py:85-105) summed over the 5 calls."""
    ns = nx + nu
    return (2.0 * ns * nx * nx + float(ns) * (ns + 1) * nx + ns ** 3 / 3.0 + float(nx) * nu * nu
            + 2.0 * nx * nx * nx)
