"""Benchmark: batched FP64 panel-major BLAS/LAPACK on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5|c6|pack] [--weak]

Default workload = BASELINE.json configs[1] ("C2"): batched dpotrf_l sweep,
n = 4, 8, 16, 32, 64, 128, 256, SPD = M M^T + n I with M ~ U[-1,1], batch
per point = round(2^34 / (n^3/3)), split batch layout (data plane + diag
plane, matstore.py), D separate from C.  One STEP = the whole sweep (every
point's full batch).  Points whose batch does not fit the device run as a
resident chunk x repetitions, the last repetition on the remainder, so
every configured item is factored exactly once per step (inputs > L2
everywhere, so no flush is needed).  metric = aggregate GFLOP/s =
sum(flops) / step time.  Per point: GFLOP/s, HBM GB/s of algorithmic bytes,
roofline fraction (roofline = min(FP64 peak, AI x HBM BW)).

The default run also carries, as sub-objects of the same JSON line:
  * "gemm": the metric's dgemm_nt half -- C1 (configs[0], 64^3, beta=1,
    batch 4096) and the C3 sweep (configs[2], n = 4..300 step 4, batch
    round(2^36 / 2n^3) per point), each point timed on the device;
  * "inplace": the C2 sweep factored in place (D == C), the reference's
    in-place form (tests/test_level3.py:319-325); C is restored from a
    pristine copy before every timed launch, outside the timed window;
  * "e2e": C2 through level3.potrf_l from pinned HOST buffers;
  * "cpu_baseline": the reference's own CPU path on the host cores.

Multi-GPU (N > 1; torchrun, or --gpus N spawns it): every point's batch is
SHARDED over the ranks (multigpu.shard_range, contiguous, sizes differ by
<= 1; strong scaling), no collective on the data path; time = max over
ranks; value = configured flops / that time.  --weak gives every rank the
full configured batch instead (value counts world x batch).

--impl reference times the reference's own CPU implementation on all host
cores: its public ``panelblas.level3`` API from ``baseline/_ref`` (the
unmodified reference, pip-installed), else its compiled core
(``oracle/_ref``), else the C restatement (``oracle/``).
"""
from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import socket
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "batched FP64 GFLOP/s (dgemm_nt, dpotrf_l) vs n, fraction of FP64/HBM roofline"
GRAPH_LAUNCHES = [0]  # kernels launched through CUDA-graph replay (not seen by the ABI counter)
FP64_PEAK_GFLOPS = 37150.0  # measured DMMA/DFMA microbench, profiles/r01_fp64_peak.log
FP64_PEAK_SRC = "measured (tools/fp64_peak.cu, DMMA m8n8k4 37.15 TF/s; cuBLAS DGEMM 35.5 TF/s)"


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


HBM_GBS, HBM_SRC = load_peaks()


# ---------------------------------------------------------------------------
# workloads


def _ru(x, t):
    return -(-x // t) * t


def split_bytes(m, n):
    """Bytes of one item in the split layout: data plane + diag plane."""
    return 8 * (_ru(m, 4) * _ru(n, 4) + min(m, n))


class Point:
    """One (routine, shape) point of a sweep: flops (reference flop_count,
    bench.py:85-105), algorithmic bytes and device footprint."""

    def __init__(self, op, m, n, k, batch, alpha=1.0, beta=0.0, cap_bytes=12e9):
        self.op, self.m, self.n, self.k = op, m, n, k
        self.alpha, self.beta = alpha, beta
        self.batch = batch
        self.cap_bytes = cap_bytes
        sb = split_bytes
        if op == "potrf_l":
            self.flops_item = n ** 3 / 3.0
            self.bytes_item = 8.0 * (n * (n + 1) + n)
            self.io_bytes = 2 * sb(n, n)  # C in, D out (+ diag_inv)
        elif op == "gemm_nt":
            self.flops_item = 2.0 * m * n * k
            self.bytes_item = 8.0 * (m * k + n * k + (m * n if beta != 0 else 0) + m * n)
            self.io_bytes = sb(m, k) + sb(n, k) + (sb(m, n) if beta != 0 else 0) + sb(m, n)
        elif op == "syrk_ln":
            self.flops_item = float(m) * (m + 1) * k
            self.bytes_item = 8.0 * (m * k + (m * (m + 1) / 2 if beta != 0 else 0) + m * (m + 1) / 2)
            self.io_bytes = sb(m + 3, k + 1) + (sb(m, m) if beta != 0 else 0) + sb(m, m)
        elif op == "trsm_rltn":
            self.flops_item = float(m) * n * n
            self.bytes_item = 8.0 * (n * (n + 1) / 2 + n + 2 * m * n)
            self.io_bytes = sb(n, n) + 2 * sb(m, n)
        elif op == "gemm_nn":
            self.flops_item = 2.0 * m * n * k
            self.bytes_item = 8.0 * (m * k + n * k + (m * n if beta != 0 else 0) + m * n)
            self.io_bytes = sb(m, k) + sb(k, n) + (sb(m, n) if beta != 0 else 0) + sb(m, n)
        elif op == "trmm_rlnn":  # reference flop_count (bench.py:90-91)
            self.flops_item = float(m) * n * n
            self.bytes_item = 8.0 * (n * (n + 1) / 2 + 2 * m * n)
            self.io_bytes = sb(n, n) + 2 * sb(m, n)
        elif op == "syrk_potrf_ln":  # m x m, A = B (m x k); bench.py:94-95
            self.flops_item = float(m) * (m + 1) * k + m ** 3 / 3.0
            self.bytes_item = 8.0 * (m * k + m * (m + 1) + m)
            self.io_bytes = sb(m, k) + 2 * sb(m, m)
        elif op == "getrf":  # getrf_pivot, square; reference flop_count 2m^3/3 (bench.py:97-98)
            self.flops_item = 2.0 * m ** 3 / 3.0
            self.bytes_item = 8.0 * (2 * m * n + min(m, n)) + 8.0 * min(m, n)  # C in, D + diag_inv + ipiv out
            self.io_bytes = 2 * sb(m, n) + 8 * min(m, n)
        elif op == "riccati_fact":  # apps.riccati_factorize: m = nx, n = nu, k = N; bench.py:98-101
            nx, nu, ns = m, n, m + n
            self.flops_item = k * (float(ns) * nx * nx + float(ns) * (ns + 1) * nx + ns ** 3 / 3.0)
            # per stage: read [B';A'], L_next (lower), [R S;S' Q] (lower); write cbuf, read it back; write F + diag_inv
            self.bytes_item = k * 8.0 * (3 * ns * nx + nx * (nx + 1) / 2 + ns * (ns + 1) + ns)
            self.io_bytes = (k + 1) * (sb(ns, nx) + 2 * sb(ns, ns))
        elif op == "riccati":  # m = nx, n = nu, k = N stages
            nx, nu, ns = m, n, m + n
            per_stage = (2.0 * ns * nx * nx + float(ns) * (ns + 1) * nx + ns ** 3 / 3.0 + float(nx) * nu * nu
                         + 2.0 * nx * nx * nx)
            self.flops_item = k * per_stage
            # per stage: read BAt,P,RQ,W,M,F; write W,M,F,K,P (algorithmic, lower halves where symmetric)
            self.bytes_item = k * 8.0 * (2 * ns * nx + 2 * nx * nx + 3 * ns * (ns + 1) / 2 + ns * nx + nx * nu)
            self.io_bytes = 8 * sb(ns, ns)
        elif op in ("pack", "unpack"):  # column-major <-> panel-major copy of an n x n item
            self.flops_item = 0.0
            self.bytes_item = 16.0 * n * n
            self.io_bytes = 8 * n * n + sb(n, n)
        else:
            raise ValueError(op)

    @property
    def label(self):
        if self.op == "riccati_fact":
            return f"riccati_factorize nx={self.m} nu={self.n} N={self.k}"
        if self.op in ("gemm_nn", "syrk_potrf_ln"):
            return f"{self.op} {self.m}x{self.n}x{self.k}"
        if self.op == "getrf":
            return f"getrf_pivot {self.m}x{self.n}"
        if self.op == "riccati":
            return f"riccati nx={self.m} nu={self.n} N={self.k}"
        if self.op == "potrf_l":
            return f"potrf_l n={self.n}"
        if self.op == "gemm_nt":
            return f"gemm_nt {self.m}x{self.n}x{self.k}"
        if self.op in ("pack", "unpack"):
            return f"{self.op} n={self.n}"
        return f"{self.op} {self.m}x{self.n if self.op == 'trsm_rltn' else self.k}"

    def roofline_gflops(self):
        if self.flops_item == 0:
            return None
        ai = self.flops_item / self.bytes_item
        return min(FP64_PEAK_GFLOPS, ai * HBM_GBS)

    def hbm_bound(self):
        return self.flops_item == 0 or self.flops_item / self.bytes_item * HBM_GBS < FP64_PEAK_GFLOPS


def config_points(name):
    if name == "c2":
        return [Point("potrf_l", n, n, 0, round(2 ** 34 / (n ** 3 / 3.0))) for n in (4, 8, 16, 32, 64, 128, 256)], \
            "C2 batched dpotrf_l sweep n=4..256, ~2^34 flop per point (BASELINE configs[1])"
    if name == "c1":
        return [Point("gemm_nt", 64, 64, 64, 4096, 1.0, 1.0)], \
            "C1 batched dgemm_nt 64^3 alpha=beta=1, batch 4096 (BASELINE configs[0])"
    if name == "c3":
        pts = [Point("gemm_nt", n, n, n, max(1, round(2 ** 36 / (2.0 * n ** 3))), cap_bytes=3e9)
               for n in range(4, 301, 4)]
        return pts, "C3 batched dgemm_nt sweep n=4..300 step 4, beta=0, batch round(2^36/2n^3) (BASELINE configs[2])"
    if name == "c4":
        return [Point("syrk_ln", 96, 96, 40, 8192, -1.0, 1.0), Point("trsm_rltn", 72, 48, 0, 8192, 1.0)], \
            "C4 dsyrk_ln 96x40 at (3,1) alpha=-1 beta=1 + dtrsm_rltn 72x48 (diag_inv reused), batch 8192"
    if name == "c5":
        return [Point("riccati", 32, 8, 50, 1024)], \
            "C5 Riccati-style chain: 1024 problems x N=50 stages, nx=32 nu=8 (gemm_nt, syrk_ln, potrf_l, trsm_rltn, gemm_nt per stage)"
    if name == "c6":
        return [Point("gemm_nn", 64, 64, 64, 4096, 1.0, 1.0), Point("trmm_rlnn", 40, 32, 0, 16384, 1.0),
                Point("syrk_potrf_ln", 40, 40, 32, 16384), Point("riccati_fact", 32, 8, 50, 1024),
                Point("getrf", 32, 32, 0, 16384)], \
            ("C6 next tier (SURVEY §8f): dgemm_nn 64^3 batch 4096, dtrmm_rlnn 40x32 and dsyrk_potrf_ln 40x40 k=32 "
             "batch 16384, apps.riccati_factorize nx=32 nu=8 N=50 x 1024 problems, dgetrf_pivot 32x32 batch 16384")
    if name == "pack":
        pts = []
        for n in (4, 16, 64):
            for op in ("pack", "unpack"):
                pts.append(Point(op, n, n, 0, max(1 << 20, round(4e9 / (16 * n * n))), cap_bytes=8e9))
        return pts, "panel-major pack/unpack (kpack_cm / kunpack_cm) n = 4, 16, 64, >= 1M items, ~4 GB moved per point"
    raise SystemExit(f"unknown config {name}")


# ---------------------------------------------------------------------------
# sharding and accounting (pure host logic; tests/test_bench_sharding.py)


def plan_point(pt, rank, world, weak=False):
    """This rank's share of a point: (lo, hi, chunk, reps, last).

    Strong scaling (default): the configured batch is split into contiguous
    ranges (multigpu.shard_range); weak: every rank takes the whole batch.
    The share runs as ``reps`` launches over a resident chunk of ``chunk``
    items (bounded by the point's device-memory cap); the last launch covers
    ``last`` items, so exactly hi - lo items are processed."""
    from paper_1704_02457_b200.multigpu import shard_range
    lo, hi = (0, pt.batch) if weak else shard_range(pt.batch, rank, world)
    items = hi - lo
    if items == 0:
        return lo, hi, 0, 0, 0
    reps = max(1, math.ceil(items * pt.io_bytes / pt.cap_bytes))
    chunk = math.ceil(items / reps)
    reps = math.ceil(items / chunk)
    last = items - chunk * (reps - 1)
    return lo, hi, chunk, reps, last


def items_of(plan):
    lo, hi, chunk, reps, last = plan
    return 0 if reps == 0 else chunk * (reps - 1) + last


# ---------------------------------------------------------------------------
# GPU arm


class GpuPoint:
    """Device-resident inputs/outputs for one point (this rank's chunk)."""

    def __init__(self, pt, plan, device, seed, inplace=False):
        import torch
        import paper_1704_02457_b200 as pb
        from paper_1704_02457_b200 import pack
        self.pt, self.plan = pt, plan
        self.inplace = inplace
        lo, hi, chunk, reps, last = plan
        nb = self.nb = max(chunk, 1)
        g = torch.Generator(device=device).manual_seed(seed)
        m, n, k = pt.m, pt.n, pt.k
        u = lambda *s: torch.rand(s, dtype=torch.float64, device=device, generator=g) * 2 - 1  # noqa: E731
        self.ops = {}
        if pt.op == "potrf_l":
            C = pb.allocate_panel_batch(nb, n, n, device=device)
            step = max(1, (1 << 26) // (n * n))
            for s0 in range(0, nb, step):
                s1 = min(nb, s0 + step)
                M = u(s1 - s0, n, n)
                a = torch.baddbmm(torch.eye(n, dtype=torch.float64, device=device).expand(s1 - s0, n, n) * n,
                                  M, M.transpose(1, 2))
                pack.pack_array_into(a, C.shard(s0, s1))
            if inplace:
                self.pristine = C.storage.clone()
                self.ops = {"C": C, "D": C}
            else:
                self.ops = {"C": C, "D": pb.allocate_panel_batch(nb, n, n, device=device, zero=True)}
        elif pt.op == "gemm_nt":
            A = pb.allocate_panel_batch(nb, m, k, device=device)
            B = pb.allocate_panel_batch(nb, n, k, device=device)
            D = pb.allocate_panel_batch(nb, m, n, device=device, zero=True)
            if pt.beta == 0.0:
                for x in (A, B):
                    x.storage.normal_(generator=g)  # C3: N(0,1)
                C = D  # beta == 0: C is never read (ccore.pyx:36)
            else:
                C = pb.allocate_panel_batch(nb, m, n, device=device)
                for x in (A, B, C):
                    x.storage.uniform_(-1, 1, generator=g)  # C1: U[-1,1]
            self.ops = {"A": A, "B": B, "C": C, "D": D}
        elif pt.op == "syrk_ln":
            A = pb.allocate_panel_batch(nb, m + 3, k + 1, device=device)
            A.storage.uniform_(-1, 1, generator=g)
            C = pb.allocate_panel_batch(nb, m, m, device=device)
            C.storage.uniform_(-1, 1, generator=g)
            self.ops = {"A": A, "C": C, "D": pb.allocate_panel_batch(nb, m, m, device=device, zero=True)}
        elif pt.op == "riccati":
            from paper_1704_02457_b200.chain import RiccatiChain
            nx, nu = m, n
            Ad = torch.randn((nb, nx, nx), dtype=torch.float64, device=device, generator=g)
            rho = torch.linalg.eigvals(Ad).abs().amax(dim=1)
            Ad *= (0.95 / rho)[:, None, None]
            Bd = torch.randn((nb, nx, nu), dtype=torch.float64, device=device, generator=g)
            G = torch.randn((nb, nx, nx), dtype=torch.float64, device=device, generator=g)
            H = torch.randn((nb, nu, nu), dtype=torch.float64, device=device, generator=g)
            Q = 0.1 * torch.eye(nx, dtype=torch.float64, device=device) + G @ G.transpose(1, 2) / nx
            R = torch.eye(nu, dtype=torch.float64, device=device) + H @ H.transpose(1, 2) / nu
            ch = RiccatiChain(nb, nx, nu, device=device)
            pack.pack_array_into(torch.cat([Bd.transpose(1, 2), Ad.transpose(1, 2)], dim=1).contiguous(), ch.BAt)
            RQ = torch.zeros((nb, nx + nu, nx + nu), dtype=torch.float64, device=device)
            RQ[:, :nu, :nu] = R
            RQ[:, nu:, nu:] = Q
            pack.pack_array_into(RQ, ch.RQ)
            self.Q = pb.allocate_panel_batch(nb, nx, nx, device=device)
            pack.pack_array_into(Q.contiguous(), self.Q)
            ch.P.storage.copy_(self.Q.storage)
            self.fused = ch.fused_supported()
            if not self.fused:
                ch.capture(k)
            self.chain = ch
        elif pt.op == "gemm_nn":
            A = pb.allocate_panel_batch(nb, m, k, device=device)
            B = pb.allocate_panel_batch(nb, k, n, device=device)
            C = pb.allocate_panel_batch(nb, m, n, device=device)
            for x in (A, B, C):
                x.storage.uniform_(-1, 1, generator=g)
            self.ops = {"A": A, "B": B, "C": C, "D": pb.allocate_panel_batch(nb, m, n, device=device, zero=True)}
        elif pt.op == "trmm_rlnn":
            A = pb.allocate_panel_batch(nb, n, n, device=device)
            A.storage.uniform_(-1, 1, generator=g)
            B = pb.allocate_panel_batch(nb, m, n, device=device)
            B.storage.uniform_(-1, 1, generator=g)
            self.ops = {"A": A, "B": B, "D": pb.allocate_panel_batch(nb, m, n, device=device, zero=True)}
        elif pt.op == "syrk_potrf_ln":
            A = pb.allocate_panel_batch(nb, m, k, device=device)
            A.storage.uniform_(-1, 1, generator=g)
            C = pb.allocate_panel_batch(nb, m, m, device=device)
            Md = u(nb, m, m)
            pack.pack_array_into(torch.baddbmm(torch.eye(m, dtype=torch.float64, device=device).expand(nb, m, m) * m,
                                               Md, Md.transpose(1, 2)), C)
            self.ops = {"A": A, "C": C, "D": pb.allocate_panel_batch(nb, m, m, device=device, zero=True)}
        elif pt.op == "getrf":
            C = pb.allocate_panel_batch(nb, m, n, device=device)
            C.storage.uniform_(-1, 1, generator=g)
            self.ops = {"C": C, "D": pb.allocate_panel_batch(nb, m, n, device=device, zero=True)}
            self.ipiv = torch.zeros((nb, min(m, n)), dtype=torch.int64, device=device)
        elif pt.op == "riccati_fact":
            from paper_1704_02457_b200 import composite
            nx, nu, N = m, n, k
            ns = nx + nu
            self.bat, self.rsq = [], []
            for _ in range(N):
                Ad = u(nb, nx, nx) * 0.5 + 0.8 * torch.eye(nx, dtype=torch.float64, device=device)
                Bd = u(nb, nx, nu)
                self.bat.append(pack.panel_from_array(torch.cat([Bd.transpose(1, 2), Ad.transpose(1, 2)], 1)
                                                      .contiguous()))
                Gd = u(nb, ns, ns)
                self.rsq.append(pack.panel_from_array(
                    torch.baddbmm(torch.eye(ns, dtype=torch.float64, device=device).expand(nb, ns, ns) * ns,
                                  Gd, Gd.transpose(1, 2))))
            Gp = u(nb, nx, nx)
            self.Pn = pack.panel_from_array(torch.baddbmm(torch.eye(nx, dtype=torch.float64, device=device)
                                                          .expand(nb, nx, nx) * nx, Gp, Gp.transpose(1, 2)))
            self.ws = composite.RiccatiBatchWorkspace(nb, nx, nu, N, device=device)
            composite.riccati_factorize(nx, nu, N, self.bat, self.rsq, self.Pn, workspace=self.ws)  # checked once
            torch.cuda.synchronize()
            from paper_1704_02457_b200 import _native as _nm
            c0 = _nm.launch_count()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                composite.riccati_factorize(nx, nu, N, self.bat, self.rsq, self.Pn, workspace=self.ws, check=False)
            self.graph_kernels = _nm.launch_count() - c0
        elif pt.op == "trsm_rltn":
            from paper_1704_02457_b200 import level3
            M = u(nb, n, n)
            spd = torch.baddbmm(torch.eye(n, dtype=torch.float64, device=device).expand(nb, n, n) * n,
                                M, M.transpose(1, 2))
            S = pack.panel_from_array(spd)
            A = pb.allocate_panel_batch(nb, n, n, device=device, zero=True)
            level3.potrf_l(n, S, A)  # diag_inv valid -> reused by trsm (level3.py:169-170)
            del S
            B = pb.allocate_panel_batch(nb, m, n, device=device)
            B.storage.uniform_(-1, 1, generator=g)
            self.ops = {"A": A, "B": B, "D": pb.allocate_panel_batch(nb, m, n, device=device, zero=True)}
        elif pt.op in ("pack", "unpack"):
            C = pb.allocate_panel_batch(nb, n, n, device=device)
            cm = torch.empty((nb, n * n), dtype=torch.float64, device=device)
            cm.uniform_(-1, 1, generator=g)
            if pt.op == "unpack":
                pack.pack_matrix(pack.ColBatch(n, n, n, cm), n, n, C)
            self.ops = {"P": C, "X": pack.ColBatch(n, n, n, cm)}
        # views over the first `last` items for the final (partial) repetition
        self.part = None
        if 0 < last < chunk and self.ops:
            self.part = {kk: (v.shard(0, last) if hasattr(v, "shard") else
                              __import__("paper_1704_02457_b200").pack.ColBatch(v.rows, v.cols, v.lda, v.data[:last]))
                         for kk, v in self.ops.items()}

    def restore(self):
        """In-place variant: put the pristine inputs back (untimed)."""
        self.ops["C"].storage.copy_(self.pristine)

    def _run(self, o, cnt):
        from paper_1704_02457_b200 import level3, pack
        pt = self.pt
        if pt.op == "potrf_l":
            level3.potrf_l(pt.n, o["C"], o["D"], check=False)
        elif pt.op == "gemm_nt":
            level3.gemm_nt(pt.m, pt.n, pt.k, pt.alpha, o["A"], o["B"], pt.beta, o["C"], o["D"])
        elif pt.op == "syrk_ln":
            a = o["A"].ref(3, 1)
            level3.syrk_ln(pt.m, pt.k, pt.alpha, a, a, pt.beta, o["C"], o["D"])
        elif pt.op == "trsm_rltn":
            level3.trsm_rltn(pt.m, pt.n, pt.alpha, o["A"], o["B"], o["D"], check=False)
        elif pt.op == "gemm_nn":
            level3.gemm_nn(pt.m, pt.n, pt.k, pt.alpha, o["A"], o["B"], pt.beta, o["C"], o["D"])
        elif pt.op == "trmm_rlnn":
            level3.trmm_rlnn(pt.m, pt.n, pt.alpha, o["A"], o["B"], o["D"])
        elif pt.op == "syrk_potrf_ln":
            level3.syrk_potrf_ln(pt.m, pt.k, o["A"], o["A"], o["C"], o["D"], check=False)
        elif pt.op == "getrf":
            level3.getrf_pivot(pt.m, pt.n, o["C"], o["D"], ipiv=self.ipiv[:cnt], check=False)
        elif pt.op == "pack":
            pack.pack_matrix(o["X"], pt.n, pt.n, o["P"])
        elif pt.op == "unpack":
            pack.unpack_matrix(o["P"], pt.n, pt.n, o["X"])

    def launch(self, only_rep=None):
        """This rank's whole share of the point (reference-facing level3 API,
        no host sync); ``only_rep`` runs just that repetition."""
        lo, hi, chunk, reps, last = self.plan
        pt = self.pt
        for r in (range(reps) if only_rep is None else [only_rep]):
            cnt = chunk if r < reps - 1 else last
            if pt.op == "riccati_fact":
                self.graph.replay()  # whole backward sweep: one graph of trmm + syrk/gemm + potrf per stage
                GRAPH_LAUNCHES[0] += self.graph_kernels
            elif pt.op == "riccati":
                # P_N = Q, then the N-stage sweep (one persistent kernel)
                self.chain.P.storage.copy_(self.Q.storage)
                if self.fused:
                    self.chain.run_fused(pt.k)
                else:
                    self.chain.replay()
                    GRAPH_LAUNCHES[0] += 5 * pt.k
            else:
                self._run(self.ops if cnt == chunk or self.part is None else self.part, cnt)


def nvsmi_sampler(path):
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        return subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100",
                                 "-i", str(int(os.environ.get("LOCAL_RANK", "0")))],
                                stdout=open(path, "w"), stderr=subprocess.DEVNULL)
    except Exception:
        return None


def parse_clocks(path):
    try:
        rows = [r.split(",") for r in open(path).read().strip().splitlines() if r.strip()]
    except Exception:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
    sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
    mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
    reasons = set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for r in rows:
        if len(r) < 9:
            continue
        for i, nm in enumerate(names):
            if r[5 + i].strip().lower() == "active":
                reasons.add(nm)
    return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "samples": len(sm), "reasons": sorted(reasons)}


def traffic_from_profile(pt, chunk):
    """ncu dram bytes per launch of this point's kernel (profiles/traffic.json), scaled to `chunk` items."""
    p = os.path.join(REPO, "profiles", "traffic.json")
    try:
        d = json.load(open(p))[pt.label]
        return d["dram_bytes_per_launch"] * chunk / d["items_per_launch"], d
    except Exception:
        return None, None


def point_record(pt, items, ms, world_factor=1):
    """Per-point numbers from `items` processed in `ms` (summed over ranks)."""
    sec = ms / 1e3
    rec = {"point": pt.label, "items": items, "ms": ms, "gbs_alg": items * pt.bytes_item / sec / 1e9}
    if pt.flops_item:
        gfl = items * pt.flops_item / sec / 1e9
        roof = pt.roofline_gflops() * world_factor
        rec.update({"gflops": gfl, "roofline_gflops": roof, "roofline_frac": gfl / roof,
                    "bound": "hbm" if pt.hbm_bound() else "fp64"})
    else:
        rec.update({"roofline_frac": rec["gbs_alg"] / (HBM_GBS * world_factor), "bound": "hbm"})
    return rec


def _max_over_ranks(vals, device, world):
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t]


def _sum_over_ranks(vals, device, world):
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t]


def time_points_separately(pts, args, device, rank, world, inplace=False, seed0=5000):
    """Each point on its own: build, warm up, time args.steps launches of this
    rank's share with CUDA events (max over ranks), free.  Used by the
    "gemm" and "inplace" sub-objects."""
    import torch
    steps = max(1, min(args.steps, args.sub_steps))
    out = []
    stream = torch.cuda.current_stream()
    for i, pt in enumerate(pts):
        plan = plan_point(pt, rank, world, args.weak)
        gp = GpuPoint(pt, plan, device, seed=seed0 + 1000 * i + 17 * rank, inplace=inplace)
        for _ in range(args.warmup):
            for r in range(plan[3]):
                if inplace:
                    gp.restore()
                gp.launch(r)
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        tot = 0.0
        if inplace:  # every repetition on restored inputs; restores outside the timed windows
            evs = []
            for _ in range(steps):
                for r in range(plan[3]):
                    gp.restore()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    gp.launch(r)
                    e1.record(stream)
                    evs.append((e0, e1))
            torch.cuda.synchronize()
            tot = sum(a.elapsed_time(b) for a, b in evs)
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                gp.launch()
            e1.record(stream)
            torch.cuda.synchronize()
            tot = e0.elapsed_time(e1)
        ms = _max_over_ranks([tot / steps], device, world)[0]
        items = int(_sum_over_ranks([items_of(plan)], device, world)[0])
        rec = point_record(pt, items, ms, world)
        rec["per_rank_launches"] = plan[3]
        out.append(rec)
        del gp
        torch.cuda.empty_cache()
    return out


def gemm_subobject(args, device, rank, world):
    """The metric's dgemm_nt half: C1 and the full-config C3 sweep."""
    c1, _ = config_points("c1")
    c3, _ = config_points("c3")
    r1 = time_points_separately(c1, args, device, rank, world, seed0=7000)
    r3 = time_points_separately(c3, args, device, rank, world, seed0=9000)
    fl = sum(p["items"] * q.flops_item for p, q in zip(r3, c3))
    ms = sum(p["ms"] for p in r3)
    fr = [p["roofline_frac"] for p, q in zip(r3, c3) if q.n >= 64]
    fr_small = [p["roofline_frac"] for p, q in zip(r3, c3) if q.n <= 16]
    return {
        "c1": dict(r1[0], workload="C1 dgemm_nt 64^3 alpha=beta=1 batch 4096 (BASELINE configs[0])"),
        "c3": {"workload": "C3 dgemm_nt n=4..300 step 4, beta=0, batch round(2^36/2n^3) (BASELINE configs[2])",
               "value": fl / (ms / 1e3) / 1e9, "unit": "GFLOP/s", "sweep_ms": ms,
               "frac_n_ge_64": {"median": statistics.median(fr), "min": min(fr)},
               "frac_n_le_16": {"median": statistics.median(fr_small), "min": min(fr_small)},
               "points": r3},
    }


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1704_02457_b200 as pb
    from paper_1704_02457_b200 import _native

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    pts, desc = config_points(args.config)
    if args.only:
        keep = [x.strip() for x in args.only.split(",")]
        pts = [p for p in pts if p.label in keep]
        desc += " [subset: %s]" % args.only
    pb.load_native()

    plans = [plan_point(pt, rank, world, args.weak) for pt in pts]
    gps = [GpuPoint(pt, plan, device, seed=1000 * i + 17 * rank) for i, (pt, plan) in enumerate(zip(pts, plans))]
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def step(evs=None):
        for i, gp in enumerate(gps):
            if evs is not None:
                evs[i][0].record(stream)
            gp.launch()
            if evs is not None:
                evs[i][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk_path = os.path.join(REPO, "gpurun_out" if os.path.isdir(os.path.join(REPO, "gpurun_out")) else ".",
                            f".clocks_rank{rank}.csv")
    sampler = nvsmi_sampler(clk_path)
    time.sleep(0.3)
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in gps]
           for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _native.launch_count(reset=True)
    GRAPH_LAUNCHES[0] = 0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0.record(stream)
    for s in range(args.steps):
        step([evs[s][i] for i in range(len(gps))])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = _native.launch_count() + GRAPH_LAUNCHES[0]
    if sampler:
        sampler.terminate()
        sampler.wait()
    total_ms = t0.elapsed_time(t1)
    pt_ms = [sum(evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(args.steps)) / args.steps
             for i in range(len(gps))]
    mx = _max_over_ranks([total_ms] + pt_ms, device, world)
    total_ms, pt_ms = mx[0], mx[1:]
    items_all = [int(x) for x in _sum_over_ranks([items_of(p) for p in plans], device, world)]
    launches = int(_sum_over_ranks([launches], device, world)[0])
    clocks = parse_clocks(clk_path)

    points = []
    tot_flops = 0.0
    wf = world  # per-point roofline scales with the GPUs working on it
    for i, gp in enumerate(gps):
        pt = gp.pt
        rec = point_record(pt, items_all[i], pt_ms[i], wf)
        rec.update({"chunk": gp.plan[2], "launches_per_rank": gp.plan[3]})
        points.append(rec)
        tot_flops += items_all[i] * pt.flops_item
    step_ms = total_ms / args.steps
    value = tot_flops / (step_ms / 1e3) / 1e9
    roof_time = sum(p["items"] * gp.pt.flops_item / (p["roofline_gflops"] * 1e9)
                    for p, gp in zip(points, gps) if p.get("roofline_gflops"))

    # dominant kernel (largest share of the step): its roofline, per launch, per GPU
    dom = max(range(len(points)), key=lambda i: points[i]["ms"])
    dp, dgp = points[dom], gps[dom]
    dpt, dplan = dgp.pt, dgp.plan
    launch_ms = dp["ms"] / max(1, dplan[3])
    chunk = dplan[2]
    if dpt.hbm_bound():
        ach = chunk * dpt.bytes_item / (launch_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": ach, "peak": HBM_GBS, "unit": "GB/s", "frac": ach / HBM_GBS,
                    "peak_src": HBM_SRC, "alg_bytes_per_item": dpt.bytes_item}
    else:
        ach = chunk * dpt.flops_item / (launch_ms * 1e-3) / 1e9
        roofline = {"bound": "fp64", "achieved": ach, "peak": FP64_PEAK_GFLOPS, "unit": "GFLOP/s",
                    "frac": ach / FP64_PEAK_GFLOPS, "peak_src": FP64_PEAK_SRC, "flops_per_item": dpt.flops_item}
    traffic, tsrc = traffic_from_profile(dpt, chunk)
    roofline.update({"kernel": dp["point"], "items_per_launch": chunk, "share_of_step": dp["ms"] / step_ms,
                     "launch_ms": launch_ms, "traffic": traffic})
    if traffic:
        dram = traffic / (launch_ms * 1e-3) / 1e9
        roofline.update({"traffic_src": tsrc.get("source"), "dram_gbs": dram, "dram_frac": dram / HBM_GBS,
                         "traffic_alg_ratio": traffic / (dpt.bytes_item * chunk)})

    # free the headline's buffers before the sub-objects
    e2e = None
    if not args.no_e2e and args.config == "c2":
        e2e = run_e2e(args, gps, device, world, rank)
    del gps
    torch.cuda.empty_cache()
    gemm = inplace = None
    if args.config == "c2" and not args.only and not args.no_gemm:
        gemm = gemm_subobject(args, device, rank, world)
    if args.config == "c2" and not args.no_inplace:
        ipts = [Point(p.op, p.m, p.n, p.k, p.batch) for p in pts]  # footprint: C (== D) + pristine copy
        ir = time_points_separately(ipts, args, device, rank, world, inplace=True, seed0=3000)
        fl = sum(p["items"] * q.flops_item for p, q in zip(ir, ipts))
        ms = sum(p["ms"] for p in ir)
        inplace = {"workload": desc + ", factored in place (D == C), C restored between launches (untimed)",
                   "value": fl / (ms / 1e3) / 1e9, "unit": "GFLOP/s", "sweep_ms": ms, "points": ir}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(pts, budget_s=args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded torch Philox on device; SPD = M M^T + n I, M~U[-1,1])",
            "config": {"workload": desc, "config": args.config,
                       "parallelism": (f"batch replicated x{world} (weak)" if args.weak
                                       else f"batch-sharded x{world} (contiguous ranges, no collective)"),
                       "layout": "split (data plane + diag_inv plane), D != C",
                       "l2": "inputs > L2 (126 MB) at every point; no flush needed",
                       "roofline_gflops_step": tot_flops / roof_time / 1e9 if roof_time else None,
                       "frac_of_step_roofline": value / (tot_flops / roof_time / 1e9) if roof_time else None},
            "points": points,
            "roofline": roofline,
            "clocks": clocks,
            "gpu_launches": launches,
            "e2e": e2e,
            "gemm": gemm,
            "inplace": inplace,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
        if args.csv:
            emit_csv(csv_rows(points, pts), args.csv)
        if args.csv_ext:
            emit_csv_ext(csv_rows(points, pts), points, pts, world, args.csv_ext)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def csv_rows(points, pts, impl="b200"):
    """Rows in the reference's sweep CSV schema (bench.py:436-462):
    routine,impl,m,n,k,seconds,gflops -- seconds = per-call time amortised
    over the batch (so rows compare 1:1 with the reference's per-call rows)."""
    rows = []
    for p, pt in zip(points, pts):
        if pt.op == "potrf_l":
            m = n = k = pt.n
        else:
            m, n, k = pt.m, pt.n, pt.k
        sec = p["ms"] / 1e3 / max(1, p["items"])
        rows.append((pt.op, impl, m, n, k, sec, p.get("gflops", 0.0)))
    return rows


def emit_csv(rows, path):
    """Write rows sorted by (routine, impl, m) with 17 significant digits."""
    with open(path, "w") as fh:
        fh.write("routine,impl,m,n,k,seconds,gflops\n")
        for r in sorted(rows, key=lambda r: (r[0], r[1], r[2])):
            fh.write(f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]},{r[5]:.17g},{r[6]:.17g}\n")


def emit_csv_ext(rows, points, pts, world, path):
    """The reference's seven columns (same order and formatting) followed by
    gpus, batch, hbm_gbs_alg, roofline_gflops, roofline_frac;
    a separate file, because the reference's parse_csv accepts only its exact header."""
    with open(path, "w") as fh:
        fh.write("routine,impl,m,n,k,seconds,gflops,gpus,batch,hbm_gbs_alg,roofline_gflops,roofline_frac\n")
        order = sorted(range(len(rows)), key=lambda i: (rows[i][0], rows[i][1], rows[i][2]))
        for i in order:
            r, p, pt = rows[i], points[i], pts[i]
            fh.write(f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]},{r[5]:.17g},{r[6]:.17g},{world},{p['items']},"
                     f"{p['gbs_alg']:.17g},{p.get('roofline_gflops') or 0.0:.17g},{p['roofline_frac']:.17g}\n")


def run_e2e(args, gps, device, world, rank):
    """C2 through the public API with HOST buffers: every step copies each
    point's inputs host->device from pinned memory (C's data plane), runs
    level3.potrf_l, and reads the results device->host (D's data plane and
    diag_inv plane); four streams with their own device staging buffers
    keep both copy directions busy (a stream's next upload waits only for
    its own previous download).  A bounded pinned host buffer per point
    holds one sub-chunk of inputs; it is re-sent for every sub-chunk (the
    data are synthetic either way)."""
    import torch
    import paper_1704_02457_b200 as pb
    from paper_1704_02457_b200 import level3

    streams = [torch.cuda.Stream(device) for _ in range(4)]
    plans = []
    for gp in gps:
        pt = gp.pt
        if pt.op != "potrf_l":
            return None
        n = pt.n
        sub = max(1, min(gp.nb, int(128e6 // split_bytes(n, n))))
        host_in = gp.ops["C"].storage[:sub].cpu().pin_memory()  # this point's inputs (per point)
        plans.append((gp, sub, host_in))
    # per-stream result / staging buffers shared by all points (host pinned
    # memory stays ~1.5 GB per rank however many points)
    out_elems = max(sub * (pb.panel_data_elems(gp.pt.n, gp.pt.n) + gp.pt.n) for gp, sub, _ in plans)
    host_raw = [torch.empty(out_elems, dtype=torch.float64).pin_memory() for _ in streams]
    dev_raw = [(torch.empty(out_elems, dtype=torch.float64, device=device),
                torch.empty(out_elems, dtype=torch.float64, device=device)) for _ in streams]

    vcache = {}

    def views(k, n, cnt):
        key = (k, n, cnt)
        if key in vcache:
            return vcache[key]
        de = pb.panel_data_elems(n, n)
        hr = host_raw[k]
        hd, hg = hr[: cnt * de].view(cnt, de), hr[cnt * de: cnt * de + cnt * n].view(cnt, n)
        ci, co = dev_raw[k]
        cin = pb.create_panel_batch(cnt, n, n, ci[: cnt * de], ci[cnt * de: cnt * de + cnt * n])
        dout = pb.create_panel_batch(cnt, n, n, co[: cnt * de], co[cnt * de: cnt * de + cnt * n])
        vcache[key] = (hd, hg, cin, dout)
        return vcache[key]

    h2d = d2h = 0

    def one_step(count=False):
        nonlocal h2d, d2h
        k = 0
        for gp, sub, host_in in plans:
            n_items = items_of(gp.plan)
            for s0 in range(0, n_items, sub):
                cnt = min(sub, n_items - s0)
                st = streams[k % len(streams)]
                hd, hg, cin, dout = views(k % len(streams), gp.pt.n, cnt)
                k += 1
                with torch.cuda.stream(st):
                    cin.storage.copy_(host_in[:cnt], non_blocking=True)
                    level3.potrf_l(gp.pt.n, cin, dout, check=False)
                    hd.copy_(dout.storage, non_blocking=True)
                    hg.copy_(dout.diag_storage, non_blocking=True)
                if count:
                    h2d += cin.storage.numel() * 8
                    d2h += (dout.storage.numel() + dout.diag_storage.numel()) * 8
        for st in streams:
            st.synchronize()

    one_step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    steps = max(1, min(args.steps, args.e2e_steps))
    t0 = time.perf_counter()
    for i in range(steps):
        one_step(count=(i == 0))
    torch.cuda.synchronize()
    el = _max_over_ranks([time.perf_counter() - t0], device, world)[0]
    tot = _sum_over_ranks([sum(items_of(gp.plan) * gp.pt.flops_item for gp in gps), h2d, d2h], device, world)
    return {"value": tot[0] * steps / el / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(tot[1]),
            "d2h_bytes_per_step": int(tot[2]), "steps": steps,
            "how": "level3.potrf_l on pinned host panel-major planes (C data in; D data + diag_inv out), "
                   "H2D + compute + D2H overlapped on 4 streams; wall clock, max over ranks"}


# ---------------------------------------------------------------------------
# CPU reference arm / cpu_baseline


def _ref_path():
    p = os.path.join(REPO, "baseline", "_ref")
    return p if os.path.isdir(os.path.join(p, "panelblas")) else None


def _ref_core():
    import glob
    import importlib.util
    so = glob.glob(os.path.join(REPO, "oracle", "_ref", "ccore*.so"))
    if not so:
        return None
    spec = importlib.util.spec_from_file_location("ccore", so[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _llc_bytes():
    best = 0
    base = "/sys/devices/system/cpu/cpu0/cache"
    try:
        for d in os.listdir(base):
            try:
                lvl = int(open(os.path.join(base, d, "level")).read())
                sz = open(os.path.join(base, d, "size")).read().strip()
                mult = {"K": 1 << 10, "M": 1 << 20}.get(sz[-1], 1)
                v = int(sz.rstrip("KM")) * mult
                if lvl >= 3:
                    best = max(best, v)
            except Exception:
                pass
    except Exception:
        pass
    return best or (32 << 20)


_CALLS_CACHE = {}  # per worker process: (op, shape, pool size) -> prepared calls (built once, reused by later steps)


def _cpu_worker(job):
    """Time the reference on one point's sample in one process.

    With the reference package (baseline/_ref) every call goes through its
    public ``panelblas.level3`` API on PanelMatrix items wrapped zero-copy
    (``create_panel_matrix``) from one host pool in the reference layout;
    the pool is larger than this worker's share of the LLC and is streamed
    item by item (no item is reused before the whole pool has been)."""
    op, m, n, k, alpha, beta, seconds, seed, pool_bytes = job
    key = (op, m, n, k, alpha, beta, pool_bytes)
    if key not in _CALLS_CACHE:
        _CALLS_CACHE[key] = _prepare_calls(op, m, n, k, alpha, beta, seed, pool_bytes)
    calls, flops_item = _CALLS_CACHE[key]
    # timed loop, bounded by `seconds`
    done = 0
    t0 = time.perf_counter()
    while True:
        for c in calls:
            c()
        done += len(calls)
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done, el, done * flops_item


def _prepare_calls(op, m, n, k, alpha, beta, seed, pool_bytes):
    import numpy as np
    rp = _ref_path()
    if rp and rp not in sys.path:
        sys.path.insert(0, rp)
    rng = np.random.default_rng(seed)
    ru4 = lambda x: -(-x // 4) * 4  # noqa: E731
    level3 = matstore = None
    if rp:
        from panelblas import level3, matstore  # noqa: F811
    core = None if rp else _ref_core()

    def offs(mm, nn, cn):
        ii, jj = np.meshgrid(np.arange(mm), np.arange(nn), indexing="ij")
        return ((ii - (ii & 3)) * cn + 4 * jj + (ii & 3)).ravel()

    def memsize(mm, nn):
        return -(-(ru4(mm) * ru4(nn) * 8) // 64) * 64 + -(-(min(mm, nn) * 8) // 64) * 64

    def pool_of(mm, nn, count, fill):
        """count items of the reference layout in one buffer; fill(cnt) -> [cnt, mm, nn] values"""
        per = memsize(mm, nn) // 8
        buf = np.zeros(count * per + 8)
        shift = (-buf.ctypes.data % 64) // 8
        buf = buf[shift: shift + count * per].reshape(count, per)
        o = offs(mm, nn, ru4(nn))
        for s0 in range(0, count, 4096):
            s1 = min(count, s0 + 4096)
            buf[s0:s1, o] = fill(s1 - s0).reshape(s1 - s0, -1)
        if matstore is not None:
            return buf, [matstore.create_panel_matrix(mm, nn, buf[i]) for i in range(count)]
        return buf, None

    def spd(cnt, nn):
        g = rng.uniform(-1, 1, (cnt, nn, nn))
        return g @ g.transpose(0, 2, 1) + nn * np.eye(nn)

    uni = lambda mm, nn: (lambda c: rng.uniform(-1, 1, (c, mm, nn)))  # noqa: E731
    if op == "potrf_l":
        count = max(64, min(300000, 2 * pool_bytes // memsize(n, n)))
        count //= 2  # C and D both streamed
        cbuf, Cs = pool_of(n, n, count, lambda c: spd(c, n))
        dbuf, Ds = pool_of(n, n, count, uni(n, n))
        flops_item = n ** 3 / 3.0
        if level3 is not None:
            calls = [(lambda c=Cs[i], d=Ds[i]: level3.potrf_l(n, c, d)) for i in range(count)]
        else:
            ck = ru4(n)
            dv = np.zeros(n)
            calls = [(lambda c=cbuf[i], d=dbuf[i]: core.potrf_drv(n, n, c, 0, 0, ck, d, 0, 0, ck, dv, 0))
                     for i in range(count)]
    elif op == "gemm_nt":
        per = memsize(m, k) + memsize(n, k) + memsize(m, n) * (2 if beta != 0 else 1)
        count = max(8, min(100000, pool_bytes // per))
        abuf, As = pool_of(m, k, count, uni(m, k))
        bbuf, Bs = pool_of(n, k, count, uni(n, k))
        cbuf, Cs = pool_of(m, n, count if beta != 0 else 1, uni(m, n))
        dbuf, Ds = pool_of(m, n, count, uni(m, n))
        flops_item = 2.0 * m * n * k
        if level3 is not None:
            calls = [(lambda i=i: level3.gemm_nt(m, n, k, alpha, As[i], Bs[i], beta, Cs[i if beta != 0 else 0],
                                                 Ds[i])) for i in range(count)]
        else:
            sk, sn = ru4(k), ru4(n)
            calls = [(lambda i=i: core.gemm_nt_drv(m, n, k, alpha, abuf[i], 0, 0, sk, bbuf[i], 0, 0, sk, beta,
                                                   cbuf[i if beta != 0 else 0], 0, 0, sn, dbuf[i], 0, 0, sn))
                     for i in range(count)]
    elif op == "syrk_ln":
        count = max(8, min(100000, pool_bytes // (memsize(m + 3, k + 1) + 2 * memsize(m, m))))
        abuf, As = pool_of(m + 3, k + 1, count, uni(m + 3, k + 1))
        cbuf, Cs = pool_of(m, m, count, uni(m, m))
        dbuf, Ds = pool_of(m, m, count, uni(m, m))
        flops_item = float(m) * (m + 1) * k
        if level3 is not None:
            calls = [(lambda i=i: level3.syrk_ln(m, k, alpha, As[i].ref(3, 1), As[i].ref(3, 1), beta, Cs[i], Ds[i]))
                     for i in range(count)]
        else:
            raise RuntimeError("syrk_ln CPU sample needs the reference package (baseline/_ref)")
    elif op == "trsm_rltn":
        count = max(8, min(100000, pool_bytes // (2 * memsize(m, n))))
        lbuf, Ls = pool_of(n, n, 1, lambda c: np.linalg.cholesky(spd(c, n)))
        bbuf, Bs = pool_of(m, n, count, uni(m, n))
        dbuf, Ds = pool_of(m, n, count, uni(m, n))
        flops_item = float(m) * n * n
        if level3 is None:
            raise RuntimeError("trsm_rltn CPU sample needs the reference package (baseline/_ref)")
        A = Ls[0]
        spdm = matstore.allocate_panel_matrix(n, n)
        sb, _ = pool_of(n, n, 1, lambda c: spd(c, n))
        spdm.data[:] = sb[0][: spdm.data.size]
        level3.potrf_l(n, spdm, A)  # diag_inv valid -> reused (level3.py:169-170)
        calls = [(lambda i=i: level3.trsm_rltn(m, n, alpha, A, Bs[i], Ds[i])) for i in range(count)]
    elif op == "riccati":
        if level3 is None:
            raise RuntimeError("riccati CPU sample needs the reference package (baseline/_ref)")
        nx, nu, N = m, n, k
        ns = nx + nu
        _, (BAt,) = pool_of(ns, nx, 1, lambda c: rng.standard_normal((c, ns, nx)) * 0.2)
        _, (RQ,) = pool_of(ns, ns, 1, lambda c: (1.0 + ns) * np.eye(ns)[None].repeat(c, 0))
        _, (P,) = pool_of(nx, nx, 1, lambda c: np.eye(nx)[None].repeat(c, 0))
        W, M, F = matstore.allocate_panel_matrix(ns, nx), matstore.allocate_panel_matrix(ns, ns), \
            matstore.allocate_panel_matrix(ns, ns)
        K = matstore.allocate_panel_matrix(nx, nu)
        for x in (W, M, F, K):
            x.data[:] = 0.0  # step 5 reads F's strict upper, which potrf_l never writes (SURVEY §8a chain note)

        def chain():
            for _ in range(N):
                level3.gemm_nt(ns, nx, nx, 1.0, BAt, P, 0.0, W, W)
                level3.syrk_ln(ns, nx, 1.0, W, BAt, 1.0, RQ, M)
                level3.potrf_l(ns, M, F)
                level3.trsm_rltn(nx, nu, -1.0, F.ref(0, 0), F.ref(nu, 0), K)
                level3.gemm_nt(nx, nx, nx, 1.0, F.ref(nu, nu), F.ref(nu, nu), 0.0, P, P)
        flops_item = N * (2.0 * ns * nx * nx + float(ns) * (ns + 1) * nx + ns ** 3 / 3.0 + float(nx) * nu * nu
                          + 2.0 * nx * nx * nx)
        calls = [chain]
    elif op in ("gemm_nn", "trmm_rlnn", "syrk_potrf_ln", "getrf", "riccati_fact"):
        if level3 is None:
            raise RuntimeError(f"{op} CPU sample needs the reference package (baseline/_ref)")
        if op == "gemm_nn":
            _, As = pool_of(m, k, 64, uni(m, k))
            _, Bs = pool_of(k, n, 64, uni(k, n))
            _, Cs = pool_of(m, n, 64, uni(m, n))
            _, Ds = pool_of(m, n, 64, uni(m, n))
            calls = [(lambda i=i: level3.gemm_nn(m, n, k, alpha, As[i], Bs[i], beta, Cs[i], Ds[i])) for i in range(64)]
            flops_item = 2.0 * m * n * k
        elif op == "trmm_rlnn":
            _, As = pool_of(n, n, 64, uni(n, n))
            _, Bs = pool_of(m, n, 64, uni(m, n))
            _, Ds = pool_of(m, n, 64, uni(m, n))
            calls = [(lambda i=i: level3.trmm_rlnn(m, n, alpha, As[i], Bs[i], Ds[i])) for i in range(64)]
            flops_item = float(m) * n * n
        elif op == "syrk_potrf_ln":
            _, As = pool_of(m, k, 64, lambda c: rng.uniform(-1, 1, (c, m, k)))
            _, Cs = pool_of(m, m, 64, lambda c: (1.0 + m * k) * np.eye(m)[None].repeat(c, 0))
            _, Ds = pool_of(m, m, 64, uni(m, m))
            calls = [(lambda i=i: level3.syrk_potrf_ln(m, k, As[i], As[i], Cs[i], Ds[i])) for i in range(64)]
            flops_item = float(m) * (m + 1) * k + m ** 3 / 3.0
        elif op == "getrf":
            _, Cs = pool_of(m, n, 64, uni(m, n))
            _, Ds = pool_of(m, n, 64, uni(m, n))
            calls = [(lambda i=i: level3.getrf_pivot(m, n, Cs[i], Ds[i])) for i in range(64)]
            flops_item = 2.0 * m ** 3 / 3.0
        else:  # apps.riccati_factor_step x N through level3 (apps.py:218-228)
            nx, nu, N = m, n, k
            ns = nx + nu
            _, bats = pool_of(ns, nx, 4, uni(ns, nx))
            _, (RSQ,) = pool_of(ns, ns, 1, lambda c: (1.0 + ns) * np.eye(ns)[None].repeat(c, 0))
            _, (Lt,) = pool_of(nx, nx, 1, lambda c: np.eye(nx)[None].repeat(c, 0))
            cb = matstore.allocate_panel_matrix(ns, nx)
            Fs = [matstore.allocate_panel_matrix(ns, ns) for _ in range(N)]
            for x in [cb] + Fs:
                x.data[:] = 0.0

            def fact():
                T = Lt.ref(0, 0)
                for st in range(N - 1, -1, -1):
                    level3.trmm_rlnn(ns, nx, 1.0, T, bats[st & 3], cb)
                    level3.syrk_potrf_ln(ns, nx, cb, cb, RSQ, Fs[st])
                    T = Fs[st].ref(nu, nu)
            calls = [fact]
            flops_item = N * (float(ns) * nx * nx + float(ns) * (ns + 1) * nx + ns ** 3 / 3.0)
    else:
        raise ValueError(op)
    return calls, flops_item


def _kind():
    if _ref_path():
        return "reference", "panelblas.level3 public API (baseline/_ref: the unmodified reference, pip-installed; " \
                            "compiled ccore backend 'c', -O3)"
    if _ref_core() is not None:
        return "reference", "the reference's compiled core ccore.pyx (oracle/_ref), driver entry points"
    return "port", "oracle/libpb_oracle.so (C restatement)"


def _worker_loop(conn):
    while True:
        job = conn.recv()
        if job is None:
            break
        try:
            conn.send(("ok", _cpu_worker(job)))
        except Exception as exc:  # reported by the caller
            conn.send(("err", f"{type(exc).__name__}: {exc}"))


class CpuWorkers:
    """One long-lived process per host core; job i always goes to worker i,
    so each worker's prepared input pools (built on first use) are reused by
    later steps instead of being rebuilt."""

    def __init__(self, n):
        ctx = mp.get_context("spawn")
        self.conns, self.procs = [], []
        for _ in range(n):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker_loop, args=(b,), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)

    def map(self, jobs):
        for c, j in zip(self.conns, jobs):
            c.send(j)
        res = [c.recv() for c in self.conns[: len(jobs)]]
        bad = [r[1] for r in res if r[0] != "ok"]
        if bad:
            raise RuntimeError(bad[0])
        return [r[1] for r in res]

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=10)


def cpu_baseline(pts, budget_s=12.0, workers=None):
    """The reference's CPU path on all host cores (one process per core) and
    on 1 core (worker 0 alone, same input pool), a bounded sample per point;
    rates extrapolated to the configured sweep as sum(F) / sum(F / R)."""
    cores = len(os.sched_getaffinity(0))
    kind, impl = _kind()
    llc = _llc_bytes()
    per_point = max(0.1, budget_s / len(pts) / 1.5)
    pool_b = max(48 << 20, 2 * llc // cores)
    rates, rates1, samples = [], [], []
    own = workers is None
    if own:
        workers = CpuWorkers(cores)
    t_start = time.perf_counter()
    try:
        for i, pt in enumerate(pts):
            if pt.op in ("pack", "unpack"):
                rates.append(None)
                rates1.append(None)
                continue
            jobs = [(pt.op, pt.m, pt.n, pt.k, pt.alpha, pt.beta, per_point, 7919 * i + w, pool_b)
                    for w in range(cores)]
            try:
                res = workers.map(jobs)
                one = workers.map([jobs[0][:6] + (per_point / 2,) + jobs[0][7:]])[0]
            except Exception as exc:  # an op without a CPU sample path: reported, not fatal
                rates.append(None)
                rates1.append(None)
                samples.append(f"{pt.label}: unavailable ({exc})")
                continue
            items = sum(r[0] for r in res)
            wall = max(r[1] for r in res)
            rates.append(sum(r[2] for r in res) / wall / 1e9)
            rates1.append(one[2] / one[1] / 1e9)
            samples.append(f"{pt.label}: {items} calls on {cores} cores in {wall:.2f}s, {one[0]} on 1 core")
    finally:
        if own:
            workers.close()
    wall_total = time.perf_counter() - t_start
    ok = [(pt, r, r1) for pt, r, r1 in zip(pts, rates, rates1) if r]
    tot = sum(pt.batch * pt.flops_item for pt, _, _ in ok)
    tim = sum(pt.batch * pt.flops_item / (r * 1e9) for pt, r, _ in ok)
    tim1 = sum(pt.batch * pt.flops_item / (r1 * 1e9) for pt, _, r1 in ok)
    return {"value": tot / tim / 1e9 if tim else None, "unit": "GFLOP/s", "cores": cores, "kind": kind,
            "value_1core": tot / tim1 / 1e9 if tim1 else None,
            "sample": "; ".join(samples) + f" (each worker streams its own input pool of >= {pool_b >> 20} MB, "
                                           f"LLC {llc >> 20} MB; per-point rates extrapolated to the configured "
                                           f"sweep as sum F / sum F/R)",
            "sample_wall_s": wall_total,
            "extrapolated_sweep_s": tim if tim else None,
            "per_point_gflops": {pt.label: r for pt, r in zip(pts, rates)},
            "per_point_gflops_1core": {pt.label: r for pt, r in zip(pts, rates1)},
            "impl": impl}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pts, desc = config_points(args.config)
    if args.only:
        keep = [x.strip() for x in args.only.split(",")]
        pts = [p for p in pts if p.label in keep]
        desc += " [subset: %s]" % args.only
    workers = CpuWorkers(len(os.sched_getaffinity(0)))
    vals, walls, r = [], [], None
    for s in range(max(1, args.warmup) + args.steps):  # warm-up steps build every worker's input pools
        t0 = time.perf_counter()
        r = cpu_baseline(pts, budget_s=args.ref_seconds if s >= max(1, args.warmup) else 0.1, workers=workers)
        if s >= max(1, args.warmup):
            walls.append(time.perf_counter() - t0)
            vals.append(r["value"])
    workers.close()
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC,
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(walls) * 1e3,
            "ms_per_step_note": "measured wall of one bounded CPU sample of the sweep (all points); the configured "
                                "sweep itself would take extrapolated_sweep_s",
            "extrapolated_sweep_s": r["extrapolated_sweep_s"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (numpy, same distributions)",
            "config": {"workload": desc, "config": args.config, "parallelism": "CPU processes (batch-parallel)"},
            "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": r["cores"], "kind": r["kind"],
                             "sample": r["sample"], "value_1core": r["value_1core"], "impl": r["impl"]},
            "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "per_point_gflops": r["per_point_gflops"], "per_point_gflops_1core": r["per_point_gflops_1core"]}
    print(json.dumps(line), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--weak", action="store_true", help="every rank runs the full configured batch (weak scaling)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-gemm", action="store_true", help="skip the C1/C3 dgemm_nt sub-object")
    ap.add_argument("--no-inplace", action="store_true", help="skip the in-place C2 sub-object")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--sub-steps", type=int, default=5, help="timed launches per point in the sub-objects")
    ap.add_argument("--cpu-seconds", type=float, default=14.0)
    ap.add_argument("--ref-seconds", type=float, default=7.0)
    ap.add_argument("--csv", default=None, help="also write per-point rows in the reference's sweep CSV schema")
    ap.add_argument("--csv-ext", default=None,
                    help="also write the reference's columns + gpus, batch, algorithmic GB/s and roofline fraction")
    ap.add_argument("--only", default=None,
                    help="comma-separated point labels to keep (tuning runs only, e.g. 'potrf_l n=4')")
    args = ap.parse_args(argv)
    config_points(args.config)  # reject an unknown --config before touching CUDA
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # not launched by torchrun: spawn one rank per GPU ourselves
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
        cmd += sys.argv[1:] if argv is None else argv
        sys.exit(subprocess.call(cmd))
    if world is not None and int(world) != args.gpus:
        print(f"error: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
