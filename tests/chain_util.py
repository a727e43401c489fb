"""Seeded C5 problem data (BASELINE configs[4]) and the oracle version of the chain."""
import numpy as np

from oracle import oracle as O


def make_problems(nb, nx, nu, seed=0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((nb, nx, nx))
    rho = np.max(np.abs(np.linalg.eigvals(A)), axis=1)
    A *= (0.95 / rho)[:, None, None]
    B = rng.standard_normal((nb, nx, nu))
    G = rng.standard_normal((nb, nx, nx))
    H = rng.standard_normal((nb, nu, nu))
    Q = 0.1 * np.eye(nx) + G @ G.transpose(0, 2, 1) / nx
    R = np.eye(nu) + H @ H.transpose(0, 2, 1) / nu
    return A, B, Q, R


def packed_inputs(A, B, Q, R):
    """BAt = [B^T; A^T] (ns x nx), RQ = blkdiag(R, Q), P_N = Q, as dense arrays."""
    nb, nx, nu = B.shape
    BAt = np.concatenate([B.transpose(0, 2, 1), A.transpose(0, 2, 1)], axis=1)
    RQ = np.zeros((nb, nx + nu, nx + nu))
    RQ[:, :nu, :nu] = R
    RQ[:, nu:, nu:] = Q
    return BAt, RQ, Q.copy()


def oracle_chain(BAt, RQ, P0, nx, nu, stages):
    nb = BAt.shape[0]
    ns = nx + nu
    hB = O.HostBatch(nb, ns, nx)
    hB.set_window(0, 0, BAt)
    hRQ = O.HostBatch(nb, ns, ns)
    hRQ.set_window(0, 0, RQ)
    hP = O.HostBatch(nb, nx, nx)
    hP.set_window(0, 0, P0)
    hW, hM, hF, hK = O.HostBatch(nb, ns, nx), O.HostBatch(nb, ns, ns), O.HostBatch(nb, ns, ns), O.HostBatch(nb, nx, nu)
    for _ in range(stages):
        O.gemm_nt(ns, nx, nx, 1.0, hB, 0, 0, hP, 0, 0, 0.0, hW, 0, 0, hW, 0, 0)
        O.syrk_ln(ns, nx, 1.0, hW, 0, 0, hB, 0, 0, 1.0, hRQ, 0, 0, hM, 0, 0)
        info = O.potrf_l(ns, hM, 0, 0, hF, 0, 0)
        assert np.all(info < 0)
        O.trsm_rltn(nx, nu, -1.0, hF, 0, 0, hF, nu, 0, hK, 0, 0)
        O.gemm_nt(nx, nx, nx, 1.0, hF, nu, nu, hF, nu, nu, 0.0, hP, 0, 0, hP, 0, 0)
    return hP.window(0, 0, nx, nx), hK.window(0, 0, nx, nu)


def dense_riccati(A, B, Q, R, stages):
    """Independent dense check: P <- Q + A'PA - A'PB (R + B'PB)^-1 B'PA."""
    P = Q.copy()
    for _ in range(stages):
        BtP = B.transpose(0, 2, 1) @ P
        S = R + BtP @ B
        AtPB = A.transpose(0, 2, 1) @ P @ B
        P = Q + A.transpose(0, 2, 1) @ P @ A - AtPB @ np.linalg.solve(S, AtPB.transpose(0, 2, 1))
        P = 0.5 * (P + P.transpose(0, 2, 1))
    return P
