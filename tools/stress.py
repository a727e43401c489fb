"""Randomised parity sweep of the batched routines against the oracle (GPU; run by hand).

Each case draws shapes, window offsets and batch sizes at random and compares the full item
storage (FP within 50*n*eps on the written window, every other byte exact; integer outputs exact).
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tests")
import paper_1704_02457_b200 as pb  # noqa: E402
from paper_1704_02457_b200 import level3  # noqa: E402
from oracle import oracle as O  # noqa: E402


def dev(h):
    return pb.create_panel_batch(h.batch, h.rows, h.cols, torch.from_numpy(h.storage.copy()).cuda())


def host(d):
    return d.storage.cpu().numpy()


def check(name, got, want, mask, n):
    g, w = got[:, : want.shape[1]], want
    if not np.array_equal(g[:, ~mask].view(np.uint64), w[:, ~mask].view(np.uint64)):
        raise AssertionError(f"{name}: bytes outside the write set changed")
    a, b = g[:, mask], w[:, mask]
    den = max(np.linalg.norm(b), 1e-300)
    err = np.linalg.norm(a - b) / den
    if err > 50 * max(n, 1) * 2.0 ** -52:
        raise AssertionError(f"{name}: rel err {err:.3e}")


def potrf_case(rng):
    # mostly the register/team sizes, sometimes the blocked driver (n > 128) and tall windows (m > n, any m)
    n = int(rng.integers(1, 81)) if rng.random() < 0.7 else int(rng.integers(81, 301))
    m = n if rng.random() < 0.7 else n + int(rng.integers(1, 4 if n > 200 else 400))
    nb = int(rng.integers(1, 40 if n <= 80 else 5))
    oc = (int(rng.integers(0, 6)), int(rng.integers(0, 4)))
    od = (int(rng.integers(0, 3)) * 4 if rng.random() < 0.7 else int(rng.integers(0, 6)), int(rng.integers(0, 4)))
    g = rng.uniform(-1, 1, (nb, n, n))
    a = np.zeros((nb, m, n))
    a[:, :n] = g @ g.transpose(0, 2, 1) + n * np.eye(n)
    a[:, n:] = rng.uniform(-1, 1, (nb, m - n, n))
    for b in range(nb):
        if rng.random() < 0.15:
            f = int(rng.integers(0, n))
            a[b, f, f] = -1.0
    C = O.HostBatch(nb, oc[0] + m + 1, oc[1] + n + 2)
    C.storage[:] = rng.uniform(-1, 1, C.storage.shape)
    C.set_window(oc[0], oc[1], a)
    D = O.HostBatch(nb, max(od[0], od[1]) + m + 2, od[1] + n + 1)  # diag_inv must hold dj + n
    D.storage[:] = rng.uniform(-1, 1, D.storage.shape)
    dC, dD = dev(C), dev(D)
    info = level3.potrf_l(m, dC.ref(*oc), dD.ref(*od), n=n, check=False).cpu().numpy()
    winfo = O.potrf_l(m, C, *oc, D, *od, n=n)
    assert np.array_equal(info, winfo), ("potrf info", m, n, oc, od)
    mask = np.zeros(D.storage.shape[1], dtype=bool)
    for j in range(n):
        for i in range(j, m):
            mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
    mask[D.diag_off + od[1]: D.diag_off + od[1] + n] = True
    ok = winfo < 0
    got = host(dD)
    if ok.any():
        check(f"potrf {m}x{n} {oc}{od}", got[ok], D.storage[ok], mask, m)
    # failing items: exactly the reference's partial write set (elementwise, FP tolerance)
    for b in np.nonzero(~ok)[0]:
        gb, wb = got[b, : D.storage.shape[1]], D.storage[b]
        same = np.isclose(gb, wb, rtol=1e-10, atol=1e-10) | (np.isnan(gb) & np.isnan(wb))
        assert same.all(), ("potrf failing item", m, n, oc, od, int(winfo[b]))


def getrf_case(rng):
    m, n = int(rng.integers(1, 60)), int(rng.integers(1, 60))
    nb = int(rng.integers(1, 30))
    oc = (int(rng.integers(0, 6)), int(rng.integers(0, 4)))
    od = (int(rng.integers(0, 6)), int(rng.integers(0, 4)))
    pivot = bool(rng.random() < 0.7)
    a = rng.uniform(-1, 1, (nb, m, n)) + (0 if pivot else 3.0 * np.eye(m, n))
    C = O.HostBatch(nb, oc[0] + m + 1, oc[1] + n + 2)
    C.storage[:] = rng.uniform(-1, 1, C.storage.shape)
    C.set_window(oc[0], oc[1], a)
    D = O.HostBatch(nb, max(od[0] + m, od[1] + min(m, n)) + 2, od[1] + n + 1)
    D.storage[:] = rng.uniform(-1, 1, D.storage.shape)
    dC, dD = dev(C), dev(D)
    k = min(m, n)
    ipiv = torch.full((nb, k), -7, dtype=torch.int64, device="cuda")
    if pivot:
        level3.getrf_pivot(m, n, dC.ref(*oc), dD.ref(*od), ipiv=ipiv, check=False)
    else:
        level3.getrf_nopivot(m, n, dC.ref(*oc), dD.ref(*od), check=False)
    wpiv = np.full((nb, k), -7, dtype=np.int64)
    _, wpiv = O.getrf(m, n, C, *oc, D, *od, pivot, ipiv=wpiv)
    assert np.array_equal(host(dD).view(np.uint64), D.storage.view(np.uint64)), ("getrf", m, n, oc, od, pivot)
    if pivot:
        assert np.array_equal(ipiv.cpu().numpy(), wpiv), ("getrf ipiv", m, n)


def gemm_case(rng):
    m, n, k = (int(rng.integers(1, 90)) for _ in range(3))
    nb = int(rng.integers(1, 20))
    alpha, beta = float(rng.choice([1.0, -1.0, 0.5, 0.0])), float(rng.choice([0.0, 1.0, -0.5]))
    oa, ob, oc, od = ((int(rng.integers(0, 5)), int(rng.integers(0, 3))) for _ in range(4))
    A = O.HostBatch(nb, oa[0] + m, oa[1] + k)
    B = O.HostBatch(nb, ob[0] + n, ob[1] + k)
    C = O.HostBatch(nb, oc[0] + m, oc[1] + n)
    D = O.HostBatch(nb, od[0] + m + 1, od[1] + n)
    for X in (A, B, C, D):
        X.storage[:] = rng.uniform(-1, 1, X.storage.shape)
    dA, dB, dC, dD = dev(A), dev(B), dev(C), dev(D)
    level3.gemm_nt(m, n, k, alpha, dA.ref(*oa), dB.ref(*ob), beta, dC.ref(*oc), dD.ref(*od))
    O.gemm_nt(m, n, k, alpha, A, *oa, B, *ob, beta, C, *oc, D, *od)
    mask = np.zeros(D.storage.shape[1], dtype=bool)
    for j in range(n):
        for i in range(m):
            mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
    check(f"gemm {m}x{n}x{k} a={alpha} b={beta}", host(dD), D.storage, mask, max(m, n, k))


def syrk_case(rng):
    m, k = int(rng.integers(1, 90)), int(rng.integers(0, 60))
    nb = int(rng.integers(1, 20))
    alpha, beta = float(rng.choice([1.0, -1.0, 0.0])), float(rng.choice([0.0, 1.0, 0.5]))
    oa, oc, od = ((int(rng.integers(0, 5)), int(rng.integers(0, 3))) for _ in range(3))
    same = bool(rng.random() < 0.5)
    A = O.HostBatch(nb, oa[0] + m, oa[1] + max(k, 1))
    B = A if same else O.HostBatch(nb, oa[0] + m, oa[1] + max(k, 1))
    C = O.HostBatch(nb, oc[0] + m, oc[1] + m)
    D = O.HostBatch(nb, od[0] + m + 1, od[1] + m)
    for X in {id(x): x for x in (A, B, C, D)}.values():
        X.storage[:] = rng.uniform(-1, 1, X.storage.shape)
    dA = dev(A)
    dB = dA if same else dev(B)
    dC, dD = dev(C), dev(D)
    level3.syrk_ln(m, k, alpha, dA.ref(*oa), dB.ref(*oa), beta, dC.ref(*oc), dD.ref(*od))
    O.syrk_ln(m, k, alpha, A, *oa, B, *oa, beta, C, *oc, D, *od)
    mask = np.zeros(D.storage.shape[1], dtype=bool)
    for j in range(m):
        for i in range(j, m):
            mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
    check(f"syrk {m}x{k} a={alpha} b={beta}", host(dD), D.storage, mask, max(m, k))


def trsm_case(rng):
    wide = rng.random() < 0.3  # the register-strip kernel: m >= 64, 64 <= n <= 128, panel-aligned A
    m, n = (int(rng.integers(64, 200)), int(rng.integers(64, 129))) if wide else (int(rng.integers(1, 90)), int(rng.integers(1, 70)))
    nb = int(rng.integers(1, 6 if wide else 20))
    alpha = float(rng.choice([1.0, -1.0, 0.5]))
    g = rng.uniform(-1, 1, (nb, n, n))
    a = np.linalg.cholesky(g @ g.transpose(0, 2, 1) + n * np.eye(n))
    oa, ob, od = ((int(rng.integers(0, 5)), int(rng.integers(0, 3))) for _ in range(3))
    if wide and rng.random() < 0.8:
        oa = (4 * int(rng.integers(0, 2)), oa[1])
    A = O.HostBatch(nb, oa[0] + n, oa[1] + n)
    A.storage[:] = rng.uniform(-1, 1, A.storage.shape)
    A.set_window(oa[0], oa[1], a)
    B = O.HostBatch(nb, ob[0] + m, ob[1] + n)
    D = O.HostBatch(nb, od[0] + m + 1, od[1] + n)
    for X in (B, D):
        X.storage[:] = rng.uniform(-1, 1, X.storage.shape)
    dA, dB, dD = dev(A), dev(B), dev(D)
    level3.trsm_rltn(m, n, alpha, dA.ref(*oa), dB.ref(*ob), dD.ref(*od))
    O.trsm_rltn(m, n, alpha, A, *oa, B, *ob, D, *od)
    mask = np.zeros(D.storage.shape[1], dtype=bool)
    for j in range(n):
        for i in range(m):
            mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
    check(f"trsm {m}x{n}", host(dD), D.storage, mask, max(m, n))


def syrk_potrf_case(rng):
    m, k = int(rng.integers(1, 70)), int(rng.integers(0, 40))
    nb = int(rng.integers(1, 20))
    g = rng.uniform(-1, 1, (nb, m, m))
    c = g @ g.transpose(0, 2, 1) + m * np.eye(m)
    oa, oc = ((int(rng.integers(0, 5)), int(rng.integers(0, 3))) for _ in range(2))
    od = (4 * int(rng.integers(0, 2)), int(rng.integers(0, 3)))
    A = O.HostBatch(nb, oa[0] + m, oa[1] + max(k, 1))
    A.storage[:] = rng.uniform(-0.3, 0.3, A.storage.shape)
    C = O.HostBatch(nb, oc[0] + m, oc[1] + m)
    C.storage[:] = rng.uniform(-1, 1, C.storage.shape)
    C.set_window(oc[0], oc[1], c)
    D = O.HostBatch(nb, max(od[0], od[1]) + m + 1, od[1] + m)
    D.storage[:] = rng.uniform(-1, 1, D.storage.shape)
    dA, dC, dD = dev(A), dev(C), dev(D)
    info = level3.syrk_potrf_ln(m, k, dA.ref(*oa), dA.ref(*oa), dC.ref(*oc), dD.ref(*od), check=False)
    winfo = O.syrk_potrf_ln(m, k, A, *oa, A, *oa, C, *oc, D, *od)
    if info is not None:
        assert np.array_equal(info.cpu().numpy(), winfo), ("syrk_potrf info", m, k)
    mask = np.zeros(D.storage.shape[1], dtype=bool)
    for j in range(m):
        for i in range(j, m):
            mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
    mask[D.diag_off + od[1]: D.diag_off + od[1] + m] = True
    check(f"syrk_potrf {m}x{k}", host(dD), D.storage, mask, max(m, k))


def gemm_nn_case(rng):
    m, n, k = (int(rng.integers(1, 80)) for _ in range(3))
    nb = int(rng.integers(1, 16))
    alpha, beta = float(rng.choice([1.0, -1.0, 0.0])), float(rng.choice([0.0, 1.0]))
    oa, ob, oc, od = ((int(rng.integers(0, 5)), int(rng.integers(0, 3))) for _ in range(4))
    A = O.HostBatch(nb, oa[0] + m, oa[1] + k)
    B = O.HostBatch(nb, ob[0] + k, ob[1] + n)
    C = O.HostBatch(nb, oc[0] + m, oc[1] + n)
    D = O.HostBatch(nb, od[0] + m + 1, od[1] + n)
    for X in (A, B, C, D):
        X.storage[:] = rng.uniform(-1, 1, X.storage.shape)
    dA, dB, dC, dD = dev(A), dev(B), dev(C), dev(D)
    level3.gemm_nn(m, n, k, alpha, dA.ref(*oa), dB.ref(*ob), beta, dC.ref(*oc), dD.ref(*od))
    O.gemm_nn(m, n, k, alpha, A, *oa, B, *ob, beta, C, *oc, D, *od)
    mask = np.zeros(D.storage.shape[1], dtype=bool)
    for j in range(n):
        for i in range(m):
            mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
    check(f"gemm_nn {m}x{n}x{k}", host(dD), D.storage, mask, max(m, n, k))


def main(cases=300, seed=0):
    rng = np.random.default_rng(seed)
    counts = {}
    for t in range(cases):
        fns = {"potrf": potrf_case, "getrf": getrf_case, "gemm": gemm_case, "syrk": syrk_case, "trsm": trsm_case,
               "syrk_potrf": syrk_potrf_case, "gemm_nn": gemm_nn_case}
        kind = list(fns)[t % len(fns)]
        fns[kind](rng)
        counts[kind] = counts.get(kind, 0) + 1
    print("stress ok", counts)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 300, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
