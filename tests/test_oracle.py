"""CPU: pin the oracle (oracle/pb_oracle.c) to the reference.

1. Bit-exact reproduction of every golden case recorded from the
   reference's own public API (tests/golden/make_golden.py).
2. Bit-exact agreement with the reference's compiled core itself
   (oracle/_ref, cythonized from ccore.pyx) on random panel data, when
   that build is present (it is built in the build container only).
3. The reference's known-answer tests for the layout (matstore KATs).
"""
import glob
import importlib.util
import os

import numpy as np
import pytest

from conftest import REPO, load_golden
from golden_util import host_inputs, out_labels, run_oracle
from oracle import oracle as O


def test_layout_kats():
    # tests/test_matstore.py:14-17, 42-47 of the reference
    lib = O.lib()
    assert lib.po_element_offset(6, 3, 8) == 46
    assert lib.po_element_offset(4, 0, 8) == 32
    assert lib.po_memsize(4, 4) == 192
    assert lib.po_memsize(5, 3) == 320
    assert O.memsize(4, 4) == 192 and O.memsize(5, 3) == 320


def test_golden_cases_bit_exact():
    z, cases = load_golden()
    assert len(cases) >= 70
    for case in cases:
        mats = host_inputs(z, case)
        st = run_oracle(case, mats, z)
        assert st == case["status"], (case["name"], st, case["status"])
        for lab in out_labels(case):
            want = z[f"{case['key']}/out/{lab}"]
            got = mats[lab].storage[0, : want.size]
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (case["name"], lab)
        if case["op"] in ("potrf_l", "syrk_potrf_ln"):
            d = mats[case["alias"].get("D", "D")]
            assert [d.diag_lo, d.diag_hi] == case["valid_out"]["D"], case["name"]


def test_golden_getrf_bit_exact():
    """§8f getrf (level3.py:405-498): storage, status, ipiv and diag validity
    bit-exact against the reference's own outputs."""
    z, cases = load_golden("golden_getrf_v1.npz")
    assert len(cases) >= 25
    for case in cases:
        mats = host_inputs(z, case)
        st = run_oracle(case, mats, z)
        assert st == case["status"], (case["name"], st, case["status"])
        for lab in out_labels(case):
            want = z[f"{case['key']}/out/{lab}"]
            got = mats[lab].storage[0, : want.size]
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (case["name"], lab)
        want_piv = z[f"{case['key']}/ipiv"]
        if case["params"]["pivot"]:
            assert np.array_equal(mats["_ipiv"][0][: want_piv.size], want_piv), case["name"]
        d = mats[case["alias"].get("D", "D")]
        assert [d.diag_lo, d.diag_hi] == case["valid_out"]["D"], case["name"]


def _load_ref_core():
    so = glob.glob(os.path.join(REPO, "oracle", "_ref", "ccore*.so"))
    if not so:
        return None
    spec = importlib.util.spec_from_file_location("ccore", so[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


ref_core = _load_ref_core()


@pytest.mark.skipif(ref_core is None, reason="oracle/_ref not built (make -C oracle ref)")
def test_oracle_matches_compiled_reference_core():
    rng = np.random.default_rng(7)
    for trial in range(40):
        m, n, k = (int(x) for x in rng.integers(1, 40, 3))
        sd_a, sd_b, sd_c, sd_d = (int(x) * 4 + 4 * ((k + 3) // 4 + 3) for x in rng.integers(1, 4, 4))
        sd_c = sd_d = max(sd_c, 4 * ((n + 3) // 4) + 8)
        rows = 4 * ((m + 3) // 4) + 8
        A = rng.standard_normal(rows * sd_a)
        B = rng.standard_normal((4 * ((n + 3) // 4) + 8) * sd_b)
        C = rng.standard_normal(rows * sd_c)
        D1 = rng.standard_normal(rows * sd_d)
        D2 = D1.copy()
        ci, cj, di = int(rng.integers(0, 4)), int(rng.integers(0, 3)), int(rng.integers(0, 4))
        alpha, beta = float(rng.choice([1.0, -1.5, 0.0])), float(rng.choice([0.0, 0.5, 1.0]))
        ref_core.gemm_nt_drv(m, n, k, alpha, A, 0, 1, sd_a, B, 4, 2, sd_b, beta, C, ci, cj, sd_c, D1, di, 1, sd_d)
        O.lib().po_gemm_nt(*[O._L(x) for x in (m, n, k)], O._D(alpha),
                           A.ctypes.data_as(O.ctypes.c_void_p), O._L(0), O._L(1), O._L(sd_a),
                           B.ctypes.data_as(O.ctypes.c_void_p), O._L(4), O._L(2), O._L(sd_b), O._D(beta),
                           C.ctypes.data_as(O.ctypes.c_void_p), O._L(ci), O._L(cj), O._L(sd_c),
                           D2.ctypes.data_as(O.ctypes.c_void_p), O._L(di), O._L(1), O._L(sd_d))
        assert np.array_equal(D1.view(np.uint64), D2.view(np.uint64)), ("gemm", trial)
        # syrk (square m), shared A/B stream at an aligned row
        sd_s = 4 * ((m + 3) // 4) + 8
        C = rng.standard_normal(rows * sd_s)
        S1 = rng.standard_normal(rows * sd_s)
        S2 = S1.copy()
        sd_c = sd_d = sd_s
        ref_core.syrk_ln_drv(m, k, alpha, A, 4, 0, sd_a, A, 4, 0, sd_a, beta, C, ci, 0, sd_c, S1, di, 0, sd_d)
        O.lib().po_syrk_ln(O._L(m), O._L(k), O._D(alpha),
                           A.ctypes.data_as(O.ctypes.c_void_p), O._L(4), O._L(0), O._L(sd_a),
                           A.ctypes.data_as(O.ctypes.c_void_p), O._L(4), O._L(0), O._L(sd_a), O._D(beta),
                           C.ctypes.data_as(O.ctypes.c_void_p), O._L(ci), O._L(0), O._L(sd_c),
                           S2.ctypes.data_as(O.ctypes.c_void_p), O._L(di), O._L(0), O._L(sd_d))
        assert np.array_equal(S1.view(np.uint64), S2.view(np.uint64)), ("syrk", trial)


@pytest.mark.skipif(ref_core is None, reason="oracle/_ref not built (make -C oracle ref)")
def test_oracle_factorizations_match_compiled_reference_core():
    rng = np.random.default_rng(8)
    for trial in range(30):
        n = int(rng.integers(1, 45))
        m = n + int(rng.integers(0, 9))
        sd = 4 * ((n + 3) // 4)
        rows = 4 * ((m + 3) // 4)
        g = rng.uniform(-1, 1, (m, n))
        full = np.zeros((m, n))
        full[:n] = g[:n] @ g[:n].T + n * np.eye(n)
        full[n:] = g[n:]
        if trial % 5 == 4:
            f = int(rng.integers(0, n))
            full[f, f] = -1.0
        C = np.zeros(rows * sd)
        for i in range(m):
            for j in range(n):
                C[O.element_offset(i, j, sd)] = full[i, j]
        D1 = np.full(rows * sd, 7.0)
        D2 = D1.copy()
        v1 = np.zeros(n)
        v2 = np.zeros(n)
        st1 = ref_core.potrf_drv(m, n, C, 0, 0, sd, D1, 0, 0, sd, v1, 0)
        st2 = O.lib().po_potrf_l(O._L(m), O._L(n), C.ctypes.data_as(O.ctypes.c_void_p), O._L(0), O._L(0), O._L(sd),
                                 D2.ctypes.data_as(O.ctypes.c_void_p), O._L(0), O._L(0), O._L(sd),
                                 v2.ctypes.data_as(O.ctypes.c_void_p), O._L(0))
        assert st1 == st2, trial
        assert np.array_equal(D1.view(np.uint64), D2.view(np.uint64)), ("potrf", trial)
        assert np.array_equal(v1.view(np.uint64), v2.view(np.uint64)), ("dinv", trial)
        if st1 >= 0:
            continue
        # trsm_rltn against the fresh factor, reusing its reciprocals
        mm = int(rng.integers(1, 30))
        rows_b = 4 * ((mm + 3) // 4)
        B = rng.uniform(-1, 1, rows_b * sd)
        X1 = np.zeros(rows_b * sd)
        X2 = X1.copy()
        ref_core.trsm_rltn_drv(mm, n, 1.5, D1, 0, 0, sd, False, B, 0, 0, sd, X1, 0, 0, sd, v1, 0)
        O.lib().po_trsm_rltn(O._L(mm), O._L(n), O._D(1.5), D2.ctypes.data_as(O.ctypes.c_void_p), O._L(0), O._L(0),
                             O._L(sd), O.ctypes.c_int(0), B.ctypes.data_as(O.ctypes.c_void_p), O._L(0), O._L(0),
                             O._L(sd), X2.ctypes.data_as(O.ctypes.c_void_p), O._L(0), O._L(0), O._L(sd),
                             v2.ctypes.data_as(O.ctypes.c_void_p), O._L(0))
        assert np.array_equal(X1.view(np.uint64), X2.view(np.uint64)), ("trsm", trial)


def test_oracle_potrf_against_numpy():
    rng = np.random.default_rng(9)
    for n in (1, 3, 8, 17, 40):
        g = rng.uniform(-1, 1, (n, n))
        a = g @ g.T + n * np.eye(n)
        C = O.HostBatch(1, n, n)
        C.set_window(0, 0, a[None])
        D = O.HostBatch(1, n, n)
        info = O.potrf_l(n, C, 0, 0, D, 0, 0)
        assert info[0] == -1
        got = np.tril(D.window(0, 0, n, n)[0])
        assert O.rel_fro(got, np.linalg.cholesky(a)) < O.tol(n)
        dinv = D.storage[0, D.diag_off: D.diag_off + n]
        assert np.max(np.abs(dinv * np.diag(got) - 1.0)) <= 1e-15  # tests/test_acceptance.py:266-267


def test_oracle_chain_matches_dense_riccati():
    """The C5 chain run on the oracle equals the dense
    Riccati recursion: P_next = Q + A'PA - A'PB (R + B'PB)^-1 B'PA."""
    from chain_util import dense_riccati, make_problems, oracle_chain, packed_inputs
    A, B, Q, R = make_problems(3, 32, 8, seed=1)
    BAt, RQ, P0 = packed_inputs(A, B, Q, R)
    P, K = oracle_chain(BAt, RQ, P0, 32, 8, 12)
    Pd = dense_riccati(A, B, Q, R, 12)
    Pfull = np.tril(P) + np.tril(P, -1).transpose(0, 2, 1)
    assert np.max(np.abs(Pfull - Pd)) / np.max(np.abs(Pd)) < 1e-12


@pytest.mark.skipif(ref_core is None, reason="oracle/_ref not built (make -C oracle ref)")
def test_oracle_next_tier_matches_compiled_reference_core():
    """gemm_nn, trmm_rlnn and the fused syrk_potrf
    restated in pb_oracle.c are bit-identical to the reference's own core."""
    rng = np.random.default_rng(17)
    P = O.ctypes.c_void_p
    for trial in range(25):
        m, n, k = (int(x) for x in rng.integers(1, 30, 3))
        sd = 4 * ((max(m, n, k) + 3) // 4) + 8
        rows = sd
        A, B, C = (rng.standard_normal(rows * sd) for _ in range(3))
        D1 = rng.standard_normal(rows * sd)
        D2 = D1.copy()
        ci, di, bi = int(rng.integers(0, 4)), int(rng.integers(0, 4)), int(rng.integers(0, 4))
        alpha, beta = float(rng.choice([1.0, -0.5, 0.0])), float(rng.choice([0.0, 2.0]))
        ref_core.gemm_nn_drv(m, n, k, alpha, A, 0, 1, sd, B, bi, 2, sd, beta, C, ci, 0, sd, D1, di, 1, sd)
        O.lib().po_gemm_nn(*[O._L(x) for x in (m, n, k)], O._D(alpha), A.ctypes.data_as(P), O._L(0), O._L(1),
                           O._L(sd), B.ctypes.data_as(P), O._L(bi), O._L(2), O._L(sd), O._D(beta),
                           C.ctypes.data_as(P), O._L(ci), O._L(0), O._L(sd), D2.ctypes.data_as(P), O._L(di),
                           O._L(1), O._L(sd))
        assert np.array_equal(D1.view(np.uint64), D2.view(np.uint64)), ("gemm_nn", trial)
        # trmm_rlnn: X m x n, T n x n lower (strict upper poisoned: never read)
        T = rng.standard_normal(rows * sd)
        for i in range(n):
            for j in range(i + 1, n):
                T[O.element_offset(i, j, sd)] = np.nan
        ti = int(rng.integers(0, 4))
        for i in range(n):
            for j in range(i + 1, n):
                T[O.element_offset(ti + i, j, sd)] = np.nan
        E1 = rng.standard_normal(rows * sd)
        E2 = E1.copy()
        ref_core.trmm_rlnn_drv(m, n, alpha, A, 0, 0, sd, T, ti, 0, sd, E1, di, 0, sd)
        O.lib().po_trmm_rlnn(O._L(m), O._L(n), O._D(alpha), T.ctypes.data_as(P), O._L(ti), O._L(0), O._L(sd),
                             A.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd), E2.ctypes.data_as(P), O._L(di),
                             O._L(0), O._L(sd))
        assert np.array_equal(E1.view(np.uint64), E2.view(np.uint64)), ("trmm", trial)
        # syrk_potrf: C + A A^T with C = g g^T + shift (SPD), tall when m > n
        nn = min(n, m)
        g = rng.uniform(-1, 1, (m, m))
        spd = g @ g.T + m * np.eye(m)
        Cs = np.zeros(rows * sd)
        for i in range(m):
            for j in range(nn):
                Cs[O.element_offset(i, j, sd)] = spd[i, j]
        F1 = np.full(rows * sd, 3.0)
        F2 = F1.copy()
        v1, v2 = np.zeros(sd), np.zeros(sd)
        st1 = ref_core.syrk_potrf_drv(m, nn, k, A, 0, 0, sd, A, 0, 0, sd, Cs, 0, 0, sd, F1, 0, 0, sd, v1, 0)
        st2 = O.lib().po_syrk_potrf_ln(O._L(m), O._L(nn), O._L(k), A.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd),
                                       A.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd), Cs.ctypes.data_as(P), O._L(0),
                                       O._L(0), O._L(sd), F2.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd),
                                       v2.ctypes.data_as(P), O._L(0))
        assert st1 == st2, trial
        assert np.array_equal(F1.view(np.uint64), F2.view(np.uint64)), ("syrk_potrf", trial)
        assert np.array_equal(v1.view(np.uint64), v2.view(np.uint64)), ("syrk_potrf dinv", trial)


def test_oracle_riccati_composition_bit_exact_vs_reference_golden():
    """The oracle's trmm_rlnn + syrk_potrf_ln, composed as apps.riccati_factorize
    (apps.py:218-254), reproduce the reference's stage factors bit for bit."""
    import json
    z, _ = load_golden()
    rics = json.loads(str(z["manifest"]))["riccati"]
    for r in rics:
        nx, nu, N = r["nx"], r["nu"], r["N"]
        ns = nx + nu
        term = O.HostBatch(1, nx, nx)
        P = O.HostBatch(1, nx, nx, z[f"{r['key']}/P"][None, :].copy())
        info = O.potrf_l(nx, P, 0, 0, term, 0, 0)
        assert info[0] < 0
        lnext, li = term, 0
        failed = -1
        for n in range(N - 1, -1, -1):
            bat = O.HostBatch(1, ns, nx, z[f"{r['key']}/bat{n}"][None, :].copy())
            rsq = O.HostBatch(1, ns, ns, z[f"{r['key']}/rsq{n}"][None, :].copy())
            cbuf, F = O.HostBatch(1, ns, nx), O.HostBatch(1, ns, ns)
            O.trmm_rlnn(ns, nx, 1.0, lnext, li, li, bat, 0, 0, cbuf, 0, 0)
            st = O.syrk_potrf_ln(ns, nx, cbuf, 0, 0, cbuf, 0, 0, rsq, 0, 0, F, 0, 0)[0]
            if st >= 0:
                failed = st
                assert r["msg"].startswith(f"stage {n}:"), r
                break
            if r["status"] < 0:  # the reference keeps factors only for a completed sweep
                want = z[f"{r['key']}/F{n}"]
                assert np.array_equal(F.storage[0, : want.size].view(np.uint64), want.view(np.uint64)), (r["name"], n)
            lnext, li = F, nu
        assert failed == r["status"], r["name"]


@pytest.mark.skipif(ref_core is None, reason="oracle/_ref not built (make -C oracle ref)")
@pytest.mark.parametrize("n", [64, 128, 256, 300])
def test_oracle_matches_reference_core_at_baseline_sizes(n):
    """The restatement against the reference's compiled core at the sizes the
    BASELINE configs run (C1/C2/C3 up to n = 300), bit for bit: gemm_nt,
    syrk_ln, potrf_l (+ diag_inv) and trsm_rltn reusing the fresh factor."""
    rng = np.random.default_rng(1000 + n)
    P = O.ctypes.c_void_p
    sd = 4 * ((n + 3) // 4)
    rows = sd
    A = rng.standard_normal(rows * sd)
    B = rng.standard_normal(rows * sd)
    C = rng.standard_normal(rows * sd)
    D1 = rng.standard_normal(rows * sd)
    D2 = D1.copy()
    ref_core.gemm_nt_drv(n, n, n, 1.0, A, 0, 0, sd, B, 0, 0, sd, 0.5, C, 0, 0, sd, D1, 0, 0, sd)
    O.lib().po_gemm_nt(*[O._L(x) for x in (n, n, n)], O._D(1.0), A.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd),
                       B.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd), O._D(0.5), C.ctypes.data_as(P), O._L(0),
                       O._L(0), O._L(sd), D2.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd))
    assert np.array_equal(D1.view(np.uint64), D2.view(np.uint64)), ("gemm", n)
    S1 = rng.standard_normal(rows * sd)
    S2 = S1.copy()
    ref_core.syrk_ln_drv(n, n, -1.0, A, 0, 0, sd, A, 0, 0, sd, 1.0, C, 0, 0, sd, S1, 0, 0, sd)
    O.lib().po_syrk_ln(O._L(n), O._L(n), O._D(-1.0), A.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd),
                       A.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd), O._D(1.0), C.ctypes.data_as(P), O._L(0),
                       O._L(0), O._L(sd), S2.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd))
    assert np.array_equal(S1.view(np.uint64), S2.view(np.uint64)), ("syrk", n)
    g = rng.uniform(-1, 1, (n, n))
    spd = g @ g.T + n * np.eye(n)
    Cs = np.zeros(rows * sd)
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    Cs[((ii - (ii & 3)) * sd + 4 * jj + (ii & 3)).ravel()] = spd.ravel()
    L1 = np.full(rows * sd, 3.0)
    L2 = L1.copy()
    v1, v2 = np.zeros(n), np.zeros(n)
    st1 = ref_core.potrf_drv(n, n, Cs, 0, 0, sd, L1, 0, 0, sd, v1, 0)
    st2 = O.lib().po_potrf_l(O._L(n), O._L(n), Cs.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd),
                             L2.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd), v2.ctypes.data_as(P), O._L(0))
    assert st1 == st2 == -1
    assert np.array_equal(L1.view(np.uint64), L2.view(np.uint64)), ("potrf", n)
    assert np.array_equal(v1.view(np.uint64), v2.view(np.uint64)), ("dinv", n)
    X1 = np.zeros(rows * sd)
    X2 = X1.copy()
    ref_core.trsm_rltn_drv(n, n, 1.0, L1, 0, 0, sd, False, B, 0, 0, sd, X1, 0, 0, sd, v1, 0)
    O.lib().po_trsm_rltn(O._L(n), O._L(n), O._D(1.0), L2.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd),
                         O.ctypes.c_int(0), B.ctypes.data_as(P), O._L(0), O._L(0), O._L(sd), X2.ctypes.data_as(P),
                         O._L(0), O._L(0), O._L(sd), v2.ctypes.data_as(P), O._L(0))
    assert np.array_equal(X1.view(np.uint64), X2.view(np.uint64)), ("trsm", n)


def test_oracle_pinned_to_reference_at_large_sizes():
    """The oracle at C2/C3 sizes (potrf 128/256, gemm 128/300, trsm 128)
    against digests of the REFERENCE's own outputs on the same seeded inputs
    (tests/golden/make_golden_large.py): whole item storage, bit for bit."""
    import hashlib
    import json
    import sys as _sys
    _sys.path.insert(0, os.path.join(REPO, "tests", "golden"))
    spec = json.load(open(os.path.join(REPO, "tests", "golden", "golden_large_v1.json")))

    def inputs(case):  # same generator as make_golden_large.inputs (no reference import here)
        rng = np.random.default_rng(case["seed"])
        n = case["n"]
        if case["op"] == "potrf_l":
            g = rng.uniform(-1, 1, (n, n))
            return {"C": g @ g.T + n * np.eye(n)}
        if case["op"] == "gemm_nt":
            return {"A": rng.standard_normal((n, n)), "B": rng.standard_normal((n, n))}
        g = rng.uniform(-1, 1, (n, n))
        return {"S": g @ g.T + n * np.eye(n), "B": rng.uniform(-1, 1, (n, n))}

    def hb(arr):
        h = O.HostBatch(1, *arr.shape)
        h.set_window(0, 0, arr[None])
        return h

    for case in spec["cases"]:
        n, a = case["n"], inputs(case)
        if case["op"] == "potrf_l":
            out = O.HostBatch(1, n, n)
            assert O.potrf_l(n, hb(a["C"]), 0, 0, out, 0, 0)[0] == -1
        elif case["op"] == "gemm_nt":
            out = O.HostBatch(1, n, n)
            O.gemm_nt(n, n, n, 1.0, hb(a["A"]), 0, 0, hb(a["B"]), 0, 0, 0.0, out, 0, 0, out, 0, 0)
        else:
            L = O.HostBatch(1, n, n)
            O.potrf_l(n, hb(a["S"]), 0, 0, L, 0, 0)
            out = O.HostBatch(1, n, n)
            O.trsm_rltn(n, n, 1.0, L, 0, 0, hb(a["B"]), 0, 0, out, 0, 0)
        raw = out.storage[0].view(np.uint8).tobytes()
        assert len(raw) == case["bytes"], case["name"]
        for p, v in case["samples"].items():
            assert out.storage[0, int(p)] == float.fromhex(v), (case["name"], p)
        assert hashlib.sha256(raw).hexdigest() == case["sha256"], case["name"]
