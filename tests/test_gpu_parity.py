"""GPU parity: the CUDA path (through the C ABI) against the oracle.

* every golden case recorded from the reference, run as a batch;
* seeded random batches at every kernel-dispatch regime (direct,
  tiled-32, tiled-64, team sizes, blocked composites) against the
  oracle (pinned bit-exact to the reference in test_oracle.py);
* the reference's discrete semantics (alpha/beta/k/m/n zero cases,
  windows never left, aliasing bit-equal, determinism, failure indices
  and partial writes), all exact;
* full BASELINE-size batches through size-independent properties.

Tolerance (north_star): relative Frobenius error <= 50 * n * eps_fp64 on
floating-point results; bit-exact for pack/unpack/copies, untouched
storage and info.
"""
import numpy as np
import pytest

from conftest import cuda_ok, load_golden
from golden_util import host_inputs, out_labels, run_oracle, written_mask
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

torch = pytest.importorskip("torch")
import paper_1704_02457_b200 as pb  # noqa: E402
from paper_1704_02457_b200 import level3, pack  # noqa: E402

EPS = np.finfo(np.float64).eps


# Every test runs on both batch layouts (matstore.py): "split" (data plane +
# diag plane, the default) and "interleaved" (the reference's item layout).
LAYOUT = "split"
_ORIG = {}  # id(PanelBatch) -> host storage it was made from (padding bytes of a split batch)


@pytest.fixture(autouse=True, params=["split", "interleaved"])
def layout(request):
    global LAYOUT
    LAYOUT = request.param
    _ORIG.clear()
    yield request.param
    _ORIG.clear()


def alloc(nb, m, n, zero=False):
    return pb.allocate_panel_batch(nb, m, n, zero=zero, layout=LAYOUT)


def dev(h):
    """HostBatch -> PanelBatch on cuda:0 (same bytes) in the current layout."""
    if LAYOUT == "interleaved":
        t = torch.from_numpy(h.storage.copy()).cuda()
        p = pb.create_panel_batch(h.batch, h.rows, h.cols, t)
    else:
        de, dn = pb.panel_data_elems(h.rows, h.cols), min(h.rows, h.cols)
        data = torch.from_numpy(np.ascontiguousarray(h.storage[:, :de])).cuda()
        diag = torch.from_numpy(np.ascontiguousarray(h.storage[:, h.diag_off: h.diag_off + dn])).cuda()
        p = pb.create_panel_batch(h.batch, h.rows, h.cols, data.reshape(-1), diag.reshape(-1))
        _ORIG[id(p)] = (p, h.storage.copy())
    p.diag_lo, p.diag_hi = h.diag_lo, h.diag_hi
    return p


def host(p):
    """Reference item layout of a device batch (numpy [batch, memsize/8])."""
    st = p.item_storage().detach().cpu().numpy()
    if p.layout == "split" and id(p) in _ORIG:  # padding slots as they were on the host
        base = _ORIG[id(p)][1].copy()
        de, dn = pb.panel_data_elems(p.rows, p.cols), min(p.rows, p.cols)
        doff = p.memsize // 8 - (-(-dn * 8 // 64) * 8)
        base[:, :de] = st[:, :de]
        base[:, doff: doff + dn] = st[:, doff: doff + dn]
        return base
    return st


def fp_close(got, want, n, what=""):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    both_nan = np.isnan(got) & np.isnan(want)
    assert not np.any(np.isnan(got) ^ np.isnan(want)), f"NaN pattern differs {what}"
    d = np.where(both_nan, 0.0, got - want)
    w = np.where(both_nan, 0.0, want)
    den = np.linalg.norm(w)
    err = np.linalg.norm(d) / den if den > 0 else np.linalg.norm(d)
    assert err <= 50 * max(n, 1) * EPS, f"rel Frobenius {err:.3e} > {50 * max(n, 1) * EPS:.3e} {what}"


def compare_storage(got, want, mask, n, what):
    """mask True: FP tolerance; mask False: bit-exact."""
    gu, wu = got.view(np.uint64), want.view(np.uint64)
    assert np.array_equal(gu[..., ~mask], wu[..., ~mask]), f"untouched storage changed {what}"
    fp_close(got[..., mask], want[..., mask], n, what)


def run_product(case, mats):
    p = case["params"]
    op = case["op"]
    if op == "gemm_nt":
        level3.gemm_nt(p["m"], p["n"], p["k"], p["alpha"], mats["A"].ref(p["ai"], p["aj"]),
                       mats["B"].ref(p["bi"], p["bj"]), p["beta"], mats["C"].ref(p["ci"], p["cj"]),
                       mats["D"].ref(p["di"], p["dj"]))
        return None
    if op == "syrk_ln":
        level3.syrk_ln(p["m"], p["k"], p["alpha"], mats["A"].ref(p["ai"], p["aj"]), mats["B"].ref(p["bi"], p["bj"]),
                       p["beta"], mats["C"].ref(p["ci"], p["cj"]), mats["D"].ref(p["di"], p["dj"]))
        return None
    if op == "trsm_rltn":
        return level3.trsm_rltn(p["m"], p["n"], p["alpha"], mats["A"].ref(p["ai"], p["aj"]),
                                mats["B"].ref(p["bi"], p["bj"]), mats["D"].ref(p["di"], p["dj"]), check=False)
    if op == "potrf_l":
        return level3.potrf_l(p["m"], mats["C"].ref(p["ci"], p["cj"]), mats["D"].ref(p["di"], p["dj"]), n=p["n"],
                              check=False)
    if op == "gemm_nn":
        level3.gemm_nn(p["m"], p["n"], p["k"], p["alpha"], mats["A"].ref(p["ai"], p["aj"]),
                       mats["B"].ref(p["bi"], p["bj"]), p["beta"], mats["C"].ref(p["ci"], p["cj"]),
                       mats["D"].ref(p["di"], p["dj"]))
        return None
    if op == "trmm_rlnn":
        level3.trmm_rlnn(p["m"], p["n"], p["alpha"], mats["A"].ref(p["ai"], p["aj"]),
                         mats["B"].ref(p["bi"], p["bj"]), mats["D"].ref(p["di"], p["dj"]))
        return None
    if op == "syrk_potrf_ln":
        return level3.syrk_potrf_ln(p["m"], p["k"], mats["A"].ref(p["ai"], p["aj"]), mats["B"].ref(p["bi"], p["bj"]),
                                    mats["C"].ref(p["ci"], p["cj"]), mats["D"].ref(p["di"], p["dj"]), n=p["n"],
                                    check=False)
    if op == "getrf":
        nb = mats["D"].batch
        mn = max(min(p["m"], p["n"]), 1)
        ipiv = torch.full((nb, mn), -7, dtype=torch.int64, device="cuda")
        fn = level3.getrf_pivot if p["pivot"] else level3.getrf_nopivot
        args = (p["m"], p["n"], mats["C"].ref(p["ci"], p["cj"]), mats["D"].ref(p["di"], p["dj"]))
        if p["pivot"]:
            fn(*args, ipiv=ipiv, check=False)
        else:
            fn(*args, check=False)
        mats["_ipiv"] = ipiv
        return None
    raise ValueError(op)


def dims_n(case):
    p = case["params"]
    return max(p.get("m", 1), p.get("n", 1), p.get("k", 1))


@pytest.mark.parametrize("batch", [1, 5])
def test_golden_cases(batch):
    z, cases = load_golden()
    for case in cases:
        if case["op"] == "pack":
            continue
        hm = host_inputs(z, case, batch)
        dm = {}
        for lab, h in hm.items():
            if lab not in case["alias"]:
                dm[lab] = dev(h)
        for lab, tgt in case["alias"].items():
            dm[lab] = dm[tgt]
        info = run_product(case, dm)
        torch.cuda.synchronize()
        if info is not None:
            assert np.all(info.cpu().numpy() == case["status"]), (case["name"], info.cpu().numpy(), case["status"])
        for lab in out_labels(case):
            want = z[f"{case['key']}/out/{lab}"]
            got = host(dm[lab])[:, : want.size]
            h = hm[lab]
            mask = written_mask(case, lab, want.size, h.cn, case["status"])
            if case["op"] in ("potrf_l", "syrk_potrf_ln") and lab == case["alias"].get("D", "D"):
                mask[h.diag_off + case["params"]["dj"]: h.diag_off + case["params"]["dj"] + case["params"]["n"]] = True
            for b in range(batch):
                compare_storage(got[b], want, mask, dims_n(case), f"{case['name']}/{lab}/item{b}")


# ---------------------------------------------------------------------------
# random batches against the oracle


def rand_batch(rng, nb, m, n, fill=None):
    h = O.HostBatch(nb, m, n)
    h.storage[:] = rng.uniform(-1, 1, h.storage.shape) if fill is None else fill
    return h


GEMM_SHAPES = [(4, 4, 4), (4, 4, 8), (3, 2, 16), (4, 3, 13), (8, 8, 8), (12, 12, 12), (16, 16, 16), (20, 20, 20), (24, 24, 24), (3, 17, 5),
               (28, 28, 28), (32, 32, 32), (40, 40, 40), (44, 36, 52), (64, 64, 64), (72, 72, 72), (100, 100, 100),
               (128, 128, 128), (300, 300, 300), (65, 130, 7), (9, 70, 33)]


@pytest.mark.parametrize("mnk", GEMM_SHAPES)
def test_gemm_nt_random_vs_oracle(mnk):
    m, n, k = mnk
    rng = np.random.default_rng(m * 10007 + n * 101 + k)
    nb = 3 if m >= 128 else 17
    for (oa, ob, oc, od, alpha, beta) in [((0, 0), (0, 0), (0, 0), (0, 0), 1.0, 1.0),
                                          ((3, 1), (1, 2), (2, 0), (1, 3), -1.5, 0.5),
                                          ((4, 0), (0, 4), (0, 0), (4, 1), 1.0, 0.0)]:
        A = rand_batch(rng, nb, oa[0] + m + 1, oa[1] + k + 2)
        B = rand_batch(rng, nb, ob[0] + n + 2, ob[1] + k + 1)
        C = rand_batch(rng, nb, oc[0] + m, oc[1] + n)
        D = rand_batch(rng, nb, od[0] + m + 3, od[1] + n + 1)
        dA, dB, dC, dD = dev(A), dev(B), dev(C), dev(D)
        level3.gemm_nt(m, n, k, alpha, dA.ref(*oa), dB.ref(*ob), beta, dC.ref(*oc), dD.ref(*od))
        O.gemm_nt(m, n, k, alpha, A, *oa, B, *ob, beta, C, *oc, D, *od)
        mask = np.zeros(D.per, dtype=bool)
        for i in range(m):
            for j in range(n):
                mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
        compare_storage(host(dD), D.storage, mask, max(m, n, k), f"gemm {mnk} {oa}{od}")


@pytest.mark.parametrize("mk", [(4, 3), (8, 8), (13, 5), (24, 24), (33, 17), (40, 40), (64, 64), (96, 40),
                                (128, 64), (200, 31)])
def test_syrk_ln_random_vs_oracle(mk):
    m, k = mk
    rng = np.random.default_rng(m * 31 + k)
    nb = 9
    for (oa, same, od, alpha, beta) in [((0, 0), False, (0, 0), 1.0, 1.0), ((3, 1), True, (0, 0), -1.0, 1.0),
                                        ((3, 1), True, (3, 1), -1.0, 1.0), ((1, 0), False, (2, 2), 0.5, 0.0)]:
        A = rand_batch(rng, nb, oa[0] + m + 2, oa[1] + k + 1)
        B = A if same else rand_batch(rng, nb, m + 1, k + 2)
        ob = oa if same else (0, 1)
        if not same:
            ob = (1, 1)
            B = rand_batch(rng, nb, ob[0] + m, ob[1] + k)
        C = rand_batch(rng, nb, m + 1, m + 2)
        D = rand_batch(rng, nb, od[0] + m + 1, od[1] + m)
        dA = dev(A)
        dB = dA if same else dev(B)
        dC, dD = dev(C), dev(D)
        level3.syrk_ln(m, k, alpha, dA.ref(*oa), dB.ref(*ob), beta, dC.ref(1, 0), dD.ref(*od))
        O.syrk_ln(m, k, alpha, A, *oa, B, *ob, beta, C, 1, 0, D, *od)
        mask = np.zeros(D.per, dtype=bool)
        for j in range(m):
            for i in range(j, m):
                mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
        compare_storage(host(dD), D.storage, mask, max(m, k), f"syrk {mk} {oa}{od}")


def spd_batch(rng, nb, n, shift=None):
    g = rng.uniform(-1, 1, (nb, n, n))
    return g @ g.transpose(0, 2, 1) + (n if shift is None else shift) * np.eye(n)


@pytest.mark.parametrize("mn", [(4, 4), (8, 8), (11, 11), (16, 16), (17, 17), (24, 24), (32, 32), (37, 37), (41, 41),
                                (57, 57), (63, 63), (64, 64), (65, 65), (72, 72), (90, 90), (96, 96), (113, 113),
                                (120, 120), (128, 128), (129, 129), (136, 136), (160, 160), (200, 200), (232, 232),
                                (256, 256), (300, 300), (29, 13), (256, 128), (70, 33), (320, 240), (300, 264),
                                (520, 40), (600, 20), (600, 200), (520, 520)])
def test_potrf_l_random_vs_oracle(mn):
    m, n = mn
    rng = np.random.default_rng(m * 7 + n)
    nb = 4 if m >= 128 else 13
    for (oc, od) in [((0, 0), (0, 0)), ((3, 2), (4, 1)), ((1, 1), (1, 1))]:
        a = spd_batch(rng, nb, m)[:, :, :n]
        if m > n:
            a[:, n:, :] = rng.uniform(-1, 1, (nb, m - n, n))
        C = rand_batch(rng, nb, oc[0] + m + 1, oc[1] + n + 2)
        C.set_window(oc[0], oc[1], a)
        D = rand_batch(rng, nb, od[0] + m, od[1] + n + 1, fill=1.25)
        dC, dD = dev(C), dev(D)
        info = level3.potrf_l(m, dC.ref(*oc), dD.ref(*od), n=n, check=False)
        winfo = O.potrf_l(m, C, *oc, D, *od, n=n)
        assert np.array_equal(info.cpu().numpy(), winfo)
        mask = np.zeros(D.per, dtype=bool)
        for j in range(n):
            for i in range(j, m):
                mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
        mask[D.diag_off + od[1]: D.diag_off + od[1] + n] = True
        compare_storage(host(dD), D.storage, mask, m, f"potrf {mn} {oc}{od}")


@pytest.mark.parametrize("mnf", [(109, 31, 29), (109, 31, 3), (391, 55, 54), (200, 101, 100), (90, 70, 69), (40, 13, 12)])
@pytest.mark.parametrize("off", [(0, 0), (1, 3)])
def test_potrf_tall_failure_in_last_row_panel(mnf, off):
    """Tall window, n % 4 != 0, failing pivot in the square's last row panel: that panel reaches into the rows
    below the square, and the reference's row-panel order has solved them against the columns left of the
    panel before it stops (ccore.pyx:884-899).  The factor + solve path must write exactly that."""
    m, n, f = mnf
    rng = np.random.default_rng(m + n + f)
    nb = 5
    a = np.zeros((nb, m, n))
    a[:, :n] = spd_batch(rng, nb, n)
    a[:, n:] = rng.uniform(-1, 1, (nb, m - n, n))
    a[1, f, f] = -3.0
    a[3, f // 2, f // 2] = -1.0
    C = rand_batch(rng, nb, off[0] + m + 1, off[1] + n + 2)
    C.set_window(off[0], off[1], a)
    D = rand_batch(rng, nb, m + 2, n + 3, fill=0.75)
    dC, dD = dev(C), dev(D)
    info = level3.potrf_l(m, dC.ref(*off), dD, n=n, check=False).cpu().numpy()
    winfo = O.potrf_l(m, C, off[0], off[1], D, 0, 0, n=n)
    assert np.array_equal(info, winfo) and winfo[1] == f
    got = host(dD)
    for b in range(nb):
        gb, wb = got[b, : D.storage.shape[1]], D.storage[b]
        assert np.allclose(gb, wb, rtol=1e-10, atol=1e-10, equal_nan=True), (mnf, off, b)


@pytest.mark.parametrize("n", [4, 8, 12, 16, 17, 24, 40, 57, 64, 72, 100, 128, 136, 200, 256, 300])
@pytest.mark.parametrize("off", [(0, 0), (1, 1)])
def test_potrf_failure_index_and_partial_writes(n, off):
    """Bad pivots: info equals the reference's index, and the failing item is
    written exactly as far as the reference writes it (ccore.pyx:884-899);
    an unaligned D window (di % 4 != 0) of a failing item is left untouched
    except for diag_inv (level3.py:338-344)."""
    rng = np.random.default_rng(n)
    nb = 16
    a = spd_batch(rng, nb, n)
    fails = rng.integers(0, n, nb)
    for b in range(nb):
        if b % 3 != 2:  # keep some items healthy
            a[b, fails[b], fails[b]] = -10.0 * n
    a[5, 0, 0] = np.nan  # NaN passes the d <= 0 test (ccore.pyx:423)
    C = rand_batch(rng, nb, n + off[0], n + off[1])
    C.set_window(off[0], off[1], a)
    D = rand_batch(rng, nb, n + off[0], n + off[1], fill=2.5)
    dC, dD = dev(C), dev(D)
    info = level3.potrf_l(n, dC.ref(*off), dD.ref(*off), check=False).cpu().numpy()
    winfo = O.potrf_l(n, C, off[0], off[1], D, off[0], off[1])
    assert np.array_equal(info, winfo)
    got = host(dD)
    for b in range(nb):
        g, w = got[b], D.storage[b]
        gn, wn = np.isnan(g), np.isnan(w)
        assert np.array_equal(gn, wn), b
        same = np.isclose(g, w, rtol=1e-11, atol=1e-11) | (gn & wn)
        assert np.all(same), (b, info[b])
    with pytest.raises(pb.NotPositiveDefiniteError) as ei:
        level3.potrf_l(n, dC.ref(*off), dD.ref(*off))
    first = int(np.nonzero(winfo >= 0)[0][0])
    assert ei.value.batch_index == first and ei.value.index == winfo[first]
    assert not dD.diag_inv_valid(0, n)


@pytest.mark.parametrize("n", [24, 40, 57, 64])
def test_potrf_nonfinite_inputs_keep_reference_pattern(n):
    """A NaN / Inf off the diagonal (17 <= n <= 64, the register-tile
    kernel): the NaN/Inf pattern of D and info equal the reference's -- such
    items are redone in the reference's own operation order (pb_exact.cu);
    finite entries agree within tolerance."""
    rng = np.random.default_rng(100 + n)
    nb = 6
    a = spd_batch(rng, nb, n)
    i0 = n // 2 + 3
    a[0, i0, 5] = np.nan           # row i0, early column
    a[1, n - 1, n - 3] = np.nan     # last row
    a[2, i0, i0 - 1] = np.inf       # next to the diagonal
    a[3, 9, 2] = -np.inf
    C = rand_batch(rng, nb, n, n)
    C.set_window(0, 0, a)
    D = rand_batch(rng, nb, n, n, fill=0.5)
    dC, dD = dev(C), dev(D)
    info = level3.potrf_l(n, dC, dD, check=False).cpu().numpy()
    winfo = O.potrf_l(n, C, 0, 0, D, 0, 0)
    assert np.array_equal(info, winfo)
    got = host(dD)
    for b in range(nb):
        g, w = got[b], D.storage[b]
        assert np.array_equal(np.isnan(g), np.isnan(w)), (n, b)
        assert np.array_equal(np.isinf(g), np.isinf(w)), (n, b)
        fin = np.isfinite(w)
        assert np.allclose(g[fin], w[fin], rtol=1e-11, atol=1e-11), (n, b)


@pytest.mark.parametrize("mn", [(12, 8), (40, 24), (72, 48), (30, 64), (80, 72)])
def test_trsm_reuse_after_unchecked_failing_potrf(mn):
    """potrf_l(check=False) with failing items, then trsm_rltn on the factor:
    healthy items reuse diag_inv, failed items recompute 1/A[j,j] like the
    reference, whose failed potrf invalidates diag_inv (level3.py:346-349)."""
    m, n = mn
    rng = np.random.default_rng(m + 31 * n)
    nb = 9
    a = spd_batch(rng, nb, n)
    bad = [1, 4, 7]
    for b in bad:
        f = int(rng.integers(1, n))
        a[b, f, f] = -5.0 * n
    a[4, 0, 0] = 0.0  # fails at pivot 0: its L is untouched, 1/A[0,0] of the old D -> zero pivot below
    C = rand_batch(rng, nb, n, n)
    C.set_window(0, 0, a)
    L = rand_batch(rng, nb, n, n, fill=0.75)
    dC, dL = dev(C), dev(L)
    pinfo = level3.potrf_l(n, dC, dL, check=False)
    winfo = O.potrf_l(n, C, 0, 0, L, 0, 0)
    assert np.array_equal(pinfo.cpu().numpy(), winfo)
    assert dL.diag_inv_valid(0, n) and dL.diag_info is not None
    if 4 in bad:  # force a zero pivot on the failed item 4's stale diagonal
        L.storage[4, O.element_offset(0, 0, L.cn)] = 0.0
        dL = dev(L)
        dL.diag_lo, dL.diag_hi, dL.diag_info = 0, n, pinfo
    B = rand_batch(rng, nb, m, n)
    X = rand_batch(rng, nb, m, n, fill=-2.0)
    dB, dX = dev(B), dev(X)
    info = level3.trsm_rltn(m, n, 1.0, dL, dB, dX, check=False).cpu().numpy()
    got = host(dX)
    ok = [b for b in range(nb) if b not in bad]
    for idx, valid in ((ok, True), (bad, False)):
        hL = O.HostBatch(len(idx), n, n, L.storage[idx].copy())
        if valid:
            hL.diag_lo, hL.diag_hi = 0, n
        hB = O.HostBatch(len(idx), m, n, B.storage[idx].copy())
        hX = O.HostBatch(len(idx), m, n, X.storage[idx].copy())
        want_info = O.trsm_rltn(m, n, 1.0, hL, 0, 0, hB, 0, 0, hX, 0, 0)
        assert np.array_equal(info[idx], want_info), (idx, info[idx], want_info)
        mask = window_mask(hX, (0, 0), m, n)
        for k, b in enumerate(idx):
            compare_storage(got[b], hX.storage[k], mask, n, f"trsm reuse item {b}")
    assert info[4] == 0
    with pytest.raises(pb.SingularMatrixError) as ei:
        level3.trsm_rltn(m, n, 1.0, dL, dB, dX)
    assert ei.value.batch_index == 4


def test_potrf_concurrent_streams_disjoint_items():
    """Two streams factor disjoint item ranges of one batch at the same time
    (the stream contract in include/pb_b200.h): the result equals one call."""
    rng = np.random.default_rng(77)
    for n in (4, 8, 32, 100):
        nb = 4096 if n <= 8 else 512
        C = rand_batch(rng, nb, n, n)
        C.set_window(0, 0, spd_batch(rng, nb, n))
        dC = dev(C)
        ref = alloc(nb, n, n, zero=True)
        level3.potrf_l(n, dC, ref)
        out = alloc(nb, n, n, zero=True)
        half = nb // 2 + 1
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            level3.potrf_l(n, dC.shard(0, half), out.shard(0, half), check=False)
        with torch.cuda.stream(s2):
            level3.potrf_l(n, dC.shard(half, nb), out.shard(half, nb), check=False)
        torch.cuda.synchronize()
        assert torch.equal(out.item_storage(), ref.item_storage()), n


@pytest.mark.parametrize("mn", [(2, 2), (5, 3), (8, 8), (3, 9), (13, 6), (72, 48), (40, 64), (33, 100), (16, 232),
                                (24, 256), (9, 300),
                                # register-strip kernel (m >= 64, 64 <= n <= 128, aligned A): full / ragged strips and blocks
                                (72, 64), (100, 72), (130, 125), (64, 128)])
def test_trsm_rltn_random_vs_oracle(mn):
    m, n = mn
    rng = np.random.default_rng(m * 3 + n)
    nb = 6
    L = np.linalg.cholesky(spd_batch(rng, nb, n))
    for (oa, ob, od, reuse) in [((0, 0), (0, 0), (0, 0), False), ((3, 3), (1, 1), (1, 2), False),
                                ((0, 0), (0, 0), (0, 0), True), ((4, 4), (2, 0), (0, 0), True)]:
        A = rand_batch(rng, nb, oa[0] + n + 1, oa[1] + n + 2)
        if reuse:
            S = rand_batch(rng, nb, oa[0] + n + 1, oa[1] + n + 2)
            S.set_window(oa[0], oa[1], spd_batch(rng, nb, n))
            O.potrf_l(n, S, *oa, A, *oa)  # oracle factor + valid diag_inv (level3.py:169-170)
            dA = dev(A)
            assert dA.diag_inv_valid(oa[1], n)
        else:
            A.set_window(oa[0], oa[1], L)
            dA = dev(A)
        B = rand_batch(rng, nb, ob[0] + m, ob[1] + n + 1)
        D = rand_batch(rng, nb, od[0] + m + 2, od[1] + n)
        dB, dD = dev(B), dev(D)
        info = level3.trsm_rltn(m, n, -1.5, dA.ref(*oa), dB.ref(*ob), dD.ref(*od), check=False)
        winfo = O.trsm_rltn(m, n, -1.5, A, *oa, B, *ob, D, *od)
        if info is not None:
            assert np.array_equal(info.cpu().numpy(), winfo)
        mask = np.zeros(D.per, dtype=bool)
        for i in range(m):
            for j in range(n):
                mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
        compare_storage(host(dD), D.storage, mask, n, f"trsm {mn} {oa}{od} reuse={reuse}")


def test_trsm_zero_pivot_leaves_item_untouched():
    rng = np.random.default_rng(3)
    for n, m in ((4, 7), (48, 7), (256, 7), (96, 70)):
        nb = 5
        L = np.linalg.cholesky(spd_batch(rng, nb, n))
        L[2, n // 2, n // 2] = 0.0
        A = rand_batch(rng, nb, n, n)
        A.set_window(0, 0, L)
        B = rand_batch(rng, nb, m, n)
        D = rand_batch(rng, nb, m, n, fill=4.0)
        dA, dB, dD = dev(A), dev(B), dev(D)
        info = level3.trsm_rltn(m, n, 1.0, dA, dB, dD, check=False).cpu().numpy()
        assert list(info) == [-1, -1, n // 2, -1, -1]
        assert np.all(host(dD)[2] == 4.0)
        with pytest.raises(pb.SingularMatrixError) as ei:
            level3.trsm_rltn(m, n, 1.0, dA, dB, dD)
        assert ei.value.index == n // 2 and ei.value.batch_index == 2


# ---------------------------------------------------------------------------
# discrete semantics (exact)


def test_gemm_special_cases_exact():
    rng = np.random.default_rng(5)
    for (m, n, k) in [(3, 5, 7), (8, 2, 7), (40, 40, 40), (70, 66, 9), (4, 4, 4)]:  # 4x4x4: the staged kernel
        nb = 4 if m != 4 else 300  # more than one 128-item round, ragged last round
        c = rng.uniform(-1, 1, (nb, m, n))
        dC = pack.panel_from_array(c)
        nanA = pack.panel_from_array(np.full((nb, m, k), np.nan))
        nanB = pack.panel_from_array(np.full((nb, n, k), np.nan))
        dD = alloc(nb, m, n, zero=True)
        level3.gemm_nt(m, n, k, 0.0, nanA, nanB, 1.0, dC, dD)  # alpha=0: A*B ignored even if NaN
        assert np.array_equal(pack.panel_to_array(dD).cpu().numpy(), c)
        level3.gemm_nt(m, n, k, 0.0, nanA, nanB, -2.0, dC, dD)
        assert np.array_equal(pack.panel_to_array(dD).cpu().numpy(), -2.0 * c)
        a = pack.panel_from_array(rng.uniform(-1, 1, (nb, m, k)))
        b = pack.panel_from_array(rng.uniform(-1, 1, (nb, n, k)))
        nanC = pack.panel_from_array(np.full((nb, m, n), np.nan))
        level3.gemm_nt(m, n, k, 1.0, a, b, 0.0, nanC, dD)  # beta=0: C never read
        assert not torch.isnan(pack.panel_to_array(dD)).any()
        level3.gemm_nt(m, n, 0, 1.0, a, b, 0.5, dC, dD)  # k=0: D = beta*C
        assert np.array_equal(pack.panel_to_array(dD).cpu().numpy(), 0.5 * c)
        before = dD.storage.clone()
        level3.gemm_nt(0, n, k, 1.0, a, b, 0.0, dC, dD)  # m=0 / n=0: no-op
        level3.gemm_nt(m, 0, k, 1.0, a, b, 0.0, dC, dD)
        assert torch.equal(before, dD.storage)


def test_gemm4_staged_inplace_broadcast_and_window():
    """m = n = k = 4 (cooperatively staged kernel): D == C in place, a broadcast B (stride 0), column-offset
    windows and several rounds with a ragged tail, against the oracle item by item."""
    rng = np.random.default_rng(44)
    nb = 389
    A = rand_batch(rng, nb, 4, 9)
    B = rand_batch(rng, 1, 4, 6)
    C = rand_batch(rng, nb, 8, 7)
    dA, dB, dC = dev(A), dev(B), dev(C)
    want = C.storage.copy()
    for b in range(nb):
        a = A.window(0, 5, 4, 4)[b]
        bm = B.window(0, 2, 4, 4)[0]
        c = C.window(4, 3, 4, 4)[b]
        res = np.zeros((4, 4))
        for i in range(4):
            for j in range(4):
                acc = 0.0
                for l in range(4):
                    acc = np.float64(a[i, l]) * bm[j, l] + acc
                res[i, j] = 0.75 * acc + (-0.5) * c[i, j]
        for i in range(4):
            for j in range(4):
                want[b, O.element_offset(4 + i, 3 + j, C.cn)] = res[i, j]
    level3.gemm_nt(4, 4, 4, 0.75, dA.ref(0, 5), dB.ref(0, 2), -0.5, dC.ref(4, 3), dC.ref(4, 3))
    got = host(dC)
    mask = np.zeros(C.per, dtype=bool)
    for i in range(4):
        for j in range(4):
            mask[O.element_offset(4 + i, 3 + j, C.cn)] = True
    compare_storage(got, want, mask, 4, "gemm4 staged in place")


def test_aliasing_and_determinism_bit_exact():
    rng = np.random.default_rng(6)
    for (m, k) in [(9, 5), (40, 33), (96, 40)]:
        nb = 6
        a = pack.panel_from_array(rng.uniform(-1, 1, (nb, m, k)))
        c = rng.uniform(-1, 1, (nb, m, m))
        alias = pack.panel_from_array(c)
        sep = alloc(nb, m, m, zero=True)
        level3.gemm_nt(m, m, k, 1.0, a, a, 0.5, alias, alias)
        level3.gemm_nt(m, m, k, 1.0, a, a, 0.5, pack.panel_from_array(c), sep)
        assert torch.equal(pack.panel_to_array(alias), pack.panel_to_array(sep))
        alias = pack.panel_from_array(c)
        sep2 = alloc(nb, m, m, zero=True)
        level3.syrk_ln(m, k, 1.0, a, a, 0.5, alias, alias)
        level3.syrk_ln(m, k, 1.0, a, a, 0.5, pack.panel_from_array(c), sep2)
        assert torch.equal(torch.tril(pack.panel_to_array(alias)), torch.tril(pack.panel_to_array(sep2)))
        s = spd_batch(rng, nb, m)
        inplace = pack.panel_from_array(s)
        out = alloc(nb, m, m, zero=True)
        level3.potrf_l(m, inplace, inplace)
        level3.potrf_l(m, pack.panel_from_array(s), out)
        assert torch.equal(torch.tril(pack.panel_to_array(inplace)), torch.tril(pack.panel_to_array(out)))
        assert torch.equal(inplace.diag_inv, out.diag_inv)
        bm = pack.panel_from_array(rng.uniform(-1, 1, (nb, 7, m)))
        x1 = alloc(nb, 7, m, zero=True)
        level3.trsm_rltn(7, m, 1.0, out, bm, x1)
        x2 = alloc(nb, 7, m, zero=True)
        pack.gecp(7, m, bm, x2)
        level3.trsm_rltn(7, m, 1.0, out, x2, x2)  # D == B in place
        assert torch.equal(x1.storage, x2.storage)
        # determinism: same inputs, bit-identical outputs run to run
        x3 = alloc(nb, 7, m, zero=True)
        level3.trsm_rltn(7, m, 1.0, out, bm, x3)
        assert torch.equal(x1.storage, x3.storage)
        if m >= 64:  # register-strip trsm kernel (m >= 64 rows): D == B in place, bit for bit
            bw = pack.panel_from_array(rng.uniform(-1, 1, (nb, 70, m)))
            y1 = alloc(nb, 70, m, zero=True)
            level3.trsm_rltn(70, m, 1.0, out, bw, y1)
            y2 = alloc(nb, 70, m, zero=True)
            pack.gecp(70, m, bw, y2)
            level3.trsm_rltn(70, m, 1.0, out, y2, y2)
            assert torch.equal(y1.storage, y2.storage)


def test_broadcast_operand():
    rng = np.random.default_rng(11)
    nb, m, n, k = 8, 12, 10, 9
    a = rng.uniform(-1, 1, (nb, m, k))
    b1 = rng.uniform(-1, 1, (1, n, k))
    dA, dB1 = pack.panel_from_array(a), pack.panel_from_array(b1)
    dD = alloc(nb, m, n, zero=True)
    level3.gemm_nt(m, n, k, 1.0, dA, dB1, 0.0, dD, dD)
    want = a @ b1[0].T
    assert O.rel_fro(pack.panel_to_array(dD).cpu().numpy(), want) < O.tol(k)


# ---------------------------------------------------------------------------
# pack / unpack / gecp: bit-exact


def test_pack_unpack_roundtrip_bit_exact():
    rng = np.random.default_rng(2)
    for trial in range(60):
        nb = int(rng.integers(1, 6))
        m, n = int(rng.integers(0, 40)), int(rng.integers(0, 40))
        ai, aj = int(rng.integers(0, 9)), int(rng.integers(0, 9))
        arr = rng.uniform(-1, 1, (nb, m, n))
        big = alloc(nb, ai + m + 3, aj + n + 3, zero=True)
        src = pack.ColBatch.from_array(arr)
        pack.pack_matrix(src, m, n, big.ref(ai, aj))
        out = pack.ColBatch.from_array(np.zeros((nb, m, n)))
        pack.unpack_matrix(big.ref(ai, aj), m, n, out)
        assert np.array_equal(out.to_array().cpu().numpy(), arr), (m, n, ai, aj)
        # panel bytes equal the oracle's kpack_cm (and padding untouched)
        h = O.HostBatch(nb, ai + m + 3, aj + n + 3)
        cm = np.ascontiguousarray(arr.transpose(0, 2, 1)).reshape(nb, -1)
        if m * n:
            O.pack_cm(m, n, cm.reshape(-1), max(m, 1), m * n, h, ai, aj)
        assert np.array_equal(host(big).view(np.uint64), h.storage.view(np.uint64))
        # row-major bridges
        back = pack.panel_to_array(big.ref(ai, aj), m, n).cpu().numpy()
        assert np.array_equal(back, arr)
        big2 = alloc(nb, ai + m + 3, aj + n + 3, zero=True)
        pack.gecp(m, n, big.ref(ai, aj), big2.ref(ai, aj))
        assert torch.equal(big.storage, big2.storage)


def test_pack_kat_element_46():
    d = alloc(2, 8, 8, zero=True)
    pack.pack_matrix(pack.ColBatch.from_array(np.full((2, 1, 1), 5.0)), 1, 1, d.ref(6, 3))
    assert torch.all(d.data[:, 46] == 5.0) and float(d.data.abs().sum()) == 10.0


# ---------------------------------------------------------------------------
# BASELINE-size batches: sampled oracle + size-independent properties


def test_config1_full_batch_sampled():
    """C1: gemm_nt 64^3, alpha=beta=1, batch 4096 (BASELINE configs[0])."""
    nb, s = 4096, 64
    g = torch.Generator(device="cuda").manual_seed(1)
    A, B, C = (alloc(nb, s, s) for _ in range(3))
    for x in (A, B, C):
        x.storage.uniform_(-1, 1, generator=g)
    D = alloc(nb, s, s, zero=True)
    level3.gemm_nt(s, s, s, 1.0, A, B, 1.0, C, D)
    # linearity: gemm(2A) - 2 gemm(A) with beta=0 is exactly zero
    D2 = alloc(nb, s, s, zero=True)
    A2 = pb.create_panel_batch(nb, s, s, A.storage * 2.0,
                               None if A.diag_storage is None else A.diag_storage.clone())
    level3.gemm_nt(s, s, s, 1.0, A2, B, 0.0, C, D2)
    D1 = alloc(nb, s, s, zero=True)
    level3.gemm_nt(s, s, s, 1.0, A, B, 0.0, C, D1)
    assert torch.equal(D2.data, 2.0 * D1.data)
    idx = np.random.default_rng(0).choice(nb, 12, replace=False)
    sub = torch.as_tensor(idx, device="cuda")
    hA, hB, hC = (O.HostBatch(12, s, s, x.item_storage()[sub].cpu().numpy()) for x in (A, B, C))
    hD = O.HostBatch(12, s, s)
    O.gemm_nt(s, s, s, 1.0, hA, 0, 0, hB, 0, 0, 1.0, hC, 0, 0, hD, 0, 0)
    fp_close(D.data[sub].cpu().numpy(), hD.storage[:, : 64 * 64], s, "C1 sample")


@pytest.mark.parametrize("n", [4, 16, 64, 256])
def test_config2_potrf_large_batch_residual(n):
    """C2: potrf at large batch: residual ||L L^T - A|| / ||A|| and sampled oracle."""
    nb = {4: 1 << 20, 16: 1 << 16, 64: 8192, 256: 256}[n]
    g = torch.Generator(device="cuda").manual_seed(n)
    M = torch.rand((nb, n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = M @ M.transpose(1, 2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
    C = pack.panel_from_array(a)
    D = alloc(nb, n, n, zero=True)
    info = level3.potrf_l(n, C, D)
    assert int((info >= 0).sum()) == 0
    L = torch.tril(pack.panel_to_array(D))
    res = torch.linalg.matrix_norm(L @ L.transpose(1, 2) - a) / torch.linalg.matrix_norm(a)
    assert float(res.max()) <= 50 * n * EPS
    dinv = D.diag_inv
    assert float((dinv * torch.diagonal(L, dim1=1, dim2=2) - 1).abs().max()) <= 4 * EPS
    idx = torch.as_tensor(np.random.default_rng(n).choice(nb, 8, replace=False), device="cuda")
    hC = O.HostBatch(8, n, n, C.item_storage()[idx].cpu().numpy())
    hD = O.HostBatch(8, n, n)
    O.potrf_l(n, hC, 0, 0, hD, 0, 0)
    fp_close(torch.tril(L[idx]).cpu().numpy(), np.tril(hD.window(0, 0, n, n)), n, "C2 sample")


@pytest.mark.parametrize("n", list(range(1, 17)))
def test_potrf_small_bit_exact(n):
    """n <= 16 runs the register kernel that follows the reference's operation
    order exactly: factor and diag_inv are bit-identical to the oracle (and so
    to the reference's compiled core), including failing items."""
    rng = np.random.default_rng(100 + n)
    nb = 300
    a = spd_batch(rng, nb, n)
    for b in range(0, nb, 7):
        f = int(rng.integers(0, n))
        a[b, f, f] = -1.0 - 10.0 * n
    C = rand_batch(rng, nb, n, n)
    C.set_window(0, 0, a)
    D = rand_batch(rng, nb, n, n, fill=-3.25)
    dC, dD = dev(C), dev(D)
    info = level3.potrf_l(n, dC, dD, check=False).cpu().numpy()
    winfo = O.potrf_l(n, C, 0, 0, D, 0, 0)
    assert np.array_equal(info, winfo)
    assert np.array_equal(host(dD).view(np.uint64), D.storage.view(np.uint64))


@pytest.mark.parametrize("n", list(range(1, 17)))
def test_potrf_small_in_place_and_offset_bit_exact(n):
    """D == C in place, and a D window at a column offset inside a wider
    matrix: the small kernels re-store whole 32-byte sectors of D, so every
    byte outside the reference's write set (strict upper, padding rows, the
    columns beside the window) must come back unchanged, bit for bit."""
    rng = np.random.default_rng(200 + n)
    nb = 97
    a = spd_batch(rng, nb, n)
    for b in range(3, nb, 11):
        f = int(rng.integers(0, n))
        a[b, f, f] = -2.0
    C = rand_batch(rng, nb, n, n)
    C.set_window(0, 0, a)
    dC = dev(C)
    info = level3.potrf_l(n, dC, dC, check=False).cpu().numpy()
    winfo = O.potrf_l(n, C, 0, 0, C, 0, 0)
    assert np.array_equal(info, winfo)
    assert np.array_equal(host(dC).view(np.uint64), C.storage.view(np.uint64))
    # D at (4, 3) of a (n+5) x (n+6) matrix pre-filled with random bytes
    C2 = rand_batch(rng, nb, n, n)
    C2.set_window(0, 0, a)
    D = rand_batch(rng, nb, n + 5, n + 6)
    dC2, dD = dev(C2), dev(D)
    info = level3.potrf_l(n, dC2, dD.ref(4, 3), check=False).cpu().numpy()
    winfo = O.potrf_l(n, C2, 0, 0, D, 4, 3)
    assert np.array_equal(info, winfo)
    assert np.array_equal(host(dD).view(np.uint64), D.storage.view(np.uint64))


@pytest.mark.parametrize("batch", [1, 6])
def test_getrf_golden_bit_exact(batch):
    """§8f getrf against the reference's own recorded outputs: storage
    (partial state of failing items included), ipiv and diag validity, bit
    for bit, replicated over a batch."""
    z, cases = load_golden("golden_getrf_v1.npz")
    for case in cases:
        hm = host_inputs(z, case, batch)
        dm = {}
        for lab, h in hm.items():
            if lab not in case["alias"]:
                dm[lab] = dev(h)
        for lab, tgt in case["alias"].items():
            dm[lab] = dm[tgt]
        dD = dm[case["alias"].get("D", "D")]
        nb = dD.batch
        p = case["params"]
        mn = max(min(p["m"], p["n"]), 1)
        ipiv = torch.full((nb, mn), -7, dtype=torch.int64, device="cuda")
        fn = level3.getrf_pivot if p["pivot"] else level3.getrf_nopivot
        args = (p["m"], p["n"], dm["C"].ref(p["ci"], p["cj"]), dD.ref(p["di"], p["dj"]))
        if case["status"] >= 0:
            with pytest.raises(pb.SingularMatrixError) as ei:
                fn(*args, ipiv=ipiv) if p["pivot"] else fn(*args)
            assert ei.value.index == case["status"] and ei.value.batch_index == 0, case["name"]
        else:
            fn(*args, ipiv=ipiv) if p["pivot"] else fn(*args)
        for lab in out_labels(case):
            want = z[f"{case['key']}/out/{lab}"]
            got = host(dm[lab])[:, : want.size]
            for b in range(batch):
                assert np.array_equal(got[b].view(np.uint64), want.view(np.uint64)), (case["name"], lab, b)
        if p["pivot"]:
            want_piv = z[f"{case['key']}/ipiv"]
            got_piv = ipiv.cpu().numpy()
            for b in range(batch):
                assert np.array_equal(got_piv[b, : want_piv.size], want_piv), (case["name"], b)
        assert [dD.diag_lo, dD.diag_hi] == case["valid_out"]["D"], case["name"]


@pytest.mark.parametrize("mn", [(4, 4), (9, 9), (16, 16), (23, 17), (17, 30), (32, 32), (48, 48), (64, 64), (100, 60)])
def test_getrf_random_vs_oracle_bit_exact(mn):
    """Random batches (pivot and no pivot), window offsets, in place, and a
    few singular items: storage, info and ipiv equal the oracle's bit for bit."""
    m, n = mn
    rng = np.random.default_rng(31 * m + n)
    nb = 37
    for pivot in (True, False):
        for (oc, od) in [((0, 0), (0, 0)), ((3, 2), (4, 1)), ((1, 0), (2, 3))]:
            a = rng.uniform(-1, 1, (nb, m, n))
            if not pivot:
                a += 4.0 * np.eye(m, n)
            for b in range(2, nb, 9):
                a[b, :, min(m, n) // 2] = 0.0  # singular column
            C = rand_batch(rng, nb, oc[0] + m + 1, oc[1] + n + 2)
            C.set_window(oc[0], oc[1], a)
            D = rand_batch(rng, nb, od[0] + m + 2, od[1] + n + 1)
            dC, dD = dev(C), dev(D)
            k = min(m, n)
            ipiv = torch.full((nb, k), -7, dtype=torch.int64, device="cuda")
            if pivot:
                level3.getrf_pivot(m, n, dC.ref(*oc), dD.ref(*od), ipiv=ipiv, check=False)
            else:
                info = level3.getrf_nopivot(m, n, dC.ref(*oc), dD.ref(*od), check=False)
            wpiv = np.full((nb, k), -7, dtype=np.int64)
            winfo, wpiv = O.getrf(m, n, C, *oc, D, *od, pivot, ipiv=wpiv)
            assert np.array_equal(host(dD).view(np.uint64), D.storage.view(np.uint64)), (mn, pivot, oc, od)
            if pivot:
                assert np.array_equal(ipiv.cpu().numpy(), wpiv), (mn, oc, od)
            else:
                assert np.array_equal(info.cpu().numpy(), winfo), (mn, oc, od)
    # in place (D == C)
    a = rng.uniform(-1, 1, (nb, m, n))
    C = rand_batch(rng, nb, m, n)
    C.set_window(0, 0, a)
    dC = dev(C)
    ipiv = torch.zeros((nb, min(m, n)), dtype=torch.int64, device="cuda")
    level3.getrf_pivot(m, n, dC, dC, ipiv=ipiv, check=False)
    _, wpiv = O.getrf(m, n, C, 0, 0, C, 0, 0, True)
    assert np.array_equal(host(dC).view(np.uint64), C.storage.view(np.uint64))
    assert np.array_equal(ipiv.cpu().numpy(), wpiv)


def test_getrf_reconstruction_and_edge_rules():
    """P*C = L*U to rounding; m or n == 0 is a no-op; a window too large for
    the shared-memory LU is refused before any launch."""
    rng = np.random.default_rng(5)
    nb, m = 8, 20
    a = rng.uniform(-1, 1, (nb, m, m))
    C = pack.panel_from_array(a)
    D = alloc(nb, m, m, zero=True)
    ipiv = level3.getrf_pivot(m, m, C, D)
    lu = pack.panel_to_array(D).cpu().numpy()
    piv = ipiv.cpu().numpy()
    for b in range(nb):
        lo = np.tril(lu[b], -1) + np.eye(m)
        up = np.triu(lu[b])
        pc = a[b].copy()
        for j in range(m):
            pc[[j, piv[b, j]]] = pc[[piv[b, j], j]]
        assert np.linalg.norm(lo @ up - pc) <= 1e-12 * np.linalg.norm(a[b])
        assert np.max(np.abs(D.diag_inv[b].cpu().numpy() * np.diag(up) - 1.0)) <= 1e-15
    before = D.storage.clone()
    assert level3.getrf_pivot(0, m, C, D) is None and level3.getrf_nopivot(m, 0, C, D) is None
    assert torch.equal(before, D.storage)
    big = alloc(1, 200, 200, zero=True)
    with pytest.raises(RuntimeError):
        level3.getrf_pivot(200, 200, big, big)


def test_riccati_chain_c5_vs_oracle_and_graph_replay():
    """C5 chain: gemm_nt -> syrk_ln -> potrf_l -> trsm_rltn ->
    gemm_nt per stage, batched over problems; eager and CUDA-graph replay are
    bit-identical, and both match the oracle chain."""
    from chain_util import make_problems, oracle_chain, packed_inputs
    from paper_1704_02457_b200.chain import RiccatiChain
    nb, nx, nu, N = 16, 32, 8, 50
    A, B, Q, R = make_problems(nb, nx, nu, seed=3)
    BAt, RQ, P0 = packed_inputs(A, B, Q, R)

    def fresh():
        ch = RiccatiChain(nb, nx, nu)
        pack.pack_array_into(torch.from_numpy(BAt).cuda(), ch.BAt)
        pack.pack_array_into(torch.from_numpy(RQ).cuda(), ch.RQ)
        pack.pack_array_into(torch.from_numpy(P0).cuda(), ch.P)
        return ch

    ch = fresh()
    ch.run(N)
    P = pack.panel_to_array(ch.P).cpu().numpy()
    K = pack.panel_to_array(ch.K).cpu().numpy()
    Pw, Kw = oracle_chain(BAt, RQ, P0, nx, nu, N)
    fp_close(P, Pw, nx + nu, "C5 P_0")
    fp_close(K, Kw, nx + nu, "C5 K")
    g = fresh()
    g.capture(N)  # capture records N stages after one warm-up stage
    g2 = fresh()
    g2.graph = g.graph
    # replaying the graph re-runs exactly the captured launches on g's buffers
    g.P.storage.copy_(g2.P.storage)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(g.P.storage, ch.P.storage)
    assert torch.equal(g.K.storage, ch.K.storage)


def test_riccati_chain_fused_kernel_vs_oracle():
    """The fused persistent chain kernel (pb_driccati_chain) matches the oracle
    chain and the per-stage batched path."""
    from chain_util import make_problems, oracle_chain, packed_inputs
    from paper_1704_02457_b200.chain import RiccatiChain
    for nb, nx, nu, N in [(16, 32, 8, 50), (7, 16, 8, 9), (5, 64, 8, 3), (9, 8, 8, 5), (6, 24, 8, 4), (4, 48, 8, 3)]:
        A, B, Q, R = make_problems(nb, nx, nu, seed=nx)
        BAt, RQ, P0 = packed_inputs(A, B, Q, R)
        ch = RiccatiChain(nb, nx, nu)
        pack.pack_array_into(torch.from_numpy(BAt).cuda(), ch.BAt)
        pack.pack_array_into(torch.from_numpy(RQ).cuda(), ch.RQ)
        pack.pack_array_into(torch.from_numpy(P0).cuda(), ch.P)
        info = ch.run_fused(N)
        assert int((info >= 0).sum()) == 0
        P = pack.panel_to_array(ch.P).cpu().numpy()
        K = pack.panel_to_array(ch.K).cpu().numpy()
        Pw, Kw = oracle_chain(BAt, RQ, P0, nx, nu, N)
        fp_close(P, Pw, nx + nu, f"fused P nx={nx}")
        fp_close(K, Kw, nx + nu, f"fused K nx={nx}")


def test_composite_kkt_schur_and_block_tridiag_vs_oracle():
    """§8f row 2 composites (apps.py:46-59, 268-293) batched on the GPU vs the
    same compositions on the oracle."""
    from paper_1704_02457_b200 import composite
    rng = np.random.default_rng(42)
    nb, n, m = 9, 20, 7
    H = spd_batch(rng, nb, n)
    A = rng.uniform(-1, 1, (nb, m, n))
    f = composite.kkt_schur_factor(n, m, pack.panel_from_array(H), pack.panel_from_array(A))
    hH, hA = O.HostBatch(nb, n, n), O.HostBatch(nb, m, n)
    hH.set_window(0, 0, H)
    hA.set_window(0, 0, A)
    lh, mm, sig, ls = O.HostBatch(nb, n, n), O.HostBatch(nb, m, n), O.HostBatch(nb, m, m), O.HostBatch(nb, m, m)
    O.potrf_l(n, hH, 0, 0, lh, 0, 0)
    O.trsm_rltn(m, n, 1.0, lh, 0, 0, hA, 0, 0, mm, 0, 0)
    O.syrk_ln(m, n, 1.0, mm, 0, 0, mm, 0, 0, 0.0, sig, 0, 0, sig, 0, 0)
    O.potrf_l(m, sig, 0, 0, ls, 0, 0)
    fp_close(np.tril(pack.panel_to_array(f.L_H).cpu().numpy()), np.tril(lh.window(0, 0, n, n)), n, "L_H")
    fp_close(pack.panel_to_array(f.M).cpu().numpy(), mm.window(0, 0, m, n), n, "M")
    fp_close(np.tril(pack.panel_to_array(f.L_S).cpu().numpy()), np.tril(ls.window(0, 0, m, m)), n, "L_S")
    # block tridiagonal, N blocks of nx
    N, nx = 6, 12
    D = [spd_batch(rng, nb, nx, shift=4 * nx) for _ in range(N)]
    E = [rng.uniform(-1, 1, (nb, nx, nx)) for _ in range(N - 1)]
    bt = composite.block_tridiag_chol_factor(N, [pack.panel_from_array(x) for x in D],
                                             [pack.panel_from_array(x) for x in E])
    hd = O.HostBatch(nb, nx, nx)
    hd.set_window(0, 0, D[0])
    Ld = O.HostBatch(nb, nx, nx)
    O.potrf_l(nx, hd, 0, 0, Ld, 0, 0)
    for i in range(1, N):
        he = O.HostBatch(nb, nx, nx)
        he.set_window(0, 0, E[i - 1])
        Lo = O.HostBatch(nb, nx, nx)
        O.trsm_rltn(nx, nx, 1.0, Ld, 0, 0, he, 0, 0, Lo, 0, 0)
        fp_close(pack.panel_to_array(bt.offdiag[i - 1]).cpu().numpy(), Lo.window(0, 0, nx, nx), nx, f"off {i}")
        w = O.HostBatch(nb, nx, nx)
        w.set_window(0, 0, D[i])
        O.syrk_ln(nx, nx, -1.0, Lo, 0, 0, Lo, 0, 0, 1.0, w, 0, 0, w, 0, 0)
        Ld = O.HostBatch(nb, nx, nx)
        O.potrf_l(nx, w, 0, 0, Ld, 0, 0)
        fp_close(np.tril(pack.panel_to_array(bt.diag[i]).cpu().numpy()), np.tril(Ld.window(0, 0, nx, nx)), nx,
                 f"diag {i}")
    # failure message carries the block index like the reference
    bad = [x.copy() for x in D]
    bad[0][3, 2, 2] = -1e3
    with pytest.raises(pb.NotPositiveDefiniteError, match="block 0") as ei:
        composite.block_tridiag_chol_factor(N, [pack.panel_from_array(x) for x in bad],
                                            [pack.panel_from_array(x) for x in E])
    assert ei.value.batch_index == 3 and ei.value.index == 2


# ---------------------------------------------------------------------------
# §8f next tier: gemm_nn, trmm_rlnn, syrk_potrf_ln, batched Riccati recursion

NN_SHAPES = [(4, 4, 4), (8, 8, 8), (16, 16, 16), (24, 24, 24), (3, 17, 5), (28, 28, 28), (32, 32, 32),
             (44, 36, 52), (64, 64, 64), (100, 100, 100), (128, 128, 128), (65, 130, 7), (9, 70, 33), (200, 40, 96)]


def window_mask(h, o, m, n, lower=False):
    mask = np.zeros(h.per, dtype=bool)
    for j in range(n):
        for i in range(j if lower else 0, m):
            mask[O.element_offset(o[0] + i, o[1] + j, h.cn)] = True
    return mask


@pytest.mark.parametrize("mnk", NN_SHAPES)
def test_gemm_nn_random_vs_oracle(mnk):
    m, n, k = mnk
    rng = np.random.default_rng(m * 7919 + n * 13 + k)
    nb = 3 if m >= 128 else 11
    for (oa, ob, oc, od, alpha, beta) in [((0, 0), (0, 0), (0, 0), (0, 0), 1.0, 1.0),
                                          ((3, 1), (1, 2), (2, 0), (1, 3), -1.5, 0.5),
                                          ((4, 0), (2, 4), (0, 0), (4, 1), 1.0, 0.0)]:
        A = rand_batch(rng, nb, oa[0] + m + 1, oa[1] + k + 2)
        B = rand_batch(rng, nb, ob[0] + k + 2, ob[1] + n + 1)
        C = rand_batch(rng, nb, oc[0] + m, oc[1] + n)
        D = rand_batch(rng, nb, od[0] + m + 3, od[1] + n + 1)
        dA, dB, dC, dD = dev(A), dev(B), dev(C), dev(D)
        level3.gemm_nn(m, n, k, alpha, dA.ref(*oa), dB.ref(*ob), beta, dC.ref(*oc), dD.ref(*od))
        O.gemm_nn(m, n, k, alpha, A, *oa, B, *ob, beta, C, *oc, D, *od)
        compare_storage(host(dD), D.storage, window_mask(D, od, m, n), max(m, n, k), f"gemm_nn {mnk} {oa}{od}")


@pytest.mark.parametrize("mn", [(4, 4), (9, 6), (8, 8), (13, 7), (24, 24), (30, 20), (40, 40), (72, 48), (33, 70),
                                (128, 128), (64, 200), (300, 96)])
def test_trmm_rlnn_random_vs_oracle(mn):
    m, n = mn
    rng = np.random.default_rng(m * 131 + n)
    nb = 3 if max(m, n) >= 128 else 9
    for (oa, ob, od, alpha) in [((0, 0), (0, 0), (0, 0), 1.0), ((3, 2), (1, 1), (2, 3), -0.5),
                                ((4, 4), (4, 0), (0, 4), 2.0)]:
        T = rand_batch(rng, nb, oa[0] + n + 1, oa[1] + n + 2)
        for i in range(n):  # poison the strict upper triangle: must never be read
            for j in range(i + 1, n):
                T.storage[:, O.element_offset(oa[0] + i, oa[1] + j, T.cn)] = np.nan
        X = rand_batch(rng, nb, ob[0] + m + 2, ob[1] + n + 1)
        D = rand_batch(rng, nb, od[0] + m + 1, od[1] + n + 1)
        dT, dX, dD = dev(T), dev(X), dev(D)
        level3.trmm_rlnn(m, n, alpha, dT.ref(*oa), dX.ref(*ob), dD.ref(*od))
        O.trmm_rlnn(m, n, alpha, T, *oa, X, *ob, D, *od)
        compare_storage(host(dD), D.storage, window_mask(D, od, m, n), max(m, n), f"trmm {mn} {oa}{od}")


@pytest.mark.parametrize("mn", [(8, 8), (40, 40), (64, 100)])
def test_trmm_in_place_matches_out_of_place(mn):
    m, n = mn
    rng = np.random.default_rng(5)
    T = rand_batch(rng, 4, n, n)
    X = rand_batch(rng, 4, m, n)
    dT, dX, dY = dev(T), dev(X), dev(X)
    out = dev(O.HostBatch(4, m, n))
    level3.trmm_rlnn(m, n, 1.0, dT, dX, out)
    level3.trmm_rlnn(m, n, 1.0, dT, dY, dY)
    data = ((m + 3) // 4 * 4) * ((n + 3) // 4 * 4)  # data part; diag_inv is not written
    assert np.array_equal(host(out)[:, :data].view(np.uint64), host(dY)[:, :data].view(np.uint64))


@pytest.mark.parametrize("mkn", [(4, 3, None), (8, 8, None), (13, 5, None), (24, 16, None), (40, 33, None),
                                 (64, 64, None), (100, 40, None), (136, 16, None), (20, 7, 12), (70, 9, 33)])
def test_syrk_potrf_ln_random_vs_oracle(mkn):
    m, k, n = mkn
    n = m if n is None else n
    rng = np.random.default_rng(m * 17 + k)
    nb = 5
    for (oa, oc, od) in [((0, 0), (0, 0), (0, 0)), ((1, 2), (3, 1), (4, 0)), ((0, 0), (0, 0), (2, 2))]:
        A = rand_batch(rng, nb, oa[0] + m + 1, oa[1] + k + 1)
        C = rand_batch(rng, nb, oc[0] + m + 1, oc[1] + n + 1)
        for b in range(nb):
            g = rng.uniform(-1, 1, (n, n))
            spd = g @ g.T + n * np.eye(n)
            for i in range(n):
                for j in range(n):
                    C.storage[b, O.element_offset(oc[0] + i, oc[1] + j, C.cn)] = spd[i, j]
        D = rand_batch(rng, nb, od[0] + m + 2, od[1] + n + 1)
        dA, dC, dD = dev(A), dev(C), dev(D)
        info = level3.syrk_potrf_ln(m, k, dA.ref(*oa), dA.ref(*oa), dC.ref(*oc), dD.ref(*od), n=n)
        oinfo = O.syrk_potrf_ln(m, k, A, *oa, A, *oa, C, *oc, D, *od, n=n)
        assert np.array_equal(info.cpu().numpy(), oinfo)
        mask = window_mask(D, od, m, n, lower=True)
        mask[D.diag_off + od[1]: D.diag_off + od[1] + n] = True
        compare_storage(host(dD), D.storage, mask, max(m, k), f"syrk_potrf {mkn} {oa}{od}")
        assert (dD.diag_lo, dD.diag_hi) == (D.diag_lo, D.diag_hi)


def test_syrk_potrf_failure_and_k0_rules():
    rng = np.random.default_rng(3)
    m, k = 12, 4
    A = rand_batch(rng, 3, m, k)
    C = O.HostBatch(3, m, m)
    for b in range(3):
        g = rng.uniform(-1, 1, (m, m))
        C.set_window(0, 0, np.broadcast_to(g @ g.T + m * np.eye(m), (3, m, m)))
    C.storage[1, O.element_offset(7, 7, C.cn)] = -1e4  # item 1 fails at pivot 7
    D = rand_batch(rng, 3, m, m)
    dA, dC, dD = dev(A), dev(C), dev(D)
    with pytest.raises(pb.NotPositiveDefiniteError) as ei:
        level3.syrk_potrf_ln(m, k, dA, dA, dC, dD)
    assert ei.value.index == 7 and ei.value.batch_index == 1
    oinfo = O.syrk_potrf_ln(m, k, A, 0, 0, A, 0, 0, C, 0, 0, D, 0, 0)
    assert list(oinfo) == [-1, 7, -1]
    mask = window_mask(D, (0, 0), m, m, lower=True)
    mask[D.diag_off: D.diag_off + m] = True
    compare_storage(host(dD), D.storage, mask, m, "syrk_potrf failure partial writes")
    # k = 0 (and zero factors) reduce to plain potrf_l, bit-equal (test_level3.py:343-353, 632-641)
    d1, d2 = dev(O.HostBatch(3, m, m)), dev(O.HostBatch(3, m, m))
    C.storage[1, O.element_offset(7, 7, C.cn)] = C.storage[0, O.element_offset(7, 7, C.cn)]
    dC = dev(C)
    level3.syrk_potrf_ln(m, 0, dA, dA, dC, d1)
    level3.potrf_l(m, dC, d2)
    assert np.array_equal(host(d1).view(np.uint64), host(d2).view(np.uint64))
    for mm in (12, 24, 40):  # small-kernel and team-kernel regimes
        Cz = O.HostBatch(2, mm, mm)
        g = rng.uniform(-1, 1, (mm, mm))
        Cz.set_window(0, 0, np.broadcast_to(g @ g.T + mm * np.eye(mm), (2, mm, mm)))
        dZ, dCz = dev(O.HostBatch(2, mm, 3)), dev(Cz)
        e1, e2 = dev(O.HostBatch(2, mm, mm)), dev(O.HostBatch(2, mm, mm))
        level3.syrk_potrf_ln(mm, 3, dZ, dZ, dCz, e1)
        level3.potrf_l(mm, dCz, e2)
        assert np.array_equal(host(e1), host(e2)), mm  # == (a zero product may flip -0 to +0)


def _riccati_golden_inputs(z, r, batch):
    nx, nu, N = r["nx"], r["nu"], r["N"]
    ns = nx + nu
    rep = lambda a: torch.from_numpy(np.repeat(a[None, :], batch, axis=0)).cuda()  # noqa: E731
    bat = [pb.create_panel_batch(batch, ns, nx, rep(z[f"{r['key']}/bat{n}"])) for n in range(N)]
    rsq = [pb.create_panel_batch(batch, ns, ns, rep(z[f"{r['key']}/rsq{n}"])) for n in range(N)]
    P = pb.create_panel_batch(batch, nx, nx, rep(z[f"{r['key']}/P"]))
    return bat, rsq, P


@pytest.mark.parametrize("batch", [1, 6])
def test_riccati_factorize_golden(batch):
    """Batched composite.riccati_factorize against the reference's own
    apps.riccati_factorize outputs (tests/golden, apps.py:231-254)."""
    from paper_1704_02457_b200 import composite
    z, _ = load_golden()
    import json
    rics = json.loads(str(z["manifest"]))["riccati"]
    assert len(rics) >= 4
    for r in rics:
        nx, nu, N = r["nx"], r["nu"], r["N"]
        ns = nx + nu
        bat, rsq, P = _riccati_golden_inputs(z, r, batch)
        if r["status"] >= 0:
            with pytest.raises(pb.FactorizationError) as ei:
                composite.riccati_factorize(nx, nu, N, bat, rsq, P)
            assert str(ei.value).startswith(r["msg"].split(":")[0] + ":"), (str(ei.value), r["msg"])
            assert ei.value.index == r["status"]
            continue
        ws = composite.riccati_factorize(nx, nu, N, bat, rsq, P)
        torch.cuda.synchronize()
        for n in range(N):
            want = z[f"{r['key']}/F{n}"]
            got = host(ws.factors[n])[:, : want.size]
            h = O.HostBatch(1, ns, ns)
            mask = np.zeros(want.size, dtype=bool)
            for j in range(ns):
                for i in range(j, ns):
                    mask[O.element_offset(i, j, h.cn)] = True
            mask[h.diag_off: h.diag_off + ns] = True
            for b in range(batch):
                compare_storage(got[b], want, mask, ns, f"{r['name']} stage {n} item {b}")


def test_randomised_sweep_vs_oracle():
    """250 random potrf / getrf / gemm / syrk / trsm cases (sizes, window offsets,
    alpha/beta, failing pivots, batch sizes) against the oracle: FP within
    50*n*eps on the written window, every other byte and every integer output exact."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "pb_stress", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "stress.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.main(250, 7)


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
def test_potrf_host_pinned_descriptors(n):
    """The C ABI also takes pinned (UVA-mapped) HOST storage: the kernels read
    C and write D across PCIe.  Same bytes as the oracle (bit-exact for
    n <= 16, tolerance above), info identical, and every byte outside the
    reference's write set -- D's strict upper, padding -- unchanged in host
    memory (profiles/r01_pcie_zero_copy.txt)."""
    import ctypes
    from paper_1704_02457_b200 import _native
    rng = np.random.default_rng(300 + n)
    nb = 41
    a = spd_batch(rng, nb, n)
    a[5, n // 2, n // 2] = -1.0
    C = rand_batch(rng, nb, n, n)
    C.set_window(0, 0, a)
    D = rand_batch(rng, nb, n, n, fill=-3.25)
    hC = torch.from_numpy(C.storage.copy()).pin_memory()
    hD = torch.from_numpy(D.storage.copy()).pin_memory()
    pC, pD = pb.create_panel_batch(nb, n, n, hC), pb.create_panel_batch(nb, n, n, hD)
    dc, dd = pC.descriptor(), pD.descriptor()
    info = torch.empty(nb, dtype=torch.int32, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert _native.call("pb_dpotrf_l", n, n, ctypes.byref(dc), 0, 0, ctypes.byref(dd), 0, 0,
                        ctypes.c_void_p(info.data_ptr()), None, 0, st) == 0
    torch.cuda.synchronize()
    winfo = O.potrf_l(n, C, 0, 0, D, 0, 0)
    assert np.array_equal(info.cpu().numpy(), winfo)
    got = hD.numpy()
    if n <= 16:
        assert np.array_equal(got.view(np.uint64), D.storage.view(np.uint64))
    else:
        mask = np.zeros(D.storage.shape[1], dtype=bool)
        for i in range(n):
            for j in range(i + 1):
                mask[pb.element_offset(i, j, 4, pD.panel_length)] = True
        mask[pD._diag_off:pD._diag_off + n] = True
        compare_storage(got, D.storage, mask, n, f"host-pinned n={n}")


@pytest.mark.parametrize("op,m,n,k,nb", [("gemm", 64, 64, 100, 3000), ("gemm", 48, 48, 70, 2000),
                                         ("syrk", 96, 96, 40, 1500), ("syrk", 64, 64, 130, 1200)])
def test_tma_pipeline_many_units_per_cta_beta1(op, m, n, k, nb):
    """beta != 0 through the warp-specialised TMA pipeline with many units per
    CTA and several k-chunks per unit (the producer streams A/B chunks and the
    C tile of consecutive units through shared rings): every item of a large
    batch against a dense fp64 torch reference, written window only."""
    g = torch.Generator(device="cuda").manual_seed(7)
    A = alloc(nb, m, k)
    B = A if op == "syrk" else alloc(nb, n, k)
    C = alloc(nb, m, n)
    for x in {id(x): x for x in (A, B, C)}.values():
        x.storage.uniform_(-1, 1, generator=g)
    D = alloc(nb, m, n)
    D.storage.fill_(-7.5)
    if op == "gemm":
        level3.gemm_nt(m, n, k, -0.5, A, B, 1.0, C, D)
    else:
        level3.syrk_ln(m, k, -0.5, A, A, 1.0, C, D)
    a, b, c = pack.unpack_window(A, m, k), pack.unpack_window(B, n, k), pack.unpack_window(C, m, n)
    want = -0.5 * torch.bmm(a, b.transpose(1, 2)) + c
    got = pack.unpack_window(D, m, n)
    if op == "syrk":
        low = torch.tril(torch.ones(m, n, dtype=torch.bool, device="cuda"))
        assert bool((got[:, ~low] == -7.5).all())  # strict upper untouched
        got, want = got[:, low], want[:, low]
    err = (torch.linalg.vector_norm(got - want) / torch.linalg.vector_norm(want)).item()
    assert err <= 50 * max(m, n, k) * EPS, err


@pytest.mark.gpu
@pytest.mark.parametrize("m", [260, 300])
def test_syrk_potrf_large_failure_partial_writes(m):
    """syrk_potrf_ln beyond one team (workspace + blocked potrf driver): items
    failing in the first panel and in the trailing block get the reference's
    row-panel partial writes (ccore.pyx:877-941); healthy items match."""
    rng = np.random.default_rng(m)
    k, nb = 16, 4
    A = rand_batch(rng, nb, m, k)
    C = O.HostBatch(nb, m, m)
    g = rng.uniform(-1, 1, (m, m))
    C.set_window(0, 0, np.broadcast_to(g @ g.T + m * np.eye(m), (nb, m, m)))
    C.storage[1, O.element_offset(50, 50, C.cn)] = -1e6   # fails inside the first panel
    C.storage[2, O.element_offset(m - 10, m - 10, C.cn)] = -1e6  # fails in the trailing block
    D = rand_batch(rng, nb, m, m, fill=2.5)
    dA, dC, dD = dev(A), dev(C), dev(D)
    with pytest.raises(pb.NotPositiveDefiniteError) as ei:
        level3.syrk_potrf_ln(m, k, dA, dA, dC, dD)
    assert ei.value.index == 50 and ei.value.batch_index == 1
    oinfo = O.syrk_potrf_ln(m, k, A, 0, 0, A, 0, 0, C, 0, 0, D, 0, 0)
    assert list(oinfo) == [-1, 50, m - 10, -1]
    mask = window_mask(D, (0, 0), m, m, lower=True)
    mask[D.diag_off: D.diag_off + m] = True
    compare_storage(host(dD), D.storage, mask, m, f"syrk_potrf {m} failure partial writes")


# ---------------------------------------------------------------------------
# guard bands (compute-sanitizer is closed on this GPU pool: own bounds checks)


def _guarded(nb, m, n, fill=0.0, guard=1 << 17):
    """A batch in the current layout carved from the middle of a larger
    buffer whose guard regions (before and after every plane) hold a NaN
    sentinel; returns (batch, check) where check() asserts the guards are
    bit-for-bit untouched."""
    sentinel = float.fromhex("-0x1.dead00beefp+1000")
    planes = []
    if LAYOUT == "interleaved":
        per = pb.memsize_panel_matrix(m, n) // 8
        buf = torch.full((2 * guard + nb * per,), sentinel, dtype=torch.float64, device="cuda")
        core = buf[guard: guard + nb * per]
        core.fill_(fill)
        p = pb.create_panel_batch(nb, m, n, core)
        planes.append((buf, guard, nb * per))
    else:
        de, dn = pb.panel_data_elems(m, n), min(m, n)
        bd = torch.full((2 * guard + nb * de,), sentinel, dtype=torch.float64, device="cuda")
        bg = torch.full((2 * guard + max(nb * dn, 1),), sentinel, dtype=torch.float64, device="cuda")
        cd, cg = bd[guard: guard + nb * de], bg[guard: guard + nb * dn]
        cd.fill_(fill)
        cg.fill_(fill)
        p = pb.create_panel_batch(nb, m, n, cd, cg)
        planes += [(bd, guard, nb * de), (bg, guard, nb * dn)]

    def check(what):
        torch.cuda.synchronize()
        for buf, g0, cnt in planes:
            s = torch.tensor([sentinel], dtype=torch.float64, device="cuda").view(torch.int64)
            head, tail = buf[:g0].view(torch.int64), buf[g0 + cnt:].view(torch.int64)
            assert bool((head == s).all()) and bool((tail == s).all()), f"guard band written: {what}"
    return p, check


@pytest.mark.parametrize("n", [4, 8, 16, 40, 64, 100, 128, 256, 300])
def test_guard_bands_potrf_and_trsm(n):
    """Every potrf regime (and the trsm that follows) writes nothing outside
    its operands' storage, including the blocked driver's workspace path."""
    rng = np.random.default_rng(n)
    nb = 3 if n >= 128 else 17
    C, cchk = _guarded(nb, n, n)
    pack.pack_array_into(torch.from_numpy(spd_batch(rng, nb, n)).cuda(), C)
    D, dchk = _guarded(nb, n, n, fill=2.0)
    level3.potrf_l(n, C, D, check=False)
    level3.potrf_l(n, C, C, check=False)
    X, xchk = _guarded(nb, 24, n)
    level3.trsm_rltn(24, n, 1.0, D, X, X, check=False)
    Y, ychk = _guarded(nb, 70, n)  # 70 rows: the register-strip trsm kernel for 64 <= n <= 128 (ragged last strip)
    level3.trsm_rltn(70, n, 1.0, D, Y, Y, check=False)
    for ck, w in ((cchk, "C"), (dchk, "D"), (xchk, "X"), (ychk, "Y")):
        ck(f"potrf/trsm n={n} {w}")


@pytest.mark.parametrize("mnk", [(4, 4, 4), (20, 24, 9), (64, 64, 64), (100, 72, 40), (300, 264, 40)])
def test_guard_bands_gemm_syrk_pack(mnk):
    m, n, k = mnk
    nb = max(2, 4000 // (m * n))
    A, achk = _guarded(nb, m + 3, k)
    B, bchk = _guarded(nb, n, k)
    Cm, cchk = _guarded(nb, m, max(m, n))
    D, dchk = _guarded(nb, m, max(m, n))
    for x in (A, B, Cm):
        x.storage.uniform_(-1, 1)
    level3.gemm_nt(m, n, k, 1.0, A.ref(3, 0), B, 1.0, Cm, D)
    level3.syrk_ln(m, k, -1.0, A, A, 1.0, Cm, D)
    arr = torch.rand((nb, m, n), dtype=torch.float64, device="cuda")
    pack.pack_array_into(arr, D)
    pack.unpack_window(D, m, n)
    pack.gecp(m, n, D, Cm)
    for ck, w in ((achk, "A"), (bchk, "B"), (cchk, "C"), (dchk, "D")):
        ck(f"gemm/syrk/pack {mnk} {w}")
