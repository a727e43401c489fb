"""Generate tests/golden/golden_v1.npz from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    make -C oracle ref                 # cythonize + compile the reference's own ccore
    python tests/golden/make_golden.py            # golden_v1.npz
    python tests/golden/make_golden.py --getrf    # golden_getrf_v1.npz (§8f getrf)

It imports the reference package ``panelblas`` read-only from
/root/reference/pkg/src with its compiled core from oracle/_ref (or, if
that is missing, the reference's own bit-identical pure-Python twin
pycore, _backend/__init__.py:17-26) and records, for every case, the
inputs and the outputs of the reference's public level3/pack calls as
full item storage (the create_panel_matrix byte layout: data, then
diag_inv), plus the raised pivot index.  Cases follow the reference's
own tests: the hand examples (tests/test_level3.py:31-36, 212-216,
288-293), the special cases (alpha=0 with NaN operands :39-46, k=0,
upper untouched :152-159), failure indices (:262-268, :296-305),
unaligned windows (:527-585), diag_inv reuse (:592-606), aliasing and
tall stacks.  Nothing from the reference's sources is copied; only
generated numbers are stored.
"""
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def import_reference():
    import importlib.util
    sys.path.insert(0, REF_SRC)
    refdir = os.path.join(REPO, "oracle", "_ref")
    so = [f for f in os.listdir(refdir) if f.startswith("ccore")] if os.path.isdir(refdir) else []
    so = [f for f in so if f.endswith(".so")]
    if so:
        spec = importlib.util.spec_from_file_location("panelblas._backend.ccore", os.path.join(refdir, so[0]))
        mod = importlib.util.module_from_spec(spec)
        sys.modules["panelblas._backend.ccore"] = mod
        spec.loader.exec_module(mod)
    else:
        os.environ["PANELBLAS_BACKEND"] = "py"
    import panelblas
    return panelblas


pb = import_reference()
from panelblas import level3, pack  # noqa: E402
from panelblas.errors import FactorizationError  # noqa: E402
from panelblas.matstore import allocate_panel_matrix  # noqa: E402

CASES = []
ARRAYS = {}


def zmat(m, n, fill=0.0):
    p = allocate_panel_matrix(m, n)
    raw = np.frombuffer(p._base, dtype=np.float64)
    raw[:] = 0.0
    p.data[:] = fill
    return p


def put(mat, ai, aj, arr):
    arr = np.asarray(arr, dtype=np.float64)
    for i in range(arr.shape[0]):
        for j in range(arr.shape[1]):
            mat.set(ai + i, aj + j, float(arr[i, j]))


def raw(mat):
    return np.frombuffer(mat._base, dtype=np.float64).copy()


def record(name, op, params, mats, fn):
    """mats: dict label -> (PanelMatrix); identical objects mean aliasing."""
    key = f"c{len(CASES):03d}"
    ids = {}
    alias = {}
    for lab, mat in mats.items():
        if id(mat) in ids:
            alias[lab] = ids[id(mat)]
        else:
            ids[id(mat)] = lab
            ARRAYS[f"{key}/in/{lab}"] = raw(mat)
    valid = {lab: [mat.diag_lo, mat.diag_hi] for lab, mat in mats.items()}
    status = -1
    try:
        fn()
    except FactorizationError as e:
        status = int(e.index)
    for lab, mat in mats.items():
        if lab not in alias:
            ARRAYS[f"{key}/out/{lab}"] = raw(mat)
    dims = {lab: [mat.rows, mat.cols] for lab, mat in mats.items()}
    CASES.append({"key": key, "name": name, "op": op, "params": params, "dims": dims, "alias": alias,
                  "status": status, "valid_in": valid,
                  "valid_out": {lab: [mat.diag_lo, mat.diag_hi] for lab, mat in mats.items()}})


def spd(rng, n, shift=None):
    g = rng.uniform(-1, 1, (n, n))
    return g @ g.T + (shift if shift is not None else n) * np.eye(n)


def gemm_case(name, rng, m, n, k, alpha, beta, oa=(0, 0), ob=(0, 0), oc=(0, 0), od=(0, 0),
              a=None, b=None, c=None, alias_dc=False, dfill=0.0):
    a = rng.uniform(-1, 1, (m, k)) if a is None else a
    b = rng.uniform(-1, 1, (n, k)) if b is None else b
    c = rng.uniform(-1, 1, (m, n)) if c is None else c
    A = zmat(oa[0] + m + 3, oa[1] + k + 2)
    B = zmat(ob[0] + n + 1, ob[1] + k + 3)
    C = zmat(oc[0] + m + 2, oc[1] + n + 1)
    put(A, *oa, a)
    put(B, *ob, b)
    put(C, *oc, c)
    if alias_dc:
        D, od = C, oc
    else:
        D = zmat(od[0] + m + 1, od[1] + n + 2, fill=dfill)
    p = dict(m=m, n=n, k=k, alpha=alpha, beta=beta, ai=oa[0], aj=oa[1], bi=ob[0], bj=ob[1], ci=oc[0], cj=oc[1],
             di=od[0], dj=od[1])
    record(name, "gemm_nt", p, {"A": A, "B": B, "C": C, "D": D},
           lambda: level3.gemm_nt(m, n, k, alpha, A.ref(*oa), B.ref(*ob), beta, C.ref(*oc), D.ref(*od)))


def syrk_case(name, rng, m, k, alpha, beta, oa=(0, 0), ob=(0, 0), oc=(0, 0), od=(0, 0), same_ab=False,
              alias_dc=False, dfill=0.0, a=None, b=None):
    a = rng.uniform(-1, 1, (m, k)) if a is None else a
    b = rng.uniform(-1, 1, (m, k)) if b is None else b
    c = rng.uniform(-1, 1, (m, m))
    A = zmat(oa[0] + m + 2, oa[1] + k + 1)
    put(A, *oa, a)
    if same_ab:
        B, ob = A, oa
    else:
        B = zmat(ob[0] + m + 1, ob[1] + k + 2)
        put(B, *ob, b)
    C = zmat(oc[0] + m + 1, oc[1] + m + 1)
    put(C, *oc, c)
    D = C if alias_dc else zmat(od[0] + m + 2, od[1] + m + 1, fill=dfill)
    if alias_dc:
        od = oc
    p = dict(m=m, k=k, alpha=alpha, beta=beta, ai=oa[0], aj=oa[1], bi=ob[0], bj=ob[1], ci=oc[0], cj=oc[1],
             di=od[0], dj=od[1])
    record(name, "syrk_ln", p, {"A": A, "B": B, "C": C, "D": D},
           lambda: level3.syrk_ln(m, k, alpha, A.ref(*oa), B.ref(*ob), beta, C.ref(*oc), D.ref(*od)))


def trsm_case(name, rng, m, n, alpha, oa=(0, 0), ob=(0, 0), od=(0, 0), lw=None, b=None, in_place=False,
              from_potrf=False):
    if lw is None:
        lw = np.linalg.cholesky(spd(rng, n))
    b = rng.uniform(-1, 1, (m, n)) if b is None else b
    A = zmat(oa[0] + n + 1, oa[1] + n + 2)
    if from_potrf:
        S = zmat(oa[0] + n + 1, oa[1] + n + 2)
        put(S, *oa, spd(rng, n))
        level3.potrf_l(n, S.ref(*oa), A.ref(*oa))  # A.diag_inv valid on its diagonal
    else:
        put(A, *oa, lw)
    B = zmat(ob[0] + m + 2, ob[1] + n + 1)
    put(B, *ob, b)
    if in_place:
        D, od = B, ob
    else:
        D = zmat(od[0] + m + 1, od[1] + n + 1)
    p = dict(m=m, n=n, alpha=alpha, ai=oa[0], aj=oa[1], bi=ob[0], bj=ob[1], di=od[0], dj=od[1])
    record(name, "trsm_rltn", p, {"A": A, "B": B, "D": D},
           lambda: level3.trsm_rltn(m, n, alpha, A.ref(*oa), B.ref(*ob), D.ref(*od)))


def potrf_case(name, rng, m, c, n=None, oc=(0, 0), od=(0, 0), in_place=False, dfill=0.0):
    n = m if n is None else n
    C = zmat(oc[0] + m + 2, oc[1] + n + 1)
    put(C, *oc, c)
    if in_place:
        D, od = C, oc
    else:
        D = zmat(od[0] + m + 1, od[1] + n + 3, fill=dfill)
    p = dict(m=m, n=n, ci=oc[0], cj=oc[1], di=od[0], dj=od[1])
    record(name, "potrf_l", p, {"C": C, "D": D}, lambda: level3.potrf_l(m, C.ref(*oc), D.ref(*od), n=n))


def gemm_nn_case(name, rng, m, n, k, alpha, beta, oa=(0, 0), ob=(0, 0), oc=(0, 0), od=(0, 0),
                 a=None, b=None, c=None, alias_dc=False, dfill=0.0):
    a = rng.uniform(-1, 1, (m, k)) if a is None else a
    b = rng.uniform(-1, 1, (k, n)) if b is None else b
    c = rng.uniform(-1, 1, (m, n)) if c is None else c
    A = zmat(oa[0] + m + 3, oa[1] + k + 2)
    B = zmat(ob[0] + k + 1, ob[1] + n + 3)
    C = zmat(oc[0] + m + 2, oc[1] + n + 1)
    put(A, *oa, a)
    put(B, *ob, b)
    put(C, *oc, c)
    if alias_dc:
        D, od = C, oc
    else:
        D = zmat(od[0] + m + 1, od[1] + n + 2, fill=dfill)
    p = dict(m=m, n=n, k=k, alpha=alpha, beta=beta, ai=oa[0], aj=oa[1], bi=ob[0], bj=ob[1], ci=oc[0], cj=oc[1],
             di=od[0], dj=od[1])
    record(name, "gemm_nn", p, {"A": A, "B": B, "C": C, "D": D},
           lambda: level3.gemm_nn(m, n, k, alpha, A.ref(*oa), B.ref(*ob), beta, C.ref(*oc), D.ref(*od)))


def trmm_case(name, rng, m, n, alpha, oa=(0, 0), ob=(0, 0), od=(0, 0), t=None, b=None, in_place=False,
              poison=True, dfill=0.0):
    t = np.tril(rng.uniform(-1, 1, (n, n))) if t is None else t
    if poison:
        t = t + np.triu(np.full((n, n), np.nan), 1)
    b = rng.uniform(-1, 1, (m, n)) if b is None else b
    A = zmat(oa[0] + n + 1, oa[1] + n + 2)
    put(A, *oa, t)
    B = zmat(ob[0] + m + 2, ob[1] + n + 1)
    put(B, *ob, b)
    if in_place:
        D, od = B, ob
    else:
        D = zmat(od[0] + m + 1, od[1] + n + 1, fill=dfill)
    p = dict(m=m, n=n, alpha=alpha, ai=oa[0], aj=oa[1], bi=ob[0], bj=ob[1], di=od[0], dj=od[1])
    record(name, "trmm_rlnn", p, {"A": A, "B": B, "D": D},
           lambda: level3.trmm_rlnn(m, n, alpha, A.ref(*oa), B.ref(*ob), D.ref(*od)))


def syrk_potrf_case(name, rng, m, k, n=None, oa=(0, 0), ob=(0, 0), oc=(0, 0), od=(0, 0), a=None, b=None, c=None,
                    same_ab=True, dfill=0.0):
    n = m if n is None else n
    a = rng.uniform(-1, 1, (m, k)) if a is None else a
    if c is None:
        c = rng.uniform(-1, 1, (m, n))
        c[:n, :n] = spd(rng, n)
    A = zmat(oa[0] + m + 2, oa[1] + k + 1)
    put(A, *oa, a)
    if same_ab:
        B, ob = A, oa
    else:
        b = rng.uniform(-1, 1, (n, k)) if b is None else b
        B = zmat(ob[0] + n + 1, ob[1] + k + 2)
        put(B, *ob, b)
    C = zmat(oc[0] + m + 1, oc[1] + n + 1)
    put(C, *oc, c)
    D = zmat(od[0] + m + 2, od[1] + n + 1, fill=dfill)
    p = dict(m=m, n=n, k=k, ai=oa[0], aj=oa[1], bi=ob[0], bj=ob[1], ci=oc[0], cj=oc[1], di=od[0], dj=od[1])
    record(name, "syrk_potrf_ln", p, {"A": A, "B": B, "C": C, "D": D},
           lambda: level3.syrk_potrf_ln(m, k, A.ref(*oa), B.ref(*ob), C.ref(*oc), D.ref(*od), n=n))


RICCATI = []


def riccati_case(name, rng, nx, nu, N, fail_stage=None):
    """apps.riccati_factorize on random stable data; records the packed
    stage inputs and every stage factor (apps.py:231-254)."""
    from panelblas import apps
    A = rng.uniform(-0.5, 0.5, (N, nx, nx)) + 0.8 * np.eye(nx)
    B = rng.uniform(-1, 1, (N, nx, nu))
    Q = np.stack([spd(rng, nx) for _ in range(N)])
    R = np.stack([spd(rng, nu) if nu else np.zeros((0, 0)) for _ in range(N)])
    S = rng.uniform(-0.1, 0.1, (N, nu, nx))
    P = spd(rng, nx)
    if fail_stage is not None:
        R[fail_stage][0, 0] = -1e6
    dims = apps.OcpDims(nx, nu, N)
    data = apps.OcpData.from_arrays(dims, A, B, Q, R, S, P)
    key = f"r{len(RICCATI):02d}"
    for n_, st in enumerate(data.stages):
        ARRAYS[f"{key}/bat{n_}"] = raw(st.bat)
        ARRAYS[f"{key}/rsq{n_}"] = raw(st.rsq)
    ARRAYS[f"{key}/P"] = raw(data.p_panel)
    status, msg = -1, ""
    ws = apps.RiccatiWorkspace(dims)  # zero the workspace: allocate_panel_matrix does not
    for mat in [ws.cbuf, ws.terminal] + ws.factors:
        np.frombuffer(mat._base, dtype=np.float64)[:] = 0.0
    try:
        fac = apps.riccati_factorize(data, ws)
        for n_, f in enumerate(fac):
            ARRAYS[f"{key}/F{n_}"] = raw(f.full)
            ARRAYS[f"{key}/P{n_}"] = f.cost_to_go()
    except FactorizationError as e:
        status, msg = int(e.index), str(e)
    RICCATI.append({"key": key, "name": name, "nx": nx, "nu": nu, "N": N, "status": status, "msg": msg})


def pack_case(name, rng, m, n, od):
    arr = rng.uniform(-1, 1, (m, n))
    from panelblas.matstore import ColMatrix
    D = zmat(od[0] + m + 3, od[1] + n + 3)
    ARRAYS[f"c{len(CASES):03d}/src"] = arr
    record(name, "pack", dict(m=m, n=n, di=od[0], dj=od[1]), {"D": D},
           lambda: pack.pack_matrix(ColMatrix.from_array(arr), m, n, D.ref(*od)) if m * n else None)


def getrf_case(name, rng, m, n, pivot, oc=(0, 0), od=(0, 0), c=None, in_place=False, dfill=0.0):
    """level3.getrf_pivot / getrf_nopivot (level3.py:405-498); ipiv recorded too."""
    c = rng.uniform(-1, 1, (m, n)) if c is None else np.asarray(c, dtype=np.float64)
    C = zmat(oc[0] + m + 1, oc[1] + n + 2)
    put(C, *oc, c)
    if in_place:
        D, od = C, oc
    else:
        D = zmat(od[0] + m + 2, od[1] + n + 1, fill=dfill)
    mn = min(m, n)
    ipiv = np.full(max(mn, 1), -7, dtype=np.int64)
    p = dict(m=m, n=n, pivot=int(pivot), ci=oc[0], cj=oc[1], di=od[0], dj=od[1])
    key = f"c{len(CASES):03d}"
    if pivot:
        fn = lambda: level3.getrf_pivot(m, n, C.ref(*oc), D.ref(*od), ipiv=ipiv[:mn] if mn else ipiv)  # noqa: E731
    else:
        fn = lambda: level3.getrf_nopivot(m, n, C.ref(*oc), D.ref(*od))  # noqa: E731
    record(name, "getrf", p, {"C": C, "D": D}, fn)
    ARRAYS[f"{key}/ipiv"] = ipiv.copy()


def main():
    rng = np.random.default_rng(20261020)
    # ---- gemm_nt
    gemm_case("gemm_kat_2x2", rng, 2, 2, 2, 1.0, 0.0, a=np.array([[1.0, 2], [3, 4]]),
              b=np.array([[5.0, 6], [7, 8]]))
    for m, n, k in [(5, 3, 7), (1, 1, 1), (16, 16, 16), (13, 9, 11), (4, 20, 2), (33, 7, 5), (8, 8, 8),
                    (24, 24, 24), (40, 36, 33), (64, 64, 64), (17, 70, 9)]:
        gemm_case(f"gemm_{m}x{n}x{k}", rng, m, n, k, 1.5, -0.5)
    gemm_case("gemm_beta0", rng, 9, 6, 5, 1.0, 0.0, c=np.full((9, 6), np.nan))
    gemm_case("gemm_alpha0_nan", rng, 8, 2, 7, 0.0, 1.0, a=np.full((8, 7), np.nan), b=np.full((2, 7), np.nan))
    gemm_case("gemm_alpha0_beta0", rng, 5, 5, 3, 0.0, 0.0, c=np.full((5, 5), np.nan))
    gemm_case("gemm_k0", rng, 5, 3, 0, 1.0, -2.0)
    gemm_case("gemm_unaligned", rng, 10, 10, 6, 1.0, 1.0, oa=(3, 2), ob=(1, 3), oc=(2, 2), od=(1, 1))
    gemm_case("gemm_unaligned_big", rng, 37, 45, 29, -1.0, 0.5, oa=(5, 1), ob=(2, 3), oc=(7, 2), od=(3, 1),
              dfill=3.5)
    gemm_case("gemm_alias_dc", rng, 9, 6, 5, 1.0, 0.5, alias_dc=True)
    gemm_case("gemm_surround", rng, 6, 5, 4, 1.0, 0.0, od=(2, 1), dfill=3.5)
    gemm_case("gemm_m0", rng, 0, 4, 4, 1.0, 0.0, dfill=1.0)
    # ---- syrk_ln
    syrk_case("syrk_identity", rng, 4, 4, 1.0, 0.0, a=np.eye(4), b=np.eye(4))
    syrk_case("syrk_k0", rng, 5, 0, 1.0, 2.0)
    syrk_case("syrk_7x4", rng, 7, 4, 1.0, 0.0)
    syrk_case("syrk_upper_untouched", rng, 6, 3, 1.0, 0.0, dfill=9.0)
    syrk_case("syrk_c4_like", rng, 24, 10, -1.0, 1.0, oa=(3, 1), same_ab=True)
    syrk_case("syrk_c4_shape", rng, 96, 40, -1.0, 1.0, oa=(3, 1), same_ab=True)
    syrk_case("syrk_unaligned_d", rng, 10, 4, 1.0, 0.0, oa=(3, 1), same_ab=True, od=(1, 1))
    syrk_case("syrk_alias_dc", rng, 9, 4, 1.0, 0.5, same_ab=True, alias_dc=True)
    syrk_case("syrk_33", rng, 33, 17, 1.5, -0.5, oa=(1, 2), ob=(2, 0), oc=(1, 1), od=(2, 3))
    syrk_case("syrk_alpha0", rng, 6, 5, 0.0, 1.0, a=np.full((6, 5), np.nan), b=np.full((6, 5), np.nan))
    # ---- trsm_rltn
    trsm_case("trsm_kat", rng, 2, 2, 1.0, lw=np.array([[2.0, 0.0], [1.0, 1.0]]), b=np.eye(2))
    for m, n in [(5, 3), (8, 8), (3, 9), (13, 6), (1, 1), (12, 12), (72, 48), (17, 33)]:
        trsm_case(f"trsm_{m}x{n}", rng, m, n, 1.5)
    trsm_case("trsm_in_place", rng, 6, 6, 1.0, in_place=True)
    trsm_case("trsm_reuse_dinv", rng, 5, 8, 1.0, from_potrf=True)
    trsm_case("trsm_reuse_dinv_72x48", rng, 72, 48, -1.0, from_potrf=True)
    trsm_case("trsm_unaligned", rng, 7, 10, 1.0, oa=(3, 3), ob=(1, 1), od=(1, 2))
    za = np.tril(rng.uniform(1, 2, (4, 4)))
    za[2, 2] = 0.0
    trsm_case("trsm_zero_diag", rng, 3, 4, 1.0, lw=za, b=np.ones((3, 4)))
    # ---- potrf_l
    potrf_case("potrf_identity", rng, 5, np.eye(5))
    potrf_case("potrf_kat", rng, 2, np.array([[4.0, 2.0], [2.0, 3.0]]))
    potrf_case("potrf_fail0", rng, 3, np.zeros((3, 3)))
    c6 = np.eye(6)
    c6[4, 4] = -1.0
    potrf_case("potrf_fail4", rng, 6, c6)
    for m in [1, 2, 3, 4, 5, 8, 11, 16, 21, 33, 48, 64]:
        potrf_case(f"potrf_{m}", rng, m, spd(rng, m))
    potrf_case("potrf_in_place", rng, 9, spd(rng, 9), in_place=True)
    h = spd(rng, 6)
    potrf_case("potrf_tall", rng, 11, np.vstack([h, rng.uniform(-1, 1, (5, 6))]), n=6)
    h = spd(rng, 20)
    potrf_case("potrf_tall_20x13", rng, 29, np.vstack([h, rng.uniform(-1, 1, (9, 20))])[:, :13], n=13)
    potrf_case("potrf_unaligned", rng, 10, spd(rng, 10), oc=(3, 3), od=(1, 1))
    potrf_case("potrf_upper_garbage", rng, 7, np.tril(spd(rng, 7)) + np.triu(np.full((7, 7), np.nan), 1))
    for f, nn in [(9, 12), (13, 16), (2, 17), (22, 24)]:
        c = spd(rng, nn)
        c[f, f] = -5.0 * nn
        potrf_case(f"potrf_fail{f}_of{nn}", rng, nn, c, dfill=2.5)
    c = spd(rng, 10)
    c[5, 5] = -100.0
    potrf_case("potrf_fail_unaligned", rng, 10, c, od=(1, 1), dfill=2.5)
    # ---- pack
    for (m, n, od) in [(2, 2, (0, 0)), (1, 1, (6, 3)), (7, 5, (3, 1)), (13, 9, (2, 5)), (0, 4, (1, 1))]:
        pack_case(f"pack_{m}x{n}", rng, m, n, od)

    # ---- next tier: gemm_nn, trmm_rlnn, syrk_potrf_ln, riccati
    gemm_nn_case("gemm_nn_kat_2x2", rng, 2, 2, 2, 1.0, 0.0, a=np.array([[1.0, 2], [3, 4]]),
                 b=np.array([[5.0, 6], [7, 8]]))
    for m, n, k in [(5, 3, 7), (1, 1, 1), (16, 16, 16), (13, 9, 11), (4, 20, 2), (33, 7, 5), (40, 36, 33),
                    (64, 64, 64), (70, 17, 9), (24, 130, 40)]:
        gemm_nn_case(f"gemm_nn_{m}x{n}x{k}", rng, m, n, k, 1.5, -0.5)
    gemm_nn_case("gemm_nn_k0", rng, 5, 3, 0, 1.0, -2.0)
    gemm_nn_case("gemm_nn_beta0", rng, 9, 6, 5, 1.0, 0.0, c=np.full((9, 6), np.nan))
    gemm_nn_case("gemm_nn_alpha0_nan", rng, 8, 2, 7, 0.0, 1.0, a=np.full((8, 7), np.nan),
                 b=np.full((7, 2), np.nan))
    gemm_nn_case("gemm_nn_unaligned", rng, 10, 10, 6, 1.0, 1.0, oa=(3, 2), ob=(1, 3), oc=(2, 2), od=(1, 1))
    gemm_nn_case("gemm_nn_unaligned_big", rng, 37, 45, 29, -1.0, 0.5, oa=(5, 1), ob=(2, 3), oc=(7, 2), od=(3, 1),
                 dfill=3.5)
    gemm_nn_case("gemm_nn_alias_dc", rng, 9, 6, 5, 1.0, 0.5, alias_dc=True)
    trmm_case("trmm_identity", rng, 5, 4, 2.5, t=np.eye(4), poison=False)
    trmm_case("trmm_scalar", rng, 3, 1, 1.0, t=np.array([[2.0]]), b=np.array([[1.0], [2.0], [3.0]]))
    for m, n in [(9, 6), (4, 5), (1, 1), (8, 8), (13, 7), (24, 16), (40, 40), (72, 48), (33, 70)]:
        trmm_case(f"trmm_{m}x{n}", rng, m, n, 1.0)
    trmm_case("trmm_in_place", rng, 7, 6, 1.0, in_place=True)
    trmm_case("trmm_in_place_wide", rng, 20, 40, -1.0, in_place=True)
    trmm_case("trmm_unaligned", rng, 11, 9, 0.5, oa=(3, 2), ob=(1, 1), od=(2, 3), dfill=3.5)
    trmm_case("trmm_alpha0", rng, 6, 5, 0.0)
    syrk_potrf_case("syrk_potrf_k0", rng, 6, 0)
    for m, k in [(5, 3), (12, 8), (17, 4), (8, 8), (24, 16), (40, 33)]:
        syrk_potrf_case(f"syrk_potrf_{m}x{k}", rng, m, k)
    syrk_potrf_case("syrk_potrf_rect", rng, 11, 4, n=6, same_ab=False)
    syrk_potrf_case("syrk_potrf_unaligned", rng, 10, 5, oa=(1, 2), oc=(3, 1), od=(2, 2), dfill=2.5)
    cfail = spd(rng, 9)
    cfail[6, 6] = -1e3
    syrk_potrf_case("syrk_potrf_fail6", rng, 9, 3, c=cfail, dfill=2.5)
    riccati_case("riccati_2x1x3", rng, 2, 1, 3)
    riccati_case("riccati_8x8x5", rng, 8, 8, 5)
    riccati_case("riccati_6x3x4", rng, 6, 3, 4)
    riccati_case("riccati_16x8x3", rng, 16, 8, 3)
    riccati_case("riccati_fail", rng, 4, 2, 4, fail_stage=1)

    out = os.path.join(HERE, "golden_v1.npz")
    ARRAYS["manifest"] = np.array(json.dumps({"backend": pb.backend_name(), "cases": CASES,
                                              "riccati": RICCATI}))
    np.savez_compressed(out, **ARRAYS)
    print(f"wrote {len(CASES)} cases to {out} (reference backend {pb.backend_name()})")


def main_getrf():
    """tests/golden/golden_getrf_v1.npz: the §8f getrf cases (separate file, own seed)."""
    rng = np.random.default_rng(20261021)
    getrf_case("getrf_identity", rng, 5, 5, True, c=np.eye(5))
    getrf_case("getrf_forced_swap", rng, 2, 2, True, c=np.array([[0.0, 1.0], [2.0, 3.0]]))
    for m, n in [(4, 4), (7, 7), (9, 9), (12, 12), (16, 16), (5, 11), (13, 6), (24, 24), (33, 33), (40, 17)]:
        getrf_case(f"getrf_pivot_{m}x{n}", rng, m, n, True)
        getrf_case(f"getrf_nopivot_{m}x{n}", rng, m, n, False, c=rng.uniform(-1, 1, (m, n)) + 4.0 * np.eye(m, n))
    getrf_case("getrf_pivot_ties", rng, 8, 8, True, c=np.round(rng.uniform(-2, 2, (8, 8))))
    getrf_case("getrf_pivot_unaligned", rng, 10, 9, True, oc=(3, 2), od=(1, 3), dfill=2.5)
    getrf_case("getrf_pivot_aligned_off", rng, 9, 10, True, oc=(1, 1), od=(4, 2), dfill=2.5)
    getrf_case("getrf_in_place", rng, 11, 11, True, in_place=True)
    cz = rng.uniform(-1, 1, (6, 6))
    cz[:, 3] = 0.0
    getrf_case("getrf_pivot_zero_column", rng, 6, 6, True, c=cz, dfill=2.5)
    cn = rng.uniform(-1, 1, (5, 5)) + 3 * np.eye(5)
    cn[2, 2] = 0.0
    cn[2, :2] = 0.0
    cn[:2, 2] = 0.0
    getrf_case("getrf_nopivot_zero_pivot", rng, 5, 5, False, c=cn, dfill=2.5)
    getrf_case("getrf_pivot_zero_column_unaligned", rng, 6, 6, True, c=cz, od=(2, 1), dfill=2.5)

    out = os.path.join(HERE, "golden_getrf_v1.npz")
    ARRAYS["manifest"] = np.array(json.dumps({"backend": pb.backend_name(), "cases": CASES}))
    np.savez_compressed(out, **ARRAYS)
    print(f"wrote {len(CASES)} cases to {out} (reference backend {pb.backend_name()})")


if __name__ == "__main__":
    if "--getrf" in sys.argv:
        main_getrf()
    else:
        main()
