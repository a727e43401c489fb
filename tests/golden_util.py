"""Golden-fixture plumbing shared by the CPU oracle tests and the GPU parity tests."""
import numpy as np

from oracle import oracle as O


def host_inputs(z, case, batch=1):
    """label -> HostBatch built from the recorded inputs (aliases share objects)."""
    mats = {}
    for lab, (m, n) in case["dims"].items():
        if lab in case["alias"]:
            continue
        arr = z[f"{case['key']}/in/{lab}"]
        st = np.repeat(arr[None, :], batch, axis=0)
        h = O.HostBatch(batch, m, n, st)
        h.diag_lo, h.diag_hi = case["valid_in"][lab]
        mats[lab] = h
    for lab, tgt in case["alias"].items():
        mats[lab] = mats[tgt]
    return mats


def run_oracle(case, mats, z=None):
    """Apply the case's op with the oracle; returns the status (first item)."""
    p = case["params"]
    op = case["op"]
    if op == "gemm_nt":
        O.gemm_nt(p["m"], p["n"], p["k"], p["alpha"], mats["A"], p["ai"], p["aj"], mats["B"], p["bi"], p["bj"],
                  p["beta"], mats["C"], p["ci"], p["cj"], mats["D"], p["di"], p["dj"])
        return -1
    if op == "syrk_ln":
        O.syrk_ln(p["m"], p["k"], p["alpha"], mats["A"], p["ai"], p["aj"], mats["B"], p["bi"], p["bj"],
                  p["beta"], mats["C"], p["ci"], p["cj"], mats["D"], p["di"], p["dj"])
        return -1
    if op == "trsm_rltn":
        info = O.trsm_rltn(p["m"], p["n"], p["alpha"], mats["A"], p["ai"], p["aj"], mats["B"], p["bi"], p["bj"],
                           mats["D"], p["di"], p["dj"])
        return int(info[0])
    if op == "potrf_l":
        info = O.potrf_l(p["m"], mats["C"], p["ci"], p["cj"], mats["D"], p["di"], p["dj"], n=p["n"])
        return int(info[0])
    if op == "gemm_nn":
        O.gemm_nn(p["m"], p["n"], p["k"], p["alpha"], mats["A"], p["ai"], p["aj"], mats["B"], p["bi"], p["bj"],
                  p["beta"], mats["C"], p["ci"], p["cj"], mats["D"], p["di"], p["dj"])
        return -1
    if op == "trmm_rlnn":
        O.trmm_rlnn(p["m"], p["n"], p["alpha"], mats["A"], p["ai"], p["aj"], mats["B"], p["bi"], p["bj"],
                    mats["D"], p["di"], p["dj"])
        return -1
    if op == "syrk_potrf_ln":
        info = O.syrk_potrf_ln(p["m"], p["k"], mats["A"], p["ai"], p["aj"], mats["B"], p["bi"], p["bj"],
                               mats["C"], p["ci"], p["cj"], mats["D"], p["di"], p["dj"], n=p["n"])
        return int(info[0])
    if op == "getrf":
        ipiv = np.full((mats["D"].batch, max(min(p["m"], p["n"]), 1)), -7, dtype=np.int64)
        info, ipiv = O.getrf(p["m"], p["n"], mats["C"], p["ci"], p["cj"], mats["D"], p["di"], p["dj"], p["pivot"],
                             ipiv=ipiv)
        mats["_ipiv"] = ipiv
        return int(info[0])
    if op == "pack":
        m, n = p["m"], p["n"]
        if m * n:
            src = np.asfortranarray(z[f"{case['key']}/src"]).reshape(-1, order="F").copy()
            O.pack_cm(m, n, src, max(m, 1), 0, mats["D"], p["di"], p["dj"])
        return -1
    raise ValueError(op)


def out_labels(case):
    return [lab for lab in case["dims"] if lab not in case["alias"]]


def written_mask(case, lab, per, cn, status):
    """Boolean mask over an item's storage: True where the op may write FP results."""
    p = case["params"]
    op = case["op"]
    mask = np.zeros(per, dtype=bool)
    if lab != case["alias"].get("D", "D"):
        return mask

    def eo(i, j):
        return (i - (i & 3)) * cn + 4 * j + (i & 3)

    if op in ("gemm_nt", "gemm_nn", "trmm_rlnn", "trsm_rltn", "pack"):
        m, n = p["m"], p["n"]
        for i in range(m):
            for j in range(n):
                mask[eo(p["di"] + i, p["dj"] + j)] = True
    elif op == "syrk_ln":
        m = p["m"]
        for j in range(m):
            for i in range(j, m):
                mask[eo(p["di"] + i, p["dj"] + j)] = True
    elif op in ("potrf_l", "syrk_potrf_ln"):
        m, n = p["m"], p["n"]
        for j in range(n):
            for i in range(j, m):
                mask[eo(p["di"] + i, p["dj"] + j)] = True
    return mask
