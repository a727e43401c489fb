"""Generate tests/golden/golden_large_v1.json from the REFERENCE itself.

Run in the build container (where /root/reference exists), after
``make -C oracle ref``:

    python tests/golden/make_golden_large.py

Pins the oracle at the BASELINE sizes the small golden file does not reach
(C2's potrf n = 128 / 256, C3's gemm n = 128 / 300, trsm 128 x 128): each
case's inputs come from a seeded numpy generator (reproducible), the
reference's public level3 call (panelblas imported read-only from
/root/reference/pkg/src with its compiled core from oracle/_ref, as in
make_golden.py) produces the output, and only a SHA-256 of the output item
storage (create_panel_matrix byte layout, data then diag_inv) plus a few
sampled values are stored -- a 1-MB item needs no fixture to be pinned.
tests/test_oracle.py::test_oracle_pinned_to_reference_at_large_sizes replays
the inputs through the oracle and compares digests.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402  (imports the reference read-only)

pbr = import_reference()
from panelblas import level3  # noqa: E402
from panelblas.matstore import allocate_panel_matrix, element_offset  # noqa: E402


def inputs(case):
    """Seeded inputs of a case as dense arrays (shared with the test)."""
    rng = np.random.default_rng(case["seed"])
    op, n = case["op"], case["n"]
    if op == "potrf_l":
        g = rng.uniform(-1, 1, (n, n))
        return {"C": g @ g.T + n * np.eye(n)}
    if op == "gemm_nt":
        return {"A": rng.standard_normal((n, n)), "B": rng.standard_normal((n, n))}
    if op == "trsm_rltn":
        g = rng.uniform(-1, 1, (n, n))
        return {"S": g @ g.T + n * np.eye(n), "B": rng.uniform(-1, 1, (n, n))}
    raise ValueError(op)


CASES = [
    {"name": "potrf_128", "op": "potrf_l", "n": 128, "seed": 128001},
    {"name": "potrf_256", "op": "potrf_l", "n": 256, "seed": 256001},
    {"name": "gemm_nt_128", "op": "gemm_nt", "n": 128, "seed": 128002},
    {"name": "gemm_nt_300", "op": "gemm_nt", "n": 300, "seed": 300002},
    {"name": "trsm_rltn_128", "op": "trsm_rltn", "n": 128, "seed": 128003},
]


def ref_mat(arr):
    m, n = arr.shape
    x = allocate_panel_matrix(m, n)
    np.asarray(x._base)[:] = 0  # padding slots too: the digest covers the whole item
    for i in range(m):
        for j in range(n):
            x.data[element_offset(i, j, 4, x.panel_length)] = arr[i, j]
    return x


def item_bytes(x):
    return np.asarray(x._base if x._base is not None else x.data).view(np.uint8).tobytes()


def run(case):
    n = case["n"]
    a = inputs(case)
    if case["op"] == "potrf_l":
        C = ref_mat(a["C"])
        D = ref_mat(np.zeros((n, n)))
        level3.potrf_l(n, C, D)
        out = D
    elif case["op"] == "gemm_nt":
        A, B = ref_mat(a["A"]), ref_mat(a["B"])
        D = ref_mat(np.zeros((n, n)))
        level3.gemm_nt(n, n, n, 1.0, A, B, 0.0, D, D)
        out = D
    else:
        S = ref_mat(a["S"])
        L = ref_mat(np.zeros((n, n)))
        level3.potrf_l(n, S, L)
        B = ref_mat(a["B"])
        X = ref_mat(np.zeros((n, n)))
        level3.trsm_rltn(n, n, 1.0, L, B, X)
        out = X
    raw = item_bytes(out)
    data = out.data
    picks = [0, 5, n + 3, len(data) // 2, len(data) - 1]
    return {"sha256": hashlib.sha256(raw).hexdigest(), "bytes": len(raw),
            "samples": {str(p): float(data[p]).hex() for p in picks}}


def main():
    out = []
    for c in CASES:
        rec = dict(c)
        rec.update(run(c))
        out.append(rec)
        print(c["name"], rec["sha256"][:16])
    with open(os.path.join(HERE, "golden_large_v1.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden_large.py", "cases": out}, fh, indent=1)


if __name__ == "__main__":
    main()
