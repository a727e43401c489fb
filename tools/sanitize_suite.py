"""Reduced GPU workload for compute-sanitizer (memcheck / racecheck / synccheck):
one small batch per kernel-dispatch regime of the product path, each operand
in its own exactly sized allocation (run with PYTORCH_NO_CUDA_MEMORY_CACHING=1
so every tensor is its own cudaMalloc and an access past an operand's last
item is outside any allocation).

    compute-sanitizer --tool memcheck python tools/sanitize_suite.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_02457_b200 as pb  # noqa: E402
from paper_1704_02457_b200 import level3, pack  # noqa: E402
from paper_1704_02457_b200.chain import RiccatiChain  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(0)


def spd(nb, n):
    g = rng.uniform(-1, 1, (nb, n, n))
    return torch.from_numpy(g @ g.transpose(0, 2, 1) + n * np.eye(n)).cuda()


def exact(nb, m, n, layout="split"):
    return pb.allocate_panel_batch(nb, m, n, zero=True, layout=layout)


def run():
    done = []
    # potrf: n <= 8 (small1), 16 (quad), 17..64 (register tile + exact pass), 65..128 (chain kernel),
    # 256 / 300 (blocked: trsm + syrk trapezoid + commit), tall windows, unaligned D, failing items
    for n, nb in ((4, 300), (8, 200), (16, 100), (24, 64), (64, 32), (100, 8), (128, 6), (256, 3), (300, 2)):
        for layout in ("split", "interleaved"):
            a = spd(nb, n)
            a[0, n // 2, n // 2] = -1.0  # one failing item
            if n >= 24:
                a[1, n - 1, 2] = float("nan")  # non-finite -> reference-order pass
            C = exact(nb, n, n, layout)
            pack.pack_array_into(a, C)
            D = exact(nb, n, n, layout)
            level3.potrf_l(n, C, D, check=False)
            level3.potrf_l(n, C, C, check=False)  # in place
        done.append(f"potrf n={n}")
    for m, n in ((300, 264), (320, 240), (600, 20), (520, 40), (256, 128), (109, 31)):  # tall: square factor + solve
        a = torch.from_numpy(rng.uniform(-1, 1, (2, m, n))).cuda()
        a[:, :n, :] = spd(2, n)
        C = exact(2, m, n)
        pack.pack_array_into(a, C)
        level3.potrf_l(m, C, exact(2, m, n), n=n, check=False)
        done.append(f"potrf tall {m}x{n}")
    a = spd(3, 136)
    C = exact(3, 137, 137)
    pack.pack_array_into(a, C.ref(1, 1))
    level3.potrf_l(136, C.ref(1, 1), exact(3, 137, 137).ref(1, 1), check=False)  # unaligned blocked
    done.append("potrf unaligned blocked")
    # gemm / syrk: item kernel, direct (<= 24), TMA pipeline with C through smem (beta != 0), unaligned rows
    for (m, n, k, beta) in ((4, 4, 4, 1.0), (16, 16, 16, 0.0), (24, 20, 9, 1.0), (64, 64, 64, 1.0),
                            (100, 72, 40, 1.0), (300, 300, 300, 0.0)):
        nb = max(2, 20000 // (m * n))
        A, B, Cm, D = exact(nb, m + 3, k), exact(nb, n, k), exact(nb, m, n), exact(nb, m, n)
        for x in (A, B, Cm):
            x.storage.uniform_(-1, 1)
        level3.gemm_nt(m, n, k, 1.0, A.ref(3, 0), B, beta, Cm, D)
        level3.gemm_nt(m, n, k, 1.0, A, B, beta, Cm, D)
        S = exact(nb, m, m)
        level3.syrk_ln(m, k, -1.0, A.ref(3, 0), A.ref(3, 0), beta, exact(nb, m, m), S)
        done.append(f"gemm/syrk {m}x{n}x{k}")
    # trsm (team widths), blocked trsm (n > team), gemm_nn, trmm in place (workspace), syrk_potrf fused / split
    for m, n in ((72, 48), (9, 300), (40, 64), (130, 125), (64, 128)):  # the last two: register-strip kernel
        L = exact(4, n, n)
        Cs = exact(4, n, n)
        pack.pack_array_into(spd(4, n), Cs)
        level3.potrf_l(n, Cs, L)
        X = exact(4, m, n)
        level3.trsm_rltn(m, n, 1.0, L, exact(4, m, n), X)
        level3.trsm_rltn(m, n, 1.0, L.ref(0, 0), X, X, check=False)
        done.append(f"trsm {m}x{n}")
    A, B, Cm = exact(8, 64, 64), exact(8, 64, 64), exact(8, 64, 64)
    for x in (A, B, Cm):
        x.storage.uniform_(-1, 1)
    level3.gemm_nn(64, 64, 64, 1.0, A, B, 1.0, Cm, exact(8, 64, 64))
    level3.trmm_rlnn(40, 32, 1.0, A.ref(0, 0), B, B)  # in place -> workspace copy
    Cs = exact(8, 40, 40)
    pack.pack_array_into(spd(8, 40) * 40, Cs)
    level3.syrk_potrf_ln(40, 32, A, A, Cs, exact(8, 40, 40), check=False)
    Cb = exact(2, 260, 260)
    pack.pack_array_into(spd(2, 260) * 260, Cb)
    level3.syrk_potrf_ln(260, 100, exact(2, 260, 100), exact(2, 260, 100), Cb, exact(2, 260, 260), check=False)
    done.append("gemm_nn / trmm / syrk_potrf")
    # getrf, pack / unpack chunks (col-major, row-major, partial panel), gecp, Riccati chain
    G = exact(16, 32, 32)
    G.storage.uniform_(-1, 1)
    level3.getrf_pivot(32, 32, G, exact(16, 32, 32), check=False)
    for m, n in ((4, 4), (7, 5), (64, 64)):
        arr = torch.rand((50, m, n), dtype=torch.float64, device="cuda")
        P = pack.panel_from_array(arr)
        cb = pack.ColBatch.from_array(arr)
        pack.pack_matrix(cb, m, n, P)
        pack.unpack_matrix(P, m, n, cb)
        pack.gecp(m, n, P, exact(50, m, n))
        pack.panel_to_array(P)
    ch = RiccatiChain(8, 32, 8)
    for x in (ch.BAt, ch.RQ, ch.P):
        x.storage.uniform_(-0.1, 0.1)
    ch.run_fused(3)
    done.append("getrf / pack / chain")
    torch.cuda.synchronize()
    print("sanitize suite ok:", "; ".join(done))


if __name__ == "__main__":
    run()
