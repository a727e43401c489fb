"""Time batched gemm_nt / syrk_ln / trsm_rltn at one shape (for ncu captures and sweeps)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1704_02457_b200 as pb
from paper_1704_02457_b200 import level3, pack

op = sys.argv[1]
m, n, k = (int(x) for x in sys.argv[2].split("x"))
nb = int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
beta = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
g = torch.Generator(device="cuda").manual_seed(0)
if op == "gemm":
    A = pb.allocate_panel_batch(nb, m, k); B = pb.allocate_panel_batch(nb, n, k); C = pb.allocate_panel_batch(nb, m, n)
    for x in (A, B, C):
        x.storage.uniform_(-1, 1, generator=g)
    D = pb.allocate_panel_batch(nb, m, n, zero=True)
    run = lambda: level3.gemm_nt(m, n, k, 1.0, A, B, beta, C, D)
    flops = 2.0 * m * n * k
    byts = 8.0 * (m * k + n * k + (m * n if beta else 0) + m * n)
elif op == "syrk":
    A = pb.allocate_panel_batch(nb, m + 3, k + 1); A.storage.uniform_(-1, 1, generator=g)
    C = pb.allocate_panel_batch(nb, m, m); C.storage.uniform_(-1, 1, generator=g)
    D = pb.allocate_panel_batch(nb, m, m, zero=True)
    a = A.ref(3, 1)
    run = lambda: level3.syrk_ln(m, k, -1.0, a, a, beta, C, D)
    flops = float(m) * (m + 1) * k
    byts = 8.0 * (m * k + (m * (m + 1) / 2 if beta else 0) + m * (m + 1) / 2)
elif op == "trsm":
    M = torch.rand((nb, n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    S = pack.panel_from_array(torch.baddbmm(torch.eye(n, dtype=torch.float64, device="cuda").expand(nb, n, n) * n, M, M.transpose(1, 2)))
    del M
    L = pb.allocate_panel_batch(nb, n, n, zero=True)
    level3.potrf_l(n, S, L)
    B = pb.allocate_panel_batch(nb, m, n); B.storage.uniform_(-1, 1, generator=g)
    D = pb.allocate_panel_batch(nb, m, n, zero=True)
    run = lambda: level3.trsm_rltn(m, n, 1.0, L, B, D, check=False)
    flops = float(m) * n * n
    byts = 8.0 * (n * (n + 1) / 2 + n + 2 * m * n)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
for r in range(reps):
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{op} {m}x{n}x{k} batch={nb}: {ms:.3f} ms, {nb * flops / ms / 1e6:.1f} GFLOP/s, alg {nb * byts / ms / 1e6:.1f} GB/s")
