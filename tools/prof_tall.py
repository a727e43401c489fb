"""Time batched potrf_l on tall windows (m > n): python tools/prof_tall.py [batch]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1704_02457_b200 as pb
from paper_1704_02457_b200 import level3, pack

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
for (m, n) in [(256, 128), (200, 100), (160, 96), (136, 72), (128, 128), (96, 40)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    M = torch.rand((nb, n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    a = torch.empty((nb, m, n), dtype=torch.float64, device="cuda")
    a[:, :n] = torch.baddbmm(torch.eye(n, dtype=torch.float64, device="cuda").expand(nb, n, n) * n, M, M.transpose(1, 2))
    a[:, n:] = torch.rand((nb, m - n, n), dtype=torch.float64, device="cuda", generator=g)
    C = pack.panel_from_array(a)
    D = pb.allocate_panel_batch(nb, m, n, zero=True)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for r in range(4):
        e0.record()
        level3.potrf_l(m, C, D, n=n, check=False)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    fl = nb * (n ** 3 / 3.0 + (m - n) * n * n)
    print(f"potrf {m}x{n} batch {nb}: {best:.3f} ms, {fl / best / 1e6:.0f} GFLOP/s")
