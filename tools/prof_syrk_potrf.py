"""Time batched syrk_potrf_ln beyond the register-tile sizes: python tools/prof_syrk_potrf.py [batch]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1704_02457_b200 as pb
from paper_1704_02457_b200 import level3, pack

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for (m, n, k) in [(128, 128, 64), (96, 96, 40), (100, 100, 32), (72, 72, 72), (160, 96, 40), (64, 64, 32)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = pack.panel_from_array(torch.rand((nb, m, k), dtype=torch.float64, device="cuda", generator=g) * 0.2)
    M = torch.rand((nb, m, m), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    c = torch.baddbmm(torch.eye(m, dtype=torch.float64, device="cuda").expand(nb, m, m) * m, M, M.transpose(1, 2))[:, :, :n]
    C = pack.panel_from_array(c.contiguous())
    D = pb.allocate_panel_batch(nb, m, n, zero=True)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for r in range(4):
        e0.record()
        level3.syrk_potrf_ln(m, k, A, A.ref(0, 0) if n == m else pb.SubRef(A, 0, 0), C, D, n=n, check=False)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    fl = nb * (n * (n + 1) * k + (m - n) * n * 2 * k + n ** 3 / 3.0 + (m - n) * n * n)
    print(f"syrk_potrf {m}x{n} k={k} batch {nb}: {best:.3f} ms, {fl / best / 1e6:.0f} GFLOP/s")
