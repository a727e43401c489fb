"""Run a few batched potrf_l launches at one size (for ncu captures)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1704_02457_b200 as pb
from paper_1704_02457_b200 import level3, pack

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nb = int(sys.argv[2]) if len(sys.argv) > 2 else max(1, (1 << 31) // (n * n * 8 * 4))
if nb == 0:  # C2 batch: ~2^34 flop, capped at the bench's resident chunk
    nb = min(round(2 ** 34 / (n ** 3 / 3.0)), int(6e9 // (2 * 8 * (n + 4) * (n + 4))))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
g = torch.Generator(device="cuda").manual_seed(0)
M = torch.rand((nb, n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
a = torch.baddbmm(torch.eye(n, dtype=torch.float64, device="cuda").expand(nb, n, n) * n, M, M.transpose(1, 2))
del M
C = pack.panel_from_array(a)
del a
import os
D = C if os.environ.get("INPLACE") else pb.allocate_panel_batch(nb, n, n, zero=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
for r in range(reps):
    e0.record()
    level3.potrf_l(n, C, D, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    alg = nb * 8.0 * (n * (n + 1) + n)
    print(f"potrf n={n} batch={nb}: {ms:.3f} ms, {nb * n**3 / 3 / ms / 1e6:.1f} GFLOP/s, alg {alg / ms / 1e6:.1f} GB/s")
