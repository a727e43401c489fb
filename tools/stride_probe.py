"""Probe: potrf_l time vs the item stride of the split data plane (power-of-two strides)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1704_02457_b200 as pb
from paper_1704_02457_b200 import level3, pack

torch.cuda.set_device(0)
for n, nb in ((32, 524288), (64, 98304), (16, 2097152), (8, 4194304)):
    per = pb.panel_data_elems(n, n)
    for pad in (0, 8, 16, 32, 64):
        def mk(zero):
            t = (torch.zeros if zero else torch.empty)((nb, per + pad), dtype=torch.float64, device="cuda")
            d = torch.zeros((nb, n), dtype=torch.float64, device="cuda")
            return pb.PanelBatch(nb, n, n, t[:, :per], d)
        C = mk(False)
        step = 1 << 16
        for s0 in range(0, nb, step):
            s1 = min(nb, s0 + step)
            M = torch.rand((s1 - s0, n, n), dtype=torch.float64, device="cuda") * 2 - 1
            pack.pack_array_into(M @ M.transpose(1, 2) + n * torch.eye(n, dtype=torch.float64, device="cuda"),
                                 C.shard(s0, s1))
        D = mk(True)
        for _ in range(3):
            level3.potrf_l(n, C, D, check=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            level3.potrf_l(n, C, D, check=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        alg = nb * 8.0 * (n * (n + 1) + n)
        print(f"n={n} pad={pad:3d} stride={(per + pad) * 8} B  {ms:.3f} ms  {alg / ms / 1e6:.0f} GB/s alg", flush=True)
        del C, D
        torch.cuda.empty_cache()
