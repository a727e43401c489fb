"""Raw PCIe copy bandwidth (pinned host <-> device), alone and concurrent, for the e2e ceiling."""
import time
import torch

def bw(size_mb=512, reps=8, streams=2):
    n = size_mb * 2**20 // 8
    h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(streams)]
    ho = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(streams)]
    d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(streams)]
    ss = [torch.cuda.Stream() for _ in range(streams)]
    out = {}
    for mode in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for r in range(reps):
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    if mode in ("h2d", "both"):
                        d[i].copy_(h[i], non_blocking=True)
                    if mode in ("d2h", "both"):
                        ho[i].copy_(d[i], non_blocking=True)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        out[mode] = reps * streams * n * 8 / el / 1e9
    return out

for mb, st in ((256, 2), (1024, 2), (256, 4)):
    print(mb, st, {k: round(v, 1) for k, v in bw(mb, 6, st).items()})
