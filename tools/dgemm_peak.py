"""cuBLAS DGEMM throughput via torch.matmul(float64): the library FP64 peak reference."""
import torch, json
torch.backends.cuda.matmul.allow_tf32 = False
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        e0.record(); a @ b; e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    res[n] = 2 * n**3 / best / 1e6
print(json.dumps({"dgemm_gflops": res, "name": torch.cuda.get_device_name()}))
