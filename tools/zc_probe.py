"""Probe: potrf_l on HOST (pinned, UVA-mapped) panel-major buffers, the kernel
reading C and writing D across PCIe directly, against the copy-engine
pipeline (H2D C, factor, D2H D on two streams).  Prints GB/s-equivalent
item rates and checks bit-equality with the device-resident result and
that D's strict upper (sentinel) stays untouched on the host.
Usage (GPU box): python tools/zc_probe.py [n ...]
"""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1704_02457_b200 as pb  # noqa: E402
from paper_1704_02457_b200 import _native, level3  # noqa: E402


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def main():
    ns = [int(x) for x in sys.argv[1:]] or [4, 8, 16, 32, 64]
    dev = torch.device("cuda", 0)
    pb.load_native()
    for n in ns:
        per = bench.memsize(n, n)
        nb = int(1.5e9 // per)
        pt = bench.Point("potrf_l", n, n, 0, nb)
        gp = bench.GpuPoint(pt, nb, dev, seed=5)
        hC = gp.C.storage.cpu().pin_memory()
        hD = torch.full_like(hC, float("nan")).pin_memory()
        hD2 = torch.empty_like(hC).pin_memory()
        info = torch.empty(nb, dtype=torch.int32, device=dev)
        # device-resident reference result
        level3.potrf_l(n, gp.C, gp.D, check=False)
        ref = gp.D.storage.cpu()
        st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        Ch = pb.create_panel_batch(nb, n, n, hC)
        Dh = pb.create_panel_batch(nb, n, n, hD)
        dc, dd = Ch.descriptor(), Dh.descriptor()

        def zc():
            _native.call("pb_dpotrf_l", n, n, ctypes.byref(dc), 0, 0, ctypes.byref(dd), 0, 0,
                         ctypes.c_void_p(info.data_ptr()), st)

        t_zc = timeit(zc)
        # correctness: lower + diag_inv bit-equal, strict upper still NaN
        lower = torch.zeros_like(ref[0], dtype=torch.bool)
        for i in range(n):
            for j in range(i + 1):
                lower[pb.element_offset(i, j, 4, gp.D.panel_length)] = True
        dinv0 = gp.D._diag_off
        lower[dinv0:dinv0 + n] = True
        same = bool(torch.equal(hD[:, lower], ref[:, lower]))
        upper = ~lower
        upper[dinv0:] = False
        up_ok = bool(torch.isnan(hD[:, upper]).all()) if upper.any() else True
        streams = [torch.cuda.Stream(dev) for _ in range(2)]
        sub = max(1, int(128e6 // per))

        def ce():
            k = 0
            for s0 in range(0, nb, sub):
                s1 = min(nb, s0 + sub)
                s = streams[k % 2]
                k += 1
                with torch.cuda.stream(s):
                    gp.C.storage[s0:s1].copy_(hC[s0:s1], non_blocking=True)
                    cin = pb.create_panel_batch(s1 - s0, n, n, gp.C.storage[s0:s1])
                    dout = pb.create_panel_batch(s1 - s0, n, n, gp.D.storage[s0:s1])
                    level3.potrf_l(n, cin, dout, check=False)
                    hD2[s0:s1].copy_(gp.D.storage[s0:s1], non_blocking=True)
            for s in streams:
                s.synchronize()

        t_ce = timeit(ce)
        gf = nb * (n ** 3 / 3.0) / 1e9
        print(f"n={n} items={nb} item_bytes={per}: zero-copy {t_zc * 1e3:.1f} ms ({gf / t_zc:.1f} GF/s, "
              f"{nb * per / t_zc / 1e9:.1f} GB/s item-eq) | copy-engine {t_ce * 1e3:.1f} ms ({gf / t_ce:.1f} GF/s) "
              f"| bit-equal {same} upper-untouched {up_ok}", flush=True)
        del gp, hC, hD, hD2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
