import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1704_02457_b200 as pb
from paper_1704_02457_b200 import level3
from oracle import oracle as O

def dev(h):
    return pb.create_panel_batch(h.batch, h.rows, h.cols, torch.from_numpy(h.storage.copy()).cuda())

def run(n, oc, od, nb=3, seed=1, fail=False):
    rng = np.random.default_rng(seed)
    g = rng.uniform(-1, 1, (nb, n, n)); a = g @ g.transpose(0, 2, 1) + n * np.eye(n)
    if fail: a[0, n // 2, n // 2] = -1.0
    C = O.HostBatch(nb, oc[0] + n + 1, oc[1] + n + 2); C.storage[:] = rng.uniform(-1, 1, C.storage.shape)
    C.set_window(oc[0], oc[1], a)
    D = O.HostBatch(nb, od[0] + n + 2, od[1] + n + 1); D.storage[:] = rng.uniform(-1, 1, D.storage.shape)
    dC, dD = dev(C), dev(D)
    info = level3.potrf_l(n, dC.ref(*oc), dD.ref(*od), check=False).cpu().numpy()
    winfo = O.potrf_l(n, C, *oc, D, *od)
    got = dD.storage.cpu().numpy()
    mask = np.zeros(D.storage.shape[1], dtype=bool)
    for j in range(n):
        for i in range(j, n):
            mask[O.element_offset(od[0] + i, od[1] + j, D.cn)] = True
    mask[D.diag_off + od[1]: D.diag_off + od[1] + n] = True
    bad = np.nonzero((got != D.storage) & ~mask[None, :])
    inv = {}
    for i in range(D.rows + 3):
        for j in range(D.cn):
            inv[O.element_offset(i, j, D.cn)] = (i, j)
    print(n, oc, od, "info", info, winfo, "bad", [(b, inv.get(x, ('pad/dinv', x - D.diag_off))) for b, x in zip(*bad)][:12])

for args in [(6, (2, 1), (0, 3)), (6, (0, 0), (0, 3)), (6, (2, 1), (0, 0)), (6, (0, 1), (0, 0)), (6, (4, 1), (0, 3)), (7, (1, 0), (0, 0)), (12, (3, 2), (0, 1)), (16, (1, 1), (0, 0)), (20, (1, 0), (0, 0))]:
    run(*args)
