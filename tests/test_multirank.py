"""CPU, world_size 2 over gloo: the multi-GPU host logic.

Each rank takes its contiguous shard of a seeded batch, factors it (the
oracle stands in for the device here -- no GPU in this container), and the
gathered results/statuses must equal the single-process run bit for bit;
max-over-ranks timing reduction is checked too.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1704_02457_b200.multigpu import gather_rows, max_over_ranks, shard_range
from oracle import oracle as O


def test_shard_range_partitions_exactly():
    for total in (0, 1, 7, 1273, 4096, 805306368):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _batch(nb, n, seed):
    rng = np.random.default_rng(seed)
    g = rng.uniform(-1, 1, (nb, n, n))
    a = g @ g.transpose(0, 2, 1) + n * np.eye(n)
    a[3, 2, 2] = -1.0  # one failing item
    C = O.HostBatch(nb, n, n)
    C.set_window(0, 0, a)
    return C


def _worker(rank, world, port, nb, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    C = _batch(nb, n, 5)
    lo, hi = shard_range(nb, rank, world)
    Cl = O.HostBatch(hi - lo, n, n, C.storage[lo:hi].copy())
    Dl = O.HostBatch(hi - lo, n, n)
    info = O.potrf_l(n, Cl, 0, 0, Dl, 0, 0)
    allD = gather_rows(torch.from_numpy(Dl.storage), world)
    allI = gather_rows(torch.from_numpy(info.astype(np.int64)), world)
    t = max_over_ranks(1.0 + rank)
    if rank == 0:
        q.put((allD.numpy(), allI.numpy(), t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_factorization_matches_single_process():
    nb, n, world = 37, 11, 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nb, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    D, I, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    C = _batch(nb, n, 5)
    Dref = O.HostBatch(nb, n, n)
    info = O.potrf_l(n, C, 0, 0, Dref, 0, 0)
    assert np.array_equal(I, info.astype(np.int64))
    assert np.array_equal(D.view(np.uint64), Dref.storage.view(np.uint64))
    assert t == 2.0
