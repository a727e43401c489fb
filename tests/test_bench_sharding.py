"""CPU, world_size 2 over gloo: bench.py's batch sharding and accounting.

Strong scaling (the default): the ranks' shares of every configured point
are disjoint, contiguous and together exactly the configured batch, and the
chunk x repetition plan of each share processes exactly its items.  Weak
scaling (--weak) gives every rank the whole batch.  Also: a --gpus/WORLD_SIZE
mismatch is refused.
"""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO

sys.path.insert(0, REPO)
import bench  # noqa: E402


def _all_points():
    pts = []
    for c in ("c2", "c1", "c3", "c4", "c5", "c6", "pack"):
        pts += bench.config_points(c)[0]
    return pts


def test_plan_point_covers_share_exactly():
    for pt in _all_points():
        for world in (1, 2, 3, 8):
            spans = []
            for rank in range(world):
                lo, hi, chunk, reps, last = plan = bench.plan_point(pt, rank, world)
                assert bench.items_of(plan) == hi - lo
                if reps:
                    assert 0 < last <= chunk and chunk * (reps - 1) + last == hi - lo
                    assert chunk * pt.io_bytes <= max(pt.cap_bytes, pt.io_bytes) * 1.0001
                spans.append((lo, hi))
            assert spans[0][0] == 0 and spans[-1][1] == pt.batch
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_config_batches_match_baseline():
    c2, _ = bench.config_points("c2")
    assert [p.batch for p in c2] == [round(2 ** 34 / (n ** 3 / 3.0)) for n in (4, 8, 16, 32, 64, 128, 256)]
    assert c2[0].batch == 805306368
    c3, _ = bench.config_points("c3")
    assert [p.n for p in c3] == list(range(4, 301, 4))
    assert c3[0].batch == 536870912 and c3[-1].batch == 1273  # SURVEY §8d examples
    c1, _ = bench.config_points("c1")
    assert (c1[0].m, c1[0].n, c1[0].k, c1[0].batch, c1[0].beta) == (64, 64, 64, 4096, 1.0)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pts = _all_points()
    strong = torch.tensor([bench.items_of(bench.plan_point(p, rank, world)) for p in pts], dtype=torch.float64)
    weak = torch.tensor([bench.items_of(bench.plan_point(p, rank, world, weak=True)) for p in pts],
                        dtype=torch.float64)
    dist.all_reduce(strong)
    dist.all_reduce(weak)
    # the bench's own reductions (sum of items, max of times) over gloo
    s = bench._sum_over_ranks([float(rank + 1)], None, world)
    m = bench._max_over_ranks([float(rank + 1)], None, world)
    if rank == 0:
        q.put((strong.tolist(), weak.tolist(), s, m))
    dist.destroy_process_group()


def test_bench_accounting_world2_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    strong, weak, ssum, smax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pts = _all_points()
    assert strong == [float(p.batch) for p in pts]  # strong: every configured item exactly once
    assert weak == [2.0 * p.batch for p in pts]
    assert ssum == [3.0] and smax == [2.0]


def test_gpus_world_size_mismatch_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--steps", "1"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr


def test_unknown_config_rejected():
    with pytest.raises(SystemExit):
        bench.config_points("c9")
