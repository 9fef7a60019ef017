"""Multi-rank host logic on CPU (gloo, world size 2): contiguous sharding of a level's sample
range, the all-gather of slot-ordered draws and the all-reduce of per-level sums."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_split_range_covers_exactly():
    from paper_2306_13493_b200.dist import split_range
    for count in (0, 1, 7, 64, 1000):
        for world in (1, 2, 4, 8):
            got = []
            for r in range(world):
                lo, hi, _ = split_range(10, 10 + count, r, world)
                got.extend(range(lo, hi))
            assert got == list(range(10, 10 + count))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_13493_b200.dist import Shard, level_sums, moments_from_sums, split_range
        sh = Shard()
        rng = np.random.default_rng(0)
        qf_all, qc_all = rng.standard_normal(37), rng.standard_normal(37)
        lo, hi, chunk = split_range(0, 37, rank, world)
        packed = np.stack([qf_all[lo:hi], qc_all[lo:hi]], axis=1)
        gathered = sh.all_gather_slots(packed, chunk, 37)
        ok_gather = np.array_equal(gathered[:, 0], qf_all) and np.array_equal(gathered[:, 1], qc_all)
        s = sh.all_reduce_sum(level_sums(qf_all[lo:hi], qc_all[lo:hi], 0.1, 0.2))
        n, my, vy, mq, vq = moments_from_sums(s, 0.1, 0.2)
        y = qf_all - qc_all
        ok_sums = n == 37 and abs(my - y.mean()) < 1e-12 and abs(vy - y.var(ddof=1)) < 1e-12
        q.put((rank, ok_gather, ok_sums))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_and_sums():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] and r[2] for r in res)
