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


def _stub_draw(plan, coarse_grid, tf, tc, problem, opt, lo, hi, draws, ctx=None, xi=None):
    """A deterministic per-slot 'sample' (no GPU): q_fine = sin(i), q_coarse = cos(i) (+ ξ row sum)."""
    if draws.q_fine.size < hi:
        draws.resize(hi)
    i = np.arange(lo, hi, dtype=np.float64)
    extra = 0.0 if xi is None else np.asarray(xi).reshape(hi - lo, -1).sum(axis=1)
    draws.q_fine[lo:hi] = np.sin(i) + extra
    draws.q_coarse[lo:hi] = np.cos(i)
    draws.wall[lo:hi] = 1e-3
    draws.iters_fine[lo:hi] = (i % 7).astype(np.int32)
    draws.iters_coarse[lo:hi] = (i % 5).astype(np.int32)
    return draws


def _shard_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_13493_b200 import api
        from paper_2306_13493_b200.dist import Shard
        sh = Shard(draw_fn=_stub_draw)
        ok = True
        for frm, to in [(0, 37), (5, 6), (3, 3 + 2 * world + 1), (100, 164)]:  # uneven and short ranges
            d = api.LevelDraws()
            d.resize(frm)
            d.q_fine[:] = -1.0
            xi = np.arange((to - frm) * 4, dtype=np.float64).reshape(to - frm, 4)
            sh.run_level_draws(None, None, False, False, None, None, frm, to, d, xi=xi)
            want = _stub_draw(None, None, False, False, None, None, frm, to, api.LevelDraws(), xi=xi)
            ok &= len(d) == to and np.all(d.q_fine[:frm] == -1.0)
            ok &= np.array_equal(d.q_fine[frm:to], want.q_fine[frm:to])
            ok &= np.array_equal(d.q_coarse[frm:to], want.q_coarse[frm:to])
            ok &= np.array_equal(d.iters_fine[frm:to], want.iters_fine[frm:to])
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_shard_run_level_draws(world):
    """Shard.run_level_draws over world 2 and 3 (uneven splits, ranks with empty shards): every rank
    ends with the slot-ordered draws a single process would produce, ξ rows routed to their shard."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == list(range(world))
    assert all(r[1] for r in res), res
