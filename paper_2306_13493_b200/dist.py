"""Multi-GPU sharding of a level's sample range — one process per GPU, torch.distributed
plumbing (NCCL over NVLink/NVSwitch on B200, gloo for the CPU tests).

MLMC samples are independent and sample i always uses NormalStream(seed, ℓ, i) and lands
in slot i (estimators.hpp:112-114), so [from, to) is split into contiguous per-rank chunks
(the std::thread chunking of parallel_samples, estimators.cpp:46-50) with no data-path
collective. The only exchanges are (a) one all-reduce of the per-level sums
[n, Σ(Y−K), Σ(Y−K)², Σ(q−K_q), Σ(q−K_q)²] per batch, and (b) an all-gather of the
per-sample (q_fine, q_coarse) slots (16 B/sample) so every rank can run the reference's
slot-ordered Welford (moments_of) bit-identically for any GPU count.
"""
from __future__ import annotations

import numpy as np


def split_range(frm: int, to: int, rank: int, world: int):
    """Contiguous chunk of [frm, to) owned by `rank` (chunk = ceil(count/world))."""
    count = max(0, to - frm)
    chunk = (count + world - 1) // world if world > 0 else count
    lo = min(to, frm + rank * chunk)
    hi = min(to, lo + chunk)
    return lo, hi, chunk


class Shard:
    """Shards run_level_draws over the ranks of a torch.distributed process group."""

    def __init__(self, group=None, draw_fn=None):
        """draw_fn(plan, coarse_grid, tf, tc, problem, opt, lo, hi, draws, ctx=, xi=) draws the local
        shard into `draws` (default: api.run_level_draws on this rank's GPU); tests inject a stub."""
        import torch.distributed as dist
        if not dist.is_initialized():
            raise RuntimeError("Shard needs torch.distributed to be initialised")
        self.dist = dist
        self.draw_fn = draw_fn
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def _device(self):
        import torch
        if self.backend == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    def all_reduce_sum(self, values: np.ndarray) -> np.ndarray:
        """One fp64 sum all-reduce (per-level sums), returned on the host."""
        import torch
        t = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float64), device=self._device()).clone()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def all_gather_slots(self, local: np.ndarray, chunk: int, total: int) -> np.ndarray:
        """Gather per-rank contiguous chunks (padded to `chunk`) back into slot order."""
        import torch
        buf = np.zeros((chunk,) + local.shape[1:], dtype=local.dtype)
        buf[:local.shape[0]] = local
        t = torch.as_tensor(buf, device=self._device())
        out = torch.empty((self.world * chunk,) + tuple(local.shape[1:]), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy()[:total]

    def run_level_draws(self, plan, coarse_grid, truncate_fine, truncate_coarse, problem, opt, frm,
                        to, draws, ctx=None, xi=None):
        from . import api
        lo, hi, chunk = split_range(frm, to, self.rank, self.world)
        local = api.LevelDraws()
        xi_local = None if xi is None else np.asarray(xi).reshape(to - frm, -1)[lo - frm:hi - frm]
        if hi > lo:
            fn = self.draw_fn or api.run_level_draws
            fn(plan, coarse_grid, truncate_fine, truncate_coarse, problem, opt, lo, hi, local, ctx=ctx, xi=xi_local)
        n = hi - lo
        packed = np.zeros((n, 5))
        if n:
            packed[:, 0] = local.q_fine[lo:hi]
            packed[:, 1] = local.q_coarse[lo:hi]
            packed[:, 2] = local.wall[lo:hi]
            packed[:, 3] = local.iters_fine[lo:hi]
            packed[:, 4] = local.iters_coarse[lo:hi]
        allp = self.all_gather_slots(packed, chunk, to - frm)
        if draws.q_fine.size < to:
            draws.resize(to)
        draws.q_fine[frm:to] = allp[:, 0]
        draws.q_coarse[frm:to] = allp[:, 1]
        draws.wall[frm:to] = allp[:, 2]
        draws.iters_fine[frm:to] = allp[:, 3].astype(np.int32)
        draws.iters_coarse[frm:to] = allp[:, 4].astype(np.int32)
        return draws


def level_sums(q_fine: np.ndarray, q_coarse, shift_y: float, shift_q: float) -> np.ndarray:
    """Host restatement of the device level sums (for the all-reduce path on CPU ranks). The shifts
    must be common to all ranks and close to the level means (e.g. the pilot means), so the variance
    (Σ(Y−K)² − (Σ(Y−K))²/n)/(n−1) does not cancel."""
    y = (q_fine - q_coarse if q_coarse is not None else q_fine) - shift_y
    q = q_fine - shift_q
    return np.array([q_fine.size, y.sum(), (y * y).sum(), q.sum(), (q * q).sum()])


def moments_from_sums(s: np.ndarray, shift_y: float, shift_q: float):
    """(n, mean_y, var_y, mean_q, var_q) from all-reduced shifted sums."""
    n = s[0]
    mean_y = s[1] / n + shift_y
    var_y = (s[2] - s[1] * s[1] / n) / (n - 1) if n >= 2 else 0.0
    mean_q = s[3] / n + shift_q
    var_q = (s[4] - s[3] * s[3] / n) / (n - 1) if n >= 2 else 0.0
    return int(n), mean_y, var_y, mean_q, var_q
