#!/usr/bin/env python
"""Benchmark of the MLMC sample path: MLMC samples/s per level (CE field + Darcy solve, fp64)
and its fraction of the B200 HBM roofline.

Default workload (BASELINE.json config 4, the per-level CE + MG-PCG configuration that is
sharded across GPUs): Matérn ν=0.5, σ²=2, λ=0.003; coupled (2048², 1024²) samples, batches of
64 per GPU; f = 1; homogeneous Dirichlet on all sides; MG-PCG to relative residual 1e-10; fp64.
A step = one batch of 64 coupled samples through osc_level_draws (ξ from the device Philox
stream NormalStream(seed, ℓ, i), fine + coarse fields, both solves, QoIs, level sums).
Per-GPU work is fixed as N grows (weak scaling: rank r draws its own contiguous index range).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4|1|2|3]

Rank 0 prints ONE JSON line. `--impl reference` times the reference's CPU implementation of the
same workload on the host cores (oracle/_ref for the reference's own BCs; the oracle port for
the all-Dirichlet extension the reference lacks) — rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


# ---- workloads ---------------------------------------------------------------------------------
def workload(cfg: str):
    """(name, dict) for a BASELINE config; per-sample algorithmic bytes follow SURVEY §8(d).
    `it` = the reference algorithm's median PCG iterations for that config and BC (SURVEY §8(d):
    "re-measure with the extension BCs for cfgs 1 and 4"; profiles/oracle_iters.json from
    scripts/oracle_iters.py, seed 1, sample indices 0..7), so our preconditioner does not move
    the basis."""
    if cfg == "4":
        return dict(name="cfg4: matern nu=0.5 s2=2 lam=0.003, coupled 2048^2/1024^2, dirichlet-all, f=1, MG-PCG 1e-10",
                    family="matern", sigma2=2.0, lam=0.003, nu=0.5, m=2048, coupled=True, bc=1, qoi=0,
                    batch=64, ell=1, it=(61.5, 60.5))
    if cfg == "2":
        return dict(name="cfg2: CE field sampling only, matern nu=1.5 s2=1 lam=0.01, 1024^2 (n=2048), 4096 samples/batch",
                    family="matern", sigma2=1.0, lam=0.01, nu=1.5, m=1024, coupled=False, bc=0, qoi=0,
                    batch=4096, ell=0, it=(0, 0), ce_only=True)
    if cfg == "1":
        return dict(name="cfg1: matern nu=0.5 s2=1 lam=0.1, 64^2 single-level MC, dirichlet-all, integral QoI",
                    family="matern", sigma2=1.0, lam=0.1, nu=0.5, m=64, coupled=False, bc=1, qoi=2,
                    batch=1000, ell=0, it=(17, 0))
    if cfg == "3":
        return dict(name="cfg3 level 4: sep-exp s2=1 lam=0.01, coupled 256^2/128^2, flow-cell, flux QoI",
                    family="sep", sigma2=1.0, lam=0.01, nu=1.0, m=256, coupled=True, bc=0, qoi=3,
                    batch=1024, ell=4, it=(25, 24))
    raise SystemExit(f"unknown config {cfg}")


def algorithmic_bytes_per_sample(W, n, it=None):
    """B = B_ce + B_solve(m) + B_solve(m/2), B_solve(m) = (m+1)²(200 + 251 it),
    B_ce (device ξ, √λ amortised over the batch) = 8 s/B + 32 n (n/2+1) + 8 (N_f + N_c).
    `it` overrides the basis iteration counts (fine, coarse) with measured ones."""
    m = W["m"]
    s = n * n
    Nf, Nc = (m + 1) ** 2, (m // 2 + 1) ** 2
    b_ce = 8 * s / W["batch"] + (32 * n * (n // 2 + 1) if 16 * n * (n // 2 + 1) > 227 * 1024 else 0) + \
        8 * (Nf + (Nc if W["coupled"] else 0))
    itf, itc = W["it"] if it is None else it
    b = b_ce + Nf * (200 + 251 * itf)
    if W["coupled"]:
        b += Nc * (200 + 251 * itc)
    return b


# Per-kernel compulsory HBM bytes per node of the grid the kernel runs on: every
# input read once and every output written once, for one active sample and one V-cycle / PCG
# iteration (a sample runs one of each per iteration). Level 0 keeps nodal k (8 B/node, the
# 5-point rows are rebuilt in registers); coarse levels store the 9-point Galerkin rows as an fp64
# diagonal and fp32 E, N, NE, NW couplings (24 B/node); `pw` = the four fp32 centre prolongation
# weights per coarse cell (4 B per fine node); a coarse-grid array costs ¼ of its fine-grid size.
KERNEL_BYTES = {
    "pcg_update": 8 * 8,                   # one-reduction PCG: read k, z, p_old, r, u; write p, u, r
    "pcg_apply": 4 * 8,                    # single-level PCG (m <= 4): read k, z, p_old; write p_new
    "pcg_update_down": 7 * 8,              # single-level PCG: read k, p, r, u; write u, r, z
    "mg_restrict_r.L0": 8 + 8 + 4 + 2,     # read k, r, pw (fp32); write rc (pre-smoother recomputed)
    "mg_smooth_up_r.L0": 8 + 8 + 2 + 4 + 8,  # read k, r, zc, pw (fp32); write z
    "mg_down": 8 + 16 + 8 + 4 + 2,         # fused pre + restrict: read C (fp64), E N NE NW (fp32), r, pw; write rc
    "mg_up": 8 + 16 + 8 + 2 + 4 + 8,       # prolong + post (z recomputed): read C, E..NW, r, zc, pw; write z2
}


def mg_hierarchy(m):
    """Grid sizes of the solver's levels and the first level of the CTA-resident tail, as
    solver_prepare / vcycle build them (csrc/mgpcg.cu): halve while even down to m ≤ 4; the tail
    starts at the first level l ≥ 1 with m_l ≤ 32 that has at least one level below it."""
    ms = [m]
    while ms[-1] > 4 and ms[-1] % 2 == 0 and len(ms) < 12:
        ms.append(ms[-1] // 2)
    ls = len(ms) - 1
    for l in range(1, len(ms) - 1):
        if ms[l] <= 32:
            ls = l
            break
    return ms, ls


def kernel_nodes(name, m_top):
    """(bytes per node, nodes per sample-launch summed over the levels the class covers) of a
    kernel-stats class "<base>[.L0|.Lc|.L<l>]" on the hierarchy of an m_top solve, or None."""
    base, _, lv = name.partition(".")
    if name in KERNEL_BYTES:
        per = KERNEL_BYTES[name]
        lv = "L0" if base.startswith("pcg_") or lv == "L0" else lv
    elif base in KERNEL_BYTES:
        per = KERNEL_BYTES[base]
    else:
        return None
    ms, ls = mg_hierarchy(m_top)
    if lv == "L0":
        levels = [0]
    elif lv == "Lc":
        levels = list(range(1, ls))
    elif lv.startswith("L") and lv[1:].isdigit():
        levels = [int(lv[1:])]
    else:
        return None
    return per, sum((ms[l] + 1) ** 2 for l in levels)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, period_ms: int = 200):
        # One nvidia-smi query costs the process ≈ 50 ms of stalled launches / synchronisations (NVML and
        # the CUDA driver share a lock): invisible in the 190 ms steps of config 4 (the recipe's 200 ms
        # period), but a third of a step on the host-polled 256² level of config 3 (15.8k samples/s with one
        # query inside the timed region, 20.9k without) — the small workloads sample once per second, so
        # their short timed regions are normally reported from the warm-up window (see mark()).
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def wait_ready(self, timeout: float = 10.0):
        """Block until nvidia-smi has produced its first row: its NVML start-up (hundreds of ms,
        driver calls) then lies before the timed region instead of stalling its first step."""
        t0 = time.perf_counter()
        while self.proc and not self.rows and self.proc.poll() is None and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)

    def mark(self):
        """Start of the timed region: rows sampled from here on are the ones reported. A timed region
        shorter than the 200 ms sampling period (the few-ms steps of the small configs) may end before a
        row arrives: stop() then reports the rows of the last two seconds BEFORE the mark, i.e. of the
        warm-up steps that ran back to back into the timed region, and says so in `window`."""
        self.t_mark = time.perf_counter()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts + [time.perf_counter()])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        t_mark = getattr(self, "t_mark", 0.0)
        window = "timed region"
        rows = [r for r in self.rows if r[6] >= t_mark]
        if not rows:
            rows = [r for r in self.rows if r[6] >= t_mark - 2.0]
            window = "warm-up steps under load within 2 s before the timed region (region shorter than the sampling period)"
        self.rows = rows
        self.window = window
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows),
                "window": self.window}


# ---- reference (CPU) arm --------------------------------------------------------------------------
# Nothing here imports the product package: the spectra come from the pristine reference's own
# build_operator (oracle/_ref), the samples from the pristine reference (flow-cell BCs, Point/L2 QoI)
# or, for the extensions it lacks (all-Dirichlet BCs, ∫u / flux QoIs), the oracle's C restatement.
def cpu_model() -> str:
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _ref_spectrum(W, ref, O):
    key = ("eig", W["m"], W["family"], W["lam"])
    if key not in _CACHE:
        fam = O.MATERN if W["family"] == "matern" else O.SEP_EXP
        r = ref.build_operator(W["m"], fam, W["sigma2"], W["lam"], W["nu"] if W["family"] == "matern" else 1.0)
        _CACHE[key] = (r.n, np.sqrt(np.maximum(r.eigenvalues(), 0.0)))
    return _CACHE[key]


def cpu_reference_step(W, threads: int, n_samples: int, seed_index: int, port, ref):
    """n_samples coupled samples of the workload on the CPU path with `threads` threads: the pristine
    reference (oracle/_ref: make_level_plan + coupled_sample) for its own BCs / QoIs, else the oracle
    port on the reference's spectrum."""
    from oracle import oracle as O
    m = W["m"]
    if W["bc"] == 0 and W["qoi"] in (0, 1):
        opts = O.RefOpts.make(family=O.MATERN if W["family"] == "matern" else O.SEP_EXP,
                              sigma2=W["sigma2"], lam=W["lam"], nu_or_p=W["nu"], qoi_kind=W["qoi"],
                              seed=1, threads=threads)
        key = ("plan", m)
        if key not in _CACHE:
            _CACHE[key] = ref.plan(W["ell"], 1.0 / (m >> W["ell"]), opts)
        t0 = time.perf_counter()
        ref.coupled(_CACHE[key], W["coupled"], False, False, opts, seed_index, seed_index + n_samples)
        return time.perf_counter() - t0, "reference"
    n, sl = _ref_spectrum(W, ref, O)
    t0 = time.perf_counter()
    port.coupled(m, n, sl, None, W["coupled"], 1, W["ell"], seed_index, seed_index + n_samples,
                 bc=W["bc"], qoi=W["qoi"], threads=threads)
    return time.perf_counter() - t0, "port"


_CACHE = {}


def cpu_baseline_block(W, budget_s: float):
    """cpu_baseline of our arm: all host threads on a bounded sample, plus a 1-thread rate."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    ref, port = O.Ref(), O.Port()
    if W.get("ce_only"):
        dt, kind = cpu_ce_step(W, cores, ref, O)
        dt1, _ = cpu_ce_step(W, 1, ref, O)
        return {"value": cores / dt, "unit": "samples/s", "cores": cores, "kind": kind, "cpu_model": cpu_model(),
                "value_1thread": 1.0 / dt1,
                "sample": f"{cores} CE samples (NormalStream + sample_into + restrict_to), one per thread ({dt:.1f} s)"}
    per_core = max(1, int(2e6 // (W["m"] + 1) ** 2))
    nsamp = cores * per_core
    dt, kind = cpu_reference_step(W, cores, nsamp, 0, port, ref)
    dt1, _ = cpu_reference_step(W, 1, per_core, nsamp, port, ref)
    return {"value": nsamp / dt, "unit": "samples/s", "cores": cores, "kind": kind, "cpu_model": cpu_model(),
            "value_1thread": per_core / dt1,
            "sample": f"{nsamp} samples of the same workload over {cores} host threads ({dt:.1f} s); "
                      f"{per_core} on 1 thread ({dt1:.1f} s)"}


def run_reference(args, W):
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    port = O.Port()
    ref = O.Ref()
    per_step = cores * max(1, int(2e6 // (W["m"] + 1) ** 2))  # bounded sample per step
    times, kind = [], "port"
    t_budget = time.time() + 240.0
    if W.get("ce_only"):
        per_step = cores
        for k in range(args.steps):
            dt, kind = cpu_ce_step(W, cores, ref, O)
            times.append(dt)
            if time.time() > t_budget:
                break
    else:
        for w in range(min(args.warmup, 1)):
            cpu_reference_step(W, cores, min(per_step, cores), 10_000_000 + w, port, ref)
        for k in range(args.steps):
            dt, kind = cpu_reference_step(W, cores, per_step, k * per_step, port, ref)
            times.append(dt)
            if time.time() > t_budget:
                break
    total = sum(times)
    value = per_step * len(times) / total
    line = {
        "impl": "reference", "metric": "MLMC samples/s per level (CE field + Darcy solve, fp64)",
        "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": len(times),
        "warmup": min(args.warmup, 1), "ms_per_step": 1000 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (NormalStream seed 1)",
        "config": {"workload": W["name"], "global_batch": per_step, "parallelism": f"{cores} host threads",
                   "steps_note": f"{len(times)} of {args.steps} steps within the 240 s CPU budget"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"{per_step} coupled samples per step x {len(times)} steps"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm -----------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="4")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--coarse-op", default="galerkin", choices=["galerkin", "rediscretize"],
                    help="MG coarse operators: exact Galerkin (default) or the reference's rediscretisation")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mlmc", action="store_true",
                    help="config 3/5: full adaptive MLMC(-CES) estimate over the GPU seam (wall time)")
    ap.add_argument("--setup", default="device", choices=["reference", "host", "device"],
                    help="--mlmc: who builds the levels' spectra (estimators.set_setup)")
    ap.add_argument("--eps", type=float, default=1e-3)
    ap.add_argument("--lam", type=float, default=0.01)
    args = ap.parse_args()
    W = workload(args.config)
    if args.batch:
        W["batch"] = args.batch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, W)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2306_13493_b200 import api
    ctx = api.Context(local)
    if args.mlmc:
        return run_mlmc(args, api, ctx, torch, rank)
    if W.get("ce_only"):
        return run_ce_only(args, W, api, ctx, torch, dist, rank, world, local)
    m, B = W["m"], W["batch"]
    model = (api.CovarianceModel.matern(W["sigma2"], W["lam"], W["nu"]) if W["family"] == "matern"
             else api.CovarianceModel.separable_exponential(W["sigma2"], W["lam"]))
    problem = api.ProblemSpec(model, api.QoiSpec(api.QoiKind(W["qoi"])), bc=api.BC(W["bc"]))
    opt = api.EstimatorOptions(seed=1, solver=api.SolverOptions(
        coarse_operator=api.CoarseOperator[args.coarse_op.capitalize()]))
    t_setup = time.perf_counter()
    plan = api.make_level_plan(W["ell"], 1.0 / (m >> W["ell"]), problem, opt)
    t_setup = time.perf_counter() - t_setup
    # the same level setup on the device (osc_build_spectrum_device), timed and checked once
    try:
        torch.cuda.synchronize()
        t_dev = time.perf_counter()
        op_dev = api.build_operator(plan.grid, model, device=True, ctx=ctx)
        t_dev = time.perf_counter() - t_dev
        e_h, e_d = plan.op.eigenvalues, op_dev.eigenvalues
        setup_dev = {"s": round(t_dev, 4), "host_s": round(t_setup, 4),
                     "max_rel_eig_diff": float(np.max(np.abs(e_d - e_h)) / np.max(np.abs(e_h)))}
        del op_dev, e_d
    except api.ConfigError as e:
        setup_dev = {"unsupported": str(e)}
    lev = plan.op.device_level(ctx, 0)
    coarse = api.GridSpec.square(m // 2) if W["coupled"] else None
    stream = torch.cuda.ExternalStream(ctx.stream)
    import ctypes as C
    from paper_2306_13493_b200 import _lib as L
    lib = L.lib()
    ps = api._problem_struct(problem, opt.solver)
    flags = L.DRAW_HAS_COARSE if W["coupled"] else 0
    qf, qc = np.empty(B), np.empty(B)
    itf, itc, st = (np.zeros(B, dtype=np.int32) for _ in range(3))
    sums = np.zeros(8)
    iters_total = [0, 0]

    # the level's running sums stay in HBM (osc_level_sums_reset); under torchrun each batch's one
    # collective is an NCCL all-reduce of those 5 device doubles through the C-ABI's osc_comm
    lev.sums_reset(0.0, 0.0)
    comm = None
    if dist:
        obj = [api.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = api.Comm(ctx, world, rank, obj[0])

    def step(k, xi=None, xi_next=None):
        frm = (k * world + rank) * B
        if xi_next is not None:  # cross-call prefetch: the next step's rows copy under this step
            api._check(lib.osc_level_prefetch_xi(lev.h, xi_next.ctypes.data_as(C.c_void_p), B))
        code = lib.osc_level_draws(lev.h, C.byref(ps), opt.seed, W["ell"], frm, frm + B, flags,
                                   None if xi is None else xi.ctypes.data_as(C.c_void_p),
                                   qf.ctypes.data, qc.ctypes.data, itf.ctypes.data, itc.ctypes.data,
                                   st.ctypes.data, sums.ctypes.data)
        api._check(code, status=st)
        if comm is not None:  # the batch's one collective: NCCL all-reduce of the device level sums
            comm.allreduce_level_sums(lev)
        iters_total[0] += int(itf.sum())
        iters_total[1] += int(itc.sum())

    # W warm-up steps, continued until at least 0.4 s have been spent warming up: an idle B200 sits at
    # 120 MHz and the few-ms steps of the small configs would otherwise be timed on ramping clocks
    # (config 1 measured 94k or 140k samples/s depending on it)
    # the clock sampler starts before the warm-up: nvidia-smi's NVML start-up (hundreds of ms) then
    # overlaps the warm-up instead of leaving the GPU idle (and down-clocking) right before the timed region
    clocks = ClockSampler(local, 200 if m >= 1024 else 1000)
    clocks.start()
    t_warm = time.perf_counter()
    w = 0
    while w < args.warmup - 1 or (time.perf_counter() - t_warm < 0.4 and w < 500):
        step(1_000_000 + w)
        w += 1
    warm_extra = max(0, w - (args.warmup - 1))
    # the last warm-up step is profiled (every kernel class, untimed): per-class times for the
    # kernel table and the choice of the dominant kernel; in the timed region only the dominant
    # kernel's launches carry CUDA events, so the step time is not perturbed by profiling
    ctx.set_profiling(True)
    ctx.reset_stats()
    iters_total[:] = [0, 0]
    step(1_000_000 + args.warmup)
    ctx.synchronize()
    kstats_w = ctx.kernel_stats()
    iters_w = list(iters_total)
    # the roofline kernel: the most expensive class with an algorithmic-bytes model (the
    # shared-memory-resident V-cycle tail of small grids has none)
    def _modelled(name):
        b_, _, g_ = name.partition("@")
        return bool(g_) and kernel_nodes(b_, int(g_)) is not None
    ranked = sorted(kstats_w.items(), key=lambda kv: -kv[1][1])
    dom_name = next((n for n, _ in ranked if _modelled(n)), ranked[0][0])
    # Grids up to 128² iterate inside a CUDA graph (device-side loop), which carries no per-kernel
    # events: there the timed region runs unprofiled and the roofline kernel is timed by CUDA events
    # in an eager pass of the same K steps right after it. Larger grids (config 4) keep the events
    # of the dominant kernel inside the timed region (host-polled loop).
    graph_loop = m <= 128
    if graph_loop:
        ctx.set_profiling(False)
    else:
        ctx.profile_only(dom_name)
    # timed region
    ctx.reset_stats()
    iters_total[:] = [0, 0]
    launches0 = ctx.launch_count
    if not clocks.rows:  # (long steps: the sampler had the whole warm-up; short ones: keep the GPU busy meanwhile)
        t_w = time.perf_counter()
        while not clocks.rows and clocks.proc and clocks.proc.poll() is None and time.perf_counter() - t_w < 10.0:
            step(2_000_000)
    if graph_loop:
        step(2_000_001)  # back-to-back into the timed region
    ctx.reset_stats()
    iters_total[:] = [0, 0]
    launches0 = ctx.launch_count
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    clocks.mark()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        step(k)
    e1.record(stream)
    ctx.synchronize()
    torch.cuda.synchronize()
    ck = clocks.stop()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    gpu_launches = ctx.launch_count - launches0
    iters_graph = list(iters_total)
    if graph_loop:  # the roofline kernel's events: an eager pass of the same K steps
        ctx.set_profiling(True)
        ctx.profile_only(dom_name)
        ctx.reset_stats()
        iters_total[:] = [0, 0]
        for k in range(args.steps):
            step(k)
        ctx.synchronize()
    kstats = ctx.kernel_stats()  # launch counts of every class; event times of dom_name only
    ctx.profile_only(None)
    ctx.set_profiling(False)
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    samples = args.steps * B * world
    value = samples / (ms / 1000.0)
    iters_timed = list(iters_graph)

    # roofline of the dominant kernel: compulsory bytes / its CUDA-event time on the ctx stream,
    # both over the timed region
    hbm, hbm_kind = peaks()
    dom_launches, dom_ms = kstats[dom_name]
    base, _, grid_tag = dom_name.partition("@")
    roof = {"kernel": dom_name, "bound": "hbm", "achieved": None, "peak": hbm, "unit": "GB/s",
            "frac": None, "traffic": None, "peak_kind": hbm_kind,
            "timing": ("CUDA events in an eager pass of the same K steps after the timed region (the timed "
                       "region runs the device-side CUDA-graph PCG loop)") if graph_loop else
                      "CUDA events around the kernel's launches inside the timed region"}
    kn = kernel_nodes(base, int(grid_tag)) if grid_tag else None
    if kn:
        mg = int(grid_tag)
        sample_iters = iters_total[0] if mg == m else iters_total[1]
        per_node, nodes = kn
        alg_bytes = per_node * nodes * sample_iters
        achieved = alg_bytes / (dom_ms / 1000.0) / 1e9
        roof.update(achieved=achieved, frac=achieved / hbm, alg_bytes_total=alg_bytes,
                    launches=dom_launches, avg_launch_ms=dom_ms / max(dom_launches, 1),
                    alg_bytes_per_launch=alg_bytes / max(dom_launches, 1),
                    bytes_per_node=per_node, nodes_per_sample_launch=nodes, sample_launches=sample_iters)
        # measured DRAM traffic of the same kernel (ncu --set full, profiles/ncu_traffic.json),
        # scaled to this run's node-launches like `achieved`
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                tr = json.load(f).get(base)
            if tr:
                roof["traffic"] = tr["dram_bytes_per_node"] * nodes * sample_iters / max(dom_launches, 1)
                roof["traffic_source"] = tr["source"]
                roof["traffic_over_algorithmic"] = tr["dram_bytes_per_node"] / per_node
        except (OSError, ValueError, KeyError):
            pass
    # every classified kernel's achieved bandwidth (same accounting), for DESIGN.md
    per_kernel = {}
    for name, (nl, tms) in kstats_w.items():  # the profiled warm-up step
        b_, _, g_ = name.partition("@")
        kn_ = kernel_nodes(b_, int(g_)) if g_ else None
        if kn_ and tms > 0:
            it_ = iters_w[0] if int(g_) == m else iters_w[1]
            per_kernel[name] = round(kn_[0] * kn_[1] * it_ / (tms / 1000.0) / 1e9, 1)
    n = lev.n
    b_sample = algorithmic_bytes_per_sample(W, n)
    pipeline = {"basis": "SURVEY 8(d) B per coupled sample", "bytes_per_sample": b_sample,
                "basis_iters": list(W["it"]),
                "roofline_samples_per_s_per_gpu": hbm * 1e9 / b_sample,
                "frac": value / world / (hbm * 1e9 / b_sample)}
    # the same byte model at this run's measured mean iteration counts (the basis fixes the
    # flow-cell counts of the reference algorithm; the preconditioner changes the count)
    it_meas = (iters_timed[0] / (args.steps * B), iters_timed[1] / (args.steps * B) if W["coupled"] else 0)
    b_meas = algorithmic_bytes_per_sample(W, n, it_meas)
    pipeline["measured_iters"] = [round(x, 2) for x in it_meas]
    pipeline["frac_at_measured_iters"] = value / world / (hbm * 1e9 / b_meas)

    # e2e: same metric through the C-ABI with HOST ξ (pinned), H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        s = lev.s
        pool = min(B, 8)
        try:
            buf = api.PinnedBuffer((B, s))
            pinned = True
        except MemoryError:  # e.g. 8 ranks × 8.6 GB on a small host: pageable staging instead
            buf = type("Pageable", (), {})()
            buf.array = np.empty((B, s))
            buf.free = lambda: None
            pinned = False
        # ξ rows for the step from the device Philox stream of a pool of indices (outside timing)
        tmp = np.empty((pool, s))
        lib.osc_normals(ctx.h, opt.seed, W["ell"], 0, pool, s, tmp.ctypes.data)
        for b in range(B):
            buf.array[b] = tmp[b % pool]
        del tmp
        k_e2e = max(1, args.steps)  # the same K as the device-timed region
        # warm the host-ξ paths (chunked + prefetch, then the prefetched whole batch); the first
        # timed step then copies its own rows (chunked), and step k copies step k+1's rows under
        # its solves (osc_level_prefetch_xi), so all k_e2e steps' H2D copies lie inside the region
        step(2_000_000, xi=buf.array, xi_next=buf.array)
        step(2_000_001, xi=buf.array)
        if dist:
            dist.barrier()
        ctx.synchronize()
        t0 = time.perf_counter()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for k in range(k_e2e):
            step(3_000_000 + k, xi=buf.array, xi_next=buf.array if k + 1 < k_e2e else None)
        f1.record(stream)
        ctx.synchronize()
        ems = f0.elapsed_time(f1)
        if dist:
            t = torch.tensor([ems], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        # the link bound: one plain H2D copy of the same pinned ξ (outside the timed region)
        nb = min(B, 16)
        dev = torch.empty((nb, s), dtype=torch.float64, device=f"cuda:{local}")
        src = torch.from_numpy(buf.array[:nb])
        dev.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record()
        dev.copy_(src, non_blocking=True)
        h1.record()
        torch.cuda.synchronize()
        h2d_gbs = 8.0 * s * nb / (h0.elapsed_time(h1) / 1000.0) / 1e9
        del dev, src
        e2e = {"value": k_e2e * B * world / (ems / 1000.0), "unit": "samples/s",
               "h2d_bytes_per_step": 8 * s * B, "d2h_bytes_per_step": 8 * 2 * B + 4 * 3 * B + 40,
               "xi": f"host {'pinned' if pinned else 'pageable'}, {pool} distinct Philox rows cycled over the batch",
               "steps": k_e2e, "h2d_gbs": h2d_gbs,
               "link_bound_samples_per_s": world * h2d_gbs * 1e9 / (8.0 * s),
               "note": "ξ (8 B per embedding entry per sample) crosses PCIe every step. Step 1 copies its own "
                       "rows in chunks (chunk i+1 under chunk i's solves); step k copies step k+1's rows under "
                       "its solves (osc_level_prefetch_xi), so e2e ≈ min(device rate, link rate)"}
        buf.free()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_block(W, 60.0)

    if rank == 0:
        line = {
            "metric": "MLMC samples/s per level (CE field + Darcy solve, fp64)",
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "warmup_extra_steps": warm_extra, "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: xi = NormalStream(seed 1, l, i) on device (Philox4x32-10 + Box-Muller)",
            "config": {"workload": W["name"], "global_batch": B * world, "per_gpu_batch": B,
                       "grid": f"{m}^2/{m // 2}^2" if W["coupled"] else f"{m}^2", "embedding_n": n,
                       "parallelism": f"dp{world} (contiguous sample shards)",
                       "l2": "inputs larger than L2 (>= 40 GB touched per step)" if m >= 1024 else
                       "per-step working set exceeds L2 (batch)",
                       "setup_s": round(t_setup, 2), "setup_device": setup_dev, "coarse_op": args.coarse_op,
                       "mean_iters_fine": iters_timed[0] / (args.steps * B),
                       "mean_iters_coarse": iters_timed[1] / (args.steps * B) if W["coupled"] else None},
            "roofline": roof, "kernel_gbs": per_kernel, "pipeline_roofline": pipeline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": gpu_launches, "clocks": ck,
            "kernels_ms_profiled_step": {k: round(v[1], 3) for k, v in
                                         sorted(kstats_w.items(), key=lambda kv: -kv[1][1])},
        }
        if args.config == "3" and world == 1:
            line["per_level"] = cfg3_per_level(args, api, ctx, torch, lib, hbm)
            line["per_level"]["4"] = {"grid": f"{m}^2/{m // 2}^2", "samples_per_s": value,
                                      "batch": B, "roofline_frac_at_measured_iters": pipeline["frac_at_measured_iters"]}
        print(json.dumps(line), flush=True)
    if dist:
        if comm is not None:
            comm.close()
        dist.destroy_process_group()


def cfg3_per_level(args, api, ctx, torch, lib, hbm):
    """Config 3's levels ℓ = 0..3 (16²…128² fine grids; ℓ ≤ 2 smoothed with k = s/2 as the reference's
    Adaptive + lstar_only rule gives for the separable exponential): samples/s per level, each level
    timed over `args.steps` batches with CUDA events on the context stream (ℓ = 4 is the main line)."""
    import ctypes as C
    from paper_2306_13493_b200 import _lib as L
    model = api.CovarianceModel.separable_exponential(1.0, 0.01)
    problem = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
    opt = api.EstimatorOptions(seed=1)
    ps = api._problem_struct(problem, opt.solver)
    out = {}
    stream = torch.cuda.ExternalStream(ctx.stream)
    for ell, B in [(0, 16384), (1, 8192), (2, 4096), (3, 2048)]:
        m = 16 << ell
        op = api.build_operator(api.GridSpec.square(m), model)
        k = op.s // 2 if ell <= 2 else 0
        plan = api.make_level_plan(ell, 1.0 / 16, problem, opt, operator=op, k_trunc=k)
        lev = plan.op.device_level(ctx, k)
        flags = (L.DRAW_HAS_COARSE if ell > 0 else 0) | (L.DRAW_TRUNC_FINE | L.DRAW_TRUNC_COARSE if k else 0)
        qf, qc = np.empty(B), np.empty(B)
        itf, itc, st = (np.zeros(B, dtype=np.int32) for _ in range(3))

        failed = []

        def step(kk):
            frm = kk * B
            code = lib.osc_level_draws(lev.h, C.byref(ps), 1, ell, frm, frm + B, flags, None, qf.ctypes.data,
                                       qc.ctypes.data, itf.ctypes.data, itc.ctypes.data, st.ctypes.data, None)
            if code == L.OSC_ERR_SOLVER:  # recorded in the line (the reference would raise SolverError)
                failed.extend(int(frm + i) for i in np.nonzero(st)[0][:8])
            elif code:
                api._check(code, status=st)
        t_warm, w = time.perf_counter(), 0
        while w < args.warmup or (time.perf_counter() - t_warm < 0.2 and w < 500):
            step(1_000_000 + w)
            w += 1
        ctx.synchronize()
        # a batch of the small levels takes 4–40 ms: at least 0.25 s of batches (and at least args.steps),
        # so that one host hiccup does not move the level's rate by a third
        n_steps = max(args.steps, min(200, int(0.25 * w / max(time.perf_counter() - t_warm, 1e-3)) + 1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = [0, 0]
        e0.record(stream)
        for kk in range(n_steps):
            step(kk)
            its[0] += int(itf.sum())
            its[1] += int(itc.sum())
        e1.record(stream)
        ctx.synchronize()
        ms = e0.elapsed_time(e1)
        rate = n_steps * B / (ms / 1000.0)
        Wl = dict(m=m, batch=B, coupled=ell > 0, it=(its[0] / (n_steps * B), its[1] / (n_steps * B)))
        b_meas = algorithmic_bytes_per_sample(Wl, plan.op.n)
        out[str(ell)] = {"grid": f"{m}^2" + (f"/{m // 2}^2" if ell else ""), "samples_per_s": rate, "batch": B,
                         "batches_timed": n_steps,
                         "smoothed": bool(k), "mean_iters": [round(x, 2) for x in Wl["it"]],
                         "roofline_frac_at_measured_iters": rate / (hbm * 1e9 / b_meas),
                         "non_converged_sample_indices": failed}
        plan.op._levels.clear()
    return out


def run_mlmc(args, api, ctx, torch, rank):
    """Configs 3 / 5: the reference's OWN adaptive MLMC(-CES) estimator (estimate_adaptive,
    estimators.cpp:289-378, compiled from the pristine sources with run_level_samples routed to the GPU
    seam — paper_2306_13493_b200.estimators) with every sample drawn through osc_level_draws.
    Exponential (separable, p = 1) covariance σ² = 1, flow-cell BCs, outflow-flux QoI, h0 = 1/16,
    smoothing Adaptive on the levels coarser than the resolution bound (smoothing_lstar_only), N_ℓ by
    the standard rule at RMSE eps."""
    from paper_2306_13493_b200 import estimators as E
    model = api.CovarianceModel.separable_exponential(1.0, args.lam)
    problem = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
    opt = api.EstimatorOptions(seed=1, smoothing=api.SmoothingRule.Adaptive, smoothing_lstar_only=True,
                               l_max=4)
    # build_operator of the reference's make_level_plan routed to the GPU level setup (the reference's
    # own single-threaded host setup otherwise takes a third of this run's wall time)
    E.set_setup({"reference": E.SETUP_REFERENCE, "host": E.SETUP_HOST, "device": E.SETUP_DEVICE}[args.setup])
    # a first (cold) run loads the kernels and allocates each level's workspaces; the second run,
    # identical (same seed, so the same samples), is the timed one
    t0 = time.perf_counter()
    E.mlmc_estimate(problem, opt, 1.0 / 16, args.eps, initial_levels=5)
    torch.cuda.synchronize()
    cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    rep = E.mlmc_estimate(problem, opt, 1.0 / 16, args.eps, initial_levels=5)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    total = sum(l.n for l in rep.levels)
    # the GPU-resident driver (osc_mlmc_adaptive, csrc/driver.cpp): the same estimator with the levels
    # of each allocation pass drawn at the same time, device level setup, moments as device sums;
    # first run cold, then timed; the serial variant (one level after the other) isolates the overlap
    from paper_2306_13493_b200 import mlmc as M
    drv = {}
    for name, conc in (("concurrent", True), ("serial", False)):
        M.mlmc_adaptive(problem, opt, 1.0 / 16, args.eps, 5, concurrent=conc)
        t0 = time.perf_counter()
        r = M.mlmc_adaptive(problem, opt, 1.0 / 16, args.eps, 5, concurrent=conc)
        torch.cuda.synchronize()
        w = time.perf_counter() - t0
        drv[name] = {"wall_s": w, "samples_per_s": sum(l.n for l in r.levels) / w, "setup_s": r.setup_s,
                     "draw_s": r.draw_s, "waves": r.waves, "passes": r.passes, "n": [l.n for l in r.levels],
                     "estimate": r.estimate, "sampling_error": r.sampling_error, "bias": r.bias_estimate,
                     "converged": r.converged, "gpu_launches": r.gpu_launches,
                     "same_n_as_reference_loop": [l.n for l in r.levels] == [l.n for l in rep.levels]}
    if rank == 0:
        print(json.dumps({
            "metric": "MLMC wall time and total samples/s (config 3/5, full adaptive run)",
            "driver_resident": drv,
            "value": total / wall, "unit": "samples/s", "wall_s": wall, "cold_wall_s": cold, "n_gpus": 1,
            "estimate": rep.estimate, "sampling_error": rep.sampling_error, "bias": rep.bias_estimate,
            "converged": rep.converged, "message": rep.message,
            "levels": [{"h": h, "n": l.n, "mean_y": l.mean_y, "var_y": l.var_y,
                        "wall_per_sample_s": l.cost_wall_per_sample} for h, l in zip(rep.level_h, rep.levels)],
            "config": {"workload": f"MLMC-CES sep-exp s2=1 lam={args.lam}, h0=1/16, 5 levels, flux QoI, eps={args.eps}",
                       "driver": "the reference's estimate_adaptive (C++) over the GPU seam",
                       "level_setup": args.setup},
            "dtype": "f64", "data": "synthetic: NormalStream(1, l, i)",
        }), flush=True)


def run_ce_only(args, W, api, ctx, torch, dist, rank, world, local):
    """Config 2: batched CE field sampling (K1 + K2), fields left in HBM for `value`."""
    import ctypes as C
    from paper_2306_13493_b200 import _lib as L
    lib = L.lib()
    m, B = W["m"], W["batch"]
    model = api.CovarianceModel.matern(W["sigma2"], W["lam"], W["nu"])
    t_setup = time.perf_counter()
    op = api.build_operator(api.GridSpec.square(m), model)
    t_setup = time.perf_counter() - t_setup
    lev = op.device_level(ctx, 0)
    Nf = (m + 1) ** 2
    out = torch.empty((B, Nf), dtype=torch.float64, device=f"cuda:{local}")
    stream = torch.cuda.ExternalStream(ctx.stream)
    flags = L.CE_FINE | L.CE_DEVICE_OUT

    def step(k):
        idx0 = (k * world + rank) * B
        api._check(lib.osc_ce_sample(lev.h, None, 1, W["ell"], idx0, B, flags, out.data_ptr(), None))

    clocks = ClockSampler(local)
    clocks.start()
    t_w, w = time.perf_counter(), 0
    while w < args.warmup or (not clocks.rows and clocks.proc and clocks.proc.poll() is None and time.perf_counter() - t_w < 10.0):
        step(1_000_000 + w)  # the sampler's NVML start-up overlaps the warm-up (the GPU never idles before the timed region)
        w += 1
    ctx.set_profiling(True)
    ctx.reset_stats()
    launches0 = ctx.launch_count
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    clocks.mark()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        step(k)
    e1.record(stream)
    ctx.synchronize()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1)
    kstats = ctx.kernel_stats()
    ctx.set_profiling(False)
    gpu_launches = ctx.launch_count - launches0
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = args.steps * B * world / (ms / 1000.0)
    hbm, hbm_kind = peaks()
    n = lev.n
    P = m + 1
    # compulsory bytes per sample: rows write the half-spectrum intermediate (16 n P) and read
    # √λ once per CTA sample-loop (≈ 8 s / samples per CTA, ignored); cols read it and write 8 Nf.
    per = {"ce_rows": 16 * n * P, "ce_cols": 16 * n * P + 8 * Nf}
    dom, (dl, dms) = max(kstats.items(), key=lambda kv: kv[1][1])
    ach = per[dom] * args.steps * B / (dms / 1000.0) / 1e9 if dom in per else None
    roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
            "frac": ach / hbm if ach else None, "traffic": None, "peak_kind": hbm_kind,
            "note": "algorithmic bytes count the half-spectrum round trip (1 GiB chunks: it spills to HBM); both "
                    "passes are bound by the SM's L1/shared-memory data pipe (71-76% busy: the radix-8 exchanges "
                    "through shared memory plus the scattered 8/16-byte stores), profiles/r2e_ce_stalls_staged_twiddles.txt"}
    # fp64 view: conventional FFT flops 5·n·log2(n) per length-n complex transform, n/2 row and P column
    # transforms per sample (Box-Muller log/sqrt/sincos and the exp() are not counted), against the
    # measured DFMA peak (profiles/r1_fp64_peak.json, scripts/micro/fp64bench.cu)
    fft_flops = (n // 2 + P) * 5.0 * n * math.log2(n)
    fp64_peak = 34.22
    compute_roof = {"bound": "fp64", "fft_flops_per_sample": fft_flops,
                    "achieved": fft_flops * value / world / 1e12, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": fft_flops * value / world / 1e12 / fp64_peak,
                    "peak_source": "profiles/r1_fp64_peak.json (DFMA chains, 148 SMs, 1965 MHz)",
                    "ncu": "profiles/r2e_ce_stalls_staged_twiddles.txt: fp64 pipe 49% (rows) busy, issue 62% / 36%"}
    b_sample = algorithmic_bytes_per_sample(dict(W, coupled=False, it=(0, 0)), n) - 8 * Nf * 0
    b_sample = 8 * n * n / B + 32 * n * (n // 2 + 1) + 8 * Nf  # SURVEY §8(d) B_ce, device ξ
    pipeline = {"basis": "SURVEY 8(d) B_ce (device xi)", "bytes_per_sample": b_sample,
                "roofline_samples_per_s_per_gpu": hbm * 1e9 / b_sample,
                "frac": value / world / (hbm * 1e9 / b_sample)}
    # The same pass on ξ resident in HBM (the parity mode of north_star: identical seeded Gaussian
    # vectors fed to both implementations): a ring of 64 distinct rows (2.1 GB at n = 2048, far above
    # L2), 64-sample calls; bytes per sample add the 8 s of ξ read
    xi_res = None
    if world == 1:
        R = 64
        g = torch.Generator(device=f"cuda:{local}")
        g.manual_seed(1)
        ring = torch.randn((R, lev.s), dtype=torch.float64, device=f"cuda:{local}", generator=g)
        fl = flags | L.CE_XI_DEVICE

        def xi_step():
            for c0 in range(0, B, R):
                api._check(lib.osc_ce_sample(lev.h, ring.data_ptr(), 1, W["ell"], 0, min(R, B - c0), fl,
                                             out[c0:].data_ptr(), None))
        xi_step()
        ctx.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        xi_step()
        g1.record(stream)
        ctx.synchronize()
        xms = g0.elapsed_time(g1)
        bx = 8 * n * n + 32 * n * (n // 2 + 1) + 8 * Nf
        xi_res = {"value": B / (xms / 1000.0), "unit": "samples/s", "bytes_per_sample": bx,
                  "roofline_samples_per_s": hbm * 1e9 / bx, "frac": B / (xms / 1000.0) / (hbm * 1e9 / bx),
                  "xi": "ring of 64 rows of torch.randn (seed 1) in HBM, 64-sample calls"}
        del ring
    # e2e: host ξ in (pinned pool), fields out to pinned host memory, 64-sample calls
    e2e = None
    if not args.no_e2e:
        cb = 64
        s_ = lev.s
        pool = api.PinnedBuffer((cb, s_))
        tmp = np.empty((8, s_))
        lib.osc_normals(ctx.h, 1, W["ell"], 0, 8, s_, tmp.ctypes.data)
        for bb in range(cb):
            pool.array[bb] = tmp[bb % 8]
        del tmp
        host_out = api.PinnedBuffer((cb, Nf))
        nsteps = 1
        calls = B // cb

        def e2e_step():
            for _ in range(calls):
                api._check(lib.osc_ce_sample(lev.h, pool.array.ctypes.data, 1, W["ell"], 0, cb, L.CE_FINE,
                                             host_out.array.ctypes.data, None))
        e2e_step()
        ctx.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(nsteps):
            e2e_step()
        f1.record(stream)
        ctx.synchronize()
        ems = f0.elapsed_time(f1)
        e2e = {"value": nsteps * B * world / (ems / 1000.0), "unit": "samples/s",
               "h2d_bytes_per_step": 8 * s_ * B, "d2h_bytes_per_step": 8 * Nf * B,
               "xi": "host pinned pool of 64 rows (8 distinct Philox rows), 64-sample calls", "steps": nsteps}
        pool.free()
        host_out.free()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_block(W, 60.0)
    if rank == 0:
        print(json.dumps({
            "metric": "CE field samples/s (config 2, sampling only, fp64)", "value": value,
            "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic: device Philox NormalStream(1, 0, i)",
            "config": {"workload": W["name"], "global_batch": B * world, "embedding_n": n,
                       "l2": "fields written (34 GB/step) exceed L2", "setup_s": round(t_setup, 2)},
            "roofline": roof, "compute_roofline": compute_roof, "pipeline_roofline": pipeline,
            "resident_xi": xi_res, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": gpu_launches, "clocks": ck,
            "kernels_ms": {k: round(v[1], 3) for k, v in sorted(kstats.items(), key=lambda kv: -kv[1][1])},
        }), flush=True)
    if dist:
        dist.destroy_process_group()


def cpu_ce_step(W, threads, ref, O):
    """CPU CE baseline: the pristine reference (NormalStream + sample_into + restrict_to), one sample
    per thread."""
    import threading as th
    m = W["m"]
    key = ("ceop", m)
    if key not in _CACHE:
        _CACHE[key] = ref.build_operator(m, O.MATERN, W["sigma2"], W["lam"], W["nu"])
    rop = _CACHE[key]

    def one(i):
        u = rop.sample(ref.normals(1, 0, i, rop.s))
        rop.restrict(u, m)
    ts = [th.Thread(target=one, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return time.perf_counter() - t0, "reference"


if __name__ == "__main__":
    main()
