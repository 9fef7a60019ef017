"""BASELINE config 5: MLMC cost sweep on one B200 — RMSE ε ∈ {1e-2, 3e-3, 1e-3, 3e-4} × λ ∈ {0.03, 0.01},
exponential (separable, p = 1) covariance σ² = 1, flow-cell BCs, outflow-flux QoI (config 3's).
Smoothed CE (MLMC-CES: h0 = 1/16, adaptive k_ℓ on the levels coarser than the resolution bound)
versus standard CE (no smoothing, coarsest mesh forced to resolve λ: h0 = coarsest_level_bound(λ)).

Every run is the REFERENCE'S OWN estimate_adaptive (integration/_build/liboscfield_gpu.so) with its
draws routed to the GPU seam and — in the sweep — its build_operator routed to the GPU level setup
(estimators.set_setup: the reference's single-threaded setup takes ~10 s per estimate at n = 4096).
The finest grid is capped at 2048² (l_max); a row whose bias estimate is still above ε/√2 there
reports converged = false, as the reference does.

"CPU beside it" (part 2): the pristine reference on the host cores (oracle/_ref, all threads) and the
GPU-routed run with IDENTICAL options, on the rows the CPU finishes in minutes — finest grid capped
at 256², L2-norm QoI (the pristine reference has no flux QoI) — with N_ℓ compared level by level.

Each sweep row also runs the GPU-resident driver (osc_mlmc_adaptive, csrc/driver.cpp) on the same options.

usage: python scripts/cfg5_sweep.py [eps,eps,...] [--no-cpu] [--no-driver]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13493_b200 as P  # noqa: E402
from paper_2306_13493_b200 import estimators as E  # noqa: E402
from paper_2306_13493_b200 import mlmc as M  # noqa: E402

api = P.api
ctx = api.default_context(0)
args = [a for a in sys.argv[1:] if not a.startswith("--")]
eps_list = [float(x) for x in (args[0].split(",") if args else ["1e-2", "3e-3", "1e-3", "3e-4"])]
with_cpu = "--no-cpu" not in sys.argv
with_driver = "--no-driver" not in sys.argv
rows, beside = [], []


def options(variant, l_max):
    if variant == "MLMC-CES":
        return api.EstimatorOptions(seed=1, smoothing=api.SmoothingRule.Adaptive, smoothing_lstar_only=True,
                                    l_max=l_max)
    return api.EstimatorOptions(seed=1, l_max=l_max)


setup = "--reference-setup" not in sys.argv
E.set_setup(E.SETUP_DEVICE if setup else E.SETUP_REFERENCE)
for lam in (0.03, 0.01):
    model = api.CovarianceModel.separable_exponential(1.0, lam)
    problem = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
    h_std = E.coarsest_level_bound(model)
    for eps in eps_list:
        for variant in ("MLMC-CES", "MLMC"):
            h0 = 1.0 / 16 if variant == "MLMC-CES" else h_std
            l_max = int(round(math.log2(2048 * h0)))  # finest grid at most 2048² (n = 4096)
            t0 = time.perf_counter()
            rep = E.mlmc_estimate(problem, options(variant, l_max), h0, eps)
            ctx.synchronize()
            wall = time.perf_counter() - t0
            # the GPU-resident driver (osc_mlmc_adaptive): levels of a pass drawn at the same time, levels
            # created on the device (no host sort of the n = 4096 spectrum), moments as device sums
            drv = None
            if with_driver:
                t0 = time.perf_counter()
                d = M.mlmc_adaptive(problem, options(variant, l_max), h0, eps)
                ctx.synchronize()
                dw = time.perf_counter() - t0
                drv = dict(wall_s=dw, setup_s=d.setup_s, draw_s=d.draw_s, waves=d.waves, n=[l.n for l in d.levels],
                           estimate=d.estimate, sampling_error=d.sampling_error, bias=d.bias_estimate,
                           converged=d.converged, same_n=[l.n for l in d.levels] == [l.n for l in rep.levels],
                           samples_per_s=sum(l.n for l in d.levels) / dw)
            row = dict(lam=lam, eps=eps, variant=variant, h0=h0, wall_s=wall, estimate=rep.estimate, driver=drv,
                       level_setup="device" if setup else "reference",
                       sampling_error=rep.sampling_error, bias=rep.bias_estimate, converged=rep.converged,
                       levels=len(rep.levels), n=[l.n for l in rep.levels], cost_model=rep.total_cost_model,
                       samples_per_s=sum(l.n for l in rep.levels) / wall, message=rep.message)
            rows.append(row)
            print(json.dumps(row), flush=True)

E.set_setup(E.SETUP_REFERENCE)  # the CPU comparison uses the reference's own setup on both sides
if with_cpu:
    from oracle import oracle as O
    if os.path.exists(O.REF_SO):
        ref = O.Ref()
        threads = os.cpu_count() or 1
        for lam in (0.03, 0.01):
            model = api.CovarianceModel.separable_exponential(1.0, lam)
            h_std = E.coarsest_level_bound(model)
            for eps in eps_list:
                for variant in ("MLMC-CES", "MLMC"):
                    h0 = 1.0 / 16 if variant == "MLMC-CES" else h_std
                    l_max = int(round(math.log2(256 * h0)))  # finest grid at most 256²
                    sm, lstar = (2, 1) if variant == "MLMC-CES" else (0, 0)
                    problem = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.L2Norm), bc=api.BC.FlowCell)
                    opt = options(variant, l_max)
                    t0 = time.perf_counter()
                    g = E.mlmc_estimate(problem, opt, h0, eps)
                    ctx.synchronize()
                    tg = time.perf_counter() - t0
                    o = O.RefOpts.make(family=O.SEP_EXP, sigma2=1.0, lam=lam, nu_or_p=1.0, seed=1,
                                       pilot_n=opt.pilot_n, threads=threads, l_max=l_max, smoothing=sm,
                                       lstar_only=lstar, qoi_kind=1)
                    t0 = time.perf_counter()
                    c = ref.mlmc(o, h0, eps, 1)
                    tc = time.perf_counter() - t0
                    cl = c.levels()
                    row = dict(lam=lam, eps=eps, variant=variant, h0=h0, l_max=l_max, qoi="L2 norm",
                               gpu_wall_s=tg, cpu_wall_s=tc, cpu_threads=threads, speedup=tc / tg,
                               n_gpu=[l.n for l in g.levels], n_cpu=[l["n"] for l in cl],
                               same_n=[l.n for l in g.levels] == [l["n"] for l in cl],
                               estimate_gpu=g.estimate, estimate_cpu=c.estimate,
                               converged=[bool(g.converged), bool(c.converged)])
                    beside.append(row)
                    print(json.dumps(row), flush=True)
    else:
        print(json.dumps({"cpu_beside": "oracle/_ref not built here"}), flush=True)

out = os.path.join(ROOT, "gpurun_out", "cfg5_sweep.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
json.dump({"sweep": rows, "cpu_beside": beside}, open(out, "w"), indent=1)
