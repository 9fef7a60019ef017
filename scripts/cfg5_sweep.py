"""BASELINE config 5: MLMC cost sweep on one B200 — RMSE ε × λ ∈ {0.03, 0.01}, exponential (separable,
p = 1) covariance σ² = 1, flow-cell BCs, outflow-flux QoI. Smoothed CE (MLMC-CES: h0 = 1/16, adaptive
k_ℓ on the levels coarser than the resolution bound) versus standard CE (no smoothing, coarsest mesh
forced to resolve λ: h0 = coarsest_level_bound(λ) = 1/64 resp. 1/128). Every sample goes through
osc_level_draws; wall time on the GPU + host driver (api.mlmc_estimate)."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_13493_b200 as P  # noqa: E402

api = P.api
ctx = api.default_context(0)
eps_list = [float(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1e-2", "3e-3", "1e-3"])]
rows = []
for lam in (0.03, 0.01):
    model = api.CovarianceModel.separable_exponential(1.0, lam)
    problem = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
    h_std = api.coarsest_level_bound(model)
    for eps in eps_list:
        for variant in ("MLMC-CES", "MLMC"):
            h0 = 1.0 / 16 if variant == "MLMC-CES" else h_std
            l_max = int(round(math.log2(2048 * h0)))  # finest grid at most 2048² (n = 4096)
            if variant == "MLMC-CES":
                opt = api.EstimatorOptions(seed=1, smoothing=api.SmoothingRule.Adaptive,
                                           smoothing_lstar_only=True, l_max=l_max)
            else:
                opt = api.EstimatorOptions(seed=1, l_max=l_max)
            t0 = time.perf_counter()
            rep = api.mlmc_estimate(problem, opt, h0, eps, ctx=ctx)
            ctx.synchronize()
            wall = time.perf_counter() - t0
            row = dict(lam=lam, eps=eps, variant=variant, h0=h0, wall_s=wall,
                       estimate=rep.estimate, sampling_error=rep.sampling_error, bias=rep.bias_estimate,
                       converged=rep.converged, levels=len(rep.levels),
                       n=[l.n for l in rep.levels], cost_model=rep.total_cost_model,
                       samples_per_s=sum(l.n for l in rep.levels) / wall)
            rows.append(row)
            print(json.dumps(row), flush=True)
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "cfg5_sweep.json")
json.dump(rows, open(out, "w"), indent=1)
