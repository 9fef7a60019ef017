import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_13493_b200 as P
api = P.api
ctx = api.default_context(0)
model = api.CovarianceModel.separable_exponential(1.0, 0.01)
prob = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
opt = api.EstimatorOptions(seed=1)
for m, B in [(64, 4096), (128, 2048)]:
    plan = api.make_level_plan(1, 2.0 / m, prob, opt, k_trunc=0)
    cg = api.GridSpec.square(m // 2)
    for mode in ("host", "graph", "host", "graph"):
        if mode == "host":
            ctx.set_profiling(True); ctx.profile_only("no-such-class")
        else:
            ctx.profile_only(None); ctx.set_profiling(False)
        d = api.LevelDraws()
        ctx.synchronize()
        n0 = ctx.launch_count
        t0 = time.perf_counter()
        api.run_level_draws(plan, cg, False, False, prob, opt, 0, B, d, ctx=ctx)
        ctx.synchronize()
        dt = time.perf_counter() - t0
        print(m, mode, f"{dt*1e3:.2f} ms", "launches", ctx.launch_count - n0, "iters fine max", d.iters_fine[:B].max(),
              "mean", d.iters_fine[:B].mean(), "coarse max", d.iters_coarse[:B].max(), flush=True)
ctx.profile_only(None); ctx.set_profiling(False)
