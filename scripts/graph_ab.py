"""A/B of the device-side CUDA-graph PCG loop against the host-polled loop (profiling on with an
empty class filter forces the host loop without recording events)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_13493_b200 as P  # noqa: E402

api = P.api
ctx = api.default_context(0)
model = api.CovarianceModel.separable_exponential(1.0, 0.01)
prob = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
opt = api.EstimatorOptions(seed=1)
for m, B, reps in [(64, 4096, 5), (128, 2048, 5), (256, 1024, 5), (512, 256, 3)]:
    plan = api.make_level_plan(1, 2.0 / m, prob, opt, k_trunc=0)
    cg = api.GridSpec.square(m // 2)
    res = {}
    for mode in ("host", "graph", "host", "graph"):
        if mode == "host":
            ctx.set_profiling(True)
            ctx.profile_only("no-such-class")
        else:
            ctx.profile_only(None)
            ctx.set_profiling(False)
        d = api.LevelDraws()
        api.run_level_draws(plan, cg, False, False, prob, opt, 0, B, d, ctx=ctx)  # warm
        ctx.synchronize()
        t0 = time.perf_counter()
        for r in range(reps):
            api.run_level_draws(plan, cg, False, False, prob, opt, r * B, (r + 1) * B, d, ctx=ctx)
        ctx.synchronize()
        res[mode] = reps * B / (time.perf_counter() - t0)
    ctx.profile_only(None)
    ctx.set_profiling(False)
    print(f"m={m} B={B}: host loop {res['host']:.0f} samples/s, graph loop {res['graph']:.0f} samples/s", flush=True)
