"""Kernel-class time shares of config 3's small levels (one osc_level_draws batch per level, CUDA events
per kernel class): where a 16² … 64² level spends its time.
usage: python scripts/level_breakdown.py [ell,ell,...]"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_13493_b200 as P  # noqa: E402
from paper_2306_13493_b200 import _lib as L  # noqa: E402

api = P.api
ctx = api.default_context(0)
lib = L.lib()
model = api.CovarianceModel.separable_exponential(1.0, 0.01)
problem = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
opt = api.EstimatorOptions(seed=1)
ps = api._problem_struct(problem, opt.solver)
ells = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1, 2, 3]
for ell in ells:
    m, B = 16 << ell, 16384 >> ell
    op = api.build_operator(api.GridSpec.square(m), model)
    k = op.s // 2 if ell <= 2 else 0
    lev = op.device_level(ctx, k)
    flags = (L.DRAW_HAS_COARSE if ell > 0 else 0) | (L.DRAW_TRUNC_FINE | L.DRAW_TRUNC_COARSE if k else 0)
    qf, qc = np.empty(B), np.empty(B)

    def step(kk):
        api._check(lib.osc_level_draws(lev.h, C.byref(ps), 1, ell, kk * B, (kk + 1) * B, flags, None, qf.ctypes.data,
                                       qc.ctypes.data, None, None, None, None))
    for w in range(5):
        step(100 + w)
    ctx.synchronize()
    t0 = time.perf_counter()
    for kk in range(5):
        step(kk)
    ctx.synchronize()
    wall = (time.perf_counter() - t0) / 5
    ctx.set_profiling(True)
    ctx.reset_stats()
    step(7)
    ctx.synchronize()
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    tot = sum(v[1] for v in st.values())
    print(json.dumps({"ell": ell, "grid": m, "batch": B, "wall_ms_per_batch": wall * 1e3, "samples_per_s": B / wall,
                      "profiled_ms": tot,
                      "kernels": {k_: [v[0], round(v[1], 3)] for k_, v in sorted(st.items(), key=lambda x: -x[1][1])}}),
          flush=True)
    op._levels.clear()
