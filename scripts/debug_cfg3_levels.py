"""Config-3 levels 0..4 (sep-exp λ=0.01, flow-cell, flux QoI, k = s/2 on ℓ ≤ 2): draw a batch per
level with per-slot status; report failures and replay a failing sample against the oracle port."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_13493_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

api, L = P.api, P._lib
ctx = api.default_context(0)
model = api.CovarianceModel.separable_exponential(1.0, 0.01)
prob = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
opt = api.EstimatorOptions(seed=1)
ps = api._problem_struct(prob, opt.solver)
port = O.Port()
base = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for ell, B in [(0, 16384), (1, 8192), (2, 4096), (3, 2048), (4, 256)]:
    m = 16 << ell
    op = api.build_operator(api.GridSpec.square(m), model)
    k = op.s // 2 if ell <= 2 else 0
    plan = api.make_level_plan(ell, 1.0 / 16, prob, opt, operator=op, k_trunc=k)
    lev = plan.op.device_level(ctx, k)
    flags = (L.DRAW_HAS_COARSE if ell > 0 else 0) | (L.DRAW_TRUNC_FINE | L.DRAW_TRUNC_COARSE if k else 0)
    qf, qc = np.empty(B), np.empty(B)
    itf, itc, st = (np.zeros(B, dtype=np.int32) for _ in range(3))
    frm = base * B
    rc = L.lib().osc_level_draws(lev.h, C.byref(ps), 1, ell, frm, frm + B, flags, None, qf.ctypes.data, qc.ctypes.data,
                                 itf.ctypes.data, itc.ctypes.data, st.ctypes.data, None)
    bad = np.nonzero(st)[0]
    print(f"ell={ell} m={m} rc={rc} failures={bad.size} iters fine mean {itf.mean():.2f} max {itf.max()} "
          f"coarse mean {itc.mean():.2f} max {itc.max()}", flush=True)
    if bad.size:
        i = frm + int(bad[0])
        j = int(bad[0])
        print("  first failing index", i, "status", st[j], "itf", itf[j], "itc", itc[j], "qf", qf[j], "qc", qc[j])
        sl = np.sqrt(np.maximum(op.eigenvalues, 0))
        trunc = np.sqrt(np.maximum(op.truncated(k).eigenvalues, 0)) if k else None
        pf, pc, pitf, pitc = port.coupled(m, op.n, trunc if k else sl, trunc, ell > 0, 1, ell, i, i + 1, bc=0, qoi=3)
        print("  port:", pf, pc, pitf, pitc)
        ctx.set_history(4096)
        try:
            d = api.LevelDraws()
            api.run_level_draws(plan, api.GridSpec.square(m // 2) if ell else None, bool(k), bool(k), prob, opt, i,
                                i + 1, d, ctx=ctx)
            print("  alone: ok", d.q_fine[i], d.iters_fine[i], d.iters_coarse[i])
        except api.SolverError as e:
            h = e.residual_history
            print("  alone: SolverError, history len", None if h is None else len(h), "head", None if h is None else h[:8],
                  "tail", None if h is None else h[-4:])
        ctx.set_history(0)
