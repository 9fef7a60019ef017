"""Replay single config-3 samples that failed in the per-level bench: status, residual history, and
the oracle port on the same sample."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_13493_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

api = P.api
ctx = api.default_context(0)
model = api.CovarianceModel.separable_exponential(1.0, 0.01)
prob = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
opt = api.EstimatorOptions(seed=1)
port = O.Port()
for ell, idx in [(2, 4096012249), (3, 3595)]:
    m = 16 << ell
    op = api.build_operator(api.GridSpec.square(m), model)
    k = op.s // 2 if ell <= 2 else 0
    plan = api.make_level_plan(ell, 1.0 / 16, prob, opt, operator=op, k_trunc=k)
    sq = np.sqrt(np.maximum((op.truncated(k) if k else op).eigenvalues, 0))
    # fields of the sample, solved alone: fine and coarse separately, with history
    fine, coarse = (op.truncated(k) if k else op).sample_fields(None, count=1, seed=1, ell=ell, index0=idx,
                                                                 fine=True, coarse=True, ctx=ctx)
    for name, mm, Z in [("fine", m, fine), ("coarse", m // 2, coarse)]:
        try:
            u, it, h = api.assemble_and_solve(mm, Z, prob, hist_cap=4096, ctx=ctx)
            print(ell, idx, name, "GPU alone ok, iters", it[0], "last", h[0, it[0]])
        except api.SolverError as e:
            hh = e.residual_history[0]
            nz = hh[hh != 0]
            print(ell, idx, name, "GPU alone FAIL", len(nz), "head", nz[:6], "tail", nz[-6:], "min", nz.min())
        uo, ito, rc, ho = port.solve(mm, Z[0], bc=0)
        print("   port: rc", rc, "iters", ito, "Zmin/max", Z.min(), Z.max())
    # the coupled draw alone (nested start) with history capture
    ctx.set_history(4096)
    try:
        d = api.LevelDraws()
        api.run_level_draws(plan, api.GridSpec.square(m // 2), bool(k), bool(k), prob, opt, idx, idx + 1, d, ctx=ctx)
        print(ell, idx, "coupled alone ok", d.iters_fine[idx], d.iters_coarse[idx])
    except api.SolverError as e:
        h = e.residual_history
        print(ell, idx, "coupled alone FAIL hist len", len(h), h[:6], h[-6:])
    ctx.set_history(0)
    # inside its original batch
    B = 4096 if ell == 2 else 2048
    frm = (idx // B) * B
    d = api.LevelDraws()
    try:
        api.run_level_draws(plan, api.GridSpec.square(m // 2), bool(k), bool(k), prob, opt, frm, frm + B, d, ctx=ctx)
        print(ell, "batch ok", d.iters_fine[idx], d.iters_coarse[idx])
    except api.SolverError as e:
        st = e.status
        print(ell, "batch FAIL slots", np.nonzero(st)[0][:5] + frm)
