import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2306_13493_b200 as P
api = P.api
ctx = api.default_context(0)
for m, B, bc in [(512, 4, 1), (512, 32, 1), (2048, 4, 1), (2048, 16, 1)]:
    model = api.CovarianceModel.matern(2.0, 0.003, 0.5)
    prob = api.ProblemSpec(model, bc=api.BC(bc))
    opt = api.EstimatorOptions(seed=1)
    plan = api.make_level_plan(1, 2.0 / m, prob, opt)
    d = api.LevelDraws()
    api.run_level_draws(plan, api.GridSpec.square(m // 2), False, False, prob, opt, 0, B, d, ctx=ctx)
    Zf, Zc = plan.op.sample_fields(None, count=B, seed=1, ell=1, index0=0, fine=True, coarse=True, ctx=ctx)
    u, it, _ = api.assemble_and_solve(m, Zf, prob, ctx=ctx)
    q = api.evaluate_qoi(m, u, prob, ctx=ctx)
    print(f"m={m} B={B} fused iters {d.iters_fine[:B].tolist()[:6]} unfused {it.tolist()[:6]} "
          f"max rel q diff {np.max(np.abs(q - d.q_fine[:B]) / np.abs(q)):.2e}", flush=True)
