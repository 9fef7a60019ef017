import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2306_13493_b200 as P
api = P.api
ctx = api.default_context(0)
m = int(sys.argv[1]); bc = int(sys.argv[2])
model = api.CovarianceModel.matern(2.0, 0.003, 0.5)
op = api.build_operator(api.GridSpec.square(m), model)
Z = op.sample_fields(None, count=1, seed=1, ell=0, index0=0, fine=True, ctx=ctx)
prob = api.ProblemSpec(model, bc=api.BC(bc))
t = time.time()
try:
    u, it, h = api.assemble_and_solve(m, Z, prob, api.SolverOptions(1e-10, 10), ctx=ctx, hist_cap=200)
    print(m, bc, "iters", it, f"{time.time()-t:.2f}s", np.round(h[0, :12], 4), flush=True)
except Exception as e:
    print(m, bc, "ERR", e, flush=True); h = getattr(e, "residual_history", None); print(np.round(h[0, :200:10], 5) if h is not None else None)
