import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_13493_b200 import api
m = int(sys.argv[1]) if len(sys.argv) > 1 else 128
model = api.CovarianceModel.matern(2.0, 3.0 / m, 0.5)
op = api.build_operator(api.GridSpec.square(m), model)
ctx = api.default_context()
Z = op.sample_fields(None, count=2, seed=3, ell=0, index0=0, fine=True, ctx=ctx)
prob = api.ProblemSpec(model, bc=api.BC(1))
try:
    api.assemble_and_solve(m, Z, prob, api.SolverOptions(max_iter_factor=0), ctx=ctx)
except api.SolverError:
    pass
