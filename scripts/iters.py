"""Compare PCG iteration counts of the GPU MG (red-black GS) with the oracle port (lexicographic GS)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2306_13493_b200 as P
from oracle import oracle as O
api = P.api
port = O.Port()
ctx = api.default_context(0)
for m in [int(x) for x in (sys.argv[1:] or ["64", "256", "1024"])]:
    model = api.CovarianceModel.matern(2.0, 0.003, 0.5)
    op = api.build_operator(api.GridSpec.square(m), model)
    Z = op.sample_fields(None, count=3, seed=1, ell=0, index0=0, fine=True, ctx=ctx)
    for bc in (0, 1):
        prob = api.ProblemSpec(model, bc=api.BC(bc))
        u, it, h = api.assemble_and_solve(m, Z, prob, ctx=ctx, hist_cap=400)
        itp = [port.solve(m, Z[b], bc=bc)[1] for b in range(3)] if m <= 512 else "-"
        rates = [float((h[b, it[b]] / h[b, 0]) ** (1.0 / it[b])) for b in range(3)]
        print(f"m={m} bc={bc} gpu iters {list(it)} rate {np.round(rates, 3)} port(lex GS) iters {itp}", flush=True)
