"""Residual histories of one solve with the marching vs the one-thread-per-node coarse kernels."""
import os, subprocess, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r"""
import sys, json, numpy as np
sys.path.insert(0, %r)
from paper_2306_13493_b200 import api
out = {}
for m, bc in [(256, 1), (128, 1)]:
    model = api.CovarianceModel.matern(2.0, 3.0 / m, 0.5)
    op = api.build_operator(api.GridSpec.square(m), model)
    ctx = api.default_context()
    Z = op.sample_fields(None, count=2, seed=3, ell=0, index0=0, fine=True, ctx=ctx)
    prob = api.ProblemSpec(model, bc=api.BC(bc))
    for mode in (0,):
        try:
            u, it, h = api.assemble_and_solve(m, Z, prob, api.SolverOptions(coarse_operator=api.CoarseOperator(mode), max_iter_factor=0), hist_cap=40, ctx=ctx)
            out[f"{m}_{bc}_{mode}"] = [it.tolist(), h[0][:25].tolist()]
        except api.SolverError as e:
            out[f"{m}_{bc}_{mode}"] = ["fail", e.residual_history[0][:25].tolist() if e.residual_history is not None else None]
print(json.dumps(out))
""" % ROOT
res = {}
for name, env in [("march", {}), ("simple", {"OSC_SIMPLE_COARSE": "1"}), ("sdown", {"OSC_SIMPLE_DOWN": "1"}), ("sup", {"OSC_SIMPLE_UP": "1"})]:
    e = dict(os.environ, OSC_HARD_ITER_CAP="40", **env)
    p = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600)
    res[name] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-2000:]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "debug_coarse.json"), "w") as f:
    json.dump(res, f, indent=1)
print("done")
