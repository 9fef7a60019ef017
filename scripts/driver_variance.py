import sys, time, json
sys.path.insert(0, '/root/repo')
import paper_2306_13493_b200 as P
from paper_2306_13493_b200 import mlmc as M
api = P.api
ctx = api.default_context(0)
def options(variant, l_max):
    if variant == "MLMC-CES":
        return api.EstimatorOptions(seed=1, smoothing=api.SmoothingRule.Adaptive, smoothing_lstar_only=True, l_max=l_max)
    return api.EstimatorOptions(seed=1, l_max=l_max)
import math
for lam, eps, variant, h0 in [(0.01, 0.01, "MLMC-CES", 1/16), (0.01, 0.003, "MLMC-CES", 1/16), (0.01, 0.001, "MLMC", 1/128), (0.03, 0.001, "MLMC-CES", 1/16)]:
    model = api.CovarianceModel.separable_exponential(1.0, lam)
    problem = api.ProblemSpec(model, api.QoiSpec(api.QoiKind.Flux), bc=api.BC.FlowCell)
    l_max = int(round(math.log2(2048 * h0)))
    for conc in (True, False, True, False):
        t0 = time.perf_counter()
        d = M.mlmc_adaptive(problem, options(variant, l_max), h0, eps, concurrent=conc)
        w = time.perf_counter() - t0
        print(lam, eps, variant, 'conc' if conc else 'serial', 'wall %.2f setup %.2f draw %.2f waves %d' % (w, d.setup_s, d.draw_s, d.waves), [l.n for l in d.levels], flush=True)
