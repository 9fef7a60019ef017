"""Oracle (reference-algorithm port) PCG iteration medians with the extension BCs, for the
SURVEY §8(d) roofline basis: cfg 4 (2048²/1024² coupled, homogeneous Dirichlet) and cfg 1 (64²,
Dirichlet), seed 1, sample indices 0..7. Writes profiles/oracle_iters.json."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_13493_b200 import api  # noqa: E402  (host setup only: no GPU needed)
from oracle.oracle import Port  # noqa: E402

port = Port()
out = {}
for name, m, lam, s2, coupled, ell in [("cfg1", 64, 0.1, 1.0, False, 0), ("cfg4", 2048, 0.003, 2.0, True, 1)]:
    model = api.CovarianceModel.matern(s2, lam, 0.5)
    op = api.build_operator(api.GridSpec.square(m), model)
    sl = np.sqrt(np.maximum(op.eigenvalues, 0))
    qf, qc, itf, itc = port.coupled(m, op.n, sl, None, coupled, 1, ell, 0, 8, bc=1, qoi=2 if name == "cfg1" else 0,
                                    threads=8)
    out[name] = {"fine_iters": [int(x) for x in itf], "coarse_iters": [int(x) for x in itc] if coupled else None,
                 "median_fine": float(np.median(itf)), "median_coarse": float(np.median(itc)) if coupled else None}
    print(name, out[name], flush=True)
with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "oracle_iters.json"), "w") as f:
    json.dump(out, f, indent=1)
