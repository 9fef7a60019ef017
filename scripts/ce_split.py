"""How much of the CE row pass is the Box-Muller draw: time ce_rows/ce_cols at config-2 size with
device Philox ξ and with a precomputed device ξ (OSC_CE_XI_DEVICE), same kernels otherwise."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2306_13493_b200 as P  # noqa: E402
from paper_2306_13493_b200 import _lib as L  # noqa: E402

api = P.api
lib = L.lib()
ctx = api.default_context(0)
m, B = (2048, 8) if "--n4096" in sys.argv else (1024, 31)
op = api.build_operator(api.GridSpec.square(m), api.CovarianceModel.matern(1.0, 0.01, 1.5 if m == 1024 else 0.5))
lev = op.device_level(ctx, 0)
out = torch.empty((B, (m + 1) ** 2), dtype=torch.float64, device="cuda:0")
xi = torch.randn((B, op.s), dtype=torch.float64, device="cuda:0")
res = {}
for mode in ("philox", "device_xi"):
    flags = L.CE_FINE | L.CE_DEVICE_OUT | (L.CE_XI_DEVICE if mode == "device_xi" else 0)
    ptr = xi.data_ptr() if mode == "device_xi" else None
    for _ in range(2):
        api._check(lib.osc_ce_sample(lev.h, ptr, 1, 0, 0, B, flags, out.data_ptr(), None))
    ctx.synchronize()
    ctx.set_profiling(True)
    ctx.reset_stats()
    for _ in range(3):
        api._check(lib.osc_ce_sample(lev.h, ptr, 1, 0, 0, B, flags, out.data_ptr(), None))
    ctx.synchronize()
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    res[mode] = {k: round(v[1] / (3 * B) * 1000, 2) for k, v in st.items()}  # µs per sample
print(json.dumps({"us_per_sample": res, "n": op.n, "batch": B}))
