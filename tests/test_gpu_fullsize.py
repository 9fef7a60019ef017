"""Parity at the BASELINE configs' full sizes: config 2's sample covariance against its target
kernel, config 4's n = 4096 fields against the oracle port, and the device level setup against the
pristine reference's build_operator (oracle/_ref) at the config sizes."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-10


def relmax(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_cfg2_sample_covariance_matches_matern_kernel(P, ctx):
    """BASELINE config 2: Matérn ν = 1.5, σ² = 1, λ = 0.01 on 1024² (n = 2048,
    J = 0), 4096 device-Philox samples. Per sample, the spatial averages of Z, Z² and Z(p)Z(p+h) over
    every node pair at lag h are iid across samples; their sample means must match 0, σ² and the
    target C(h) = σ²(1 + √3 r/λ) e^{−√3 r/λ} within 4 standard errors."""
    import torch
    api = P.api
    m, sigma2, lam = 1024, 1.0, 0.01
    op = api.build_operator(api.GridSpec.square(m), api.CovarianceModel.matern(sigma2, lam, 1.5))
    assert op.padding[0] == 0 and op.n == 2048
    lev = op.device_level(ctx, 0)
    lags = [(0, 0), (3, 0), (0, 3), (6, 0), (0, 12), (4, 4), (25, 0)]
    S, chunk = 4096, 256
    n0 = m + 1
    out = torch.empty((chunk, n0 * n0), dtype=torch.float64, device="cuda:0")
    stats = {"mean": [], "sq": [], **{lag: [] for lag in lags}}
    import ctypes as C
    L = P._lib
    for c0 in range(0, S, chunk):
        rc = L.lib().osc_ce_sample(lev.h, None, 1, 0, c0, chunk, L.CE_FINE | L.CE_DEVICE_OUT,
                                   C.c_void_p(out.data_ptr()), None)
        assert rc == 0, L.last_error()
        torch.cuda.synchronize()
        Z = out.view(chunk, n0, n0)  # [b][y][x]
        stats["mean"].append(Z.mean(dim=(1, 2)).cpu().numpy())
        stats["sq"].append((Z * Z).mean(dim=(1, 2)).cpu().numpy())
        for (dx, dy) in lags:
            a = Z[:, :n0 - dy, :n0 - dx]
            b = Z[:, dy:, dx:]
            stats[(dx, dy)].append((a * b).mean(dim=(1, 2)).cpu().numpy())

    def check(vals, target, what):
        v = np.concatenate(vals)
        se = v.std(ddof=1) / math.sqrt(v.size)
        print(f"{what}: {v.mean():.5f} vs {target:.5f} (SE {se:.2e})")
        assert abs(v.mean() - target) < 4 * se + 1e-12, what

    check(stats["mean"], 0.0, "mean")
    check(stats["sq"], sigma2, "variance")
    for (dx, dy) in lags:
        x = math.sqrt(3.0) * math.hypot(dx, dy) / m / lam
        check(stats[(dx, dy)], sigma2 * (1 + x) * math.exp(-x), f"C(lag {dx},{dy})")


def test_cfg4_fields_n4096_vs_port(P, ctx, port):
    """Config 4's embedding (m = 2048, n = 4096, Matérn ν = 0.5, σ² = 2, λ = 0.003): the device CE
    field (device Philox NormalStream(1, 1, i)), fine R-block and stride-2 coarse, against the port's
    sample_into + restrict_to on the same ξ, ≤ 1e-10 of max|Z|."""
    api = P.api
    m = 2048
    op = api.build_operator(api.GridSpec.square(m), api.CovarianceModel.matern(2.0, 0.003, 0.5))
    assert op.n == 4096
    fine, coarse = op.sample_fields(None, count=2, seed=1, ell=1, index0=5, fine=True, coarse=True, ctx=ctx)
    sl = np.sqrt(np.maximum(op.eigenvalues, 0))
    for b in range(2):
        u = port.sample(op.n, sl, port.normals(1, 1, 5 + b, op.s))
        assert relmax(fine[b], port.restrict(op.n, m, u, m)) < FIELD_TOL
        assert relmax(coarse[b], port.restrict(op.n, m, u, m // 2)) < FIELD_TOL


@pytest.mark.parametrize("m,model", [
    (16, ("sep", 1.0, 0.01)), (64, ("sep", 1.0, 0.01)), (256, ("sep", 1.0, 0.01)),  # config 3 levels
    (64, ("matern", 1.0, 0.1, 0.5)),                                               # config 1
    (1024, ("matern", 1.0, 0.01, 1.5)),                                            # config 2
    (2048, ("matern", 2.0, 0.003, 0.5)),                                           # config 4
    (16, ("matern", 1.0, 0.3, 1.5)),                                               # padded, J > 0
])
def test_device_setup_vs_pristine_reference(P, ctx, ref, m, model):
    """osc_build_spectrum_device (first row + spectrum FFT on the GPU) against the pristine
    reference's build_operator (oracle/_ref, embedding.cpp:67-151): same padding J, eigenvalues
    within 1e-12 of max λ."""
    from oracle import oracle as O
    api = P.api
    if model[0] == "sep":
        cov = api.CovarianceModel.separable_exponential(model[1], model[2])
        r = ref.build_operator(m, O.SEP_EXP, model[1], model[2], 1.0)
    else:
        cov = api.CovarianceModel.matern(model[1], model[2], model[3])
        r = ref.build_operator(m, O.MATERN, model[1], model[2], model[3])
    op = api.build_operator(api.GridSpec.square(m), cov, device=True, ctx=ctx)
    e = r.eigenvalues()
    assert op.padding[0] == r.J and op.s == e.size
    d = np.max(np.abs(op.eigenvalues - e)) / np.max(np.abs(e))
    print(f"m={m} {model}: J={r.J} max|Δλ|/max λ = {d:.2e}")
    assert d < 1e-12
