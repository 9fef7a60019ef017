"""Level setup that stays in HBM (osc_level_create_device / osc_level_retruncate /
osc_level_eigenvalues) and the fused smoothing-error pass (osc_smoothing_error), through the C-ABI,
against the pristine reference (oracle/_ref) and the host setup path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cov(api, O, model):
    if model[0] == "sep":
        return api.CovarianceModel.separable_exponential(model[1], model[2]), (O.SEP_EXP, model[1], model[2], 1.0)
    return api.CovarianceModel.matern(model[1], model[2], model[3]), (O.MATERN, model[1], model[2], model[3])


@pytest.mark.parametrize("m,model", [
    (16, ("sep", 1.0, 0.01)), (256, ("sep", 1.0, 0.01)),  # config 3's coarsest and finest level
    (64, ("matern", 1.0, 0.1, 0.5)),                      # config 1
    (1024, ("matern", 1.0, 0.01, 1.5)),                   # config 2
    (16, ("matern", 1.0, 0.3, 1.5)),                      # padded, J > 0 (mixed-radix CE)
    (32, ("matern", 1.5, 0.2, 0.8)), (64, ("matern", 1.0, 0.05, 2.3)),  # general ν: the device K_ν
    (16, ("matern", 1.0, 0.4, 1.0)),                      # integer ν, padded
])
def test_level_create_device_vs_pristine_reference(P, ctx, ref, m, model):
    """build_operator + from_parts + truncated in HBM: same J and eigenvalues (1e-12 of max λ) as
    the pristine reference; the device order is the stable descending order of the device's own
    eigenvalues (embedding.cpp:105-107), i.e. truncated fields are bit-identical to a level uploaded
    from those eigenvalues through the host sort."""
    from oracle import oracle as O
    api = P.api
    cov, rargs = _cov(api, O, model)
    r = ref.build_operator(m, *rargs)
    k = r.s // 2
    lev = api.DeviceLevel.from_model(ctx, api.GridSpec.square(m), cov, k_trunc=k)
    assert (lev.J, lev.s, lev.k_trunc) == (r.J, r.s, k)
    eig = lev.eigenvalues()
    e = r.eigenvalues()
    assert np.max(np.abs(eig - e)) < 1e-12 * np.max(np.abs(e)) and eig.min() >= 0.0
    host = api.DeviceLevel(ctx, m, lev.J, eig, k)  # host stable_sort of the same eigenvalues
    for trunc in (False, True):
        a = lev.sample_fields(None, count=2, seed=3, ell=1, index0=7, truncated=trunc)
        b = host.sample_fields(None, count=2, seed=3, ell=1, index0=7, truncated=trunc)
        assert np.array_equal(a, b), (m, model, trunc)
    # truncated(k') from the resident order
    k2 = max(1, r.s // 5)
    lev.retruncate(k2)
    host2 = api.DeviceLevel(ctx, m, lev.J, eig, k2)
    assert np.array_equal(lev.sample_fields(None, count=1, seed=3, ell=0, index0=1, truncated=True),
                          host2.sample_fields(None, count=1, seed=3, ell=0, index0=1, truncated=True))
    lev.retruncate(0)
    with pytest.raises(api.ConfigError):
        lev.sample_fields(None, count=1, truncated=True)  # no truncated spectrum any more
    with pytest.raises(api.ConfigError):
        lev.retruncate(r.s)
    with pytest.raises(api.ConfigError):
        host.retruncate(3)  # host-uploaded levels hold no device order
    with pytest.raises(api.ConfigError):
        host.eigenvalues()


def test_level_create_device_errors(P, ctx):
    api = P.api
    g = api.GridSpec.square(16)
    with pytest.raises(api.ConfigError):  # ν beyond the device K_ν's range
        api.DeviceLevel.from_model(ctx, g, api.CovarianceModel.matern(1.0, 0.1, 80.0))
    with pytest.raises(api.EmbeddingError):  # no SPD padding in the schedule
        api.DeviceLevel.from_model(ctx, g, api.CovarianceModel.matern(1.0, 2.0, 3.5),
                                   options=api.BuildOptions(padding_fractions=(0.5,)))


@pytest.mark.parametrize("m,model,frac", [(16, ("sep", 1.0, 0.1), 0.5), (64, ("matern", 1.0, 0.1, 0.5), 0.8),
                                          (24, ("matern", 1.0, 0.3, 1.5), 0.5)])
def test_smoothing_error_fused_pass(P, ctx, ref, m, model, frac):
    """osc_smoothing_error (one CE pass over the dropped modes, sup-norm in the column epilogue)
    against the pristine reference's two-field loop (embedding.cpp:205-228) on the same ξ and mask,
    and against the device's own two-pass difference."""
    from oracle import oracle as O
    api = P.api
    cov, rargs = _cov(api, O, model)
    r = ref.build_operator(m, *rargs)
    op = api.EmbeddingOperator(api.GridSpec.square(m), r.J, r.eigenvalues(), model[1])
    k = int(op.s * frac)
    n = 24
    lev = op.device_level(ctx, k)
    st, sups = lev.smoothing_error(n, 5, return_sups=True)
    tr = r.truncated(k)
    want = []
    for i in range(n):
        xi = ref.normals(5, 0, i, r.s)
        want.append(np.max(np.abs(r.restrict(r.sample(xi), m) - tr.restrict(tr.sample(xi), m))))
    want = np.array(want)
    assert np.max(np.abs(sups - want)) < 1e-10 * np.max(want)
    assert abs(st.mean - want.mean()) < 1e-10 * want.mean()
    assert abs(st.variance - want.var(ddof=1)) < 1e-8 * want.var(ddof=1)
    full = lev.sample_fields(None, count=n, seed=5, ell=0, index0=0)
    smooth = lev.sample_fields(None, count=n, seed=5, ell=0, index0=0, truncated=True)
    two_pass = np.max(np.abs(full - smooth), axis=1)
    assert np.max(np.abs(sups - two_pass)) < 1e-12 * np.max(two_pass)
    g = api.smoothing_error_estimate(op, k, n, seed=5, ctx=ctx)
    assert (g.mean, g.variance) == (st.mean, st.variance)
    with pytest.raises(api.ConfigError):
        api.smoothing_error_estimate(op, k, 1, seed=5, ctx=ctx)
