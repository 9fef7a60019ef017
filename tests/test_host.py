"""CPU tests of the product's host side: the C-ABI library loads and exports every symbol
include/oscfield_b200.h declares; host level setup (spectrum, padding, truncation) and the
estimator host math agree with the reference golden vectors; no GPU compute is called."""
import ctypes
import os
import re

import numpy as np
import pytest


def test_abi_exports_every_declared_symbol(P):
    from paper_2306_13493_b200 import _lib
    header = open(_lib.HEADER).read()
    declared = set(re.findall(r"\b(osc_[a-z_0-9]+)\s*\(", header))
    assert declared == set(_lib.EXPORTS)
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name


def test_library_is_sm100a(P):
    import subprocess
    from paper_2306_13493_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("name", ["sepexp_m2_l1", "sepexp_m8_l01", "matern_m8_nu05",
                                  "matern_m16_nu15_pad", "matern_m16_nu15"])
def test_host_spectrum_matches_reference(P, golden, name):
    api = P.api
    m, fam, s2, lam, nu = {"sepexp_m2_l1": (2, 1, 1.0, 1.0, 1.0), "sepexp_m8_l01": (8, 1, 1.0, 0.1, 1.0),
                           "matern_m8_nu05": (8, 0, 1.0, 0.1, 0.5),
                           "matern_m16_nu15_pad": (16, 0, 1.0, 0.3, 1.5),
                           "matern_m16_nu15": (16, 0, 2.0, 0.05, 1.5)}[name]
    model = api.CovarianceModel.matern(s2, lam, nu) if fam == 0 else \
        api.CovarianceModel.separable_exponential(s2, lam, nu)
    op = api.build_operator(api.GridSpec.square(m), model)
    ref = golden[f"eig_{name}"]
    assert op.padding[0] == int(golden[f"J_{name}"][0])
    assert np.max(np.abs(op.eigenvalues - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert abs(ref.sum() - op.s * s2) < 1e-8 * op.s * s2  # trace identity (SPEC)


def test_spec_spectrum_example(P):
    # d=1 analogue in SPEC: row (1, e^-1/2, e^-1, e^-1/2); here the 2-D m=2, λ=1 sep-exp operator
    api = P.api
    op = api.build_operator(api.GridSpec.square(2), api.CovarianceModel.separable_exponential(1, 1))
    lam1 = np.array([1 + np.exp(-1) * np.cos(np.pi * q) + 2 * np.exp(-0.5) * np.cos(np.pi * q / 2)
                     for q in range(4)])
    assert np.allclose(op.eigenvalues.reshape(4, 4), np.outer(lam1, lam1), rtol=1e-13, atol=1e-14)


def test_truncation_mask_uses_stable_descending_order(P, golden):
    api = P.api
    eig = golden["eig_matern_m16_nu15"]
    op = api.EmbeddingOperator(api.GridSpec.square(16), 0, eig, 2.0)
    assert np.array_equal(op.perm(), golden["perm_matern_m16_nu15"])
    t = op.truncated(op.s // 2)
    assert np.count_nonzero(t.eigenvalues == 0) >= op.s // 2
    with pytest.raises(api.ConfigError):
        op.truncated(op.s)


def test_osc1_roundtrip(P, tmp_path, golden):
    api = P.api
    op = api.EmbeddingOperator(api.GridSpec.square(16), 8, golden["eig_matern_m16_nu15_pad"], 1.0)
    p = str(tmp_path / "s.osc1")
    api.save_spectrum(op, p)
    op2 = api.load_spectrum(p, 1.0)
    assert op2.padding == (8, 8) and np.array_equal(op2.eigenvalues, op.eigenvalues)


def test_osc1_reads_reference_dump(P, ref, tmp_path):
    api = P.api
    r = ref.build_operator(16, 0, 1.0, 0.3, 1.5)
    p = str(tmp_path / "r.osc1")
    r.save(p)
    op = api.load_spectrum(p, 1.0)
    assert op.padding[0] == r.J and np.array_equal(op.eigenvalues, r.eigenvalues())


def test_estimator_host_math(P, golden):
    api = P.api
    ks = [api.choose_k_ell(api.CovarianceModel.separable_exponential(1, 0.01), h, 0, int((2 / h) ** 2), 1, 1)
          for h in (1 / 16, 1 / 32, 1 / 64)]
    ks += [api.choose_k_ell(api.CovarianceModel.matern(1, 0.1, 1.5), h, 0, int((2 / h) ** 2), 1, 1)
           for h in (1 / 16, 1 / 32)]
    assert ks == [int(x) for x in golden["k_ell"]]
    b = golden["coarsest_bound"]
    assert api.coarsest_level_bound(api.CovarianceModel.separable_exponential(1, 0.01)) == b[0]
    assert api.coarsest_level_bound(api.CovarianceModel.matern(1, 0.03, 1.5)) == b[1]
    with pytest.raises(api.NumericalError):
        api.richardson_bias(1.0, 1.0, 0.5, True)


def test_summarize_matches_welford(P, port):
    api = P.api
    d = api.LevelDraws()
    d.resize(50)
    rng = np.random.default_rng(4)
    d.q_fine[:] = rng.standard_normal(50)
    d.q_coarse[:] = rng.standard_normal(50)
    s = api.summarize_draws(d, True)
    o = port.moments(d.q_fine, d.q_coarse, True)
    assert (s.n, s.mean_y, s.var_y, s.mean_q, s.var_q) == (o["n"], o["mean_y"], o["var_y"], o["mean_q"], o["var_q"])


def test_config_errors(P):
    api = P.api
    with pytest.raises(api.ConfigError):
        api.CovarianceModel.matern(-1, 0.1, 0.5)
    with pytest.raises(api.ConfigError):
        api.make_level_plan(0, 0.3, api.ProblemSpec(api.CovarianceModel.matern(1, 0.1, 0.5)),
                            api.EstimatorOptions())
    with pytest.raises(api.ConfigError):
        api.EmbeddingOperator(api.GridSpec.square(4), 0, np.zeros(10), 1.0)


def test_embedding_error_when_no_spd_padding(P):
    """build_operator exhausts the padding schedule → EmbeddingError (embedding.cpp:142-149)."""
    api = P.api
    with pytest.raises(api.EmbeddingError):
        api.build_operator(api.GridSpec.square(4), api.CovarianceModel.matern(1.0, 2.0, 1.5))


def test_padded_embedding_sizes(P, ref):
    """Padding J (smooth periodisation) matches the pristine reference; n = 2(m+J) factors into 2,3,5."""
    api = P.api
    for m, lam, nu in [(4, 1.0, 1.5), (8, 0.5, 3.5), (8, 1.0, 1.5), (16, 0.3, 1.5)]:
        op = api.build_operator(api.GridSpec.square(m), api.CovarianceModel.matern(1.0, lam, nu))
        r = ref.build_operator(m, 0, 1.0, lam, nu)
        assert op.padding[0] == r.J
        e = r.eigenvalues()
        assert np.max(np.abs(op.eigenvalues - e)) <= 1e-10 * np.max(np.abs(e))
        v = op.n
        for f in (2, 3, 5):
            while v % f == 0:
                v //= f
        assert v == 1


def test_fit_rates(P):
    api = P.api
    pts = [api.RatePoint(h, 0.3 * h, 2.0 * h ** 2, 5.0 * h ** -2) for h in (1 / 8, 1 / 16, 1 / 32, 1 / 64)]
    f = api.fit_rates(pts)
    assert abs(f.alpha - 1) < 1e-12 and abs(f.beta - 2) < 1e-12 and abs(f.gamma - 2) < 1e-12
    assert abs(f.c_alpha - 0.3) < 1e-12
    w = []
    pts[0].mean_abs_y = 0.0
    f = api.fit_rates(pts, w)
    assert w and abs(f.alpha - 1) < 1e-12
    with pytest.raises(api.ConfigError):
        api.fit_rates(pts[:2])
