"""osc_mlmc_adaptive — the GPU-resident adaptive driver (csrc/driver.cpp).

CPU part: the smoothing rule against the pristine reference's choose_k_ell / coarsest_level_bound
(estimators.cpp:238-275, 487-494) and the argument checks, none of which touch the device.
GPU part: the driver against the pristine reference's own mlmc_estimate on the CPU (oracle/_ref):
both draw sample i of level ℓ from NormalStream(seed, ℓ, i) and solve to 1e-10, so they must take the
SAME decisions (levels, N_ℓ, convergence) and agree in every level moment far inside the sampling
confidence intervals north_star asks for.
"""
import os

import numpy as np
import pytest

MOMENT_TOL = 1e-6


def _opts(P, lam=0.1, smoothing=0, lstar=0, family="sep", nu=1.0, alpha=1.0, c_ratio=1.0, use_coarse=False, **kw):
    api = P.api
    model = (api.CovarianceModel.separable_exponential(1.0, lam) if family == "sep"
             else api.CovarianceModel.matern(1.0, lam, nu))
    opt = api.EstimatorOptions(smoothing=api.SmoothingRule(smoothing), smoothing_lstar_only=bool(lstar), alpha=alpha,
                               c_ratio=c_ratio, smoothing_use_coarse_s=use_coarse, **kw)
    return api.ProblemSpec(model), opt


def test_k_trunc_rule_matches_reference(P, ref):
    from oracle import oracle as O
    from paper_2306_13493_b200 import mlmc
    for family, fam_id, nu in (("sep", O.SEP_EXP, 1.0), ("matern", O.MATERN, 0.5), ("matern", O.MATERN, 1.5)):
        for lam in (0.3, 0.03, 0.01):
            for alpha, c_ratio, use_coarse in ((1.0, 1.0, False), (1.5, 0.7, True), (0.8, 2.0, False)):
                prob, opt = _opts(P, lam=lam, smoothing=2, family=family, nu=nu, alpha=alpha, c_ratio=c_ratio,
                                  use_coarse=use_coarse)
                o = mlmc.make_options(prob, opt, 1 / 8, 1e-2)
                for m, J in ((8, 0), (32, 0), (64, 16), (512, 0)):
                    s = (2 * (m + J)) ** 2
                    want = ref.choose_k_ell(fam_id, 1.0, lam, nu, 1.0 / m, J, s, alpha, c_ratio, int(use_coarse))
                    assert mlmc.k_trunc(o, 1.0 / m, J, s) == want, (family, nu, lam, alpha, m, J)
        # lstar_only: resolved levels stay unsmoothed; HalfSpectrum: s/2
        prob, opt = _opts(P, lam=0.03, smoothing=1, lstar=1, family=family, nu=nu)
        o = mlmc.make_options(prob, opt, 1 / 8, 1e-2)
        bound = ref.coarsest_level_bound(fam_id, 1.0, 0.03, nu)
        for m in (4, 8, 16, 32, 64, 128):
            h = 1.0 / m
            assert mlmc.k_trunc(o, h, 0, 4 * m * m) == (0 if h <= bound * (1 + 1e-12) else 2 * m * m)


def test_driver_argument_errors(P):
    from paper_2306_13493_b200 import mlmc
    api = P.api
    prob, opt = _opts(P)
    with pytest.raises(api.ConfigError):
        mlmc.mlmc_adaptive(prob, opt, 1 / 8, 0.0)          # eps must be positive
    with pytest.raises(api.ConfigError):
        mlmc.mlmc_adaptive(prob, opt, 0.3, 1e-2)           # h0 not a negative power of two
    with pytest.raises(api.ConfigError):
        mlmc.mlmc_adaptive(prob, opt, 1 / 8, 1e-2, 0)      # at least one level


def _same_report(gpu, cpu):
    lv = cpu.levels()
    assert len(gpu.levels) == len(lv), (len(gpu.levels), len(lv))
    for a, b in zip(gpu.levels, lv):
        assert a.n == b["n"], ("N_l differs", a.n, b["n"])
        sd_y, sd_q = np.sqrt(max(b["var_y"], 0.0)), np.sqrt(max(b["var_q"], 0.0))
        assert abs(a.mean_y - b["mean_y"]) <= MOMENT_TOL * (abs(b["mean_y"]) + sd_y)
        assert abs(a.mean_q - b["mean_q"]) <= MOMENT_TOL * (abs(b["mean_q"]) + sd_q)
        assert abs(a.var_y - b["var_y"]) <= MOMENT_TOL * b["var_y"] + 1e-300
        assert abs(a.var_q - b["var_q"]) <= MOMENT_TOL * b["var_q"] + 1e-300
    tot_sd = np.sqrt(sum(l["var_y"] / max(l["n"], 1) for l in lv))
    assert abs(gpu.estimate - cpu.estimate) <= MOMENT_TOL * (abs(cpu.estimate) + tot_sd)
    assert abs(gpu.sampling_error - cpu.sampling_error) <= MOMENT_TOL * cpu.sampling_error
    assert abs(gpu.bias_estimate - cpu.bias_estimate) <= MOMENT_TOL * (abs(cpu.bias_estimate) + tot_sd)
    assert bool(gpu.converged) == bool(cpu.converged)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["off_point", "cfg3_rule_point", "cfg3_rule_l2", "half_spectrum"])
def test_driver_vs_cpu_reference(P, ctx, ref, case):
    """'off': smoothing Off (device level setup: no truncation mask involved). 'cfg3_rule': BASELINE config
    3's rule (Adaptive + lstar_only, h0 = 1/16, sep-exp λ = 0.01) at ε = 1e-2; 'half_spectrum': every level
    smoothed, so each level extension changes the previous finest level's law and redraws it. The smoothed
    cases take the eigenvalues from the reference's build_operator (spectrum callback): the truncation mask
    cuts through groups of equal eigenvalues, whose order is only reproducible from the same bits."""
    from oracle import oracle as O
    from paper_2306_13493_b200 import mlmc
    threads = os.cpu_count() or 1
    if case == "off_point":
        lam, h0, eps, levels, sm, lstar, qk = 0.1, 1.0 / 8, 2e-3, 2, 0, 0, 0
    elif case == "half_spectrum":
        lam, h0, eps, levels, sm, lstar, qk = 0.1, 1.0 / 8, 4e-3, 1, 1, 0, 0
    else:
        lam, h0, eps, levels, sm, lstar, qk = 0.01, 1.0 / 16, 1e-2, 1, 2, 1, (1 if case.endswith("l2") else 0)
    pilot, l_max = 50, 4
    opts = O.RefOpts.make(family=O.SEP_EXP, sigma2=1.0, lam=lam, nu_or_p=1.0, seed=1, pilot_n=pilot,
                          threads=threads, l_max=l_max, smoothing=sm, lstar_only=lstar, qoi_kind=qk)
    cpu = ref.mlmc(opts, h0, eps, levels)
    api = P.api
    prob = api.ProblemSpec(api.CovarianceModel.separable_exponential(1.0, lam),
                           api.QoiSpec(api.QoiKind.L2Norm if qk else api.QoiKind.Point))
    opt = api.EstimatorOptions(seed=1, pilot_n=pilot, l_max=l_max, smoothing=api.SmoothingRule(sm),
                               smoothing_lstar_only=bool(lstar))

    def spectrum(m):
        op = ref.build_operator(m, O.SEP_EXP, 1.0, lam, 1.0)
        return op.J, op.eigenvalues()

    gpu = mlmc.mlmc_adaptive(prob, opt, h0, eps, levels, spectrum=None if sm == 0 else spectrum)
    print(case, "levels", [l.n for l in gpu.levels], "k", gpu.k_trunc, "redrawn", gpu.redrawn, "waves", gpu.waves,
          "estimate", gpu.estimate, cpu.estimate, "s", round(gpu.total_s, 3))
    _same_report(gpu, cpu)
    assert gpu.gpu_launches > 0 and gpu.samples_total >= sum(l.n for l in gpu.levels)
    if case == "half_spectrum":
        assert sum(gpu.redrawn) > 0


@pytest.mark.gpu
def test_driver_concurrent_levels_equal_serial(P, ctx):
    """Levels drawn at the same time (one stream per level) and one after the other give the same
    decisions and the same moments: every sample is a pure function of (seed, ℓ, i)."""
    from paper_2306_13493_b200 import mlmc
    api = P.api
    prob, opt = _opts(P, lam=0.1, seed=3, pilot_n=40, l_max=3)
    a = mlmc.mlmc_adaptive(prob, opt, 1 / 8, 3e-3, 2, concurrent=True)
    b = mlmc.mlmc_adaptive(prob, opt, 1 / 8, 3e-3, 2, concurrent=False)
    assert [l.n for l in a.levels] == [l.n for l in b.levels]
    for x, y in zip(a.levels, b.levels):
        assert abs(x.mean_y - y.mean_y) <= 1e-13 * (abs(y.mean_y) + np.sqrt(y.var_y))
        assert abs(x.var_y - y.var_y) <= 1e-12 * y.var_y
    assert a.waves == b.waves and a.converged == b.converged


@pytest.mark.gpu
def test_driver_matches_routed_reference_estimator_extension_qoi(P, ctx):
    """Config 3's flux QoI and the all-Dirichlet BC (extensions) through the driver and through the
    reference's own estimate_adaptive over the seam: identical N_ℓ and moments."""
    from paper_2306_13493_b200 import estimators as E
    from paper_2306_13493_b200 import mlmc
    api = P.api
    try:
        E.lib()
    except ImportError as e:
        pytest.fail(f"GPU-routed reference build missing: {e}")
    prob = api.ProblemSpec(api.CovarianceModel.separable_exponential(1.0, 0.1), api.QoiSpec(api.QoiKind.Flux))
    opt = api.EstimatorOptions(seed=5, pilot_n=40, l_max=3)
    a = mlmc.mlmc_adaptive(prob, opt, 1 / 8, 4e-3, 2)
    b = E.mlmc_estimate(prob, opt, 1 / 8, 4e-3, 2)
    E.mc_estimate_fixed_n(api.ProblemSpec(prob.model), opt, 16, 4)  # reset the seam's QoI mapping
    assert [l.n for l in a.levels] == [l.n for l in b.levels]
    for x, y in zip(a.levels, b.levels):
        assert abs(x.mean_y - y.mean_y) <= 1e-10 * (abs(y.mean_y) + np.sqrt(y.var_y))
        assert abs(x.var_y - y.var_y) <= 1e-9 * y.var_y
    assert abs(a.estimate - b.estimate) <= 1e-10 * abs(b.estimate)


@pytest.mark.gpu
def test_driver_single_level_mc(P, ctx, ref):
    """mc_estimate with a fixed mesh (estimators.cpp:398-412): one level, sampling error only."""
    from oracle import oracle as O
    from paper_2306_13493_b200 import mlmc
    api = P.api
    prob, opt = _opts(P, lam=0.1, seed=2, pilot_n=30)
    rep = mlmc.mc_adaptive(prob, opt, 2e-2, 1 / 16)
    assert len(rep.levels) == 1 and rep.converged and "single level" in rep.message
    assert rep.sampling_error ** 2 <= 0.5 * 2e-2 ** 2 * (1 + 1e-9)
    assert rep.bias_estimate == pytest.approx(1 / 16)


@pytest.mark.gpu
def test_level_sums_reshift(P, ctx):
    """osc_level_sums_reshift moves the running sums to new shifts exactly as if the samples had been
    accumulated there."""
    api = P.api
    prob = api.ProblemSpec(api.CovarianceModel.separable_exponential(1.0, 0.1))
    opt = api.EstimatorOptions(seed=1)
    plan = api.make_level_plan(1, 1 / 8, prob, opt)
    lev = plan.op.device_level(ctx)
    draws = api.LevelDraws()
    lev.sums_reset(0.0, 0.0)
    api.run_level_draws(plan, api.GridSpec.square(8), False, False, prob, opt, 0, 40, draws, ctx=ctx)
    y = draws.q_fine[:40] - draws.q_coarse[:40]
    q = draws.q_fine[:40]
    ky, kq = float(y.mean()), float(q.mean())
    lib = P._lib.lib()
    import ctypes as C
    lib.osc_level_sums_reshift.argtypes = [C.c_void_p, C.c_double, C.c_double]
    assert lib.osc_level_sums_reshift(lev.h, ky, kq) == 0
    s = lev.sums_read()
    want = [40, (y - ky).sum(), ((y - ky) ** 2).sum(), (q - kq).sum(), ((q - kq) ** 2).sum()]
    assert s[0] == 40 and s[5] == ky and s[6] == kq
    assert abs(s[2] - want[2]) <= 1e-12 * want[2] and abs(s[4] - want[4]) <= 1e-10 * want[4]
    assert abs(s[1]) <= 1e-13 * np.abs(y).sum() and abs(s[3]) <= 1e-13 * np.abs(q).sum()


@pytest.mark.gpu
def test_driver_collective_path_on_one_device(P, ctx, monkeypatch):
    """The several-device path of the driver (per-device staging of all levels' sums + one NCCL all-reduce
    per wave) on the one visible device: same decisions and bit-identical moments as the direct read."""
    from paper_2306_13493_b200 import mlmc
    prob, opt = _opts(P, lam=0.1, seed=7, pilot_n=30, l_max=3)
    a = mlmc.mlmc_adaptive(prob, opt, 1 / 8, 4e-3, 2, devices=[0])
    monkeypatch.setenv("OSC_MLMC_FORCE_GROUP", "1")
    b = mlmc.mlmc_adaptive(prob, opt, 1 / 8, 4e-3, 2, devices=[0])
    assert [l.n for l in a.levels] == [l.n for l in b.levels] and a.waves == b.waves
    assert [l.mean_y for l in a.levels] == [l.mean_y for l in b.levels]
    assert [l.var_y for l in a.levels] == [l.var_y for l in b.levels]
    assert a.estimate == b.estimate


def test_driver_struct_layout_matches_header(P, tmp_path):
    """The ctypes mirrors of osc_mlmc_options / osc_mlmc_report / osc_problem have the C layout of
    include/oscfield_b200.h (sizes and the offsets of the last fields), checked with the C compiler."""
    import ctypes as C
    import subprocess
    from paper_2306_13493_b200 import _lib, mlmc
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "oscfield_b200.h"\n'
        'int main(void) { printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(osc_mlmc_options), '
        'offsetof(osc_mlmc_options, spectrum_user), offsetof(osc_mlmc_options, seed), sizeof(osc_mlmc_report), '
        'offsetof(osc_mlmc_report, message), offsetof(osc_mlmc_report, wall_per_sample), sizeof(osc_problem)); '
        'return 0; }\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(_lib.ROOT) + "/include", "-o", str(exe), str(src)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(mlmc.Options), mlmc.Options.spectrum_user.offset, mlmc.Options.seed.offset,
            C.sizeof(mlmc.Report), mlmc.Report.message.offset, mlmc.Report.wall_per_sample.offset,
            C.sizeof(_lib.Problem)]
    assert got == want, (got, want)
