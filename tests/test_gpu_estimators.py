"""The reference's OWN estimators over the GPU seam vs the same estimators on the CPU.

integration/_build/liboscfield_gpu.so is the pristine reference (estimate_adaptive, mlmc_estimate,
mc_estimate_fixed_n: src/estimators.cpp:289-418) with run_level_samples routed to run_level_draws
→ libosc_b200.so. oracle/_ref/libosc_ref.so is the pristine reference on the CPU. Both draw sample
i from NormalStream(seed, ℓ, i) into slot i, both solve to ‖r‖/‖b‖ ≤ 1e-10, so the two runs must take
the SAME decisions (levels, N_ℓ per level, convergence) and agree in every level moment to the QoI
tolerance — far tighter than the sampling confidence intervals north_star asks for.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MOMENT_TOL = 1e-6  # relative to |value| + the level's standard deviation


@pytest.fixture(scope="module")
def E(P, ctx):
    from paper_2306_13493_b200 import estimators as E
    try:
        E.lib()
    except ImportError as e:
        pytest.fail(f"GPU-routed reference build missing: {e}")
    return E


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
    assert bool(gpu.converged) == bool(cpu.converged)


def test_mc_fixed_n_golden(P, E, golden):
    """The reference's mc_estimate_fixed_n over the seam reproduces the golden MC estimate."""
    api = P.api
    prob = api.ProblemSpec(api.CovarianceModel.matern(1.0, 0.1, 0.5), api.QoiSpec(api.QoiKind.L2Norm))
    rep = E.mc_estimate_fixed_n(prob, api.EstimatorOptions(seed=1), 16, 64)
    mean, var = golden["mc16_mean_var"]
    assert abs(rep.levels[0].mean_y - mean) < 1e-8 * abs(mean)
    assert abs(rep.levels[0].var_y - var) < 1e-5 * abs(var)


@pytest.mark.parametrize("case", ["off_point", "cfg3_rule_point", "cfg3_rule_l2"])
def test_mlmc_gpu_vs_cpu_reference(P, E, ref, case):
    """mlmc_estimate, GPU-routed vs CPU: identical N_ℓ and level moments. 'off': smoothing Off,
    sep-exp λ = 0.1, h0 = 1/8. 'cfg3_rule': BASELINE config 3's rule — SmoothingRule::Adaptive with
    smoothing_lstar_only, h0 = 1/16, sep-exp λ = 0.01, flow-cell BCs — at ε = 1e-2 (the reference's
    CPU run of ε = 1e-3 takes hours), point and L2 QoI (the reference has no flux QoI)."""
    import os
    from oracle import oracle as O
    api = P.api
    threads = os.cpu_count() or 1
    if case == "off_point":
        lam, h0, eps, levels, sm, lstar, qk = 0.1, 1.0 / 8, 2e-3, 2, 0, 0, 0
    else:
        lam, h0, eps, levels, sm, lstar, qk = 0.01, 1.0 / 16, 1e-2, 1, 2, 1, (1 if case.endswith("l2") else 0)
    pilot, l_max = 50, 4
    opts = O.RefOpts.make(family=O.SEP_EXP, sigma2=1.0, lam=lam, nu_or_p=1.0, seed=1, pilot_n=pilot,
                          threads=threads, l_max=l_max, smoothing=sm, lstar_only=lstar, qoi_kind=qk)
    cpu = ref.mlmc(opts, h0, eps, levels)
    prob = api.ProblemSpec(api.CovarianceModel.separable_exponential(1.0, lam),
                           api.QoiSpec(api.QoiKind.L2Norm if qk else api.QoiKind.Point))
    opt = api.EstimatorOptions(seed=1, pilot_n=pilot, l_max=l_max, smoothing=api.SmoothingRule(sm),
                               smoothing_lstar_only=bool(lstar))
    gpu = E.mlmc_estimate(prob, opt, h0, eps, levels)
    print(case, "levels", [l.n for l in gpu.levels], "estimate", gpu.estimate, cpu.estimate)
    _same_report(gpu, cpu)


@pytest.mark.parametrize("mode", ["host", "device"])
def test_mlmc_routed_level_setup(P, E, ref, mode):
    """build_operator of the routed estimator taken from this repo's host / GPU setup
    (build_operator_routed): with smoothing Off no truncation mask is involved, so the run must take
    the CPU reference's decisions (identical N_ℓ) and agree in every level moment."""
    import os
    from oracle import oracle as O
    api = P.api
    lam, h0, eps, pilot, l_max = 0.1, 1.0 / 8, 2e-3, 50, 4
    opts = O.RefOpts.make(family=O.SEP_EXP, sigma2=1.0, lam=lam, nu_or_p=1.0, seed=1, pilot_n=pilot,
                          threads=os.cpu_count() or 1, l_max=l_max)
    cpu = ref.mlmc(opts, h0, eps, 2)
    prob = api.ProblemSpec(api.CovarianceModel.separable_exponential(1.0, lam))
    opt = api.EstimatorOptions(seed=1, pilot_n=pilot, l_max=l_max)
    E.set_setup(E.SETUP_HOST if mode == "host" else E.SETUP_DEVICE)
    try:
        gpu = E.mlmc_estimate(prob, opt, h0, eps, 2)
    finally:
        E.set_setup(E.SETUP_REFERENCE)
    _same_report(gpu, cpu)
    with pytest.raises(api.ConfigError):
        E.set_setup(7)


def test_mlmc_group_mode_matches_single_device(P, E):
    """The seam's osc_group path (n_gpus = 1 here; contiguous per-device chunks + NCCL all-reduce of
    the level sums) gives the bit-identical estimate of the single-context path."""
    api = P.api
    prob = api.ProblemSpec(api.CovarianceModel.separable_exponential(1.0, 0.1))
    opt = api.EstimatorOptions(seed=4, pilot_n=40, l_max=2)
    a = E.mlmc_estimate(prob, opt, 1.0 / 8, 4e-3, 2, n_gpus=0)
    b = E.mlmc_estimate(prob, opt, 1.0 / 8, 4e-3, 2, n_gpus=1)
    E.mlmc_estimate(prob, opt, 1.0 / 8, 4e-3, 2, n_gpus=0)  # back to the default for later tests
    assert a.estimate == b.estimate and [l.n for l in a.levels] == [l.n for l in b.levels]
    assert [l.var_y for l in a.levels] == [l.var_y for l in b.levels]


def test_mlmc_extension_qoi_through_reference_loop(P, E, port):
    """Config 3's flux QoI (an extension the reference's QoiSpec cannot name) through the reference's
    own adaptive loop: level 0's mean equals the mean of the oracle port's flux QoIs on the same
    sample indices (the port restates the consistent reaction flux)."""
    api = P.api
    prob = api.ProblemSpec(api.CovarianceModel.separable_exponential(1.0, 0.1), api.QoiSpec(api.QoiKind.Flux))
    opt = api.EstimatorOptions(seed=2, pilot_n=24, l_max=0)
    rep = E.mc_estimate_fixed_n(prob, opt, 16, 24)
    op = api.build_operator(api.GridSpec.square(16), prob.model)
    sl = np.sqrt(np.maximum(op.eigenvalues, 0))
    qf, _, _, _ = port.coupled(16, op.n, sl, None, False, 2, 0, 0, 24, bc=0, qoi=3)
    assert abs(rep.levels[0].mean_y - qf.mean()) <= 1e-7 * abs(qf.mean())
    assert abs(rep.levels[0].var_y - qf.var(ddof=1)) <= 1e-6 * qf.var(ddof=1)
    E.mc_estimate_fixed_n(api.ProblemSpec(prob.model), opt, 16, 4)  # reset the seam's QoI mapping


def test_solver_error_carries_history_through_reference(P, E):
    """A sample that cannot converge within the cap surfaces as the reference's SolverError with
    its residual history (fem.cpp:359-379), through the reference's own estimator and the seam."""
    api = P.api
    prob = api.ProblemSpec(api.CovarianceModel.separable_exponential(1.0, 0.1))
    opt = api.EstimatorOptions(seed=1, solver=api.SolverOptions(max_iter_factor=0))
    with pytest.raises(api.SolverError) as ei:
        E.mc_estimate_fixed_n(prob, opt, 8, 4)
    h = ei.value.residual_history
    assert h is not None and len(h) >= 1 and np.all(np.isfinite(h)) and h[0] > 1e-10


def test_mlmc_estimate_gpu_drop_in(P, E, ref):
    """oscfield::mlmc_estimate_gpu — the reference's mlmc_estimate signature and report around the
    GPU-resident driver, spectra from the reference's own build_operator: under config 3's rule
    (smoothed coarse levels, whose truncation masks depend on the spectrum's bits) it takes the CPU
    reference's decisions and reproduces its level moments."""
    import os
    from oracle import oracle as O
    api = P.api
    lam, h0, eps, pilot, l_max = 0.01, 1.0 / 16, 1e-2, 50, 4
    opts = O.RefOpts.make(family=O.SEP_EXP, sigma2=1.0, lam=lam, nu_or_p=1.0, seed=1, pilot_n=pilot,
                          threads=os.cpu_count() or 1, l_max=l_max, smoothing=2, lstar_only=1, qoi_kind=0)
    cpu = ref.mlmc(opts, h0, eps, 1)
    prob = api.ProblemSpec(api.CovarianceModel.separable_exponential(1.0, lam), api.QoiSpec(api.QoiKind.Point))
    opt = api.EstimatorOptions(seed=1, pilot_n=pilot, l_max=l_max, smoothing=api.SmoothingRule.Adaptive,
                               smoothing_lstar_only=True)
    gpu = E.mlmc_estimate_resident(prob, opt, h0, eps, 1)
    _same_report(gpu, cpu)
    routed = E.mlmc_estimate(prob, opt, h0, eps, 1)
    assert [l.n for l in routed.levels] == [l.n for l in gpu.levels]
