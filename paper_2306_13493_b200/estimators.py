"""The reference's OWN estimators — mlmc_estimate / mc_estimate / mc_estimate_fixed_n
(/root/reference/proj/src/estimators.cpp:289-418) — with every sample drawn on the B200.

They live in integration/_build/liboscfield_gpu.so: the pristine reference sources compiled with
the GPU seam (integration/oscfield_gpu_seams.cpp) and the overload that routes the reference's
run_level_samples onto it (integration/route_run_level_samples.hpp). Nothing of the host control
loop is restated here: the adaptive allocation, the level extension, the Richardson bias and the
smoothing rules are the reference's C++; this module only marshals options and the report.

Built by __graft_entry__.build() (make -C integration) where the reference sources exist; the
prebuilt library travels with the repository to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from .api import (BC, ConfigError, EmbeddingError, EstimatorOptions, NumericalError, ProblemSpec,
                  QoiKind, SmoothingRule, SolverError, CovFamily)

LIB_PATH = os.path.join(_lib.ROOT, "integration", "_build", "liboscfield_gpu.so")


class _Opts(C.Structure):
    """oscgpu_opts (integration/estimator_capi.cpp)."""
    _fields_ = [
        ("family", C.c_int), ("sigma2", C.c_double), ("lambda_", C.c_double), ("nu_or_p", C.c_double),
        ("qoi_kind", C.c_int), ("qoi_x", C.c_double), ("qoi_y", C.c_double), ("forcing", C.c_int),
        ("forcing_value", C.c_double), ("seed", C.c_uint64), ("pilot_n", C.c_int), ("threads", C.c_int),
        ("gamma_model", C.c_double), ("alpha", C.c_double), ("c_alpha", C.c_double), ("c_ratio", C.c_double),
        ("c_alpha_tilde_ratio", C.c_double), ("smoothing", C.c_int), ("use_coarse_s", C.c_int),
        ("lstar_only", C.c_int), ("l_max", C.c_int), ("tol", C.c_double), ("max_iter_factor", C.c_int),
    ]


class _Report(C.Structure):
    """oscgpu_report (MlmcReport, estimators.hpp:43-62)."""
    _fields_ = [
        ("estimate", C.c_double), ("bias_estimate", C.c_double), ("sampling_error", C.c_double),
        ("total_cost_model", C.c_double), ("total_cost_wall", C.c_double), ("converged", C.c_int),
        ("n_levels", C.c_int), ("n", C.c_int64 * 32), ("mean_y", C.c_double * 32), ("var_y", C.c_double * 32),
        ("mean_q", C.c_double * 32), ("var_q", C.c_double * 32), ("h", C.c_double * 32),
        ("n_real", C.c_double * 32), ("wall", C.c_double * 32), ("message", C.c_char * 256),
    ]


@dataclass
class LevelStats:
    n: int = 0
    mean_y: float = 0.0
    var_y: float = 0.0
    mean_q: float = 0.0
    var_q: float = 0.0
    cost_wall_per_sample: float = 0.0
    n_real: float = 0.0


@dataclass
class MlmcReport:
    estimate: float = 0.0
    levels: List[LevelStats] = field(default_factory=list)
    level_h: List[float] = field(default_factory=list)
    bias_estimate: float = 0.0
    sampling_error: float = 0.0
    total_cost_model: float = 0.0
    total_cost_wall: float = 0.0
    converged: bool = True
    message: str = ""


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() where the reference sources "
                              "exist (make -C integration)")
        _lib.lib()  # libosc_b200.so first (the routed library links it)
        L = C.CDLL(LIB_PATH)
        L.oscgpu_last_error.restype = C.c_char_p
        L.oscgpu_last_history.restype = C.c_int64
        L.oscgpu_last_history.argtypes = [C.c_void_p, C.c_int64]
        L.oscgpu_configure.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int]
        L.oscgpu_set_setup.argtypes = [C.c_int]
        L.oscgpu_mlmc_estimate.argtypes = [C.POINTER(_Opts), C.c_double, C.c_double, C.c_int, C.POINTER(_Report)]
        L.oscgpu_mlmc_estimate_resident.argtypes = [C.POINTER(_Opts), C.c_double, C.c_double, C.c_int, C.c_int,
                                                    C.POINTER(_Report)]
        L.oscgpu_mc_estimate.argtypes = [C.POINTER(_Opts), C.c_double, C.c_double, C.POINTER(_Report)]
        L.oscgpu_mc_estimate_fixed_n.argtypes = [C.POINTER(_Opts), C.c_int, C.c_int64, C.POINTER(_Report)]
        L.oscgpu_coarsest_level_bound.restype = C.c_double
        L.oscgpu_coarsest_level_bound.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        _LIB = L
    return _LIB


SETUP_REFERENCE, SETUP_HOST, SETUP_DEVICE = 0, 1, 2


def set_setup(mode: int) -> None:
    """Level setup of the routed estimator (integration/oscfield_gpu_seams.cpp build_operator_routed):
    SETUP_REFERENCE — the reference's own build_operator (default: same spectrum bits, hence the same
    truncation mask as the CPU reference); SETUP_HOST / SETUP_DEVICE — this repo's threaded host setup /
    the GPU setup feeding EmbeddingOperator::from_parts (~10 s → < 1 s per estimate at n = 4096)."""
    if lib().oscgpu_set_setup(int(mode)):
        raise ConfigError("oscgpu_set_setup: mode must be 0, 1 or 2")


def _configure(problem: ProblemSpec, n_gpus: int) -> None:
    """Seam settings for one estimate: n_gpus > 0 draws every batch over an osc_group of n_gpus devices
    (0: the calling thread's device). The all-Dirichlet BC and the ∫u / outflow-flux QoIs are extensions
    the reference's ProblemSpec cannot express; they are handed to the seam here, while the reference
    sees flow-cell + Point (its QoI kind is then only a placeholder)."""
    bc = -1 if problem.bc == BC.FlowCell else int(problem.bc)
    qoi = -1 if problem.qoi.kind in (QoiKind.Point, QoiKind.L2Norm) else int(problem.qoi.kind)
    if lib().oscgpu_configure(int(n_gpus), None, bc, qoi):
        raise ConfigError("oscgpu_configure: bad arguments")


def _opts(problem: ProblemSpec, opt: EstimatorOptions) -> _Opts:
    m = problem.model
    q = problem.qoi.kind
    return _Opts(0 if m.family == CovFamily.Matern else 1, m.sigma2, m.lambda_, m.param,
                 1 if q == QoiKind.L2Norm else 0, problem.qoi.x, problem.qoi.y, int(problem.forcing),
                 problem.forcing_value, int(opt.seed), int(opt.pilot_n), 0, opt.gamma_model, opt.alpha,
                 opt.c_alpha, opt.c_ratio, opt.c_alpha_tilde_ratio, int(opt.smoothing),
                 int(opt.smoothing_use_coarse_s), int(opt.smoothing_lstar_only), int(opt.l_max),
                 opt.solver.tol, int(opt.solver.max_iter_factor))


def _run(fn, *args) -> MlmcReport:
    rep = _Report()
    rc = fn(*args, C.byref(rep))
    if rc:
        msg = lib().oscgpu_last_error().decode()
        if rc == -2:
            raise ConfigError(msg)
        if rc == -4:
            n = lib().oscgpu_last_history(None, 0)
            h = np.empty(max(n, 0))
            if n > 0:
                lib().oscgpu_last_history(h.ctypes.data_as(C.c_void_p), n)
            raise SolverError(msg, residual_history=h)
        if rc == -5:
            raise EmbeddingError(msg)
        raise NumericalError(msg)
    out = MlmcReport(rep.estimate, [], [], rep.bias_estimate, rep.sampling_error, rep.total_cost_model,
                     rep.total_cost_wall, bool(rep.converged), rep.message.decode())
    for i in range(rep.n_levels):
        out.levels.append(LevelStats(int(rep.n[i]), rep.mean_y[i], rep.var_y[i], rep.mean_q[i], rep.var_q[i],
                                     rep.wall[i], rep.n_real[i]))
        out.level_h.append(rep.h[i])
    return out


def mlmc_estimate(problem: ProblemSpec, opt: EstimatorOptions, h0: float, eps: float,
                  initial_levels: int = 1, n_gpus: int = 0) -> MlmcReport:
    """The reference's mlmc_estimate (estimators.cpp:414-418 → estimate_adaptive :289-378)."""
    _configure(problem, n_gpus)
    o = _opts(problem, opt)
    return _run(lib().oscgpu_mlmc_estimate, C.byref(o), float(h0), float(eps), int(initial_levels))


def mlmc_estimate_resident(problem: ProblemSpec, opt: EstimatorOptions, h0: float, eps: float,
                           initial_levels: int = 1, n_gpus: int = 0) -> MlmcReport:
    """oscfield::mlmc_estimate_gpu (integration/oscfield_gpu_seams.cpp): the reference's ProblemSpec /
    EstimatorOptions / MlmcReport around the GPU-resident driver osc_mlmc_adaptive, with the levels'
    spectra from the routed build_operator (set_setup)."""
    _configure(problem, 0)
    o = _opts(problem, opt)
    return _run(lib().oscgpu_mlmc_estimate_resident, C.byref(o), float(h0), float(eps), int(initial_levels),
                int(n_gpus))


def mc_estimate(problem: ProblemSpec, opt: EstimatorOptions, eps: float, fixed_h: Optional[float] = None,
                n_gpus: int = 0) -> MlmcReport:
    """The reference's mc_estimate (estimators.cpp:398-412)."""
    _configure(problem, n_gpus)
    o = _opts(problem, opt)
    return _run(lib().oscgpu_mc_estimate, C.byref(o), float(eps), float(fixed_h or 0.0))


def mc_estimate_fixed_n(problem: ProblemSpec, opt: EstimatorOptions, m: int, n: int,
                        n_gpus: int = 0) -> MlmcReport:
    """The reference's mc_estimate_fixed_n (estimators.cpp:382-396) on the m×m grid."""
    _configure(problem, n_gpus)
    o = _opts(problem, opt)
    return _run(lib().oscgpu_mc_estimate_fixed_n, C.byref(o), int(m), int(n))


def coarsest_level_bound(model) -> float:
    """The reference's coarsest_level_bound (estimators.cpp:487-494): the largest h = 2^-k that resolves
    the correlation length (the standard-CE coarsest mesh of BASELINE config 5)."""
    return lib().oscgpu_coarsest_level_bound(0 if model.family == CovFamily.Matern else 1, model.sigma2,
                                             model.lambda_, model.param)
