"""osc_mlmc_adaptive — the GPU-resident adaptive MLMC driver (include/oscfield_b200.h).

The reference's estimate_adaptive (/root/reference/proj/src/estimators.cpp:289-378) with each allocation
pass run as a wave: all levels that need samples draw at the same time (one context and host thread per
level and device), the level moments stay in HBM as running sums. The control loop is host C++ inside
libosc_b200.so (csrc/driver.cpp); this module only marshals options and the report.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib
from .api import (BC, CovFamily, EstimatorOptions, ProblemSpec, _check, _problem_struct)
from .estimators import LevelStats, MlmcReport

MAX_LEVELS = 26
SPECTRUM_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                          C.POINTER(C.POINTER(C.c_double)))


class Options(C.Structure):
    """osc_mlmc_options."""
    _fields_ = [
        ("family", C.c_int), ("sigma2", C.c_double), ("lambda_", C.c_double), ("nu_or_p", C.c_double),
        ("h0", C.c_double), ("eps", C.c_double), ("initial_levels", C.c_int), ("l_max", C.c_int),
        ("allow_extension", C.c_int), ("seed", C.c_uint64), ("pilot_n", C.c_int),
        ("gamma_model", C.c_double), ("alpha", C.c_double), ("c_alpha", C.c_double), ("c_ratio", C.c_double),
        ("c_alpha_tilde_ratio", C.c_double), ("smoothing", C.c_int), ("use_coarse_s", C.c_int),
        ("lstar_only", C.c_int), ("concurrent_levels", C.c_int), ("spectrum", SPECTRUM_FN),
        ("spectrum_user", C.c_void_p),
    ]


_ARR_I = C.c_int64 * MAX_LEVELS
_ARR_D = C.c_double * MAX_LEVELS


class Report(C.Structure):
    """osc_mlmc_report."""
    _fields_ = [
        ("estimate", C.c_double), ("bias_estimate", C.c_double), ("sampling_error", C.c_double),
        ("total_cost_model", C.c_double), ("total_cost_wall", C.c_double), ("converged", C.c_int),
        ("n_levels", C.c_int), ("passes", C.c_int), ("waves", C.c_int),
        ("n", _ARR_I), ("k_trunc", _ARR_I), ("redrawn", _ARR_I),
        ("mean_y", _ARR_D), ("var_y", _ARR_D), ("mean_q", _ARR_D), ("var_q", _ARR_D), ("h", _ARR_D),
        ("n_real", _ARR_D), ("wall_per_sample", _ARR_D),
        ("setup_s", C.c_double), ("draw_s", C.c_double), ("total_s", C.c_double),
        ("samples_total", C.c_int64), ("gpu_launches", C.c_int64), ("message", C.c_char * 256),
    ]


def _bind():
    L = _lib.lib()
    L.osc_mlmc_adaptive.argtypes = [C.c_int, C.c_void_p, C.POINTER(_lib.Problem), C.POINTER(Options),
                                    C.POINTER(Report)]
    L.osc_mlmc_k_trunc.argtypes = [C.POINTER(Options), C.c_double, C.c_int, C.c_int64]
    L.osc_mlmc_k_trunc.restype = C.c_int64
    return L


def make_options(problem: ProblemSpec, opt: EstimatorOptions, h0: float, eps: float, initial_levels: int = 1,
                 allow_extension: bool = True, concurrent: bool = True) -> Options:
    m = problem.model
    return Options(0 if m.family == CovFamily.Matern else 1, m.sigma2, m.lambda_, m.param, float(h0), float(eps),
                   int(initial_levels), int(opt.l_max), int(allow_extension), int(opt.seed), int(opt.pilot_n),
                   opt.gamma_model, opt.alpha, opt.c_alpha, opt.c_ratio, opt.c_alpha_tilde_ratio,
                   int(opt.smoothing), int(opt.smoothing_use_coarse_s), int(opt.smoothing_lstar_only),
                   int(concurrent), SPECTRUM_FN(), None)


def k_trunc(o: Options, h: float, J: int, s: int) -> int:
    """The truncation count the driver uses on mesh width h (make_level_plan's rule, estimators.cpp:183-194)."""
    return int(_bind().osc_mlmc_k_trunc(C.byref(o), float(h), int(J), int(s)))


class DriverReport(MlmcReport):
    """MlmcReport plus what the driver measured: waves, seconds (setup / draws / total), launches."""
    passes: int = 0
    waves: int = 0
    setup_s: float = 0.0
    draw_s: float = 0.0
    total_s: float = 0.0
    samples_total: int = 0
    gpu_launches: int = 0
    k_trunc: list = []
    redrawn: list = []


def mlmc_adaptive(problem: ProblemSpec, opt: EstimatorOptions, h0: float, eps: float, initial_levels: int = 1, *,
                  n_devices: int = 0, devices: Optional[Sequence[int]] = None, allow_extension: bool = True,
                  concurrent: bool = True,
                  spectrum: Optional[Callable[[int], tuple]] = None) -> DriverReport:
    """mlmc_estimate (estimators.cpp:414-418) on the GPU-resident driver. `spectrum(m) -> (J, eigenvalues)`
    supplies a level's eigenvalues (e.g. the reference's build_operator, so that a truncation mask is
    bit-identical to the reference's); without it the levels are set up on the device."""
    L = _bind()
    o = make_options(problem, opt, h0, eps, initial_levels, allow_extension, concurrent)
    libc = C.CDLL(None)
    libc.malloc.restype = C.c_void_p
    libc.malloc.argtypes = [C.c_size_t]
    keep = None
    if spectrum is not None:
        def cb(_user, m, J_out, s_out, eig_out):
            try:
                J, eig = spectrum(int(m))
                eig = np.ascontiguousarray(eig, dtype=np.float64)
                buf = libc.malloc(eig.nbytes)
                if not buf:
                    return 1
                C.memmove(buf, eig.ctypes.data, eig.nbytes)
                J_out[0] = int(J)
                s_out[0] = eig.size
                eig_out[0] = C.cast(buf, C.POINTER(C.c_double))
                return 0
            except Exception:  # reported by the driver as OSC_ERR_EMBEDDING
                return 1
        keep = SPECTRUM_FN(cb)
        o.spectrum = keep
    ps = _problem_struct(problem, opt.solver)
    rep = Report()
    dev = None
    if devices is not None:
        dev = (C.c_int * len(devices))(*devices)
        n_devices = len(devices)
    _check(L.osc_mlmc_adaptive(int(n_devices), dev, C.byref(ps), C.byref(o), C.byref(rep)))
    out = DriverReport(rep.estimate, [], [], rep.bias_estimate, rep.sampling_error, rep.total_cost_model,
                       rep.total_cost_wall, bool(rep.converged), rep.message.decode())
    for i in range(rep.n_levels):
        out.levels.append(LevelStats(int(rep.n[i]), rep.mean_y[i], rep.var_y[i], rep.mean_q[i], rep.var_q[i],
                                     rep.wall_per_sample[i], rep.n_real[i]))
        out.level_h.append(rep.h[i])
    out.passes, out.waves = rep.passes, rep.waves
    out.setup_s, out.draw_s, out.total_s = rep.setup_s, rep.draw_s, rep.total_s
    out.samples_total, out.gpu_launches = int(rep.samples_total), int(rep.gpu_launches)
    out.k_trunc = [int(rep.k_trunc[i]) for i in range(rep.n_levels)]
    out.redrawn = [int(rep.redrawn[i]) for i in range(rep.n_levels)]
    return out


def mc_adaptive(problem: ProblemSpec, opt: EstimatorOptions, eps: float, h: float, **kw) -> DriverReport:
    """mc_estimate with a fixed mesh (estimators.cpp:398-412): one level, smoothing off, no extension."""
    import dataclasses
    from .api import SmoothingRule
    o = dataclasses.replace(opt, smoothing=SmoothingRule.Off, l_max=0)
    return mlmc_adaptive(problem, o, h, eps, 1, allow_extension=False, **kw)
