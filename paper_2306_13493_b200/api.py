"""Host-side mirror of the reference's sampler / solver / estimator interface
(namespace oscfield, /root/reference/proj/include/oscfield/*.hpp), backed by the sm_100a
C-ABI (include/oscfield_b200.h). Same names, argument meaning and error behaviour:

  GridSpec, CovarianceModel, EmbeddingOperator, build_operator, load_spectrum/save_spectrum
      ← grid.hpp, covariance.hpp, embedding.hpp
  ProblemSpec, QoiSpec, EstimatorOptions, SolverOptions, LevelPlan, make_level_plan,
  run_level_draws, summarize_draws, choose_k_ell, richardson_bias, coarsest_level_bound,
  mc_estimate_fixed_n, mc_estimate, mlmc_estimate, fit_rates
      ← estimators.hpp (host control logic restated from src/estimators.cpp)
  assemble_and_solve / evaluate_qoi (batched) ← fem.hpp

Errors map onto ConfigError / NumericalError / SolverError / EmbeddingError (errors.hpp).
Per-sample work never runs on the CPU: every draw goes through libosc_b200.so.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import struct
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L


# ---- errors (errors.hpp:10-29) ------------------------------------------------------------------
class ConfigError(ValueError):
    """Invalid configuration or arguments (CLI exit code 2)."""


class NumericalError(RuntimeError):
    """Numerical failure at run time (CLI exit code 3)."""


class SolverError(NumericalError):
    def __init__(self, what: str, residual_history=None, status=None):
        super().__init__(what)
        self.residual_history = residual_history
        self.status = status


class EmbeddingError(NumericalError):
    pass


def _check(code: int, **extra):
    if code == L.OSC_OK:
        return
    msg = L.last_error()
    if code == L.OSC_ERR_CONFIG:
        raise ConfigError(msg)
    if code == L.OSC_ERR_SOLVER:
        raise SolverError(msg, **extra)
    if code == L.OSC_ERR_EMBEDDING:
        raise EmbeddingError(msg)
    if code == L.OSC_ERR_NUMERICAL:
        raise NumericalError(msg)
    raise RuntimeError(f"CUDA failure: {msg}")


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---- grid / covariance (grid.hpp, covariance.hpp) -------------------------------------------------
@dataclass(frozen=True)
class GridSpec:
    dim: int
    cells: tuple

    @staticmethod
    def square(m: int) -> "GridSpec":
        if m < 1:
            raise ConfigError("GridSpec: resolution must be >= 1")
        return GridSpec(2, (int(m), int(m)))

    def m(self, i: int = 0) -> int:
        return self.cells[i]

    def nodes(self, i: int = 0) -> int:
        return self.cells[i] + 1

    def node_count(self) -> int:
        return (self.cells[0] + 1) * (self.cells[1] + 1)

    def refines(self, coarse: "GridSpec") -> bool:
        return coarse.dim == self.dim and all(a % b == 0 for a, b in zip(self.cells, coarse.cells))


class CovFamily(enum.IntEnum):
    Matern = L.COV_MATERN
    SeparableExponential = L.COV_SEPARABLE_EXP


@dataclass(frozen=True)
class CovarianceModel:
    family: CovFamily
    sigma2: float
    lambda_: float
    nu: float = 1.0
    p_norm: float = 1.0

    def __post_init__(self):
        if not (self.sigma2 > 0 and math.isfinite(self.sigma2)):
            raise ConfigError("CovarianceModel: sigma2 must be positive")
        if not (self.lambda_ > 0 and math.isfinite(self.lambda_)):
            raise ConfigError("CovarianceModel: lambda must be positive")
        if self.family == CovFamily.Matern and not (self.nu > 0 and math.isfinite(self.nu)):
            raise ConfigError("CovarianceModel: nu must be positive")
        if self.family == CovFamily.SeparableExponential and not (self.p_norm > 0):
            raise ConfigError("CovarianceModel: p must be positive")

    @staticmethod
    def matern(sigma2: float, lam: float, nu: float) -> "CovarianceModel":
        return CovarianceModel(CovFamily.Matern, sigma2, lam, nu, 2.0)

    @staticmethod
    def separable_exponential(sigma2: float, lam: float, p: float = 1.0) -> "CovarianceModel":
        return CovarianceModel(CovFamily.SeparableExponential, sigma2, lam, 1.0, p)

    @property
    def param(self) -> float:
        return self.nu if self.family == CovFamily.Matern else self.p_norm

    def describe(self) -> str:
        if self.family == CovFamily.Matern:
            return f"matern(sigma2={self.sigma2}, lambda={self.lambda_}, nu={self.nu})"
        return f"exponential(sigma2={self.sigma2}, lambda={self.lambda_}, p={self.p_norm})"


# ---- device context -------------------------------------------------------------------------------
class Context:
    """One osc_ctx per device (one host thread drives one GPU, embedding.hpp:24-35)."""

    def __init__(self, device: int = 0):
        self._lib = L.lib()
        h = C.c_void_p()
        _check(self._lib.osc_ctx_create(int(device), C.byref(h)))
        self.h = h.value
        self.device = int(device)

    def close(self):
        if getattr(self, "h", None):
            self._lib.osc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return self._lib.osc_ctx_stream(self.h)

    def synchronize(self):
        _check(self._lib.osc_ctx_synchronize(self.h))

    def set_profiling(self, on: bool):
        _check(self._lib.osc_ctx_set_profiling(self.h, 1 if on else 0))

    def profile_only(self, kernel_class: str | None):
        """Time only `kernel_class` (events around its launches); None times every class."""
        _check(self._lib.osc_ctx_profile_only(self.h, kernel_class.encode() if kernel_class else None))

    def set_mem_budget(self, nbytes: int):
        _check(self._lib.osc_ctx_set_mem_budget(self.h, int(nbytes)))

    def reset_stats(self):
        _check(self._lib.osc_ctx_reset_stats(self.h))

    def kernel_stats(self) -> dict:
        out, i = {}, 0
        name, n, ms = C.c_char_p(), C.c_int64(), C.c_double()
        while self._lib.osc_ctx_kernel_stats(self.h, i, C.byref(name), C.byref(n), C.byref(ms)) == 0:
            out[name.value.decode()] = (n.value, ms.value)
            i += 1
        return out

    @property
    def launch_count(self) -> int:
        return self._lib.osc_ctx_launch_count(self.h)


_CTX: dict = {}


def default_context(device: Optional[int] = None) -> Context:
    if device is None:
        import os
        device = int(os.environ.get("LOCAL_RANK", "0"))
    if device not in _CTX:
        _CTX[device] = Context(device)
    return _CTX[device]


class PinnedBuffer:
    """Page-locked host array (cudaHostAlloc) for overlapped copies."""

    def __init__(self, shape, dtype=np.float64):
        self._lib = L.lib()
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self.ptr = self._lib.osc_host_alloc(max(nbytes, 1))
        if not self.ptr:
            raise MemoryError("cudaHostAlloc failed")
        buf = (C.c_char * max(nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def free(self):
        if self.ptr:
            self.array = None
            self._lib.osc_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ---- embedding operator (embedding.hpp) ------------------------------------------------------------
@dataclass
class BuildOptions:
    tol_spd_factor: float = 1e-12
    padding_fractions: Sequence[float] = (0.5, 1.0, 2.0, 4.0, 8.0)


class EmbeddingOperator:
    """Factorised circulant embedding: eigenvalues λ (length s = n², n = 2(m+J)), the stable
    descending permutation and the truncation count (embedding.hpp:37-104). The device copy
    (√λ full and truncated) is created lazily per context."""

    def __init__(self, grid: GridSpec, padding: int, eigenvalues: np.ndarray, sigma2: float,
                 truncation_k: int = 0):
        self.grid = grid
        self.padding = (int(padding), int(padding))
        self.dims = [2 * (grid.m(0) + padding)] * 2
        self.n = self.dims[0]
        self.s = self.n * self.n
        eig = np.ascontiguousarray(eigenvalues, dtype=np.float64)
        if eig.size != self.s:
            raise ConfigError("EmbeddingOperator: eigenvalue count must equal the embedding size")
        self._eig_full = eig
        self.sigma2 = float(sigma2)
        self.truncation_k = int(truncation_k)
        self._levels = {}

    @staticmethod
    def from_parts(grid: GridSpec, padding, eigenvalues, sigma2) -> "EmbeddingOperator":
        J = padding[0] if isinstance(padding, (tuple, list)) else padding
        return EmbeddingOperator(grid, int(J), eigenvalues, sigma2)

    def perm(self) -> np.ndarray:
        return np.argsort(-self._eig_full, kind="stable")

    @property
    def eigenvalues(self) -> np.ndarray:
        if self.truncation_k == 0:
            return self._eig_full
        e = self._eig_full.copy()
        e[self.perm()[self.s - self.truncation_k:]] = 0.0
        return e

    def truncated(self, k: int) -> "EmbeddingOperator":
        if k < 0 or k >= self.s:
            raise ConfigError("truncated: k must lie in [0, s); at least one mode must survive")
        op = EmbeddingOperator(self.grid, self.padding[0], self._eig_full, self.sigma2, k)
        return op

    def device_level(self, ctx: Optional[Context] = None, k_trunc: Optional[int] = None) -> "DeviceLevel":
        ctx = ctx or default_context()
        k = self.truncation_k if k_trunc is None else int(k_trunc)
        key = (id(ctx), k)
        if key not in self._levels:
            self._levels[key] = DeviceLevel(ctx, self.grid.m(0), self.padding[0], self._eig_full, k)
        return self._levels[key]

    # sample_into + restrict_to, batched: fields on the R-block (fine) / stride-2 (coarse)
    def sample_fields(self, xi: Optional[np.ndarray] = None, *, count: Optional[int] = None,
                      seed: int = 1, ell: int = 0, index0: int = 0, fine: bool = True,
                      coarse: bool = False, exp: bool = False, ctx: Optional[Context] = None):
        lev = self.device_level(ctx, self.truncation_k)
        return lev.sample_fields(xi, count=count, seed=seed, ell=ell, index0=index0, fine=fine,
                                 coarse=coarse, exp=exp, truncated=self.truncation_k > 0)


@dataclass
class SmoothingErrorStats:
    mean: float
    variance: float


def smoothing_error_estimate(op: "EmbeddingOperator", k: int, n_samples: int, seed: int,
                             ctx: Optional[Context] = None, chunk: int = 64) -> SmoothingErrorStats:
    """Monte Carlo estimate of E‖Z − Z̃‖∞ (embedding.cpp:205-228): Z and Z̃ share the device ξ of
    NormalStream(seed, 0, i); Z̃ drops the k smallest eigenvalues. Both fields come from the
    device CE path; the sup-norm and the Welford update run on the host in index order."""
    if n_samples < 2:
        raise ConfigError("smoothing_error_estimate: need at least 2 samples")
    ctx = ctx or default_context()
    m = op.grid.m(0)
    lev = op.device_level(ctx, k)
    mean, m2 = 0.0, 0.0
    for c0 in range(0, n_samples, chunk):
        cnt = min(chunk, n_samples - c0)
        full = lev.sample_fields(None, count=cnt, seed=seed, ell=0, index0=c0, fine=True)
        smooth = lev.sample_fields(None, count=cnt, seed=seed, ell=0, index0=c0, fine=True,
                                   truncated=k > 0)
        sup = np.max(np.abs(full - smooth), axis=1)
        for j, v in enumerate(sup):
            i = c0 + j
            d = v - mean
            mean += d / (i + 1)
            m2 += d * (v - mean)
    return SmoothingErrorStats(mean, m2 / (n_samples - 1))


class DeviceLevel:
    """An osc_level: √λ (full and truncated) resident on one device."""

    def __init__(self, ctx: Context, m: int, J: int, eigenvalues: np.ndarray, k_trunc: int):
        self.ctx = ctx
        self._lib = L.lib()
        eig = np.ascontiguousarray(eigenvalues, dtype=np.float64)
        h = C.c_void_p()
        _check(self._lib.osc_level_create(ctx.h, int(m), int(J), _p(eig), int(k_trunc), C.byref(h)))
        self.h = h.value
        self.m, self.J, self.n, self.s, self.k_trunc = m, J, 2 * (m + J), (2 * (m + J)) ** 2, k_trunc

    def __del__(self):
        try:
            if self.h:
                self._lib.osc_level_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def prefetch_xi(self, xi_next: Optional[np.ndarray], count: Optional[int] = None):
        """osc_level_prefetch_xi: arm the host ξ rows of the NEXT host-ξ draw call on this level
        (copied under the following call's solves). xi_next must be a C-contiguous float64 array
        of at least count·s values (pinned for full overlap) that stays unchanged until that next
        call returns; None disarms."""
        if xi_next is None:
            self._xi_next = None
            _check(self._lib.osc_level_prefetch_xi(self.h, None, 0))
            return
        if xi_next.dtype != np.float64 or not xi_next.flags["C_CONTIGUOUS"]:
            raise ConfigError("prefetch_xi: xi_next must be a C-contiguous float64 array")
        cnt = xi_next.size // self.s if count is None else int(count)
        if cnt < 0 or cnt * self.s > xi_next.size:
            raise ConfigError("prefetch_xi: xi_next holds fewer than count*s values")
        self._xi_next = xi_next  # held until the next prefetch / disarm
        _check(self._lib.osc_level_prefetch_xi(self.h, xi_next.ctypes.data_as(C.c_void_p), cnt))

    def sample_fields(self, xi=None, *, count=None, seed=1, ell=0, index0=0, fine=True, coarse=False,
                      exp=False, truncated=False):
        if xi is not None:
            xi = np.ascontiguousarray(xi, dtype=np.float64).reshape(-1, self.s)
            count = xi.shape[0]
        if count is None:
            raise ConfigError("sample_fields: give xi or count")
        m, mc = self.m, self.m // 2
        f = np.empty((count, (m + 1) ** 2)) if fine else None
        c = np.empty((count, (mc + 1) ** 2)) if coarse else None
        flags = (L.CE_FINE if fine else 0) | (L.CE_COARSE if coarse else 0) | \
                (L.CE_EXP if exp else 0) | (L.CE_TRUNCATED if truncated else 0)
        _check(self._lib.osc_ce_sample(self.h, _p(xi), int(seed), int(ell), int(index0), int(count),
                                       flags, _p(f), _p(c)))
        return (f, c) if (fine and coarse) else (f if fine else c)


def build_operator(grid: GridSpec, model: CovarianceModel,
                   options: BuildOptions = BuildOptions(), *, device: bool = False,
                   ctx: Optional["Context"] = None) -> EmbeddingOperator:
    """build_operator (embedding.cpp:114-151): J = 0, then ceil(f·m) until SPD. device=True builds
    the first row and the spectrum on the GPU (osc_build_spectrum_device; separable exponential
    and Matérn ν = k + ½, k ≤ 3); the host C++ setup is the general path."""
    lib = L.lib()
    fr = np.ascontiguousarray(options.padding_fractions, dtype=np.float64)
    J, s, ptr = C.c_int(), C.c_int64(), C.c_void_p()
    if device:
        ctx = ctx or default_context()
        _check(lib.osc_build_spectrum_device(ctx.h, grid.m(0), int(model.family), model.sigma2,
                                             model.lambda_, model.param, _p(fr), len(fr),
                                             options.tol_spd_factor, C.byref(J), C.byref(s),
                                             C.byref(ptr)))
    else:
        _check(lib.osc_build_spectrum(grid.m(0), int(model.family), model.sigma2, model.lambda_,
                                      model.param, _p(fr), len(fr), options.tol_spd_factor,
                                      C.byref(J), C.byref(s), C.byref(ptr)))
    try:
        eig = np.ctypeslib.as_array((C.c_double * s.value).from_address(ptr.value)).copy()
    finally:
        lib.osc_free(ptr)
    return EmbeddingOperator(grid, J.value, eig, model.sigma2)


def save_spectrum(op: EmbeddingOperator, path: str) -> None:
    """OSC1 dump (embedding.hpp:131-134): "OSC1", u32 d, u32 m[d], u32 J[d], u64 s, s f64."""
    with open(path, "wb") as f:
        f.write(b"OSC1")
        f.write(struct.pack("<I", 2))
        f.write(struct.pack("<II", op.grid.m(0), op.grid.m(1)))
        f.write(struct.pack("<II", op.padding[0], op.padding[1]))
        f.write(struct.pack("<Q", op.s))
        f.write(np.ascontiguousarray(op.eigenvalues, dtype="<f8").tobytes())


def load_spectrum(path: str, sigma2: float) -> EmbeddingOperator:
    """OSC1 load (embedding.cpp:262-294) — the parity-injection format for truncation masks."""
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"OSC1":
        raise ConfigError(f"load_spectrum: bad magic in {path}")
    d = struct.unpack_from("<I", data, 4)[0]
    if d != 2:
        raise ConfigError("load_spectrum: only d = 2 is supported by the device path")
    m0, m1, J0, J1 = struct.unpack_from("<IIII", data, 8)
    s = struct.unpack_from("<Q", data, 24)[0]
    if m0 != m1 or J0 != J1 or s != (2 * (m0 + J0)) * (2 * (m1 + J1)):
        raise ConfigError(f"load_spectrum: inconsistent header in {path}")
    eig = np.frombuffer(data, dtype="<f8", count=s, offset=32)
    if eig.size != s:
        raise ConfigError(f"load_spectrum: truncated file {path}")
    return EmbeddingOperator(GridSpec.square(m0), J0, eig.astype(np.float64), sigma2)


# ---- problem / options (estimators.hpp, fem.hpp) ---------------------------------------------------
class QoiKind(enum.IntEnum):
    Point = L.QOI_POINT
    L2Norm = L.QOI_L2
    Integral = L.QOI_INTEGRAL   # extension (BASELINE config 1)
    Flux = L.QOI_FLUX           # extension (BASELINE configs 3, 5)


class BC(enum.IntEnum):
    FlowCell = L.BC_FLOWCELL
    DirichletAll = L.BC_DIRICHLET_ALL  # extension (BASELINE configs 1, 4)


class Forcing(enum.IntEnum):
    Zero = 0
    Constant = 1


@dataclass
class QoiSpec:
    kind: QoiKind = QoiKind.Point
    x: float = 7.0 / 15.0
    y: float = 7.0 / 15.0


@dataclass
class ProblemSpec:
    model: CovarianceModel
    qoi: QoiSpec = field(default_factory=QoiSpec)
    forcing: Forcing = Forcing.Constant
    forcing_value: float = 1.0
    bc: BC = BC.FlowCell


class CoarseOperator(enum.IntEnum):
    """Multigrid coarse operators and transfers (include/oscfield_b200.h OSC_COARSE_*).

    * Galerkin: operator-dependent (flux-continuous) prolongation with exact Galerkin PᵀAP coarse
      operators. About 2.5× fewer PCG iterations on rough fields.
    * Rediscretize: the reference's scheme, injected-k re-assembly with P1 transfer
      (fem.cpp:144-195, 241-244).
    * GalerkinLinear: P1 transfer with PᵀAP.

    Every mode solves the same fine system to the same tolerance.
    """
    Galerkin = 0
    Rediscretize = 1
    GalerkinLinear = 2


@dataclass
class SolverOptions:
    tol: float = 1e-10
    max_iter_factor: int = 10
    coarse_operator: CoarseOperator = CoarseOperator.Galerkin


class SmoothingRule(enum.IntEnum):
    Off = 0
    HalfSpectrum = 1
    Adaptive = 2


@dataclass
class EstimatorOptions:
    seed: int = 1
    pilot_n: int = 100
    gamma_model: float = 2.0
    alpha: float = 1.0
    c_alpha: float = 1.0
    c_ratio: float = 1.0
    c_alpha_tilde_ratio: float = 1.0
    smoothing: SmoothingRule = SmoothingRule.Off
    smoothing_use_coarse_s: bool = False
    smoothing_lstar_only: bool = False
    l_max: int = 10
    solver: SolverOptions = field(default_factory=SolverOptions)


def _problem_struct(problem: ProblemSpec, solver: SolverOptions) -> L.Problem:
    return L.Problem(int(problem.bc), int(problem.forcing), float(problem.forcing_value),
                     int(problem.qoi.kind), float(problem.qoi.x), float(problem.qoi.y),
                     float(solver.tol), int(solver.max_iter_factor), int(solver.coarse_operator))


# ---- batched FEM stages (fem.hpp) ---------------------------------------------------------------------
def assemble_and_solve(m: int, Z: np.ndarray, problem: ProblemSpec,
                       solver: SolverOptions = SolverOptions(), hist_cap: int = 0,
                       ctx: Optional[Context] = None):
    """Batched assemble_and_solve (fem.cpp:317-400) of log fields Z[count, (m+1)²].
    Returns (u, iters, history|None); raises SolverError like the reference."""
    ctx = ctx or default_context()
    Z = np.ascontiguousarray(Z, dtype=np.float64).reshape(-1, (m + 1) ** 2)
    cnt = Z.shape[0]
    u = np.empty_like(Z)
    it = np.zeros(cnt, dtype=np.int32)
    st = np.zeros(cnt, dtype=np.int32)
    hist = np.zeros((cnt, hist_cap)) if hist_cap > 0 else None
    ps = _problem_struct(problem, solver)
    code = L.lib().osc_darcy_solve(ctx.h, int(m), cnt, _p(Z), C.byref(ps), _p(u), _p(it), _p(st),
                                   _p(hist), int(hist_cap))
    _check(code, residual_history=hist, status=st)
    return u, it, hist


def evaluate_qoi(m: int, u: np.ndarray, problem: ProblemSpec, Z: Optional[np.ndarray] = None,
                 ctx: Optional[Context] = None) -> np.ndarray:
    """Batched evaluate_qoi (estimators.cpp:13-15; fem.cpp:402-436 + extensions)."""
    ctx = ctx or default_context()
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1, (m + 1) ** 2)
    Zc = None if Z is None else np.ascontiguousarray(Z, dtype=np.float64).reshape(u.shape)
    q = np.empty(u.shape[0])
    ps = _problem_struct(problem, SolverOptions())
    _check(L.lib().osc_qoi(ctx.h, int(m), u.shape[0], _p(u), _p(Zc), C.byref(ps), _p(q)))
    return q


# ---- level plans and draws (estimators.cpp) -------------------------------------------------------------
def coarsest_level_bound(model: CovarianceModel) -> float:
    """estimators.cpp:487-494."""
    limit = model.lambda_ if model.family == CovFamily.SeparableExponential else \
        math.sqrt(8.0 * model.nu) * model.lambda_
    h = 1.0
    while h > limit * (1.0 + 1e-12):
        h *= 0.5
    return h


def choose_k_ell(model: CovarianceModel, h: float, padding: int, s: int, alpha: float,
                 c_ratio: float, use_coarse_s: bool = False) -> int:
    """estimators.cpp:239-272."""
    if not alpha > 0:
        raise ConfigError("choose_k_ell: alpha must be positive")
    if not c_ratio > 0:
        raise ConfigError("choose_k_ell: c_ratio must be positive")

    def llround(x):
        return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))

    h_eff = 2.0 * h if use_coarse_s else h
    if model.family == CovFamily.SeparableExponential:
        s_formula = 4.0 / (h_eff * h_eff)
        k_real = s_formula ** ((3.0 - alpha) / 2.0) / (c_ratio + s_formula ** (-(alpha - 1.0) / 2.0))
        return min(max(llround(k_real), 0), s - 1)
    j_eff = 0.5 * padding if use_coarse_s else float(padding)
    half_width = 1.0 / h_eff + j_eff
    s_m = 4.0 * half_width * half_width
    nu = model.nu
    rhs = c_ratio * h_eff ** alpha * half_width

    def residual(k):
        return (s_m - k) ** (-(1.0 + nu) / 2.0) * k - rhs

    lo, hi = 0.0, s_m - 1.0
    if hi <= lo or residual(hi) < 0.0:
        import sys
        print(f"choose_k_ell: no root in (0, s-1) for {model.describe()} at h = {h}; "
              "smoothing disabled on this level", file=sys.stderr)
        return 0
    while hi - lo > 0.5:
        mid = 0.5 * (lo + hi)
        if residual(mid) < 0.0:
            lo = mid
        else:
            hi = mid
    return min(max(llround(0.5 * (lo + hi)), 0), s - 1)


def richardson_bias(mean_diff: float, alpha: float, c_tilde_over_c: float = 1.0,
                    smoothed_extrapolant: bool = False) -> float:
    """estimators.cpp:274-283."""
    if not alpha > 0:
        raise ConfigError("richardson_bias: alpha must be positive")
    denom = (1.0 - c_tilde_over_c * 2.0 ** alpha) if smoothed_extrapolant else (1.0 - 2.0 ** alpha)
    if abs(denom) < 0.1:
        raise NumericalError("richardson_bias: extrapolation denominator below 0.1")
    return abs(mean_diff) / abs(denom)


def _is_power_of_two_inverse(h: float) -> Optional[int]:
    if not (h > 0.0) or h > 1.0:
        return None
    inv = 1.0 / h
    m = int(round(inv))
    if abs(inv - m) > 1e-9 or m < 1 or (m & (m - 1)) != 0:
        return None
    return m


@dataclass
class LevelPlan:
    ell: int
    h: float
    grid: GridSpec
    op: EmbeddingOperator
    op_smoothed: Optional[EmbeddingOperator]
    k_trunc: int = 0


def make_level_plan(ell: int, h0: float, problem: ProblemSpec, opt: EstimatorOptions,
                    operator: Optional[EmbeddingOperator] = None) -> LevelPlan:
    """estimators.cpp:169-198. `operator` injects a prebuilt (e.g. OSC1-loaded) spectrum."""
    m0 = _is_power_of_two_inverse(h0)
    if m0 is None:
        raise ConfigError("make_level_plan: h0 must be a negative power of two")
    if ell < 0 or ell > 24:
        raise ConfigError("make_level_plan: level out of range")
    h = h0 / float(1 << ell)
    m = m0 << ell
    if m > (1 << 16):
        raise ConfigError("make_level_plan: grid too fine")
    grid = GridSpec.square(m)
    op = operator if operator is not None else build_operator(grid, problem.model)
    k = 0
    if opt.smoothing != SmoothingRule.Off:
        resolved = h <= coarsest_level_bound(problem.model) * (1.0 + 1e-12)
        if not (opt.smoothing_lstar_only and resolved):
            if opt.smoothing == SmoothingRule.HalfSpectrum:
                k = op.s // 2
            else:
                k = choose_k_ell(problem.model, h, op.padding[0], op.s, opt.alpha, opt.c_ratio,
                                 opt.smoothing_use_coarse_s)
    k = min(max(k, 0), op.s - 1)
    return LevelPlan(ell, h, grid, op, op.truncated(k) if k > 0 else None, k)


class LevelDraws:
    """Slot-indexed draws of one level (std::vector<LevelDraw>, estimators.hpp:106-110)."""

    def __init__(self):
        self.q_fine = np.zeros(0)
        self.q_coarse = np.zeros(0)
        self.wall = np.zeros(0)
        self.iters_fine = np.zeros(0, dtype=np.int32)
        self.iters_coarse = np.zeros(0, dtype=np.int32)

    def __len__(self):
        return self.q_fine.size

    def resize(self, n: int):
        def grow(a):
            out = np.zeros(n, dtype=a.dtype)
            out[:min(n, a.size)] = a[:n]
            return out
        self.q_fine, self.q_coarse, self.wall = grow(self.q_fine), grow(self.q_coarse), grow(self.wall)
        self.iters_fine, self.iters_coarse = grow(self.iters_fine), grow(self.iters_coarse)

    def clear(self):
        self.resize(0)


def run_level_draws(plan: LevelPlan, coarse_grid: Optional[GridSpec], truncate_fine: bool,
                    truncate_coarse: bool, problem: ProblemSpec, opt: EstimatorOptions, frm: int,
                    to: int, draws: LevelDraws, *, ctx: Optional[Context] = None,
                    xi: Optional[np.ndarray] = None, xi_next: Optional[np.ndarray] = None,
                    dist=None) -> LevelDraws:
    """run_level_draws (estimators.hpp:112-118): samples [frm, to) land in slots [frm, to) of
    `draws`; sample i uses NormalStream(opt.seed, ℓ, i) (or row i-frm of xi). `xi_next` (host
    ξ of the caller's next batch, see DeviceLevel.prefetch_xi) is copied under this call's solves,
    so the next call with that array runs without an exposed H2D copy. With `dist`
    (paper_2306_13493_b200.dist.Shard) the range is split into contiguous per-rank shards and
    the slots are all-gathered, so every rank ends with identical draws."""
    if to < frm:
        raise ConfigError("run_level_draws: to < from")
    if draws.q_fine.size < to:
        draws.resize(to)
    if to == frm:
        return draws
    has_coarse = coarse_grid is not None
    if has_coarse and not plan.grid.refines(coarse_grid):
        raise ConfigError("restrict: target grid is not a nested coarsening")
    if dist is not None:
        return dist.run_level_draws(plan, coarse_grid, truncate_fine, truncate_coarse, problem,
                                    opt, frm, to, draws, ctx=ctx, xi=xi)
    ctx = ctx or default_context()
    lev = plan.op.device_level(ctx, plan.k_trunc)
    cnt = to - frm
    qf, qc = np.empty(cnt), np.empty(cnt)
    itf, itc = np.zeros(cnt, dtype=np.int32), np.zeros(cnt, dtype=np.int32)
    st = np.zeros(cnt, dtype=np.int32)
    flags = (L.DRAW_HAS_COARSE if has_coarse else 0) | \
        (L.DRAW_TRUNC_FINE if truncate_fine else 0) | (L.DRAW_TRUNC_COARSE if truncate_coarse else 0)
    xi_arr = None
    if xi is not None:
        xi_arr = np.ascontiguousarray(xi, dtype=np.float64).reshape(cnt, plan.op.s)
    if xi_next is not None:
        lev.prefetch_xi(xi_next)
    ps = _problem_struct(problem, opt.solver)
    t0 = time.perf_counter()
    code = L.lib().osc_level_draws(lev.h, C.byref(ps), int(opt.seed), int(plan.ell), int(frm),
                                   int(to), flags, _p(xi_arr), _p(qf), _p(qc), _p(itf), _p(itc),
                                   _p(st), None)
    wall = time.perf_counter() - t0
    _check(code, status=st)
    draws.q_fine[frm:to] = qf
    draws.q_coarse[frm:to] = qc if has_coarse else 0.0
    draws.wall[frm:to] = wall / cnt
    draws.iters_fine[frm:to] = itf
    draws.iters_coarse[frm:to] = itc
    return draws


@dataclass
class DrawStats:
    n: int = 0
    mean_y: float = 0.0
    var_y: float = 0.0
    mean_q: float = 0.0
    var_q: float = 0.0
    mean_wall: float = 0.0


def summarize_draws(draws: LevelDraws, has_coarse: bool) -> DrawStats:
    """summarize_draws / moments_of (estimators.cpp:82-101), slot order (C-ABI osc_summarize)."""
    n = len(draws)
    out = np.zeros(5)
    qf = np.ascontiguousarray(draws.q_fine)
    qc = np.ascontiguousarray(draws.q_coarse)
    _check(L.lib().osc_summarize(_p(qf), _p(qc), n, 1 if has_coarse else 0, _p(out)))
    mean_wall = 0.0
    for i, w in enumerate(draws.wall):
        mean_wall += (w - mean_wall) / (i + 1)
    return DrawStats(int(out[0]), out[1], out[2], out[3], out[4], mean_wall)


# ---- estimators (estimators.cpp:103-418) -------------------------------------------------------------------
@dataclass
class LevelStats:
    n: int = 0
    mean_y: float = 0.0
    var_y: float = 0.0
    mean_q: float = 0.0
    var_q: float = 0.0
    cost_wall_per_sample: float = 0.0
    cost_model_per_sample: float = 0.0
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


class _LevelState:
    def __init__(self, plan: LevelPlan, has_coarse: bool):
        self.plan = plan
        self.has_coarse = has_coarse
        self.coarse = GridSpec.square(plan.grid.m(0) // 2) if has_coarse else None
        self.truncate_fine = False
        self.truncate_coarse = False
        self.draws = LevelDraws()
        self.moments = DrawStats()
        self.n_real = 0.0


def _set_mode(st: _LevelState, opt: EstimatorOptions, is_finest: bool):
    """estimators.cpp:114-122."""
    ces = opt.smoothing != SmoothingRule.Off and st.plan.k_trunc > 0
    new_fine, new_coarse = ces and not is_finest, ces
    if (new_fine != st.truncate_fine or new_coarse != st.truncate_coarse) and len(st.draws):
        st.draws.clear()
    st.truncate_fine, st.truncate_coarse = new_fine, new_coarse


def _make_state(ell, h0, problem, opt, is_finest, operators=None) -> _LevelState:
    op = operators.get(ell) if operators else None
    st = _LevelState(make_level_plan(ell, h0, problem, opt, op), ell > 0)
    _set_mode(st, opt, is_finest)
    return st


def _finalize(states, opt, bias, converged, message) -> MlmcReport:
    """estimators.cpp:147-165."""
    rep = MlmcReport(bias_estimate=bias, converged=converged, message=message)
    var_sum = 0.0
    for st in states:
        m = st.moments
        ls = LevelStats(m.n, m.mean_y, m.var_y, m.mean_q, m.var_q, m.mean_wall,
                        st.plan.h ** (-opt.gamma_model), st.n_real)
        rep.levels.append(ls)
        rep.level_h.append(st.plan.h)
        rep.estimate += ls.mean_y
        var_sum += ls.var_y / ls.n if ls.n > 0 else 0.0
        rep.total_cost_model += ls.cost_model_per_sample * ls.n
        rep.total_cost_wall += ls.cost_wall_per_sample * ls.n
    rep.sampling_error = math.sqrt(var_sum)
    return rep


def _estimate_adaptive(problem, opt, h0, eps, initial_levels, allow_extension, *, ctx=None,
                       dist=None, operators=None) -> MlmcReport:
    """estimators.cpp:289-378 over the GPU seam run_level_draws."""
    if not eps > 0:
        raise ConfigError("estimate: eps must be positive")
    eps2_half = 0.5 * eps * eps
    pilot = max(2, opt.pilot_n)
    l_start = max(0, min(initial_levels - 1, opt.l_max))
    states = [_make_state(ell, h0, problem, opt, ell == l_start, operators)
              for ell in range(l_start + 1)]
    message, converged, bias = "", True, 0.0

    def draw(st, have, target):
        run_level_draws(st.plan, st.coarse, st.truncate_fine, st.truncate_coarse, problem, opt,
                        have, target, st.draws, ctx=ctx, dist=dist)

    outer = 0
    while True:
        if outer > 64:
            converged, message = False, "sample allocation did not stabilise"
            break
        outer += 1
        drew = False
        for st in states:
            have = len(st.draws)
            if have < pilot:
                draw(st, have, pilot)
                drew = True
        for st in states:
            st.moments = summarize_draws(st.draws, st.has_coarse)
        sum_cv = sum(math.sqrt(st.plan.h ** (-opt.gamma_model) * max(st.moments.var_y, 0.0))
                     for st in states)
        for st in states:
            c_model = st.plan.h ** (-opt.gamma_model)
            st.n_real = 2.0 / (eps * eps) * sum_cv * math.sqrt(max(st.moments.var_y, 0.0) / c_model)
            target = max(int(math.ceil(st.n_real)), 2)
            have = len(st.draws)
            if target > have:
                draw(st, have, target)
                st.moments = summarize_draws(st.draws, st.has_coarse)
                drew = True
        if drew:
            continue
        finest = states[-1]
        if len(states) == 1:
            bias = opt.c_alpha * finest.plan.h ** opt.alpha
            if not allow_extension or opt.l_max == 0:
                message = "single level: bias taken from the weak-error model"
                break
        else:
            bias = richardson_bias(finest.moments.mean_y, opt.alpha, opt.c_alpha_tilde_ratio,
                                   finest.truncate_coarse and finest.plan.k_trunc > 0)
        if allow_extension and bias * bias > eps2_half:
            if len(states) - 1 >= opt.l_max:
                converged = False
                message = (f"bias {bias} still above target {math.sqrt(eps2_half)} at "
                           f"L_max = {opt.l_max}")
                break
            new_l = len(states)
            states.append(_make_state(new_l, h0, problem, opt, True, operators))
            for st in states[:-1]:
                _set_mode(st, opt, False)
            continue
        break
    rep = _finalize(states, opt, bias, converged, message)
    if rep.sampling_error ** 2 > eps2_half * (1.0 + 1e-9):
        rep.converged = False
        rep.message = (rep.message + "; " if rep.message else "") + "sampling error above target"
    return rep


def mc_estimate_fixed_n(problem: ProblemSpec, opt: EstimatorOptions, grid: GridSpec, n: int, *,
                        ctx=None, dist=None, operator=None) -> MlmcReport:
    """estimators.cpp:382-396 (smoothing forced off)."""
    if n < 2:
        raise ConfigError("mc_estimate_fixed_n: need at least 2 samples")
    import copy
    mc_opt = copy.copy(opt)
    mc_opt.smoothing = SmoothingRule.Off
    st = _make_state(0, 1.0 / grid.m(0), problem, mc_opt, True, {0: operator} if operator else None)
    run_level_draws(st.plan, None, False, False, problem, mc_opt, 0, n, st.draws, ctx=ctx, dist=dist)
    st.moments = summarize_draws(st.draws, False)
    if st.moments.var_y == 0.0:
        raise NumericalError("mc_estimate: sample variance is zero; degenerate input")
    return _finalize([st], mc_opt, opt.c_alpha * (1.0 / grid.m(0)) ** opt.alpha, True,
                     "fixed sample count")


def mc_estimate(problem: ProblemSpec, opt: EstimatorOptions, eps: float,
                fixed_h: Optional[float] = None, **kw) -> MlmcReport:
    """estimators.cpp:398-412."""
    import copy
    if fixed_h is not None:
        h = fixed_h
    else:
        target = (eps / (math.sqrt(2.0) * opt.c_alpha)) ** (1.0 / opt.alpha)
        h = 1.0
        while h >= target:
            h *= 0.5
    mc_opt = copy.copy(opt)
    mc_opt.smoothing = SmoothingRule.Off
    mc_opt.l_max = 0
    return _estimate_adaptive(problem, mc_opt, h, eps, 1, False, **kw)


def mlmc_estimate(problem: ProblemSpec, opt: EstimatorOptions, h0: float, eps: float,
                  initial_levels: int = 1, **kw) -> MlmcReport:
    """estimators.cpp:414-418."""
    if initial_levels < 1:
        raise ConfigError("mlmc_estimate: need at least one level")
    return _estimate_adaptive(problem, opt, h0, eps, initial_levels, True, **kw)


# ---- rate fits (estimators.cpp:420-485) -------------------------------------------------------------------
@dataclass
class RatePoint:
    h: float = 0.0
    mean_abs_y: float = 0.0
    var_y: float = 0.0
    cost: float = 0.0


@dataclass
class RateFit:
    alpha: float = 0.0
    c_alpha: float = 0.0
    beta: float = 0.0
    c_beta: float = 0.0
    gamma: float = 0.0
    c_gamma: float = 0.0


def fit_rates(data: Sequence[RatePoint], warnings: Optional[list] = None) -> RateFit:
    """Least-squares log-log fits of |E Y|, V[Y] and cost against h (estimators.cpp:428-485);
    non-positive points are dropped per series (noted in `warnings`), < 3 survivors is an error."""
    if len(data) < 3:
        raise ConfigError("fit_rates: need at least 3 levels")

    def fit(hs, vs, name):
        xs, ys = [], []
        for h, v in zip(hs, vs):
            if not (v > 0.0) or not math.isfinite(v):
                if warnings is not None:
                    warnings.append(f"fit_rates: dropped non-positive {name} point at h = {h}; ")
                continue
            xs.append(math.log(h))
            ys.append(math.log(v))
        if len(xs) < 3:
            raise ConfigError("fit_rates: fewer than 3 positive points for a series")
        mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
        sxx = sum((x - mx) ** 2 for x in xs)
        sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
        slope = sxy / sxx
        return slope, math.exp(my - slope * mx)

    h = [p.h for p in data]
    a, ca = fit(h, [p.mean_abs_y for p in data], "|mean Y|")
    b, cb = fit(h, [p.var_y for p in data], "var Y")
    g, cg = fit(h, [p.cost for p in data], "cost")
    return RateFit(a, ca, b, cb, -g, cg)
