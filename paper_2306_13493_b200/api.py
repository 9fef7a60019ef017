"""Host-side mirror of the reference's sampler / solver / batch-seam interface
(namespace oscfield, /root/reference/proj/include/oscfield/*.hpp), backed by the sm_100a
C-ABI (include/oscfield_b200.h). Same names, argument meaning and error behaviour:

  GridSpec, CovarianceModel, EmbeddingOperator, build_operator, load_spectrum/save_spectrum
      ← grid.hpp, covariance.hpp, embedding.hpp
  ProblemSpec, QoiSpec, EstimatorOptions, SolverOptions, LevelPlan, make_level_plan,
  run_level_draws, summarize_draws
      ← estimators.hpp (the batch seams :106-128)
  assemble_and_solve / evaluate_qoi (batched) ← fem.hpp
  DeviceGroup / GroupLevel (several GPUs, NCCL), Comm (one process per GPU)

The reference's host control loop (estimate_adaptive, mlmc_estimate, …) is NOT restated here: it
runs as the reference's own C++ over the GPU seam (integration/, Python binding `estimators.py`).

Errors map onto ConfigError / NumericalError / SolverError / EmbeddingError (errors.hpp).
Per-sample work never runs on the CPU: every draw goes through libosc_b200.so.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
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

    def set_history(self, cap: int):
        """osc_ctx_set_history: a failing draw call re-solves its first failing slot with the
        residual history kept, so SolverError carries it (fem.cpp:359-379)."""
        _check(self._lib.osc_ctx_set_history(self.h, int(cap)))

    def failure_history(self):
        """(slot, history ndarray) of the last failing osc_level_draws call, or (-1, None)."""
        slot = C.c_int64(-1)
        n = self._lib.osc_ctx_failure_history(self.h, C.byref(slot), None, 0)
        if n <= 0:
            return -1, None
        h = np.empty(n)
        self._lib.osc_ctx_failure_history(self.h, C.byref(slot), _p(h), n)
        return slot.value, h


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
                             ctx: Optional[Context] = None) -> SmoothingErrorStats:
    """Monte Carlo estimate of E‖Z − Z̃‖∞ (embedding.cpp:205-228) with ξ_i = NormalStream(seed, 0, i);
    Z̃ drops the k smallest eigenvalues. osc_smoothing_error: one CE pass per sample over the dropped
    modes (Z − Z̃ is linear in ξ) with the sup-norm reduced in the column pass's epilogue."""
    if n_samples < 2:
        raise ConfigError("smoothing_error_estimate: need at least 2 samples")
    if k < 0 or k >= op.s:
        raise ConfigError("truncated: k must lie in [0, s); at least one mode must survive")
    lev = op.device_level(ctx or default_context(), k)
    return lev.smoothing_error(n_samples, seed)


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

    @classmethod
    def from_model(cls, ctx: Context, grid: GridSpec, model: "CovarianceModel", k_trunc: int = 0,
                   options: Optional["BuildOptions"] = None) -> "DeviceLevel":
        """build_operator + from_parts + truncated in HBM (osc_level_create_device): the spectrum, the
        SPD test, √λ, the stable descending order and the mask never visit the host."""
        self = cls.__new__(cls)
        self.ctx, self._lib = ctx, L.lib()
        fr = None if options is None else np.ascontiguousarray(options.padding_fractions, dtype=np.float64)
        h = C.c_void_p()
        _check(self._lib.osc_level_create_device(
            ctx.h, grid.m(0), int(model.family), model.sigma2, model.lambda_, model.param, _p(fr),
            0 if fr is None else len(fr), 0.0 if options is None else options.tol_spd_factor, int(k_trunc),
            C.byref(h)))
        self.h = h.value
        m_, J_, n_, s_, k_ = C.c_int(), C.c_int(), C.c_int(), C.c_int64(), C.c_int64()
        _check(self._lib.osc_level_info(self.h, C.byref(m_), C.byref(J_), C.byref(n_), C.byref(s_), C.byref(k_)))
        self.m, self.J, self.n, self.s, self.k_trunc = m_.value, J_.value, n_.value, s_.value, k_.value
        return self

    def retruncate(self, k: int):
        """EmbeddingOperator::truncated(k) from the resident order (device-built levels)."""
        _check(self._lib.osc_level_retruncate(self.h, int(k)))
        self.k_trunc = int(k)

    def eigenvalues(self) -> np.ndarray:
        """The clamped eigenvalues of a device-built level (s doubles, copied to the host)."""
        out = np.empty(self.s)
        _check(self._lib.osc_level_eigenvalues(self.h, out.ctypes.data))
        return out

    def smoothing_error(self, n_samples: int, seed: int, return_sups: bool = False):
        out = (C.c_double * 2)()
        sups = np.empty(n_samples) if return_sups else None
        _check(self._lib.osc_smoothing_error(self.h, int(n_samples), int(seed), out, _p(sups)))
        st = SmoothingErrorStats(out[0], out[1])
        return (st, sups) if return_sups else st

    def __del__(self):
        try:
            if self.h:
                self._lib.osc_level_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def sums_reset(self, shift_y: float = 0.0, shift_q: float = 0.0):
        """osc_level_sums_reset: start the level's running device sums
        [n, Σ(Y−Ky), Σ(Y−Ky)², Σ(q−Kq), Σ(q−Kq)²] (every later draw call adds to them)."""
        _check(self._lib.osc_level_sums_reset(self.h, float(shift_y), float(shift_q)))

    def sums_read(self) -> np.ndarray:
        """[n, Σ(Y−Ky), Σ(Y−Ky)², Σ(q−Kq), Σ(q−Kq)², Ky, Kq] from the device."""
        out = np.zeros(7)
        _check(self._lib.osc_level_sums_read(self.h, _p(out)))
        return out

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
    the first row and the spectrum on the GPU (osc_build_spectrum_device: every model of the host setup,
    Matérn ν up to 64 through a device K_ν)."""
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
    """OSC1 dump (osc_spectrum_save; embedding.cpp:262-271)."""
    eig = np.ascontiguousarray(op.eigenvalues, dtype=np.float64)
    _check(L.lib().osc_spectrum_save(os.fsencode(path), op.grid.m(0), op.padding[0], eig.ctypes.data, eig.size))


def load_spectrum(path: str, sigma2: float) -> EmbeddingOperator:
    """OSC1 load (osc_spectrum_load; embedding.cpp:273-294) — the parity-injection format for
    truncation masks."""
    lib = L.lib()
    m, J, s_, ptr = C.c_int(), C.c_int(), C.c_int64(), C.c_void_p()
    _check(lib.osc_spectrum_load(os.fsencode(path), C.byref(m), C.byref(J), C.byref(s_), C.byref(ptr)))
    try:
        eig = np.ctypeslib.as_array((C.c_double * s_.value).from_address(ptr.value)).copy()
    finally:
        lib.osc_free(ptr)
    return EmbeddingOperator(GridSpec.square(m.value), J.value, eig, sigma2)


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


# ---- level plans and draws (estimators.hpp:34-41,106-128) ------------------------------------------------
@dataclass
class LevelPlan:
    ell: int
    h: float
    grid: GridSpec
    op: EmbeddingOperator
    op_smoothed: Optional[EmbeddingOperator]
    k_trunc: int = 0


def make_level_plan(ell: int, h0: float, problem: ProblemSpec, opt: EstimatorOptions,
                    operator: Optional[EmbeddingOperator] = None, k_trunc: Optional[int] = None) -> LevelPlan:
    """LevelPlan of level ell above h0 (estimators.cpp:169-198): grid m = 2^ell / h0, its embedding
    operator (or the injected `operator`, e.g. OSC1-loaded), and the truncation count: `k_trunc`
    when given, s/2 for SmoothingRule.HalfSpectrum, 0 for Off. The Adaptive rule (choose_k_ell) and
    smoothing_lstar_only belong to the reference's own planner, which runs over the GPU seam
    (paper_2306_13493_b200.estimators)."""
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
    if k_trunc is not None:
        k = int(k_trunc)
    elif opt.smoothing == SmoothingRule.Off:
        k = 0
    elif opt.smoothing == SmoothingRule.HalfSpectrum and not opt.smoothing_lstar_only:
        k = op.s // 2
    else:
        raise ConfigError("make_level_plan: the Adaptive / lstar_only truncation rule is the reference's "
                          "(choose_k_ell): pass k_trunc, or use paper_2306_13493_b200.estimators")
    k = min(max(k, 0), op.s - 1)
    return LevelPlan(ell, h, grid, op, op.truncated(k) if k > 0 else None, k)


def _is_power_of_two_inverse(h: float) -> Optional[int]:
    if not (h > 0.0) or h > 1.0:
        return None
    inv = 1.0 / h
    m = int(round(inv))
    if abs(inv - m) > 1e-9 or m < 1 or (m & (m - 1)) != 0:
        return None
    return m


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
                    dist=None, group: Optional["DeviceGroup"] = None) -> LevelDraws:
    """run_level_draws (estimators.hpp:112-118): samples [frm, to) land in slots [frm, to) of
    `draws`; sample i uses NormalStream(opt.seed, ℓ, i) (or row i-frm of xi). `xi_next` (host
    ξ of the caller's next batch, see DeviceLevel.prefetch_xi) is copied under this call's solves,
    so the next call with that array runs without an exposed H2D copy. With `group` (DeviceGroup,
    one process, several GPUs) or `dist` (paper_2306_13493_b200.dist.Shard, one process per GPU)
    the range is split into contiguous per-device shards; every slot still receives its own
    sample. A non-converged sample raises SolverError carrying its residual history when the
    context has history capture on (Context.set_history)."""
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
    if group is not None:
        return group.run_level_draws(plan, coarse_grid, truncate_fine, truncate_coarse, problem, opt,
                                     frm, to, draws, xi=xi)
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
    if code == L.OSC_ERR_SOLVER:
        _check(code, status=st, residual_history=ctx.failure_history()[1])
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


# ---- several GPUs (osc_group / osc_comm) ------------------------------------------------------------
class DeviceGroup:
    """osc_group: one process drives n devices (one context and one host thread per device, NCCL
    communicators). run_level_draws cuts [from, to) into contiguous per-device chunks (the chunking
    of parallel_samples, estimators.cpp:32-63); the per-level sums are reduced by one NCCL
    all-reduce of device buffers."""

    def __init__(self, n_devices: int, devices: Optional[Sequence[int]] = None):
        self._lib = L.lib()
        dv = None if devices is None else np.ascontiguousarray(devices, dtype=np.int32)
        h = C.c_void_p()
        _check(self._lib.osc_group_create(int(n_devices), _p(dv), C.byref(h)))
        self.h = h.value
        self.n = int(n_devices)
        self._levels = {}

    def close(self):
        if getattr(self, "h", None):
            for gl in self._levels.values():
                gl.close()
            self._levels.clear()
            self._lib.osc_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def level(self, op: EmbeddingOperator, k_trunc: int = 0) -> "GroupLevel":
        key = (id(op), int(k_trunc))
        if key not in self._levels:
            self._levels[key] = GroupLevel(self, op, int(k_trunc))
        return self._levels[key]

    def run_level_draws(self, plan, coarse_grid, truncate_fine, truncate_coarse, problem, opt, frm, to,
                        draws, xi=None, level_sums: Optional[np.ndarray] = None) -> LevelDraws:
        gl = self.level(plan.op, plan.k_trunc)
        cnt = to - frm
        qf, qc = np.empty(cnt), np.empty(cnt)
        itf, itc = np.zeros(cnt, dtype=np.int32), np.zeros(cnt, dtype=np.int32)
        st = np.zeros(cnt, dtype=np.int32)
        has_coarse = coarse_grid is not None
        flags = (L.DRAW_HAS_COARSE if has_coarse else 0) | \
            (L.DRAW_TRUNC_FINE if truncate_fine else 0) | (L.DRAW_TRUNC_COARSE if truncate_coarse else 0)
        xi_arr = None if xi is None else np.ascontiguousarray(xi, dtype=np.float64).reshape(cnt, plan.op.s)
        ps = _problem_struct(problem, opt.solver)
        t0 = time.perf_counter()
        code = self._lib.osc_group_level_draws(gl.h, C.byref(ps), int(opt.seed), int(plan.ell), int(frm), int(to),
                                               flags, _p(xi_arr), _p(qf), _p(qc), _p(itf), _p(itc), _p(st),
                                               _p(level_sums))
        wall = time.perf_counter() - t0
        _check(code, status=st)
        if draws.q_fine.size < to:
            draws.resize(to)
        draws.q_fine[frm:to] = qf
        draws.q_coarse[frm:to] = qc if has_coarse else 0.0
        draws.wall[frm:to] = wall / max(cnt, 1)
        draws.iters_fine[frm:to] = itf
        draws.iters_coarse[frm:to] = itc
        return draws


class GroupLevel:
    """osc_group_level: one osc_level (√λ in HBM) per device of a DeviceGroup."""

    def __init__(self, group: DeviceGroup, op: EmbeddingOperator, k_trunc: int):
        self._lib = group._lib
        h = C.c_void_p()
        eig = np.ascontiguousarray(op._eig_full, dtype=np.float64)
        _check(self._lib.osc_group_level_create(group.h, op.grid.m(0), op.padding[0], _p(eig), int(k_trunc),
                                                C.byref(h)))
        self.h = h.value

    def close(self):
        if self.h:
            self._lib.osc_group_level_destroy(self.h)
            self.h = None

    def sums_reset(self, shift_y: float = 0.0, shift_q: float = 0.0):
        _check(self._lib.osc_group_level_sums_reset(self.h, float(shift_y), float(shift_q)))

    def sums_allreduce(self) -> np.ndarray:
        """NCCL all-reduce of every device's running level sums: [5 sums, Ky, Kq]."""
        out = np.zeros(7)
        _check(self._lib.osc_group_level_sums_allreduce(self.h, _p(out)))
        return out


class Comm:
    """osc_comm: one process per GPU (torchrun). Rank 0 creates the NCCL id (Comm.unique_id()),
    the launcher broadcasts it, every rank builds its Comm on its own Context."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(L.lib().osc_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx: Context, nranks: int, rank: int, uid: bytes):
        self._lib = L.lib()
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(self._lib.osc_comm_create(ctx.h, int(nranks), int(rank), buf, C.byref(h)))
        self.h = h.value
        self.nranks, self.rank = int(nranks), int(rank)

    def close(self):
        if getattr(self, "h", None):
            self._lib.osc_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def allreduce_level_sums(self, level: DeviceLevel) -> np.ndarray:
        out = np.zeros(7)
        _check(self._lib.osc_comm_allreduce_level_sums(self.h, level.h, _p(out)))
        return out

    def allgather(self, local: np.ndarray) -> np.ndarray:
        local = np.ascontiguousarray(local, dtype=np.float64).ravel()
        out = np.empty(local.size * self.nranks)
        _check(self._lib.osc_comm_allgather(self.h, _p(local), local.size, _p(out)))
        return out
