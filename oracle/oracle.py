"""ctypes bindings for the two CPU checkers. TEST INFRASTRUCTURE ONLY.

* ``Ref``    — the PRISTINE reference (/root/reference/proj/src/*.cpp) compiled with our
               shims into oracle/_ref/libosc_ref.so (oracle/Makefile, target ``ref``).
* ``Port``   — our plain-C restatement oracle/osc_oracle.c (target ``oracle``), which also
               carries the BC/QoI extensions the reference lacks.

Neither is used by the product path; they are the checkers the parity tests, smoke()
and the bench's CPU-baseline leg call.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libosc_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libosc_oracle.so")

BC_FLOWCELL, BC_DIRICHLET_ALL = 0, 1
QOI_POINT, QOI_L2, QOI_INTEGRAL, QOI_FLUX = 0, 1, 2, 3
MATERN, SEP_EXP = 0, 1

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def build(ref: bool = True) -> None:
    """Compile the checkers (ref only when /root/reference is present)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_2306_13493_b200", "libosc_b200.so")):
            targets.append("seam_demo")  # pristine reference + seam binding + C-ABI
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class RefOpts(C.Structure):
    _fields_ = [
        ("family", C.c_int), ("sigma2", C.c_double), ("lam", C.c_double), ("nu_or_p", C.c_double),
        ("qoi_kind", C.c_int), ("qoi_x", C.c_double), ("qoi_y", C.c_double),
        ("forcing", C.c_int), ("forcing_value", C.c_double),
        ("seed", C.c_uint64), ("pilot_n", C.c_int), ("threads", C.c_int),
        ("gamma_model", C.c_double), ("alpha", C.c_double), ("c_alpha", C.c_double),
        ("c_ratio", C.c_double), ("c_alpha_tilde_ratio", C.c_double),
        ("smoothing", C.c_int), ("use_coarse_s", C.c_int), ("lstar_only", C.c_int),
        ("l_max", C.c_int), ("tol", C.c_double), ("max_iter_factor", C.c_int),
        ("precond", C.c_int),
    ]

    @classmethod
    def make(cls, family=SEP_EXP, sigma2=1.0, lam=0.3, nu_or_p=1.0, qoi_kind=QOI_POINT,
             qoi_x=7.0 / 15.0, qoi_y=7.0 / 15.0, forcing=1, forcing_value=1.0, seed=1,
             pilot_n=100, threads=1, gamma_model=2.0, alpha=1.0, c_alpha=1.0, c_ratio=1.0,
             c_alpha_tilde_ratio=1.0, smoothing=0, use_coarse_s=0, lstar_only=0, l_max=10,
             tol=1e-10, max_iter_factor=10, precond=1):
        return cls(family, sigma2, lam, nu_or_p, qoi_kind, qoi_x, qoi_y, forcing, forcing_value,
                   seed, pilot_n, threads, gamma_model, alpha, c_alpha, c_ratio,
                   c_alpha_tilde_ratio, smoothing, use_coarse_s, lstar_only, l_max, tol,
                   max_iter_factor, precond)


class RefReport(C.Structure):
    _fields_ = [
        ("estimate", C.c_double), ("bias_estimate", C.c_double), ("sampling_error", C.c_double),
        ("total_cost_model", C.c_double), ("total_cost_wall", C.c_double),
        ("converged", C.c_int), ("n_levels", C.c_int), ("n", C.c_int64 * 32),
        ("mean_y", C.c_double * 32), ("var_y", C.c_double * 32), ("mean_q", C.c_double * 32),
        ("var_q", C.c_double * 32), ("h", C.c_double * 32), ("n_real", C.c_double * 32),
    ]

    def levels(self):
        return [dict(n=self.n[i], mean_y=self.mean_y[i], var_y=self.var_y[i],
                     mean_q=self.mean_q[i], var_q=self.var_q[i], h=self.h[i],
                     n_real=self.n_real[i]) for i in range(self.n_levels)]


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference status {code}: {msg}")
        self.code = code


class Ref:
    """The pristine reference library (oracle/_ref/libosc_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_normals.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_void_p, C.c_int64]
        L.ref_op_s.restype = C.c_int64
        L.ref_op_s.argtypes = [C.c_void_p]
        L.ref_op_padding.argtypes = [C.c_void_p]
        L.ref_op_m.argtypes = [C.c_void_p]
        L.ref_op_free.argtypes = [C.c_void_p]
        L.ref_op_eigenvalues.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_op_perm.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_op_truncated.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]
        L.ref_build_operator.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.POINTER(C.c_void_p)]
        L.ref_load_spectrum.argtypes = [C.c_char_p, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_save_spectrum.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_sample.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_restrict.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.ref_build_first_row.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_double, C.c_void_p]
        L.ref_solve.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int,
                                C.c_int, C.c_void_p]
        L.ref_qoi_point.argtypes = [C.c_int, C.c_void_p, C.c_double, C.c_double, _dp]
        L.ref_qoi_l2norm.argtypes = [C.c_int, C.c_void_p, _dp]
        L.ref_plan_create.argtypes = [C.c_int, C.c_double, C.POINTER(RefOpts), C.POINTER(C.c_void_p)]
        L.ref_plan_free.argtypes = [C.c_void_p]
        L.ref_plan_k_trunc.restype = C.c_int64
        L.ref_plan_k_trunc.argtypes = [C.c_void_p]
        L.ref_plan_m.argtypes = [C.c_void_p]
        L.ref_plan_op.restype = C.c_void_p
        L.ref_plan_op.argtypes = [C.c_void_p]
        L.ref_plan_op_smoothed.restype = C.c_void_p
        L.ref_plan_op_smoothed.argtypes = [C.c_void_p]
        L.ref_coupled_samples.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(RefOpts), C.c_int64, C.c_int64, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        L.ref_mc_fixed_n.argtypes = [C.POINTER(RefOpts), C.c_int, C.c_int64, C.POINTER(RefReport)]
        L.ref_mlmc.argtypes = [C.POINTER(RefOpts), C.c_double, C.c_double, C.c_int,
                               C.POINTER(RefReport)]
        L.ref_choose_k_ell.restype = C.c_int64
        L.ref_choose_k_ell.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                       C.c_int, C.c_int64, C.c_double, C.c_double, C.c_int]
        L.ref_coarsest_level_bound.restype = C.c_double
        L.ref_coarsest_level_bound.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        L.ref_last_history.restype = C.c_int64
        L.ref_last_history.argtypes = [C.c_void_p, C.c_int64]

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, self.L.ref_last_error().decode())

    # RNG
    def philox(self, key, ctr):
        k = (C.c_uint32 * 2)(*key)
        c = (C.c_uint32 * 4)(*ctr)
        o = (C.c_uint32 * 4)()
        self.L.ref_philox_block(k, c, o)
        return list(o)

    def normals(self, seed, level, index, n):
        out = np.empty(n)
        self.L.ref_normals(seed, level, index, _ptr(out), n)
        return out

    # embedding
    class Op:
        def __init__(self, ref, h):
            self.ref, self.h = ref, h
            L = ref.L
            self.s = L.ref_op_s(h)
            self.m = L.ref_op_m(h)
            self.J = L.ref_op_padding(h)
            self.n = 2 * (self.m + self.J)

        def __del__(self):
            try:
                self.ref.L.ref_op_free(self.h)
            except Exception:
                pass

        def eigenvalues(self):
            e = np.empty(self.s)
            self.ref.L.ref_op_eigenvalues(self.h, _ptr(e))
            return e

        def perm(self):
            p = np.empty(self.s, dtype=np.int64)
            self.ref.L.ref_op_perm(self.h, _ptr(p))
            return p

        def truncated(self, k):
            h = C.c_void_p()
            self.ref._check(self.ref.L.ref_op_truncated(self.h, k, C.byref(h)))
            return Ref.Op(self.ref, h.value)

        def sample(self, xi):
            xi = np.ascontiguousarray(xi, dtype=np.float64)
            u = np.empty(self.s)
            self.ref._check(self.ref.L.ref_sample(self.h, _ptr(xi), _ptr(u)))
            return u

        def restrict(self, u, m_target):
            out = np.empty((m_target + 1) ** 2)
            u = np.ascontiguousarray(u, dtype=np.float64)
            self.ref._check(self.ref.L.ref_restrict(self.h, _ptr(u), m_target, _ptr(out)))
            return out

        def save(self, path):
            self.ref._check(self.ref.L.ref_save_spectrum(self.h, path.encode()))

    def build_operator(self, m, family, sigma2, lam, nu_or_p):
        h = C.c_void_p()
        self._check(self.L.ref_build_operator(m, family, sigma2, lam, nu_or_p, C.byref(h)))
        return Ref.Op(self, h.value)

    def load_spectrum(self, path, sigma2):
        h = C.c_void_p()
        self._check(self.L.ref_load_spectrum(path.encode(), sigma2, C.byref(h)))
        return Ref.Op(self, h.value)

    def first_row(self, m, J, family, sigma2, lam, nu_or_p):
        n = 2 * (m + J)
        out = np.empty(n * n)
        self._check(self.L.ref_build_first_row(m, J, family, sigma2, lam, nu_or_p, _ptr(out)))
        return out

    # FEM
    def solve(self, m, Z, forcing=1, forcing_value=1.0, tol=1e-10, max_iter_factor=10, precond=1):
        Z = np.ascontiguousarray(Z, dtype=np.float64)
        u = np.empty((m + 1) ** 2)
        self._check(self.L.ref_solve(m, _ptr(Z), forcing, forcing_value, tol, max_iter_factor,
                                     precond, _ptr(u)))
        return u

    def qoi_point(self, m, u, x=7 / 15, y=7 / 15):
        out = C.c_double()
        self._check(self.L.ref_qoi_point(m, _ptr(np.ascontiguousarray(u)), x, y, C.byref(out)))
        return out.value

    def qoi_l2(self, m, u):
        out = C.c_double()
        self._check(self.L.ref_qoi_l2norm(m, _ptr(np.ascontiguousarray(u)), C.byref(out)))
        return out.value

    def history(self):
        n = self.L.ref_last_history(None, 0)
        out = np.empty(n)
        self.L.ref_last_history(_ptr(out), n)
        return out

    # estimators
    class Plan:
        def __init__(self, ref, h):
            self.ref, self.h = ref, h
            self.k_trunc = ref.L.ref_plan_k_trunc(h)
            self.m = ref.L.ref_plan_m(h)

        def __del__(self):
            try:
                self.ref.L.ref_plan_free(self.h)
            except Exception:
                pass

        def op(self, smoothed=False):
            """Borrowed view of the plan's operator (kept alive by the plan)."""
            h = (self.ref.L.ref_plan_op_smoothed if smoothed else self.ref.L.ref_plan_op)(self.h)
            if not h:
                return None
            o = Ref.Op.__new__(Ref.Op)
            o.ref, o.h = self.ref, h
            L = self.ref.L
            o.s, o.m, o.J = L.ref_op_s(h), L.ref_op_m(h), L.ref_op_padding(h)
            o.n = 2 * (o.m + o.J)
            o.__class__ = _BorrowedOp
            o._plan = self
            return o

    def plan(self, ell, h0, opts: RefOpts):
        h = C.c_void_p()
        self._check(self.L.ref_plan_create(ell, h0, C.byref(opts), C.byref(h)))
        return Ref.Plan(self, h.value)

    def coupled(self, plan, has_coarse, tf, tc, opts, frm, to):
        n = to - frm
        qf, qc, wall = np.empty(n), np.empty(n), np.empty(n)
        self._check(self.L.ref_coupled_samples(plan.h, int(has_coarse), int(tf), int(tc),
                                               C.byref(opts), frm, to, _ptr(qf), _ptr(qc),
                                               _ptr(wall)))
        return qf, qc, wall

    def mc_fixed_n(self, opts, m, n):
        rep = RefReport()
        self._check(self.L.ref_mc_fixed_n(C.byref(opts), m, n, C.byref(rep)))
        return rep

    def mlmc(self, opts, h0, eps, initial_levels=1):
        rep = RefReport()
        self._check(self.L.ref_mlmc(C.byref(opts), h0, eps, initial_levels, C.byref(rep)))
        return rep

    def choose_k_ell(self, family, sigma2, lam, nu_or_p, h, padding, s, alpha=1.0, c_ratio=1.0,
                     use_coarse_s=0):
        return self.L.ref_choose_k_ell(family, sigma2, lam, nu_or_p, h, padding, s, alpha,
                                       c_ratio, use_coarse_s)

    def coarsest_level_bound(self, family, sigma2, lam, nu_or_p):
        return self.L.ref_coarsest_level_bound(family, sigma2, lam, nu_or_p)


class _BorrowedOp(Ref.Op):
    def __del__(self):
        pass


class OoLevel(C.Structure):
    _fields_ = [
        ("m", C.c_int), ("n", C.c_int), ("sqrt_fine", C.c_void_p), ("sqrt_coarse", C.c_void_p),
        ("has_coarse", C.c_int), ("seed", C.c_uint64), ("ell", C.c_uint32),
        ("bc", C.c_int), ("forcing", C.c_int), ("qoi", C.c_int), ("precond", C.c_int),
        ("max_iter_factor", C.c_int), ("forcing_value", C.c_double), ("qx", C.c_double),
        ("qy", C.c_double), ("tol", C.c_double), ("threads", C.c_int),
    ]


class Port:
    """Our plain-C restatement (oracle/_build/libosc_oracle.so)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.L = C.CDLL(path)
        L.oo_normals.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_void_p, C.c_int64]
        L.oo_sample.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oo_restrict.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
        L.oo_solve.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                               C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_int), C.c_void_p,
                               C.c_int, C.POINTER(C.c_int)]
        L.oo_qoi.restype = C.c_double
        L.oo_qoi.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                             C.c_void_p, C.c_int, C.c_double]
        L.oo_coupled.argtypes = [C.POINTER(OoLevel), C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p]
        L.oo_moments.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]

    def philox(self, key, ctr):
        k = (C.c_uint32 * 2)(*key)
        c = (C.c_uint32 * 4)(*ctr)
        o = (C.c_uint32 * 4)()
        self.L.oo_philox_block(k, c, o)
        return list(o)

    def normals(self, seed, level, index, n):
        out = np.empty(n)
        self.L.oo_normals(seed, level, index, _ptr(out), n)
        return out

    def sample(self, n, sqrt_lam, xi):
        u = np.empty(n * n)
        rc = self.L.oo_sample(n, _ptr(np.ascontiguousarray(sqrt_lam)),
                              _ptr(np.ascontiguousarray(xi)), _ptr(u))
        assert rc == 0
        return u

    def restrict(self, n, m, u, m_t):
        out = np.empty((m_t + 1) ** 2)
        self.L.oo_restrict(n, m, _ptr(np.ascontiguousarray(u)), m_t, _ptr(out))
        return out

    def solve(self, m, Z, bc=BC_FLOWCELL, forcing=1, forcing_value=1.0, tol=1e-10,
              max_iter_factor=10, precond=1, hist_cap=0):
        Z = np.ascontiguousarray(Z, dtype=np.float64)
        u = np.empty((m + 1) ** 2)
        it = C.c_int()
        hl = C.c_int()
        hist = np.empty(max(hist_cap, 1))
        rc = self.L.oo_solve(m, _ptr(Z), bc, forcing, forcing_value, tol, max_iter_factor, precond,
                             _ptr(u), C.byref(it), _ptr(hist), hist_cap, C.byref(hl))
        return u, it.value, rc, hist[:min(hl.value, hist_cap)]

    def qoi(self, m, u, bc=BC_FLOWCELL, qoi=QOI_POINT, qx=7 / 15, qy=7 / 15, Z=None, forcing=1,
            forcing_value=1.0):
        if Z is None:
            Z = np.zeros((m + 1) ** 2)
        return self.L.oo_qoi(m, _ptr(np.ascontiguousarray(u)), bc, qoi, qx, qy,
                             _ptr(np.ascontiguousarray(Z)), forcing, forcing_value)

    def coupled(self, m, n, sqrt_fine, sqrt_coarse, has_coarse, seed, ell, frm, to,
                bc=BC_FLOWCELL, forcing=1, forcing_value=1.0, qoi=QOI_POINT, qx=7 / 15,
                qy=7 / 15, tol=1e-10, max_iter_factor=10, precond=1, threads=1, xi_host=None):
        sqrt_fine = np.ascontiguousarray(sqrt_fine, dtype=np.float64)
        sc = sqrt_fine if sqrt_coarse is None else np.ascontiguousarray(sqrt_coarse, dtype=np.float64)
        L = OoLevel(m, n, sqrt_fine.ctypes.data, sc.ctypes.data, int(has_coarse), seed, ell, bc,
                    forcing, qoi, precond, max_iter_factor, forcing_value, qx, qy, tol, threads)
        cnt = to - frm
        qf, qc = np.empty(cnt), np.empty(cnt)
        itf, itc = np.zeros(cnt, dtype=np.int32), np.zeros(cnt, dtype=np.int32)
        xi_p = None if xi_host is None else _ptr(np.ascontiguousarray(xi_host, dtype=np.float64))
        rc = self.L.oo_coupled(C.byref(L), frm, to, xi_p, _ptr(qf), _ptr(qc), _ptr(itf), _ptr(itc))
        if rc != 0:
            raise RuntimeError(f"oracle port status {rc}")
        return qf, qc, itf, itc

    def moments(self, qf, qc, has_coarse):
        out = np.empty(5)
        qf = np.ascontiguousarray(qf, dtype=np.float64)
        qc = np.ascontiguousarray(qc if qc is not None else qf, dtype=np.float64)
        self.L.oo_moments(_ptr(qf), _ptr(qc), len(qf), int(has_coarse), _ptr(out))
        return dict(n=int(out[0]), mean_y=out[1], var_y=out[2], mean_q=out[3], var_q=out[4])
