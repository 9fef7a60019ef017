"""ctypes binding of the C-ABI in include/oscfield_b200.h (libosc_b200.so, built in-tree).

The product path has no CPU fallback: if the shared library is missing or cannot be loaded,
importing the package's device API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# OSC_LIB: developer override (A/B builds of the same sources); the default is the in-tree build
LIB_PATH = os.environ.get("OSC_LIB") or os.path.join(HERE, "libosc_b200.so")
HEADER = os.path.join(ROOT, "include", "oscfield_b200.h")
SOURCES = ["csrc/capi.cu", "csrc/ce_sample.cu", "csrc/mgpcg.cu", "csrc/level_setup.cu", "csrc/setup.cpp",
           "csrc/group.cpp", "csrc/driver.cpp"]
DEPS = SOURCES + ["csrc/osc_internal.cuh", "csrc/osc_device.cuh"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
]
OBJ_DIR = os.path.join(HERE, "_build")

OSC_OK, OSC_ERR_CONFIG, OSC_ERR_NUMERICAL, OSC_ERR_SOLVER, OSC_ERR_EMBEDDING, OSC_ERR_CUDA = (
    0, 2, 3, 4, 5, 6)
BC_FLOWCELL, BC_DIRICHLET_ALL = 0, 1
QOI_POINT, QOI_L2, QOI_INTEGRAL, QOI_FLUX = 0, 1, 2, 3
COV_MATERN, COV_SEPARABLE_EXP = 0, 1
COARSE_GALERKIN, COARSE_REDISCRETIZE, COARSE_GALERKIN_LINEAR = 0, 1, 2
DRAW_HAS_COARSE, DRAW_TRUNC_FINE, DRAW_TRUNC_COARSE, DRAW_XI_DEVICE = 1, 2, 4, 8
CE_TRUNCATED, CE_EXP, CE_FINE, CE_COARSE, CE_DEVICE_OUT, CE_XI_DEVICE = 1, 2, 4, 8, 16, 32

# every symbol the header declares (checked by tests/test_abi.py against the header text)
EXPORTS = [
    "osc_ctx_create", "osc_ctx_destroy", "osc_last_error", "osc_ctx_stream", "osc_ctx_synchronize",
    "osc_ctx_set_mem_budget", "osc_ctx_set_profiling", "osc_ctx_profile_only", "osc_ctx_kernel_stats", "osc_ctx_reset_stats",
    "osc_ctx_launch_count", "osc_host_alloc", "osc_host_free", "osc_free", "osc_build_spectrum",
    "osc_build_spectrum_device",
    "osc_level_create", "osc_level_create_device", "osc_level_retruncate", "osc_level_eigenvalues",
    "osc_smoothing_error", "osc_spectrum_save", "osc_spectrum_load", "osc_level_prefetch_xi", "osc_level_destroy", "osc_level_info", "osc_level_draws", "osc_summarize",
    "osc_normals", "osc_ce_sample", "osc_darcy_solve", "osc_qoi",
    "osc_level_sums_reset", "osc_level_sums_read", "osc_ctx_set_history", "osc_ctx_failure_history",
    "osc_group_create", "osc_group_destroy", "osc_group_size", "osc_group_ctx", "osc_group_level_create",
    "osc_group_level_destroy", "osc_group_level_at", "osc_group_level_draws", "osc_group_level_sums_reset",
    "osc_group_level_sums_allreduce", "osc_comm_unique_id", "osc_comm_create", "osc_comm_destroy",
    "osc_comm_allreduce_level_sums", "osc_comm_allgather",
    "osc_level_sums_reshift", "osc_mlmc_adaptive", "osc_mlmc_k_trunc",
]


class Problem(C.Structure):
    """osc_problem (flat DarcyProblem/SolverOptions/QoiSpec)."""
    _fields_ = [
        ("bc", C.c_int), ("forcing", C.c_int), ("forcing_value", C.c_double), ("qoi", C.c_int),
        ("qoi_x", C.c_double), ("qoi_y", C.c_double), ("tol", C.c_double),
        ("max_iter_factor", C.c_int), ("coarse_op", C.c_int),
    ]


def build(verbose: bool = False, force: bool = False) -> str:
    """Compile libosc_b200.so for sm_100a with nvcc (in-tree): one object per source, compiled in
    parallel, then linked. Skipped when the library is newer than every source (force=True rebuilds)."""
    from concurrent.futures import ThreadPoolExecutor
    srcs = [os.path.join(HERE, s) for s in SOURCES]
    deps = [os.path.join(HERE, s) for s in DEPS] + [HEADER]
    if not force and os.path.exists(LIB_PATH):
        t = os.path.getmtime(LIB_PATH)
        if all(os.path.getmtime(d) <= t for d in deps):
            return LIB_PATH
    os.makedirs(OBJ_DIR, exist_ok=True)
    extra = ["-Xptxas", "-v"] if verbose else []

    def compile_one(src):
        obj = os.path.join(OBJ_DIR, os.path.basename(src) + ".o")
        subprocess.run(["nvcc"] + NVCC_FLAGS + extra + ["-c", "-o", obj, src], check=True, cwd=HERE)
        return obj

    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(compile_one, srcs))
    subprocess.run(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB_PATH] + objs +
                   ["-ldl", "-lpthread"], check=True, cwd=HERE)
    return LIB_PATH


_LIB = None


def lib() -> C.CDLL:
    """Load (never silently skip) the CUDA library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                          "(the product path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, dp, ip, i64 = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_int64
    L.osc_last_error.restype = C.c_char_p
    L.osc_ctx_create.argtypes = [ip, C.POINTER(vp)]
    L.osc_ctx_destroy.argtypes = [vp]
    L.osc_ctx_destroy.restype = None
    L.osc_ctx_stream.argtypes = [vp]
    L.osc_ctx_stream.restype = vp
    L.osc_ctx_synchronize.argtypes = [vp]
    L.osc_ctx_set_mem_budget.argtypes = [vp, C.c_size_t]
    L.osc_level_prefetch_xi.argtypes = [vp, vp, i64]
    L.osc_ctx_set_profiling.argtypes = [vp, ip]
    L.osc_ctx_profile_only.argtypes = [vp, C.c_char_p]
    L.osc_ctx_kernel_stats.argtypes = [vp, ip, C.POINTER(C.c_char_p), C.POINTER(i64),
                                       C.POINTER(C.c_double)]
    L.osc_ctx_reset_stats.argtypes = [vp]
    L.osc_ctx_launch_count.argtypes = [vp]
    L.osc_ctx_launch_count.restype = i64
    L.osc_host_alloc.argtypes = [C.c_size_t]
    L.osc_host_alloc.restype = vp
    L.osc_host_free.argtypes = [vp]
    L.osc_host_free.restype = None
    L.osc_free.argtypes = [vp]
    L.osc_free.restype = None
    L.osc_build_spectrum.argtypes = [ip, ip, C.c_double, C.c_double, C.c_double, vp, ip, C.c_double,
                                     C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(vp)]
    L.osc_build_spectrum_device.argtypes = [vp, ip, ip, C.c_double, C.c_double, C.c_double, vp, ip, C.c_double,
                                            C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(vp)]
    L.osc_level_create.argtypes = [vp, ip, ip, vp, i64, C.POINTER(vp)]
    L.osc_level_create_device.argtypes = [vp, ip, ip, C.c_double, C.c_double, C.c_double, vp, ip, C.c_double,
                                          i64, C.POINTER(vp)]
    L.osc_level_retruncate.argtypes = [vp, i64]
    L.osc_level_eigenvalues.argtypes = [vp, vp]
    L.osc_smoothing_error.argtypes = [vp, ip, C.c_uint64, dp, vp]
    L.osc_spectrum_save.argtypes = [C.c_char_p, ip, ip, vp, i64]
    L.osc_spectrum_load.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(i64),
                                    C.POINTER(vp)]
    L.osc_level_destroy.argtypes = [vp]
    L.osc_level_destroy.restype = None
    L.osc_level_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(i64), C.POINTER(i64)]
    L.osc_level_draws.argtypes = [vp, C.POINTER(Problem), C.c_uint64, C.c_uint32, i64, i64, ip, vp,
                                  vp, vp, vp, vp, vp, vp]
    L.osc_summarize.argtypes = [vp, vp, i64, ip, vp]
    L.osc_normals.argtypes = [vp, C.c_uint64, C.c_uint32, C.c_uint64, i64, i64, vp]
    L.osc_ce_sample.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_uint64, i64, ip, vp, vp]
    L.osc_darcy_solve.argtypes = [vp, ip, i64, vp, C.POINTER(Problem), vp, vp, vp, vp, ip]
    L.osc_qoi.argtypes = [vp, ip, i64, vp, vp, C.POINTER(Problem), vp]
    L.osc_level_sums_reset.argtypes = [vp, C.c_double, C.c_double]
    L.osc_level_sums_read.argtypes = [vp, vp]
    L.osc_ctx_set_history.argtypes = [vp, ip]
    L.osc_ctx_failure_history.argtypes = [vp, C.POINTER(i64), vp, ip]
    L.osc_group_create.argtypes = [ip, vp, C.POINTER(vp)]
    L.osc_group_destroy.argtypes = [vp]
    L.osc_group_destroy.restype = None
    L.osc_group_size.argtypes = [vp]
    L.osc_group_ctx.argtypes = [vp, ip]
    L.osc_group_ctx.restype = vp
    L.osc_group_level_create.argtypes = [vp, ip, ip, vp, i64, C.POINTER(vp)]
    L.osc_group_level_destroy.argtypes = [vp]
    L.osc_group_level_destroy.restype = None
    L.osc_group_level_at.argtypes = [vp, ip]
    L.osc_group_level_at.restype = vp
    L.osc_group_level_draws.argtypes = [vp, C.POINTER(Problem), C.c_uint64, C.c_uint32, i64, i64, ip, vp,
                                        vp, vp, vp, vp, vp, vp]
    L.osc_group_level_sums_reset.argtypes = [vp, C.c_double, C.c_double]
    L.osc_group_level_sums_allreduce.argtypes = [vp, vp]
    L.osc_comm_unique_id.argtypes = [vp]
    L.osc_comm_create.argtypes = [vp, ip, ip, vp, C.POINTER(vp)]
    L.osc_comm_destroy.argtypes = [vp]
    L.osc_comm_destroy.restype = None
    L.osc_comm_allreduce_level_sums.argtypes = [vp, vp, vp]
    L.osc_comm_allgather.argtypes = [vp, vp, i64, vp]
    _LIB = L
    return L


def last_error() -> str:
    return lib().osc_last_error().decode()
