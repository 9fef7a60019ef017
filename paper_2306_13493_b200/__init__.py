"""paper_2306_13493_b200 — B200-native (sm_100a, fp64) MLMC sample path of arXiv 2306.13493:
circulant-embedding random field → coarse/fine restriction → batched MG-PCG Darcy solve →
QoI → per-level sums, behind the reference's oscfield interface (see api.py) and the C-ABI
include/oscfield_b200.h (libosc_b200.so)."""
from ._lib import build, lib  # noqa: F401
from .api import *  # noqa: F401,F403
from .api import (BC, BuildOptions, Context, CovarianceModel, EmbeddingOperator,  # noqa: F401
                  EstimatorOptions, GridSpec, LevelDraws, ProblemSpec, QoiKind, QoiSpec,
                  SmoothingRule, SolverOptions, assemble_and_solve, build_operator,
                  default_context, evaluate_qoi, load_spectrum, make_level_plan, run_level_draws,
                  save_spectrum, summarize_draws, DeviceGroup, Comm)
