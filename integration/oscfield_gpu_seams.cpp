// Reference-side binding: defines the two batch seams the reference DECLARES but never defines
// (include/oscfield/estimators.hpp:112-118 run_level_draws, :120-128 summarize_draws) on top of
// the B200 C-ABI (include/oscfield_b200.h). Compile this file together with the reference
// library and link libosc_b200.so; the reference's estimators then reach the GPU by calling
// run_level_draws where they call run_level_samples today (src/estimators.cpp:315-316,333-334,388).
//
//   g++ -std=c++20 -I<reference>/include -I<this repo>/include -c oscfield_gpu_seams.cpp
//   ... link with -L<repo>/paper_2306_13493_b200 -losc_b200
#include <chrono>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "oscfield/errors.hpp"
#include "oscfield/estimators.hpp"
#include "oscfield_b200.h"

namespace oscfield {
namespace {

[[noreturn]] void raise(int code, std::vector<double> history = {}) {
  const std::string msg = osc_last_error();
  switch (code) {
    case OSC_ERR_CONFIG: throw ConfigError(msg);
    case OSC_ERR_SOLVER: throw SolverError(msg, std::move(history));
    case OSC_ERR_EMBEDDING: throw EmbeddingError(msg);
    default: throw NumericalError(msg);
  }
}

// One context per host thread (one thread drives one GPU, embedding.hpp:24-35), and one device
// level per (operator, truncation) — the level owns √λ (full and truncated) in HBM.
struct DeviceState {
  osc_ctx* ctx = nullptr;
  std::map<std::pair<const EmbeddingOperator*, std::int64_t>, osc_level*> levels;
  ~DeviceState() {
    for (auto& kv : levels) osc_level_destroy(kv.second);
    if (ctx) osc_ctx_destroy(ctx);
  }
};
thread_local DeviceState g_dev;

osc_level* level_for(const LevelPlan& plan) {
  if (!g_dev.ctx) {
    if (int rc = osc_ctx_create(0, &g_dev.ctx)) raise(rc);
  }
  const auto key = std::make_pair(plan.op.get(), plan.k_trunc);
  auto it = g_dev.levels.find(key);
  if (it != g_dev.levels.end()) return it->second;
  osc_level* lev = nullptr;
  if (int rc = osc_level_create(g_dev.ctx, plan.grid.m(0), plan.op->padding()[0],
                                plan.op->eigenvalues().data(), plan.k_trunc, &lev))
    raise(rc);
  g_dev.levels.emplace(key, lev);
  return lev;
}

}  // namespace

void run_level_draws(const LevelPlan& plan, const GridSpec* coarse_grid, bool truncate_fine,
                     bool truncate_coarse, const ProblemSpec& problem,
                     const EstimatorOptions& opt, std::int64_t from, std::int64_t to,
                     std::vector<LevelDraw>& draws) {
  if (to < from) throw ConfigError("run_level_draws: to < from");
  if (static_cast<std::int64_t>(draws.size()) < to) draws.resize(static_cast<std::size_t>(to));
  if (to == from) return;
  const std::int64_t n = to - from;
  osc_problem p{};
  p.bc = OSC_BC_FLOWCELL;  // the reference's only boundary condition (fem.cpp:28-30)
  p.forcing = problem.forcing == Forcing::Constant ? 1 : 0;
  p.forcing_value = problem.forcing_value;
  p.qoi = problem.qoi.kind == QoiSpec::Kind::L2Norm ? OSC_QOI_L2 : OSC_QOI_POINT;
  p.qoi_x = problem.qoi.x;
  p.qoi_y = problem.qoi.y;
  p.tol = opt.solver.tol;
  p.max_iter_factor = opt.solver.max_iter_factor;  // preconditioner: always geometric MG
  p.coarse_op = OSC_COARSE_GALERKIN;  // same fine system and tolerance; ~2x fewer CG iterations
  const int flags = (coarse_grid ? OSC_DRAW_HAS_COARSE : 0) |
                    (truncate_fine ? OSC_DRAW_TRUNC_FINE : 0) |
                    (truncate_coarse ? OSC_DRAW_TRUNC_COARSE : 0);
  std::vector<double> qf(n), qc(n);
  std::vector<std::int32_t> status(n);
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = osc_level_draws(level_for(plan), &p, opt.seed, static_cast<std::uint32_t>(plan.ell),
                                 from, to, flags, /*xi=*/nullptr, qf.data(), qc.data(), nullptr,
                                 nullptr, status.data(), nullptr);
  if (rc) raise(rc);
  const double wall =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / n;
  for (std::int64_t i = 0; i < n; ++i)
    draws[static_cast<std::size_t>(from + i)] = {qf[i], coarse_grid ? qc[i] : 0.0, wall};
}

DrawStats summarize_draws(const std::vector<LevelDraw>& draws, bool has_coarse) {
  std::vector<double> qf(draws.size()), qc(draws.size());
  double mean_wall = 0.0;
  for (std::size_t i = 0; i < draws.size(); ++i) {
    qf[i] = draws[i].q_fine;
    qc[i] = draws[i].q_coarse;
    mean_wall += (draws[i].wall - mean_wall) / static_cast<double>(i + 1);
  }
  double out[5];
  osc_summarize(qf.data(), qc.data(), static_cast<std::int64_t>(draws.size()), has_coarse ? 1 : 0,
                out);
  DrawStats s;
  s.n = static_cast<std::int64_t>(out[0]);
  s.mean_y = out[1];
  s.var_y = out[2];
  s.mean_q = out[3];
  s.var_q = out[4];
  s.mean_wall = mean_wall;
  return s;
}

}  // namespace oscfield
