// Reference-side binding: defines the two batch seams the reference DECLARES but never defines
// (include/oscfield/estimators.hpp:112-118 run_level_draws, :120-128 summarize_draws) on top of
// the B200 C-ABI (include/oscfield_b200.h), plus the overload that routes the reference's own
// estimator loop onto them (integration/route_run_level_samples.hpp). Compile this file together
// with the reference library and link libosc_b200.so; the reference's estimators then draw every
// sample on the GPU (integration/Makefile builds exactly that: the pristine sources + this file).
//
//   g++ -std=c++20 -I<reference>/include -I<this repo>/include -c oscfield_gpu_seams.cpp
//   ... link with -L<repo>/paper_2306_13493_b200 -losc_b200
//
// Devices. By default the seam drives the calling thread's current CUDA device (or OSC_DEVICE /
// LOCAL_RANK when set): one context per host thread, as one SampleWorkspace per worker
// (embedding.hpp:24-35). oscfield_gpu_configure(n, ...) (or OSC_SEAM_GPUS=n) switches to an
// osc_group over n devices: each batch is cut into contiguous per-device chunks (the chunking of
// parallel_samples, estimators.cpp:32-63), one host thread per GPU, slot i = sample i on any count.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "oscfield/errors.hpp"
#include "oscfield/estimators.hpp"
#include "oscfield_b200.h"

namespace oscfield {
EmbeddingOperator build_operator_routed(const GridSpec& grid, const CovarianceModel& model,
                                        const BuildOptions& options);
MlmcReport mlmc_estimate_gpu(const ProblemSpec& problem, const EstimatorOptions& opt, double h0, double eps,
                             int initial_levels = 1, int n_gpus = 0);
namespace {

// cap of the residual history a SolverError carries (the failing slot is re-solved with it kept)
constexpr int kHistoryCap = 1 << 16;

[[noreturn]] void raise(int code, osc_ctx* ctx = nullptr) {
  const std::string msg = osc_last_error();
  switch (code) {
    case OSC_ERR_CONFIG: throw ConfigError(msg);
    case OSC_ERR_SOLVER: {
      std::vector<double> hist;
      if (ctx) {
        std::int64_t slot = -1;
        const int n = osc_ctx_failure_history(ctx, &slot, nullptr, 0);
        if (n > 0) {
          hist.resize(static_cast<std::size_t>(n));
          osc_ctx_failure_history(ctx, &slot, hist.data(), n);
        }
      }
      throw SolverError(msg, std::move(hist));
    }
    case OSC_ERR_EMBEDDING: throw EmbeddingError(msg);
    default: throw NumericalError(msg);
  }
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Device level per (operator, truncation). The entry holds a weak_ptr to the operator, so a freed
// plan whose successor is allocated at the same address is never mistaken for it, and the levels of
// expired operators (their √λ in HBM) are destroyed on the next lookup.
template <typename Lev>
struct LevelCache {
  struct Entry {
    std::weak_ptr<const EmbeddingOperator> op;
    Lev* lev = nullptr;
  };
  std::map<std::pair<const EmbeddingOperator*, std::int64_t>, Entry> map;
  template <typename Destroy, typename Create>
  Lev* get(const LevelPlan& plan, Destroy&& destroy, Create&& create) {
    for (auto it = map.begin(); it != map.end();) {
      if (it->second.op.expired()) {
        destroy(it->second.lev);
        it = map.erase(it);
      } else {
        ++it;
      }
    }
    const auto key = std::make_pair(plan.op.get(), plan.k_trunc);
    auto it = map.find(key);
    if (it != map.end() && it->second.op.lock() == plan.op) return it->second.lev;
    if (it != map.end()) {
      destroy(it->second.lev);
      map.erase(it);
    }
    Lev* lev = create();
    map.emplace(key, Entry{plan.op, lev});
    return lev;
  }
  template <typename Destroy>
  void clear(Destroy&& destroy) {
    for (auto& kv : map) destroy(kv.second.lev);
    map.clear();
  }
};

// single-device mode: one context per host thread
struct ThreadState {
  osc_ctx* ctx = nullptr;
  LevelCache<osc_level> levels;
  ~ThreadState() {
    levels.clear([](osc_level* l) { osc_level_destroy(l); });
    if (ctx) osc_ctx_destroy(ctx);
  }
};
thread_local ThreadState g_thread;

// group mode: one process-wide group
struct GroupState {
  std::mutex mu;
  int n_gpus = 0;  // 0: not configured (single device)
  std::vector<int> devices;
  osc_group* group = nullptr;
  LevelCache<osc_group_level> levels;
  int bc = -1, qoi = -1;  // extension overrides (-1: the reference's own BC / QoI mapping)
  int setup_mode = -1;    // build_operator_routed: -1 = OSC_SEAM_SETUP, 0 reference, 1 host, 2 device
  ~GroupState() { reset(); }
  void reset() {
    levels.clear([](osc_group_level* l) { osc_group_level_destroy(l); });
    if (group) osc_group_destroy(group);
    group = nullptr;
  }
};
GroupState& group_state() {
  static GroupState g;
  static std::once_flag once;
  std::call_once(once, [] { g.n_gpus = env_int("OSC_SEAM_GPUS", 0); });
  return g;
}

osc_ctx* thread_ctx() {
  if (!g_thread.ctx) {
    const int dev = env_int("OSC_DEVICE", env_int("LOCAL_RANK", -1));  // -1: current CUDA device
    if (int rc = osc_ctx_create(dev, &g_thread.ctx)) raise(rc);
    osc_ctx_set_history(g_thread.ctx, kHistoryCap);
  }
  return g_thread.ctx;
}

osc_problem problem_of(const ProblemSpec& problem, const EstimatorOptions& opt, const GroupState& gs) {
  osc_problem p{};
  p.bc = gs.bc >= 0 ? gs.bc : OSC_BC_FLOWCELL;  // the reference's only BC (fem.cpp:28-30)
  p.forcing = problem.forcing == Forcing::Constant ? 1 : 0;
  p.forcing_value = problem.forcing_value;
  p.qoi = gs.qoi >= 0 ? gs.qoi : (problem.qoi.kind == QoiSpec::Kind::L2Norm ? OSC_QOI_L2 : OSC_QOI_POINT);
  p.qoi_x = problem.qoi.x;
  p.qoi_y = problem.qoi.y;
  p.tol = opt.solver.tol;
  p.max_iter_factor = opt.solver.max_iter_factor;  // preconditioner: always geometric MG
  p.coarse_op = OSC_COARSE_GALERKIN;  // same fine system and tolerance; ~2.5x fewer CG iterations
  return p;
}

}  // namespace

void run_level_draws(const LevelPlan& plan, const GridSpec* coarse_grid, bool truncate_fine,
                     bool truncate_coarse, const ProblemSpec& problem,
                     const EstimatorOptions& opt, std::int64_t from, std::int64_t to,
                     std::vector<LevelDraw>& draws) {
  if (to < from) throw ConfigError("run_level_draws: to < from");
  if (static_cast<std::int64_t>(draws.size()) < to) draws.resize(static_cast<std::size_t>(to));
  if (to == from) return;
  if (coarse_grid && !plan.grid.refines(*coarse_grid))
    throw ConfigError("restrict: target grid is not a nested coarsening");
  const std::int64_t n = to - from;
  GroupState& gs = group_state();
  const osc_problem p = problem_of(problem, opt, gs);
  const int flags = (coarse_grid ? OSC_DRAW_HAS_COARSE : 0) |
                    (truncate_fine ? OSC_DRAW_TRUNC_FINE : 0) |
                    (truncate_coarse ? OSC_DRAW_TRUNC_COARSE : 0);
  std::vector<double> qf(n), qc(n);
  std::vector<std::int32_t> status(n);
  const int m = plan.grid.m(0), J = plan.op->padding()[0];
  const double* eig = plan.op->eigenvalues().data();
  const auto t0 = std::chrono::steady_clock::now();
  if (gs.n_gpus > 0) {
    std::lock_guard<std::mutex> lk(gs.mu);
    if (!gs.group) {
      if (int rc = osc_group_create(gs.n_gpus, gs.devices.empty() ? nullptr : gs.devices.data(), &gs.group))
        raise(rc);
      for (int i = 0; i < gs.n_gpus; ++i) osc_ctx_set_history(osc_group_ctx(gs.group, i), kHistoryCap);
    }
    osc_group_level* lev = gs.levels.get(
        plan, [](osc_group_level* l) { osc_group_level_destroy(l); },
        [&] {
          osc_group_level* l = nullptr;
          if (int rc = osc_group_level_create(gs.group, m, J, eig, plan.k_trunc, &l)) raise(rc);
          return l;
        });
    const int rc = osc_group_level_draws(lev, &p, opt.seed, static_cast<std::uint32_t>(plan.ell), from, to,
                                         flags, /*xi=*/nullptr, qf.data(), qc.data(), nullptr, nullptr,
                                         status.data(), nullptr);
    if (rc) {
      osc_ctx* failed = nullptr;  // the device whose shard holds the first failing slot
      for (int i = 0; i < gs.n_gpus && !failed; ++i) {
        std::int64_t slot = -1;
        if (osc_ctx_failure_history(osc_group_ctx(gs.group, i), &slot, nullptr, 0) > 0) failed = osc_group_ctx(gs.group, i);
      }
      raise(rc, failed);
    }
  } else {
    osc_ctx* ctx = thread_ctx();
    osc_level* lev = g_thread.levels.get(
        plan, [](osc_level* l) { osc_level_destroy(l); },
        [&] {
          osc_level* l = nullptr;
          if (int rc = osc_level_create(ctx, m, J, eig, plan.k_trunc, &l)) raise(rc);
          return l;
        });
    const int rc = osc_level_draws(lev, &p, opt.seed, static_cast<std::uint32_t>(plan.ell), from, to, flags,
                                   /*xi=*/nullptr, qf.data(), qc.data(), nullptr, nullptr, status.data(), nullptr);
    if (rc) raise(rc, ctx);
  }
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

// Level setup of the routed estimator. integration/Makefile compiles the pristine estimators.cpp
// with -Dbuild_operator=build_operator_routed, so make_level_plan (estimators.cpp:181) lands here.
// Mode 0 (default) is the reference's own build_operator (bit-identical spectrum, hence the same
// truncation mask as the CPU reference: the parity tests). Modes 1 / 2 take the spectrum from this
// repo's threaded host setup / from the GPU (osc_build_spectrum[_device]: same padding schedule, SPD
// test and clamp, eigenvalues equal to rounding) and hand it to EmbeddingOperator::from_parts — at
// n = 4096 the reference's single-threaded first row + FFT take ~10 s per estimate, these < 1 s.
EmbeddingOperator build_operator_routed(const GridSpec& grid, const CovarianceModel& model,
                                        const BuildOptions& options) {
  static const int env_mode = env_int("OSC_SEAM_SETUP", 0);
  const int mode = group_state().setup_mode >= 0 ? group_state().setup_mode : env_mode;
  if (mode == 0 || grid.dim() != 2 || grid.m(0) != grid.m(1)) return build_operator(grid, model, options);
  const int family = model.family() == CovFamily::Matern ? OSC_COV_MATERN : OSC_COV_SEPARABLE_EXP;
  const double nu_or_p = family == OSC_COV_MATERN ? model.nu() : model.p_norm();
  int J = 0;
  std::int64_t s = 0;
  double* eig = nullptr;
  const int rc = mode == 2 ? osc_build_spectrum_device(thread_ctx(), grid.m(0), family, model.sigma2(), model.lambda(),
                                                       nu_or_p, options.padding_fractions.data(),
                                                       static_cast<int>(options.padding_fractions.size()),
                                                       options.tol_spd_factor, &J, &s, &eig)
                           : osc_build_spectrum(grid.m(0), family, model.sigma2(), model.lambda(), nu_or_p,
                                                options.padding_fractions.data(),
                                                static_cast<int>(options.padding_fractions.size()),
                                                options.tol_spd_factor, &J, &s, &eig);
  if (rc) raise(rc);
  std::vector<double> ev(eig, eig + s);
  osc_free(eig);
  return EmbeddingOperator::from_parts(grid, {J, J}, std::move(ev), model.sigma2());
}

// The reference's estimators call the file-local run_level_samples (estimators.cpp:315-316,333-334,
// 388) with a non-const LevelPlan; this overload (declared by route_run_level_samples.hpp) is the
// better match there and forwards to the GPU seam. Same arguments, same slot contract.
void run_level_samples(LevelPlan& plan, const GridSpec* coarse_grid, bool truncate_fine, bool truncate_coarse,
                       const ProblemSpec& problem, const EstimatorOptions& opt, std::int64_t from,
                       std::int64_t to, std::vector<LevelDraw>& draws) {
  draws.resize(static_cast<std::size_t>(to));  // run_level_samples' own contract (estimators.cpp:69)
  run_level_draws(plan, coarse_grid, truncate_fine, truncate_coarse, problem, opt, from, to, draws);
}

// mlmc_estimate (estimators.hpp; estimators.cpp:414-418) on the GPU-resident driver
// (osc_mlmc_adaptive, include/oscfield_b200.h): same arguments and report type as the reference's
// mlmc_estimate, so a caller switches by name. All levels of an allocation pass draw concurrently and
// the level moments stay in HBM; the levels' spectra come from the routed build_operator (the
// reference's own by default, so truncation masks match the CPU reference bit for bit; modes 1 / 2 of
// oscfield_gpu_set_setup hand the driver this repo's host spectrum or let it build them on the
// device). n_gpus = 0 draws on the calling thread's device, n > 0 over devices 0..n-1.
namespace {
struct SpectrumSource {
  const CovarianceModel* model;
};
extern "C" int oscfield_gpu_spectrum_cb(void* user, int m, int* J, std::int64_t* s, double** eig) {
  try {
    const auto* src = static_cast<const SpectrumSource*>(user);
    const EmbeddingOperator op = build_operator_routed(GridSpec::square(m), *src->model, BuildOptions{});
    *J = op.padding()[0];
    *s = op.s();
    *eig = static_cast<double*>(std::malloc(sizeof(double) * static_cast<std::size_t>(op.s())));
    if (!*eig) return 1;
    const auto ev = op.eigenvalues();
    for (std::int64_t i = 0; i < op.s(); ++i) (*eig)[i] = ev[static_cast<std::size_t>(i)];
    return 0;
  } catch (...) {
    return 1;
  }
}
}  // namespace

MlmcReport mlmc_estimate_gpu(const ProblemSpec& problem, const EstimatorOptions& opt, double h0, double eps,
                             int initial_levels, int n_gpus) {
  GroupState& gs = group_state();
  const osc_problem p = problem_of(problem, opt, gs);
  const CovarianceModel& model = problem.model;
  osc_mlmc_options o{};
  o.family = model.family() == CovFamily::Matern ? OSC_COV_MATERN : OSC_COV_SEPARABLE_EXP;
  o.sigma2 = model.sigma2();
  o.lambda = model.lambda();
  o.nu_or_p = o.family == OSC_COV_MATERN ? model.nu() : model.p_norm();
  o.h0 = h0;
  o.eps = eps;
  o.initial_levels = initial_levels;
  o.l_max = opt.l_max;
  o.allow_extension = 1;
  o.seed = opt.seed;
  o.pilot_n = opt.pilot_n;
  o.gamma_model = opt.gamma_model;
  o.alpha = opt.alpha;
  o.c_alpha = opt.c_alpha;
  o.c_ratio = opt.c_ratio;
  o.c_alpha_tilde_ratio = opt.c_alpha_tilde_ratio;
  o.smoothing = opt.smoothing == SmoothingRule::Off            ? OSC_SMOOTHING_OFF
                : opt.smoothing == SmoothingRule::HalfSpectrum ? OSC_SMOOTHING_HALF_SPECTRUM
                                                               : OSC_SMOOTHING_ADAPTIVE;
  o.use_coarse_s = opt.smoothing_use_coarse_s ? 1 : 0;
  o.lstar_only = opt.smoothing_lstar_only ? 1 : 0;
  o.concurrent_levels = 1;
  static const int env_mode = env_int("OSC_SEAM_SETUP", 0);
  const int mode = gs.setup_mode >= 0 ? gs.setup_mode : env_mode;
  SpectrumSource src{&model};
  if (mode != 2) {  // 2: the driver's own device level setup
    o.spectrum = oscfield_gpu_spectrum_cb;
    o.spectrum_user = &src;
  }
  osc_mlmc_report r{};
  if (int rc = osc_mlmc_adaptive(n_gpus, nullptr, &p, &o, &r)) raise(rc);
  MlmcReport rep;
  rep.estimate = r.estimate;
  rep.bias_estimate = r.bias_estimate;
  rep.sampling_error = r.sampling_error;
  rep.total_cost_model = r.total_cost_model;
  rep.total_cost_wall = r.total_cost_wall;
  rep.converged = r.converged != 0;
  rep.message = r.message;
  for (int i = 0; i < r.n_levels; ++i) {
    LevelStats l;
    l.n = r.n[i];
    l.mean_y = r.mean_y[i];
    l.var_y = r.var_y[i];
    l.mean_q = r.mean_q[i];
    l.var_q = r.var_q[i];
    l.cost_wall_per_sample = r.wall_per_sample[i];
    l.cost_model_per_sample = std::pow(r.h[i], -opt.gamma_model);
    l.n_real = r.n_real[i];
    rep.levels.push_back(l);
    rep.level_h.push_back(r.h[i]);
  }
  return rep;
}

}  // namespace oscfield

extern "C" {
// Seam settings (process-wide; call before the first draw or between estimates):
//   n_gpus  > 0: draw every batch over an osc_group of n_gpus devices (devices NULL → 0..n-1);
//           0: the calling thread's device (default; OSC_SEAM_GPUS sets the initial value).
//   bc, qoi ≥ 0: the extension BC / QoI of include/oscfield_b200.h (OSC_BC_DIRICHLET_ALL,
//           OSC_QOI_INTEGRAL, OSC_QOI_FLUX), which the reference's ProblemSpec cannot express;
//           -1 keeps the reference's flow-cell BC and its Point / L2 QoI.
int oscfield_gpu_configure(int n_gpus, const int* devices, int bc, int qoi) {
  oscfield::GroupState& gs = oscfield::group_state();
  std::lock_guard<std::mutex> lk(gs.mu);
  if (n_gpus < 0) return OSC_ERR_CONFIG;
  std::vector<int> devs(devices ? devices : nullptr, devices ? devices + n_gpus : nullptr);
  if (n_gpus != gs.n_gpus || devs != gs.devices) {
    gs.reset();
    gs.n_gpus = n_gpus;
    gs.devices = devs;
  }
  gs.bc = bc;
  gs.qoi = qoi;
  return OSC_OK;
}

// Level setup of the routed estimator: 0 the reference's own build_operator (default), 1 this repo's
// host setup, 2 the GPU setup (see build_operator_routed); -1 returns to OSC_SEAM_SETUP.
int oscfield_gpu_set_setup(int mode) {
  if (mode < -1 || mode > 2) return OSC_ERR_CONFIG;
  oscfield::GroupState& gs = oscfield::group_state();
  std::lock_guard<std::mutex> lk(gs.mu);
  gs.setup_mode = mode;
  return OSC_OK;
}
}
