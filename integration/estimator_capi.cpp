// extern "C" entry points of the GPU-routed reference build (integration/_build/liboscfield_gpu.so):
// the reference's OWN estimators — mlmc_estimate, mc_estimate, mc_estimate_fixed_n
// (src/estimators.cpp:382-418, the adaptive loop :289-378) — compiled from the pristine sources with
// run_level_samples routed to the GPU seam (route_run_level_samples.hpp, oscfield_gpu_seams.cpp).
// The host control loop is the reference's C++; every sample is drawn by libosc_b200.so.
// Flat structs so any FFI (ctypes here) can call it; errors as negative codes + message.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "oscfield/errors.hpp"
#include "oscfield/estimators.hpp"

using namespace oscfield;

namespace oscfield {
MlmcReport mlmc_estimate_gpu(const ProblemSpec& problem, const EstimatorOptions& opt, double h0, double eps,
                             int initial_levels, int n_gpus);
}
extern "C" int oscfield_gpu_configure(int n_gpus, const int* devices, int bc, int qoi);
extern "C" int oscfield_gpu_set_setup(int mode);

namespace {
thread_local std::string g_err;
thread_local std::vector<double> g_hist;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const SolverError& e) {
    g_err = e.what();
    g_hist = e.residual_history;
    return -4;
  } catch (const EmbeddingError& e) {
    g_err = e.what();
    return -5;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return -3;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
}  // namespace

extern "C" {

// ProblemSpec + EstimatorOptions (estimators.hpp:25-30,66-80), flat
struct oscgpu_opts {
  int family;  // 0 Matern, 1 separable exponential (covariance.hpp:10)
  double sigma2, lambda, nu_or_p;
  int qoi_kind;  // 0 Point, 1 L2Norm
  double qoi_x, qoi_y;
  int forcing;  // 0 Zero, 1 Constant
  double forcing_value;
  uint64_t seed;
  int pilot_n, threads;
  double gamma_model, alpha, c_alpha, c_ratio, c_alpha_tilde_ratio;
  int smoothing;  // 0 Off, 1 HalfSpectrum, 2 Adaptive
  int use_coarse_s, lstar_only, l_max;
  double tol;
  int max_iter_factor;
};

// MlmcReport (estimators.hpp:43-62), levels truncated to 32
struct oscgpu_report {
  double estimate, bias_estimate, sampling_error, total_cost_model, total_cost_wall;
  int converged;
  int n_levels;
  int64_t n[32];
  double mean_y[32], var_y[32], mean_q[32], var_q[32], h[32], n_real[32], wall[32];
  char message[256];
};

const char* oscgpu_last_error() { return g_err.c_str(); }
int64_t oscgpu_last_history(double* out, int64_t cap) {
  const int64_t n = static_cast<int64_t>(g_hist.size());
  for (int64_t i = 0; i < std::min(n, cap); ++i) out[i] = g_hist[i];
  return n;
}

int oscgpu_configure(int n_gpus, const int* devices, int bc, int qoi) {
  return oscfield_gpu_configure(n_gpus, devices, bc, qoi);
}

int oscgpu_set_setup(int mode) { return oscfield_gpu_set_setup(mode); }

}  // extern "C"

namespace {
ProblemSpec problem_of(const oscgpu_opts& o) {
  const CovarianceModel model = o.family == 0 ? CovarianceModel::matern(o.sigma2, o.lambda, o.nu_or_p)
                                              : CovarianceModel::separable_exponential(o.sigma2, o.lambda, o.nu_or_p);
  ProblemSpec p{model, QoiSpec{}, o.forcing ? Forcing::Constant : Forcing::Zero, o.forcing_value};
  p.qoi.kind = o.qoi_kind ? QoiSpec::Kind::L2Norm : QoiSpec::Kind::Point;
  p.qoi.x = o.qoi_x;
  p.qoi.y = o.qoi_y;
  return p;
}

EstimatorOptions options_of(const oscgpu_opts& o) {
  EstimatorOptions e;
  e.seed = o.seed;
  e.pilot_n = o.pilot_n;
  e.threads = o.threads;
  e.gamma_model = o.gamma_model;
  e.alpha = o.alpha;
  e.c_alpha = o.c_alpha;
  e.c_ratio = o.c_ratio;
  e.c_alpha_tilde_ratio = o.c_alpha_tilde_ratio;
  e.smoothing = o.smoothing == 0 ? SmoothingRule::Off
                : o.smoothing == 1 ? SmoothingRule::HalfSpectrum : SmoothingRule::Adaptive;
  e.smoothing_use_coarse_s = o.use_coarse_s != 0;
  e.smoothing_lstar_only = o.lstar_only != 0;
  e.l_max = o.l_max;
  e.solver = SolverOptions{o.tol, o.max_iter_factor, Preconditioner::Multigrid};
  return e;
}

void fill(const MlmcReport& r, oscgpu_report* out) {
  std::memset(out, 0, sizeof(*out));
  out->estimate = r.estimate;
  out->bias_estimate = r.bias_estimate;
  out->sampling_error = r.sampling_error;
  out->total_cost_model = r.total_cost_model;
  out->total_cost_wall = r.total_cost_wall;
  out->converged = r.converged ? 1 : 0;
  out->n_levels = static_cast<int>(std::min<std::size_t>(r.levels.size(), 32));
  for (int i = 0; i < out->n_levels; ++i) {
    const LevelStats& l = r.levels[i];
    out->n[i] = l.n;
    out->mean_y[i] = l.mean_y;
    out->var_y[i] = l.var_y;
    out->mean_q[i] = l.mean_q;
    out->var_q[i] = l.var_q;
    out->h[i] = r.level_h[i];
    out->n_real[i] = l.n_real;
    out->wall[i] = l.cost_wall_per_sample;
  }
  std::strncpy(out->message, r.message.c_str(), sizeof(out->message) - 1);
}
}  // namespace

extern "C" {

int oscgpu_mlmc_estimate(const oscgpu_opts* o, double h0, double eps, int initial_levels, oscgpu_report* out) {
  return guard([&] { fill(mlmc_estimate(problem_of(*o), options_of(*o), h0, eps, initial_levels), out); });
}

// the same estimate on the GPU-resident driver (mlmc_estimate_gpu, oscfield_gpu_seams.cpp)
int oscgpu_mlmc_estimate_resident(const oscgpu_opts* o, double h0, double eps, int initial_levels, int n_gpus,
                                  oscgpu_report* out) {
  return guard([&] { fill(mlmc_estimate_gpu(problem_of(*o), options_of(*o), h0, eps, initial_levels, n_gpus), out); });
}

int oscgpu_mc_estimate(const oscgpu_opts* o, double eps, double fixed_h /* <= 0: none */, oscgpu_report* out) {
  return guard([&] {
    std::optional<double> fh;
    if (fixed_h > 0) fh = fixed_h;
    fill(mc_estimate(problem_of(*o), options_of(*o), eps, fh), out);
  });
}

double oscgpu_coarsest_level_bound(int family, double sigma2, double lambda, double nu_or_p) {
  const CovarianceModel model = family == 0 ? CovarianceModel::matern(sigma2, lambda, nu_or_p)
                                            : CovarianceModel::separable_exponential(sigma2, lambda, nu_or_p);
  return coarsest_level_bound(model);
}

int oscgpu_mc_estimate_fixed_n(const oscgpu_opts* o, int m, int64_t n, oscgpu_report* out) {
  return guard([&] { fill(mc_estimate_fixed_n(problem_of(*o), options_of(*o), GridSpec::square(m), n), out); });
}

}  // extern "C"
