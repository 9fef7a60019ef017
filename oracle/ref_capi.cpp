// extern "C" wrapper around the PRISTINE reference library (oscfield) —
// TEST INFRASTRUCTURE ONLY. Compiled together with the unmodified sources under
// /root/reference/proj/src into oracle/_ref/libosc_ref.so (see Makefile), so
// Python tests (ctypes) can run the reference itself as the parity checker and
// as the CPU baseline (`bench.py --impl reference`). Nothing in the product
// (paper_2306_13493_b200/) links or loads this.
//
// Every function returns 0 on success, or a negative status after storing the
// exception text (ref_last_error): -2 ConfigError, -3 NumericalError,
// -4 SolverError, -5 EmbeddingError, -1 other.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>
#include <mutex>
#include <thread>
#include <algorithm>

#include "oscfield/embedding.hpp"
#include "oscfield/errors.hpp"
#include "oscfield/estimators.hpp"
#include "oscfield/fem.hpp"
#include "oscfield/rng.hpp"

using namespace oscfield;

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

CovarianceModel make_model(int family, double sigma2, double lambda, double nu_or_p) {
  return family == 0 ? CovarianceModel::matern(sigma2, lambda, nu_or_p)
                     : CovarianceModel::separable_exponential(sigma2, lambda, nu_or_p);
}
}  // namespace

extern "C" {

// Flat mirror of ProblemSpec + EstimatorOptions (estimators.hpp:16-80).
struct ref_opts {
  int family;          // 0 Matern, 1 SeparableExponential
  double sigma2, lambda, nu_or_p;
  int qoi_kind;        // 0 Point, 1 L2Norm
  double qoi_x, qoi_y;
  int forcing;         // 0 Zero, 1 Constant
  double forcing_value;
  uint64_t seed;
  int pilot_n;
  int threads;
  double gamma_model, alpha, c_alpha, c_ratio, c_alpha_tilde_ratio;
  int smoothing;       // 0 Off, 1 HalfSpectrum, 2 Adaptive
  int use_coarse_s, lstar_only, l_max;
  double tol;
  int max_iter_factor;
  int precond;         // 0 Jacobi, 1 Multigrid
};

const char* ref_last_error() { return g_err.c_str(); }
int64_t ref_last_history(double* out, int64_t cap) {
  const int64_t n = static_cast<int64_t>(g_hist.size());
  if (out) std::memcpy(out, g_hist.data(), sizeof(double) * static_cast<size_t>(n < cap ? n : cap));
  return n;
}

void ref_philox_block(const uint32_t key[2], const uint32_t ctr[4], uint32_t out[4]) {
  Philox4x32 g{{key[0], key[1]}};
  const auto r = g.block({ctr[0], ctr[1], ctr[2], ctr[3]});
  for (int i = 0; i < 4; ++i) out[i] = r[i];
}

void ref_normals(uint64_t seed, uint32_t level, uint64_t index, double* out, int64_t n) {
  NormalStream s(seed, level, index);
  s.fill(std::span<double>(out, static_cast<size_t>(n)));
}

// ---- embedding operator ---------------------------------------------------
int ref_build_operator(int m, int family, double sigma2, double lambda, double nu_or_p,
                       void** op_out) {
  return guard([&] {
    auto op = std::make_unique<EmbeddingOperator>(
        build_operator(GridSpec::square(m), make_model(family, sigma2, lambda, nu_or_p)));
    *op_out = op.release();
  });
}
int ref_load_spectrum(const char* path, double sigma2, void** op_out) {
  return guard([&] {
    *op_out = new EmbeddingOperator(load_spectrum(path, sigma2));
  });
}
int ref_save_spectrum(void* op, const char* path) {
  return guard([&] { save_spectrum(*static_cast<EmbeddingOperator*>(op), path); });
}
void ref_op_free(void* op) { delete static_cast<EmbeddingOperator*>(op); }
int64_t ref_op_s(void* op) { return static_cast<EmbeddingOperator*>(op)->s(); }
int ref_op_padding(void* op) { return static_cast<EmbeddingOperator*>(op)->padding()[0]; }
int ref_op_m(void* op) { return static_cast<EmbeddingOperator*>(op)->grid().m(0); }
void ref_op_eigenvalues(void* op, double* out) {
  const auto& e = static_cast<EmbeddingOperator*>(op)->eigenvalues();
  std::memcpy(out, e.data(), sizeof(double) * e.size());
}
void ref_op_perm(void* op, int64_t* out) {
  const auto& p = static_cast<EmbeddingOperator*>(op)->perm();
  std::memcpy(out, p.data(), sizeof(int64_t) * p.size());
}
int ref_op_truncated(void* op, int64_t k, void** out) {
  return guard([&] {
    *out = new EmbeddingOperator(static_cast<EmbeddingOperator*>(op)->truncated(k));
  });
}
int ref_sample(void* op, const double* xi, double* u) {
  return guard([&] {
    auto* o = static_cast<EmbeddingOperator*>(op);
    SampleWorkspace ws;
    const size_t s = static_cast<size_t>(o->s());
    o->sample_into(std::span<const double>(xi, s), ws, std::span<double>(u, s));
  });
}
int ref_restrict(void* op, const double* u, int m_target, double* out) {
  return guard([&] {
    auto* o = static_cast<EmbeddingOperator*>(op);
    const FieldSample f = o->restrict_to(std::span<const double>(u, static_cast<size_t>(o->s())),
                                         GridSpec::square(m_target));
    std::memcpy(out, f.values.data(), sizeof(double) * f.values.size());
  });
}
int ref_build_first_row(int m, int J, int family, double sigma2, double lambda, double nu_or_p,
                        double* out) {
  return guard([&] {
    const auto row = build_first_row(GridSpec::square(m), make_model(family, sigma2, lambda, nu_or_p),
                                     {J, J});
    std::memcpy(out, row.data(), sizeof(double) * row.size());
  });
}

// ---- FEM --------------------------------------------------------------------
int ref_solve(int m, const double* Z, int forcing, double forcing_value, double tol,
              int max_iter_factor, int precond, double* u_out) {
  return guard([&] {
    GridSpec g = GridSpec::square(m);
    FieldSample fs{g, std::vector<double>(Z, Z + g.node_count())};
    DarcyProblem p{g, fs, forcing ? Forcing::Constant : Forcing::Zero, forcing_value};
    SolverOptions so{tol, max_iter_factor, precond ? Preconditioner::Multigrid : Preconditioner::Jacobi};
    const FeSolution sol = assemble_and_solve(p, so);
    std::memcpy(u_out, sol.u.data(), sizeof(double) * sol.u.size());
  });
}
int ref_qoi_point(int m, const double* u, double x, double y, double* out) {
  return guard([&] {
    GridSpec g = GridSpec::square(m);
    FeSolution s{g, std::vector<double>(u, u + g.node_count())};
    *out = qoi_point(s, x, y);
  });
}
int ref_qoi_l2norm(int m, const double* u, double* out) {
  return guard([&] {
    GridSpec g = GridSpec::square(m);
    FeSolution s{g, std::vector<double>(u, u + g.node_count())};
    *out = qoi_l2norm(s);
  });
}

// ---- estimators ---------------------------------------------------------------
static ProblemSpec problem_of(const ref_opts& o) {
  ProblemSpec p{make_model(o.family, o.sigma2, o.lambda, o.nu_or_p), QoiSpec{}, Forcing::Constant, 1.0};
  p.qoi.kind = o.qoi_kind ? QoiSpec::Kind::L2Norm : QoiSpec::Kind::Point;
  p.qoi.x = o.qoi_x;
  p.qoi.y = o.qoi_y;
  p.forcing = o.forcing ? Forcing::Constant : Forcing::Zero;
  p.forcing_value = o.forcing_value;
  return p;
}
static EstimatorOptions options_of(const ref_opts& o) {
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
  e.solver = SolverOptions{o.tol, o.max_iter_factor,
                           o.precond ? Preconditioner::Multigrid : Preconditioner::Jacobi};
  return e;
}

struct ref_plan {
  LevelPlan plan;
};

int ref_plan_create(int ell, double h0, const ref_opts* o, void** out) {
  return guard([&] {
    auto* p = new ref_plan{make_level_plan(ell, h0, problem_of(*o), options_of(*o))};
    *out = p;
  });
}
void ref_plan_free(void* p) { delete static_cast<ref_plan*>(p); }
int64_t ref_plan_k_trunc(void* p) { return static_cast<ref_plan*>(p)->plan.k_trunc; }
int ref_plan_m(void* p) { return static_cast<ref_plan*>(p)->plan.grid.m(0); }
void* ref_plan_op(void* p) { return const_cast<EmbeddingOperator*>(static_cast<ref_plan*>(p)->plan.op.get()); }
void* ref_plan_op_smoothed(void* p) {
  return const_cast<EmbeddingOperator*>(static_cast<ref_plan*>(p)->plan.op_smoothed.get());
}

// Runs coupled_sample (estimators.cpp:200-237) for indices [from, to) on ONE thread
// (or opt.threads std::threads over contiguous chunks), writing q_fine/q_coarse by slot.
int ref_coupled_samples(void* plan, int has_coarse, int truncate_fine, int truncate_coarse,
                        const ref_opts* o, int64_t from, int64_t to, double* q_fine,
                        double* q_coarse, double* wall) {
  return guard([&] {
    auto* p = static_cast<ref_plan*>(plan);
    const ProblemSpec prob = problem_of(*o);
    const EstimatorOptions opt = options_of(*o);
    GridSpec coarse = GridSpec::square(p->plan.grid.m(0) >= 2 ? p->plan.grid.m(0) / 2 : 1);
    const int64_t count = to - from;
    int workers = o->threads > 0 ? o->threads : 1;
    if (workers > count) workers = static_cast<int>(count > 0 ? count : 1);
    std::vector<std::thread> pool;
    std::exception_ptr err;
    std::mutex mu;
    const int64_t chunk = (count + workers - 1) / workers;
    for (int w = 0; w < workers; ++w) {
      const int64_t lo = from + w * chunk, hi = std::min<int64_t>(to, lo + chunk);
      if (lo >= hi) break;
      pool.emplace_back([&, lo, hi] {
        try {
          SampleWorkspace ws;
          for (int64_t i = lo; i < hi; ++i) {
            const CoupledResult r = coupled_sample(p->plan, has_coarse ? &coarse : nullptr,
                                                   truncate_fine != 0, truncate_coarse != 0, prob,
                                                   opt, static_cast<uint64_t>(i), ws);
            q_fine[i - from] = r.q_fine;
            if (q_coarse) q_coarse[i - from] = r.has_coarse ? r.q_coarse : 0.0;
            if (wall) wall[i - from] = r.wall_seconds;
          }
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          if (!err) err = std::current_exception();
        }
      });
    }
    for (auto& t : pool) t.join();
    if (err) std::rethrow_exception(err);
  });
}

// Flat MlmcReport (estimators.hpp:43-62); levels truncated to cap.
struct ref_report {
  double estimate, bias_estimate, sampling_error, total_cost_model, total_cost_wall;
  int converged;
  int n_levels;
  int64_t n[32];
  double mean_y[32], var_y[32], mean_q[32], var_q[32], h[32], n_real[32];
};

static void fill_report(const MlmcReport& r, ref_report* out) {
  std::memset(out, 0, sizeof(*out));
  out->estimate = r.estimate;
  out->bias_estimate = r.bias_estimate;
  out->sampling_error = r.sampling_error;
  out->total_cost_model = r.total_cost_model;
  out->total_cost_wall = r.total_cost_wall;
  out->converged = r.converged ? 1 : 0;
  out->n_levels = static_cast<int>(std::min<size_t>(r.levels.size(), 32));
  for (int i = 0; i < out->n_levels; ++i) {
    out->n[i] = r.levels[i].n;
    out->mean_y[i] = r.levels[i].mean_y;
    out->var_y[i] = r.levels[i].var_y;
    out->mean_q[i] = r.levels[i].mean_q;
    out->var_q[i] = r.levels[i].var_q;
    out->h[i] = r.level_h[i];
    out->n_real[i] = r.levels[i].n_real;
  }
}

int ref_mc_fixed_n(const ref_opts* o, int m, int64_t n, ref_report* out) {
  return guard([&] {
    fill_report(mc_estimate_fixed_n(problem_of(*o), options_of(*o), GridSpec::square(m), n), out);
  });
}
int ref_mlmc(const ref_opts* o, double h0, double eps, int initial_levels, ref_report* out) {
  return guard([&] {
    fill_report(mlmc_estimate(problem_of(*o), options_of(*o), h0, eps, initial_levels), out);
  });
}
int64_t ref_choose_k_ell(int family, double sigma2, double lambda, double nu_or_p, double h,
                         int padding, int64_t s, double alpha, double c_ratio, int use_coarse_s) {
  int64_t k = -1;
  guard([&] {
    k = choose_k_ell(make_model(family, sigma2, lambda, nu_or_p), h, padding, s, alpha, c_ratio,
                     use_coarse_s != 0);
  });
  return k;
}
double ref_coarsest_level_bound(int family, double sigma2, double lambda, double nu_or_p) {
  return coarsest_level_bound(make_model(family, sigma2, lambda, nu_or_p));
}

}  // extern "C"
