// GPU-resident adaptive MLMC driver (include/oscfield_b200.h, osc_mlmc_adaptive).
//
// The reference's estimate_adaptive (src/estimators.cpp:289-378) walks the levels one after the other
// and keeps every draw in host vectors. Two facts of that loop make it a device-resident one:
//   * inside one allocation pass the targets N_ℓ of ALL levels are functions of the moments at the
//     start of the pass (:322-338: sum_cv is formed once, each level's variance is only refreshed after
//     its own draws), and the pilot fills (:310-319) are independent as well — so a pass is a WAVE of
//     independent per-level batches that can run at the same time;
//   * the allocation only needs (n, mean, variance) per level, i.e. the five running sums the draw
//     kernels already accumulate in HBM (osc_level_sums_*).
// Here every level owns one context (stream + workspaces) per device and one host thread per context
// while a wave runs; the small levels, which cannot fill the GPU alone, execute under the large
// ones. Between waves the host reads 5 doubles per level (all levels of all devices combined by one
// all-reduce when several devices take part) and takes the reference's decisions.
//
// Shifts of the running sums: unknown before a level's first batch, so that batch accumulates at
// shift 0 and the sums are then re-centred on its mean on the device (osc_level_sums_reshift); every
// later, larger batch accumulates without cancellation.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "osc_internal.cuh"

struct osc_group;
namespace osc {
void draws_checked(Level* L, const osc_problem* prob, uint64_t seed, uint32_t ell, int64_t from, int64_t to,
                   int flags, const double* xi, double* q_fine, double* q_coarse, int32_t* iters_fine,
                   int32_t* iters_coarse, int32_t* status, double* level_sums);
int c_api_error(const std::exception_ptr& e);
void group_allreduce_f64(osc_group* g, double* const* send, double* const* recv, size_t count);
}  // namespace osc

using namespace osc;

namespace {

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

// h = 2^-j for an integer j ≥ 0 → cells per side 2^j (make_level_plan's precondition, :173-175)
bool cells_of(double h, int& m) {
  if (!(h > 0.0) || h > 1.0) return false;
  int e = 0;
  if (std::frexp(h, &e) != 0.5) return false;  // exactly a power of two
  m = 1 << (1 - e);
  return 1 - e <= 16;
}

// the largest mesh width 2^-j that resolves the correlation length (coarsest_level_bound, :487-494)
double resolving_width(const osc_mlmc_options& o) {
  const double len = o.family == OSC_COV_SEPARABLE_EXP ? o.lambda : std::sqrt(8.0 * o.nu_or_p) * o.lambda;
  double h = 1.0;
  while (h > len * (1.0 + 1e-12)) h *= 0.5;
  return h;
}

int64_t clamp_k(double k, int64_t s) { return std::min<int64_t>(std::max<int64_t>(std::llround(k), 0), s - 1); }

// choose_k_ell (:238-275): the number of smallest modes dropped on mesh width h
int64_t adaptive_k(const osc_mlmc_options& o, double h, int J, int64_t s) {
  OSC_REQUIRE(o.alpha > 0.0, "smoothing rule: alpha must be positive");
  OSC_REQUIRE(o.c_ratio > 0.0, "smoothing rule: c_ratio must be positive");
  const double hs = o.use_coarse_s ? 2.0 * h : h;  // the rule may be evaluated on the coarse partner's mesh
  if (o.family == OSC_COV_SEPARABLE_EXP) {
    // closed form for the separable exponential: k = S^((3-α)/2) / (c + S^(-(α-1)/2)), S = 4/h²
    const double S = 4.0 / (hs * hs);
    return clamp_k(std::pow(S, 0.5 * (3.0 - o.alpha)) / (o.c_ratio + std::pow(S, -0.5 * (o.alpha - 1.0))), s);
  }
  // Matérn: the root of k (S − k)^(-(1+ν)/2) = c h^α W on (0, S − 1), W the embedding half width
  const double W = 1.0 / hs + (o.use_coarse_s ? 0.5 * J : (double)J);
  const double S = 4.0 * W * W, target = o.c_ratio * std::pow(hs, o.alpha) * W, ex = -0.5 * (1.0 + o.nu_or_p);
  auto excess = [&](double k) { return k * std::pow(S - k, ex) - target; };
  double a = 0.0, b = S - 1.0;
  if (!(b > a) || excess(b) < 0.0) {
    std::fprintf(stderr, "osc_mlmc: smoothing rule has no root at h = %g; level left unsmoothed\n", h);
    return 0;
  }
  while (b - a > 0.5) {
    const double mid = 0.5 * (a + b);
    if (excess(mid) < 0.0) a = mid; else b = mid;
  }
  return clamp_k(0.5 * (a + b), s);
}

int64_t k_trunc_rule(const osc_mlmc_options& o, double h, int J, int64_t s) {
  if (o.smoothing == OSC_SMOOTHING_OFF) return 0;
  // lstar_only: levels whose mesh already resolves the correlation length stay unsmoothed (:185-186)
  if (o.lstar_only && h <= resolving_width(o) * (1.0 + 1e-12)) return 0;
  const int64_t k = o.smoothing == OSC_SMOOTHING_HALF_SPECTRUM ? s / 2 : adaptive_k(o, h, J, s);
  return std::min<int64_t>(std::max<int64_t>(k, 0), s - 1);
}

struct Moments {
  int64_t n = 0;
  double mean_y = 0, var_y = 0, mean_q = 0, var_q = 0;
};

// one MLMC level: a context and a device level per participating device
struct LevelRun {
  int ell = 0, m = 0;
  double h = 0;
  int64_t k_trunc = 0;
  bool trunc_fine = false, trunc_coarse = false;
  std::vector<osc_ctx*> ctx;
  std::vector<osc_level*> lev;
  int64_t have = 0;      // samples drawn under the current sampling law
  bool centred = false;  // running sums already re-centred on the first batch's mean
  double shift_y = 0, shift_q = 0;
  Moments mom;
  double n_real = 0, busy_s = 0;
  int64_t redrawn = 0;   // samples discarded because the level's sampling law changed
  int64_t launches_gone = 0;  // launches of contexts already replaced
  ~LevelRun() {
    for (osc_level* l : lev) osc_level_destroy(l);
    for (osc_ctx* c : ctx) osc_ctx_destroy(c);
  }
};

struct Driver {
  const osc_problem& prob;
  const osc_mlmc_options& opt;
  std::vector<int> devices;
  osc_group* group = nullptr;            // several devices: communicators + one staging context each
  std::vector<DevBuf> stage;             // per device: [levels × 8] sums in, [levels × 8] reduced
  std::vector<std::unique_ptr<LevelRun>> levels;
  int waves = 0;
  double setup_s = 0, draw_s = 0;
  int64_t samples = 0;

  Driver(const osc_problem& p, const osc_mlmc_options& o) : prob(p), opt(o) {}
  ~Driver() {
    levels.clear();
    for (size_t g = 0; g < stage.size(); ++g) {
      cudaSetDevice(devices[g]);
      stage[g].release();
    }
    if (group) osc_group_destroy(group);
  }
  int G() const { return (int)devices.size(); }

  // run fn(j) for j < n on n host threads (or in order when n == 1 / serial); the first failure in
  // index order is rethrown once every thread has finished, like parallel_samples (:52-63)
  template <typename F>
  void fan_out(int n, bool serial, F&& fn) {
    std::vector<std::exception_ptr> errs((size_t)n);
    if (serial || n == 1) {
      for (int j = 0; j < n; ++j) {
        try { fn(j); } catch (...) { errs[(size_t)j] = std::current_exception(); }
      }
    } else {
      std::vector<std::thread> pool;
      pool.reserve((size_t)n);
      for (int j = 0; j < n; ++j)
        pool.emplace_back([&, j] {
          try { fn(j); } catch (...) { errs[(size_t)j] = std::current_exception(); }
        });
      for (auto& t : pool) t.join();
    }
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }

  static size_t held_bytes(const Ctx* c) {
    return c->ce_inter.bytes + c->xi_dev.bytes + c->fields_fine.bytes + c->fields_coarse.bytes + c->solver.mem.bytes +
           c->out_q.bytes + c->out_i.bytes + c->retry_k.bytes + c->retry_q.bytes;
  }

  // Equal shares of each device's memory for the batch workspaces of the active levels (under the MLMC
  // allocation N_ℓ · bytes per sample is roughly level-independent). A context whose workspaces have
  // grown beyond the new share is replaced, so that memory returns to the pool; the others keep their
  // workspaces (and their instantiated PCG-loop graphs) and only get the new budget.
  void rebalance() {
    for (int g = 0; g < G(); ++g) {
      OSC_CUDA(cudaSetDevice(devices[g]));
      size_t fr = 0, tot = 0, held = 0;
      OSC_CUDA(cudaMemGetInfo(&fr, &tot));
      for (auto& L : levels) held += held_bytes(L->ctx[g]);
      const size_t share = std::max<size_t>((size_t)(0.85 * (double)(fr + held) / (double)levels.size()), (size_t)64 << 20);
      for (auto& L : levels) {
        if (held_bytes(L->ctx[g]) > share) {
          L->launches_gone += L->ctx[g]->launches;
          osc_ctx* fresh = nullptr;
          if (int rc = osc_ctx_create(devices[g], &fresh)) throw Error(rc, osc_last_error());
          osc_ctx_destroy(L->ctx[g]);
          L->ctx[g] = fresh;
          L->lev[g]->ctx = fresh;
        }
        osc_ctx_set_mem_budget(L->ctx[g], share);
      }
    }
  }

  void set_law(LevelRun& L, bool is_finest) {
    // set_mode (:114-122): a smoothed level truncates its coarse term always, its fine term unless it
    // is the finest level; a changed law discards the level's samples
    const bool ces = opt.smoothing != OSC_SMOOTHING_OFF && L.k_trunc > 0;
    const bool tf = ces && !is_finest, tc = ces;
    if ((tf != L.trunc_fine || tc != L.trunc_coarse) && L.have > 0) {
      L.redrawn += L.have;
      L.have = 0;
      L.mom = Moments{};
    }
    L.trunc_fine = tf;
    L.trunc_coarse = tc;
  }

  void add_levels(int first, int last, int finest) {
    const auto t0 = Clock::now();
    int m0 = 0;
    OSC_REQUIRE(cells_of(opt.h0, m0), "osc_mlmc: h0 must be a negative power of two");
    const size_t base = levels.size();
    for (int ell = first; ell <= last; ++ell) {
      OSC_REQUIRE(ell >= 0 && ell <= 24, "osc_mlmc: level out of range");
      const int64_t m = (int64_t)m0 << ell;
      OSC_REQUIRE(m <= (1 << 16), "osc_mlmc: grid too fine");
      auto L = std::make_unique<LevelRun>();
      L->ell = ell;
      L->m = (int)m;
      L->h = opt.h0 / (double)((int64_t)1 << ell);
      L->ctx.assign((size_t)G(), nullptr);
      L->lev.assign((size_t)G(), nullptr);
      levels.push_back(std::move(L));
    }
    const int nl = last - first + 1;
    // caller-supplied spectra: one call per level, from this thread only (the callback may be a host
    // setup that is not re-entrant), shared by the level's devices
    struct Spectrum {
      int J = 0;
      int64_t s = 0;
      double* eig = nullptr;
    };
    std::vector<Spectrum> spectra((size_t)nl);
    struct FreeAll {
      std::vector<Spectrum>& v;
      ~FreeAll() {
        for (auto& sp : v) std::free(sp.eig);
      }
    } free_all{spectra};
    if (opt.spectrum)
      for (int i = 0; i < nl; ++i) {
        Spectrum& sp = spectra[(size_t)i];
        if (opt.spectrum(opt.spectrum_user, levels[base + (size_t)i]->m, &sp.J, &sp.s, &sp.eig) != 0 || !sp.eig)
          throw Error(OSC_ERR_EMBEDDING, "osc_mlmc: the spectrum callback failed");
      }
    // setup of the new levels: all (level, device) pairs at once, each on its own stream
    fan_out(nl * G(), !opt.concurrent_levels, [&](int j) {
      LevelRun& L = *levels[base + (size_t)(j / G())];
      const int g = j % G();
      OSC_CUDA(cudaSetDevice(devices[g]));
      if (int rc = osc_ctx_create(devices[g], &L.ctx[g])) throw Error(rc, osc_last_error());
      if (opt.spectrum) {
        const Spectrum& sp = spectra[(size_t)(j / G())];
        const int64_t k = k_trunc_rule(opt, L.h, sp.J, sp.s);
        if (int rc = osc_level_create(L.ctx[g], L.m, sp.J, sp.eig, k, &L.lev[g])) throw Error(rc, osc_last_error());
      } else {
        if (int rc = osc_level_create_device(L.ctx[g], L.m, opt.family, opt.sigma2, opt.lambda, opt.nu_or_p, nullptr,
                                             0, 0.0, 0, &L.lev[g]))
          throw Error(rc, osc_last_error());
        const int64_t k = k_trunc_rule(opt, L.h, L.lev[g]->J, L.lev[g]->s);
        if (k > 0)
          if (int rc = osc_level_retruncate(L.lev[g], k)) throw Error(rc, osc_last_error());
      }
    });
    for (size_t i = base; i < levels.size(); ++i) {
      levels[i]->k_trunc = levels[i]->lev[0]->k_trunc;
      set_law(*levels[i], levels[i]->ell == finest);
    }
    rebalance();
    setup_s += seconds_since(t0);
  }

  struct Job {
    LevelRun* L;
    int64_t from, to;
  };

  // One wave: every job's range cut into contiguous per-device chunks (parallel_samples' chunking,
  // :36-41), one host thread per (level, device); then the moments of the waved levels are refreshed
  // from the device sums.
  void run_wave(const std::vector<Job>& jobs) {
    const auto t0 = Clock::now();
    ++waves;
    struct Piece {
      LevelRun* L;
      int g;
      int64_t lo, hi;
    };
    std::vector<Piece> pieces;
    for (const Job& j : jobs) {
      LevelRun& L = *j.L;
      if (L.have == 0) {  // first batch under this law: sums restart at shift 0
        for (int g = 0; g < G(); ++g)
          if (int rc = osc_level_sums_reset(L.lev[g], 0.0, 0.0)) throw Error(rc, osc_last_error());
        L.centred = false;
        L.shift_y = L.shift_q = 0.0;
      }
      const int64_t count = j.to - j.from, chunk = (count + G() - 1) / G();
      for (int g = 0; g < G(); ++g) {
        const int64_t lo = std::min(j.to, j.from + g * chunk), hi = std::min(j.to, lo + chunk);
        if (hi > lo) pieces.push_back({&L, g, lo, hi});
      }
    }
    // the largest pieces start first
    std::stable_sort(pieces.begin(), pieces.end(), [](const Piece& a, const Piece& b) {
      return (double)(a.hi - a.lo) * a.L->m * a.L->m > (double)(b.hi - b.lo) * b.L->m * b.L->m;
    });
    fan_out((int)pieces.size(), !opt.concurrent_levels, [&](int i) {
      const Piece& p = pieces[(size_t)i];
      LevelRun& L = *p.L;
      const auto tp = Clock::now();
      const int flags = (L.ell > 0 ? OSC_DRAW_HAS_COARSE : 0) | (L.trunc_fine ? OSC_DRAW_TRUNC_FINE : 0) |
                        (L.trunc_coarse ? OSC_DRAW_TRUNC_COARSE : 0);
      draws_checked(L.lev[p.g], &prob, opt.seed, (uint32_t)L.ell, p.lo, p.hi, flags, nullptr, nullptr, nullptr, nullptr,
                    nullptr, nullptr, nullptr);
      if (p.g == 0) L.busy_s += seconds_since(tp);
    });
    for (const Job& j : jobs) {
      j.L->have = j.to;
      samples += j.to - j.from;
    }
    refresh(jobs);
    draw_s += seconds_since(t0);
  }

  void refresh(const std::vector<Job>& jobs) {
    const size_t nl = levels.size();
    std::vector<double> sums(8 * nl, 0.0);
    if (!group) {
      for (const Job& j : jobs) {
        double out[7];
        if (int rc = osc_level_sums_read(j.L->lev[0], out)) throw Error(rc, osc_last_error());
        std::copy(out, out + 5, sums.begin() + 8 * index_of(j.L));
      }
    } else {
      // all levels' sums of a device → its staging buffer, one all-reduce over the devices
      std::vector<double*> send((size_t)G()), recv((size_t)G());
      for (int g = 0; g < G(); ++g) {
        OSC_CUDA(cudaSetDevice(devices[g]));
        stage[(size_t)g].ensure(sizeof(double) * 16 * OSC_MLMC_MAX_LEVELS);
        double* st = stage[(size_t)g].as<double>();
        cudaStream_t s = osc_group_ctx(group, g)->stream;
        OSC_CUDA(cudaMemsetAsync(st, 0, sizeof(double) * 8 * nl, s));
        for (const Job& j : jobs)
          OSC_CUDA(cudaMemcpyAsync(st + 8 * index_of(j.L), j.L->lev[(size_t)g]->run_sums.p, sizeof(double) * 5,
                                   cudaMemcpyDeviceToDevice, s));
        send[(size_t)g] = st;
        recv[(size_t)g] = st + 8 * OSC_MLMC_MAX_LEVELS;
      }
      group_allreduce_f64(group, send.data(), recv.data(), 8 * nl);
      OSC_CUDA(cudaSetDevice(devices[0]));
      OSC_CUDA(cudaMemcpy(sums.data(), recv[0], sizeof(double) * 8 * nl, cudaMemcpyDeviceToHost));
    }
    for (const Job& j : jobs) {
      LevelRun& L = *j.L;
      const double* s = sums.data() + 8 * index_of(&L);
      const double n = s[0];
      if ((int64_t)n != L.have)
        throw Error(OSC_ERR_CUDA, "osc_mlmc: device sample count differs from the schedule");
      Moments mo;
      mo.n = L.have;
      mo.mean_y = L.shift_y + s[1] / n;
      mo.mean_q = L.shift_q + s[3] / n;
      if (mo.n >= 2) {  // moments_of divides by n − 1 from two samples on (:97-99)
        mo.var_y = std::max(0.0, (s[2] - s[1] * s[1] / n) / (n - 1.0));
        mo.var_q = std::max(0.0, (s[4] - s[3] * s[3] / n) / (n - 1.0));
      }
      L.mom = mo;
      if (!L.centred) {
        for (int g = 0; g < G(); ++g)
          if (int rc = osc_level_sums_reshift(L.lev[(size_t)g], mo.mean_y, mo.mean_q)) throw Error(rc, osc_last_error());
        L.shift_y = mo.mean_y;
        L.shift_q = mo.mean_q;
        L.centred = true;
      }
    }
  }

  size_t index_of(const LevelRun* L) const {
    for (size_t i = 0; i < levels.size(); ++i)
      if (levels[i].get() == L) return i;
    return 0;
  }
};

void copy_message(char (&dst)[256], const std::string& msg) {
  std::snprintf(dst, sizeof dst, "%s", msg.c_str());
}

void run(int n_devices, const int* devs, const osc_problem& prob, const osc_mlmc_options& o, osc_mlmc_report& rep) {
  const auto t_all = Clock::now();
  OSC_REQUIRE(o.eps > 0.0, "osc_mlmc: eps must be positive");
  OSC_REQUIRE(o.initial_levels >= 1, "osc_mlmc: need at least one level");
  OSC_REQUIRE(o.family == OSC_COV_MATERN || o.family == OSC_COV_SEPARABLE_EXP, "osc_mlmc: unknown covariance family");
  OSC_REQUIRE(o.smoothing >= OSC_SMOOTHING_OFF && o.smoothing <= OSC_SMOOTHING_ADAPTIVE, "osc_mlmc: unknown smoothing rule");
  OSC_REQUIRE(o.alpha > 0.0, "osc_mlmc: alpha must be positive");
  int m0 = 0;
  OSC_REQUIRE(cells_of(o.h0, m0), "osc_mlmc: h0 must be a negative power of two");
  OSC_REQUIRE(o.l_max < OSC_MLMC_MAX_LEVELS, "osc_mlmc: l_max beyond OSC_MLMC_MAX_LEVELS");

  Driver d(prob, o);
  if (n_devices <= 0) {
    int cur = 0;
    OSC_CUDA(cudaGetDevice(&cur));
    d.devices = {cur};
  } else {
    for (int i = 0; i < n_devices; ++i) d.devices.push_back(devs ? devs[i] : i);
  }
  // several devices: NCCL communicators + one staging context per device (OSC_MLMC_FORCE_GROUP=1 takes
  // this path on a single device too, so the collective path can be exercised on a one-GPU box)
  const char* force = std::getenv("OSC_MLMC_FORCE_GROUP");
  if (d.G() > 1 || (force && force[0] == '1')) {
    if (int rc = osc_group_create(d.G(), d.devices.data(), &d.group)) throw Error(rc, osc_last_error());
    d.stage.resize((size_t)d.G());
  }

  const double half_eps2 = 0.5 * o.eps * o.eps;
  const int64_t pilot = std::max(2, o.pilot_n);
  const int l_first = std::max(0, std::min(o.initial_levels - 1, o.l_max));
  d.add_levels(0, l_first, l_first);

  std::string message;
  bool converged = true;
  double bias = 0.0;
  int passes = 0;
  for (;; ++passes) {
    if (passes > 64) {
      converged = false;
      message = "sample allocation did not stabilise";
      break;
    }
    // wave 1 of the pass: levels below the pilot count
    std::vector<Driver::Job> jobs;
    for (auto& L : d.levels)
      if (L->have < pilot) jobs.push_back({L.get(), L->have, pilot});
    const bool filled = !jobs.empty();
    if (filled) d.run_wave(jobs);
    // wave 2: the allocation from the moments all levels hold now
    double cv = 0.0;
    for (auto& L : d.levels) cv += std::sqrt(std::pow(L->h, -o.gamma_model) * std::max(L->mom.var_y, 0.0));
    jobs.clear();
    for (auto& L : d.levels) {
      const double cost = std::pow(L->h, -o.gamma_model);
      L->n_real = 2.0 / (o.eps * o.eps) * cv * std::sqrt(std::max(L->mom.var_y, 0.0) / cost);
      const int64_t want = std::max<int64_t>((int64_t)std::ceil(L->n_real), 2);
      if (want > L->have) jobs.push_back({L.get(), L->have, want});
    }
    if (!jobs.empty()) {
      d.run_wave(jobs);
      continue;
    }
    if (filled) continue;

    const LevelRun& top = *d.levels.back();
    if (d.levels.size() == 1) {
      bias = o.c_alpha * std::pow(top.h, o.alpha);  // no pair to extrapolate from: the weak-error model
      if (!o.allow_extension || o.l_max == 0) {
        message = "single level: bias taken from the weak-error model";
        break;
      }
    } else {
      const bool smoothed_pair = top.trunc_coarse && top.k_trunc > 0;
      const double denom = 1.0 - (smoothed_pair ? o.c_alpha_tilde_ratio : 1.0) * std::pow(2.0, o.alpha);
      if (std::abs(denom) < 0.1)
        throw Error(OSC_ERR_NUMERICAL, "osc_mlmc: Richardson extrapolation denominator below 0.1");
      bias = std::abs(top.mom.mean_y) / std::abs(denom);
    }
    if (o.allow_extension && bias * bias > half_eps2) {
      const int L_now = (int)d.levels.size() - 1;
      if (L_now >= o.l_max) {
        converged = false;
        char buf[160];
        std::snprintf(buf, sizeof buf, "bias %g still above target %g at L_max = %d", bias, std::sqrt(half_eps2), o.l_max);
        message = buf;
        break;
      }
      d.add_levels(L_now + 1, L_now + 1, L_now + 1);
      for (size_t i = 0; i + 1 < d.levels.size(); ++i) d.set_law(*d.levels[i], false);
      continue;
    }
    break;
  }

  std::memset(&rep, 0, sizeof rep);
  rep.bias_estimate = bias;
  rep.n_levels = (int)d.levels.size();
  rep.passes = passes + (passes <= 64 ? 1 : 0);
  rep.waves = d.waves;
  double var_sum = 0.0;
  for (size_t i = 0; i < d.levels.size(); ++i) {
    const LevelRun& L = *d.levels[i];
    rep.n[i] = L.mom.n;
    rep.k_trunc[i] = L.k_trunc;
    rep.redrawn[i] = L.redrawn;
    rep.mean_y[i] = L.mom.mean_y;
    rep.var_y[i] = L.mom.var_y;
    rep.mean_q[i] = L.mom.mean_q;
    rep.var_q[i] = L.mom.var_q;
    rep.h[i] = L.h;
    rep.n_real[i] = L.n_real;
    rep.wall_per_sample[i] = L.mom.n > 0 ? L.busy_s / (double)(L.mom.n + L.redrawn) : 0.0;
    rep.estimate += L.mom.mean_y;
    if (L.mom.n > 0) var_sum += L.mom.var_y / (double)L.mom.n;
    rep.total_cost_model += std::pow(L.h, -o.gamma_model) * (double)L.mom.n;
    rep.total_cost_wall += rep.wall_per_sample[i] * (double)L.mom.n;
    rep.gpu_launches += L.launches_gone;
    for (osc_ctx* c : L.ctx) rep.gpu_launches += c->launches;
  }
  rep.sampling_error = std::sqrt(var_sum);
  if (rep.sampling_error * rep.sampling_error > half_eps2 * (1.0 + 1e-9)) {
    converged = false;
    message += message.empty() ? "sampling error above target" : "; sampling error above target";
  }
  rep.converged = converged ? 1 : 0;
  rep.setup_s = d.setup_s;
  rep.draw_s = d.draw_s;
  rep.samples_total = d.samples;
  copy_message(rep.message, message);
  rep.total_s = seconds_since(t_all);
}

}  // namespace

extern "C" {

int osc_mlmc_adaptive(int n_devices, const int* devices, const osc_problem* problem, const osc_mlmc_options* options,
                      osc_mlmc_report* report) {
  try {
    OSC_REQUIRE(problem && options && report, "osc_mlmc_adaptive: null argument");
    run(n_devices, devices, *problem, *options, *report);
    return OSC_OK;
  } catch (...) {
    return c_api_error(std::current_exception());
  }
}

int64_t osc_mlmc_k_trunc(const osc_mlmc_options* options, double h, int J, int64_t s) {
  try {
    if (!options || s < 1) return 0;
    return k_trunc_rule(*options, h, J, s);
  } catch (...) {
    c_api_error(std::current_exception());
    return -1;
  }
}

}  // extern "C"
