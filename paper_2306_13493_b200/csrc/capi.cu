// C-ABI (include/oscfield_b200.h): context / level lifetime, the fused per-level batch
// osc_level_draws (the reference's run_level_draws seam, estimators.hpp:112-118) and the
// unfused single-stage entry points. Host C++; every kernel runs on the context stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "osc_internal.cuh"

namespace osc {
struct SetupError {
  int code;
  std::string msg;
};
std::vector<double> build_spectrum(int m, int family, double sigma2, double lambda, double nu_or_p,
                                   const double* fractions, int n_fractions, double tol_factor,
                                   int* J_out);
std::vector<double> build_spectrum_with(int m, int family, double sigma2, double lambda, double nu_or_p,
                                        const double* fractions, int n_fractions, double tol_factor, int* J_out,
                                        const std::function<std::vector<double>(int)>& attempt_spectrum);
void sqrt_spectra(const double* eig, int64_t s, int64_t k_trunc, std::vector<double>& full,
                  std::vector<double>& trunc);
}  // namespace osc

using namespace osc;

namespace {
thread_local std::string g_last_error;
}  // namespace

namespace osc {
// exception → osc_status, message kept for osc_last_error() of the calling thread
int c_api_error(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const osc::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const osc::SetupError& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return OSC_ERR_NUMERICAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return OSC_ERR_CONFIG;
  } catch (...) {
    g_last_error = "unknown error";
    return OSC_ERR_CONFIG;
  }
}
}  // namespace osc

namespace {
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return OSC_OK;
  } catch (...) {
    return c_api_error(std::current_exception());
  }
}

void set_device(Ctx* c) { OSC_CUDA(cudaSetDevice(c->device)); }

constexpr int kXiChunks = 4;  // host-ξ batches: up to 4 chunks, so only the first chunk's H2D is exposed

size_t budget_of(Ctx* c) {
  if (c->mem_budget) return c->mem_budget;
  size_t fr = 0, tot = 0;
  OSC_CUDA(cudaMemGetInfo(&fr, &tot));
  // what the context already holds is reusable
  size_t held = c->ce_inter.bytes + c->xi_dev.bytes + c->fields_fine.bytes + c->fields_coarse.bytes +
                c->solver.mem.bytes + c->out_q.bytes + c->out_i.bytes + c->xi_pref[0].bytes + c->xi_pref[1].bytes;
  return (size_t)(0.6 * (double)(fr + held));
}

void h2d(Ctx* c, void* dst, const void* src, size_t bytes) {
  OSC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
}
void d2h(Ctx* c, void* dst, const void* src, size_t bytes) {
  OSC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
}
}  // namespace

// ---- per-device kernel attributes ---------------------------------------------------------------
namespace osc {
void smem_attr_raw(const void* fn, size_t bytes) {
  // the attribute is a maximum: keep the largest size set so far per (device, kernel), never lower it
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set_max;
  int dev = 0;
  OSC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = set_max[{dev, fn}];
  if (bytes <= cur) return;
  OSC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  cur = bytes;
}
}  // namespace osc

// ---- profiling ---------------------------------------------------------------------------------
namespace osc {
int Ctx::stat_class(const char* name) {
  for (size_t i = 0; i < stats.size(); ++i)
    if (stats[i].name == name) return (int)i;
  stats.push_back(KernelStat{name});
  return (int)stats.size() - 1;
}

void Ctx::flush_stats() {
  for (auto& s : stats) {
    for (auto& pr : s.pending) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) s.total_ms += ms;
    }
    s.pending.clear();
  }
  ev_next = 0;  // every pooled event has been read: reuse them
}

cudaEvent_t Ctx::pool_event() {
  if (ev_next == ev_pool.size()) {
    cudaEvent_t e = nullptr;
    OSC_CUDA(cudaEventCreate(&e));
    ev_pool.push_back(e);
  }
  return ev_pool[ev_next++];
}

// Without profiling a scope only counts launches (no string work on the launch path). With OSC_NVTX=1
// (read at context creation) every scope is also an NVTX range named "<class>:<grid>" (SURVEY §5:
// NVTX ranges per kernel; ':' because '@' separates the domain in ncu's filter syntax), so ncu / nsys
// can select a kernel class at one grid size:
//   OSC_NVTX=1 ncu --nvtx --nvtx-include "mg_up.Lc:2048/" ...
KScope::KScope(Ctx* c, const char* name, int n_launches) : ctx(c), cls(-1) {
  c->launches += n_launches;
  if (c->nvtx) {
    const std::string full = c->tag.empty() ? std::string(name) : std::string(name) + ":" + c->tag;
    nvtxRangePushA(full.c_str());
  }
  if (!c->profiling) return;
  const std::string full = c->tag.empty() ? std::string(name) : std::string(name) + "@" + c->tag;
  cls = c->stat_class(full.c_str());
  c->stats[cls].launches += n_launches;
  if (!c->profile_only.empty() && c->profile_only != full) return;
  e0 = c->pool_event();
  e1 = c->pool_event();
  cudaEventRecord(e0, c->stream);
}

KScope::~KScope() {
  if (ctx->nvtx) nvtxRangePop();
  if (e0) {
    cudaEventRecord(e1, ctx->stream);
    ctx->stats[cls].pending.emplace_back(e0, e1);
  }
}
}  // namespace osc

extern "C" {

const char* osc_last_error(void) { return g_last_error.c_str(); }

int osc_ctx_create(int device, osc_ctx** out) {
  return guarded([&] {
    OSC_REQUIRE(out != nullptr, "osc_ctx_create: null out");
    if (device < 0) OSC_CUDA(cudaGetDevice(&device));  // the calling thread's current device
    auto* c = new osc_ctx();
    c->device = device;
    const char* nv = std::getenv("OSC_NVTX");
    c->nvtx = nv && std::atoi(nv) != 0;
    try {
      OSC_CUDA(cudaSetDevice(device));
      OSC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      OSC_CUDA(cudaHostAlloc(&c->h_pinned_int, 64, cudaHostAllocDefault));
      OSC_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
      for (int i = 0; i < 4; ++i) OSC_CUDA(cudaEventCreateWithFlags(&c->ev_poll[i], cudaEventDisableTiming));
      for (int i = 0; i < 2; ++i) {
        OSC_CUDA(cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming));
        OSC_CUDA(cudaEventCreateWithFlags(&c->ev_ce_done[i], cudaEventDisableTiming));
      }
      for (int t = 0; t < 2; ++t) {
        OSC_CUDA(cudaEventCreateWithFlags(&c->ev_pref_read[t], cudaEventDisableTiming));
        for (int j = 0; j < Ctx::kPrefParts; ++j)
          OSC_CUDA(cudaEventCreateWithFlags(&c->ev_pref_part[t][j], cudaEventDisableTiming));
      }
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void osc_ctx_destroy(osc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->flush_stats();
  cudaStreamSynchronize(c->copy_stream);
  for (DevBuf* b : {&c->ce_inter, &c->xi_dev, &c->fields_fine, &c->fields_coarse, &c->out_q,
                    &c->out_i, &c->tmp_host_stage, &c->sums, &c->solver.mem, &c->xi_pref[0], &c->xi_pref[1],
                    &c->retry_k, &c->retry_q})
    b->release();
  for (int t = 0; t < 2; ++t) {
    if (c->ev_pref_read[t]) cudaEventDestroy(c->ev_pref_read[t]);
    for (int j = 0; j < Ctx::kPrefParts; ++j)
      if (c->ev_pref_part[t][j]) cudaEventDestroy(c->ev_pref_part[t][j]);
  }
  if (c->h_pinned_int) cudaFreeHost(c->h_pinned_int);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (int i = 0; i < 4; ++i)
    if (c->ev_poll[i]) cudaEventDestroy(c->ev_poll[i]);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
    if (c->ev_ce_done[i]) cudaEventDestroy(c->ev_ce_done[i]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  cudaStreamDestroy(c->stream);
  delete c;
}

void* osc_ctx_stream(osc_ctx* c) { return c ? (void*)c->stream : nullptr; }

int osc_ctx_synchronize(osc_ctx* c) {
  return guarded([&] {
    set_device(c);
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    c->flush_stats();
  });
}

int osc_level_prefetch_xi(osc_level* next_level, const double* xi_next, int64_t count) {
  return guarded([&] {
    OSC_REQUIRE(next_level && next_level->ctx, "osc_level_prefetch_xi: null level");
    OSC_REQUIRE(count >= 0, "osc_level_prefetch_xi: negative count");
    Ctx* c = next_level->ctx;
    const bool on = count > 0 && xi_next != nullptr;
    c->next_xi = on ? xi_next : nullptr;
    c->next_count = on ? count : 0;
    c->next_s = on ? next_level->s : 0;
  });
}

int osc_ctx_set_mem_budget(osc_ctx* c, size_t bytes) {
  c->mem_budget = bytes;
  return OSC_OK;
}

int osc_ctx_set_profiling(osc_ctx* c, int on) {
  return guarded([&] {
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    c->flush_stats();
    c->profiling = on != 0;
  });
}

int osc_ctx_profile_only(osc_ctx* c, const char* kernel_class) {
  return guarded([&] {
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    c->flush_stats();
    c->profile_only = kernel_class ? kernel_class : "";
  });
}

int osc_ctx_kernel_stats(osc_ctx* c, int i, const char** name, int64_t* launches, double* total_ms) {
  if (i < 0 || i >= (int)c->stats.size()) return OSC_ERR_CONFIG;
  if (name) *name = c->stats[i].name.c_str();
  if (launches) *launches = c->stats[i].launches;
  if (total_ms) *total_ms = c->stats[i].total_ms;
  return OSC_OK;
}

int osc_ctx_reset_stats(osc_ctx* c) {
  return guarded([&] {
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    c->flush_stats();
    for (auto& s : c->stats) {
      s.launches = 0;
      s.total_ms = 0.0;
    }
  });
}

int64_t osc_ctx_launch_count(osc_ctx* c) { return c ? c->launches : 0; }

void* osc_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) return nullptr;
  return p;
}
void osc_host_free(void* p) {
  if (p) cudaFreeHost(p);
}
void osc_free(void* p) { std::free(p); }

// ---- level setup -----------------------------------------------------------------------------
int osc_build_spectrum(int m, int family, double sigma2, double lambda, double nu_or_p,
                       const double* fractions, int n_fractions, double tol_spd_factor, int* J_out,
                       int64_t* s_out, double** eig_out) {
  return guarded([&] {
    OSC_REQUIRE(family == OSC_COV_MATERN || family == OSC_COV_SEPARABLE_EXP,
                "osc_build_spectrum: unknown covariance family");
    int J = 0;
    std::vector<double> eig = build_spectrum(m, family, sigma2, lambda, nu_or_p, fractions,
                                             n_fractions, tol_spd_factor, &J);
    if (J_out) *J_out = J;
    if (s_out) *s_out = (int64_t)eig.size();
    if (eig_out) {
      double* buf = static_cast<double*>(std::malloc(sizeof(double) * eig.size()));
      if (!buf) throw std::bad_alloc();
      std::memcpy(buf, eig.data(), sizeof(double) * eig.size());
      *eig_out = buf;
    }
  });
}

int osc_build_spectrum_device(osc_ctx* c, int m, int family, double sigma2, double lambda, double nu_or_p,
                              const double* fractions, int n_fractions, double tol_spd_factor, int* J_out,
                              int64_t* s_out, double** eig_out) {
  return guarded([&] {
    OSC_REQUIRE(c, "osc_build_spectrum_device: null context");
    OSC_REQUIRE(family == OSC_COV_MATERN || family == OSC_COV_SEPARABLE_EXP,
                "osc_build_spectrum_device: unknown covariance family");
    OSC_REQUIRE(spectrum_device_supported(family, nu_or_p),
                "osc_build_spectrum_device: Matern nu must lie in (0, 64] (use osc_build_spectrum)");
    set_device(c);
    int J = 0;
    std::vector<double> eig = build_spectrum_with(
        m, family, sigma2, lambda, nu_or_p, fractions, n_fractions, tol_spd_factor, &J,
        [&](int Jt) { return spectrum_device(c, m, Jt, family, sigma2, lambda, nu_or_p); });
    if (J_out) *J_out = J;
    if (s_out) *s_out = (int64_t)eig.size();
    if (eig_out) {
      double* buf = static_cast<double*>(std::malloc(sizeof(double) * eig.size()));
      if (!buf) throw std::bad_alloc();
      std::memcpy(buf, eig.data(), sizeof(double) * eig.size());
      *eig_out = buf;
    }
  });
}

int osc_level_create(osc_ctx* c, int m, int J, const double* eigenvalues, int64_t k_trunc,
                     osc_level** out) {
  return guarded([&] {
    OSC_REQUIRE(c && out && eigenvalues, "osc_level_create: null argument");
    OSC_REQUIRE(m >= 1 && J >= 0, "osc_level_create: m >= 1, J >= 0 required");
    set_device(c);
    auto* L = new osc_level();
    L->ctx = c;
    L->m = m;
    L->J = J;
    L->n = 2 * (m + J);
    L->s = (int64_t)L->n * L->n;
    OSC_REQUIRE(k_trunc >= 0 && k_trunc < L->s,
                "truncated: k must lie in [0, s); at least one mode must survive");
    L->k_trunc = k_trunc;
    try {
      std::vector<double> full, trunc;
      sqrt_spectra(eigenvalues, L->s, k_trunc, full, trunc);
      L->sqrt_full.ensure(sizeof(double) * L->s);
      OSC_CUDA(cudaMemcpy(L->sqrt_full.p, full.data(), sizeof(double) * L->s, cudaMemcpyHostToDevice));
      if (k_trunc > 0) {
        L->sqrt_trunc.ensure(sizeof(double) * L->s);
        OSC_CUDA(cudaMemcpy(L->sqrt_trunc.p, trunc.data(), sizeof(double) * L->s, cudaMemcpyHostToDevice));
      }
      upload_twiddles(L);
    } catch (...) {
      L->sqrt_full.release();
      L->sqrt_trunc.release();
      L->twiddle.release();
      delete L;
      throw;
    }
    *out = L;
  });
}

void osc_level_destroy(osc_level* L) {
  if (!L) return;
  cudaSetDevice(L->ctx->device);
  cudaStreamSynchronize(L->ctx->stream);
  for (DevBuf* b : {&L->sqrt_full, &L->sqrt_trunc, &L->twiddle, &L->eig, &L->perm, &L->sqrt_comp, &L->run_sums})
    b->release();
  delete L;
}

int osc_level_info(const osc_level* L, int* m, int* J, int* n, int64_t* s, int64_t* k_trunc) {
  if (!L) return OSC_ERR_CONFIG;
  if (m) *m = L->m;
  if (J) *J = L->J;
  if (n) *n = L->n;
  if (s) *s = L->s;
  if (k_trunc) *k_trunc = L->k_trunc;
  return OSC_OK;
}

// ---- the fused per-level batch -----------------------------------------------------------------
}  // extern "C"

namespace osc {
// Body of osc_level_draws without the error mapping: returns (any non-finite field, any solver
// failure). hist_cap > 0 keeps every solve's residual history (the failure re-run below);
// hist_out (host, hist_cap per solve) then receives the fine solve's history, hist_coarse the
// coarse one's. level_sums: this call's sums (per-call semantics of the header); with the level's
// running sums enabled they are also added to L->run_sums on the device.
std::pair<bool, bool> draws_impl(Level* L, const osc_problem* prob, uint64_t seed, uint32_t ell, int64_t from,
                                 int64_t to, int flags, const double* xi, double* q_fine, double* q_coarse,
                                 int32_t* iters_fine, int32_t* iters_coarse, int32_t* status, double* level_sums,
                                 int hist_cap, double* hist_fine, double* hist_coarse) {
  {
    OSC_REQUIRE(L && prob, "osc_level_draws: null argument");
    OSC_REQUIRE(to >= from && from >= 0, "osc_level_draws: need 0 <= from <= to");
    OSC_REQUIRE(prob->bc == OSC_BC_FLOWCELL || prob->bc == OSC_BC_DIRICHLET_ALL, "unknown bc");
    OSC_REQUIRE(prob->qoi >= OSC_QOI_POINT && prob->qoi <= OSC_QOI_FLUX, "unknown qoi");
    OSC_REQUIRE(!(prob->qoi == OSC_QOI_POINT && (prob->qoi_x < 0 || prob->qoi_x > 1 ||
                                                 prob->qoi_y < 0 || prob->qoi_y > 1)),
                "qoi_point: point outside [0,1]^2");
    Ctx* c = L->ctx;
    set_device(c);
    const int64_t count = to - from;
    if (count == 0) {
      if (level_sums) {  // an empty shard still contributes zeros (group / comm reductions)
        c->sums.ensure(sizeof(double) * 8);
        OSC_CUDA(cudaMemsetAsync(c->sums.p, 0, sizeof(double) * 8, c->stream));
        for (int j = 0; j < 5; ++j) level_sums[j] = 0.0;
      }
      return {false, false};
    }
    const bool has_coarse = (flags & OSC_DRAW_HAS_COARSE) != 0;
    OSC_REQUIRE(!has_coarse || (L->m % 2 == 0 && L->m >= 2),
                "restrict: target grid is not a nested coarsening");
    // coupled_sample: the smoothed operator is used only when it exists (estimators.cpp:211-223)
    const double* sq_f = (flags & OSC_DRAW_TRUNC_FINE) && L->k_trunc > 0 ? L->sqrt_trunc.as<double>()
                                                                         : L->sqrt_full.as<double>();
    const double* sq_c = (flags & OSC_DRAW_TRUNC_COARSE) && L->k_trunc > 0 ? L->sqrt_trunc.as<double>()
                                                                           : L->sqrt_full.as<double>();
    const bool shared_field = sq_f == sq_c;
    const int m = L->m, mc = m / 2;
    const int64_t Nf = (int64_t)(m + 1) * (m + 1), Nc = (int64_t)(mc + 1) * (mc + 1);
    const bool xi_host = xi != nullptr && !(flags & OSC_DRAW_XI_DEVICE);
    // batch size from the memory budget
    size_t per = sizeof(double) * (Nf + (has_coarse ? Nc : 0)) + ce_inter_bytes(L, 1, 1) +
                 solver_bytes(m, 1, 0) + 64;
    if (xi_host) per += sizeof(double) * L->s;
    // cross-call prefetch (osc_level_prefetch_xi): this call's rows may already be resident in
    // xi_pref (copied under the previous call's solves), and the next call's rows may be armed
    const bool arm = xi_host && c->next_xi != nullptr && c->next_count > 0 && c->next_s > 0;
    const bool pref_hit = xi_host && c->pref_xi == xi && c->pref_count == count && c->pref_s == L->s;
    if (xi_host && !pref_hit) c->pref_xi = nullptr;  // stale rows: dropped (the copy stream orders reuse)
    if (arm || pref_hit) per += 2 * sizeof(double) * L->s;
    const size_t budget = budget_of(c);
    int64_t Bmax = std::max<int64_t>(1, (int64_t)(budget / per));
    Bmax = std::min<int64_t>(Bmax, 1 << 16);
    constexpr int NP = Ctx::kPrefParts;
    const int cur = c->pref_slot;  // the buffer holding this call's prefetched rows
    // whole-batch mode: the rows have arrived, so one chunk (full batch, no per-chunk overhead);
    // parts mode: they are still arriving (the copy engine is behind, e.g. right after a start-up
    // call that copied its own rows and the next batch's), so the call runs part by part as they land
    bool pref_ready = false;
    int64_t max_part = 0;
    if (pref_hit) {
      const cudaError_t q = cudaEventQuery(c->ev_pref_part[cur][NP - 1]);
      if (q != cudaSuccess && q != cudaErrorNotReady) OSC_CUDA(q);
      pref_ready = q == cudaSuccess;
      for (int j = 0; j < NP; ++j) max_part = std::max(max_part, c->pref_part_end[j] - (j ? c->pref_part_end[j - 1] : 0));
    }
    const bool whole = pref_hit && count <= Bmax && pref_ready;
    const bool parts = pref_hit && !whole && max_part <= Bmax;
    if (pref_hit && !whole && !parts) c->pref_xi = nullptr;  // not consumed: never reused by a later call
    const bool from_pref = whole || parts;
    const bool xi_chunked = xi_host && !from_pref;
    int64_t nchunks = (count + Bmax - 1) / Bmax;
    // host ξ: several chunks, so chunk i+1's H2D copy (copy stream, double-buffered) runs under
    // chunk i's solve and only the first chunk's copy is exposed (up to 4 chunks of ≥ 8 samples);
    // device ξ / Philox: one chunk when it fits
    if (xi_chunked && count >= 2)
      nchunks = std::max<int64_t>(nchunks, std::min<int64_t>(kXiChunks, std::max<int64_t>(2, count / 8)));
    const int Bc = (int)((count + nchunks - 1) / nchunks);
    // chunk schedule. Host ξ with large uniform chunks (≥ 256 MB of ξ each): a ramp — a small
    // first chunk (its copy is the only exposed one), then each chunk ≤ OSC_XI_RAMP × the previous,
    // so chunk i+1's copy still fits under chunk i's solves (copy ≈ 0.6 × solve per sample on
    // cfg 4), capped at the uniform size Bc. Small ξ (cfg 1) keeps the uniform chunks: there the
    // per-chunk launch overhead outweighs the exposed copy.
    std::vector<std::pair<int64_t, int>> sched;
    {
      auto env_num = [](const char* k, double d) { const char* v = std::getenv(k); return v ? std::atof(v) : d; };
      const double ramp = 1.35;
      const int first_div = 16;
      const double min_mb = env_num("OSC_XI_RAMP_MIN_MB", 256);  // tests lower it to reach the ramp
      int sz = Bc;
      const bool big = sizeof(double) * (double)L->s * Bc >= min_mb * (1 << 20);
      if (xi_chunked && big && first_div > 0 && ramp > 1.0 && count >= 16)
        sz = (int)std::max<int64_t>(1, std::min<int64_t>(Bc, count / first_div));
      if (parts) {
        for (int j = 0; j < NP; ++j) {
          const int64_t a = j ? c->pref_part_end[j - 1] : 0;
          if (c->pref_part_end[j] > a) sched.emplace_back(a, (int)(c->pref_part_end[j] - a));
        }
      } else {
        for (int64_t a = 0; a < count;) {
          const int nb = (int)std::min<int64_t>(sz, count - a);
          sched.emplace_back(a, nb);
          a += nb;
          sz = std::min(Bc, std::max(sz + 1, (int)std::ceil(sz * ramp)));
        }
      }
    }
    c->fields_fine.ensure(sizeof(double) * Nf * Bc);
    if (has_coarse) c->fields_coarse.ensure(sizeof(double) * Nc * Bc);
    c->out_q.ensure(sizeof(double) * 2 * Bc);
    c->out_i.ensure(sizeof(int) * 2 * Bc);
    c->sums.ensure(sizeof(double) * 8);
    if (xi_chunked) c->xi_dev.ensure(2 * sizeof(double) * L->s * Bc);
    auto xi_buf = [&](int64_t chunk) { return c->xi_dev.as<double>() + (chunk & 1) * L->s * Bc; };
    auto issue_copy = [&](int64_t chunk) {  // H2D of chunk `chunk` on the copy stream
      if (chunk >= (int64_t)sched.size()) return;
      const int64_t a = sched[chunk].first;
      const int64_t nb = sched[chunk].second;
      if (chunk >= 2)  // the CE of chunk-2 used this buffer
        OSC_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev_ce_done[chunk & 1], 0));
      OSC_CUDA(cudaMemcpyAsync(xi_buf(chunk), xi + a * L->s, sizeof(double) * L->s * nb,
                               cudaMemcpyHostToDevice, c->copy_stream));
      OSC_CUDA(cudaEventRecord(c->ev_copied[chunk & 1], c->copy_stream));
    };
    // the armed next call's rows → the other prefetch buffer, in NP parts, queued on the copy stream
    // behind this call's own copies and after the last read of that buffer (ev_pref_read)
    auto issue_prefetch = [&] {
      if (!arm) return;
      const int nxt = 1 - cur;
      const int64_t rows = c->next_count, sn = c->next_s;
      const size_t bytes = sizeof(double) * sn * rows;
      if (c->xi_pref[nxt].bytes < bytes) {
        OSC_CUDA(cudaStreamSynchronize(c->copy_stream));
        c->xi_pref[nxt].ensure(bytes);
      }
      OSC_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev_pref_read[nxt], 0));
      for (int j = 0; j < NP; ++j) {
        const int64_t a = rows * j / NP, e = rows * (j + 1) / NP;
        if (e > a)
          OSC_CUDA(cudaMemcpyAsync(c->xi_pref[nxt].as<double>() + a * sn, c->next_xi + a * sn,
                                   sizeof(double) * sn * (e - a), cudaMemcpyHostToDevice, c->copy_stream));
        OSC_CUDA(cudaEventRecord(c->ev_pref_part[nxt][j], c->copy_stream));
        c->pref_part_end[j] = e;
      }
      c->pref_slot = nxt;
      c->pref_xi = c->next_xi;
      c->pref_count = rows;
      c->pref_s = sn;
      c->next_xi = nullptr;
      c->next_count = 0;
      c->next_s = 0;
    };
    if (xi_chunked) {
      issue_copy(0);
      if (sched.size() == 1) issue_prefetch();
    } else if (from_pref) {
      issue_prefetch();  // nothing of this call's own is queued on the copy stream
    }
    double* xi_cur = from_pref ? c->xi_pref[cur].as<double>() : nullptr;
    double* d_qf = c->out_q.as<double>();
    double* d_qc = d_qf + Bc;
    int* d_bad = c->out_i.as<int>();
    double* d_sums = c->sums.as<double>();
    if (level_sums) {
      OSC_CUDA(cudaMemsetAsync(d_sums, 0, sizeof(double) * 8, c->stream));
    }
    bool any_bad = false, any_fail = false;
    std::vector<int32_t> it_tmp(Bc), st_tmp(Bc), bad_tmp(Bc);
    constexpr bool nested = true;  // the fine solve starts from the prolonged coarse solution
    for (int64_t chunk = 0; chunk < (int64_t)sched.size(); ++chunk) {
      const int64_t c0 = sched[chunk].first;
      const int B = sched[chunk].second;
      const double* xi_chunk = nullptr;
      if (xi) {
        if (from_pref) {
          OSC_CUDA(cudaStreamWaitEvent(c->stream, c->ev_pref_part[cur][whole ? NP - 1 : chunk], 0));
          xi_chunk = xi_cur + c0 * L->s;
        } else if (xi_host) {
          OSC_CUDA(cudaStreamWaitEvent(c->stream, c->ev_copied[chunk & 1], 0));
          xi_chunk = xi_buf(chunk);
        } else {
          xi_chunk = xi + c0 * L->s;
        }
      }
      OSC_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int) * B, c->stream));
      double* kf = c->fields_fine.as<double>();
      double* kc = has_coarse ? c->fields_coarse.as<double>() : nullptr;
      const uint64_t idx0 = (uint64_t)(from + c0);
      if (shared_field || !has_coarse) {
        ce_sample_launch(c, L, sq_f, xi_chunk, seed, ell, idx0, B, true, kf, kc, d_bad);
      } else {
        ce_sample_launch(c, L, sq_f, xi_chunk, seed, ell, idx0, B, true, kf, nullptr, d_bad);
        ce_sample_launch(c, L, sq_c, xi_chunk, seed, ell, idx0, B, true, nullptr, kc, d_bad);
      }
      if (from_pref) {
        if (chunk + 1 == (int64_t)sched.size()) {  // the prefetch buffer consumed: a later prefetch may refill it
          OSC_CUDA(cudaEventRecord(c->ev_pref_read[cur], c->stream));
          if (c->pref_slot == cur) c->pref_xi = nullptr;  // (a prefetch issued by this call lives in the other slot)
        }
      } else if (xi_host) {  // ξ buffer consumed: start the next chunk's copy under this chunk's solves
        OSC_CUDA(cudaEventRecord(c->ev_ce_done[chunk & 1], c->stream));
        issue_copy(chunk + 1);
        if (chunk + 1 == (int64_t)sched.size() - 1) issue_prefetch();
      }
      // Coupled draws solve the coarse field first: its solution, prolonged (P1), starts the fine
      // PCG (nested iteration), which then needs fewer iterations to the same 1e-10 stopping test.
      // The coarse conductivity buffer holds the guess once the coarse QoI has been evaluated.
      std::vector<int32_t> itc_tmp(B), stc_tmp(B);
      const double* guess = nullptr;
      if (has_coarse) {
        solver_prepare(c, mc, B, hist_cap);
        c->solver.lev[0].k = kc;
        solver_run(c, prob, B);
        qoi_launch(c, prob, B, d_qc);
        solver_results(c, B, itc_tmp.data(), stc_tmp.data(), hist_coarse);
        if (nested) {
          OSC_CUDA(cudaMemcpyAsync(kc, c->solver.u, sizeof(double) * Nc * B, cudaMemcpyDeviceToDevice, c->stream));
          guess = kc;
        }
      }
      // fine solve + QoI
      solver_prepare(c, m, B, hist_cap);
      c->solver.lev[0].k = kf;
      solver_run(c, prob, B, guess);
      qoi_launch(c, prob, B, d_qf);
      solver_results(c, B, it_tmp.data(), st_tmp.data(), hist_fine);
      if (guess) {
        // A nested start that fails to converge (rare: ~1 in 2·10⁴ config-3 samples, where the
        // one-reduction recurrence loses conjugacy) is re-solved from the reference's Dirichlet lift
        // (fem.cpp:335-339): the failing samples' fields are compacted into a small batch.
        std::vector<int> redo;
        for (int b = 0; b < B; ++b)
          if (st_tmp[b] == OSC_ERR_SOLVER) redo.push_back(b);
        if (!redo.empty()) {
          const int nr = (int)redo.size();
          c->retry_k.ensure(sizeof(double) * Nf * nr);
          c->retry_q.ensure(sizeof(double) * nr);
          double* rk = c->retry_k.as<double>();
          for (int j = 0; j < nr; ++j)
            OSC_CUDA(cudaMemcpyAsync(rk + (int64_t)j * Nf, kf + (int64_t)redo[j] * Nf, sizeof(double) * Nf,
                                     cudaMemcpyDeviceToDevice, c->stream));
          solver_prepare(c, m, nr, hist_cap);
          c->solver.lev[0].k = rk;
          solver_run(c, prob, nr, nullptr);
          qoi_launch(c, prob, nr, c->retry_q.as<double>());
          std::vector<int32_t> itr(nr), str(nr);
          solver_results(c, nr, itr.data(), str.data(), nullptr);
          for (int j = 0; j < nr; ++j) {
            OSC_CUDA(cudaMemcpyAsync(d_qf + redo[j], c->retry_q.as<double>() + j, sizeof(double),
                                     cudaMemcpyDeviceToDevice, c->stream));
            it_tmp[redo[j]] = itr[j];
            st_tmp[redo[j]] = str[j];
          }
        }
      }
      d2h(c, bad_tmp.data(), d_bad, sizeof(int) * B);
      OSC_CUDA(cudaStreamSynchronize(c->stream));
      for (int b = 0; b < B; ++b) {
        int s = bad_tmp[b] ? OSC_ERR_NUMERICAL : st_tmp[b];
        any_bad |= bad_tmp[b] != 0;
        any_fail |= st_tmp[b] != 0;
        if (iters_fine) iters_fine[c0 + b] = it_tmp[b];
        if (status) status[c0 + b] = s;
      }
      if (has_coarse) {
        for (int b = 0; b < B; ++b) {
          any_fail |= stc_tmp[b] != 0;
          if (iters_coarse) iters_coarse[c0 + b] = itc_tmp[b];
          if (status && status[c0 + b] == 0) status[c0 + b] = stc_tmp[b];
        }
      }
      if (level_sums)
        level_sums_launch(c, d_qf, has_coarse ? d_qc : nullptr, B, level_sums[5], level_sums[6], d_sums);
      if (L->sums_on)
        level_sums_launch(c, d_qf, has_coarse ? d_qc : nullptr, B, L->shift_y, L->shift_q, L->run_sums.as<double>());
      if (q_fine) d2h(c, q_fine + c0, d_qf, sizeof(double) * B);
      if (q_coarse) {
        if (has_coarse) d2h(c, q_coarse + c0, d_qc, sizeof(double) * B);
        else std::memset(q_coarse + c0, 0, sizeof(double) * B);
      }
    }
    if (level_sums) d2h(c, level_sums, d_sums, sizeof(double) * 5);
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    c->flush_stats();
    return {any_bad, any_fail};
  }
}

// The error mapping of osc_level_draws (also used by the group's per-device workers). A solver
// failure with osc_ctx_set_history on re-draws the first failing slot alone with the residual history
// kept: sample i is a pure function of (seed, ℓ, i) (or xi row i), so the re-run repeats the failure
// bit for bit and SolverError can carry the reference's residual_history (fem.cpp:359-379).
void draws_checked(Level* L, const osc_problem* prob, uint64_t seed, uint32_t ell, int64_t from, int64_t to,
                   int flags, const double* xi, double* q_fine, double* q_coarse, int32_t* iters_fine,
                   int32_t* iters_coarse, int32_t* status, double* level_sums) {
  OSC_REQUIRE(L, "osc_level_draws: null level");
  Ctx* c = L->ctx;
  std::vector<int32_t> st_local;
  if (!status && c->hist_req > 0 && to > from) {
    st_local.resize((size_t)(to - from));
    status = st_local.data();
  }
  const auto r = draws_impl(L, prob, seed, ell, from, to, flags, xi, q_fine, q_coarse, iters_fine, iters_coarse,
                            status, level_sums, 0, nullptr, nullptr);
  if (r.first) throw osc::Error(OSC_ERR_NUMERICAL, "assemble_and_solve: non-finite log-field value");
  if (!r.second) return;
  c->fail_slot = -1;
  c->fail_hist.clear();
  if (c->hist_req > 0) {
    int64_t i = from;
    while (i < to && status[i - from] != OSC_ERR_SOLVER) ++i;
    if (i < to) {
      const int cap = c->hist_req;
      std::vector<double> hf(cap, 0.0), hc(cap, 0.0);
      double qf1, qc1;
      int32_t itf1, itc1, st1;
      const double* xi1 = xi ? xi + (i - from) * L->s : nullptr;
      const bool host_pref = c->next_xi != nullptr;  // keep an armed prefetch for the caller's next call
      const double* nx = c->next_xi;
      const int64_t ncount = c->next_count, ns = c->next_s;
      c->next_xi = nullptr;
      draws_impl(L, prob, seed, ell, i, i + 1, flags, xi1, &qf1, &qc1, &itf1, &itc1, &st1, nullptr, cap, hf.data(),
                 hc.data());
      if (host_pref) {
        c->next_xi = nx;
        c->next_count = ncount;
        c->next_s = ns;
      }
      // the failing solve's history (entries after the last iteration stay 0): the fine one when its
      // last recorded ‖r‖/‖b‖ is above tol, else the coarse one
      auto len_of = [&](const std::vector<double>& h) {
        int n = 1;
        while (n < cap && h[n] != 0.0) ++n;
        return n;
      };
      const int lf = len_of(hf);
      const bool fine_failed = !(hf[lf - 1] <= prob->tol);
      const std::vector<double>& h = fine_failed ? hf : hc;
      c->fail_slot = i;
      c->fail_hist.assign(h.begin(), h.begin() + (fine_failed ? lf : len_of(hc)));
    }
  }
  throw osc::Error(OSC_ERR_SOLVER, "CG did not reach the relative residual within the iteration cap");
}
}  // namespace osc

extern "C" {

int osc_level_draws(osc_level* L, const osc_problem* prob, uint64_t seed, uint32_t ell,
                    int64_t from, int64_t to, int flags, const double* xi, double* q_fine,
                    double* q_coarse, int32_t* iters_fine, int32_t* iters_coarse, int32_t* status,
                    double* level_sums) {
  return guarded([&] {
    draws_checked(L, prob, seed, ell, from, to, flags, xi, q_fine, q_coarse, iters_fine, iters_coarse, status,
                  level_sums);
  });
}

int osc_ctx_set_history(osc_ctx* c, int hist_cap) {
  return guarded([&] {
    OSC_REQUIRE(c && hist_cap >= 0, "osc_ctx_set_history: null context or negative cap");
    c->hist_req = hist_cap;
  });
}

int osc_ctx_failure_history(osc_ctx* c, int64_t* slot, double* out, int cap) {
  if (!c) return -1;
  if (slot) *slot = c->fail_slot;
  const int n = (int)c->fail_hist.size();
  for (int j = 0; j < std::min(n, cap); ++j) out[j] = c->fail_hist[j];
  return n;
}

int osc_level_sums_reset(osc_level* L, double shift_y, double shift_q) {
  return guarded([&] {
    OSC_REQUIRE(L, "osc_level_sums_reset: null level");
    set_device(L->ctx);
    L->run_sums.ensure(sizeof(double) * 16);
    OSC_CUDA(cudaMemsetAsync(L->run_sums.p, 0, sizeof(double) * 16, L->ctx->stream));
    L->shift_y = shift_y;
    L->shift_q = shift_q;
    L->sums_on = true;
  });
}

int osc_level_sums_reshift(osc_level* L, double shift_y, double shift_q) {
  return guarded([&] {
    OSC_REQUIRE(L, "osc_level_sums_reshift: null level");
    OSC_REQUIRE(L->sums_on, "osc_level_sums_reshift: running sums not enabled (osc_level_sums_reset)");
    set_device(L->ctx);
    level_sums_reshift_launch(L->ctx, L->run_sums.as<double>(), shift_y - L->shift_y, shift_q - L->shift_q);
    L->shift_y = shift_y;
    L->shift_q = shift_q;
  });
}

int osc_level_sums_read(osc_level* L, double out[7]) {
  return guarded([&] {
    OSC_REQUIRE(L && out, "osc_level_sums_read: null argument");
    OSC_REQUIRE(L->sums_on, "osc_level_sums_read: running sums not enabled (osc_level_sums_reset)");
    set_device(L->ctx);
    d2h(L->ctx, out, L->run_sums.p, sizeof(double) * 5);
    OSC_CUDA(cudaStreamSynchronize(L->ctx->stream));
    out[5] = L->shift_y;
    out[6] = L->shift_q;
  });
}


int osc_summarize(const double* qf, const double* qc, int64_t n, int has_coarse, double out[5]) {
  // moments_of (estimators.cpp:82-101), slot order
  double mean_y = 0.0, mean_q = 0.0, m2y = 0.0, m2q = 0.0;
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double y = has_coarse ? qf[i] - qc[i] : qf[i];
    ++cnt;
    double d = y - mean_y;
    mean_y += d / cnt;
    m2y += d * (y - mean_y);
    d = qf[i] - mean_q;
    mean_q += d / cnt;
    m2q += d * (qf[i] - mean_q);
  }
  out[0] = (double)cnt;
  out[1] = mean_y;
  out[2] = cnt >= 2 ? m2y / (cnt - 1) : 0.0;
  out[3] = mean_q;
  out[4] = cnt >= 2 ? m2q / (cnt - 1) : 0.0;
  return OSC_OK;
}

// ---- unfused stages ------------------------------------------------------------------------------
int osc_normals(osc_ctx* c, uint64_t seed, uint32_t ell, uint64_t index0, int64_t count, int64_t s,
                double* out) {
  return guarded([&] {
    set_device(c);
    OSC_REQUIRE(count >= 0 && s >= 0, "osc_normals: negative size");
    if (count == 0 || s == 0) return;
    c->xi_dev.ensure(sizeof(double) * s * count);
    normals_launch(c, seed, ell, index0, (int)count, s, c->xi_dev.as<double>());
    d2h(c, out, c->xi_dev.p, sizeof(double) * s * count);
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    c->flush_stats();
  });
}

int osc_ce_sample(osc_level* L, const double* xi, uint64_t seed, uint32_t ell, uint64_t index0,
                  int64_t count, int flags, double* fine_out, double* coarse_out) {
  return guarded([&] {
    Ctx* c = L->ctx;
    set_device(c);
    if (count <= 0) return;
    const bool want_f = (flags & OSC_CE_FINE) != 0, want_c = (flags & OSC_CE_COARSE) != 0;
    const bool dev_out = (flags & OSC_CE_DEVICE_OUT) != 0, dev_xi = (flags & OSC_CE_XI_DEVICE) != 0;
    OSC_REQUIRE(want_f || want_c, "osc_ce_sample: request FINE and/or COARSE output");
    OSC_REQUIRE(!want_c || L->m % 2 == 0, "restrict: target grid is not a nested coarsening");
    OSC_REQUIRE(!(flags & OSC_CE_TRUNCATED) || L->k_trunc > 0, "osc_ce_sample: level has no truncated spectrum");
    OSC_REQUIRE(!dev_out || ((!want_f || fine_out) && (!want_c || coarse_out)),
                "osc_ce_sample: OSC_CE_DEVICE_OUT needs device output pointers");
    const double* sq = (flags & OSC_CE_TRUNCATED) ? L->sqrt_trunc.as<double>() : L->sqrt_full.as<double>();
    const int m = L->m, mc = m / 2;
    const int64_t Nf = (int64_t)(m + 1) * (m + 1), Nc = (int64_t)(mc + 1) * (mc + 1);
    // host-facing calls stage through device buffers in chunks bounded by the memory budget
    const size_t per = (size_t)(dev_out ? 0 : 8 * (Nf * want_f + Nc * want_c)) +
                       (size_t)((xi && !dev_xi) ? 8 * L->s : 0) + ce_inter_bytes(L, 1, 1) + 64;
    int64_t chunk = dev_out && (!xi || dev_xi) ? count
                                               : std::max<int64_t>(1, std::min<int64_t>(count, budget_of(c) / per));
    if (!dev_out) {
      if (want_f) c->fields_fine.ensure(sizeof(double) * Nf * chunk);
      if (want_c) c->fields_coarse.ensure(sizeof(double) * Nc * chunk);
    }
    if (xi && !dev_xi) c->xi_dev.ensure(sizeof(double) * L->s * chunk);
    c->out_i.ensure(sizeof(int) * count);
    OSC_CUDA(cudaMemsetAsync(c->out_i.p, 0, sizeof(int) * count, c->stream));
    for (int64_t c0 = 0; c0 < count; c0 += chunk) {
      const int64_t cnt = std::min<int64_t>(chunk, count - c0);
      const double* xd = nullptr;
      if (xi) {
        if (dev_xi) {
          xd = xi + c0 * L->s;
        } else {
          h2d(c, c->xi_dev.p, xi + c0 * L->s, sizeof(double) * L->s * cnt);
          xd = c->xi_dev.as<double>();
        }
      }
      double* of = want_f ? (dev_out ? fine_out + c0 * Nf : c->fields_fine.as<double>()) : nullptr;
      double* oc = want_c ? (dev_out ? coarse_out + c0 * Nc : c->fields_coarse.as<double>()) : nullptr;
      ce_sample_launch(c, L, sq, xd, seed, ell, index0 + (uint64_t)c0, (int)cnt, (flags & OSC_CE_EXP) != 0,
                       of, oc, c->out_i.as<int>() + c0);
      if (!dev_out) {
        if (want_f && fine_out) d2h(c, fine_out + c0 * Nf, of, sizeof(double) * Nf * cnt);
        if (want_c && coarse_out) d2h(c, coarse_out + c0 * Nc, oc, sizeof(double) * Nc * cnt);
      }
    }
    std::vector<int> bad(count);
    d2h(c, bad.data(), c->out_i.p, sizeof(int) * count);
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    c->flush_stats();
    for (int64_t b = 0; b < count; ++b)
      if (bad[b]) throw osc::Error(OSC_ERR_NUMERICAL, "sample: non-finite field value");
  });
}

int osc_darcy_solve(osc_ctx* c, int m, int64_t count, const double* Z, const osc_problem* prob,
                    double* u_out, int32_t* iters, int32_t* status, double* history, int hist_cap) {
  return guarded([&] {
    set_device(c);
    OSC_REQUIRE(m >= 1, "assemble_and_solve: m >= 1 required");
    OSC_REQUIRE(prob && Z, "osc_darcy_solve: null argument");
    if (count <= 0) return;
    const int64_t N = (int64_t)(m + 1) * (m + 1);
    c->fields_fine.ensure(sizeof(double) * N * count);
    c->xi_dev.ensure(sizeof(double) * N * count);
    c->out_i.ensure(sizeof(int) * count);
    h2d(c, c->xi_dev.p, Z, sizeof(double) * N * count);
    OSC_CUDA(cudaMemsetAsync(c->out_i.p, 0, sizeof(int) * count, c->stream));
    solver_prepare(c, m, (int)count, history ? hist_cap : 0);
    exp_field_launch(c, c->xi_dev.as<double>(), c->fields_fine.as<double>(), N * count, c->out_i.as<int>());
    std::vector<int> bad(count);
    d2h(c, bad.data(), c->out_i.p, sizeof(int) * count);
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    for (int64_t b = 0; b < count; ++b)
      if (bad[b]) throw osc::Error(OSC_ERR_NUMERICAL, "assemble_and_solve: non-finite log-field value");
    c->solver.lev[0].k = c->fields_fine.as<double>();
    solver_run(c, prob, (int)count);
    std::vector<int32_t> it(count), st(count);
    solver_results(c, (int)count, it.data(), st.data(), history);
    if (u_out) d2h(c, u_out, c->solver.u, sizeof(double) * N * count);
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    c->flush_stats();
    bool fail = false;
    for (int64_t b = 0; b < count; ++b) {
      if (iters) iters[b] = it[b];
      if (status) status[b] = st[b];
      fail |= st[b] != 0;
    }
    if (fail) throw osc::Error(OSC_ERR_SOLVER, "CG did not reach the relative residual within the iteration cap");
  });
}

int osc_qoi(osc_ctx* c, int m, int64_t count, const double* u, const double* Z,
            const osc_problem* prob, double* q_out) {
  return guarded([&] {
    set_device(c);
    OSC_REQUIRE(prob && u && q_out, "osc_qoi: null argument");
    OSC_REQUIRE(prob->qoi != OSC_QOI_FLUX || Z != nullptr, "osc_qoi: FLUX needs the log field Z");
    if (count <= 0) return;
    const int64_t N = (int64_t)(m + 1) * (m + 1);
    solver_prepare(c, m, (int)count, 0);
    c->fields_fine.ensure(sizeof(double) * N * count);
    c->out_q.ensure(sizeof(double) * count);
    c->out_i.ensure(sizeof(int) * count);
    h2d(c, c->solver.u, u, sizeof(double) * N * count);
    if (Z) {
      c->xi_dev.ensure(sizeof(double) * N * count);
      h2d(c, c->xi_dev.p, Z, sizeof(double) * N * count);
      exp_field_launch(c, c->xi_dev.as<double>(), c->fields_fine.as<double>(), N * count, c->out_i.as<int>());
    }
    c->solver.lev[0].k = c->fields_fine.as<double>();
    qoi_launch(c, prob, (int)count, c->out_q.as<double>());
    d2h(c, q_out, c->out_q.p, sizeof(double) * count);
    OSC_CUDA(cudaStreamSynchronize(c->stream));
    c->flush_stats();
  });
}

}  // extern "C"
