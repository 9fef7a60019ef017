// Multi-GPU layer of the C-ABI (include/oscfield_b200.h, osc_group_* / osc_comm_*).
//
// MLMC samples shard with no data-path exchange: sample i always uses NormalStream(seed, ℓ, i) and
// lands in slot i (estimators.hpp:112-114), so a level's range [from, to) is cut into contiguous
// per-device chunks exactly like parallel_samples cuts it into per-thread chunks
// (src/estimators.cpp:32-63): chunk = ceil(count / G), device g draws [from + g·chunk, …). Each
// device runs the fused osc_level_draws batch on its own host thread (one thread drives one GPU,
// embedding.hpp:24-35), writing its slots of the caller's arrays in place. The only collective is
// the per-level sums: one ncclAllReduce (fp64, sum) of the 5 device-resident values per batch over
// NVLink/NVSwitch — the values never leave HBM before the reduction.
//
//  * osc_group: one process, G devices, one osc_ctx and one host worker thread per device, NCCL
//    communicators from ncclCommInitAll.
//  * osc_comm: one process per GPU (torchrun-style launch); ranks join through an NCCL unique id.
//
// NCCL is loaded with dlopen on first use (libnccl.so.2; inside a torch process this resolves to the
// NCCL torch already mapped), so single-GPU users never need it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "osc_internal.cuh"

namespace osc {
std::pair<bool, bool> draws_impl(Level* L, const osc_problem* prob, uint64_t seed, uint32_t ell, int64_t from,
                                 int64_t to, int flags, const double* xi, double* q_fine, double* q_coarse,
                                 int32_t* iters_fine, int32_t* iters_coarse, int32_t* status, double* level_sums,
                                 int hist_cap, double* hist_fine, double* hist_coarse);
void draws_checked(Level* L, const osc_problem* prob, uint64_t seed, uint32_t ell, int64_t from, int64_t to,
                   int flags, const double* xi, double* q_fine, double* q_coarse, int32_t* iters_fine,
                   int32_t* iters_coarse, int32_t* status, double* level_sums);
int c_api_error(const std::exception_ptr& e);  // capi.cu: exception → status + thread-local message

namespace {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl api;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    if (!h) {
      err = std::string("NCCL not available: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p && err.empty()) err = std::string("NCCL symbol missing: ") + n;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw Error(OSC_ERR_CONFIG, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(OSC_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

// contiguous chunk of [from, to) owned by shard g of G (parallel_samples' chunking)
void shard_range(int64_t from, int64_t to, int g, int G, int64_t& lo, int64_t& hi) {
  const int64_t count = to - from, chunk = (count + G - 1) / G;
  lo = std::min(to, from + g * chunk);
  hi = std::min(to, lo + chunk);
}

}  // namespace
}  // namespace osc

using namespace osc;

struct osc_group;
namespace osc {
// one grouped fp64 sum all-reduce over the group's communicators (device buffers, one per device, on
// each device's group-context stream), then a synchronise: the collective of the MLMC driver
void group_allreduce_f64(osc_group* g, double* const* send, double* const* recv, size_t count);
}

struct osc_group {
  std::vector<int> devices;
  std::vector<osc_ctx*> ctx;
  std::vector<ncclComm_t> comm;
};

struct osc_group_level {
  osc_group* g = nullptr;
  std::vector<osc_level*> lev;
};

struct osc_comm {
  osc_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  DevBuf stage;
};

namespace {
template <typename F>
int guard(F&& f) {
  try {
    f();
    return OSC_OK;
  } catch (...) {
    return c_api_error(std::current_exception());
  }
}

// Run fn(i) on one host thread per device (device i current); the first failure (lowest device)
// is rethrown after all threads joined, like parallel_samples (estimators.cpp:52-63).
template <typename F>
void per_device(const osc_group* g, F&& fn) {
  const int G = (int)g->devices.size();
  std::vector<std::exception_ptr> errs(G);
  std::vector<std::thread> pool;
  pool.reserve(G);
  for (int i = 0; i < G; ++i)
    pool.emplace_back([&, i] {
      try {
        OSC_CUDA(cudaSetDevice(g->devices[i]));
        fn(i);
      } catch (...) {
        errs[i] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}
}  // namespace

void osc::group_allreduce_f64(osc_group* g, double* const* send, double* const* recv, size_t count) {
  const int G = (int)g->devices.size();
  const Nccl& N = nccl();
  nccl_check(N.GroupStart(), "ncclGroupStart");
  for (int i = 0; i < G; ++i) {
    OSC_CUDA(cudaSetDevice(g->devices[i]));
    nccl_check(N.AllReduce(send[i], recv[i], count, ncclFloat64, ncclSum, g->comm[i], g->ctx[i]->stream),
               "ncclAllReduce");
  }
  nccl_check(N.GroupEnd(), "ncclGroupEnd");
  for (int i = 0; i < G; ++i) {
    OSC_CUDA(cudaSetDevice(g->devices[i]));
    OSC_CUDA(cudaStreamSynchronize(g->ctx[i]->stream));
  }
}

extern "C" {

int osc_group_create(int n_devices, const int* devices, osc_group** out) {
  return guard([&] {
    OSC_REQUIRE(out && n_devices >= 1, "osc_group_create: need at least one device");
    int avail = 0;
    OSC_CUDA(cudaGetDeviceCount(&avail));
    auto* g = new osc_group();
    try {
      for (int i = 0; i < n_devices; ++i) {
        const int d = devices ? devices[i] : i;
        OSC_REQUIRE(d >= 0 && d < avail, "osc_group_create: device index out of range");
        OSC_REQUIRE(std::find(g->devices.begin(), g->devices.end(), d) == g->devices.end(),
                    "osc_group_create: duplicate device");
        g->devices.push_back(d);
      }
      for (int d : g->devices) {
        osc_ctx* c = nullptr;
        if (int rc = osc_ctx_create(d, &c)) throw Error(rc, osc_last_error());
        g->ctx.push_back(c);
      }
      g->comm.assign(n_devices, nullptr);
      nccl_check(nccl().CommInitAll(g->comm.data(), n_devices, g->devices.data()), "ncclCommInitAll");
    } catch (...) {
      osc_group_destroy(g);
      throw;
    }
    *out = g;
  });
}

void osc_group_destroy(osc_group* g) {
  if (!g) return;
  for (ncclComm_t cm : g->comm)
    if (cm) nccl().CommDestroy(cm);
  for (osc_ctx* c : g->ctx) osc_ctx_destroy(c);
  delete g;
}

int osc_group_size(const osc_group* g) { return g ? (int)g->devices.size() : 0; }

osc_ctx* osc_group_ctx(osc_group* g, int i) {
  return (g && i >= 0 && i < (int)g->ctx.size()) ? g->ctx[i] : nullptr;
}

int osc_group_level_create(osc_group* g, int m, int J, const double* eigenvalues, int64_t k_trunc,
                           osc_group_level** out) {
  return guard([&] {
    OSC_REQUIRE(g && out && eigenvalues, "osc_group_level_create: null argument");
    auto* gl = new osc_group_level();
    gl->g = g;
    gl->lev.assign(g->devices.size(), nullptr);
    try {
      // host setup is shared; each device uploads its own √λ (8·s bytes, once per level)
      per_device(g, [&](int i) {
        if (int rc = osc_level_create(g->ctx[i], m, J, eigenvalues, k_trunc, &gl->lev[i]))
          throw Error(rc, osc_last_error());
      });
    } catch (...) {
      osc_group_level_destroy(gl);
      throw;
    }
    *out = gl;
  });
}

void osc_group_level_destroy(osc_group_level* gl) {
  if (!gl) return;
  for (osc_level* L : gl->lev) osc_level_destroy(L);
  delete gl;
}

osc_level* osc_group_level_at(osc_group_level* gl, int i) {
  return (gl && i >= 0 && i < (int)gl->lev.size()) ? gl->lev[i] : nullptr;
}

int osc_group_level_draws(osc_group_level* gl, const osc_problem* prob, uint64_t seed, uint32_t ell,
                          int64_t from, int64_t to, int flags, const double* xi, double* q_fine,
                          double* q_coarse, int32_t* iters_fine, int32_t* iters_coarse, int32_t* status,
                          double* level_sums) {
  return guard([&] {
    OSC_REQUIRE(gl && prob, "osc_group_level_draws: null argument");
    OSC_REQUIRE(to >= from && from >= 0, "osc_level_draws: need 0 <= from <= to");
    OSC_REQUIRE(!(flags & OSC_DRAW_XI_DEVICE), "osc_group_level_draws: xi must be host memory (or NULL)");
    osc_group* g = gl->g;
    const int G = (int)g->devices.size();
    const int64_t s = gl->lev[0]->s;
    std::vector<double> part(8 * (size_t)G, 0.0);
    std::vector<int> failed(G, 0);
    std::vector<std::exception_ptr> errs(G);
    per_device(g, [&](int i) {
      int64_t lo, hi;
      shard_range(from, to, i, G, lo, hi);
      double* ls = level_sums ? part.data() + 8 * i : nullptr;
      if (ls) {
        ls[5] = level_sums[5];
        ls[6] = level_sums[6];
      }
      const int64_t o = lo - from;
      try {
        draws_checked(gl->lev[i], prob, seed, ell, lo, std::max(lo, hi), flags, xi ? xi + o * s : nullptr,
                      q_fine ? q_fine + o : nullptr, q_coarse ? q_coarse + o : nullptr,
                      iters_fine ? iters_fine + o : nullptr, iters_coarse ? iters_coarse + o : nullptr,
                      status ? status + o : nullptr, ls);
      } catch (const Error& e) {
        if (e.code != OSC_ERR_SOLVER) throw;  // a non-converged sample still lets the batch finish
        failed[i] = 1;
        errs[i] = std::current_exception();
      }
    });
    if (level_sums) {
      // one fp64 all-reduce of the devices' per-call sums (left in each context's sums buffer)
      const Nccl& N = nccl();
      nccl_check(N.GroupStart(), "ncclGroupStart");
      for (int i = 0; i < G; ++i) {
        OSC_CUDA(cudaSetDevice(g->devices[i]));
        double* d = g->ctx[i]->sums.as<double>();
        nccl_check(N.AllReduce(d, d, 5, ncclFloat64, ncclSum, g->comm[i], g->ctx[i]->stream), "ncclAllReduce");
      }
      nccl_check(N.GroupEnd(), "ncclGroupEnd");
      for (int i = 0; i < G; ++i) {
        OSC_CUDA(cudaSetDevice(g->devices[i]));
        OSC_CUDA(cudaStreamSynchronize(g->ctx[i]->stream));
      }
      OSC_CUDA(cudaSetDevice(g->devices[0]));
      OSC_CUDA(cudaMemcpy(level_sums, g->ctx[0]->sums.p, sizeof(double) * 5, cudaMemcpyDeviceToHost));
    }
    for (int i = 0; i < G; ++i)
      if (failed[i]) std::rethrow_exception(errs[i]);
  });
}

int osc_group_level_sums_reset(osc_group_level* gl, double shift_y, double shift_q) {
  return guard([&] {
    OSC_REQUIRE(gl, "osc_group_level_sums_reset: null level");
    for (osc_level* L : gl->lev)
      if (int rc = osc_level_sums_reset(L, shift_y, shift_q)) throw Error(rc, osc_last_error());
  });
}

int osc_group_level_sums_allreduce(osc_group_level* gl, double out[7]) {
  return guard([&] {
    OSC_REQUIRE(gl && out, "osc_group_level_sums_allreduce: null argument");
    osc_group* g = gl->g;
    const int G = (int)g->devices.size();
    for (int i = 0; i < G; ++i) OSC_REQUIRE(gl->lev[i]->sums_on, "running sums not enabled (osc_group_level_sums_reset)");
    const Nccl& N = nccl();
    nccl_check(N.GroupStart(), "ncclGroupStart");
    for (int i = 0; i < G; ++i) {
      OSC_CUDA(cudaSetDevice(g->devices[i]));
      double* d = gl->lev[i]->run_sums.as<double>();
      nccl_check(N.AllReduce(d, d + 8, 5, ncclFloat64, ncclSum, g->comm[i], g->ctx[i]->stream), "ncclAllReduce");
    }
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
    for (int i = 0; i < G; ++i) {
      OSC_CUDA(cudaSetDevice(g->devices[i]));
      OSC_CUDA(cudaStreamSynchronize(g->ctx[i]->stream));
    }
    OSC_CUDA(cudaSetDevice(g->devices[0]));
    OSC_CUDA(cudaMemcpy(out, gl->lev[0]->run_sums.as<double>() + 8, sizeof(double) * 5, cudaMemcpyDeviceToHost));
    out[5] = gl->lev[0]->shift_y;
    out[6] = gl->lev[0]->shift_q;
  });
}

// ---- one process per GPU ------------------------------------------------------------------------
int osc_comm_unique_id(unsigned char id[128]) {
  return guard([&] {
    OSC_REQUIRE(id, "osc_comm_unique_id: null buffer");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int osc_comm_create(osc_ctx* ctx, int nranks, int rank, const unsigned char id[128], osc_comm** out) {
  return guard([&] {
    OSC_REQUIRE(ctx && id && out, "osc_comm_create: null argument");
    OSC_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "osc_comm_create: bad rank");
    OSC_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto* c = new osc_comm();
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    try {
      nccl_check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void osc_comm_destroy(osc_comm* c) {
  if (!c) return;
  if (c->comm) nccl().CommDestroy(c->comm);
  c->stage.release();
  delete c;
}

int osc_comm_allreduce_level_sums(osc_comm* c, osc_level* L, double out[7]) {
  return guard([&] {
    OSC_REQUIRE(c && L, "osc_comm_allreduce_level_sums: null argument");
    OSC_REQUIRE(L->ctx == c->ctx, "osc_comm_allreduce_level_sums: level of another context");
    OSC_REQUIRE(L->sums_on, "running sums not enabled (osc_level_sums_reset)");
    OSC_CUDA(cudaSetDevice(c->ctx->device));
    double* d = L->run_sums.as<double>();
    nccl_check(nccl().AllReduce(d, d + 8, 5, ncclFloat64, ncclSum, c->comm, c->ctx->stream), "ncclAllReduce");
    if (out) {
      OSC_CUDA(cudaMemcpyAsync(out, d + 8, sizeof(double) * 5, cudaMemcpyDeviceToHost, c->ctx->stream));
      OSC_CUDA(cudaStreamSynchronize(c->ctx->stream));
      out[5] = L->shift_y;
      out[6] = L->shift_q;
    }
  });
}

int osc_comm_allgather(osc_comm* c, const double* local, int64_t n_per_rank, double* all) {
  return guard([&] {
    OSC_REQUIRE(c && local && all && n_per_rank >= 0, "osc_comm_allgather: null argument");
    if (n_per_rank == 0) return;
    OSC_CUDA(cudaSetDevice(c->ctx->device));
    const size_t bytes = sizeof(double) * (size_t)n_per_rank;
    c->stage.ensure(bytes * (size_t)(c->nranks + 1));
    double* send = c->stage.as<double>();
    double* recv = send + n_per_rank;
    cudaStream_t st = c->ctx->stream;
    OSC_CUDA(cudaMemcpyAsync(send, local, bytes, cudaMemcpyHostToDevice, st));
    nccl_check(nccl().AllGather(send, recv, (size_t)n_per_rank, ncclFloat64, c->comm, st), "ncclAllGather");
    OSC_CUDA(cudaMemcpyAsync(all, recv, bytes * (size_t)c->nranks, cudaMemcpyDeviceToHost, st));
    OSC_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
