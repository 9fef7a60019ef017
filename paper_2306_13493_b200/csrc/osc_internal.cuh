// Internal declarations shared by the sm_100a kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/oscfield_b200.h"

namespace osc {

// ---- errors -------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define OSC_CUDA(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      throw ::osc::Error(OSC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define OSC_REQUIRE(cond, msg) \
  do {                         \
    if (!(cond)) throw ::osc::Error(OSC_ERR_CONFIG, msg); \
  } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies per device: set once per (current device,
// kernel, size); thread-safe (one host thread per device may launch concurrently).
void smem_attr_raw(const void* fn, size_t bytes);
template <class K>
inline void smem_attr(K* fn, size_t bytes) {
  smem_attr_raw(reinterpret_cast<const void*>(fn), bytes);
}

// ---- device buffer (grow-only) --------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    OSC_CUDA(cudaMalloc(&p, n));
    bytes = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// ---- per-kernel-class profiling on the context stream -------------------------------------
struct KernelStat {
  std::string name;
  int64_t launches = 0;
  double total_ms = 0.0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
};

struct Ctx;
// RAII scope: records start/stop events around the launches of one kernel class.
struct KScope {
  Ctx* ctx;
  int cls;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  KScope(Ctx* c, const char* name, int n_launches = 1);
  ~KScope();
};

// ---- solver workspace (one MG hierarchy for a batch of B samples) ----------------------------
struct SolverLevel {
  int m = 0;       // cells per side
  int64_t N = 0;   // nodes (m+1)^2
  double* k = nullptr;  // level 0: nodal conductivity (5-point stencil rebuilt in-kernel)
  // levels ≥ 1: symmetric 9-point operator, Dirichlet-eliminated (identity rows): diagonal C and
  // the couplings to the E, N, NE, NW neighbours (W, S, SW, SE are the neighbours' E, N, NE, NW)
  // Stored as fp64 diagonal + fp32 couplings: the preconditioner only steers the iteration (PCG
  // still stops on the fp64 residual of the fp64 level-0 system), and the diagonal is raised by the
  // couplings' fp32 rounding bound so the stored operator stays SPD (mgpcg.cu, store_row9).
  double* C = nullptr;
  float *E = nullptr, *Nw = nullptr, *NE = nullptr, *NW = nullptr;
  // prolongation weights of this level's cell-centre nodes (odd, odd) to the SW, SE, NW, NE coarse
  // corners, one value per cell (m/2 × m/2 per sample); edge-node weights are rebuilt from the stencil
  float* pw[4] = {nullptr, nullptr, nullptr, nullptr};
  double *r = nullptr, *z = nullptr;   // MG residual / pre-smoothed correction
  double* z2 = nullptr;                // post-smoothed correction (no in-place halo race)
};

struct SolverWork {
  int m = 0;
  int B = 0;
  int nlev = 0;
  int nc = 0;  // coarsest node count
  SolverLevel lev[24];
  double *u = nullptr, *p0 = nullptr, *p1 = nullptr, *Ap = nullptr;  // level-0 PCG vectors
  double* r2 = nullptr;  // level-0 residual ping-pong partner (pcg_update_down reads a halo of r)
  double* r_cur = nullptr;
  double* chol = nullptr;   // B * nc * nc
  double* scal = nullptr;   // per-sample scalars (see mgpcg.cu)
  double* partial = nullptr;
  unsigned* counter = nullptr;
  int* flags = nullptr;     // per-sample: active, iters, status
  int* n_active = nullptr;
  double* hist = nullptr;   // B * hist_cap (optional)
  int hist_cap = 0;
  int max_parts = 0;
  int opdep = 1;  // operator-dependent transfers (OSC_COARSE_GALERKIN) vs P1 linear
  DevBuf mem;
  // Device-side PCG loops (CUDA graphs with a conditional WHILE node), one per solve shape; the key
  // covers every value the captured kernels bake in (shape, tolerance, buffers).
  struct LoopGraph {
    int m = 0, B = 0, bc = 0, opdep = 0, hist_cap = 0;
    long hard_cap = -1;
    double tol = 0.0;
    const void *k = nullptr, *mem = nullptr;
    size_t mem_bytes = 0;
    cudaGraphExec_t exec = nullptr;
    int body_launches = 0;  // kernels per body run (two PCG iterations)
    uint64_t last_use = 0;
  };
  std::vector<LoopGraph> graphs;
  uint64_t graph_clock = 0;
  int pending_body_launches = 0;  // launches of the last graph solve, counted once its runs are known
  ~SolverWork() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
  }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  size_t mem_budget = 0;
  bool profiling = false;
  bool nvtx = false;  // OSC_NVTX=1: every kernel-class scope is an NVTX range "<class>:<grid>"
  std::string profile_only;  // non-empty: events only around this kernel class's launches
  std::vector<cudaEvent_t> ev_pool;  // timing events, reused across profiled launches
  size_t ev_next = 0;
  int64_t launches = 0;
  std::string tag;  // appended to kernel-class names ("name@tag"), e.g. the solve grid m
  std::vector<KernelStat> stats;
  // reusable workspaces
  DevBuf ce_inter, xi_dev, fields_fine, fields_coarse, out_q, out_i, tmp_host_stage, sums;
  DevBuf retry_k, retry_q;  // nested-start failures re-solved from the lift (osc_level_draws)
  SolverWork solver;
  int* h_pinned_int = nullptr;  // small pinned staging for n_active (16 ints; [4..7]: polling ring)
  cudaEvent_t ev_poll[4] = {nullptr, nullptr, nullptr, nullptr};  // lagged convergence polling
  cudaStream_t copy_stream = nullptr;           // host-ξ H2D overlapped with the previous chunk's solve
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_ce_done[2] = {nullptr, nullptr};
  // cross-call ξ prefetch (osc_level_prefetch_xi): the armed host rows of the NEXT osc_level_draws
  // call are copied into xi_pref on the copy stream under this call's solves
  const double* next_xi = nullptr;
  int64_t next_count = 0, next_s = 0;  // rows and embedding size s of the armed level
  // Two buffers: a call that reads one may already copy the following call's rows into the other.
  // Each prefetch is copied in kPrefParts parts with an event per part, so a call whose rows are
  // still arriving consumes them part by part instead of waiting for the whole batch.
  static constexpr int kPrefParts = 4;
  const double* pref_xi = nullptr;  // rows resident (or in flight) in xi_pref[pref_slot]
  int64_t pref_count = 0, pref_s = 0;
  int pref_slot = 0;
  int64_t pref_part_end[kPrefParts] = {0, 0, 0, 0};  // row ends of the parts
  DevBuf xi_pref[2];
  cudaEvent_t ev_pref_part[2][kPrefParts] = {};
  cudaEvent_t ev_pref_read[2] = {nullptr, nullptr};  // last read of each buffer (main stream)
  // residual history of failing samples (osc_ctx_set_history): the first failing slot of the last
  // osc_level_draws call is re-solved with the history kept (fem.cpp:359-379 SolverError::history)
  int hist_req = 0;
  int64_t fail_slot = -1;
  std::vector<double> fail_hist;
  int stat_class(const char* name);
  cudaEvent_t pool_event();
  void flush_stats();
};

struct Level {
  Ctx* ctx = nullptr;
  int m = 0, J = 0, n = 0;
  int64_t s = 0, k_trunc = 0;
  DevBuf sqrt_full, sqrt_trunc, twiddle;  // twiddle: n complex exp(+2πi t/n)
  // device-built levels (osc_level_create_device): the clamped eigenvalues and their stable
  // descending order stay resident, so re-truncation and OSC1 dumps need no host setup
  DevBuf eig, perm;  // perm: uint32 indices, largest eigenvalue first
  DevBuf sqrt_comp;  // √λ of the dropped modes (osc_smoothing_error), built on first use
  // running per-level sums in HBM (osc_level_sums_reset): [0..4] = [n, Σ(Y−Ky), Σ(Y−Ky)², Σ(q−Kq),
  // Σ(q−Kq)²] accumulated by every osc_level_draws call; [8..12] receive the cross-rank reduction
  DevBuf run_sums;
  bool sums_on = false;
  double shift_y = 0.0, shift_q = 0.0;
};

// ---- launchers --------------------------------------------------------------------------
// CE sample (ce_sample.cu). Produces fields for samples [0, count) of a chunk:
//  xi_dev != nullptr: ξ rows in device memory (count*s), else device Philox of indices
//  index0 + b. out_fine/out_coarse (device, may be null) receive exp(Z) (if do_exp) or Z.
//  col_stride 2 computes only the even columns/rows (coarse-only pass).
//  sup_out (device, count words, zeroed by the caller): the bit pattern of max |Z| over the fine
//  window per sample (the column pass's epilogue reduction; the outputs may then be null).
void ce_sample_launch(Ctx* ctx, const Level* L, const double* sqrt_lam, const double* xi_dev,
                      uint64_t seed, uint32_t ell, uint64_t index0, int count, bool do_exp,
                      double* out_fine, double* out_coarse, int* bad_flag,
                      unsigned long long* sup_out = nullptr);
size_t ce_inter_bytes(const Level* L, int count, int col_stride);
void upload_twiddles(Level* L);
// Level setup on the device (ce_sample.cu): raw spectrum (s = (2(m+J))² entries, host vector) of
// the padding-J embedding; supported for separable exponential and Matérn ν = k + ½, k ≤ 3.
bool spectrum_device_supported(int family, double nu_or_p);
std::vector<double> spectrum_device(Ctx* ctx, int m, int J, int family, double sigma2, double lambda,
                                    double nu_or_p);
void spectrum_device_into(Ctx* ctx, int m, int J, int family, double sigma2, double lambda, double nu_or_p,
                          double* eig_dev);

// Batched MG-PCG (mgpcg.cu). k (device, B*(m+1)^2) is consumed as level-0 conductivity.
void solver_prepare(Ctx* ctx, int m, int B, int hist_cap);
size_t solver_bytes(int m, int B, int hist_cap);
void solver_run(Ctx* ctx, const osc_problem* prob, int B, const double* uc_guess = nullptr);
// after solver_run: per-sample iters/status/u on device
void qoi_launch(Ctx* ctx, const osc_problem* prob, int B, double* q_dev);
void level_sums_launch(Ctx* ctx, const double* qf, const double* qc, int B, double shift_y,
                       double shift_q, double* sums_dev);
void level_sums_reshift_launch(Ctx* ctx, double* sums_dev, double dy, double dq);
// per-sample iterations / status (and history) of the last solver_run, copied to host
void solver_results(Ctx* ctx, int B, int32_t* iters, int32_t* status, double* hist_host);
void exp_field_launch(Ctx* ctx, const double* Z, double* k, int64_t total, int* bad_flag);
void normals_launch(Ctx* ctx, uint64_t seed, uint32_t ell, uint64_t index0, int count,
                    int64_t s, double* out);

}  // namespace osc

// the C-ABI's opaque handles are the internal objects
struct osc_ctx : osc::Ctx {};
struct osc_level : osc::Level {};
