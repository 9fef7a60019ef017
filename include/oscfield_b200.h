/*
 * oscfield_b200.h — C-ABI of the B200-native MLMC sample path
 * (circulant-embedding field → coarse/fine restriction → batched fp64 Darcy MG-PCG →
 * QoI → per-level sums). Implemented by paper_2306_13493_b200/libosc_b200.so
 * (hand-written sm_100a CUDA + host C++). Plain pointers and sizes only.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj):
 *
 *   osc_level_draws     ← run_level_draws (include/oscfield/estimators.hpp:112-118, declared
 *                         but undefined in the reference; its body today is run_level_samples,
 *                         src/estimators.cpp:65-75 → coupled_sample :200-237 per index)
 *   osc_summarize       ← summarize_draws (estimators.hpp:120-128; body = moments_of,
 *                         src/estimators.cpp:82-101)
 *   osc_ce_sample       ← EmbeddingOperator::sample_into + restrict_to
 *                         (include/oscfield/embedding.hpp:63-69, src/embedding.cpp:165-203)
 *   osc_darcy_solve     ← assemble_and_solve (include/oscfield/fem.hpp:47, src/fem.cpp:317-400)
 *   osc_qoi             ← evaluate_qoi / qoi_point / qoi_l2norm (estimators.hpp:23,
 *                         fem.hpp:51-54, src/fem.cpp:402-436)
 *   osc_build_spectrum  ← build_operator (embedding.hpp:112-113, src/embedding.cpp:114-151)
 *   osc_build_spectrum_device ← build_operator with build_first_row + spectrum on the device
 *   osc_level_create    ← EmbeddingOperator::from_parts + truncated (embedding.cpp:90-112,153-163)
 *   osc_mlmc_adaptive   ← estimate_adaptive (src/estimators.cpp:289-378; mlmc_estimate / mc_estimate
 *                         :398-418) as a GPU-resident driver: all levels of a round draw concurrently,
 *                         the moments stay in HBM as running sums
 *   osc_normals         ← NormalStream::fill (include/oscfield/rng.hpp:30-43, src/rng.cpp:42-67)
 *
 * Errors: every function returns an osc_status. Non-zero codes map onto the reference's
 * exception taxonomy (include/oscfield/errors.hpp:10-29): OSC_ERR_CONFIG → ConfigError,
 * OSC_ERR_NUMERICAL → NumericalError, OSC_ERR_SOLVER → SolverError (per-sample status[]
 * says which samples, the optional history buffer carries the residual history),
 * OSC_ERR_EMBEDDING → EmbeddingError. The message is available from osc_last_error().
 *
 * Threading: one osc_ctx per device, driven by one host thread (mirrors one
 * SampleWorkspace per worker, embedding.hpp:24-35). Device buffers are owned by the
 * context/level and stay resident across calls; host buffers are owned by the caller.
 *
 * Layouts: nodal arrays are fp64, x fastest, index p0 + (m+1)*p1 (grid.hpp:13-15,39-41).
 * ξ is fp64 of length s = n*n in NormalStream::fill order (q0 + n*q1).
 */
#ifndef OSCFIELD_B200_H
#define OSCFIELD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  OSC_OK = 0,
  OSC_ERR_CONFIG = 2,     /* ConfigError (CLI exit 2) */
  OSC_ERR_NUMERICAL = 3,  /* NumericalError (CLI exit 3) */
  OSC_ERR_SOLVER = 4,     /* SolverError: CG did not reach tol within the cap */
  OSC_ERR_EMBEDDING = 5,  /* EmbeddingError: no SPD embedding within the padding schedule */
  OSC_ERR_CUDA = 6        /* device / driver failure */
} osc_status;

/* Boundary conditions. FLOWCELL is the reference's (fem.hpp:11-16, fem.cpp:28-30):
 * u=1 at x=0, u=0 at x=1, zero flux on y∈{0,1}. DIRICHLET_ALL (u=0 on all sides) is an
 * extension required by BASELINE configs 1 and 4 (parity unpinned by the reference). */
enum { OSC_BC_FLOWCELL = 0, OSC_BC_DIRICHLET_ALL = 1 };
/* QoIs: POINT, L2 as the reference (estimators.hpp:16-21); INTEGRAL (∫u dx) and FLUX
 * (outflow flux through x=1) are extensions for BASELINE configs 1/3/5. */
enum { OSC_QOI_POINT = 0, OSC_QOI_L2 = 1, OSC_QOI_INTEGRAL = 2, OSC_QOI_FLUX = 3 };
/* Covariance families (covariance.hpp:10). */
enum { OSC_COV_MATERN = 0, OSC_COV_SEPARABLE_EXP = 1 };

/* osc_level_draws flags */
enum {
  OSC_DRAW_HAS_COARSE = 1,      /* level ℓ>0: also solve on the coarse grid m/2 */
  OSC_DRAW_TRUNC_FINE = 2,      /* fine field from the truncated (smoothed) spectrum */
  OSC_DRAW_TRUNC_COARSE = 4,    /* coarse field from the truncated spectrum */
  OSC_DRAW_XI_DEVICE = 8        /* xi points to DEVICE memory (else host memory) */
};
/* osc_ce_sample flags */
enum {
  OSC_CE_TRUNCATED = 1,         /* use the truncated spectrum */
  OSC_CE_EXP = 2,               /* write k = exp(Z) instead of Z */
  OSC_CE_FINE = 4,              /* write the fine field (m+1)^2 */
  OSC_CE_COARSE = 8,            /* write the stride-2 coarse field (m/2+1)^2 */
  OSC_CE_DEVICE_OUT = 16,       /* fine_out / coarse_out are DEVICE pointers (no D2H copy) */
  OSC_CE_XI_DEVICE = 32         /* xi is a DEVICE pointer (no H2D copy) */
};

/* Coarse-grid operators and transfers of the multigrid preconditioner. The preconditioner only
 * changes the iteration path: every mode solves the same fine system to the same ‖r‖/‖b‖ ≤ tol.
 * GALERKIN (default): operator-dependent prolongation (flux-continuous weights from the stencil:
 *   edge nodes collapse the stencil along the line, cell centres interpolate from their four
 *   edge neighbours) and exact Galerkin coarse operators A_c = Pᵀ A P (9-point below level 0).
 *   It needs about 2.5× fewer PCG iterations than the reference on rough fields.
 * REDISCRETIZE: the reference's scheme (fem.cpp:144-195, 241-244):
 *   - coarse matrices re-assembled from injected nodal k;
 *   - P1 linear transfer.
 * GALERKIN_LINEAR: P1 linear transfer with Galerkin coarse operators. This is the coarse P1 matrix
 *   whose triangle conductivity is the mean of the 4 fine triangles inside each coarse triangle. */
enum { OSC_COARSE_GALERKIN = 0, OSC_COARSE_REDISCRETIZE = 1, OSC_COARSE_GALERKIN_LINEAR = 2 };

/* Flat mirror of DarcyProblem / SolverOptions / QoiSpec (fem.hpp:17-35,
 * estimators.hpp:16-30). The preconditioner is always geometric multigrid (the estimator
 * default, estimators.hpp:79):
 *   - red-black Gauss-Seidel V(1,1);
 *   - transfers and coarse operators per `coarse_op`;
 *   - a per-sample dense factor on the coarsest grid. */
typedef struct {
  int bc;               /* OSC_BC_* */
  int forcing;          /* 0 = Forcing::Zero, 1 = Forcing::Constant */
  double forcing_value; /* f */
  int qoi;              /* OSC_QOI_* */
  double qoi_x, qoi_y;  /* point QoI location, default (7/15, 7/15) */
  double tol;           /* relative residual target, default 1e-10 */
  int max_iter_factor;  /* CG cap = factor * node count, default 10 */
  int coarse_op;        /* OSC_COARSE_*, default (0) GALERKIN */
} osc_problem;

typedef struct osc_ctx osc_ctx;
typedef struct osc_level osc_level;

/* ---- context --------------------------------------------------------------- */
/* device < 0: the calling thread's current CUDA device */
int osc_ctx_create(int device, osc_ctx** out);
void osc_ctx_destroy(osc_ctx* ctx);
/* Thread-local message of the last failing call. */
const char* osc_last_error(void);
/* The cudaStream_t (as void*) every kernel of this context is launched on. */
void* osc_ctx_stream(osc_ctx* ctx);
int osc_ctx_synchronize(osc_ctx* ctx);
/* Device memory budget (bytes) for batch workspaces; 0 = 60% of free memory. */
int osc_ctx_set_mem_budget(osc_ctx* ctx, size_t bytes);
/* Per-kernel-class timing with CUDA events on the context stream (0 off / 1 on). */
int osc_ctx_set_profiling(osc_ctx* ctx, int on);
/* Restrict profiling events to one kernel class ("name@grid", as osc_ctx_kernel_stats reports it);
 * launch counts of every class are still kept. NULL or "" lifts the restriction. */
int osc_ctx_profile_only(osc_ctx* ctx, const char* kernel_class);
/* Number of kernel classes with stats; name/launch count/total ms of class i. */
int osc_ctx_kernel_stats(osc_ctx* ctx, int i, const char** name, int64_t* launches,
                         double* total_ms);
int osc_ctx_reset_stats(osc_ctx* ctx);
/* Kernels launched by this context since creation (all classes). */
int64_t osc_ctx_launch_count(osc_ctx* ctx);

/* Pinned host memory for overlapped H2D/D2H (cudaHostAlloc). */
void* osc_host_alloc(size_t bytes);
void osc_host_free(void* p);
/* Library-allocated host buffer release (osc_build_spectrum output). */
void osc_free(void* p);

/* ---- level setup (host C++) ---------------------------------------------------- */
/* build_operator: first row (embedding.cpp:22-65) → spectrum (:67-88) with padding
 * schedule J = 0, then ceil(f*m) for f in fractions (:132-141) until min λ ≥ -tol_spd
 * (tol_spd = tol_spd_factor * s * sigma2), negatives clamped to 0. Returns J and a
 * malloc'd eigenvalue array of s = (2(m+J))^2 entries (release with osc_free).
 * fractions = NULL → {0.5, 1, 2, 4, 8}; tol_spd_factor ≤ 0 → 1e-12. */
int osc_build_spectrum(int m, int family, double sigma2, double lambda, double nu_or_p,
                       const double* fractions, int n_fractions, double tol_spd_factor,
                       int* J_out, int64_t* s_out, double** eig_out);
/* build_operator with the first row and the spectrum FFT on the device (same padding schedule,
 * SPD test, clamping and output contract as osc_build_spectrum). Separable exponential and
 * Matern (covariance.cpp:53-62): closed forms for nu = k + 1/2 (k <= 3), a device K_nu (Temme's series /
 * Steed's continued fraction + upward recurrence) for any other nu in (0, 64].
 * Eigenvalues agree with the host setup to rounding (~1e-15 of max λ); ties of equal λ may then
 * order differently in a truncation mask (use the host or OSC1 spectrum for mask parity). */
int osc_build_spectrum_device(osc_ctx* ctx, int m, int family, double sigma2, double lambda, double nu_or_p,
                              const double* fractions, int n_fractions, double tol_spd_factor,
                              int* J_out, int64_t* s_out, double** eig_out);
/* Upload one level: n = 2(m+J); eigenvalues (s entries) → √max(λ,0) on device, plus the
 * truncated copy zeroing the k_trunc smallest by a stable descending sort
 * (embedding.cpp:105-110,153-163). k_trunc = 0 → no truncated copy. */
int osc_level_create(osc_ctx* ctx, int m, int J, const double* eigenvalues, int64_t k_trunc,
                     osc_level** out);
/* build_operator + from_parts + truncated (embedding.cpp:90-163) entirely in HBM: the spectrum as in
 * osc_build_spectrum_device, its minimum (the SPD test; the only value that reaches the host), the
 * clamp, √max(λ,0), the stable descending order (a stable radix sort of (λ, index) pairs, i.e.
 * std::stable_sort by a > b, :105-107) and the truncation mask. The eigenvalues and the order stay
 * resident: osc_level_retruncate(k) is truncated(k) without a rebuild, osc_level_eigenvalues copies
 * the clamped λ to the host (s doubles; e.g. for osc_spectrum_save or the estimator's k_ℓ rule). J from
 * osc_level_info. Same model support as osc_build_spectrum_device. */
int osc_level_create_device(osc_ctx* ctx, int m, int family, double sigma2, double lambda, double nu_or_p,
                            const double* fractions, int n_fractions, double tol_spd_factor,
                            int64_t k_trunc, osc_level** out);
int osc_level_retruncate(osc_level* level, int64_t k_trunc);
int osc_level_eigenvalues(osc_level* level, double* out);
/* smoothing_error_estimate (embedding.cpp:205-228): mean and sample variance of ‖Z − Z̃‖∞ over
 * n_samples draws ξ_i = NormalStream(seed, 0, i), Z̃ from the level's truncated spectrum. Z − Z̃ is
 * linear in ξ, so each sample is ONE CE pass with the dropped modes' √λ whose column pass reduces
 * sup|·| over the (m+1)² window in its epilogue; no field is stored or copied. out = [mean, variance]
 * (Welford in index order); sup_out (may be NULL) receives the n_samples sup-norms. A level with
 * k_trunc = 0 gives zeros. */
int osc_smoothing_error(osc_level* level, int n_samples, uint64_t seed, double out[2], double* sup_out);
/* OSC1 spectrum files (save_spectrum / load_spectrum, embedding.cpp:262-294; d = 2, square grids):
 * "OSC1", u32 d, u32 m[d], u32 J[d], u64 s, s little-endian f64. load returns a malloc'd array
 * (release with osc_free). Errors as the reference's ConfigError cases. */
int osc_spectrum_save(const char* path, int m, int J, const double* eigenvalues, int64_t s);
int osc_spectrum_load(const char* path, int* m_out, int* J_out, int64_t* s_out, double** eig_out);

/* Cross-call ξ prefetch for a streaming caller (the reference's estimate_adaptive issues
 * consecutive run_level_draws batches, estimators.cpp:304-369). Arms the host rows xi_next
 * (count·s doubles, s = next_level's embedding size; pinned for full overlap) of the NEXT host-ξ
 * osc_level_draws call on next_level: the following host-ξ call on the same context copies them
 * to the device on the copy stream under its own solves, and the call on next_level with exactly
 * that pointer and count then runs as one batch without an exposed H2D copy. Any other pointer,
 * count or embedding size drops the prefetched rows (plain chunked path). Contract: xi_next holds
 * count·s doubles and stays valid and unchanged until that next call returns. NULL / 0 disarms.
 * No reference counterpart. */
int osc_level_prefetch_xi(osc_level* next_level, const double* xi_next, int64_t count);
void osc_level_destroy(osc_level* level);
/* m, J, n, s and k_trunc of a level. */
int osc_level_info(const osc_level* level, int* m, int* J, int* n, int64_t* s, int64_t* k_trunc);

/* ---- the fused per-level batch (the drop-in seam) ------------------------------ */
/* Draws samples [from, to) on one level: ξ_i = NormalStream(seed, ell, i) generated on
 * device (xi == NULL) or taken from xi (row i-from, s doubles; host or device memory per
 * OSC_DRAW_XI_DEVICE); fine field (and, with OSC_DRAW_HAS_COARSE, the stride-2 coarse
 * field of the same ξ — from the other spectrum when the TRUNC flags differ,
 * estimators.cpp:221-234); batched MG-PCG solves; QoIs. Slot i-from of q_fine / q_coarse
 * / iters_* / status receives sample i, so results do not depend on how [from,to) is
 * split across calls, ranks or devices (estimators.hpp:112-114). Any output pointer
 * may be NULL. level_sums (may be NULL) receives, accumulated in slot order on device,
 * [count, Σ(Y-shift), Σ(Y-shift)², Σ(q_f-shift_q), Σ(q_f-shift_q)²] with
 * Y = q_fine - q_coarse (or q_fine) and shifts given in level_sums[5], level_sums[6]
 * on input. Returns OSC_ERR_SOLVER if any sample failed to converge (its status[] slot
 * is OSC_ERR_SOLVER), OSC_ERR_NUMERICAL on a non-finite field. */
int osc_level_draws(osc_level* level, const osc_problem* problem, uint64_t seed, uint32_t ell,
                    int64_t from, int64_t to, int flags, const double* xi, double* q_fine,
                    double* q_coarse, int32_t* iters_fine, int32_t* iters_coarse,
                    int32_t* status, double* level_sums);

/* Running per-level sums in HBM (north_star subsystem 4; the moments of estimators.cpp:82-101,320,335
 * as shifted sums). After osc_level_sums_reset(level, Ky, Kq) every osc_level_draws call on the level
 * adds its samples to [n, Σ(Y−Ky), Σ(Y−Ky)², Σ(q_f−Kq), Σ(q_f−Kq)²] on the device (no host round trip;
 * Y = q_fine − q_coarse, or q_fine without a coarse grid). Use shifts near the level means (e.g. the
 * pilot means) so the variance (Σ(Y−K)² − (Σ(Y−K))²/n)/(n−1) does not cancel. osc_level_sums_read copies
 * out = [5 sums, Ky, Kq]. The sums of one call sequence are bit-identical run to run; a different
 * chunking of the same samples changes the summation order (~1e-16 relative). */
int osc_level_sums_reset(osc_level* level, double shift_y, double shift_q);
int osc_level_sums_read(osc_level* level, double out[7]);
/* Moves the running sums to new shifts without the samples (device side, one thread):
 * Σ(v−K') = Σ(v−K) − n·d and Σ(v−K')² = Σ(v−K)² − 2d·Σ(v−K) + n·d² with d = K' − K. A driver that
 * cannot know the level mean before its first batch starts at shift 0 and re-centres after the pilot,
 * so the later (much larger) batches accumulate without cancellation. */
int osc_level_sums_reshift(osc_level* level, double shift_y, double shift_q);

/* Residual history of failing samples (SolverError::history, fem.cpp:359-379). With hist_cap > 0, an
 * osc_level_draws call that returns OSC_ERR_SOLVER re-draws its first failing slot alone with the
 * per-iteration ‖r‖/‖b‖ kept (sample i is a pure function of (seed, ℓ, i) or of xi row i, so the
 * failure repeats bit for bit); osc_ctx_failure_history then returns that slot and up to cap entries
 * (history[0] = initial residual) and the history length (0 when no failure was recorded). */
int osc_ctx_set_history(osc_ctx* ctx, int hist_cap);
int osc_ctx_failure_history(osc_ctx* ctx, int64_t* slot, double* out, int cap);

/* ---- several GPUs -------------------------------------------------------------------------------
 * Samples shard with no data-path exchange: [from, to) is cut into contiguous per-device chunks
 * (chunk = ceil(count/G), the chunking of parallel_samples, estimators.cpp:32-63), so slot i receives
 * sample i for any device count. The only collective is an fp64 ncclAllReduce of the 5 device-resident
 * level sums per batch. NCCL is loaded at run time (dlopen libnccl.so.2).
 *
 * osc_group: one process drives G devices, one osc_ctx and one host thread per device. */
typedef struct osc_group osc_group;
typedef struct osc_group_level osc_group_level;
int osc_group_create(int n_devices, const int* devices /* NULL → 0..n-1 */, osc_group** out);
void osc_group_destroy(osc_group* group);
int osc_group_size(const osc_group* group);
osc_ctx* osc_group_ctx(osc_group* group, int i);
/* osc_level_create on every device (same host eigenvalues, same truncation mask). */
int osc_group_level_create(osc_group* group, int m, int J, const double* eigenvalues, int64_t k_trunc,
                           osc_group_level** out);
void osc_group_level_destroy(osc_group_level* level);
osc_level* osc_group_level_at(osc_group_level* level, int i);
/* osc_level_draws over the group: device g draws its contiguous chunk into its slots of the caller's
 * (host) arrays; xi is host memory or NULL (device Philox). level_sums as in osc_level_draws, summed
 * over the devices by one NCCL all-reduce of the device buffers. A solver failure on any device lets
 * every device finish, then returns OSC_ERR_SOLVER. */
int osc_group_level_draws(osc_group_level* level, const osc_problem* problem, uint64_t seed, uint32_t ell,
                          int64_t from, int64_t to, int flags, const double* xi, double* q_fine,
                          double* q_coarse, int32_t* iters_fine, int32_t* iters_coarse, int32_t* status,
                          double* level_sums);
int osc_group_level_sums_reset(osc_group_level* level, double shift_y, double shift_q);
/* all-reduce of the devices' running level sums (device to device), out = [5 sums, Ky, Kq] */
int osc_group_level_sums_allreduce(osc_group_level* level, double out[7]);

/* osc_comm: one process per GPU (e.g. torchrun). Rank 0 makes the id, the launcher broadcasts it. */
typedef struct osc_comm osc_comm;
int osc_comm_unique_id(unsigned char id[128]);
int osc_comm_create(osc_ctx* ctx, int nranks, int rank, const unsigned char id[128], osc_comm** out);
void osc_comm_destroy(osc_comm* comm);
/* ncclAllReduce of the level's running sums into a separate device buffer (the running sums keep
 * accumulating); out (may be NULL) = [5 reduced sums, Ky, Kq] */
int osc_comm_allreduce_level_sums(osc_comm* comm, osc_level* level, double out[7]);
/* ncclAllGather of n_per_rank doubles per rank (host in, host out, rank order): the (q_f, q_c) slots
 * of contiguous shards, so every rank can run the reference's slot-order Welford bit-identically. */
int osc_comm_allgather(osc_comm* comm, const double* local, int64_t n_per_rank, double* all);

/* ---- GPU-resident adaptive MLMC driver ---------------------------------------
 * estimate_adaptive (src/estimators.cpp:289-378) with the level loop turned into waves: within one
 * allocation pass every level's target N_ℓ = ⌈2ε⁻²·(Σ_j √(C_j V_j))·√(V_ℓ/C_ℓ)⌉ (C_ℓ = h_ℓ^−γ) depends
 * only on the moments at the start of the pass (:322-338), so all levels that need samples draw AT THE
 * SAME TIME — one context (stream + workspace) and one host thread per level and device — instead of
 * one level after the other; small levels, which cannot fill 148 SMs alone, run under the large ones.
 * The moments never pass through per-sample host arrays: each level accumulates its running sums in
 * HBM (osc_level_sums_*), re-centred on the pilot mean after the first wave; with several devices
 * each level's range is cut into contiguous per-device chunks and ONE all-reduce per wave combines
 * the sums of all levels (8 doubles per level). Levels are set up on the device
 * (osc_level_create_device) unless `spectrum` supplies the eigenvalues.
 * The decisions follow the reference: pilot = max(2, pilot_n) samples per level, at most 64 passes,
 * bias from the weak-error model c_α h^α on a single level, else Richardson |E[Y_L]|/|1 − r·2^α|
 * (r = c_alpha_tilde_ratio when the finest difference has a smoothed coarse term, else 1; a
 * denominator below 0.1 is OSC_ERR_NUMERICAL), a new finest level while bias² > ε²/2 and L < l_max
 * (the previous finest level then changes its sampling law and is redrawn when it was smoothed),
 * the smoothing rule of make_level_plan (:169-198, choose_k_ell :238-275, coarsest_level_bound
 * :487-494). Sample i of level ℓ is NormalStream(seed, ℓ, i), as in every other entry point. */
enum { OSC_SMOOTHING_OFF = 0, OSC_SMOOTHING_HALF_SPECTRUM = 1, OSC_SMOOTHING_ADAPTIVE = 2 };
#define OSC_MLMC_MAX_LEVELS 26

/* Optional source of a level's eigenvalues (OSC1 files, the reference's build_operator, …): fills J, s
 * and a malloc'd array of s = (2(m+J))² eigenvalues that the driver releases with free(). Non-zero
 * return = failure (reported as OSC_ERR_EMBEDDING). Called once per level, always from the thread that
 * called osc_mlmc_adaptive (it need not be re-entrant). */
typedef int (*osc_spectrum_fn)(void* user, int m, int* J, int64_t* s, double** eigenvalues);

typedef struct {
  int family;            /* OSC_COV_* */
  double sigma2, lambda, nu_or_p;
  double h0;             /* coarsest mesh width, a negative power of two */
  double eps;            /* RMSE target */
  int initial_levels;    /* ≥ 1 */
  int l_max;             /* finest admissible level index */
  int allow_extension;   /* 1 = mlmc_estimate; 0 = the single-grid mc_estimate path (sampling error only) */
  uint64_t seed;
  int pilot_n;
  double gamma_model, alpha, c_alpha, c_ratio, c_alpha_tilde_ratio; /* EstimatorOptions, estimators.hpp:66-80 */
  int smoothing;         /* OSC_SMOOTHING_* */
  int use_coarse_s, lstar_only;
  int concurrent_levels; /* 1 (default use): all levels of a wave at once; 0: one level after the other */
  osc_spectrum_fn spectrum; /* NULL: device level setup */
  void* spectrum_user;
} osc_mlmc_options;

typedef struct {
  double estimate, bias_estimate, sampling_error, total_cost_model, total_cost_wall;
  int converged, n_levels, passes, waves;
  int64_t n[OSC_MLMC_MAX_LEVELS], k_trunc[OSC_MLMC_MAX_LEVELS], redrawn[OSC_MLMC_MAX_LEVELS];
  double mean_y[OSC_MLMC_MAX_LEVELS], var_y[OSC_MLMC_MAX_LEVELS], mean_q[OSC_MLMC_MAX_LEVELS],
      var_q[OSC_MLMC_MAX_LEVELS], h[OSC_MLMC_MAX_LEVELS], n_real[OSC_MLMC_MAX_LEVELS],
      wall_per_sample[OSC_MLMC_MAX_LEVELS];
  double setup_s, draw_s, total_s; /* level setup, waves (elapsed, levels overlapped), whole call */
  int64_t samples_total, gpu_launches;
  char message[256];
} osc_mlmc_report;

/* devices NULL → 0..n_devices-1; n_devices ≤ 0 → the calling thread's current device. */
int osc_mlmc_adaptive(int n_devices, const int* devices, const osc_problem* problem,
                      const osc_mlmc_options* options, osc_mlmc_report* report);
/* The truncation count k_ℓ the driver uses on mesh width h for an embedding with padding J and s
 * entries (0: no smoothing on that level). */
int64_t osc_mlmc_k_trunc(const osc_mlmc_options* options, double h, int J, int64_t s);

/* summarize_draws: one-pass Welford over slot-ordered draws (estimators.cpp:82-101).
 * out = [n, mean_y, var_y, mean_q, var_q]; var only when n ≥ 2. q_coarse may be NULL. */
int osc_summarize(const double* q_fine, const double* q_coarse, int64_t n, int has_coarse,
                  double out[5]);

/* ---- unfused stages (single-sample reference APIs, unit tests) -------------------- */
/* NormalStream(seed, ell, index0 + j).fill for j < count on device; out host (count*s). */
int osc_normals(osc_ctx* ctx, uint64_t seed, uint32_t ell, uint64_t index0, int64_t count,
                int64_t s, double* out);
/* CE sample of `count` samples: xi (count*s; host, or device with OSC_CE_XI_DEVICE) or NULL for
 * device Philox of indices [index0, index0+count) at (seed, ell); writes fine ((m+1)^2 each)
 * and/or coarse ((m/2+1)^2 each) fields to host (or to device with OSC_CE_DEVICE_OUT) per the
 * OSC_CE_* flags. Large batches are processed in L2-sized chunks internally. */
int osc_ce_sample(osc_level* level, const double* xi, uint64_t seed, uint32_t ell,
                  uint64_t index0, int64_t count, int flags, double* fine_out,
                  double* coarse_out);
/* Batched assemble_and_solve of `count` log fields Z (host, count*(m+1)^2) on grid m.
 * u_out (host, may be NULL), iters/status per sample (may be NULL); history (may be NULL)
 * receives hist_cap relative residuals per sample (the reference's residual_history,
 * fem.cpp:364-365,388), padded with 0. */
int osc_darcy_solve(osc_ctx* ctx, int m, int64_t count, const double* Z,
                    const osc_problem* problem, double* u_out, int32_t* iters, int32_t* status,
                    double* history, int hist_cap);
/* QoI of `count` nodal solutions u (host) on grid m; Z (host) needed only for FLUX. */
int osc_qoi(osc_ctx* ctx, int m, int64_t count, const double* u, const double* Z,
            const osc_problem* problem, double* q_out);

#ifdef __cplusplus
}
#endif
#endif /* OSCFIELD_B200_H */
