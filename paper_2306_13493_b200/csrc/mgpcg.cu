// K3: batched fp64 Darcy solve −∇·(k∇u) = f with P1 elements and geometric-multigrid-
// preconditioned CG, one independent solve per sample (gridDim.y = sample).
// Replaces assemble (src/fem.cpp:38-138), Multigrid (src/fem.cpp:140-307) and the PCG loop of
// assemble_and_solve (src/fem.cpp:317-400).
//
// Matrix-free: the P1 matrix of the lower-left/upper-right triangulation with vertex-mean
// element conductivity is a 5-point stencil (the diagonal couplings vanish exactly). Per node
// we keep D (diagonal = −Σ raw couplings, i.e. before Dirichlet elimination) and the east/north
// couplings E, N after symmetric Dirichlet elimination (zero when either end is Dirichlet);
// Dirichlet rows are identity (D = 1). Edge weights:
//   E(i,j) = −½[K_low(i,j) + K_up(i,j−1)],  N(i,j) = −½[K_up(i,j) + K_low(i−1,j)],
//   K_low(i,j) = (k_ij + k_i+1,j + k_i+1,j+1)/3,  K_up(i,j) = (k_ij + k_i+1,j+1 + k_i,j+1)/3.
// Preconditioner: V(1,1) with red-black Gauss–Seidel (red→black before the coarse correction,
// black→red after: symmetric, so CG stays valid — the reference uses lexicographic forward/
// backward GS, fem.cpp:197-212,288-303), R = Pᵀ with the P1 prolongation (fem.cpp:144-195),
// coarse operators rediscretised from injected nodal k (fem.cpp:241-244), coarsening while
// m > 4 and even (fem.cpp:239), dense per-sample Cholesky on the coarsest grid (:255-286).
// PCG and its stopping rule ‖r‖₂/‖b‖₂ ≤ tol over all rows incl. Dirichlet identity rows, with
// the Dirichlet lift as initial guess and cap max_iter_factor·N, follow fem.cpp:335-397.
// Per-sample reductions are deterministic (fixed-order last-block reduction).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "osc_device.cuh"
#include "osc_internal.cuh"

namespace osc {

namespace {

constexpr int NT = 256;  // threads per node block

// per-sample scalars (double) and flags (int)
enum { S_BNORM = 0, S_RZ, S_ALPHA, S_BETA, S_REL, S_NSCAL = 8 };
enum { F_ACTIVE = 0, F_ITERS, F_STATUS, F_FIRST, F_MAXIT, F_NFLAGS = 8 };

struct Geo {
  int m, n0;
  int64_t N;
};

__device__ __forceinline__ bool is_dir(int bc, int m, int p0, int p1) {
  return p0 == 0 || p0 == m || (bc == OSC_BC_DIRICHLET_ALL && (p1 == 0 || p1 == m));
}

// Fixed-order per-sample reduction of up to two values across the CTAs of one sample.
// Returns true in the last CTA; totals valid in thread 0 of that CTA.
__device__ __forceinline__ bool reduce2_last(double v0, double v1, double2* partial, int maxp,
                                             unsigned* counter, int b, double& t0, double& t1) {
  __shared__ double sh[32];
  __shared__ int last;
  const double s0 = block_sum(v0, sh);
  __syncthreads();
  const double s1 = block_sum(v1, sh);
  const int nparts = gridDim.x;
  if (threadIdx.x == 0) {
    partial[(int64_t)b * maxp + blockIdx.x] = make_double2(s0, s1);
    __threadfence();
    const unsigned prev = atomicAdd(counter + b, 1u);
    last = (prev == (unsigned)nparts - 1) ? 1 : 0;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double a0 = 0.0, a1 = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    const double2 pv = __ldcg(partial + (int64_t)b * maxp + i);
    a0 += pv.x;
    a1 += pv.y;
  }
  __syncthreads();
  t0 = block_sum(a0, sh);
  __syncthreads();
  t1 = block_sum(a1, sh);
  if (threadIdx.x == 0) counter[b] = 0u;
  return true;
}

// ---- setup: stencil from nodal k (+ injection to the next level) --------------------------
__global__ void __launch_bounds__(NT) setup_level_kernel(Geo g, int bc, const double* __restrict__ k,
                                                         double* __restrict__ D, double* __restrict__ E,
                                                         double* __restrict__ Nw, double* __restrict__ kc) {
  const int b = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x;
  if (i >= g.N) return;
  const int m = g.m, n0 = g.n0;
  const int p1 = (int)(i / n0), p0 = (int)(i - (int64_t)p1 * n0);
  const double* kb = k + (int64_t)b * g.N;
  auto K = [&](int a0, int a1) { return __ldg(kb + (int64_t)a1 * n0 + a0); };
  auto klow = [&](int c0, int c1) { return (K(c0, c1) + K(c0 + 1, c1) + K(c0 + 1, c1 + 1)) / 3.0; };
  auto kup = [&](int c0, int c1) { return (K(c0, c1) + K(c0 + 1, c1 + 1) + K(c0, c1 + 1)) / 3.0; };
  // raw couplings of the 4 edges at this node
  double e_east = 0.0, e_west = 0.0, e_north = 0.0, e_south = 0.0;
  if (p0 < m) e_east = -0.5 * ((p1 < m ? klow(p0, p1) : 0.0) + (p1 > 0 ? kup(p0, p1 - 1) : 0.0));
  if (p0 > 0) e_west = -0.5 * ((p1 < m ? klow(p0 - 1, p1) : 0.0) + (p1 > 0 ? kup(p0 - 1, p1 - 1) : 0.0));
  if (p1 < m) e_north = -0.5 * ((p0 < m ? kup(p0, p1) : 0.0) + (p0 > 0 ? klow(p0 - 1, p1) : 0.0));
  if (p1 > 0) e_south = -0.5 * ((p0 < m ? kup(p0, p1 - 1) : 0.0) + (p0 > 0 ? klow(p0 - 1, p1 - 1) : 0.0));
  const bool dself = is_dir(bc, m, p0, p1);
  const int64_t o = (int64_t)b * g.N + i;
  D[o] = dself ? 1.0 : -(e_east + e_west + e_north + e_south);
  E[o] = (p0 < m && !dself && !is_dir(bc, m, p0 + 1, p1)) ? e_east : 0.0;
  Nw[o] = (p1 < m && !dself && !is_dir(bc, m, p0, p1 + 1)) ? e_north : 0.0;
  if (kc && ((p0 | p1) & 1) == 0) {
    const int mc = m / 2;
    kc[(int64_t)b * (mc + 1) * (mc + 1) + (int64_t)(p1 >> 1) * (mc + 1) + (p0 >> 1)] = K(p0, p1);
  }
}

// Dense Cholesky of the coarsest operator, one thread per sample (fem.cpp:255-272).
__global__ void coarse_factor_kernel(Geo g, int B, const double* __restrict__ D,
                                     const double* __restrict__ E, const double* __restrict__ Nw,
                                     double* __restrict__ chol) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int n = (int)g.N, n0 = g.n0;
  double* L = chol + (int64_t)b * n * n;
  const double* Db = D + (int64_t)b * n;
  const double* Eb = E + (int64_t)b * n;
  const double* Nb = Nw + (int64_t)b * n;
  for (int i = 0; i < n * n; ++i) L[i] = 0.0;
  for (int i = 0; i < n; ++i) {
    const int p1 = i / n0, p0 = i - p1 * n0;
    L[i * n + i] = Db[i];
    if (p0 + 1 < n0) { L[i * n + i + 1] = Eb[i]; L[(i + 1) * n + i] = Eb[i]; }
    if (p1 + 1 < n0) { L[i * n + i + n0] = Nb[i]; L[(i + n0) * n + i] = Nb[i]; }
  }
  for (int j = 0; j < n; ++j) {
    double d = L[j * n + j];
    for (int q = 0; q < j; ++q) d -= L[j * n + q] * L[j * n + q];
    L[j * n + j] = sqrt(d);
    const double inv = 1.0 / L[j * n + j];
    for (int i = j + 1; i < n; ++i) {
      double v = L[i * n + j];
      for (int q = 0; q < j; ++q) v -= L[i * n + q] * L[j * n + q];
      L[i * n + j] = v * inv;
    }
  }
}

// ---- stencil helpers --------------------------------------------------------------------------
struct St {
  const double* __restrict__ D;
  const double* __restrict__ E;
  const double* __restrict__ Nw;
};

// Σ_nb A(i,nb) x(nb) (off-diagonal part) at node (p0,p1) of sample slice x.
__device__ __forceinline__ double offdiag(const St& s, const double* __restrict__ x, int64_t i,
                                          int p0, int p1, int m, int n0) {
  double acc = 0.0;
  if (p0 < m) acc += __ldg(s.E + i) * x[i + 1];
  if (p0 > 0) acc += __ldg(s.E + i - 1) * x[i - 1];
  if (p1 < m) acc += __ldg(s.Nw + i) * x[i + n0];
  if (p1 > 0) acc += __ldg(s.Nw + i - n0) * x[i - n0];
  return acc;
}

#define NODE_PROLOGUE                                                     \
  const int b = blockIdx.y;                                               \
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;                            \
  const int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x;               \
  const int m = g.m, n0 = g.n0;                                           \
  const int p1 = (int)(i / n0), p0 = (int)(i - (int64_t)p1 * n0);         \
  const int64_t off = (int64_t)b * g.N;                                   \
  const bool in = i < g.N;

// ---- PCG init: u = lift, r = b − A u (= b on interior rows, 0 on Dirichlet rows) -------------
__global__ void __launch_bounds__(NT) pcg_init_kernel(Geo g, int bc, int forcing, double fval,
                                                      double tol, int max_iter_factor,
                                                      const double* __restrict__ k,
                                                      double* __restrict__ u, double* __restrict__ r,
                                                      double* scal, int* flags, double2* partial,
                                                      int maxp, unsigned* counter, int* n_active,
                                                      double* hist, int hist_cap) {
  const int b = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x;
  const int m = g.m, n0 = g.n0;
  const int p1 = (int)(i / n0), p0 = (int)(i - (int64_t)p1 * n0);
  const int64_t off = (int64_t)b * g.N;
  double bb = 0.0, rr = 0.0;
  if (i < g.N) {
    const bool dself = is_dir(bc, m, p0, p1);
    const double g_self = (bc == OSC_BC_FLOWCELL && p0 == 0) ? 1.0 : 0.0;
    double bi;
    if (dself) {
      bi = g_self;
      u[off + i] = g_self;
      r[off + i] = 0.0;
    } else {
      // load: f·area/3 per incident triangle (fem.cpp:85-86)
      const int tri = 2 * (p0 < m && p1 < m) + (p0 > 0 && p1 < m) + 2 * (p0 > 0 && p1 > 0) +
                      (p0 < m && p1 > 0);
      const double h = 1.0 / m;
      bi = forcing ? tri * (fval * (0.5 * h * h) / 3.0) : 0.0;
      // symmetric elimination of the u=1 column at x=0 (fem.cpp:109-114)
      if (bc == OSC_BC_FLOWCELL && p0 == 1) {
        const double* kb = k + off;
        auto K = [&](int a0, int a1) { return kb[(int64_t)a1 * n0 + a0]; };
        const double e = -0.5 * ((p1 < m ? (K(0, p1) + K(1, p1) + K(1, p1 + 1)) / 3.0 : 0.0) +
                                 (p1 > 0 ? (K(0, p1 - 1) + K(1, p1) + K(0, p1)) / 3.0 : 0.0));
        bi -= e * 1.0;
      }
      u[off + i] = 0.0;
      r[off + i] = bi;
      rr = bi * bi;
    }
    bb = bi * bi;
  }
  double tb, tr;
  if (reduce2_last(bb, rr, partial, maxp, counter, b, tb, tr) && threadIdx.x == 0) {
    const double bnorm = sqrt(tb);
    const double rel = sqrt(tr) / bnorm;
    scal[b * S_NSCAL + S_BNORM] = bnorm;
    scal[b * S_NSCAL + S_REL] = rel;
    scal[b * S_NSCAL + S_RZ] = 0.0;
    scal[b * S_NSCAL + S_BETA] = 0.0;
    const int act = rel > tol ? 1 : 0;  // NaN (b = 0) → converged, as in fem.cpp:367
    flags[b * F_NFLAGS + F_ACTIVE] = act;
    flags[b * F_NFLAGS + F_ITERS] = 0;
    flags[b * F_NFLAGS + F_STATUS] = 0;
    flags[b * F_NFLAGS + F_FIRST] = 1;
    const int64_t cap = (int64_t)max_iter_factor * g.N;
    flags[b * F_NFLAGS + F_MAXIT] = (int)(cap < 0x7fffffff ? cap : 0x7fffffff);
    if (hist && hist_cap > 0) hist[(int64_t)b * hist_cap] = rel;
    if (act) atomicAdd(n_active, 1);
  }
}

// ---- PCG: p = z + βp (p = z first), Ap, <p,Ap> → α -----------------------------------------------
__global__ void __launch_bounds__(NT) pcg_apply_kernel(Geo g, St s, const double* __restrict__ z,
                                                       const double* __restrict__ p_old,
                                                       double* __restrict__ p_new,
                                                       double* __restrict__ Ap, double* scal,
                                                       int* flags, double2* partial, int maxp,
                                                       unsigned* counter) {
  NODE_PROLOGUE
  const bool first = flags[b * F_NFLAGS + F_FIRST] != 0;
  const double beta = scal[b * S_NSCAL + S_BETA];
  double pap = 0.0;
  if (in) {
    const double* zb = z + off;
    const double* pb = p_old + off;
    auto P = [&](int64_t j) { return first ? zb[j] : fma(beta, pb[j], zb[j]); };
    const double pc = P(i);
    double acc = __ldg(s.D + off + i) * pc;
    if (p0 < m) acc += __ldg(s.E + off + i) * P(i + 1);
    if (p0 > 0) acc += __ldg(s.E + off + i - 1) * P(i - 1);
    if (p1 < m) acc += __ldg(s.Nw + off + i) * P(i + n0);
    if (p1 > 0) acc += __ldg(s.Nw + off + i - n0) * P(i - n0);
    p_new[off + i] = pc;
    Ap[off + i] = acc;
    pap = pc * acc;
  }
  double t0, t1;
  if (reduce2_last(pap, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    scal[b * S_NSCAL + S_ALPHA] = scal[b * S_NSCAL + S_RZ] / t0;
    flags[b * F_NFLAGS + F_FIRST] = 0;
  }
}

// ---- PCG: u += αp, r −= αAp, ‖r‖ → convergence ----------------------------------------------------
__global__ void __launch_bounds__(NT) pcg_update_kernel(Geo g, double tol, const double* __restrict__ p,
                                                        const double* __restrict__ Ap,
                                                        double* __restrict__ u, double* __restrict__ r,
                                                        double* scal, int* flags, double2* partial,
                                                        int maxp, unsigned* counter, int* n_active,
                                                        double* hist, int hist_cap) {
  NODE_PROLOGUE
  (void)p0; (void)p1; (void)m; (void)n0;
  const double alpha = scal[b * S_NSCAL + S_ALPHA];
  double rr = 0.0;
  if (in) {
    u[off + i] = fma(alpha, p[off + i], u[off + i]);
    const double rn = fma(-alpha, Ap[off + i], r[off + i]);
    r[off + i] = rn;
    rr = rn * rn;
  }
  double t0, t1;
  if (reduce2_last(rr, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    const double rel = sqrt(t0) / scal[b * S_NSCAL + S_BNORM];
    const int it = flags[b * F_NFLAGS + F_ITERS] + 1;
    flags[b * F_NFLAGS + F_ITERS] = it;
    scal[b * S_NSCAL + S_REL] = rel;
    if (hist && it < hist_cap) hist[(int64_t)b * hist_cap + it] = rel;
    if (rel <= tol) {
      flags[b * F_NFLAGS + F_ACTIVE] = 0;
      atomicSub(n_active, 1);
    } else if (!isfinite(rel)) {  // breakdown (non-finite residual): fail fast, never spin to the cap
      flags[b * F_NFLAGS + F_ACTIVE] = 0;
      flags[b * F_NFLAGS + F_STATUS] = OSC_ERR_SOLVER;
      atomicSub(n_active, 1);
    } else if (it >= flags[b * F_NFLAGS + F_MAXIT]) {
      flags[b * F_NFLAGS + F_ACTIVE] = 0;
      flags[b * F_NFLAGS + F_STATUS] = OSC_ERR_SOLVER;
      atomicSub(n_active, 1);
    }
  }
}

// ---- V-cycle pieces ----------------------------------------------------------------------------------
// pre-smooth from z = 0: red z = r/D, then black z = (r − Σ A z_red)/D
__global__ void __launch_bounds__(NT) smooth_down_kernel(Geo g, St s, const double* __restrict__ r,
                                                         double* __restrict__ z, const int* flags) {
  NODE_PROLOGUE
  if (!in) return;
  const St sb{s.D + off, s.E + off, s.Nw + off};
  const double* rb = r + off;
  double val;
  if (((p0 + p1) & 1) == 0) {
    val = rb[i] / __ldg(sb.D + i);
  } else {
    double acc = 0.0;
    if (p0 < m) acc += __ldg(sb.E + i) * (rb[i + 1] / __ldg(sb.D + i + 1));
    if (p0 > 0) acc += __ldg(sb.E + i - 1) * (rb[i - 1] / __ldg(sb.D + i - 1));
    if (p1 < m) acc += __ldg(sb.Nw + i) * (rb[i + n0] / __ldg(sb.D + i + n0));
    if (p1 > 0) acc += __ldg(sb.Nw + i - n0) * (rb[i - n0] / __ldg(sb.D + i - n0));
    val = (rb[i] - acc) / __ldg(sb.D + i);
  }
  z[off + i] = val;
}

// residual t = r − A z at fine node (a0,a1)
__device__ __forceinline__ double resid_at(const St& sb, const double* __restrict__ rb,
                                           const double* __restrict__ zb, int a0, int a1, int m,
                                           int n0) {
  const int64_t j = (int64_t)a1 * n0 + a0;
  return rb[j] - __ldg(sb.D + j) * zb[j] - offdiag(sb, zb, j, a0, a1, m, n0);
}

// coarse residual rc = Pᵀ (r − A z), zero at coarse Dirichlet nodes (fem.cpp:168-195)
__global__ void __launch_bounds__(NT) restrict_kernel(Geo g, Geo gc, int bc, St s,
                                                      const double* __restrict__ r,
                                                      const double* __restrict__ z,
                                                      double* __restrict__ rc, const int* flags) {
  const int b = blockIdx.y;
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;
  const int64_t ic = blockIdx.x * (int64_t)NT + threadIdx.x;
  if (ic >= gc.N) return;
  const int mc = gc.m;
  const int J = (int)(ic / gc.n0), I = (int)(ic - (int64_t)J * gc.n0);
  double acc = 0.0;
  if (!is_dir(bc, mc, I, J)) {
    const int64_t off = (int64_t)b * g.N;
    const St sb{s.D + off, s.E + off, s.Nw + off};
    const double* rb = r + off;
    const double* zb = z + off;
    const int m = g.m, n0 = g.n0;
    const int f0 = 2 * I, f1 = 2 * J;
    acc = resid_at(sb, rb, zb, f0, f1, m, n0);
    double half = 0.0;
    if (f0 > 0) half += resid_at(sb, rb, zb, f0 - 1, f1, m, n0);
    if (f0 < m) half += resid_at(sb, rb, zb, f0 + 1, f1, m, n0);
    if (f1 > 0) half += resid_at(sb, rb, zb, f0, f1 - 1, m, n0);
    if (f1 < m) half += resid_at(sb, rb, zb, f0, f1 + 1, m, n0);
    if (f0 < m && f1 < m) half += resid_at(sb, rb, zb, f0 + 1, f1 + 1, m, n0);
    if (f0 > 0 && f1 > 0) half += resid_at(sb, rb, zb, f0 - 1, f1 - 1, m, n0);
    acc += 0.5 * half;
  }
  rc[(int64_t)b * gc.N + ic] = acc;
}

// P1 prolongation of the coarse correction at fine node (a0,a1) (fem.cpp:144-165)
__device__ __forceinline__ double prolong_at(const double* __restrict__ zc, int a0, int a1,
                                             int nc0) {
  const bool ex = (a0 & 1) == 0, ey = (a1 & 1) == 0;
  auto Z = [&](int c0, int c1) { return zc[(int64_t)c1 * nc0 + c0]; };
  if (ex && ey) return Z(a0 >> 1, a1 >> 1);
  if (!ex && ey) return 0.5 * (Z((a0 - 1) >> 1, a1 >> 1) + Z((a0 + 1) >> 1, a1 >> 1));
  if (ex && !ey) return 0.5 * (Z(a0 >> 1, (a1 - 1) >> 1) + Z(a0 >> 1, (a1 + 1) >> 1));
  return 0.5 * (Z((a0 - 1) >> 1, (a1 - 1) >> 1) + Z((a0 + 1) >> 1, (a1 + 1) >> 1));
}

// post-smooth part 1: black z = (r − Σ A (z_red + P zc)_nb)/D ; red untouched
__global__ void __launch_bounds__(NT) smooth_up_black_kernel(Geo g, Geo gc, St s,
                                                             const double* __restrict__ r,
                                                             double* __restrict__ z,
                                                             const double* __restrict__ zc,
                                                             const int* flags) {
  NODE_PROLOGUE
  if (!in || ((p0 + p1) & 1) == 0) return;
  const St sb{s.D + off, s.E + off, s.Nw + off};
  const double* zb = z + off;
  const double* zcb = zc + (int64_t)b * gc.N;
  const int nc0 = gc.n0;
  auto V = [&](int64_t j, int a0, int a1) { return zb[j] + prolong_at(zcb, a0, a1, nc0); };
  double acc = 0.0;
  if (p0 < m) acc += __ldg(sb.E + i) * V(i + 1, p0 + 1, p1);
  if (p0 > 0) acc += __ldg(sb.E + i - 1) * V(i - 1, p0 - 1, p1);
  if (p1 < m) acc += __ldg(sb.Nw + i) * V(i + n0, p0, p1 + 1);
  if (p1 > 0) acc += __ldg(sb.Nw + i - n0) * V(i - n0, p0, p1 - 1);
  z[off + i] = (r[off + i] - acc) / __ldg(sb.D + i);
}

// post-smooth part 2: red z = (r − Σ A z_black)/D; on level 0 also <r,z> → β
__global__ void __launch_bounds__(NT) smooth_up_red_kernel(Geo g, St s, const double* __restrict__ r,
                                                           double* __restrict__ z, int finest,
                                                           double* scal, int* flags,
                                                           double2* partial, int maxp,
                                                           unsigned* counter) {
  NODE_PROLOGUE
  double rz = 0.0;
  if (in) {
    const St sb{s.D + off, s.E + off, s.Nw + off};
    const double* zb = z + off;
    const double ri = r[off + i];
    double zi;
    if (((p0 + p1) & 1) == 0) {
      zi = (ri - offdiag(sb, zb, i, p0, p1, m, n0)) / __ldg(sb.D + i);
      z[off + i] = zi;
    } else {
      zi = zb[i];
    }
    rz = ri * zi;
  }
  if (!finest) return;
  double t0, t1;
  if (reduce2_last(rz, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    const double old = scal[b * S_NSCAL + S_RZ];
    scal[b * S_NSCAL + S_BETA] = flags[b * F_NFLAGS + F_ITERS] == 0 ? 0.0 : t0 / old;
    scal[b * S_NSCAL + S_RZ] = t0;
  }
}

// single-level case (no coarser grid): <r,z> → β
__global__ void __launch_bounds__(NT) dot_rz_kernel(Geo g, const double* __restrict__ r,
                                                    const double* __restrict__ z, double* scal,
                                                    int* flags, double2* partial, int maxp,
                                                    unsigned* counter) {
  NODE_PROLOGUE
  (void)p0; (void)p1; (void)m; (void)n0;
  const double rz = in ? r[off + i] * z[off + i] : 0.0;
  double t0, t1;
  if (reduce2_last(rz, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    const double old = scal[b * S_NSCAL + S_RZ];
    scal[b * S_NSCAL + S_BETA] = flags[b * F_NFLAGS + F_ITERS] == 0 ? 0.0 : t0 / old;
    scal[b * S_NSCAL + S_RZ] = t0;
  }
}

// coarsest solve z = L⁻ᵀ L⁻¹ r, one thread per sample (fem.cpp:274-286)
__global__ void coarse_solve_kernel(int n, int B, const double* __restrict__ chol,
                                    const double* __restrict__ r, double* __restrict__ z,
                                    const int* flags) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || !flags[b * F_NFLAGS + F_ACTIVE]) return;
  const double* L = chol + (int64_t)b * n * n;
  const double* rb = r + (int64_t)b * n;
  double* zb = z + (int64_t)b * n;
  for (int i = 0; i < n; ++i) {
    double v = rb[i];
    for (int q = 0; q < i; ++q) v -= L[i * n + q] * zb[q];
    zb[i] = v / L[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double v = zb[i];
    for (int q = i + 1; q < n; ++q) v -= L[q * n + i] * zb[q];
    zb[i] = v / L[i * n + i];
  }
}

// ---- QoIs (fem.cpp:402-436 + extensions) -------------------------------------------------------------
__global__ void __launch_bounds__(NT) qoi_kernel(Geo g, int qoi, double qx, double qy, int forcing,
                                                 double fval, const double* __restrict__ u,
                                                 const double* __restrict__ k,
                                                 double* __restrict__ q, double2* partial, int maxp,
                                                 unsigned* counter) {
  const int b = blockIdx.y;
  const int m = g.m, n0 = g.n0;
  const double* ub = u + (int64_t)b * g.N;
  if (qoi == OSC_QOI_POINT) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      int i = (int)(qx * m), j = (int)(qy * m);
      i = min(i, m - 1);
      j = min(j, m - 1);
      const double xi = qx * m - i, eta = qy * m - j;
      const double ull = ub[j * n0 + i], ulr = ub[j * n0 + i + 1], uur = ub[(j + 1) * n0 + i + 1],
                   uul = ub[(j + 1) * n0 + i];
      q[b] = (eta <= xi) ? (1.0 - xi) * ull + (xi - eta) * ulr + eta * uur
                         : (1.0 - eta) * ull + xi * uur + (eta - xi) * uul;
    }
    return;
  }
  const int64_t t = blockIdx.x * (int64_t)NT + threadIdx.x;
  double v = 0.0;
  const double h = 1.0 / m;
  if (qoi == OSC_QOI_FLUX) {
    // −Σ_{p1} (K_raw u − F) at the x = 1 nodes (reaction flux of the un-eliminated rows)
    if (t <= m) {
      const int p1 = (int)t, p0 = m;
      const double* kb = k + (int64_t)b * g.N;
      auto K = [&](int a0, int a1) { return kb[(int64_t)a1 * n0 + a0]; };
      auto U = [&](int a0, int a1) { return ub[(int64_t)a1 * n0 + a0]; };
      const double ew = -0.5 * ((p1 < m ? (K(p0 - 1, p1) + K(p0, p1) + K(p0, p1 + 1)) / 3.0 : 0.0) +
                                (p1 > 0 ? (K(p0 - 1, p1 - 1) + K(p0, p1) + K(p0 - 1, p1)) / 3.0 : 0.0));
      const double en = p1 < m ? -0.5 * (K(p0 - 1, p1) + K(p0, p1) + K(p0, p1 + 1)) / 3.0 : 0.0;
      const double es = p1 > 0 ? -0.5 * (K(p0 - 1, p1 - 1) + K(p0, p1 - 1) + K(p0, p1)) / 3.0 : 0.0;
      const double d = -(ew + en + es);
      double Ku = d * U(p0, p1) + ew * U(p0 - 1, p1);
      if (p1 < m) Ku += en * U(p0, p1 + 1);
      if (p1 > 0) Ku += es * U(p0, p1 - 1);
      const int tri = (p1 < m) + 2 * (p1 > 0);
      const double F = forcing ? tri * (fval * (0.5 * h * h) / 3.0) : 0.0;
      v = -(Ku - F);
    }
  } else {
    // triangle sums over cell t = (ci, cj)
    if (t < (int64_t)m * m) {
      const int cj = (int)(t / m), ci = (int)(t - (int64_t)cj * m);
      const int64_t a = (int64_t)cj * n0 + ci;
      const double area = 0.5 * h * h;
      const double u00 = ub[a], u10 = ub[a + 1], u11 = ub[a + n0 + 1], u01 = ub[a + n0];
      if (qoi == OSC_QOI_L2) {
        const double s1 = u00 + u10 + u11, s2 = u00 + u11 + u01;
        v = area / 12.0 * (u00 * u00 + u10 * u10 + u11 * u11 + s1 * s1) +
            area / 12.0 * (u00 * u00 + u11 * u11 + u01 * u01 + s2 * s2);
      } else {
        v = area * (u00 + u10 + u11) / 3.0 + area * (u00 + u11 + u01) / 3.0;
      }
    }
  }
  double t0, t1;
  if (reduce2_last(v, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0)
    q[b] = (qoi == OSC_QOI_L2) ? sqrt(t0) : t0;
}

__global__ void exp_field_kernel(const double* __restrict__ Z, double* __restrict__ k,
                                 int64_t total, int64_t per_sample, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double z = Z[i];
    if (!isfinite(z)) atomicOr(bad + i / per_sample, 1);
    k[i] = exp(z);
  }
}

// per-level sums in slot order: [n, Σ(Y−K), Σ(Y−K)², Σ(q−Kq), Σ(q−Kq)²], one CTA
__global__ void level_sums_kernel(const double* __restrict__ qf, const double* __restrict__ qc,
                                  int B, double ky, double kq, double* sums) {
  __shared__ double sh[32];
  double a[4] = {0, 0, 0, 0};
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const double y = (qc ? qf[i] - qc[i] : qf[i]) - ky;
    const double q = qf[i] - kq;
    a[0] += y; a[1] += y * y; a[2] += q; a[3] += q * q;
  }
  for (int j = 0; j < 4; ++j) {
    const double t = block_sum(a[j], sh);
    __syncthreads();
    if (threadIdx.x == 0) sums[1 + j] += t;
  }
  if (threadIdx.x == 0) sums[0] += B;
}

inline int nblocks(int64_t N) { return (int)((N + NT - 1) / NT); }

}  // namespace

size_t solver_bytes(int m, int B, int hist_cap) {
  size_t tot = 0;
  int g = m, lev = 0;
  for (;;) {
    const size_t N = (size_t)(g + 1) * (g + 1);
    tot += N * B * sizeof(double) * (lev == 0 ? 10 : 6);
    ++lev;
    if (g <= 4 || g % 2 != 0) { tot += N * N * B * sizeof(double); break; }
    g /= 2;
  }
  tot += (size_t)B * (S_NSCAL * 8 + F_NFLAGS * 4 + 8) + (size_t)B * hist_cap * 8;
  tot += (size_t)B * ((size_t)(m + 1) * (m + 1) / NT + 2) * 16;
  return tot + 4096 * 16;
}

void solver_prepare(Ctx* ctx, int m, int B, int hist_cap) {
  SolverWork& w = ctx->solver;
  OSC_REQUIRE(m >= 1, "solve: m must be >= 1");
  w.m = m;
  w.B = B;
  w.hist_cap = hist_cap;
  // hierarchy geometry
  int g = m, nl = 0;
  for (;;) {
    w.lev[nl].m = g;
    w.lev[nl].N = (int64_t)(g + 1) * (g + 1);
    ++nl;
    if (g <= 4 || g % 2 != 0 || nl == 24) break;
    g /= 2;
  }
  w.nlev = nl;
  w.nc = (int)w.lev[nl - 1].N;
  OSC_REQUIRE(w.nc <= 1089, "solve: coarsest multigrid grid too large (m must be 2^j * c, c <= 32)");
  w.max_parts = nblocks(w.lev[0].N);
  w.mem.ensure(solver_bytes(m, B, hist_cap));
  char* p = static_cast<char*>(w.mem.p);
  auto take = [&](size_t bytes) {
    void* q = p;
    p += (bytes + 255) & ~size_t(255);
    return q;
  };
  for (int l = 0; l < nl; ++l) {
    SolverLevel& L = w.lev[l];
    const size_t vb = sizeof(double) * L.N * B;
    if (l > 0) L.k = (double*)take(vb);  // level 0's k is provided by the caller buffer
    L.D = (double*)take(vb);
    L.E = (double*)take(vb);
    L.Nw = (double*)take(vb);
    L.r = (double*)take(vb);
    L.z = (double*)take(vb);
  }
  const size_t vb0 = sizeof(double) * w.lev[0].N * B;
  w.u = (double*)take(vb0);
  w.p0 = (double*)take(vb0);
  w.p1 = (double*)take(vb0);
  w.Ap = (double*)take(vb0);
  w.chol = (double*)take(sizeof(double) * (size_t)w.nc * w.nc * B);
  w.scal = (double*)take(sizeof(double) * S_NSCAL * B);
  w.flags = (int*)take(sizeof(int) * F_NFLAGS * B);
  w.counter = (unsigned*)take(sizeof(unsigned) * B);
  w.n_active = (int*)take(sizeof(int) * 4);
  w.partial = (double*)take(sizeof(double2) * (size_t)w.max_parts * B);
  w.hist = hist_cap > 0 ? (double*)take(sizeof(double) * (size_t)hist_cap * B) : nullptr;
  OSC_REQUIRE((size_t)(p - static_cast<char*>(w.mem.p)) <= w.mem.bytes, "solver workspace overflow");
  OSC_CUDA(cudaMemsetAsync(w.counter, 0, sizeof(unsigned) * B, ctx->stream));
  OSC_CUDA(cudaMemsetAsync(w.n_active, 0, sizeof(int) * 4, ctx->stream));
  if (w.hist) OSC_CUDA(cudaMemsetAsync(w.hist, 0, sizeof(double) * (size_t)hist_cap * B, ctx->stream));
}

namespace {

Geo geo_of(const SolverLevel& L) { return Geo{L.m, L.m + 1, L.N}; }
St st_of(const SolverLevel& L) { return St{L.D, L.E, L.Nw}; }

void vcycle(Ctx* ctx, int bc, int B) {
  SolverWork& w = ctx->solver;
  cudaStream_t st = ctx->stream;
  double2* part = reinterpret_cast<double2*>(w.partial);
  if (w.nlev == 1) {
    {
      KScope ks(ctx, "mg_coarse_solve");
      coarse_solve_kernel<<<(B + 63) / 64, 64, 0, st>>>(w.nc, B, w.chol, w.lev[0].r, w.lev[0].z, w.flags);
    }
    KScope ks(ctx, "pcg_dot_rz");
    dot_rz_kernel<<<dim3(nblocks(w.lev[0].N), B), NT, 0, st>>>(geo_of(w.lev[0]), w.lev[0].r, w.lev[0].z,
                                                              w.scal, w.flags, part, w.max_parts, w.counter);
    return;
  }
  for (int l = 0; l + 1 < w.nlev; ++l) {
    const SolverLevel& L = w.lev[l];
    const SolverLevel& C = w.lev[l + 1];
    {
      KScope ks(ctx, "mg_smooth_down");
      smooth_down_kernel<<<dim3(nblocks(L.N), B), NT, 0, st>>>(geo_of(L), st_of(L), L.r, L.z, w.flags);
    }
    KScope ks(ctx, "mg_restrict");
    restrict_kernel<<<dim3(nblocks(C.N), B), NT, 0, st>>>(geo_of(L), geo_of(C), bc, st_of(L), L.r, L.z,
                                                         C.r, w.flags);
  }
  {
    const SolverLevel& C = w.lev[w.nlev - 1];
    KScope ks(ctx, "mg_coarse_solve");
    coarse_solve_kernel<<<(B + 63) / 64, 64, 0, st>>>(w.nc, B, w.chol, C.r, C.z, w.flags);
  }
  for (int l = w.nlev - 2; l >= 0; --l) {
    const SolverLevel& L = w.lev[l];
    const SolverLevel& C = w.lev[l + 1];
    {
      KScope ks(ctx, "mg_smooth_up_black");
      smooth_up_black_kernel<<<dim3(nblocks(L.N), B), NT, 0, st>>>(geo_of(L), geo_of(C), st_of(L), L.r,
                                                                   L.z, C.z, w.flags);
    }
    KScope ks(ctx, "mg_smooth_up_red");
    smooth_up_red_kernel<<<dim3(nblocks(L.N), B), NT, 0, st>>>(geo_of(L), st_of(L), L.r, L.z, l == 0 ? 1 : 0,
                                                               w.scal, w.flags, part, w.max_parts,
                                                               w.counter);
  }
  OSC_CUDA(cudaGetLastError());
}

}  // namespace

// Solve the batch whose level-0 conductivity sits in ctx->solver.lev[0].k (set by caller).
void solver_run(Ctx* ctx, const osc_problem* prob, int B) {
  SolverWork& w = ctx->solver;
  cudaStream_t st = ctx->stream;
  double2* part = reinterpret_cast<double2*>(w.partial);
  const int bc = prob->bc;
  struct TagGuard {
    Ctx* c;
    ~TagGuard() { c->tag.clear(); }
  } tg{ctx};
  ctx->tag = std::to_string(w.m);
  // setup: stencils + injection + coarse factor
  {
    KScope ks(ctx, "mg_setup", w.nlev + 1);
    for (int l = 0; l < w.nlev; ++l) {
      SolverLevel& L = w.lev[l];
      double* kc = (l + 1 < w.nlev) ? w.lev[l + 1].k : nullptr;
      setup_level_kernel<<<dim3(nblocks(L.N), B), NT, 0, st>>>(geo_of(L), bc, L.k, L.D, L.E, L.Nw, kc);
    }
    const SolverLevel& C = w.lev[w.nlev - 1];
    coarse_factor_kernel<<<(B + 63) / 64, 64, 0, st>>>(geo_of(C), B, C.D, C.E, C.Nw, w.chol);
    OSC_CUDA(cudaGetLastError());
  }
  SolverLevel& L0 = w.lev[0];
  const Geo g0 = geo_of(L0);
  const int nb0 = nblocks(L0.N);
  OSC_CUDA(cudaMemsetAsync(w.n_active, 0, sizeof(int), st));
  {
    KScope ks(ctx, "pcg_init");
    pcg_init_kernel<<<dim3(nb0, B), NT, 0, st>>>(g0, bc, prob->forcing, prob->forcing_value, prob->tol,
                                                 prob->max_iter_factor, L0.k, w.u, L0.r, w.scal, w.flags,
                                                 part, w.max_parts, w.counter, w.n_active, w.hist,
                                                 w.hist_cap);
  }
  vcycle(ctx, bc, B);  // z = M r, rz = <r,z>
  double* p_old = w.p0;
  double* p_new = w.p1;
  const int check_every = L0.N >= 65536 ? 1 : 4;
  for (int it = 0;; ++it) {
    if (it % check_every == 0) {
      OSC_CUDA(cudaMemcpyAsync(ctx->h_pinned_int, w.n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
      OSC_CUDA(cudaStreamSynchronize(st));
      if (*ctx->h_pinned_int <= 0) break;
    }
    {
      KScope ks(ctx, "pcg_apply");
      pcg_apply_kernel<<<dim3(nb0, B), NT, 0, st>>>(g0, st_of(L0), L0.z, p_old, p_new, w.Ap, w.scal,
                                                    w.flags, part, w.max_parts, w.counter);
    }
    {
      KScope ks(ctx, "pcg_update");
      pcg_update_kernel<<<dim3(nb0, B), NT, 0, st>>>(g0, prob->tol, p_new, w.Ap, w.u, L0.r, w.scal,
                                                     w.flags, part, w.max_parts, w.counter, w.n_active,
                                                     w.hist, w.hist_cap);
    }
    vcycle(ctx, bc, B);
    std::swap(p_old, p_new);
  }
}

void qoi_launch(Ctx* ctx, const osc_problem* prob, int B, double* q_dev) {
  SolverWork& w = ctx->solver;
  const SolverLevel& L0 = w.lev[0];
  const int m = L0.m;
  ctx->tag = std::to_string(m);
  struct TagGuard {
    Ctx* c;
    ~TagGuard() { c->tag.clear(); }
  } tg{ctx};
  int64_t items = 1;
  if (prob->qoi == OSC_QOI_FLUX) items = m + 1;
  else if (prob->qoi != OSC_QOI_POINT) items = (int64_t)m * m;
  KScope ks(ctx, "qoi");
  qoi_kernel<<<dim3(nblocks(items), B), NT, 0, ctx->stream>>>(
      geo_of(L0), prob->qoi, prob->qoi_x, prob->qoi_y, prob->forcing, prob->forcing_value, w.u, L0.k,
      q_dev, reinterpret_cast<double2*>(w.partial), w.max_parts, w.counter);
  OSC_CUDA(cudaGetLastError());
}

void solver_results(Ctx* ctx, int B, int32_t* iters, int32_t* status, double* hist_host) {
  SolverWork& w = ctx->solver;
  std::vector<int> fl((size_t)B * F_NFLAGS);
  OSC_CUDA(cudaMemcpyAsync(fl.data(), w.flags, sizeof(int) * fl.size(), cudaMemcpyDeviceToHost, ctx->stream));
  if (hist_host && w.hist)
    OSC_CUDA(cudaMemcpyAsync(hist_host, w.hist, sizeof(double) * (size_t)B * w.hist_cap,
                             cudaMemcpyDeviceToHost, ctx->stream));
  OSC_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int b = 0; b < B; ++b) {
    if (iters) iters[b] = fl[(size_t)b * F_NFLAGS + F_ITERS];
    if (status) status[b] = fl[(size_t)b * F_NFLAGS + F_STATUS];
  }
}

void level_sums_launch(Ctx* ctx, const double* qf, const double* qc, int B, double shift_y,
                       double shift_q, double* sums_dev) {
  KScope ks(ctx, "level_sums");
  level_sums_kernel<<<1, 256, 0, ctx->stream>>>(qf, qc, B, shift_y, shift_q, sums_dev);
  OSC_CUDA(cudaGetLastError());
}

void exp_field_launch(Ctx* ctx, const double* Z, double* k, int64_t total, int* bad_flag) {
  const int64_t per = ctx->solver.lev[0].N;
  KScope ks(ctx, "exp_field");
  exp_field_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 8192), 256, 0, ctx->stream>>>(
      Z, k, total, per, bad_flag);
  OSC_CUDA(cudaGetLastError());
}

}  // namespace osc
