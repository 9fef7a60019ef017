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
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

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
  const int part = blockIdx.y * gridDim.x + blockIdx.x;
  const int nparts = gridDim.x * gridDim.y;
  __shared__ double sh[32];
  __shared__ int last;
  const double s0 = block_sum(v0, sh);
  __syncthreads();
  const double s1 = block_sum(v1, sh);
  if (threadIdx.x == 0) {
    partial[(int64_t)b * maxp + part] = make_double2(s0, s1);
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

struct Sten {
  double d, e, w, n, s;  // raw diagonal (1 on Dirichlet rows) and eliminated couplings
};

// ---- setup: coarse-level operators -------------------------------------------------------------------
// Level l ≥ 1 keeps its raw edge weights E, N in HBM (before Dirichlet elimination; built once per
// solve). They come from per-triangle conductivities Klo(I,J), Kup(I,J) of the level's cells.
// The triangles of cell (i,j) are lower (i,j),(i+1,j),(i+1,j+1) and upper (i,j),(i+1,j+1),(i,j+1)
// (fem.cpp:62-63). The two coarse-operator modes differ only in those conductivities:
//  * REDISCRETIZE is the reference: vertex means of the injected nodal k (fem.cpp:241-244).
//  * GALERKIN is A_c = Pᵀ A P exactly. The coarse P1 basis functions have constant gradients on
//    each coarse triangle, so Pᵀ A P is the coarse P1 matrix whose triangle conductivity is the
//    mean of the 4 equal-area fine triangles inside it:
//      coarse lower(I,J) = lower(2I,2J), lower(2I+1,2J), upper(2I+1,2J), lower(2I+1,2J+1)
//      coarse upper(I,J) = upper(2I,2J), lower(2I,2J+1), upper(2I,2J+1), upper(2I+1,2J+1)
//    (tests/test_host.py::test_galerkin_coarse_operator_identity checks this against Pᵀ A P).
//    It is still a 5-point stencil, and it cuts the PCG iterations about 2× on rough fields.
// Triangle conductivities of level l+1 are written cell-wise ([J·n0c + I]) into that level's z (lo)
// and z2 (up) buffers, which are free until the solve starts.
// mode: OSC_COARSE_* ; src_lo/src_up = level-l triangles (GALERKIN, l ≥ 1) or null (from k0);
// stride = 2^(l+1) in level-0 nodes (REDISCRETIZE; 1 builds level 0's own triangles).
__global__ void __launch_bounds__(NT) coarsen_tri_kernel(int mode, Geo g0, Geo gf, Geo gc, int stride,
                                                         const double* __restrict__ k0,
                                                         const double* __restrict__ src_lo,
                                                         const double* __restrict__ src_up,
                                                         double* __restrict__ clo, double* __restrict__ cup) {
  const int b = blockIdx.y;
  const int mc = gc.m;
  const int64_t ic = blockIdx.x * (int64_t)NT + threadIdx.x;
  if (ic >= (int64_t)mc * mc) return;
  const int J = (int)(ic / mc), I = (int)(ic - (int64_t)J * mc);
  constexpr double third = 1.0 / 3.0;
  const double* kb = k0 + (int64_t)b * g0.N;
  double lo, up;
  if (mode == OSC_COARSE_REDISCRETIZE) {
    auto K = [&](int x, int y) { return __ldg(kb + (int64_t)(y * stride) * g0.n0 + (int64_t)x * stride); };
    lo = (K(I, J) + K(I + 1, J) + K(I + 1, J + 1)) * third;
    up = (K(I, J) + K(I + 1, J + 1) + K(I, J + 1)) * third;
  } else {
    double fl[4], fu[4];  // fine cells (2I,2J), (2I+1,2J), (2I,2J+1), (2I+1,2J+1)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * I + (c & 1), j = 2 * J + (c >> 1);
      if (src_lo) {
        fl[c] = __ldg(src_lo + (int64_t)b * gf.N + (int64_t)j * gf.n0 + i);
        fu[c] = __ldg(src_up + (int64_t)b * gf.N + (int64_t)j * gf.n0 + i);
      } else {
        auto K = [&](int x, int y) { return __ldg(kb + (int64_t)y * g0.n0 + x); };
        fl[c] = (K(i, j) + K(i + 1, j) + K(i + 1, j + 1)) * third;
        fu[c] = (K(i, j) + K(i + 1, j + 1) + K(i, j + 1)) * third;
      }
    }
    lo = 0.25 * (fl[0] + fl[1] + fu[1] + fl[3]);
    up = 0.25 * (fu[0] + fl[2] + fu[2] + fu[3]);
  }
  const int64_t o = (int64_t)b * gc.N + (int64_t)J * gc.n0 + I;
  clo[o] = lo;
  cup[o] = up;
}

// Raw edge weights of one level from its triangle conductivities:
//   E(x,y) = −½[Klo(x,y) + Kup(x,y−1)],  N(x,y) = −½[Kup(x,y) + Klo(x−1,y)],  zero off the grid.
// With REDISCRETIZE conductivities this is bit-identical to edges_pair on the injected k.
__global__ void __launch_bounds__(NT) edges_kernel(Geo g, const double* __restrict__ klo,
                                                   const double* __restrict__ kup, double* __restrict__ E,
                                                   double* __restrict__ Nn) {
  const int b = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x;
  if (i >= g.N) return;
  const int y = (int)(i / g.n0), x = (int)(i - (int64_t)y * g.n0), m = g.m;
  const double* lo = klo + (int64_t)b * g.N;
  const double* up = kup + (int64_t)b * g.N;
  double e = 0.0, n = 0.0;
  if (x < m) e = -0.5 * ((y < m ? lo[i] : 0.0) + (y > 0 ? up[i - g.n0] : 0.0));
  if (y < m) n = -0.5 * ((x < m ? up[i] : 0.0) + (x > 0 ? lo[i - 1] : 0.0));
  E[(int64_t)b * g.N + i] = e;
  Nn[(int64_t)b * g.N + i] = n;
}

// 5-point row of node (x, y) from stored raw edges (Dirichlet rows identity, couplings to
// Dirichlet nodes eliminated).
__device__ __forceinline__ Sten sten_edges(const double* E, const double* Nn, int n0, int m, int x, int y, int bc) {
  Sten st;
  if (is_dir(bc, m, x, y)) {
    st.d = 1.0;
    st.e = st.w = st.n = st.s = 0.0;
    return st;
  }
  const int i = y * n0 + x;
  const double e = E[i], w = x > 0 ? E[i - 1] : 0.0, n = Nn[i], s = y > 0 ? Nn[i - n0] : 0.0;
  st.d = -(e + w + n + s);
  st.e = is_dir(bc, m, x + 1, y) ? 0.0 : e;
  st.w = is_dir(bc, m, x - 1, y) ? 0.0 : w;
  st.n = is_dir(bc, m, x, y + 1) ? 0.0 : n;
  st.s = is_dir(bc, m, x, y - 1) ? 0.0 : s;
  return st;
}

// Coarsest operator and its explicit inverse, one warp per sample. The reference factors the
// coarsest matrix by dense Cholesky (fem.cpp:255-272) and back-substitutes per V-cycle
// (:274-286); here the SPD matrix is inverted once per solve by Gauss–Jordan (no pivoting
// needed for SPD; lane i owns row i of [A | I] in shared memory), so every V-cycle's coarsest
// solve is one warp-parallel matvec. n ≤ 32 uses this path; larger coarsest grids fall back to
// the per-thread Cholesky + inverse below.
constexpr int CF_WARPS = 2;
__global__ void __launch_bounds__(32 * CF_WARPS) coarse_factor_warp_kernel(Geo g, int bc, int B,
                                                                          const double* __restrict__ E,
                                                                          const double* __restrict__ Nn,
                                                                          double* __restrict__ chol) {
  __shared__ double aug[CF_WARPS][32][65];  // row i: A(i, 0..n−1) | I(i, 0..n−1), padded
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * CF_WARPS + w;
  if (b >= B) return;
  const int n = (int)g.N, n0 = g.n0, m = g.m;
  double(*A)[65] = aug[w];
  if (lane < n) {
    for (int j = 0; j < 2 * n; ++j) A[lane][j] = (j == n + lane) ? 1.0 : 0.0;
    const int gy = lane / n0, gx = lane - gy * n0;
    const Sten st = sten_edges(E + (int64_t)b * n, Nn + (int64_t)b * n, n0, m, gx, gy, bc);
    A[lane][lane] = st.d;
    if (gx + 1 < n0) A[lane][lane + 1] = st.e;
    if (gx > 0) A[lane][lane - 1] = st.w;
    if (gy + 1 < n0) A[lane][lane + n0] = st.n;
    if (gy > 0) A[lane][lane - n0] = st.s;
  }
  __syncwarp();
  for (int c = 0; c < n; ++c) {
    const double inv_p = 1.0 / A[c][c];
    const double f = (lane < n && lane != c) ? A[lane][c] * inv_p : 0.0;
    __syncwarp();
    if (lane < n && lane != c)
      for (int j = c; j < 2 * n; ++j) A[lane][j] = fma(-f, A[c][j], A[lane][j]);
    __syncwarp();
    if (lane == c)
      for (int j = c; j < 2 * n; ++j) A[c][j] *= inv_p;
    __syncwarp();
  }
  double* X = chol + (int64_t)b * 2 * n * n + (int64_t)n * n;
  for (int idx = lane; idx < n * n; idx += 32) X[idx] = A[idx / n][n + idx % n];
}

// Dense Cholesky of the coarsest operator, one thread per sample (fem.cpp:255-272).
__global__ void coarse_factor_kernel(Geo g, int bc, int B, const double* __restrict__ E,
                                     const double* __restrict__ Nn, double* __restrict__ chol) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int n = (int)g.N, n0 = g.n0, m = g.m;
  double* L = chol + (int64_t)b * 2 * n * n;
  for (int i = 0; i < n * n; ++i) L[i] = 0.0;
  for (int i = 0; i < n; ++i) {
    const int gy = i / n0, gx = i - gy * n0;
    const Sten st = sten_edges(E + (int64_t)b * n, Nn + (int64_t)b * n, n0, m, gx, gy, bc);
    L[i * n + i] = st.d;
    if (gx + 1 < n0) L[i * n + i + 1] = st.e;
    if (gx > 0) L[i * n + i - 1] = st.w;
    if (gy + 1 < n0) L[i * n + i + n0] = st.n;
    if (gy > 0) L[i * n + i - n0] = st.s;
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
  // explicit inverse A⁻¹ = L⁻ᵀ L⁻¹ (column by column), so each V-cycle's coarsest solve is one
  // warp-parallel matvec instead of two serial triangular sweeps
  double* X = L + (int64_t)n * n;
  for (int c = 0; c < n; ++c) {
    for (int i = 0; i < n; ++i) {  // forward: L y = e_c
      double v = (i == c) ? 1.0 : 0.0;
      for (int q = 0; q < i; ++q) v -= L[i * n + q] * X[q * n + c];
      X[i * n + c] = v / L[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {  // backward: Lᵀ x = y
      double v = X[i * n + c];
      for (int q = i + 1; q < n; ++q) v -= L[q * n + i] * X[q * n + c];
      X[i * n + c] = v / L[i * n + i];
    }
  }
}

// ---- PCG init: u = lift, r = b − A u (= b on interior rows, 0 on Dirichlet rows) -------------
__global__ void __launch_bounds__(NT) pcg_init_kernel(Geo g, int bc, int forcing, double fval,
                                                      double tol, int max_iter_factor,
                                                      const double* __restrict__ k,
                                                      double* __restrict__ u, double* __restrict__ r,
                                                      double* scal, int* flags, double2* partial,
                                                      int maxp, unsigned* counter, int* n_active,
                                                      double* hist, int hist_cap) {
  const int b = blockIdx.z;
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

// ---- register-marching MG-PCG kernels -----------------------------------------------------------
// One lane per grid column; a warp owns a strip of 32 columns (the outer HX lanes are x-halo) and
// marches up a chunk of LY rows, keeping the few rows each stage needs in registers. x-neighbours
// come from warp shuffles, y-neighbours from the register pipeline: no shared-memory staging and
// no barriers on the data path. The 5-point stencil is recomputed from nodal k per row (8 B/node
// of HBM instead of 24 B/node for stored D/E/N).
constexpr int MW = 4;        // warps (strips) per CTA
constexpr int MT = 32 * MW;  // threads per CTA
constexpr int LY = 32;       // output rows per warp on large grids
// rows marched per warp: long chunks amortise the 2-row warm-up on large grids; short chunks
// cut the serial row-latency chain (and add CTAs) on the small, latency-bound MG levels.
__host__ __device__ __forceinline__ int rows_per_warp(int m) { return m >= 512 ? LY : (m >= 64 ? 16 : 8); }
constexpr int LYC = 16;      // coarse output rows per warp (restriction) on large grids
__host__ __device__ __forceinline__ int coarse_rows_per_warp(int mc) { return mc >= 256 ? LYC : 4; }
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double shup(double v) { return __shfl_up_sync(FULL, v, 1); }
__device__ __forceinline__ double shdn(double v) { return __shfl_down_sync(FULL, v, 1); }

// Load one node; INT (interior warp-chunk) skips the bounds test.
template <bool INT>
__device__ __forceinline__ double ldv(const double* __restrict__ base, int gx, int gy, int n0) {
  if (INT) return __ldg(base + (int64_t)gy * n0 + gx);
  return ((unsigned)gx < (unsigned)n0 && (unsigned)gy < (unsigned)n0)
             ? __ldg(base + (int64_t)gy * n0 + gx) : 0.0;
}

// 1/d to full double precision: MUFU approximation + two Newton steps (no DDIV sequence).
__device__ __forceinline__ double rcp64(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = fma(y, fma(-d, y, 1.0), y);
  y = fma(y, fma(-d, y, 1.0), y);
  return y;
}

// ---- column-pair marching ------------------------------------------------------------------------
// Lane l owns the column pair xa = 60·strip − 2 + 2l (even) and xb = xa + 1, so every row gives
// each lane exactly one red and one black node: the red-black sweeps run without divergence and
// every load instruction moves two independent rows' worth of work. Lanes 0 and 31 are the
// 2-column x-halo; lanes 1..30 write.
struct Pair {
  double a, b;
};

template <bool INT>
__device__ __forceinline__ Pair ld2(const double* __restrict__ base, int xa, int y, int n0) {
  return Pair{ldv<INT>(base, xa, y, n0), ldv<INT>(base, xa + 1, y, n0)};
}

// Edge weights of row y at both columns from k rows y−1, y, y+1. Triangle means in the
// reference's vertex order with ·(1/3) instead of /3 (≤ 1 ulp per coefficient); each edge is
// formed once, so both rows of A see the same double. INT: every edge of the pair is interior.
template <bool INT>
__device__ __forceinline__ void edges_pair(Pair km, Pair k0, Pair kp, int xa, int y, int m, Pair& E,
                                           Pair& N) {
  constexpr double third = 1.0 / 3.0;
  const double k0a_e = shdn(k0.a), kpa_e = shdn(kp.a), k0b_w = shup(k0.b);  // k(xb+1,y), k(xb+1,y+1), k(xa−1,y)
  if (INT) {
    E.a = -0.5 * ((k0.a + k0.b + kp.b) * third + (km.a + k0.b + k0.a) * third);
    E.b = -0.5 * ((k0.b + k0a_e + kpa_e) * third + (km.b + k0a_e + k0.b) * third);
    N.a = -0.5 * ((k0.a + kp.b + kp.a) * third + (k0b_w + k0.a + kp.a) * third);
    N.b = -0.5 * ((k0.b + kpa_e + kp.b) * third + (k0.a + k0.b + kp.b) * third);
    return;
  }
  const int xb = xa + 1;
  E.a = E.b = N.a = N.b = 0.0;
  if (y >= 0 && y <= m) {
    if (xa >= 0 && xa < m)
      E.a = -0.5 * ((y < m ? (k0.a + k0.b + kp.b) * third : 0.0) + (y > 0 ? (km.a + k0.b + k0.a) * third : 0.0));
    if (xb >= 0 && xb < m)
      E.b = -0.5 * ((y < m ? (k0.b + k0a_e + kpa_e) * third : 0.0) + (y > 0 ? (km.b + k0a_e + k0.b) * third : 0.0));
  }
  if (y >= 0 && y < m) {
    if (xa >= 0 && xa <= m)
      N.a = -0.5 * ((xa < m ? (k0.a + kp.b + kp.a) * third : 0.0) + (xa > 0 ? (k0b_w + k0.a + kp.a) * third : 0.0));
    if (xb >= 0 && xb <= m)
      N.b = -0.5 * ((xb < m ? (k0.b + kpa_e + kp.b) * third : 0.0) + (xb > 0 ? (k0.a + k0.b + kp.b) * third : 0.0));
  }
}

template <bool INT>
__device__ __forceinline__ Sten mk_sten(double E, double W, double N, double S, int x, int y, int m, int bc) {
  Sten st;
  if (INT) {  // interior node with interior neighbours: no Dirichlet elimination
    st.d = -(E + W + N + S);
    st.e = E;
    st.w = W;
    st.n = N;
    st.s = S;
    return st;
  }
  if (x < 0 || x > m || y < 0 || y > m || is_dir(bc, m, x, y)) {
    st.d = 1.0;
    st.e = st.w = st.n = st.s = 0.0;
    return st;
  }
  st.d = -(E + W + N + S);
  st.e = is_dir(bc, m, x + 1, y) ? 0.0 : E;
  st.w = is_dir(bc, m, x - 1, y) ? 0.0 : W;
  st.n = is_dir(bc, m, x, y + 1) ? 0.0 : N;
  st.s = is_dir(bc, m, x, y - 1) ? 0.0 : S;
  return st;
}

struct Sten2 {
  Sten a, b;
};

// 5-point rows at (xa, y) and (xb, y) from this row's E, N and the previous row's N.
template <bool INT>
__device__ __forceinline__ Sten2 sten_pair(Pair E, Pair N, Pair Nm, int xa, int y, int m, int bc) {
  const double Wa = shup(E.b);  // E(xa−1) lives in the previous lane's b column
  return Sten2{mk_sten<INT>(E.a, Wa, N.a, Nm.a, xa, y, m, bc), mk_sten<INT>(E.b, E.a, N.b, Nm.b, xa + 1, y, m, bc)};
}

// Off-diagonal part Σ A(x,nb) v(nb) at both columns of row y from v rows y−1, y, y+1.
__device__ __forceinline__ Pair offd_pair(const Sten2& st, Pair vm, Pair v0, Pair vp) {
  const double va_e = shdn(v0.a), vb_w = shup(v0.b);
  return Pair{st.a.e * v0.b + st.a.w * vb_w + st.a.n * vp.a + st.a.s * vm.a,
              st.b.e * va_e + st.b.w * v0.a + st.b.n * vp.b + st.b.s * vm.b};
}

// Raw edge weights (E, N) of consecutive rows r0, r0+1, … of one warp strip, with one row of loads
// in flight. EN = false (level 0) rebuilds them from nodal k (three k rows in registers); EN = true
// (levels ≥ 1) loads the stored E/N rows of the coarse operator. Every kernel uses only N of the
// first row, so the k row below it is never loaded.
template <bool INT, bool EN>
struct EdgeRows;

template <bool INT>
struct EdgeRows<INT, false> {
  const double* kb;
  int xa, n0, m, r;
  Pair k0, k1, kq;
  __device__ __forceinline__ EdgeRows(const double* k, const double*, int xa_, int n0_, int m_, int r0)
      : kb(k), xa(xa_), n0(n0_), m(m_), r(r0) {
    k0 = Pair{0.0, 0.0};
    k1 = ld2<INT>(kb, xa, r0, n0);
    kq = ld2<INT>(kb, xa, r0 + 1, n0);
  }
  __device__ __forceinline__ void next(Pair& E, Pair& N) {
    const Pair kp = kq;
    kq = ld2<INT>(kb, xa, r + 2, n0);
    edges_pair<INT>(k0, k1, kp, xa, r, m, E, N);
    k0 = k1;
    k1 = kp;
    ++r;
  }
};

template <bool INT>
struct EdgeRows<INT, true> {
  const double *Eb, *Nb;
  int xa, n0, r;
  Pair eq, nq;
  __device__ __forceinline__ EdgeRows(const double* E, const double* N, int xa_, int n0_, int, int r0)
      : Eb(E), Nb(N), xa(xa_), n0(n0_), r(r0) {
    eq = ld2<INT>(Eb, xa, r0, n0);
    nq = ld2<INT>(Nb, xa, r0, n0);
  }
  __device__ __forceinline__ void next(Pair& E, Pair& N) {
    E = eq;
    N = nq;
    eq = ld2<INT>(Eb, xa, r + 1, n0);
    nq = ld2<INT>(Nb, xa, r + 1, n0);
    ++r;
  }
};

struct PairCtx {
  int b, lane, m, n0, xa, xb, y0, y1;
  bool outa, outb;
  int64_t off;
};

// Per-warp context; `interior` = every node this warp-chunk touches (rows y0−2 … y1+2, columns
// xa(lane 0)−1 … xb(lane 31)+1) is an in-grid non-Dirichlet node with in-grid neighbours, so the
// warp can run the branch-free body.
#define PAIR_PROLOGUE                                                                   \
  const int b = blockIdx.z;                                                             \
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;                                          \
  PairCtx c;                                                                            \
  {                                                                                     \
    const int lane = threadIdx.x & 31;                                                  \
    const int strip = blockIdx.x * MW + (threadIdx.x >> 5);                             \
    const int ly = rows_per_warp(g.m);                                                  \
    c.b = b;                                                                            \
    c.lane = lane;                                                                      \
    c.m = g.m;                                                                          \
    c.n0 = g.n0;                                                                        \
    c.xa = strip * 60 - 2 + 2 * lane;                                                   \
    c.xb = c.xa + 1;                                                                    \
    c.outa = lane >= 1 && lane < 31 && c.xa <= g.m;                                     \
    c.outb = lane >= 1 && lane < 31 && c.xb <= g.m;                                     \
    c.y0 = blockIdx.y * ly;                                                             \
    c.y1 = min(c.y0 + ly, g.n0);                                                        \
    c.off = (int64_t)b * g.N;                                                           \
  }                                                                                     \
  const int strip0 = blockIdx.x * MW + (threadIdx.x >> 5);                              \
  const bool interior = strip0 * 60 - 2 >= 2 && strip0 * 60 + 61 <= g.m - 2 &&          \
                        c.y0 >= 3 && c.y1 <= g.m - 2;

#define PAIR_UNPACK                                                                     \
  const int b = c.b, m = c.m, n0 = c.n0, xa = c.xa, xb = c.xb, y0 = c.y0, y1 = c.y1;    \
  const bool outa = c.outa, outb = c.outb;                                              \
  const int64_t off = c.off;                                                            \
  (void)b; (void)xb; (void)outa; (void)outb;

// red column of row y: a (even xa) when y is even, b otherwise
#define RED_IS_A(y) (((y) & 1) == 0)

// ---- PCG: p = z + βp (p = z first), <p, A p> → α  (Ap itself is recomputed where needed) --------
template <bool INT>
__device__ __forceinline__ double pcg_apply_kernel_body(Geo g, int bc, const double* __restrict__ k,
                                                       const double* __restrict__ z,
                                                       const double* __restrict__ p_old,
                                                       double* __restrict__ p_new, double* scal,
                                                       int* flags, double2* partial, int maxp,
                                                       unsigned* counter, const PairCtx& c) {
  PAIR_UNPACK

  const bool first = flags[b * F_NFLAGS + F_FIRST] != 0;
  const double beta = scal[b * S_NSCAL + S_BETA];
  const double *kb = k + off, *zb = z + off, *pb = p_old + off;
  auto comb = [&](Pair zz, Pair oo) {
    return first ? zz : Pair{fma(beta, oo.a, zz.a), fma(beta, oo.b, zz.b)};
  };
  const Pair zero{0.0, 0.0};
  Pair km = ld2<INT>(kb, xa, y0 - 1, n0), k0 = ld2<INT>(kb, xa, y0, n0);
  Pair pm = comb(ld2<INT>(zb, xa, y0 - 1, n0), first ? zero : ld2<INT>(pb, xa, y0 - 1, n0));
  Pair p0 = comb(ld2<INT>(zb, xa, y0, n0), first ? zero : ld2<INT>(pb, xa, y0, n0));
  Pair Nm, Ed;
  edges_pair<INT>(zero, km, k0, xa, y0 - 1, m, Ed, Nm);
  Pair kq = ld2<INT>(kb, xa, y0 + 1, n0), zq = ld2<INT>(zb, xa, y0 + 1, n0);
  Pair oq = first ? zero : ld2<INT>(pb, xa, y0 + 1, n0);
  double pap = 0.0;
  for (int y = y0; y < y1; ++y) {
    const Pair kp = kq, pp = comb(zq, oq);  // row y+1 (raw rows loaded one iteration ahead)
    kq = ld2<INT>(kb, xa, y + 2, n0);
    zq = ld2<INT>(zb, xa, y + 2, n0);
    if (!first) oq = ld2<INT>(pb, xa, y + 2, n0);
    Pair E, N;
    edges_pair<INT>(km, k0, kp, xa, y, m, E, N);
    const Sten2 st = sten_pair<INT>(E, N, Nm, xa, y, m, bc);
    const Pair od = offd_pair(st, pm, p0, pp);
    double* out = p_new + off + (int64_t)y * n0;
    if (outa) {
      out[xa] = p0.a;
      pap = fma(p0.a, fma(st.a.d, p0.a, od.a), pap);
    }
    if (outb) {
      out[xb] = p0.b;
      pap = fma(p0.b, fma(st.b.d, p0.b, od.b), pap);
    }
    km = k0; k0 = kp; pm = p0; p0 = pp; Nm = N;
  }
  return pap;
}

__global__ void __launch_bounds__(MT) pcg_apply_kernel(Geo g, int bc, const double* __restrict__ k,
                                                       const double* __restrict__ z,
                                                       const double* __restrict__ p_old,
                                                       double* __restrict__ p_new, double* scal,
                                                       int* flags, double2* partial, int maxp,
                                                       unsigned* counter) {
  PAIR_PROLOGUE
  const double pap = interior ? pcg_apply_kernel_body<true>(g, bc, k, z, p_old, p_new, scal, flags, partial, maxp, counter, c) : pcg_apply_kernel_body<false>(g, bc, k, z, p_old, p_new, scal, flags, partial, maxp, counter, c);
  double t0, t1;
  if (reduce2_last(pap, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    scal[b * S_NSCAL + S_ALPHA] = scal[b * S_NSCAL + S_RZ] / t0;
    flags[b * F_NFLAGS + F_FIRST] = 0;
  }
}

// ---- PCG update fused with the level-0 pre-smoother:
//   u += αp, r −= αAp (Ap recomputed from p), ‖r‖ → convergence,
//   then z_red = r/D, z_black = (r − Σ A z_red)/D  (red-black GS from z = 0)
template <bool INT>
__device__ __forceinline__ double pcg_update_down_kernel_body(
    Geo g, int bc, double tol, const double* __restrict__ k, const double* __restrict__ p,
    double* __restrict__ u, const double* __restrict__ r, double* __restrict__ r_out,
    double* __restrict__ z, double* scal, int* flags, double2* partial, int maxp, unsigned* counter,
    int* n_active, double* hist, int hist_cap, const PairCtx& c) {
  PAIR_UNPACK

  const double alpha = scal[b * S_NSCAL + S_ALPHA];
  const double *kb = k + off, *pb = p + off, *rb = r + off;
  const Pair zero{0.0, 0.0};
  // state for output row t: k/p rows t, t+1; N_t; r_new(t); z_red rows t−1, t; stencil(t)
  Pair ka = ld2<INT>(kb, xa, y0 - 2, n0), kb1 = ld2<INT>(kb, xa, y0 - 1, n0);
  Pair pa = ld2<INT>(pb, xa, y0 - 2, n0), pb1 = ld2<INT>(pb, xa, y0 - 1, n0);
  Pair Nt, Ed;
  edges_pair<INT>(zero, ka, kb1, xa, y0 - 2, m, Ed, Nt);
  Pair rn0 = zero;
  double zrm = 0.0, zr0 = 0.0;        // red z of rows t−1, t (the black entries are 0)
  Sten sb0{1.0, 0.0, 0.0, 0.0, 0.0};  // stencil of row t's black column (all the output needs)
  Pair kq = ld2<INT>(kb, xa, y0, n0), pq = ld2<INT>(pb, xa, y0, n0), rq = ld2<INT>(rb, xa, y0 - 1, n0);
  Pair uq = ld2<INT>(u + off, xa, y0 - 2, n0);
  double rr = 0.0;
#ifdef OSC_UD_UNROLL2
  // rows alternate parity: run them in (even, odd) pairs so the red/black roles are static
  auto step = [&](int t, auto ra) {
    constexpr bool ra0 = decltype(ra)::value, ra1 = !ra0;  // red column of row t is a
    const Pair kc = kq, pc = pq, r1 = rq, u0 = uq;  // rows t+2 / t+1 / t, loaded one iteration ahead
    kq = ld2<INT>(kb, xa, t + 3, n0);
    pq = ld2<INT>(pb, xa, t + 3, n0);
    rq = ld2<INT>(rb, xa, t + 2, n0);
    uq = ld2<INT>(u + off, xa, t + 1, n0);
    Pair E1, N1;
    edges_pair<INT>(ka, kb1, kc, xa, t + 1, m, E1, N1);
    const Sten2 st1 = sten_pair<INT>(E1, N1, Nt, xa, t + 1, m, bc);
    const Pair od1 = offd_pair(st1, pa, pb1, pc);
    const Pair rn1{fma(-alpha, fma(st1.a.d, pb1.a, od1.a), r1.a), fma(-alpha, fma(st1.b.d, pb1.b, od1.b), r1.b)};
    const double zrp = ra1 ? rn1.a * rcp64(st1.a.d) : rn1.b * rcp64(st1.b.d);
    const double zbl = ra0 ? (rn0.b - (sb0.e * shdn(zr0) + sb0.w * zr0 + sb0.n * zrp + sb0.s * zrm)) * rcp64(sb0.d)
                           : (rn0.a - (sb0.e * zr0 + sb0.w * shup(zr0) + sb0.n * zrp + sb0.s * zrm)) * rcp64(sb0.d);
    const Pair zv = ra0 ? Pair{zr0, zbl} : Pair{zbl, zr0};
    if (t >= y0) {
      const int64_t row = off + (int64_t)t * n0;
      if (outa) {
        u[row + xa] = fma(alpha, pa.a, u0.a);
        r_out[row + xa] = rn0.a;
        z[row + xa] = zv.a;
        rr = fma(rn0.a, rn0.a, rr);
      }
      if (outb) {
        u[row + xb] = fma(alpha, pa.b, u0.b);
        r_out[row + xb] = rn0.b;
        z[row + xb] = zv.b;
        rr = fma(rn0.b, rn0.b, rr);
      }
    }
    ka = kb1; kb1 = kc; pa = pb1; pb1 = pc; Nt = N1;
    rn0 = rn1; zrm = zr0; zr0 = zrp; sb0 = ra1 ? st1.b : st1.a;
  };
  for (int t = y0 - 2; t < y1; t += 2) {  // y0 is even
    step(t, std::true_type{});
    if (t + 1 < y1) step(t + 1, std::false_type{});
  }
#else
  for (int t = y0 - 2; t < y1; ++t) {
    const Pair kc = kq, pc = pq, r1 = rq, u0 = uq;  // rows t+2 / t+1 / t, loaded one iteration ahead
    kq = ld2<INT>(kb, xa, t + 3, n0);
    pq = ld2<INT>(pb, xa, t + 3, n0);
    rq = ld2<INT>(rb, xa, t + 2, n0);
    uq = ld2<INT>(u + off, xa, t + 1, n0);
    Pair E1, N1;
    edges_pair<INT>(ka, kb1, kc, xa, t + 1, m, E1, N1);
    const Sten2 st1 = sten_pair<INT>(E1, N1, Nt, xa, t + 1, m, bc);
    const Pair od1 = offd_pair(st1, pa, pb1, pc);
    const Pair rn1{fma(-alpha, fma(st1.a.d, pb1.a, od1.a), r1.a), fma(-alpha, fma(st1.b.d, pb1.b, od1.b), r1.b)};
    // z_red on row t+1
    const bool ra0 = RED_IS_A(t), ra1 = !ra0;
    const double zrp = (ra1 ? rn1.a : rn1.b) * rcp64(ra1 ? st1.a.d : st1.b.d);
    // output row t: black column = (r − Σ A z_red)/D, red column = z_red. Black at xb (ra0):
    // east = next lane's xa, west = own xa; black at xa: east = own xb, west = previous lane's xb
    const double zr0_e = shdn(zr0), zr0_w = shup(zr0);
    const double zbl = ((ra0 ? rn0.b : rn0.a) - (sb0.e * (ra0 ? zr0_e : zr0) + sb0.w * (ra0 ? zr0 : zr0_w) +
                                                 sb0.n * zrp + sb0.s * zrm)) * rcp64(sb0.d);
    const Pair zv = ra0 ? Pair{zr0, zbl} : Pair{zbl, zr0};
    if (t >= y0) {
      const int64_t row = off + (int64_t)t * n0;
      if (outa) {
        u[row + xa] = fma(alpha, pa.a, u0.a);
        r_out[row + xa] = rn0.a;
        z[row + xa] = zv.a;
        rr = fma(rn0.a, rn0.a, rr);
      }
      if (outb) {
        u[row + xb] = fma(alpha, pa.b, u0.b);
        r_out[row + xb] = rn0.b;
        z[row + xb] = zv.b;
        rr = fma(rn0.b, rn0.b, rr);
      }
    }
    ka = kb1; kb1 = kc; pa = pb1; pb1 = pc; Nt = N1;
    rn0 = rn1; zrm = zr0; zr0 = zrp; sb0 = ra1 ? st1.b : st1.a;
  }
#endif
  return rr;
}

#ifndef OSC_UD_MINB
#define OSC_UD_MINB 4
#endif
__global__ void __launch_bounds__(MT, OSC_UD_MINB) pcg_update_down_kernel(
    Geo g, int bc, double tol, const double* __restrict__ k, const double* __restrict__ p,
    double* __restrict__ u, const double* __restrict__ r, double* __restrict__ r_out,
    double* __restrict__ z, double* scal, int* flags, double2* partial, int maxp, unsigned* counter,
    int* n_active, double* hist, int hist_cap) {
  PAIR_PROLOGUE
#ifdef OSC_UD_INTERIOR
  const double rr = interior ? pcg_update_down_kernel_body<true>(g, bc, tol, k, p, u, r, r_out, z, scal, flags, partial, maxp, counter, n_active, hist, hist_cap, c)
                             : pcg_update_down_kernel_body<false>(g, bc, tol, k, p, u, r, r_out, z, scal, flags, partial, maxp, counter, n_active, hist, hist_cap, c);
#else
  // generic body only: the interior specialisation pushes this kernel past 128 registers (spills)
  (void)interior;
  const double rr = pcg_update_down_kernel_body<false>(g, bc, tol, k, p, u, r, r_out, z, scal, flags, partial, maxp, counter, n_active, hist, hist_cap, c);
#endif
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

// ---- residual restriction rc = Pᵀ(r − A z) after the red-black pre-smoother (fem.cpp:168-195).
// After the black sweep the residual vanishes on black nodes and equals −Σ A z_black on red
// nodes, so rc(I,J) = t(2I,2J) + ½[t(2I+1,2J+1) + t(2I−1,2J−1)]; zero at coarse Dirichlet nodes.
// Lane l owns fine columns xa = 2I, xb = 2I+1 of coarse column I (the column-pair layout of the
// marching kernels); lanes 0 and 31 are halo.
// −Σ A z_black at the red node of row y: column a (RA, y even) or b (y odd). E/N: row y's raw edges,
// Nm: row y−1's; zm/z0/zp: z rows y−1, y, y+1. All lanes must call it (shuffles).
template <bool INT, bool RA>
__device__ __forceinline__ double red_resid(Pair E, Pair N, Pair Nm, Pair zm, Pair z0, Pair zp, int xa, int y,
                                            int m, int bc) {
  const double Ew = shup(E.b);                      // E(xa−1)
  const double zw = RA ? shup(z0.b) : z0.a;         // z west of the red node
  const double ze = RA ? z0.b : shdn(z0.a);         // z east
  const double e0 = RA ? E.a : E.b, w0 = RA ? Ew : E.a, n0_ = RA ? N.a : N.b, s0 = RA ? Nm.a : Nm.b;
  const double zn = RA ? zp.a : zp.b, zs = RA ? zm.a : zm.b;
  if (INT) return -(e0 * ze + w0 * zw + n0_ * zn + s0 * zs);
  const int x = RA ? xa : xa + 1;
  if (x < 0 || x > m || y < 0 || y > m || is_dir(bc, m, x, y)) return 0.0;
  const double e = is_dir(bc, m, x + 1, y) ? 0.0 : e0, w = is_dir(bc, m, x - 1, y) ? 0.0 : w0;
  const double n = is_dir(bc, m, x, y + 1) ? 0.0 : n0_, sv = is_dir(bc, m, x, y - 1) ? 0.0 : s0;
  return -(e * ze + w * zw + n * zn + sv * zs);
}

template <bool INT, bool EN>
__device__ __forceinline__ void restrict_z_body(Geo g, Geo gc, int bc, const double* __restrict__ ca,
                                              const double* __restrict__ cb, const double* __restrict__ z,
                                              double* __restrict__ rc, int b, int I, bool outI, int J0, int J1) {
  const int m = g.m, n0 = g.n0, mc = gc.m;
  const int xa = 2 * I;
  const int64_t off = (int64_t)b * g.N;
  const double* zb = z + off;
  // fine rows y = 2J0−1 (odd: t at (xb, 2J0−1)), then pairs (2J, 2J+1) for J = J0 … J1−1;
  // state: z rows y−1, y (+ y+1 in flight), N of row y−1
  const int ys = 2 * J0 - 1;
  EdgeRows<INT, EN> er(ca + off, EN ? cb + off : nullptr, xa, n0, m, ys - 1);
  Pair E, N, Nm;
  er.next(E, Nm);
  Pair zm = ld2<INT>(zb, xa, ys - 1, n0), z0 = ld2<INT>(zb, xa, ys, n0);
  Pair zq = ld2<INT>(zb, xa, ys + 1, n0);
  double* rcb = rc + (int64_t)b * gc.N;
  auto advance = [&](int y, Pair& zp) {  // row y's edges and z row y+1; prefetch z row y+2
    zp = zq;
    zq = ld2<INT>(zb, xa, y + 2, n0);
    er.next(E, N);
  };
  Pair zp;
  advance(ys, zp);
  double t_prev = red_resid<INT, false>(E, N, Nm, zm, z0, zp, xa, ys, m, bc);  // (xb, 2J0−1)
  zm = z0; z0 = zp; Nm = N;
  for (int J = J0; J < J1; ++J) {
    const int y = 2 * J;
    advance(y, zp);
    const double t_even = red_resid<INT, true>(E, N, Nm, zm, z0, zp, xa, y, m, bc);  // (xa, 2J)
    zm = z0; z0 = zp; Nm = N;
    advance(y + 1, zp);
    const double t = red_resid<INT, false>(E, N, Nm, zm, z0, zp, xa, y + 1, m, bc);  // (xb, 2J+1)
    zm = z0; z0 = zp; Nm = N;
    const double t_w = shup(t_prev);  // t at (xa−1, 2J−1): previous lane's xb
    if (outI) rcb[(int64_t)J * gc.n0 + I] = is_dir(bc, mc, I, J) ? 0.0 : t_even + 0.5 * (t + t_w);
    t_prev = t;
  }
}

// ---- pre-smoother + residual restriction, fused (fem.cpp:288-295, 168-195) ----------------------------
// The pre-smoother is red-black GS from z = 0:
//   red sweep:   z_red = r/D;
//   black sweep: z_black = (r − Σ A z_red)/D.
// The residual r − A z then vanishes on black nodes and equals t = −Σ A z_black on red nodes, so
//   rc(I,J) = t(2I,2J) + ½[t(2I+1,2J+1) + t(2I−1,2J−1)]   (zero at coarse Dirichlet nodes).
// z is never stored. The post-smoother (smooth_up) recomputes z_red = r/D with the same operands,
// and its black sweep overwrites the black values. Fine rows are ingested one at a time: ingesting
// row y gives z_red(y), z_black(y−1) and t(y−2). Lane l owns fine columns xa = 2I, xb = 2I+1 of
// coarse column I (the column-pair layout); lanes 0 and 31 are halo.
template <bool INT, bool EN>
__device__ __forceinline__ void restrict_body(Geo g, Geo gc, int bc, const double* __restrict__ ca,
                                              const double* __restrict__ cb, const double* __restrict__ r,
                                              double* __restrict__ rc, int b, int I, bool outI, int J0, int J1) {
  const int m = g.m, n0 = g.n0, mc = gc.m;
  const int xa = 2 * I;
  const int64_t off = (int64_t)b * g.N;
  const double* rb = r + off;
  const int yf = 2 * J0 - 3;  // first ingested row (odd)
  EdgeRows<INT, EN> er(ca + off, EN ? cb + off : nullptr, xa, n0, m, yf - 1);
  Pair E, N, Nm;
  er.next(E, Nm);  // N of row yf−1
  Pair rq = ld2<INT>(rb, xa, yf, n0);
  const Sten unit{1.0, 0.0, 0.0, 0.0, 0.0};
  double zr_m = 0.0, zr_0 = 0.0;  // z_red of rows y−2, y−1 (y = the row being ingested)
  double rb_0 = 0.0;              // r at the black node of row y−1
  Sten sb_0 = unit;               // black stencil of row y−1
  double zb_m = 0.0, zb_0 = 0.0;  // z_black of rows y−3, y−2
  Sten sr_m = unit, sr_0 = unit;  // red stencils of rows y−2, y−1
  // RN: the red column of the ingested row y is a (y even). Returns t(y−2).
  auto ingest = [&](int y, auto ra) {
    constexpr bool RN = decltype(ra)::value;
    const Pair r1 = rq;
    rq = ld2<INT>(rb, xa, y + 1, n0);
    er.next(E, N);
    const Sten2 st = sten_pair<INT>(E, N, Nm, xa, y, m, bc);
    Nm = N;
    const Sten srn = RN ? st.a : st.b, sbn = RN ? st.b : st.a;
    // red sweep, row y
    const double zr_p = (RN ? r1.a : r1.b) * rcp64(srn.d);
    // black sweep, row y−1 (black column: a if RN). Black at a: east = own xb, west = previous
    // lane's xb; black at b: east = next lane's xa, west = own xa; north/south = red of rows y, y−2
    const double zr0_e = shdn(zr_0), zr0_w = shup(zr_0);
    const double zb_p = (rb_0 - (sb_0.e * (RN ? zr_0 : zr0_e) + sb_0.w * (RN ? zr0_w : zr_0) +
                                 sb_0.n * zr_p + sb_0.s * zr_m)) * rcp64(sb_0.d);
    // residual at the red node of row y−2 (red column: a if RN)
    const double zb0_e = shdn(zb_0), zb0_w = shup(zb_0);
    const double t = -(sr_m.e * (RN ? zb_0 : zb0_e) + sr_m.w * (RN ? zb0_w : zb_0) + sr_m.n * zb_p +
                       sr_m.s * zb_m);
    zr_m = zr_0; zr_0 = zr_p;
    rb_0 = RN ? r1.b : r1.a;
    sb_0 = sbn;
    zb_m = zb_0; zb_0 = zb_p;
    sr_m = sr_0; sr_0 = srn;
    return t;
  };
  using EVEN = std::true_type;
  using ODD = std::false_type;
  ingest(yf, ODD{});
  ingest(yf + 1, EVEN{});
  ingest(yf + 2, ODD{});
  ingest(yf + 3, EVEN{});
  double t_prev = ingest(yf + 4, ODD{});  // t(2J0−1)
  double* rcb = rc + (int64_t)b * gc.N;
  for (int J = J0; J < J1; ++J) {
    const double t_even = ingest(2 * J + 2, EVEN{});  // t(2J)   at (xa, 2J)
    const double t_odd = ingest(2 * J + 3, ODD{});    // t(2J+1) at (xb, 2J+1)
    const double t_w = shup(t_prev);                  // t(2J−1) at (xa−1): previous lane's xb
    if (outI) rcb[(int64_t)J * gc.n0 + I] = is_dir(bc, mc, I, J) ? 0.0 : t_even + 0.5 * (t_odd + t_w);
    t_prev = t_odd;
  }
}

// Level 0 (EN = false): restriction of the residual left by the pre-smoother that pcg_update_down
// fused (reads k, z). Coarse levels (EN = true): pre-smoother fused here (reads E, N, r; z never
// stored). Both give the same rc.
template <bool EN, bool ZIN>
__global__ void __launch_bounds__(MT) restrict_kernel(Geo g, Geo gc, int bc, const double* __restrict__ ca,
                                                      const double* __restrict__ cb,
                                                      const double* __restrict__ r,
                                                      const double* __restrict__ z,
                                                      double* __restrict__ rc, const int* flags) {
  const int b = blockIdx.z;
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;
  const int lane = threadIdx.x & 31;
  const int strip = blockIdx.x * MW + (threadIdx.x >> 5);
  const int I = strip * 30 - 1 + lane;
  const bool outI = lane >= 1 && lane < 31 && I <= gc.m;
  const int lyc = coarse_rows_per_warp(gc.m);
  const int J0 = blockIdx.y * lyc, J1 = min(J0 + lyc, gc.n0);
  // interior: fine rows 2J0−4 … 2J1+3 and columns xa(lane 0)−1 … xb(lane 31)+1 are in-grid,
  // non-Dirichlet nodes with in-grid neighbours
  const bool interior = strip * 60 - 2 >= 2 && strip * 60 + 61 <= g.m - 2 && 2 * J0 - 4 >= 2 &&
                        2 * J1 + 4 <= g.m - 1;
  if (!ZIN) {  // coarse levels, and level 0 of the first V-cycle (no fused pre-smoother ran yet)
    if (interior) restrict_body<true, EN>(g, gc, bc, ca, cb, r, rc, b, I, outI, J0, J1);
    else restrict_body<false, EN>(g, gc, bc, ca, cb, r, rc, b, I, outI, J0, J1);
  } else {
    if (interior) restrict_z_body<true, false>(g, gc, bc, ca, cb, z, rc, b, I, outI, J0, J1);
    else restrict_z_body<false, false>(g, gc, bc, ca, cb, z, rc, b, I, outI, J0, J1);
  }
}

// ---- prolongation + post-smoother, level 0: reads the pre-smoothed z written by pcg_update_down ---------
template <bool INT, bool EN>
__device__ __forceinline__ double smooth_up_z_body(Geo g, Geo gc, int bc,
                                                       const double* __restrict__ ca,
                                                       const double* __restrict__ cb,
                                                       const double* __restrict__ r,
                                                       const double* __restrict__ z,
                                                       double* __restrict__ z_out,
                                                       const double* __restrict__ zc, int finest,
                                                       double* scal, int* flags, double2* partial,
                                                       int maxp, unsigned* counter, const PairCtx& c) {
  PAIR_UNPACK

  const double *rb = r + off, *zbp = z + off, *zcb = zc + (int64_t)b * gc.N;
  const int nc0 = gc.n0;
  const Pair zero{0.0, 0.0};
  // Red node of row y after prolongation: z_red + P zc (fem.cpp:144-165). Row y even: red at xa
  // (even, even) → zc(xa/2, y/2). Row y odd: red at xb (odd, odd) → ½[zc(xa/2, (y−1)/2) +
  // zc(xa/2+1, (y+1)/2)]. Raw values are loaded one row ahead and combined when used.
  struct ZRaw {
    double z, c0, c1;
  };
  const int I = xa >> 1;
  // red value of row y after prolongation (the black column's entry is 0 until the black sweep)
  auto ZL = [&](int y) {
    ZRaw v{0.0, 0.0, 0.0};
    if (!INT && (unsigned)y >= (unsigned)n0) return v;
    if (RED_IS_A(y)) {
      if (INT || (unsigned)xa < (unsigned)n0) {
        v.z = __ldg(zbp + (int64_t)y * n0 + xa);
        v.c0 = __ldg(zcb + (int64_t)(y >> 1) * nc0 + I);
      }
    } else if (INT || (unsigned)xb < (unsigned)n0) {
      v.z = __ldg(zbp + (int64_t)y * n0 + xb);
      v.c0 = __ldg(zcb + (int64_t)(y >> 1) * nc0 + I);
      v.c1 = __ldg(zcb + (int64_t)((y + 1) >> 1) * nc0 + I + 1);
    }
    return v;
  };
  auto ZC = [&](const ZRaw& v, int y) { return RED_IS_A(y) ? v.z + v.c0 : v.z + 0.5 * (v.c0 + v.c1); };
  EdgeRows<INT, EN> er(ca + off, EN ? cb + off : nullptr, xa, n0, m, y0 - 2);
  // scalars: qa/qb/qc = red values of rows t, t+1, t+2; zbm/zb0 = black values of rows t−1, t
  double qa = ZC(ZL(y0 - 2), y0 - 2), qb = ZC(ZL(y0 - 1), y0 - 1);
  Pair Nt, Ed;
  er.next(Ed, Nt);
  Pair r0 = zero;
  double zbm = 0.0, zb0 = 0.0;
  Sten sr0{1.0, 0.0, 0.0, 0.0, 0.0};  // stencil of row t's red column
  Pair rq = ld2<INT>(rb, xa, y0 - 1, n0);
  ZRaw zq = ZL(y0);
  double rz = 0.0;
  for (int t = y0 - 2; t < y1; ++t) {
    const bool ra1 = RED_IS_A(t + 1);  // row t+1: red column a, black b (else the reverse)
    const Pair r1 = rq;
    const double qc = ZC(zq, t + 2);
    zq = ZL(t + 3);
    rq = ld2<INT>(rb, xa, t + 2, n0);
    Pair E1, N1;
    er.next(E1, N1);
    const Sten2 st1 = sten_pair<INT>(E1, N1, Nt, xa, t + 1, m, bc);
    // black node of row t+1: (r − Σ A z_red_prolonged)/D; its x-neighbours are row t+1's red
    // nodes (own column and the next/previous lane's)
    const double qb_e = shdn(qb), qb_w = shup(qb);
    const Sten sb = ra1 ? st1.b : st1.a;
    const double odb = sb.e * (ra1 ? qb_e : qb) + sb.w * (ra1 ? qb : qb_w) + sb.n * qc + sb.s * qa;
    const double zbp1 = ((ra1 ? r1.b : r1.a) - odb) * rcp64(sb.d);
    // output row t: red column = (r − Σ A z_black)/D, black column = z_black
    const double zb0_e = shdn(zb0), zb0_w = shup(zb0);
    const bool ra0 = !ra1;
    const double zred = ((ra0 ? r0.a : r0.b) - (sr0.e * (ra0 ? zb0 : zb0_e) + sr0.w * (ra0 ? zb0_w : zb0) +
                                                 sr0.n * zbp1 + sr0.s * zbm)) * rcp64(sr0.d);
    const Pair zv = ra0 ? Pair{zred, zb0} : Pair{zb0, zred};
    if (t >= y0) {
      double* out = z_out + off + (int64_t)t * n0;
      if (outa) {
        out[xa] = zv.a;
        rz = fma(r0.a, zv.a, rz);
      }
      if (outb) {
        out[xb] = zv.b;
        rz = fma(r0.b, zv.b, rz);
      }
    }
    qa = qb; qb = qc; Nt = N1;
    r0 = r1; zbm = zb0; zb0 = zbp1; sr0 = ra1 ? st1.a : st1.b;
  }
  return rz;
}

// ---- prolongation + post-smoother (black then red); on level 0 also <r, z> → β -------------------
// The pre-smoothed red values are recomputed as z_red = r/D (restrict_body's red sweep, same
// operands), so the only field reads are the coefficients, r and the coarse correction zc.
template <bool INT, bool EN>
__device__ __forceinline__ double smooth_up_kernel_body(Geo g, Geo gc, int bc,
                                                       const double* __restrict__ ca,
                                                       const double* __restrict__ cb,
                                                       const double* __restrict__ r,
                                                       double* __restrict__ z_out,
                                                       const double* __restrict__ zc, const PairCtx& c) {
  PAIR_UNPACK

  const double *rb = r + off, *zcb = zc + (int64_t)b * gc.N;
  const int nc0 = gc.n0;
  const Pair zero{0.0, 0.0};
  const int I = xa >> 1;
  // coarse correction at the red node of row y (fem.cpp:144-165): row y even → red at xa (even,
  // even): zc(I, y/2); row y odd → red at xb (odd, odd): ½[zc(I, (y−1)/2) + zc(I+1, (y+1)/2)].
  // Raw values are loaded ahead and combined when used.
  struct CRaw {
    double c0, c1;
  };
  auto CL = [&](int y) {
    CRaw v{0.0, 0.0};
    if ((unsigned)y >= (unsigned)n0) return v;
    if (RED_IS_A(y)) {
      if (INT || (unsigned)xa < (unsigned)n0) v.c0 = __ldg(zcb + (int64_t)(y >> 1) * nc0 + I);
    } else if (INT || (unsigned)xb < (unsigned)n0) {
      v.c0 = __ldg(zcb + (int64_t)(y >> 1) * nc0 + I);
      v.c1 = __ldg(zcb + (int64_t)((y + 1) >> 1) * nc0 + I + 1);
    }
    return v;
  };
  // red value of row y after the pre-smoother and the coarse correction: r/D + P zc, with D the
  // raw diagonal of the red node from row y's edges and row y−1's N
  auto qred = [&](Pair E, Pair N, Pair Nm, Pair rr, const CRaw& cv, int y) {
    const double Wa = shup(E.b);
    const double d = RED_IS_A(y) ? mk_sten<INT>(E.a, Wa, N.a, Nm.a, xa, y, m, bc).d
                                 : mk_sten<INT>(E.b, E.a, N.b, Nm.b, xb, y, m, bc).d;
    return RED_IS_A(y) ? rr.a * rcp64(d) + cv.c0 : rr.b * rcp64(d) + 0.5 * (cv.c0 + cv.c1);
  };
  EdgeRows<INT, EN> er(ca + off, EN ? cb + off : nullptr, xa, n0, m, y0 - 3);
  Pair N0, E1, N1, Ed;
  er.next(Ed, N0);  // N of row y0−3
  er.next(E1, N1);  // row y0−2
  const Pair r_a = ld2<INT>(rb, xa, y0 - 2, n0), r_b = ld2<INT>(rb, xa, y0 - 1, n0);
  double qa = qred(E1, N1, N0, r_a, CL(y0 - 2), y0 - 2);
  N0 = N1;
  er.next(E1, N1);  // row y0−1
  double qb = qred(E1, N1, N0, r_b, CL(y0 - 1), y0 - 1);
  // scalars: qa/qb/qc = red values of rows t, t+1, t+2; zbm/zb0 = black values of rows t−1, t
  Pair r0 = zero, r1 = r_b;
  double zbm = 0.0, zb0 = 0.0;
  Sten sr0{1.0, 0.0, 0.0, 0.0, 0.0};  // stencil of row t's red column
  Pair rq = ld2<INT>(rb, xa, y0, n0);
  CRaw cq = CL(y0);
  double rz = 0.0;
  for (int t = y0 - 2; t < y1; ++t) {
    const bool ra1 = RED_IS_A(t + 1);  // row t+1: red column a, black b (else the reverse)
    const Pair r2 = rq;
    const CRaw c2 = cq;
    rq = ld2<INT>(rb, xa, t + 3, n0);
    cq = CL(t + 3);
    Pair E2, N2;
    er.next(E2, N2);
    const double qc = qred(E2, N2, N1, r2, c2, t + 2);
    const Sten2 st1 = sten_pair<INT>(E1, N1, N0, xa, t + 1, m, bc);
    // black node of row t+1: (r − Σ A z_red_prolonged)/D; its x-neighbours are row t+1's red
    // nodes (own column and the next/previous lane's)
    const double qb_e = shdn(qb), qb_w = shup(qb);
    const Sten sb = ra1 ? st1.b : st1.a;
    const double odb = sb.e * (ra1 ? qb_e : qb) + sb.w * (ra1 ? qb : qb_w) + sb.n * qc + sb.s * qa;
    const double zbp1 = ((ra1 ? r1.b : r1.a) - odb) * rcp64(sb.d);
    // output row t: red column = (r − Σ A z_black)/D, black column = z_black
    const double zb0_e = shdn(zb0), zb0_w = shup(zb0);
    const bool ra0 = !ra1;
    const double zred = ((ra0 ? r0.a : r0.b) - (sr0.e * (ra0 ? zb0 : zb0_e) + sr0.w * (ra0 ? zb0_w : zb0) +
                                                 sr0.n * zbp1 + sr0.s * zbm)) * rcp64(sr0.d);
    const Pair zv = ra0 ? Pair{zred, zb0} : Pair{zb0, zred};
    if (t >= y0) {
      double* out = z_out + off + (int64_t)t * n0;
      if (outa) {
        out[xa] = zv.a;
        rz = fma(r0.a, zv.a, rz);
      }
      if (outb) {
        out[xb] = zv.b;
        rz = fma(r0.b, zv.b, rz);
      }
    }
    qa = qb; qb = qc;
    N0 = N1; E1 = E2; N1 = N2;
    r0 = r1; r1 = r2;
    zbm = zb0; zb0 = zbp1; sr0 = ra1 ? st1.a : st1.b;
  }
  return rz;
}

// EN = false: level 0 (a = nodal k, z = pre-smoothed z), also <r, z> → β; EN = true: levels ≥ 1
// (a = E, b = N; z_red recomputed from r)
template <bool EN, bool ZIN>
__global__ void __launch_bounds__(MT, 4) smooth_up_kernel(Geo g, Geo gc, int bc,
                                                       const double* __restrict__ a,
                                                       const double* __restrict__ bN,
                                                       const double* __restrict__ r,
                                                       const double* __restrict__ z,
                                                       double* __restrict__ z_out,
                                                       const double* __restrict__ zc,
                                                       double* scal, int* flags, double2* partial,
                                                       int maxp, unsigned* counter) {
  PAIR_PROLOGUE
  double rz;
  if (!ZIN)
    rz = interior ? smooth_up_kernel_body<true, EN>(g, gc, bc, a, bN, r, z_out, zc, c)
                  : smooth_up_kernel_body<false, EN>(g, gc, bc, a, bN, r, z_out, zc, c);
  else
    rz = interior ? smooth_up_z_body<true, false>(g, gc, bc, a, bN, r, z, z_out, zc, 1, scal, flags, partial, maxp, counter, c)
                  : smooth_up_z_body<false, false>(g, gc, bc, a, bN, r, z, z_out, zc, 1, scal, flags, partial, maxp, counter, c);
  if (EN) return;
  double t0, t1;
  if (reduce2_last(rz, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    const double old = scal[b * S_NSCAL + S_RZ];
    scal[b * S_NSCAL + S_BETA] = flags[b * F_NFLAGS + F_ITERS] == 0 ? 0.0 : t0 / old;
    scal[b * S_NSCAL + S_RZ] = t0;
  }
}

// ---- CTA-resident solver for small grids (m ≤ 64) ----------------------------------------------------
// One CTA owns one sample's whole solve: the edge weights E/N of every MG level, r, z (and p on
// level 0) live in shared memory (≤ 221 KB at m = 64), u stays in global memory, and the entire
// PCG loop (same algorithm and stopping rule as the multi-kernel path) runs inside one launch —
// no per-iteration launches, host polling or grid-wide reductions for the latency-bound levels
// that dominate MLMC's coarse levels (BASELINE configs 1, 3, 5).
constexpr int SM_THREADS = 1024;

struct SLev {
  double *E, *N, *r, *z;
  int m, n0, N_;
};

__device__ __forceinline__ Sten sten_smem(const SLev& L, int x, int y, int bc) {
  const int m = L.m, n0 = L.n0, c = y * n0 + x;
  Sten st;
  if (is_dir(bc, m, x, y)) {
    st.d = 1.0;
    st.e = st.w = st.n = st.s = 0.0;
    return st;
  }
  const double e = L.E[c], w = x > 0 ? L.E[c - 1] : 0.0, n = L.N[c], s = y > 0 ? L.N[c - n0] : 0.0;
  st.d = -(e + w + n + s);
  st.e = is_dir(bc, m, x + 1, y) ? 0.0 : e;
  st.w = is_dir(bc, m, x - 1, y) ? 0.0 : w;
  st.n = is_dir(bc, m, x, y + 1) ? 0.0 : n;
  st.s = is_dir(bc, m, x, y - 1) ? 0.0 : s;
  return st;
}

__device__ __forceinline__ double offd_smem(const Sten& st, const double* v, int c, int n0) {
  double a = 0.0;
  if (st.e != 0.0) a += st.e * v[c + 1];
  if (st.w != 0.0) a += st.w * v[c - 1];
  if (st.n != 0.0) a += st.n * v[c + n0];
  if (st.s != 0.0) a += st.s * v[c - n0];
  return a;
}

// red (color 0) or black (color 1) Gauss–Seidel half sweep: z = (r − Σ A z)/D on that color
__device__ __forceinline__ void gs_color(const SLev& L, int color, int bc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int y = warp; y < L.n0; y += nw) {
    for (int x = 2 * lane + ((y + color) & 1); x < L.n0; x += 64) {
      const int i = y * L.n0 + x;
      const Sten st = sten_smem(L, x, y, bc);
      L.z[i] = (L.r[i] - offd_smem(st, L.z, i, L.n0)) * rcp64(st.d);
    }
  }
}

// V(1,1) on levels l..L−1, input L[l].r, output L[l].z (same algorithm as the multi-kernel path)
__device__ void vcycle_smem(SLev* lev, int nlev, const double* Ainv, int bc) {
  for (int l = 0; l + 1 < nlev; ++l) {
    const SLev& F = lev[l];
    for (int i = threadIdx.x; i < F.N_; i += blockDim.x) F.z[i] = 0.0;
    __syncthreads();
    gs_color(F, 0, bc);
    __syncthreads();
    gs_color(F, 1, bc);
    __syncthreads();
    // rc = Pᵀ(r − A z): the residual vanishes on black nodes, is −Σ A z_black on red nodes
    const SLev& C = lev[l + 1];
    for (int ic = threadIdx.x; ic < C.N_; ic += blockDim.x) {
      const int J = ic / C.n0, I = ic - J * C.n0;
      double acc = 0.0;
      if (!is_dir(bc, C.m, I, J)) {
        auto t_at = [&](int fx, int fy) {
          if (fx < 0 || fx > F.m || fy < 0 || fy > F.m) return 0.0;
          const Sten st = sten_smem(F, fx, fy, bc);
          return -offd_smem(st, F.z, fy * F.n0 + fx, F.n0);
        };
        acc = t_at(2 * I, 2 * J) + 0.5 * (t_at(2 * I + 1, 2 * J + 1) + t_at(2 * I - 1, 2 * J - 1));
      }
      C.r[ic] = acc;
    }
    __syncthreads();
  }
  {  // coarsest: z = A⁻¹ r
    const SLev& C = lev[nlev - 1];
    for (int i = threadIdx.x; i < C.N_; i += blockDim.x) {
      double v = 0.0;
      for (int j = 0; j < C.N_; ++j) v = fma(Ainv[i * C.N_ + j], C.r[j], v);
      C.z[i] = v;
    }
    __syncthreads();
  }
  for (int l = nlev - 2; l >= 0; --l) {
    const SLev& F = lev[l];
    const SLev& C = lev[l + 1];
    // prolongation onto the red nodes (black values are overwritten by the black sweep)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int y = warp; y < F.n0; y += nw)
      for (int x = 2 * lane + (y & 1); x < F.n0; x += 64) {
      const int i = y * F.n0 + x;
      const double pz = (x & 1) == 0 ? C.z[(y >> 1) * C.n0 + (x >> 1)]
                                     : 0.5 * (C.z[(y >> 1) * C.n0 + (x >> 1)] + C.z[((y + 1) >> 1) * C.n0 + ((x + 1) >> 1)]);
      F.z[i] += pz;
    }
    __syncthreads();
    gs_color(F, 1, bc);
    __syncthreads();
    gs_color(F, 0, bc);
    __syncthreads();
  }
}

__device__ __forceinline__ double block_sum_s(double v) {
  __shared__ double sh[32];
  const double t = block_sum(v, sh);
  __shared__ double res;
  if (threadIdx.x == 0) res = t;
  __syncthreads();
  return res;
}

size_t small_smem_bytes(int m, int* nlev_out) {
  size_t tot = 0;
  int g = m, nl = 0, nc = 0;
  for (;;) {
    const size_t N = (size_t)(g + 1) * (g + 1);
    tot += N * (nl == 0 ? 5 : 4) * sizeof(double);
    ++nl;
    if (g <= 4 || g % 2 != 0) { nc = (int)N; break; }
    g /= 2;
  }
  if (nlev_out) *nlev_out = nl;
  return tot + (size_t)nc * nc * sizeof(double) + 64 * sizeof(SLev) + 256;
}

// Edge weights E/N of every level of a CTA-resident hierarchy. Level 0 comes from nodal k (global).
// Level l ≥ 1 comes from its triangle conductivities, built in that level's r (lower) / z (upper)
// buffers (free until the V-cycle runs):
//  * REDISCRETIZE: vertex means of the injected k;
//  * GALERKIN: means of the 4 fine triangles (from k for level 1, from level l−1's r/z after that).
// Same formulas as coarsen_tri_kernel / edges_kernel.
__device__ void smem_hierarchy(SLev* lev, int nlev, int coarse_op, const double* __restrict__ k0, int m0) {
  constexpr double third = 1.0 / 3.0;
  const int n00 = m0 + 1;
  auto K = [&](int x, int y, int st) { return __ldg(k0 + (int64_t)(y * st) * n00 + x * st); };
  for (int l = 1; l < nlev; ++l) {
    const SLev L = lev[l];
    const int mc = L.m;
    for (int ic = threadIdx.x; ic < mc * mc; ic += blockDim.x) {
      const int J = ic / mc, I = ic - J * mc;
      double lo, up;
      if (coarse_op == OSC_COARSE_REDISCRETIZE) {
        const int st = 1 << l;
        lo = (K(I, J, st) + K(I + 1, J, st) + K(I + 1, J + 1, st)) * third;
        up = (K(I, J, st) + K(I + 1, J + 1, st) + K(I, J + 1, st)) * third;
      } else {
        double fl[4], fu[4];
        for (int c = 0; c < 4; ++c) {
          const int i = 2 * I + (c & 1), j = 2 * J + (c >> 1);
          if (l == 1) {
            fl[c] = (K(i, j, 1) + K(i + 1, j, 1) + K(i + 1, j + 1, 1)) * third;
            fu[c] = (K(i, j, 1) + K(i + 1, j + 1, 1) + K(i, j + 1, 1)) * third;
          } else {
            fl[c] = lev[l - 1].r[j * lev[l - 1].n0 + i];
            fu[c] = lev[l - 1].z[j * lev[l - 1].n0 + i];
          }
        }
        lo = 0.25 * (fl[0] + fl[1] + fu[1] + fl[3]);
        up = 0.25 * (fu[0] + fl[2] + fu[2] + fu[3]);
      }
      L.r[J * L.n0 + I] = lo;
      L.z[J * L.n0 + I] = up;
    }
    __syncthreads();
  }
  for (int l = 0; l < nlev; ++l) {
    const SLev L = lev[l];
    const int m = L.m;
    for (int i = threadIdx.x; i < L.N_; i += blockDim.x) {
      const int y = i / L.n0, x = i - y * L.n0;
      double e = 0.0, n = 0.0;
      if (l == 0) {
        if (x < m) {
          const double lo = y < m ? (K(x, y, 1) + K(x + 1, y, 1) + K(x + 1, y + 1, 1)) * third : 0.0;
          const double up = y > 0 ? (K(x, y - 1, 1) + K(x + 1, y, 1) + K(x, y, 1)) * third : 0.0;
          e = -0.5 * (lo + up);
        }
        if (y < m) {
          const double up = x < m ? (K(x, y, 1) + K(x + 1, y + 1, 1) + K(x, y + 1, 1)) * third : 0.0;
          const double lo = x > 0 ? (K(x - 1, y, 1) + K(x, y, 1) + K(x, y + 1, 1)) * third : 0.0;
          n = -0.5 * (up + lo);
        }
      } else {
        if (x < m) e = -0.5 * ((y < m ? L.r[i] : 0.0) + (y > 0 ? L.z[i - L.n0] : 0.0));
        if (y < m) n = -0.5 * ((x < m ? L.z[i] : 0.0) + (x > 0 ? L.r[i - 1] : 0.0));
      }
      L.E[i] = e;
      L.N[i] = n;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(SM_THREADS) small_pcg_kernel(int m0, int nlev, int bc, int coarse_op, int forcing,
                                                               double fval, double tol, int max_iter_factor,
                                                               const double* __restrict__ kin,
                                                               double* __restrict__ uout, int* flags,
                                                               double* scal) {
  extern __shared__ double smem[];
  __shared__ SLev lev[12];
  const int b = blockIdx.x;
  const int N0 = (m0 + 1) * (m0 + 1);
  const double* k0 = kin + (int64_t)b * N0;
  double* u = uout + (int64_t)b * N0;
  // carve shared memory
  double* p = smem;
  double* cur = smem + N0;
  {
    int g = m0;
    for (int l = 0; l < nlev; ++l) {
      const int n0 = g + 1, N = n0 * n0;
      if (threadIdx.x == 0) lev[l] = SLev{cur, cur + N, cur + 2 * N, cur + 3 * N, g, n0, N};
      cur += 4 * N;
      g /= 2;
    }
  }
  double* Ainv = cur;
  __syncthreads();
  // level-0 edge weights from nodal k (same formulas and operand order as the streaming kernels),
  // coarse levels from their triangle conductivities (coarsen_tri_kernel / edges_kernel semantics)
  smem_hierarchy(lev, nlev, coarse_op, k0, m0);
  {  // coarsest operator → in-place Gauss–Jordan inverse (SPD, no pivoting)
    const SLev C = lev[nlev - 1];
    const int n = C.N_;
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) Ainv[idx] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int y = i / C.n0, x = i - y * C.n0;
      const Sten st = sten_smem(C, x, y, bc);
      Ainv[i * n + i] = st.d;
      if (x + 1 < C.n0) Ainv[i * n + i + 1] = st.e;
      if (x > 0) Ainv[i * n + i - 1] = st.w;
      if (y + 1 < C.n0) Ainv[i * n + i + C.n0] = st.n;
      if (y > 0) Ainv[i * n + i - C.n0] = st.s;
    }
    __syncthreads();
    for (int kk = 0; kk < n; ++kk) {
      const double piv = 1.0 / Ainv[kk * n + kk];
      __syncthreads();
      // row kk scaled; column kk of other rows folded (in-place Gauss–Jordan)
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (i == kk) continue;
        const double f = Ainv[i * n + kk] * piv;
        for (int j = 0; j < n; ++j) {
          if (j == kk) continue;
          Ainv[i * n + j] = fma(-f, Ainv[kk * n + j], Ainv[i * n + j]);
        }
        Ainv[i * n + kk] = -f;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int j = 0; j < n; ++j) Ainv[kk * n + j] = (j == kk) ? piv : Ainv[kk * n + j] * piv;
      }
      __syncthreads();
    }
  }
  // PCG init (fem.cpp:335-365): u = lift, r = b − A u
  const SLev L0 = lev[0];
  const int m = m0;
  double bb = 0.0, rr0 = 0.0;
  for (int i = threadIdx.x; i < N0; i += blockDim.x) {
    const int y = i / L0.n0, x = i - y * L0.n0;
    const double gs = (bc == OSC_BC_FLOWCELL && x == 0) ? 1.0 : 0.0;
    double bi;
    if (is_dir(bc, m, x, y)) {
      bi = gs;
      u[i] = gs;
      L0.r[i] = 0.0;
    } else {
      const int tri = 2 * (x < m && y < m) + (x > 0 && y < m) + 2 * (x > 0 && y > 0) + (x < m && y > 0);
      const double h = 1.0 / m;
      bi = forcing ? tri * (fval * (0.5 * h * h) / 3.0) : 0.0;
      if (bc == OSC_BC_FLOWCELL && x == 1) bi -= L0.E[i - 1] * 1.0;  // raw coupling to u = 1 at x = 0
      u[i] = 0.0;
      L0.r[i] = bi;
      rr0 += bi * bi;
    }
    bb += bi * bi;
  }
  const double bnorm = sqrt(block_sum_s(bb));
  double rel = sqrt(block_sum_s(rr0)) / bnorm;
  int it = 0, status = 0;
  const int64_t cap64 = (int64_t)max_iter_factor * N0;
  const int cap = (int)(cap64 < 0x7fffffff ? cap64 : 0x7fffffff);
  if (rel > tol) {
    vcycle_smem(lev, nlev, Ainv, bc);
    double rz = 0.0;
    for (int i = threadIdx.x; i < N0; i += blockDim.x) {
      p[i] = L0.z[i];
      rz += L0.r[i] * L0.z[i];
    }
    rz = block_sum_s(rz);
    for (;;) {
      if (it >= cap) {
        status = OSC_ERR_SOLVER;
        break;
      }
      ++it;
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
      double pap = 0.0;
      for (int y = warp; y < L0.n0; y += nw)
        for (int x = lane; x < L0.n0; x += 32) {
          const int i = y * L0.n0 + x;
          const Sten st = sten_smem(L0, x, y, bc);
          pap += p[i] * (st.d * p[i] + offd_smem(st, p, i, L0.n0));
        }
      const double alpha = rz / block_sum_s(pap);
      double rr = 0.0;
      for (int y = warp; y < L0.n0; y += nw)
        for (int x = lane; x < L0.n0; x += 32) {
        const int i = y * L0.n0 + x;
        const Sten st = sten_smem(L0, x, y, bc);
        u[i] = fma(alpha, p[i], u[i]);
        const double rn = fma(-alpha, st.d * p[i] + offd_smem(st, p, i, L0.n0), L0.r[i]);
        L0.r[i] = rn;
        rr += rn * rn;
      }
      rel = sqrt(block_sum_s(rr)) / bnorm;
      if (rel <= tol) break;
      if (!isfinite(rel)) {
        status = OSC_ERR_SOLVER;
        break;
      }
      vcycle_smem(lev, nlev, Ainv, bc);
      double rzn = 0.0;
      for (int i = threadIdx.x; i < N0; i += blockDim.x) rzn += L0.r[i] * L0.z[i];
      rzn = block_sum_s(rzn);
      const double beta = rzn / rz;
      rz = rzn;
      for (int i = threadIdx.x; i < N0; i += blockDim.x) p[i] = fma(beta, p[i], L0.z[i]);
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    flags[b * F_NFLAGS + F_ACTIVE] = 0;
    flags[b * F_NFLAGS + F_ITERS] = it;
    flags[b * F_NFLAGS + F_STATUS] = status;
    scal[b * S_NSCAL + S_REL] = rel;
    scal[b * S_NSCAL + S_BNORM] = bnorm;
  }
}


// ---- CTA-resident tail of the V-cycle (levels with m ≤ 32) ---------------------------------------------
// On large solves the coarsest few levels are launch/latency-bound (≈ 20 µs per kernel whatever
// their size). One CTA per sample runs the whole sub-V-cycle from level ls down, in shared memory.
// It reads the stored edge weights of each level and the coarsest inverse from the setup.
constexpr int SUB_THREADS = 256;
struct SubLevels {
  const double* E[12];
  const double* N[12];
};
__global__ void __launch_bounds__(SUB_THREADS) sub_vcycle_kernel(int m_ls, int nlev, int bc, SubLevels sl,
                                                                 const double* __restrict__ r_ls,
                                                                 double* __restrict__ z_out,
                                                                 const double* __restrict__ chol,
                                                                 const int* flags) {
  extern __shared__ double smem[];
  __shared__ SLev lev[12];
  const int b = blockIdx.x;
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;
  const int N_ls = (m_ls + 1) * (m_ls + 1);
  double* cur = smem;
  {
    int g = m_ls;
    for (int l = 0; l < nlev; ++l) {
      const int n0 = g + 1, N = n0 * n0;
      if (threadIdx.x == 0) lev[l] = SLev{cur, cur + N, cur + 2 * N, cur + 3 * N, g, n0, N};
      cur += 4 * N;
      g /= 2;
    }
  }
  double* Ainv = cur;
  __syncthreads();
  for (int l = 0; l < nlev; ++l) {
    const SLev L = lev[l];
    const double* Eg = sl.E[l] + (int64_t)b * L.N_;
    const double* Ng = sl.N[l] + (int64_t)b * L.N_;
    for (int i = threadIdx.x; i < L.N_; i += blockDim.x) {
      L.E[i] = __ldg(Eg + i);
      L.N[i] = __ldg(Ng + i);
    }
  }
  {
    const int nc = lev[nlev - 1].N_;
    const double* X = chol + (int64_t)b * 2 * nc * nc + (int64_t)nc * nc;
    for (int i = threadIdx.x; i < nc * nc; i += blockDim.x) Ainv[i] = X[i];
  }
  const double* rb = r_ls + (int64_t)b * N_ls;
  for (int i = threadIdx.x; i < N_ls; i += blockDim.x) lev[0].r[i] = rb[i];
  __syncthreads();
  vcycle_smem(lev, nlev, Ainv, bc);
  double* zb = z_out + (int64_t)b * N_ls;
  for (int i = threadIdx.x; i < N_ls; i += blockDim.x) zb[i] = lev[0].z[i];
}

size_t sub_smem_bytes(int m_ls, int nlev) {
  size_t tot = 0;
  int g = m_ls, nc = 0;
  for (int l = 0; l < nlev; ++l) {
    const size_t N = (size_t)(g + 1) * (g + 1);
    tot += 4 * N * sizeof(double);
    nc = (int)N;
    g /= 2;
  }
  return tot + (size_t)nc * nc * sizeof(double);
}

__global__ void mark_active_failed_kernel(int B, int* flags) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B && flags[b * F_NFLAGS + F_ACTIVE]) {
    flags[b * F_NFLAGS + F_ACTIVE] = 0;
    flags[b * F_NFLAGS + F_STATUS] = OSC_ERR_SOLVER;
  }
}

// single-level case (no coarser grid): <r,z> → β
__global__ void __launch_bounds__(NT) dot_rz_kernel(Geo g, const double* __restrict__ r,
                                                    const double* __restrict__ z, double* scal,
                                                    int* flags, double2* partial, int maxp,
                                                    unsigned* counter) {
  const int b = blockIdx.z;
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;
  const int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x;
  const int64_t off = (int64_t)b * g.N;
  const double rz = i < g.N ? r[off + i] * z[off + i] : 0.0;
  double t0, t1;
  if (reduce2_last(rz, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    const double old = scal[b * S_NSCAL + S_RZ];
    scal[b * S_NSCAL + S_BETA] = flags[b * F_NFLAGS + F_ITERS] == 0 ? 0.0 : t0 / old;
    scal[b * S_NSCAL + S_RZ] = t0;
  }
}

// coarsest solve z = A⁻¹ r (the Cholesky solve of fem.cpp:274-286 via the precomputed inverse),
// one warp per sample: lane i forms row i of the matvec
__global__ void coarse_solve_kernel(int n, int B, const double* __restrict__ chol,
                                    const double* __restrict__ r, double* __restrict__ z,
                                    const int* flags) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B || !flags[b * F_NFLAGS + F_ACTIVE]) return;
  const double* X = chol + (int64_t)b * 2 * n * n + (int64_t)n * n;
  const double* rb = r + (int64_t)b * n;
  double* zb = z + (int64_t)b * n;
  for (int i = lane; i < n; i += 32) {
    double v = 0.0;
    for (int j = 0; j < n; ++j) v = fma(X[i * n + j], __ldg(rb + j), v);
    zb[i] = v;
  }
}

// ---- QoIs (fem.cpp:402-436 + extensions) -------------------------------------------------------------
__global__ void __launch_bounds__(NT) qoi_kernel(Geo g, int qoi, double qx, double qy, int forcing,
                                                 double fval, const double* __restrict__ u,
                                                 const double* __restrict__ k,
                                                 double* __restrict__ q, double2* partial, int maxp,
                                                 unsigned* counter) {
  const int b = blockIdx.z;
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
inline int march_strips(int m) { return (m + 1 + 59) / 60; }  // 60 written columns per warp strip
inline dim3 march_grid(int m, int /*hx*/, int B) {
  const int ly = rows_per_warp(m);
  return dim3((unsigned)((march_strips(m) + MW - 1) / MW), (unsigned)((m + 1 + ly - 1) / ly), (unsigned)B);
}
inline dim3 restrict_grid(int mc, int B) {
  const int lyc = coarse_rows_per_warp(mc);
  return dim3((unsigned)(((mc + 1 + 29) / 30 + MW - 1) / MW), (unsigned)((mc + 1 + lyc - 1) / lyc), (unsigned)B);
}
inline int64_t tile_parts(int m) {
  const dim3 a = march_grid(m, 1, 1), b = march_grid(m, 2, 1);
  return std::max<int64_t>((int64_t)a.x * a.y, (int64_t)b.x * b.y);
}

}  // namespace

size_t solver_bytes(int m, int B, int hist_cap) {
  size_t tot = 0;
  int g = m, lev = 0;
  for (;;) {
    const size_t N = (size_t)(g + 1) * (g + 1);
    // level 0: u r r2 z z2 p0 p1 (+k by caller); levels ≥ 1: E N r z z2
    tot += N * B * sizeof(double) * (lev == 0 ? 8 : 5);
    ++lev;
    if (g <= 4 || g % 2 != 0) {
      tot += 2 * N * N * B * sizeof(double);
      if (lev == 1) tot += 2 * N * B * sizeof(double);  // single level: E N of level 0 for the factor
      break;
    }
    g /= 2;
  }
  tot += (size_t)B * (S_NSCAL * 8 + F_NFLAGS * 4 + 8) + (size_t)B * hist_cap * 8;
  tot += (size_t)B * (tile_parts(m) + (size_t)(m + 1) * (m + 1) / NT + 2) * 16;
  return tot + 8192 * 16;
}

void solver_prepare(Ctx* ctx, int m, int B, int hist_cap) {
  SolverWork& w = ctx->solver;
  OSC_REQUIRE(m >= 1, "solve: m must be >= 1");
  OSC_REQUIRE(B >= 1 && B <= 65535, "solve: batch must be in [1, 65535]");
  w.m = m;
  w.B = B;
  w.hist_cap = hist_cap;
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
  w.max_parts = (int)std::max<int64_t>(tile_parts(m), nblocks(w.lev[0].N));
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
    L.k = nullptr;  // level 0's k is the caller's buffer; coarse levels keep edge weights instead
    L.D = nullptr;
    const bool edges = l > 0 || nl == 1;
    L.E = edges ? (double*)take(vb) : nullptr;
    L.Nw = edges ? (double*)take(vb) : nullptr;
    L.r = (double*)take(vb);
    L.z = (double*)take(vb);
    L.z2 = (double*)take(vb);
  }
  const size_t vb0 = sizeof(double) * w.lev[0].N * B;
  w.u = (double*)take(vb0);
  w.r2 = (double*)take(vb0);
  w.r_cur = w.lev[0].r;
  w.p0 = (double*)take(vb0);
  w.p1 = (double*)take(vb0);
  w.Ap = nullptr;
  w.chol = (double*)take(sizeof(double) * 2 * (size_t)w.nc * w.nc * B);
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

// kernel-class name of a coarse level: "<base>.Lc", or "<base>.L<l>" with OSC_LEVEL_STATS set
std::string lvl_name(const char* base, int l) {
  static const bool per_level = std::getenv("OSC_LEVEL_STATS") != nullptr;
  return std::string(base) + (per_level ? ".L" + std::to_string(l) : std::string(".Lc"));
}

// Preconditioner z = M r on level 0 (input w.r_cur, output lev[0].z2). z0_fresh: lev[0].z holds the
// level-0 pre-smoothed correction (written by pcg_update_down); otherwise the fused restriction
// runs the level-0 pre-smoother itself.
void vcycle(Ctx* ctx, int bc, int B, bool z0_fresh) {
  SolverWork& w = ctx->solver;
  cudaStream_t st = ctx->stream;
  double2* part = reinterpret_cast<double2*>(w.partial);
  if (w.nlev == 1) {
    {
      KScope ks(ctx, "mg_coarse_solve");
      coarse_solve_kernel<<<(B + 3) / 4, 128, 0, st>>>(w.nc, B, w.chol, w.r_cur, w.lev[0].z2, w.flags);
    }
    KScope ks(ctx, "pcg_dot_rz");
    dot_rz_kernel<<<dim3(nblocks(w.lev[0].N), 1, B), NT, 0, st>>>(geo_of(w.lev[0]), w.r_cur, w.lev[0].z2,
                                                                 w.scal, w.flags, part, w.max_parts, w.counter);
    OSC_CUDA(cudaGetLastError());
    return;
  }
  // first level handled by the CTA-resident tail (m ≤ 32, at least two levels below it)
  static const bool sub_off = std::getenv("OSC_NO_SUB_VCYCLE") != nullptr;
  int ls = w.nlev - 1;
  if (!sub_off)
    for (int l = 1; l < w.nlev - 1; ++l)
      if (w.lev[l].m <= 32) { ls = l; break; }
  // down: pre-smoother + restriction, one fused pass per level
  for (int l = 0; l + 1 < w.nlev && l < ls; ++l) {
    const SolverLevel& L = w.lev[l];
    const SolverLevel& C = w.lev[l + 1];
    KScope ks(ctx, l > 0 ? lvl_name("mg_restrict", l).c_str() : z0_fresh ? "mg_restrict.L0" : "mg_restrict.L0first");
    if (l == 0 && z0_fresh)
      restrict_kernel<false, true><<<restrict_grid(C.m, B), MT, 0, st>>>(geo_of(L), geo_of(C), bc, L.k, nullptr, w.r_cur,
                                                                         L.z, C.r, w.flags);
    else if (l == 0)
      restrict_kernel<false, false><<<restrict_grid(C.m, B), MT, 0, st>>>(geo_of(L), geo_of(C), bc, L.k, nullptr, w.r_cur,
                                                                          nullptr, C.r, w.flags);
    else
      restrict_kernel<true, false><<<restrict_grid(C.m, B), MT, 0, st>>>(geo_of(L), geo_of(C), bc, L.E, L.Nw, L.r, nullptr, C.r, w.flags);
  }
  if (ls < w.nlev - 1) {
    const SolverLevel& S = w.lev[ls];
    const int nl = w.nlev - ls;
    const size_t sm = sub_smem_bytes(S.m, nl);
    OSC_CUDA(cudaFuncSetAttribute(sub_vcycle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    SubLevels sl{};
    for (int l = 0; l < nl; ++l) {
      sl.E[l] = w.lev[ls + l].E;
      sl.N[l] = w.lev[ls + l].Nw;
    }
    KScope ks(ctx, "mg_sub_vcycle");
    sub_vcycle_kernel<<<B, SUB_THREADS, sm, st>>>(S.m, nl, bc, sl, S.r, S.z2, w.chol, w.flags);
  } else {
    const SolverLevel& C = w.lev[w.nlev - 1];
    KScope ks(ctx, "mg_coarse_solve");
    coarse_solve_kernel<<<(B + 3) / 4, 128, 0, st>>>(w.nc, B, w.chol, C.r, C.z2, w.flags);
  }
  // up: prolongation + post-smoother per level
  for (int l = ls - 1; l >= 0; --l) {
    const SolverLevel& L = w.lev[l];
    const SolverLevel& C = w.lev[l + 1];
    KScope ks(ctx, l > 0 ? lvl_name("mg_smooth_up", l).c_str() : z0_fresh ? "mg_smooth_up.L0" : "mg_smooth_up.L0first");
    if (l == 0 && z0_fresh)
      smooth_up_kernel<false, true><<<march_grid(L.m, 2, B), MT, 0, st>>>(geo_of(L), geo_of(C), bc, L.k, nullptr, w.r_cur,
                                                              L.z,
                                                              L.z2, C.z2, w.scal, w.flags, part, w.max_parts, w.counter);
    else if (l == 0)
      smooth_up_kernel<false, false><<<march_grid(L.m, 2, B), MT, 0, st>>>(geo_of(L), geo_of(C), bc, L.k, nullptr, w.r_cur,
                                                              nullptr,
                                                              L.z2, C.z2, w.scal, w.flags, part, w.max_parts, w.counter);
    else
      smooth_up_kernel<true, false><<<march_grid(L.m, 2, B), MT, 0, st>>>(geo_of(L), geo_of(C), bc, L.E, L.Nw, L.r, nullptr,
                                                             L.z2, C.z2, w.scal, w.flags, part, w.max_parts, w.counter);
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
  OSC_REQUIRE(prob->coarse_op == OSC_COARSE_GALERKIN || prob->coarse_op == OSC_COARSE_REDISCRETIZE,
              "solve: unknown coarse_op");
  struct TagGuard {
    Ctx* c;
    ~TagGuard() { c->tag.clear(); }
  } tg{ctx};
  ctx->tag = std::to_string(w.m);
  SolverLevel& L0 = w.lev[0];
  const Geo g0 = geo_of(L0);
  w.r_cur = L0.r;
  static const bool small_off = std::getenv("OSC_NO_SMALL_PCG") != nullptr;
  if (w.m <= 64 && w.hist_cap == 0 && !small_off) {
    // whole solve CTA-resident (one CTA per sample, one launch)
    int nl = 0;
    const size_t sm = small_smem_bytes(w.m, &nl);
    OSC_CUDA(cudaFuncSetAttribute(small_pcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    KScope ks(ctx, "small_pcg");
    small_pcg_kernel<<<B, SM_THREADS, sm, st>>>(w.m, nl, bc, prob->coarse_op, prob->forcing, prob->forcing_value, prob->tol,
                                               prob->max_iter_factor, L0.k, w.u, w.flags, w.scal);
    OSC_CUDA(cudaGetLastError());
    return;
  }
  {  // hierarchy: coarse operators (triangle conductivities → edge weights) + coarsest inverse
    KScope ks(ctx, "mg_setup", 2 * w.nlev);
    const int mode = prob->coarse_op;
    if (w.nlev == 1) {  // single level: level 0's own edges (vertex means of k) for the factor
      SolverLevel& L = w.lev[0];
      coarsen_tri_kernel<<<dim3(nblocks((int64_t)L.m * L.m), B), NT, 0, st>>>(
          OSC_COARSE_REDISCRETIZE, g0, g0, g0, 1, L0.k, nullptr, nullptr, L.z, L.z2);
      edges_kernel<<<dim3(nblocks(L.N), B), NT, 0, st>>>(g0, L.z, L.z2, L.E, L.Nw);
    }
    for (int l = 0; l + 1 < w.nlev; ++l) {
      const SolverLevel& F = w.lev[l];
      const SolverLevel& C = w.lev[l + 1];
      const bool from_k = mode == OSC_COARSE_REDISCRETIZE || l == 0;
      coarsen_tri_kernel<<<dim3(nblocks((int64_t)C.m * C.m), B), NT, 0, st>>>(
          mode, g0, geo_of(F), geo_of(C), 2 << l, L0.k, from_k ? nullptr : F.z, from_k ? nullptr : F.z2,
          C.z, C.z2);
      edges_kernel<<<dim3(nblocks(C.N), B), NT, 0, st>>>(geo_of(C), C.z, C.z2, C.E, C.Nw);
    }
    const SolverLevel& C = w.lev[w.nlev - 1];
    if (w.nc <= 32)
      coarse_factor_warp_kernel<<<(B + CF_WARPS - 1) / CF_WARPS, 32 * CF_WARPS, 0, st>>>(geo_of(C), bc, B, C.E, C.Nw, w.chol);
    else
      coarse_factor_kernel<<<(B + 63) / 64, 64, 0, st>>>(geo_of(C), bc, B, C.E, C.Nw, w.chol);
    OSC_CUDA(cudaGetLastError());
  }

  OSC_CUDA(cudaMemsetAsync(w.n_active, 0, sizeof(int), st));
  {
    KScope ks(ctx, "pcg_init");
    pcg_init_kernel<<<dim3(nblocks(L0.N), 1, B), NT, 0, st>>>(
        g0, bc, prob->forcing, prob->forcing_value, prob->tol, prob->max_iter_factor, L0.k, w.u, w.r_cur,
        w.scal, w.flags, part, w.max_parts, w.counter, w.n_active, w.hist, w.hist_cap);
  }
  vcycle(ctx, bc, B, false);  // z = M r0, rz = <r0, z>
  double* p_old = w.p0;
  double* p_new = w.p1;
  const int check_every = L0.N >= 65536 ? 1 : 4;
  // optional host-side safety valve (debugging): OSC_HARD_ITER_CAP stops the loop early; the
  // samples still active are reported as not converged by solver_results().
  static const long hard_cap = [] {
    const char* e = std::getenv("OSC_HARD_ITER_CAP");
    return e ? std::atol(e) : -1L;
  }();
  for (int it = 0;; ++it) {
    if (hard_cap >= 0 && it >= hard_cap) {
      mark_active_failed_kernel<<<(B + 255) / 256, 256, 0, st>>>(B, w.flags);
      break;
    }
    if (it % check_every == 0) {
      OSC_CUDA(cudaMemcpyAsync(ctx->h_pinned_int, w.n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
      OSC_CUDA(cudaStreamSynchronize(st));
      if (*ctx->h_pinned_int <= 0) break;
    }
    {
      KScope ks(ctx, "pcg_apply");
      pcg_apply_kernel<<<march_grid(L0.m, 1, B), MT, 0, st>>>(g0, bc, L0.k, L0.z2, p_old, p_new, w.scal, w.flags,
                                                        part, w.max_parts, w.counter);
    }
    {
      KScope ks(ctx, "pcg_update_down");
      double* r_next = (w.r_cur == L0.r) ? w.r2 : L0.r;
      pcg_update_down_kernel<<<march_grid(L0.m, 2, B), MT, 0, st>>>(g0, bc, prob->tol, L0.k, p_new, w.u, w.r_cur,
                                                              r_next, L0.z, w.scal, w.flags, part, w.max_parts,
                                                              w.counter, w.n_active, w.hist, w.hist_cap);
    }
    w.r_cur = (w.r_cur == L0.r) ? w.r2 : L0.r;
    vcycle(ctx, bc, B, true);  // level-0 pre-smoother ran inside pcg_update_down
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
  qoi_kernel<<<dim3(nblocks(items), 1, B), NT, 0, ctx->stream>>>(
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
