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
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

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

// 1/d to full double precision: MUFU approximation + two Newton steps (no DDIV sequence).
__device__ __forceinline__ double rcp64(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = fma(y, fma(-d, y, 1.0), y);
  y = fma(y, fma(-d, y, 1.0), y);
  return y;
}

// Reciprocal of the smoothing sweeps: one Newton step on the 2^-23 hardware estimate (relative error
// ≈ 2^-46). The sweeps divide by stencil diagonals inside the preconditioner, where 1e-14 is a
// perturbation of the smoother far below the fp32 couplings'; setup (transfer weights, Galerkin
// products) keeps rcp64.
__device__ __forceinline__ double rcp64s(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  return fma(y, fma(-d, y, 1.0), y);
}

// ---- multigrid hierarchy: rows, transfers, coarse operators -----------------------------------------
// Level 0 is the fine P1 system: a 5-point stencil rebuilt from nodal k in every kernel. Levels ≥ 1
// keep a symmetric 9-point operator in HBM, stored with Dirichlet elimination already applied
// (identity rows, zero couplings to Dirichlet nodes): diagonal C and the couplings to the E, N, NE
// and NW neighbours. The W, S, SW and SE couplings are read from the neighbours' E, N, NE and NW.
//
// Prolongation P by node parity (x, y):
//   C point (even, even)    injection;
//   H-edge (odd, even)      from its W and E coarse neighbours;
//   V-edge (even, odd)      from its S and N coarse neighbours;
//   centre (odd, odd)       from the SW, SE, NW, NE coarse corners.
// The weights depend on coarse_op:
//   * GALERKIN: operator-dependent, flux-continuous weights (Dendy's black-box MG).
//     - An edge node collapses its stencil along its line: for an H-edge,
//       w_W = −(a_w + a_nw + a_sw)/(a_c + a_n + a_s).
//     - A centre solves its own row with its four edge neighbours interpolated:
//       P(centre, SW) = −(a_w P(W, SW) + a_s P(S, SW) + a_sw)/a_c, …
//   * REDISCRETIZE / GALERKIN_LINEAR: the P1 weights of fem.cpp:144-165 (edges ½, ½; centres ½
//     to SW and NE).
// Weights to Dirichlet coarse nodes are dropped (fem.cpp:191-194 zeroes them after restriction).
// Coarse operators:
//   * GALERKIN, GALERKIN_LINEAR: A_c = Pᵀ A P over the free nodes.
//   * REDISCRETIZE: re-assembled from injected k (fem.cpp:241-244).
struct S9 {
  double c, e, w, n, s, ne, nw, se, sw;
};

// Eliminated P1 row of node (x, y) of a grid with m cells whose nodal k is read at stride `st`
// from the level-0 array kb (row length n00): st = 1 gives the level-0 row, st = 2^l the reference's
// rediscretised level-l row (fem.cpp:38-138 / 241-244). Same formulas and operand order as
// edges_pair + mk_sten.
__device__ S9 row_k(const double* __restrict__ kb, int n00, int st, int m, int bc, int x, int y) {
  S9 r{0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (x < 0 || x > m || y < 0 || y > m || is_dir(bc, m, x, y)) {
    r.c = 1.0;
    return r;
  }
  constexpr double third = 1.0 / 3.0;
  auto K = [&](int a, int b2) { return __ldg(kb + (int64_t)(b2 * st) * n00 + (int64_t)a * st); };
  auto Ed = [&](int a, int b2) -> double {  // raw edge (a, b2)–(a+1, b2)
    if (a < 0 || a >= m) return 0.0;
    return -0.5 * ((b2 < m ? (K(a, b2) + K(a + 1, b2) + K(a + 1, b2 + 1)) * third : 0.0) +
                   (b2 > 0 ? (K(a, b2 - 1) + K(a + 1, b2) + K(a, b2)) * third : 0.0));
  };
  auto Nd = [&](int a, int b2) -> double {  // raw edge (a, b2)–(a, b2+1)
    if (b2 < 0 || b2 >= m) return 0.0;
    return -0.5 * ((a < m ? (K(a, b2) + K(a + 1, b2 + 1) + K(a, b2 + 1)) * third : 0.0) +
                   (a > 0 ? (K(a - 1, b2) + K(a, b2) + K(a, b2 + 1)) * third : 0.0));
  };
  const double E = Ed(x, y), W = Ed(x - 1, y), N = Nd(x, y), S = Nd(x, y - 1);
  r.c = -(E + W + N + S);
  r.e = is_dir(bc, m, x + 1, y) ? 0.0 : E;
  r.w = is_dir(bc, m, x - 1, y) ? 0.0 : W;
  r.n = is_dir(bc, m, x, y + 1) ? 0.0 : N;
  r.s = is_dir(bc, m, x, y - 1) ? 0.0 : S;
  return r;
}

// Stored coarse rows: fp64 diagonal, fp32 couplings. Rounding a coupling a to fp32 moves it by at
// most 2^-24·|a|; raising the diagonal by that bound summed over the row's eight couplings makes the
// stored operator A' = A + E with E symmetric and diagonally dominant with a non-negative diagonal
// (Gershgorin: E ⪰ 0), so A' stays SPD whenever A is, and the V-cycle stays a valid PCG
// preconditioner. (1 + 2^-20) covers the few-ulp difference between a row's own value of a W/S
// coupling and the neighbour's stored E/N of the same pair.
__device__ __forceinline__ double fp32_rounding_margin(double sum_abs_couplings) {
  return sum_abs_couplings * (0x1p-24 * (1.0 + 0x1p-20));
}

// A stored 9-point level (one sample's arrays start at off = b·N).
struct L9 {
  const double* C;
  const float *E, *N, *NE, *NW;
  int m, n0;
  int64_t Nn;
};

__device__ __forceinline__ S9 row_s(const L9& L, int64_t off, int x, int y) {
  S9 r{0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (x < 0 || x > L.m || y < 0 || y > L.m) {
    r.c = 1.0;
    return r;
  }
  const int64_t i = off + (int64_t)y * L.n0 + x;
  r.c = L.C[i];
  r.e = L.E[i];
  r.n = L.N[i];
  if (x > 0) r.w = L.E[i - 1];
  if (y > 0) r.s = L.N[i - L.n0];
  if (L.NE) {  // 9-point level (level 0 keeps 5-point rows)
    r.ne = L.NE[i];
    r.nw = L.NW[i];
    if (x > 0 && y > 0) r.sw = L.NE[i - L.n0 - 1];
    if (x < L.m && y > 0) r.se = L.NW[i - L.n0 + 1];
  }
  return r;
}

// Level-0 rows from nodal k, stored once per setup (C, E, N; 5-point) so the transfer and Galerkin
// kernels read every level the same way.
__global__ void __launch_bounds__(NT) rows0_kernel(Geo g, int bc, const double* __restrict__ k,
                                                   double* __restrict__ C, float* __restrict__ E,
                                                   float* __restrict__ Nn) {
  const int b = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x;
  if (i >= g.N) return;
  const int y = (int)((unsigned)i / (unsigned)g.n0), x = (int)i - y * g.n0;  // N < 2^31
  const S9 r = row_k(k + (int64_t)b * g.N, g.n0, 1, g.m, bc, x, y);
  const int64_t o = (int64_t)b * g.N + i;
  C[o] = r.c;
  E[o] = r.e;
  Nn[o] = r.n;
}

// Raw (un-eliminated) level-0 edge weights E(x,y) = A((x,y),(x+1,y)), N(x,y) = A((x,y),(x,y+1)) in fp32
// for the level-0 preconditioner sweeps (the Galerkin setup writes them as a by-product of its tile;
// this kernel serves the rediscretised hierarchy). Same formulas as edges_pair.
__global__ void __launch_bounds__(NT) edges0_kernel(Geo g, const double* __restrict__ k, float* __restrict__ E,
                                                    float* __restrict__ Nn) {
  const int b = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x;
  if (i >= g.N) return;
  const int m = g.m, n0 = g.n0;
  const int y = (int)((unsigned)i / (unsigned)n0), x = (int)i - y * n0;
  const double* kb = k + (int64_t)b * g.N;
  constexpr double third = 1.0 / 3.0;
  auto K = [&](int a, int b2) { return __ldg(kb + (int64_t)b2 * n0 + a); };
  double e = 0.0, nn = 0.0;
  if (x < m)
    e = -0.5 * ((y < m ? (K(x, y) + K(x + 1, y) + K(x + 1, y + 1)) * third : 0.0) +
                (y > 0 ? (K(x, y - 1) + K(x + 1, y) + K(x, y)) * third : 0.0));
  if (y < m)
    nn = -0.5 * ((x < m ? (K(x, y) + K(x + 1, y + 1) + K(x, y + 1)) * third : 0.0) +
                 (x > 0 ? (K(x - 1, y) + K(x, y) + K(x, y + 1)) * third : 0.0));
  const int64_t o = (int64_t)b * g.N + i;
  E[o] = (float)e;
  Nn[o] = (float)nn;
}

__device__ __forceinline__ bool dir_or_out(int bc, int m, int x, int y) {
  return x < 0 || x > m || y < 0 || y > m || is_dir(bc, m, x, y);
}

// Edge-node weights from the node's row (opdep) or ½ (P1); zero to Dirichlet coarse parents and
// for Dirichlet fine nodes. H-edge (odd x, even y): w0 → ((x−1)/2, y/2), w1 → ((x+1)/2, y/2).
// V-edge (even x, odd y): w0 → (x/2, (y−1)/2), w1 → (x/2, (y+1)/2).
__device__ __forceinline__ void edge_w(const S9& r, bool horiz, bool opdep, bool fine_dir, bool d0, bool d1,
                                       double& w0, double& w1) {
  if (fine_dir) {
    w0 = w1 = 0.0;
    return;
  }
  if (opdep) {
    if (horiz) {
      const double ic = rcp64(r.c + r.n + r.s);
      w0 = -(r.w + r.nw + r.sw) * ic;
      w1 = -(r.e + r.ne + r.se) * ic;
    } else {
      const double ic = rcp64(r.c + r.w + r.e);
      w0 = -(r.s + r.sw + r.se) * ic;
      w1 = -(r.n + r.nw + r.ne) * ic;
    }
  } else {
    w0 = w1 = 0.5;
  }
  if (d0) w0 = 0.0;
  if (d1) w1 = 0.0;
}

// Centre (odd x, odd y) weights to SW, SE, NW, NE; `row(x, y)` gives the level's S9 row of a node.
// INT: the node, its neighbours and their coarse parents are interior (no Dirichlet / off-grid tests).
template <bool INT = false, class RowF>
__device__ __forceinline__ void centre_w_f(RowF row, int bc, int m, int x, int y, bool opdep, double w[4]) {
  const int mc = m / 2;
  const int I = (x - 1) >> 1, J = (y - 1) >> 1;
  const bool dSW = !INT && is_dir(bc, mc, I, J), dSE = !INT && is_dir(bc, mc, I + 1, J),
             dNW = !INT && is_dir(bc, mc, I, J + 1), dNE = !INT && is_dir(bc, mc, I + 1, J + 1);
  if (!opdep) {
    w[0] = dSW ? 0.0 : 0.5;
    w[1] = 0.0;
    w[2] = 0.0;
    w[3] = dNE ? 0.0 : 0.5;
    return;
  }
  const S9 rc = row(x, y);
  double wWs, wWn, wEs, wEn, wSw, wSe, wNw, wNe;  // V-edges W, E: (S, N); H-edges S, N: (W, E)
  edge_w(row(x - 1, y), false, true, !INT && dir_or_out(bc, m, x - 1, y), dSW, dNW, wWs, wWn);
  edge_w(row(x + 1, y), false, true, !INT && dir_or_out(bc, m, x + 1, y), dSE, dNE, wEs, wEn);
  edge_w(row(x, y - 1), true, true, !INT && dir_or_out(bc, m, x, y - 1), dSW, dSE, wSw, wSe);
  edge_w(row(x, y + 1), true, true, !INT && dir_or_out(bc, m, x, y + 1), dNW, dNE, wNw, wNe);
  const double ic = rcp64(rc.c);
  w[0] = dSW ? 0.0 : -(rc.w * wWs + rc.s * wSw + rc.sw) * ic;
  w[1] = dSE ? 0.0 : -(rc.e * wEs + rc.s * wSe + rc.se) * ic;
  w[2] = dNW ? 0.0 : -(rc.w * wWn + rc.n * wNw + rc.nw) * ic;
  w[3] = dNE ? 0.0 : -(rc.e * wEn + rc.n * wNe + rc.ne) * ic;
}

__device__ void centre_w(const L9& R, int bc, int b, int x, int y, bool opdep, double w[4]) {
  const int64_t off = (int64_t)b * R.Nn;
  centre_w_f([&](int xx, int yy) { return row_s(R, off, xx, yy); }, bc, R.m, x, y, opdep, w);
}

// P row of node (x, y) (weights to its coarse parents, meaning by parity; see prow_kernel)
template <bool INT = false, class RowF>
__device__ __forceinline__ void prow_f(RowF row, int bc, int m, int x, int y, bool opdep, double w[4]) {
  const int mc = m / 2;
  w[0] = w[1] = w[2] = w[3] = 0.0;
  if (!INT && (x < 0 || x > m || y < 0 || y > m)) return;
  const bool fdir = !INT && is_dir(bc, m, x, y);
  if ((x & 1) == 0 && (y & 1) == 0) {
    w[0] = fdir ? 0.0 : 1.0;
  } else if ((x & 1) && (y & 1)) {
    centre_w_f<INT>(row, bc, m, x, y, opdep, w);
  } else {
    const bool horiz = (x & 1) != 0;
    const int I0 = horiz ? (x - 1) >> 1 : x >> 1, J0 = horiz ? y >> 1 : (y - 1) >> 1;
    const int I1 = horiz ? I0 + 1 : I0, J1 = horiz ? J0 : J0 + 1;
    const S9 r = opdep ? row(x, y) : S9{};
    edge_w(r, horiz, opdep, fdir, !INT && is_dir(bc, mc, I0, J0), !INT && is_dir(bc, mc, I1, J1), w[0], w[1]);
  }
}

// P rows of every node of a level (scratch P0..P3, per node, meaning by parity as above) and the
// level's centre weights per cell (pw, m/2 × m/2 per sample) for the V-cycle transfers.
__global__ void __launch_bounds__(NT) prow_kernel(L9 R, int bc, int opdep, double* __restrict__ P0,
                                                  double* __restrict__ P1, double* __restrict__ P2,
                                                  double* __restrict__ P3, float* __restrict__ pw0,
                                                  float* __restrict__ pw1, float* __restrict__ pw2,
                                                  float* __restrict__ pw3) {
  const int b = blockIdx.y;
  const int m = R.m, n0 = m + 1, mc = m / 2;
  const int64_t N = (int64_t)n0 * n0;
  const int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x;
  if (i >= N) return;
  const int y = (int)((unsigned)i / (unsigned)n0), x = (int)i - y * n0;  // N < 2^31
  double w[4] = {0.0, 0.0, 0.0, 0.0};
  const bool fdir = is_dir(bc, m, x, y);
  if ((x & 1) == 0 && (y & 1) == 0) {
    w[0] = fdir ? 0.0 : 1.0;
  } else if ((x & 1) && (y & 1)) {
    centre_w(R, bc, b, x, y, opdep != 0, w);
    const int64_t cell = (int64_t)b * mc * mc + (int64_t)((y - 1) >> 1) * mc + ((x - 1) >> 1);
    pw0[cell] = w[0];
    pw1[cell] = w[1];
    pw2[cell] = w[2];
    pw3[cell] = w[3];
  } else {
    const bool horiz = (x & 1) != 0;
    const int I0 = horiz ? (x - 1) >> 1 : x >> 1, J0 = horiz ? y >> 1 : (y - 1) >> 1;
    const int I1 = horiz ? I0 + 1 : I0, J1 = horiz ? J0 : J0 + 1;
    const S9 r = opdep ? row_s(R, (int64_t)b * N, x, y) : S9{};
    edge_w(r, horiz, opdep != 0, fdir, is_dir(bc, mc, I0, J0), is_dir(bc, mc, I1, J1), w[0], w[1]);
  }
  const int64_t o = (int64_t)b * N + i;
  P0[o] = w[0];
  P1[o] = w[1];
  P2[o] = w[2];
  P3[o] = w[3];
}

// Fused Galerkin setup of one level pair, tiled in shared memory: the fine rows (level 0: rebuilt
// from nodal k; levels ≥ 1: the stored 9-point rows) of a halo'd tile are staged once, the P rows of
// the tile's fine nodes are formed in shared memory (prow_f, the arithmetic of prow_kernel), and each
// thread forms one coarse Galerkin row (the loop of rap_kernel) and the centre weights pw of its
// cell. HBM traffic is the fine input (k or C…NW, plus L2-served halo) and the coarse output, instead
// of the stored rows, P rows and their re-reads of the unfused rows0/prow/rap sequence.
// Tile: GT_X × GT_Y coarse nodes, one per thread. Fine regions (global coordinates):
//   P rows  x ∈ [2I0−2, 2I0+2GT_X], y ∈ [2J0−2, 2J0+2GT_Y]
//   rows    read at x ∈ [2I0−4, 2I0+2GT_X+2], y ∈ [2J0−4, 2J0+2GT_Y+1]
//   k (L0)  x ∈ [2I0−5, 2I0+2GT_X+3], y ∈ [2J0−5, 2J0+2GT_Y+2]
constexpr int GT_X = 16, GT_Y = 8, GT_THREADS = GT_X * GT_Y;
constexpr int GA_W = 2 * GT_X + 7, GA_H = 2 * GT_Y + 6;
constexpr int GP_W = 2 * GT_X + 3, GP_H = 2 * GT_Y + 3;
constexpr int GK_W = 2 * GT_X + 9, GK_H = 2 * GT_Y + 8;
constexpr size_t galerkin_tile_smem(bool l0) {
  return sizeof(double) * ((l0 ? 3 : 5) * GA_W * GA_H + 4 * GP_W * GP_H + (l0 ? GK_W * GK_H : 0));
}

// INT: every node the tile touches (k region included) is in-grid and non-Dirichlet, and so are
// the coarse nodes of the tile: no bounds / Dirichlet tests (most tiles of a large level).
template <bool L0K, bool INT>
__device__ __forceinline__ void galerkin_tile_body(const double* __restrict__ k0, const L9& F, int bc, int opdep,
                                                   const Geo& gc, double* __restrict__ Cc, float* __restrict__ Ec,
                                                   float* __restrict__ Nc, float* __restrict__ NEc,
                                                   float* __restrict__ NWc, float* __restrict__ pw0,
                                                   float* __restrict__ pw1, float* __restrict__ pw2,
                                                   float* __restrict__ pw3, double* gsm,
                                                   float* __restrict__ E0 = nullptr,
                                                   float* __restrict__ N0 = nullptr) {
  const int b = blockIdx.z;
  const int I0 = blockIdx.x * GT_X, J0 = blockIdx.y * GT_Y;
  const int m = F.m, n0 = F.n0, mc = gc.m, mcl = m / 2;
  const int ax = 2 * I0 - 4, ay = 2 * J0 - 4, px = 2 * I0 - 2, py = 2 * J0 - 2;
  constexpr int NA = L0K ? 3 : 5;
  double* sA = gsm;                          // raw rows: C, E, N [, NE, NW], each GA_H × GA_W
  double* sP = gsm + NA * GA_W * GA_H;       // P rows: 4 × GP_H × GP_W
  auto A = [&](int q, int lx, int ly) -> double& { return sA[(q * GA_H + ly) * GA_W + lx]; };
  auto P = [&](int q, int lx, int ly) -> double& { return sP[(q * GP_H + ly) * GP_W + lx]; };
  const int tid = threadIdx.x;
  if constexpr (L0K) {
    double* sK = sP + 4 * GP_W * GP_H;
    const double* kb = k0 + (int64_t)b * F.Nn;
    const int kx = ax - 1, ky = ay - 1;
    {  // all of a thread's k loads are issued before the first is stored (the rolled load → store loop
       // serialised eight DRAM latencies: a quarter of this kernel's stall samples)
      constexpr int NKQ = (GK_W * GK_H + GT_THREADS - 1) / GT_THREADS;
      double kv[NKQ];
#pragma unroll
      for (int q = 0; q < NKQ; ++q) {
        const int i = tid + q * GT_THREADS;
        const int lx = i % GK_W, ly = i / GK_W, x = kx + lx, y = ky + ly;
        kv[q] = (i < GK_W * GK_H && (unsigned)x < (unsigned)n0 && (unsigned)y < (unsigned)n0)
                    ? __ldg(kb + (int64_t)y * n0 + x)
                    : 0.0;
      }
#pragma unroll
      for (int q = 0; q < NKQ; ++q) {
        const int i = tid + q * GT_THREADS;
        if (i < GK_W * GK_H) sK[i] = kv[q];
      }
    }
    __syncthreads();
    // level-0 rows (row_k, stride 1) of the raw region from the staged k
    constexpr double third = 1.0 / 3.0;
    auto K = [&](int x, int y) { return sK[(y - ky) * GK_W + (x - kx)]; };
    for (int i = tid; i < GA_W * GA_H; i += GT_THREADS) {
      const int lx = i % GA_W, ly = i / GA_W, x = ax + lx, y = ay + ly;
      double c = 1.0, e = 0.0, nn = 0.0;
      auto Ed = [&](int a, int b2) -> double {
        if (a < 0 || a >= m) return 0.0;
        return -0.5 * ((b2 < m ? (K(a, b2) + K(a + 1, b2) + K(a + 1, b2 + 1)) * third : 0.0) +
                       (b2 > 0 ? (K(a, b2 - 1) + K(a + 1, b2) + K(a, b2)) * third : 0.0));
      };
      auto Nd = [&](int a, int b2) -> double {
        if (b2 < 0 || b2 >= m) return 0.0;
        return -0.5 * ((a < m ? (K(a, b2) + K(a + 1, b2 + 1) + K(a, b2 + 1)) * third : 0.0) +
                       (a > 0 ? (K(a - 1, b2) + K(a, b2) + K(a, b2 + 1)) * third : 0.0));
      };
      const bool in_grid = INT || !(x < 0 || x > m || y < 0 || y > m);
      double E = 0.0, Nn = 0.0;
      if (in_grid) {
        E = Ed(x, y);
        Nn = Nd(x, y);
      }
      if (INT || (in_grid && !is_dir(bc, m, x, y))) {
        const double W = Ed(x - 1, y), S = Nd(x, y - 1);
        c = -(E + W + Nn + S);
        e = (!INT && is_dir(bc, m, x + 1, y)) ? 0.0 : E;
        nn = (!INT && is_dir(bc, m, x, y + 1)) ? 0.0 : Nn;
      }
      // raw (un-eliminated) edge weights of the tile's own fine nodes for the level-0 sweeps, fp32
      if (E0 && in_grid && x >= 2 * I0 && x < 2 * I0 + 2 * GT_X && y >= 2 * J0 && y < 2 * J0 + 2 * GT_Y) {
        const int64_t o = (int64_t)b * F.Nn + (int64_t)y * n0 + x;
        E0[o] = (float)E;
        N0[o] = (float)Nn;
      }
      A(0, lx, ly) = c;
      A(1, lx, ly) = e;
      A(2, lx, ly) = nn;
    }
  } else {
    const int64_t off = (int64_t)b * F.Nn;
    const float* src[4] = {F.E + off, F.N + off, F.NE + off, F.NW + off};
#pragma unroll 2
    for (int i = tid; i < GA_W * GA_H; i += GT_THREADS) {  // two nodes' ten loads in flight per thread
      const int lx = i % GA_W, ly = i / GA_W, x = ax + lx, y = ay + ly;
      const bool in = INT || ((unsigned)x < (unsigned)n0 && (unsigned)y < (unsigned)n0);
      const int64_t o = (int64_t)y * n0 + x;
      A(0, lx, ly) = in ? __ldg(F.C + off + o) : 1.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) A(q + 1, lx, ly) = in ? (double)__ldg(src[q] + o) : 0.0;
    }
  }
  __syncthreads();
  // S9 row of fine node (x, y) from the staged rows (row_s semantics)
  auto RS = [&](int x, int y) -> S9 {
    S9 r{0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (!INT && (x < 0 || x > m || y < 0 || y > m)) {
      r.c = 1.0;
      return r;
    }
    const int lx = x - ax, ly = y - ay;
    r.c = A(0, lx, ly);
    r.e = A(1, lx, ly);
    r.n = A(2, lx, ly);
    if (INT || x > 0) r.w = A(1, lx - 1, ly);
    if (INT || y > 0) r.s = A(2, lx, ly - 1);
    if constexpr (!L0K) {
      r.ne = A(3, lx, ly);
      r.nw = A(4, lx, ly);
      if (INT || (x > 0 && y > 0)) r.sw = A(3, lx - 1, ly - 1);
      if (INT || (x < m && y > 0)) r.se = A(4, lx + 1, ly - 1);
    }
    return r;
  };
  // P rows of the tile's fine region; centres of the tile's own cells also store pw. The region
  // origin is even, so local parity = node type: one loop per type keeps every warp on one path
  // of prow_f (centres, H-edges, V-edges, C points).
  const int64_t cb0 = (int64_t)b * mcl * mcl;
  constexpr int NXo = GP_W / 2, NXe = (GP_W + 1) / 2, NYo = GP_H / 2, NYe = (GP_H + 1) / 2;
  auto doP = [&](int lx, int ly) {
    const int x = px + lx, y = py + ly;
    double w[4];
    prow_f<INT>(RS, bc, m, x, y, opdep != 0, w);
    P(0, lx, ly) = w[0];
    P(1, lx, ly) = w[1];
    P(2, lx, ly) = w[2];
    P(3, lx, ly) = w[3];
    if ((x & 1) && (y & 1) && x < m && y < m) {
      const int Ic = (x - 1) >> 1, Jc = (y - 1) >> 1;
      if (Ic >= I0 && Ic < I0 + GT_X && Jc >= J0 && Jc < J0 + GT_Y) {
        const int64_t cell = cb0 + (int64_t)Jc * mcl + Ic;
        pw0[cell] = w[0];
        pw1[cell] = w[1];
        pw2[cell] = w[2];
        pw3[cell] = w[3];
      }
    }
  };
  for (int i = tid; i < NXo * NYo; i += GT_THREADS) doP(2 * (i % NXo) + 1, 2 * (i / NXo) + 1);  // centres
  for (int i = tid; i < NXo * NYe; i += GT_THREADS) doP(2 * (i % NXo) + 1, 2 * (i / NXo));      // H-edges
  for (int i = tid; i < NXe * NYo; i += GT_THREADS) doP(2 * (i % NXe), 2 * (i / NXe) + 1);      // V-edges
  for (int i = tid; i < NXe * NYe; i += GT_THREADS) doP(2 * (i % NXe), 2 * (i / NXe));          // C points
  __syncthreads();
  // coarse Galerkin row of (I, J) (rap_kernel's loop over the staged P rows and fine rows)
  const int I = I0 + tid % GT_X, J = J0 + tid / GT_X;
  if (I > mc || J > mc) return;
  const int64_t o = (int64_t)b * gc.N + (int64_t)J * gc.n0 + I;
  if (!INT && is_dir(bc, mc, I, J)) {
    Cc[o] = 1.0;
    Ec[o] = Nc[o] = NEc[o] = NWc[o] = 0.0;
    return;
  }
  double acc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
  for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
    for (int di = -1; di <= 1; ++di) {
      const int xi = 2 * I + di, yi = 2 * J + dj;
      if (!INT && (xi < 0 || xi > m || yi < 0 || yi > m)) continue;
      const int lxi = xi - px, lyi = yi - py;
      double pic;
      if (di == 0 && dj == 0) pic = P(0, lxi, lyi);
      else if (dj == 0) pic = di > 0 ? P(0, lxi, lyi) : P(1, lxi, lyi);
      else if (di == 0) pic = dj > 0 ? P(0, lxi, lyi) : P(1, lxi, lyi);
      else pic = dj > 0 ? (di > 0 ? P(0, lxi, lyi) : P(1, lxi, lyi)) : (di > 0 ? P(2, lxi, lyi) : P(3, lxi, lyi));
      if (!INT && pic == 0.0) continue;
      const S9 r = RS(xi, yi);
#pragma unroll
      for (int ey = -1; ey <= 1; ++ey)
#pragma unroll
        for (int ex = -1; ex <= 1; ++ex) {
          if constexpr (L0K) {  // level 0 is 5-point: the corner couplings are exact zeros
            if (ex != 0 && ey != 0) continue;
          }
          const double a = ey < 0 ? (ex < 0 ? r.sw : ex == 0 ? r.s : r.se)
                                  : ey == 0 ? (ex < 0 ? r.w : ex == 0 ? r.c : r.e)
                                            : (ex < 0 ? r.nw : ex == 0 ? r.n : r.ne);
          const int xj = xi + ex, yj = yi + ey;
          if (!INT && (a == 0.0 || xj < 0 || xj > m || yj < 0 || yj > m)) continue;
          const int lxj = xj - px, lyj = yj - py;
          const double pa = pic * a;
          const int dx = di + ex, dy = dj + ey;
          const bool ox = (dx & 1) != 0, oy = (dy & 1) != 0;
          const int bx = dx >> 1, by = dy >> 1;
          if (!ox && !oy) {
            acc[by + 1][bx + 1] += pa * P(0, lxj, lyj);
          } else if (ox && !oy) {
            acc[by + 1][bx + 1] += pa * P(0, lxj, lyj);
            acc[by + 1][bx + 2] += pa * P(1, lxj, lyj);
          } else if (!ox && oy) {
            acc[by + 1][bx + 1] += pa * P(0, lxj, lyj);
            acc[by + 2][bx + 1] += pa * P(1, lxj, lyj);
          } else {
            acc[by + 1][bx + 1] += pa * P(0, lxj, lyj);
            acc[by + 1][bx + 2] += pa * P(1, lxj, lyj);
            acc[by + 2][bx + 1] += pa * P(2, lxj, lyj);
            acc[by + 2][bx + 2] += pa * P(3, lxj, lyj);
          }
        }
    }
  const double margin = fp32_rounding_margin(fabs(acc[0][0]) + fabs(acc[0][1]) + fabs(acc[0][2]) + fabs(acc[1][0]) +
                                             fabs(acc[1][2]) + fabs(acc[2][0]) + fabs(acc[2][1]) + fabs(acc[2][2]));
  Cc[o] = acc[1][1] + margin;
  Ec[o] = (float)acc[1][2];
  Nc[o] = (float)acc[2][1];
  NEc[o] = (float)acc[2][2];
  NWc[o] = (float)acc[2][0];
}

template <bool L0K>
__global__ void __launch_bounds__(GT_THREADS) galerkin_tile_kernel(const double* __restrict__ k0, L9 F, int bc,
                                                                   int opdep, Geo gc, double* __restrict__ Cc,
                                                                   float* __restrict__ Ec, float* __restrict__ Nc,
                                                                   float* __restrict__ NEc,
                                                                   float* __restrict__ NWc, float* __restrict__ pw0,
                                                                   float* __restrict__ pw1, float* __restrict__ pw2,
                                                                   float* __restrict__ pw3, float* __restrict__ E0,
                                                                   float* __restrict__ N0) {
  extern __shared__ double gsm[];
  const int I0 = blockIdx.x * GT_X, J0 = blockIdx.y * GT_Y, m = F.m;
  const bool interior = 2 * I0 - 5 >= 1 && 2 * I0 + 2 * GT_X + 3 <= m - 1 && 2 * J0 - 5 >= 1 &&
                        2 * J0 + 2 * GT_Y + 3 <= m - 1;
  if (interior)
    galerkin_tile_body<L0K, true>(k0, F, bc, opdep, gc, Cc, Ec, Nc, NEc, NWc, pw0, pw1, pw2, pw3, gsm, E0, N0);
  else
    galerkin_tile_body<L0K, false>(k0, F, bc, opdep, gc, Cc, Ec, Nc, NEc, NWc, pw0, pw1, pw2, pw3, gsm, E0, N0);
}

// Reference rediscretisation (fem.cpp:241-244): the level-l row from the injected nodal k,
// stored in the 9-point format (zero diagonal couplings).
__global__ void __launch_bounds__(NT) rediscretize_kernel(const double* __restrict__ k0, Geo g0, int stride,
                                                          int bc, Geo gc, double* __restrict__ Cc,
                                                          float* __restrict__ Ec, float* __restrict__ Nc,
                                                          float* __restrict__ NEc, float* __restrict__ NWc) {
  const int b = blockIdx.y;
  const int64_t ic = blockIdx.x * (int64_t)NT + threadIdx.x;
  if (ic >= gc.N) return;
  const int J = (int)(ic / gc.n0), I = (int)(ic - (int64_t)J * gc.n0);
  const S9 r = row_k(k0 + (int64_t)b * g0.N, g0.n0, stride, gc.m, bc, I, J);
  const int64_t o = (int64_t)b * gc.N + ic;
  Cc[o] = r.c + fp32_rounding_margin(fabs(r.e) + fabs(r.w) + fabs(r.n) + fabs(r.s));
  Ec[o] = (float)r.e;
  Nc[o] = (float)r.n;
  NEc[o] = 0.0f;
  NWc[o] = 0.0f;
}

// Coarsest operator (stored 9-point rows) and its explicit inverse, one warp per sample. The
// reference factors the coarsest matrix by dense Cholesky (fem.cpp:255-272) and back-substitutes
// per V-cycle (:274-286); here the SPD matrix is inverted once per solve by in-place Gauss–Jordan (lane i
// owns row i), so every coarsest solve is one warp matvec. n ≤ 32 uses this path.
constexpr int CF_WARPS = 2;
// Row i of the coarsest operator: the stored level, or — when the whole grid is the coarsest level
// (k0 != null) — the exact fp64 P1 row rebuilt from k, so that single-level solves keep the exact
// inverse as preconditioner (one PCG step, as the reference's Cholesky, fem.cpp:255-292).
__device__ __forceinline__ void dense_row(const L9& L, int64_t off, int i, double* row, int n,
                                          const double* k0, int bc) {
  const int n0 = L.n0, y = i / n0, x = i - y * n0;
  const S9 r = k0 ? row_k(k0 + off, n0, 1, L.m, bc, x, y) : row_s(L, off, x, y);
  row[i] = r.c;
  if (x + 1 < n0) row[i + 1] = r.e;
  if (x > 0) row[i - 1] = r.w;
  if (y + 1 < n0) {
    row[i + n0] = r.n;
    if (x + 1 < n0) row[i + n0 + 1] = r.ne;
    if (x > 0) row[i + n0 - 1] = r.nw;
  }
  if (y > 0) {
    row[i - n0] = r.s;
    if (x + 1 < n0) row[i - n0 + 1] = r.se;
    if (x > 0) row[i - n0 - 1] = r.sw;
  }
  (void)n;
}

__global__ void __launch_bounds__(32 * CF_WARPS) coarse_factor_warp_kernel(L9 L, int B, double* __restrict__ chol,
                                                                           const double* __restrict__ k0, int bc) {
  __shared__ double mat[CF_WARPS][32][33];  // row i of A, inverted in place (odd pitch: conflict-free columns)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * CF_WARPS + w;
  if (b >= B) return;
  const int n = (int)L.Nn;
  double(*A)[33] = mat[w];
  if (lane < n) {
    for (int j = 0; j < n; ++j) A[lane][j] = 0.0;
    dense_row(L, (int64_t)b * n, lane, A[lane], n, k0, bc);
  }
  __syncwarp();
  // In-place Gauss–Jordan (no pivoting: A is SPD): after pivot c, column c holds the c-th column of the
  // running inverse. Per pivot every row does n updates (the augmented [A | I] form did 2n − c).
  for (int c = 0; c < n; ++c) {
    const double inv_p = 1.0 / A[c][c];
    const bool other = lane < n && lane != c;
    const double f = other ? A[lane][c] * inv_p : 0.0;
    __syncwarp();
    if (other) {
      for (int j = 0; j < n; ++j) A[lane][j] = fma(-f, A[c][j], A[lane][j]);
      A[lane][c] = -f;
    }
    __syncwarp();
    if (lane == c) {
      for (int j = 0; j < n; ++j) A[c][j] *= inv_p;
      A[c][c] = inv_p;
    }
    __syncwarp();
  }
  double* X = chol + (int64_t)b * 2 * n * n + (int64_t)n * n;
  for (int idx = lane; idx < n * n; idx += 32) X[idx] = A[idx / n][idx % n];
}

// Dense Cholesky + explicit inverse of the coarsest operator, one thread per sample (n > 32).
__global__ void coarse_factor_kernel(L9 Lv, int B, double* __restrict__ chol, const double* __restrict__ k0, int bc) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int n = (int)Lv.Nn;
  double* L = chol + (int64_t)b * 2 * n * n;
  for (int i = 0; i < n * n; ++i) L[i] = 0.0;
  for (int i = 0; i < n; ++i) dense_row(Lv, (int64_t)b * n, i, L + (int64_t)i * n, n, k0, bc);
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

// Coarsest grids above 1089 nodes (m = 2^j·c with odd c ≥ 33: the reference Cholesky-factors whatever
// grid is left when m stops being even, fem.cpp:239,255-272): a banded Cholesky instead of the dense
// inverse. The operator is a 9-point stencil, so its half-bandwidth is w = n0 + 1; L keeps that band,
// Lb[i·(w+1) + d] = L(i, i − w + d), d = w the diagonal. One CTA (warp) per sample, right-looking: the
// w + 1 rows a pivot touches sit in a shared-memory window that slides down the band.
constexpr int kBandMaxM = 128;  // coarsest cells per side supported by the window ((w+1)² doubles of smem)
__host__ __device__ inline size_t band_doubles(int n0) { return (size_t)n0 * n0 * (n0 + 2); }

__global__ void __launch_bounds__(32) coarse_band_factor_kernel(L9 Lv, int B, double* __restrict__ band,
                                                                const double* __restrict__ k0, int bc) {
  extern __shared__ double win[];  // rows j … j + w of the band, row i in slot i mod (w+1)
  const int b = blockIdx.x, lane = threadIdx.x;
  const int n0 = Lv.n0, n = (int)Lv.Nn, w = n0 + 1, W1 = w + 1;
  double* Lb = band + (int64_t)b * band_doubles(n0);
  // lower band of row i into window slot (zeros outside the stencil)
  auto load_row = [&](int i) {
    double* row = win + (size_t)(i % W1) * W1;
    for (int d = lane; d < W1; d += 32) row[d] = 0.0;
    __syncwarp();
    if (lane == 0) {
      const int y = i / n0, x = i - y * n0;
      const S9 r = k0 ? row_k(k0 + (int64_t)b * n, n0, 1, Lv.m, bc, x, y) : row_s(Lv, (int64_t)b * n, x, y);
      row[w] = r.c;
      if (x > 0) row[w - 1] = r.w;
      if (y > 0) {
        row[w - n0] = r.s;
        if (x + 1 < n0) row[w - n0 + 1] = r.se;
        if (x > 0) row[w - n0 - 1] = r.sw;
      }
    }
    __syncwarp();
  };
  for (int i = 0; i < min(n, W1); ++i) load_row(i);
  for (int j = 0; j < n; ++j) {
    double* rj = win + (size_t)(j % W1) * W1;
    const double d = sqrt(rj[w]);
    const double inv = 1.0 / d;
    __syncwarp();
    if (lane == 0) rj[w] = d;
    const int cnt = min(w, n - 1 - j);
    // column j below the diagonal: L(i, j) sits at slot w − (i − j) of row i
    for (int t = lane; t < cnt; t += 32) win[(size_t)((j + 1 + t) % W1) * W1 + (w - 1 - t)] *= inv;
    __syncwarp();
    // trailing update A(i, q) −= L(i, j) L(q, j), j < q ≤ i ≤ j + cnt
    for (int t1 = 0; t1 < cnt; ++t1) {
      double* ri = win + (size_t)((j + 1 + t1) % W1) * W1;
      const double lij = ri[w - 1 - t1];
      if (lij != 0.0)
        for (int t2 = lane; t2 <= t1; t2 += 32)
          ri[w - (t1 - t2)] = fma(-lij, win[(size_t)((j + 1 + t2) % W1) * W1 + (w - 1 - t2)], ri[w - (t1 - t2)]);
    }
    __syncwarp();
    // row j is final: write it out, then its slot takes row j + w + 1
    for (int dd = lane; dd < W1; dd += 32) Lb[(int64_t)j * W1 + dd] = rj[dd];
    __syncwarp();
    if (j + W1 < n) load_row(j + W1);
  }
}

// z = A⁻¹ r through the banded factor (fem.cpp:274-286): forward then backward substitution, one warp
// per sample; a row's dot product over the band is spread over the lanes.
__global__ void __launch_bounds__(32) coarse_band_solve_kernel(int n0, int B, const double* __restrict__ band,
                                                               const double* __restrict__ r, double* __restrict__ z,
                                                               const int* flags) {
  extern __shared__ double y[];  // n doubles
  const int b = blockIdx.x, lane = threadIdx.x;
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;
  const int n = n0 * n0, w = n0 + 1, W1 = w + 1;
  const double* Lb = band + (int64_t)b * band_doubles(n0);
  const double* rb = r + (int64_t)b * n;
  double* zb = z + (int64_t)b * n;
  for (int i = 0; i < n; ++i) {  // L y = r
    const double* row = Lb + (int64_t)i * W1;
    double acc = 0.0;
    for (int d = lane; d < w; d += 32) {
      const int q = i - w + d;
      if (q >= 0) acc = fma(row[d], y[q], acc);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[i] = (rb[i] - acc) / row[w];
    __syncwarp();
  }
  for (int i = n - 1; i >= 0; --i) {  // Lᵀ z = y: column i of L below the diagonal is L(i + t, i), t ≤ w
    double acc = 0.0;
    for (int t = 1 + lane; t <= w; t += 32) {
      const int q = i + t;
      if (q < n) acc = fma(Lb[(int64_t)q * W1 + (w - t)], y[q], acc);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[i] = (y[i] - acc) / Lb[(int64_t)i * W1 + w];
    __syncwarp();
  }
  for (int i = lane; i < n; i += 32) zb[i] = y[i];
}

// ---- coarse levels (9-point): red-black GS V(1,1), one thread per node -------------------------------
// Red = (x + y) even. Within a color the nodes update simultaneously (Jacobi for the same-color
// diagonal neighbours), so every sweep is a parallel, deterministic pass; the V-cycle stays
// symmetric (pre red→black, post black→red) and CG-valid. From z = 0 the pre-smoother's diagonal
// terms vanish: red z = r/C, black z = (r − Σ_WENS a z_red)/C.

// ---- PCG init: u = lift (or the nested-iteration guess), r = b − A u, ‖b‖, ‖r‖ -------------------
// One thread per column marching INIT_RY rows, so a CTA covers NT × INIT_RY nodes and does one
// fixed-order reduction (a CTA per 256 nodes made the init launch-/reduction-bound: 1M CTAs per
// config-4 batch).
constexpr int INIT_RY = 16;

// b_i for a free node (fem.cpp:85-86 load, :109-114 flow-cell column elimination)
__device__ __forceinline__ double init_rhs(const double* __restrict__ kb, int bc, int forcing, double fval, int m,
                                           int n0, int p0, int p1) {
  const int tri = 2 * (p0 < m && p1 < m) + (p0 > 0 && p1 < m) + 2 * (p0 > 0 && p1 > 0) + (p0 < m && p1 > 0);
  const double h = 1.0 / m;
  double bi = forcing ? tri * (fval * (0.5 * h * h) / 3.0) : 0.0;
  if (bc == OSC_BC_FLOWCELL && p0 == 1) {
    auto K = [&](int a0, int a1) { return kb[(int64_t)a1 * n0 + a0]; };
    const double e = -0.5 * ((p1 < m ? (K(0, p1) + K(1, p1) + K(1, p1 + 1)) / 3.0 : 0.0) +
                             (p1 > 0 ? (K(0, p1 - 1) + K(1, p1) + K(0, p1)) / 3.0 : 0.0));
    bi -= e * 1.0;
  }
  return bi;
}

// u0 = P₁ u_c at fine node (x, y): the reference's P1 transfer (fem.cpp:144-165: C points injected,
// edge nodes ½·(two parents), cell centres ½·(SW + NE) along the triangulation's diagonal).
__device__ __forceinline__ double nested_guess(const double* __restrict__ ucb, int nc0, int x, int y) {
  const int I = x >> 1, J = y >> 1;
  const double* u = ucb + (int64_t)J * nc0 + I;
  const bool ox = x & 1, oy = y & 1;
  if (!ox && !oy) return u[0];
  if (ox && !oy) return 0.5 * (u[0] + u[1]);
  if (!ox && oy) return 0.5 * (u[0] + u[nc0]);
  return 0.5 * (u[0] + u[nc0 + 1]);
}

__device__ __forceinline__ void init_finish(const Geo& g, double tol, int max_iter_factor, double bb, double rr,
                                            double* scal, int* flags, double2* partial, int maxp,
                                            unsigned* counter, int* n_active, double* hist, int hist_cap) {
  const int b = blockIdx.z;
  double tb, tr;
  if (reduce2_last(bb, rr, partial, maxp, counter, b, tb, tr) && threadIdx.x == 0) {
    const double bnorm = sqrt(tb);
    const double rel = sqrt(tr) / bnorm;
    scal[b * S_NSCAL + S_BNORM] = bnorm;
    scal[b * S_NSCAL + S_REL] = rel;
    scal[b * S_NSCAL + S_RZ] = 0.0;
    scal[b * S_NSCAL + S_BETA] = 0.0;
    const int64_t cap = (int64_t)max_iter_factor * g.N;
    // NaN (b = 0) → converged, as in fem.cpp:367; a zero cap fails before the first iteration
    // (fem.cpp:374: iter++ >= max_iter)
    const int act = (rel > tol && cap > 0) ? 1 : 0;
    flags[b * F_NFLAGS + F_ACTIVE] = act;
    flags[b * F_NFLAGS + F_ITERS] = 0;
    flags[b * F_NFLAGS + F_STATUS] = (rel > tol && cap <= 0) ? OSC_ERR_SOLVER : 0;
    flags[b * F_NFLAGS + F_FIRST] = 1;
    flags[b * F_NFLAGS + F_MAXIT] = (int)(cap < 0x7fffffff ? cap : 0x7fffffff);
    if (hist && hist_cap > 0) hist[(int64_t)b * hist_cap] = rel;
    if (act) atomicAdd(n_active, 1);
  }
}

// uc == nullptr: the reference's Dirichlet lift (fem.cpp:335-339), u = g on Dirichlet rows and 0
// elsewhere, r = b. uc != nullptr: nested iteration, u0 = P₁ u_c (the coarse coupled solve) on the
// free rows and r0 = b − A u0 (A rows rebuilt from k as row_k; eliminated rows have no Dirichlet
// couplings). ‖b‖ and the stopping test are the same in both cases.
__global__ void __launch_bounds__(NT) pcg_init_kernel(Geo g, int bc, int forcing, double fval, double tol,
                                                      int max_iter_factor, const double* __restrict__ k,
                                                      const double* __restrict__ uc, double* __restrict__ u,
                                                      double* __restrict__ r, double* scal, int* flags,
                                                      double2* partial, int maxp, unsigned* counter,
                                                      int* n_active, double* hist, int hist_cap) {
  const int b = blockIdx.z;
  const int m = g.m, n0 = g.n0, nc0 = m / 2 + 1;
  const int x = blockIdx.x * NT + threadIdx.x;
  const int y0 = blockIdx.y * INIT_RY, y1 = min(y0 + INIT_RY, n0);
  const int64_t off = (int64_t)b * g.N;
  const double* kb = k + off;
  const double* ucb = uc ? uc + (int64_t)b * nc0 * nc0 : nullptr;
  double bb = 0.0, rr = 0.0;
  if (x < n0) {
    for (int y = y0; y < y1; ++y) {
      const int64_t i = off + (int64_t)y * n0 + x;
      double bi;
      if (is_dir(bc, m, x, y)) {
        bi = (bc == OSC_BC_FLOWCELL && x == 0) ? 1.0 : 0.0;
        u[i] = bi;
        r[i] = 0.0;
      } else {
        bi = init_rhs(kb, bc, forcing, fval, m, n0, x, y);
        double ri = bi, u0 = 0.0;
        if (ucb) {
          const S9 a = row_k(kb, n0, 1, m, bc, x, y);
          u0 = nested_guess(ucb, nc0, x, y);
          double au = a.c * u0;
          if (a.e != 0.0) au += a.e * nested_guess(ucb, nc0, x + 1, y);
          if (a.w != 0.0) au += a.w * nested_guess(ucb, nc0, x - 1, y);
          if (a.n != 0.0) au += a.n * nested_guess(ucb, nc0, x, y + 1);
          if (a.s != 0.0) au += a.s * nested_guess(ucb, nc0, x, y - 1);
          ri = bi - au;
        }
        u[i] = u0;
        r[i] = ri;
        rr += ri * ri;
      }
      bb += bi * bi;
    }
  }
  init_finish(g, tol, max_iter_factor, bb, rr, scal, flags, partial, maxp, counter, n_active, hist, hist_cap);
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
__host__ __device__ __forceinline__ int rows_per_warp(int m) {
  // 64 rows at m ≥ 1024 halve the ring warm-up and the per-CTA reduction tail of the level-0 sweeps
  // (config 4: smooth_up 40.4 → 38.2 ms, pcg_update 45.3 → 44.6 ms per step)
  return m >= 1024 ? 2 * LY : (m >= 512 ? LY : (m >= 64 ? 16 : 8));
}
constexpr int LYC = 16;      // coarse output rows per warp (restriction) on large grids
__host__ __device__ __forceinline__ int coarse_rows_per_warp(int mc) {
  return mc >= 512 ? 32 : (mc >= 256 ? LYC : 4);
}
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

// Storage types of the level-0 search direction p and preconditioned residual z. fp32 storage (fp64
// arithmetic; u and r keep using one fp64 p, so r stays the residual of u) was measured twice, before
// and after the pcg_update prefetch: same iteration counts; the up sweep gains 4–7% from the narrower
// z store, pcg_update loses up to 8% at 1024² on the float loads and conversions; the step is
// unchanged within the run-to-run spread, so both stay fp64 (profiles/ab_r2/pz32_vs_pz64.txt).
using p_t = double;
using z_t = double;

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
#define PAIR_PROLOGUE PAIR_PROLOGUE_W(MW)
#define PAIR_PROLOGUE_W(WPB)                                                            \
  const int b = blockIdx.z;                                                             \
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;                                          \
  PairCtx c;                                                                            \
  {                                                                                     \
    const int lane = threadIdx.x & 31;                                                  \
    const int strip = blockIdx.x * (WPB) + (threadIdx.x >> 5);                          \
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
  const int strip0 = blockIdx.x * (WPB) + (threadIdx.x >> 5);                           \
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

// ---- PCG step of the one-reduction (Chronopoulos–Gear) iteration, fused with the search direction:
//   p = z + βp (p = z first), u += αp, r −= αAp (Ap recomputed from p), ‖r‖ → convergence.
// α and β come from the previous V-cycle's epilogue (smooth_up_kernel: γ = ⟨r, z⟩, δ = ⟨z, Az⟩,
// β = γ/γ_old, α = γ/(δ − βγ/α_old)), so no ⟨p, Ap⟩ reduction (and no pcg_apply pass) precedes
// the update. Reads k, z, p_old, r, u; writes p_new, u, r_next.
template <bool INT>
__device__ __forceinline__ double pcg_update_cg_body(Geo g, int bc, const double* __restrict__ k,
                                                     const z_t* __restrict__ z, const p_t* __restrict__ p_old,
                                                     p_t* __restrict__ p_new, double* __restrict__ u,
                                                     const double* __restrict__ r, double* __restrict__ r_out,
                                                     double* scal, int* flags, const PairCtx& c) {
  PAIR_UNPACK

  const bool first = flags[b * F_NFLAGS + F_FIRST] != 0;
  const double beta = first ? 0.0 : scal[b * S_NSCAL + S_BETA];
  const double alpha = scal[b * S_NSCAL + S_ALPHA];
  const double *kb = k + off, *rb = r + off;
  const z_t* zb = z + off;
  const p_t* pb = p_old + off;
  double* ub = u + off;
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
  Pair rq = ld2<INT>(rb, xa, y0, n0), uq = ld2<INT>(ub, xa, y0, n0);
  double rr = 0.0;
  // L2 prefetch PU_PREFETCH rows ahead of the register pipeline (which holds one row of loads): the
  // kernel is latency-bound on DRAM (70% of its stall samples are long-scoreboard waits at 16 warps per
  // SM), and the prefetched rows turn those into L2 hits without spending registers. Every fourth
  // lane's address covers the 64 bytes its four lanes will load. Measured at 2048² (A/B of the
  // distance, profiles/ab_r2/pcg_update_prefetch.txt): none 5.37, 3 rows 5.68, 4 rows 5.71, 6 rows
  // 5.66, 8 rows 5.45, 12 rows 4.66 TB/s.
  constexpr int PU_PREFETCH = 4;
  const bool pf_lane = (c.lane & 3) == 0;
  for (int y = y0; y < y1; ++y) {
    if (INT && pf_lane && y + PU_PREFETCH < y1 + 2) {
      const int64_t o = (int64_t)(y + PU_PREFETCH) * n0 + xa;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(kb + o));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(zb + o));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + o));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(rb + o));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(ub + o));
    }
    const Pair kp = kq, pp = comb(zq, oq);  // row y+1 (raw rows loaded one iteration ahead)
    const Pair r0 = rq, u0 = uq;            // row y
    kq = ld2<INT>(kb, xa, y + 2, n0);
    zq = ld2<INT>(zb, xa, y + 2, n0);
    if (!first) oq = ld2<INT>(pb, xa, y + 2, n0);
    rq = ld2<INT>(rb, xa, y + 1, n0);
    uq = ld2<INT>(ub, xa, y + 1, n0);
    Pair E, N;
    edges_pair<INT>(km, k0, kp, xa, y, m, E, N);
    const Sten2 st = sten_pair<INT>(E, N, Nm, xa, y, m, bc);
    const Pair od = offd_pair(st, pm, p0, pp);
    const int64_t row = off + (int64_t)y * n0;
    if (outa) {
      const double rn = fma(-alpha, fma(st.a.d, p0.a, od.a), r0.a);
      p_new[row + xa] = (p_t)p0.a;
      u[row + xa] = fma(alpha, p0.a, u0.a);
      r_out[row + xa] = rn;
      rr = fma(rn, rn, rr);
    }
    if (outb) {
      const double rn = fma(-alpha, fma(st.b.d, p0.b, od.b), r0.b);
      p_new[row + xb] = (p_t)p0.b;
      u[row + xb] = fma(alpha, p0.b, u0.b);
      r_out[row + xb] = rn;
      rr = fma(rn, rn, rr);
    }
    km = k0; k0 = kp; pm = p0; p0 = pp; Nm = N;
  }
  return rr;
}

constexpr int PU_W = 4;  // warps per CTA of pcg_update (A/B knob: 1 and 2 warps are no faster, it is DRAM-bound)
__global__ void __launch_bounds__(32 * PU_W, 16 / PU_W) pcg_update_cg_kernel(Geo g, int bc, double tol, const double* __restrict__ k,
                                                              const z_t* __restrict__ z,
                                                              const p_t* __restrict__ p_old,
                                                              p_t* __restrict__ p_new, double* __restrict__ u,
                                                              const double* __restrict__ r, double* __restrict__ r_out,
                                                              double* scal, int* flags, double2* partial, int maxp,
                                                              unsigned* counter, int* n_active, double* hist,
                                                              int hist_cap) {
  PAIR_PROLOGUE_W(PU_W)
  const double rr = interior ? pcg_update_cg_body<true>(g, bc, k, z, p_old, p_new, u, r, r_out, scal, flags, c)
                             : pcg_update_cg_body<false>(g, bc, k, z, p_old, p_new, u, r, r_out, scal, flags, c);
  double t0, t1;
  if (reduce2_last(rr, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    flags[b * F_NFLAGS + F_FIRST] = 0;
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

// ---- nested-iteration start, column-pair marching: after pcg_init (u = lift, r = b, ‖b‖), add the
// prolonged coarse coupled solution g = P₁ u_c (zero on Dirichlet rows) to u and form r = b − A g with
// A rebuilt from k in registers, exactly as pcg_update_cg forms r − αAp (α = 1, p = g). Lane l's
// columns xa (even) and xa + 1 (odd) share the coarse column I = xa/2, so the two P₁ cases per row
// are static; each coarse row pair is read once per fine row.
template <bool INT>
__device__ __forceinline__ Pair nested_pair(const double* __restrict__ ucb, int nc0, int xa, int y, int m, int bc) {
  if (!INT) {
    const double va = ((unsigned)xa <= (unsigned)m && (unsigned)y <= (unsigned)m && !is_dir(bc, m, xa, y))
                          ? nested_guess(ucb, nc0, xa, y) : 0.0;
    const double vb = ((unsigned)(xa + 1) <= (unsigned)m && (unsigned)y <= (unsigned)m && !is_dir(bc, m, xa + 1, y))
                          ? nested_guess(ucb, nc0, xa + 1, y) : 0.0;
    return Pair{va, vb};
  }
  const double* u = ucb + (int64_t)(y >> 1) * nc0 + (xa >> 1);
  const double u00 = __ldg(u), u01 = __ldg(u + 1);
  if (!(y & 1)) return Pair{u00, 0.5 * (u00 + u01)};
  return Pair{0.5 * (u00 + __ldg(u + nc0)), 0.5 * (u00 + __ldg(u + nc0 + 1))};
}

// Raw coarse values of fine row y for the interior path: (u_c[J][I], u_c[J][I+1]) and, when y is
// odd, row J+1 as well (J = y/2, I = xa/2); loaded one row ahead of use.
struct CoarseRaw {
  double a0, a1, b0, b1;
};
__device__ __forceinline__ CoarseRaw coarse_raw(const double* __restrict__ ucb, int nc0, int xa, int y) {
  const double* u = ucb + (int64_t)(y >> 1) * nc0 + (xa >> 1);
  CoarseRaw c{__ldg(u), __ldg(u + 1), 0.0, 0.0};
  if (y & 1) {
    c.b0 = __ldg(u + nc0);
    c.b1 = __ldg(u + nc0 + 1);
  }
  return c;
}
__device__ __forceinline__ Pair coarse_pair(const CoarseRaw& c, int y) {
  if (!(y & 1)) return Pair{c.a0, 0.5 * (c.a0 + c.a1)};
  return Pair{0.5 * (c.a0 + c.b0), 0.5 * (c.a0 + c.b1)};
}

// Whole start of a nested solve in one marching pass: b (init_rhs), the lift on Dirichlet rows
// (u = g, r = 0), u = g_guess and r = b − A·g_guess on the free rows, and ‖b‖², ‖r‖² for the stopping
// test. Returns (Σ b², Σ r²) of this lane's output nodes.
template <bool INT>
__device__ __forceinline__ double2 init_nested_body(Geo g, int bc, int forcing, double fval,
                                                    const double* __restrict__ k, const double* __restrict__ uc,
                                                    double* __restrict__ u, double* __restrict__ r, const PairCtx& c) {
  PAIR_UNPACK
  const int nc0 = m / 2 + 1;
  const double* ucb = uc + (int64_t)b * nc0 * nc0;
  const double* kb = k + off;
  const Pair zero{0.0, 0.0};
  const double h = 1.0 / m;
  const double b_int = forcing ? 6 * (fval * (0.5 * h * h) / 3.0) : 0.0;  // init_rhs of an interior node
  auto guess = [&](int y) { return nested_pair<INT>(ucb, nc0, xa, y, m, bc); };
  Pair km = ld2<INT>(kb, xa, y0 - 1, n0), k0 = ld2<INT>(kb, xa, y0, n0);
  Pair pm = guess(y0 - 1), p0 = guess(y0);
  Pair Nm, Ed;
  edges_pair<INT>(zero, km, k0, xa, y0 - 1, m, Ed, Nm);
  // rows loaded one iteration ahead: k, coarse raw values and the guess of row y+1
  Pair kq = ld2<INT>(kb, xa, y0 + 1, n0);
  CoarseRaw cq{};
  Pair pq = zero;
  if (INT) cq = coarse_raw(ucb, nc0, xa, y0 + 1);
  else pq = guess(y0 + 1);
  double bb = 0.0, rr = 0.0;
  auto node = [&](int x, int y, int64_t i, const Sten& st, double pv, double odv) {
    double bi;
    if (!INT && is_dir(bc, m, x, y)) {
      bi = (bc == OSC_BC_FLOWCELL && x == 0) ? 1.0 : 0.0;
      u[i] = bi;
      r[i] = 0.0;
    } else {
      bi = INT ? b_int : init_rhs(kb, bc, forcing, fval, m, n0, x, y);
      const double rn = bi - fma(st.d, pv, odv);
      u[i] = pv;
      r[i] = rn;
      rr = fma(rn, rn, rr);
    }
    bb = fma(bi, bi, bb);
  };
  for (int y = y0; y < y1; ++y) {
    const Pair kp = kq;
    const Pair pp = INT ? coarse_pair(cq, y + 1) : pq;
    kq = ld2<INT>(kb, xa, y + 2, n0);
    if (INT) cq = coarse_raw(ucb, nc0, xa, y + 2);
    else pq = guess(y + 2);
    Pair E, N;
    edges_pair<INT>(km, k0, kp, xa, y, m, E, N);
    const Sten2 st = sten_pair<INT>(E, N, Nm, xa, y, m, bc);
    const Pair od = offd_pair(st, pm, p0, pp);
    const int64_t row = off + (int64_t)y * n0;
    if (outa) node(xa, y, row + xa, st.a, p0.a, od.a);
    if (outb) node(xb, y, row + xb, st.b, p0.b, od.b);
    km = k0; k0 = kp; pm = p0; p0 = pp; Nm = N;
  }
  return make_double2(bb, rr);
}

// No active-flag test in the prologue: this kernel initialises the flags.
__global__ void __launch_bounds__(MT, 4) pcg_init_nested_kernel(Geo g, int bc, int forcing, double fval, double tol,
                                                                int max_iter_factor, const double* __restrict__ k,
                                                                const double* __restrict__ uc, double* __restrict__ u,
                                                                double* __restrict__ r, double* scal, int* flags,
                                                                double2* partial, int maxp, unsigned* counter,
                                                                int* n_active, double* hist, int hist_cap) {
  PairCtx c;
  {
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * MW + (threadIdx.x >> 5);
    const int ly = rows_per_warp(g.m);
    c.b = blockIdx.z;
    c.lane = lane;
    c.m = g.m;
    c.n0 = g.n0;
    c.xa = strip * 60 - 2 + 2 * lane;
    c.xb = c.xa + 1;
    c.outa = lane >= 1 && lane < 31 && c.xa <= g.m;
    c.outb = lane >= 1 && lane < 31 && c.xb <= g.m;
    c.y0 = blockIdx.y * ly;
    c.y1 = min(c.y0 + ly, g.n0);
    c.off = (int64_t)c.b * g.N;
  }
  const int strip0 = blockIdx.x * MW + (threadIdx.x >> 5);
  const bool interior = strip0 * 60 - 2 >= 2 && strip0 * 60 + 61 <= g.m - 2 && c.y0 >= 3 && c.y1 <= g.m - 2;
  const double2 br = interior ? init_nested_body<true>(g, bc, forcing, fval, k, uc, u, r, c)
                              : init_nested_body<false>(g, bc, forcing, fval, k, uc, u, r, c);
  init_finish(g, tol, max_iter_factor, br.x, br.y, scal, flags, partial, maxp, counter, n_active, hist, hist_cap);
}

// ---- PCG update fused with the level-0 pre-smoother:
//   u += αp, r −= αAp (Ap recomputed from p), ‖r‖ → convergence,
//   then z_red = r/D, z_black = (r − Σ A z_red)/D  (red-black GS from z = 0)
template <bool INT>
__device__ __forceinline__ double pcg_update_down_kernel_body(
    Geo g, int bc, double tol, const double* __restrict__ k, const double* __restrict__ p,
    double* __restrict__ u, const double* __restrict__ r, double* __restrict__ r_out,
    double* __restrict__ z, double* scal, int* flags, double2* partial, int maxp, unsigned* counter,
    int* n_active, double* hist, int hist_cap, int init, const PairCtx& c) {
  PAIR_UNPACK

  const double alpha = init ? 0.0 : scal[b * S_NSCAL + S_ALPHA];
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
  return rr;
}

__global__ void __launch_bounds__(MT, 4) pcg_update_down_kernel(
    Geo g, int bc, double tol, const double* __restrict__ k, const double* __restrict__ p,
    double* __restrict__ u, const double* __restrict__ r, double* __restrict__ r_out,
    double* __restrict__ z, double* scal, int* flags, double2* partial, int maxp, unsigned* counter,
    int* n_active, double* hist, int hist_cap, int init) {
  PAIR_PROLOGUE
  // generic body only: the interior specialisation pushes this kernel past 128 registers (spills)
  (void)interior;
  const double rr = pcg_update_down_kernel_body<false>(g, bc, tol, k, p, u, r, r_out, z, scal, flags, partial, maxp, counter, n_active, hist, hist_cap, init, c);
  if (init) return;  // the first V-cycle's pre-smoother pass (α = 0): no PCG bookkeeping
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
// After the black sweep the residual vanishes on black nodes and equals −Σ A z_black on red nodes
// (C points and cell centres). So
//   rc(I,J) = t(2I,2J) + Σ over the 4 centres around (2I,2J) of P(centre, (I,J))·t(centre),
// with the centre weights from the level's pw cells (operator-dependent, or ½ to SW/NE for P1:
// t(2I+1,2J+1) + t(2I−1,2J−1) halves as in fem.cpp:168-195). Zero at coarse Dirichlet nodes.
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

struct PW4 {
  const float *w0, *w1, *w2, *w3;  // centre weights to SW, SE, NW, NE per cell (m/2 × m/2 per sample)
};

// ---- coarse levels (9-point): row-marching kernels ----------------------------------------------------
// The same column-pair layout as level 0: lane l owns the even column xa and xb = xa + 1 of its
// 64-column strip, so each row gives every lane one red and one black node. The stored operator
// rows are loaded as pairs; the W, S, SW, SE couplings come from the previous lane (shuffles) and
// from the previous row (carried).
struct R9 {
  Pair C, E, N, NE, NW;
};

// 9-point rows of both columns of row y from its loads and row y−1's N, NE, NW.
__device__ __forceinline__ void st9_pair(const R9& q, Pair Nm, Pair NEm, Pair NWm, S9& A, S9& Bc) {
  A.c = q.C.a;  A.e = q.E.a;  A.w = shup(q.E.b);  A.n = q.N.a;  A.s = Nm.a;
  A.ne = q.NE.a;  A.nw = q.NW.a;  A.sw = shup(NEm.b);  A.se = NWm.b;
  Bc.c = q.C.b;  Bc.e = q.E.b;  Bc.w = q.E.a;  Bc.n = q.N.b;  Bc.s = Nm.b;
  Bc.ne = q.NE.b;  Bc.nw = q.NW.b;  Bc.sw = NEm.a;  Bc.se = shdn(NWm.a);
}

// Σ over the 8 neighbours of node a / node b of row y, from value pairs of rows y−1 (vm), y (v0), y+1 (vp)
__device__ __forceinline__ double dot8_a(const S9& A, Pair vm, Pair v0, Pair vp) {
  return A.e * v0.b + A.w * shup(v0.b) + A.n * vp.a + A.s * vm.a + A.ne * vp.b + A.nw * shup(vp.b) +
         A.se * vm.b + A.sw * shup(vm.b);
}
__device__ __forceinline__ double dot8_b(const S9& B, Pair vm, Pair v0, Pair vp) {
  return B.e * shdn(v0.a) + B.w * v0.a + B.n * vp.b + B.s * vm.b + B.ne * shdn(vp.a) + B.nw * vp.a +
         B.se * shdn(vm.a) + B.sw * vm.a;
}
// diagonal part only
__device__ __forceinline__ double diag_a(const S9& A, Pair vm, Pair vp) {
  return A.ne * vp.b + A.nw * shup(vp.b) + A.se * vm.b + A.sw * shup(vm.b);
}
__device__ __forceinline__ double diag_b(const S9& B, Pair vm, Pair vp) {
  return B.ne * shdn(vp.a) + B.nw * vp.a + B.se * shdn(vm.a) + B.sw * vm.a;
}

constexpr int CU_W = 1;  // warps per CTA of the coarse ring up sweep
#define C9_PROLOGUE C9_PROLOGUE_W(MW)
#define C9_PROLOGUE_W(WPB)                                                            \
  const int b = blockIdx.z;                                                           \
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;                                        \
  const int lane = threadIdx.x & 31;                                                  \
  const int strip = blockIdx.x * (WPB) + (threadIdx.x >> 5);                          \
  const int m = L.m, n0 = L.n0;                                                       \
  const int xa = strip * 60 - 2 + 2 * lane, xb = xa + 1;                              \
  const bool outa = lane >= 1 && lane < 31 && xa <= m;                                \
  const bool outb = lane >= 1 && lane < 31 && xb <= m;                                \
  const int ly = rows_per_warp(m);                                                    \
  const int y0 = blockIdx.y * ly, y1 = min(y0 + ly, n0);                              \
  const int64_t off = (int64_t)b * L.Nn;                                              \
  (void)outa; (void)outb;

// ---- coarse levels: cp.async-staged marching ------------------------------------------------------
// The register-marching coarse kernels above hold the next row's loads in registers (≈190
// registers for the up kernel: 2 CTAs per SM, one row of loads in flight per warp, ≈30% of HBM).
// The ring variants stage each lane's raw row data P rows ahead in a per-thread slot of shared
// memory with cp.async (the slot is written and read by the same thread, so no barriers): loads
// in flight no longer cost registers, and the zc / pw gathers of the prolongation are prefetched
// with the rest.
// 8-byte async copy global → shared; !ok zero-fills without reading (g is then never dereferenced,
// so callers pass the unclamped address)
__device__ __forceinline__ void cpa8(double* s, const double* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"((unsigned)ok << 3)
               : "memory");
}
// 4-byte variant for the fp32 couplings and transfer weights
__device__ __forceinline__ void cpa4(float* s, const float* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(g), "r"((unsigned)ok << 2)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Ring rows are laid out per warp: for each staged array the 64 consecutive columns x0 … x0+63 of
// the warp's strip (x0 = xa of lane 0), so lane l's cp.async pair covers columns x0+l and x0+32+l
// (each warp instruction moves 256 contiguous bytes) and lane l reads its own column pair back as
// one 16-byte shared load. A __syncwarp orders the cp.async data with the other lanes' reads.
//   up:   C E N NE NW r [z]  (64 each), zc of coarse rows Jc, Jc+1 (33 each: coarse columns
//         x0/2 … x0/2+32), pw of the odd rows' cells (4 × 32), 3 halo couplings
// Ring row of the up sweep, in doubles: C and r (64 columns each, fp64), the fp32 couplings E N NE NW
// (64 each), zc of coarse rows Jc, Jc+1 (33 each), then fp32: pw of the odd rows' cells (4 × 32) and
// 3 halo couplings.
struct UpLayout {
  static constexpr int C = 0, R = 64, CPL = 128;     // CPL: float region, E N NE NW at CPL*2 + k*64
  static constexpr int ZC0 = CPL + 128, ZC1 = ZC0 + 33, PW = ZC1 + 33, X = PW + 64;  // PW, X: floats
  static constexpr int WORDS = (X + 2 + 1) & ~1;   // doubles per warp-row (even: 16-byte alignment)
};
enum { UP_E = 0, UP_N = 1, UP_NE = 2, UP_NW = 3 };
// rows staged per warp: 3 rows. A/B with one-warp CTAs (fp64 couplings): 4 or 5 rows were slower
// (coarse up sweep 19.4 → 28 ms per config-4 step: fewer resident warps)
constexpr int UP_RING = 3;
template <bool RZ>
constexpr size_t up_ring_smem() { return sizeof(double) * UP_RING * CU_W * UpLayout::WORDS; }

// Prolongation + post-smoother, ring-staged (same algorithm as c_up_march_kernel; pending smoother
// rows carry partial sums). RZ: the pre-smoothed z is recomputed from r and the operator (red z =
// r/C, black z = (r − Σ_WENS a z_red)/C, as c_pre_march_kernel) instead of loaded, so the down
// sweep need not store it.
template <bool RZ>
__global__ void __launch_bounds__(32 * CU_W, 3 * 4 / CU_W) c_up_ring_kernel(L9 L, int bc, int opdep, const double* __restrict__ r,
                                                          const double* __restrict__ z, PW4 pw, Geo gc,
                                                          const double* __restrict__ zc, double* __restrict__ z2,
                                                          const int* flags) {
  C9_PROLOGUE_W(CU_W)
  static_assert(RZ, "the up sweep recomputes the pre-smoothed z");
  using LY = UpLayout;
  extern __shared__ __align__(16) double ring[];
  const int warp = threadIdx.x >> 5;
  const double *rb = r + off, *zb = z + off, *zcb = zc + (int64_t)b * gc.N;
  const int x0 = xa - 2 * lane, I0 = x0 >> 1, nc0 = gc.n0;
  const int mcl = m / 2;
  const int64_t cb0 = (int64_t)b * mcl * mcl;
  const float* cpl[4] = {L.E + off, L.N + off, L.NE + off, L.NW + off};
  (void)zb;
  auto slot = [&](int y) {
    return ring + ((size_t)((unsigned)(y - (y0 - 4)) % UP_RING) * CU_W + warp) * LY::WORDS;
  };
  // stage row y into its slot (off-grid values are zero-filled); rows past the last one the chunk
  // reads are skipped (their groups stay empty)
  const int ylast = y1 + 1 + (RZ ? 1 : 0);
  auto issue = [&](int y) {
    if (y > ylast) return;
    double* S = slot(y);
    const bool yok = (unsigned)y < (unsigned)n0;
    const int c0 = x0 + lane, c1 = c0 + 32;
    const bool ok0 = yok && (unsigned)c0 < (unsigned)n0, ok1 = yok && (unsigned)c1 < (unsigned)n0;
    const int64_t i0 = (int64_t)y * n0 + c0;
    cpa8(S + LY::C + lane, L.C + off + i0, ok0);
    cpa8(S + LY::C + 32 + lane, L.C + off + i0 + 32, ok1);
    cpa8(S + LY::R + lane, rb + i0, ok0);
    cpa8(S + LY::R + 32 + lane, rb + i0 + 32, ok1);
    float* SF = reinterpret_cast<float*>(S + LY::CPL);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cpa4(SF + k * 64 + lane, cpl[k] + i0, ok0);
      cpa4(SF + k * 64 + 32 + lane, cpl[k] + i0 + 32, ok1);
    }
    // coarse values of the prolongation: row Jc (and Jc+1 on odd rows), columns I0 … I0+32
    const int Jc = y >> 1, ci = I0 + lane;
    const bool cok = (unsigned)ci < (unsigned)nc0, cok2 = (unsigned)(ci + 32) < (unsigned)nc0;
    const bool j0 = (unsigned)Jc < (unsigned)nc0, j1 = (unsigned)(Jc + 1) < (unsigned)nc0;
    const double* zr0 = zcb + (int64_t)Jc * nc0 + ci;
    cpa8(S + LY::ZC0 + lane, zr0, j0 && cok);
    if (lane == 0) cpa8(S + LY::ZC0 + 32, zr0 + 32, j0 && cok2);
    if (y & 1) {
      cpa8(S + LY::ZC1 + lane, zr0 + nc0, j1 && cok);
      if (lane == 0) cpa8(S + LY::ZC1 + 32, zr0 + nc0 + 32, j1 && cok2);
      const bool ok = ci >= 0 && ci < mcl && Jc >= 0 && Jc < mcl;
      const int64_t cell = cb0 + (int64_t)Jc * mcl + ci;
      float* SP = reinterpret_cast<float*>(S + LY::PW);
      cpa4(SP + 0 * 32 + lane, pw.w0 + cell, ok);
      cpa4(SP + 1 * 32 + lane, pw.w1 + cell, ok);
      cpa4(SP + 2 * 32 + lane, pw.w2 + cell, ok);
      cpa4(SP + 3 * 32 + lane, pw.w3 + cell, ok);
    }
    // halo couplings from beyond the warp: E(x0−1, y), NE(x0−1, y−1), NW(x0+64, y−1)
    if (lane == 0) {
      const bool xk = (unsigned)(x0 - 1) < (unsigned)n0;
      float* SX = reinterpret_cast<float*>(S + LY::X);
      cpa4(SX + 0, cpl[UP_E] + (i0 - 1), yok && xk);
      cpa4(SX + 1, cpl[UP_NE] + (i0 - n0 - 1), (unsigned)(y - 1) < (unsigned)n0 && xk);
    } else if (lane == 31) {
      const bool xk = (unsigned)(x0 + 64) < (unsigned)n0;
      cpa4(reinterpret_cast<float*>(S + LY::X) + 2, cpl[UP_NW] + (i0 - n0 + 33),
           (unsigned)(y - 1) < (unsigned)n0 && xk);
    }
  };
  auto P2 = [&](const double* S, int base) {  // fp64 pair of this lane's columns
    const double2 v = *reinterpret_cast<const double2*>(S + base + 2 * lane);
    return Pair{v.x, v.y};
  };
  auto F2 = [&](const double* S, int k) {  // fp32 coupling pair
    const float2 v = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(S + LY::CPL) + k * 64 + 2 * lane);
    return Pair{(double)v.x, (double)v.y};
  };
  auto raw9 = [&](const double* S, int y) {
    R9 q{P2(S, LY::C), F2(S, UP_E), F2(S, UP_N), F2(S, UP_NE), F2(S, UP_NW)};
    const bool yok = (unsigned)y < (unsigned)n0;
    if (!(yok && (unsigned)xa < (unsigned)n0)) q.C.a = 1.0;
    if (!(yok && (unsigned)xb < (unsigned)n0)) q.C.b = 1.0;
    return q;
  };
  const Pair zero{0.0, 0.0};
  int y = y0 - 3;  // y0 is even (rows per warp are even): the march starts on an odd row
  // prologue: rows y0−4 (for the carried N/NE/NW), y0−3, … staged
  for (int j = 0; j < UP_RING; ++j) {
    issue(y - 1 + j);
    cpa_commit();
  }
  cpa_wait<UP_RING - 1>();
  __syncwarp();
  Pair Nm, NEm, NWm;
  {
    const double* S = slot(y - 1);
    Nm = F2(S, UP_N);
    NEm = F2(S, UP_NE);
    NWm = F2(S, UP_NW);
  }
  __syncwarp();
  issue(y - 1 + UP_RING);
  cpa_commit();
  double zrm = 0.0, zr0 = 0.0;  // RZ: red pre-smoothed z of rows y−1, y
  if (RZ) {
    cpa_wait<UP_RING - 1>();
    __syncwarp();
    const double* S = slot(y);
    const R9 q = raw9(S, y);
    zr0 = P2(S, LY::R).b * rcp64s(q.C.b);  // row y0−3 is odd: red at b
  }
  // Pending smoother rows carry partial sums instead of stencils: every neighbour term is folded in
  // as soon as its value exists, so only the couplings still to be applied stay live.
  //   black node of row y−1: Σ over the S/E/W-side neighbours done; N, NE, NW wait for v(y)
  //   red node of row y−1:   S (black new of row y−2) and SE/SW (v(y−2)) done; E/W (black new of
  //                          row y−1) and NE/NW (v(y)) arrive now, N (black new of row y) next step
  //   red node of row y−2:   only N (black new of row y−1) left
  struct PendB { double n, ne, nw, ic, rr; };
  struct PendR1 { double e, w, ne, nw, n, ic, rr; };
  struct PendR2 { double n, ic, rr; };
  PendB pb{0, 0, 0, 0, 0};
  PendR1 pr1{0, 0, 0, 0, 0, 0, 0};
  PendR2 pr2{0, 0, 0};
  Pair vm1 = zero;     // v of row y−1
  double zbn1 = 0.0;   // black new of row y−2 (output with the red of row y−2)
  // one row; RA = red at column a in row y (row parity is static: the loop is unrolled by 2)
  auto step = [&](auto RA, int y) {
    constexpr bool ra0 = decltype(RA)::value;
    // row y (RZ: and y+1) resident; groups complete in issue order
    cpa_wait<RZ ? UP_RING - 2 : UP_RING - 1>();
    __syncwarp();
    const double* S = slot(y);
    const R9 qc = raw9(S, y);
    const Pair rc0 = P2(S, LY::R);
    Pair zc0;
    if constexpr (RZ) {
      const double* S1 = slot(y + 1);
      // row y+1 has its red node in the other column
      const bool ok1 = (unsigned)(y + 1) < (unsigned)n0 && (unsigned)(ra0 ? xb : xa) < (unsigned)n0;
      const double c1 = ok1 ? S1[LY::C + 2 * lane + (ra0 ? 1 : 0)] : 1.0;
      const double zrp = S1[LY::R + 2 * lane + (ra0 ? 1 : 0)] * rcp64s(c1);
      const double zr0_e = shdn(zr0), zr0_w = shup(zr0);
      if constexpr (ra0) {
        const double zbl = (rc0.b - (qc.E.b * zr0_e + qc.E.a * zr0 + qc.N.b * zrp + Nm.b * zrm)) * rcp64s(qc.C.b);
        zc0 = Pair{zr0, zbl};
      } else {
        const double Ew = shup(qc.E.b);
        const double zbl = (rc0.a - (qc.E.a * zr0 + Ew * zr0_w + qc.N.a * zrp + Nm.a * zrm)) * rcp64s(qc.C.a);
        zc0 = Pair{zbl, zr0};
      }
      zrm = zr0;
      zr0 = zrp;
    } else {
      zc0 = Pair{0.0, 0.0};
    }
    S9 A, Bc;
    st9_pair(qc, Nm, NEm, NWm, A, Bc);
    if (lane == 0) {
      A.w = reinterpret_cast<const float*>(S + LY::X)[0];
      A.sw = reinterpret_cast<const float*>(S + LY::X)[1];
    } else if (lane == 31) {
      Bc.se = reinterpret_cast<const float*>(S + LY::X)[2];
    }
    Nm = qc.N; NEm = qc.NE; NWm = qc.NW;
    // v(y) = z + P zc
    Pair v0 = zc0;
    {
      double w0, w1;
      if constexpr (ra0) {  // a = C point, b = H-edge
        const double c0 = S[LY::ZC0 + lane], c1 = S[LY::ZC0 + lane + 1];
        v0.a += c0;
        edge_w(Bc, true, opdep != 0, false, false, false, w0, w1);
        v0.b += w0 * c0 + w1 * c1;
      } else {  // a = V-edge, b = centre
        const double c00 = S[LY::ZC0 + lane], c10 = S[LY::ZC0 + lane + 1], c01 = S[LY::ZC1 + lane],
                     c11 = S[LY::ZC1 + lane + 1];
        edge_w(A, false, opdep != 0, false, false, false, w0, w1);
        v0.a += w0 * c00 + w1 * c01;
        const float* SP = reinterpret_cast<const float*>(S + LY::PW);
        v0.b += (double)SP[lane] * c00 + (double)SP[32 + lane] * c10 + (double)SP[64 + lane] * c01 +
                (double)SP[96 + lane] * c11;
      }
      const bool yin = (unsigned)y <= (unsigned)m;
      if (!yin || (unsigned)xa > (unsigned)m || is_dir(bc, m, xa, y)) v0.a = 0.0;
      if (!yin || (unsigned)xb > (unsigned)m || is_dir(bc, m, xb, y)) v0.b = 0.0;
    }
    // the slot of row y is consumed (by every lane): stage row y + UP_RING into it
    __syncwarp();
    issue(y + UP_RING);
    cpa_commit();
    // neighbours in row y of a node of row y−1 at column a / b: N, NE, NW
    const double v0a_e = shdn(v0.a), v0b_w = shup(v0.b);
    // black new of row y−1 (its black column is a when row y is red-at-a)
    const double zbn0 = ra0 ? (pb.rr - (pb.n * v0.a + pb.ne * v0.b + pb.nw * v0b_w)) * pb.ic
                            : (pb.rr - (pb.n * v0.b + pb.ne * v0a_e + pb.nw * v0.a)) * pb.ic;
    // red new of row y−2 (same column as the black of row y−1): its N neighbour
    const double zrn = (pr2.rr - pr2.n * zbn0) * pr2.ic;
    const int yo = y - 2;
    if (yo >= y0 && yo < y1) {
      double* out = z2 + off + (int64_t)yo * n0;
      if (outa) out[xa] = ra0 ? zrn : zbn1;
      if (outb) out[xb] = ra0 ? zbn1 : zrn;
    }
    // red of row y−1 (column b when row y is red-at-a): E/W black new of row y−1, NE/NW v(y)
    {
      const double zbn0_e = shdn(zbn0), zbn0_w = shup(zbn0);
      const double e_b = ra0 ? zbn0_e : zbn0, w_b = ra0 ? zbn0 : zbn0_w;
      // red at b: NE = (xb+1, y) = next lane's a, NW = (xa, y); red at a: NE = (xb, y), NW = (xa−1, y)
      const double d_ne = ra0 ? v0a_e : v0.b, d_nw = ra0 ? v0.a : v0b_w;
      pr2 = PendR2{pr1.n, pr1.ic, pr1.rr - (pr1.e * e_b + pr1.w * w_b + pr1.ne * d_ne + pr1.nw * d_nw)};
    }
    // new pending nodes of row y: black (S side + E/W from v(y−1), v(y)) and red (S = black new of
    // row y−1, SE/SW = v(y−1))
    const double vm1a_e = shdn(vm1.a), vm1b_w = shup(vm1.b);
    if constexpr (ra0) {  // red a, black b
      const S9& K = Bc;    // black at b: E = next lane's a, W = own a; S row: S = vm1.b, SE = next a, SW = vm1.a
      pb = PendB{K.n, K.ne, K.nw, rcp64s(K.c),
                 rc0.b - (K.e * v0a_e + K.w * v0.a + K.s * vm1.b + K.se * vm1a_e + K.sw * vm1.a)};
      const S9& R = A;     // red at a: S = black new of row y−1 at a (= zbn0), SE = vm1.b, SW = prev lane's b
      pr1 = PendR1{R.e, R.w, R.ne, R.nw, R.n, rcp64s(R.c), rc0.a - (R.s * zbn0 + R.se * vm1.b + R.sw * vm1b_w)};
    } else {  // red b, black a
      const S9& K = A;     // black at a: E = own b, W = prev lane's b; SE = vm1.b, SW = prev lane's b
      pb = PendB{K.n, K.ne, K.nw, rcp64s(K.c),
                 rc0.a - (K.e * v0.b + K.w * v0b_w + K.s * vm1.a + K.se * vm1.b + K.sw * vm1b_w)};
      const S9& R = Bc;    // red at b: S = zbn0 (black new of row y−1 at b), SE = next lane's a, SW = vm1.a
      pr1 = PendR1{R.e, R.w, R.ne, R.nw, R.n, rcp64s(R.c), rc0.b - (R.s * zbn0 + R.se * vm1a_e + R.sw * vm1.a)};
    }
    vm1 = v0;
    zbn1 = zbn0;
  };
  for (; y < y1 + 2; y += 2) {
    step(std::false_type{}, y);
    step(std::true_type{}, y + 1);
  }
  cpa_wait<0>();
}

// Fused pre-smoother + residual + restriction, ring-staged: z (red r/C, black (r − Σ_WENS a z_red)/C,
// as c_pre_march_kernel) is formed in registers two rows ahead of the residual and never stored;
// the residual and rc = Pᵀ t follow c_restrict_march_kernel. Reads C, E, N, NE, NW, r, pw; writes
// rc. Ring rows use the warp layout of the up kernel (C E N NE NW r, 64 columns each); the centre
// weights of the odd rows are loaded into registers one row pair ahead.
// Ring row, in doubles: C, r (64 columns each, fp64), then the fp32 couplings E N NE NW (64 each).
enum { DN_C = 0, DN_R = 64, DN_CPL = 128, DN_WORDS = 256 };
enum { DN_E = 0, DN_N = 1, DN_NE = 2, DN_NW = 3 };  // fp32 arrays of the coupling region
constexpr int DN_RING = 4;  // rows y … y+2 resident + one in flight; 4 × 4 warps × 256 × 8 B = 32 KB
constexpr int CD_W = 4;  // warps per CTA of the coarse ring down sweep
constexpr size_t DN_RING_SMEM = sizeof(double) * DN_RING * CD_W * DN_WORDS;

__global__ void __launch_bounds__(32 * CD_W, 4 * 4 / CD_W) c_down_ring_kernel(L9 L, int bc, int opdep, const double* __restrict__ r,
                                                            PW4 pw, Geo gc, double* __restrict__ rc,
                                                            const int* flags) {
  const int b = blockIdx.z;
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;
  extern __shared__ __align__(16) double ring[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int strip = blockIdx.x * CD_W + warp;
  const int I = strip * 30 - 1 + lane;
  const bool outI = lane >= 1 && lane < 31 && I <= gc.m;
  const int lyc = coarse_rows_per_warp(gc.m);
  const int J0 = blockIdx.y * lyc, J1 = min(J0 + lyc, gc.n0);
  const int m = L.m, n0 = L.n0, mc = gc.m, xa = 2 * I, xb = xa + 1, x0 = xa - 2 * lane;
  const int64_t off = (int64_t)b * L.Nn;
  const int mcl = m / 2;
  const int64_t cb0 = (int64_t)b * mcl * mcl;
  const float* cpl[4] = {L.E + off, L.N + off, L.NE + off, L.NW + off};
  const double *Cb = L.C + off, *rb = r + off;
  const int ys = 2 * J0 - 1;
  const int ylast = 2 * J1 + 1;  // residual rows end at 2J1 − 1; their z needs raw rows up to 2J1 + 1
  auto slot = [&](int y) {
    return ring + ((size_t)((unsigned)(y - (ys - 2)) % DN_RING) * CD_W + warp) * DN_WORDS;
  };
  auto issue = [&](int y) {
    if (y > ylast) return;
    double* S = slot(y);
    const bool yok = (unsigned)y < (unsigned)n0;
    const int c0 = x0 + lane, c1 = c0 + 32;
    const bool ok0 = yok && (unsigned)c0 < (unsigned)n0, ok1 = yok && (unsigned)c1 < (unsigned)n0;
    const int64_t i0 = (int64_t)y * n0 + c0;
    cpa8(S + DN_C + lane, Cb + i0, ok0);
    cpa8(S + DN_C + 32 + lane, Cb + i0 + 32, ok1);
    cpa8(S + DN_R + lane, rb + i0, ok0);
    cpa8(S + DN_R + 32 + lane, rb + i0 + 32, ok1);
    float* SF = reinterpret_cast<float*>(S + DN_CPL);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cpa4(SF + k * 64 + lane, cpl[k] + i0, ok0);
      cpa4(SF + k * 64 + 32 + lane, cpl[k] + i0 + 32, ok1);
    }
  };
  auto P2 = [&](const double* S, int base) {  // fp64 pair of this lane's columns
    const double2 v = *reinterpret_cast<const double2*>(S + base + 2 * lane);
    return Pair{v.x, v.y};
  };
  auto F2 = [&](const double* S, int k) {  // fp32 coupling pair
    const float2 v = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(S + DN_CPL) + k * 64 + 2 * lane);
    return Pair{(double)v.x, (double)v.y};
  };
  auto Cpair = [&](const double* S, int y) {  // off-grid rows are identity
    Pair c = P2(S, DN_C);
    const bool yok = (unsigned)y < (unsigned)n0;
    if (!(yok && (unsigned)xa < (unsigned)n0)) c.a = 1.0;
    if (!(yok && (unsigned)xb < (unsigned)n0)) c.b = 1.0;
    return c;
  };
  // red pre-smoothed z of row y (its red column): r/C
  auto zred = [&](int y) {
    const double* S = slot(y);
    const Pair c = Cpair(S, y), rr = P2(S, DN_R);
    return RED_IS_A(y) ? rr.a * rcp64s(c.a) : rr.b * rcp64s(c.b);
  };
  // pre-smoothed pair of row y from its red value zr0 and the red values of rows y∓1 (zrm, zrp);
  // Nm = N of row y − 1
  auto zpair = [&](int y, double zrm, double zr0, double zrp, Pair Nm) {
    const double* S = slot(y);
    const Pair c = Cpair(S, y), E0 = F2(S, DN_E), N0 = F2(S, DN_N), r0 = P2(S, DN_R);
    const double zr0_e = shdn(zr0), zr0_w = shup(zr0), Ew = shup(E0.b);
    if (RED_IS_A(y)) {
      const double zbl = (r0.b - (E0.b * zr0_e + E0.a * zr0 + N0.b * zrp + Nm.b * zrm)) * rcp64s(c.b);
      return Pair{zr0, zbl};
    }
    const double zbl = (r0.a - (E0.a * zr0 + Ew * zr0_w + N0.a * zrp + Nm.a * zrm)) * rcp64s(c.a);
    return Pair{zbl, zr0};
  };
  // centre weights of cell (I, Jc) (odd row 2Jc+1); 0 off the cells
  // fp32 weights stay fp32 in registers until their use (a conversion right after the load would
  // wait on it there and expose the load latency the row-pair prefetch is meant to hide)
  auto W4 = [&](int Jc, float w[4]) {
    const bool ok = I >= 0 && I < mcl && Jc >= 0 && Jc < mcl;
    const int64_t cell = cb0 + (int64_t)Jc * mcl + I;
    w[0] = ok ? __ldg(pw.w0 + cell) : 0.0f;
    w[1] = ok ? __ldg(pw.w1 + cell) : 0.0f;
    w[2] = ok ? __ldg(pw.w2 + cell) : 0.0f;
    w[3] = ok ? __ldg(pw.w3 + cell) : 0.0f;
  };
  float wn[4];
  W4(J0 - 1, wn);
  // prologue: rows ys−2 … ys+1 staged; z of rows ys−1, ys
  for (int j = 0; j < DN_RING; ++j) {
    issue(ys - 2 + j);
    cpa_commit();
  }
  cpa_wait<1>();  // rows ys−2, ys−1, ys
  __syncwarp();
  const double zr_m2 = zred(ys - 2), zr_m1 = zred(ys - 1), zr_0 = zred(ys);
  const Pair N_m2 = F2(slot(ys - 2), DN_N);
  Pair zm = zpair(ys - 1, zr_m2, zr_m1, zr_0, N_m2);
  Pair Nm, NEm, NWm;
  {
    const double* S = slot(ys - 1);
    Nm = F2(S, DN_N);
    NEm = F2(S, DN_NE);
    NWm = F2(S, DN_NW);
  }
  __syncwarp();
  issue(ys + 2);  // into the slot of row ys−2
  cpa_commit();
  cpa_wait<1>();  // row ys+1
  __syncwarp();
  double zrA = zr_0, zrB = zred(ys + 1);  // red z of rows y, y+1 entering row(y)
  Pair z0 = zpair(ys, zr_m1, zr_0, zrB, Nm);
  __syncwarp();
  issue(ys + 3);  // into the slot of row ys−1
  cpa_commit();
  // residuals of row y (both columns) and the row's stencils; advances the state to row y+1 and
  // stages row y+4 into row y's slot
  auto row = [&](int y, double& ta, double& tb, S9& A, S9& Bc) {
    cpa_wait<1>();  // row y+2
    __syncwarp();
    const double zrC = zred(y + 2);
    const double* S = slot(y);
    const R9 q{Cpair(S, y), F2(S, DN_E), F2(S, DN_N), F2(S, DN_NE), F2(S, DN_NW)};
    const Pair zp = zpair(y + 1, zrA, zrB, zrC, q.N);
    __syncwarp();
    issue(y + 4);
    cpa_commit();
    st9_pair(q, Nm, NEm, NWm, A, Bc);
    const bool red_a = RED_IS_A(y);
    ta = red_a ? -dot8_a(A, zm, z0, zp) : -diag_a(A, zm, zp);
    tb = red_a ? -diag_b(Bc, zm, zp) : -dot8_b(Bc, zm, z0, zp);
    if (is_dir(bc, m, xa, y) || (unsigned)xa > (unsigned)m || (unsigned)y > (unsigned)m) ta = 0.0;
    if (is_dir(bc, m, xb, y) || (unsigned)xb > (unsigned)m || (unsigned)y > (unsigned)m) tb = 0.0;
    Nm = q.N; NEm = q.NE; NWm = q.NW;
    zm = z0; z0 = zp;
    zrA = zrB; zrB = zrC;
  };
  double w[4], ta, tb, w0, w1;
  S9 A, Bc;
  // odd row 2J0−1: contributions to coarse row J0 (V-edge N weight, centre NW own / NE previous lane)
  row(ys, ta, tb, A, Bc);
  w[0] = wn[0]; w[1] = wn[1]; w[2] = wn[2]; w[3] = wn[3];
  W4(J0, wn);
  edge_w(A, false, opdep != 0, false, false, false, w0, w1);
  double carry_own = w1 * ta + w[2] * tb, carry_ne = w[3] * tb;
  double* rcb = rc + (int64_t)b * gc.N;
  for (int J = J0; J < J1; ++J) {
    // even row 2J: C point (a) and H-edge (b)
    row(2 * J, ta, tb, A, Bc);
    edge_w(Bc, true, opdep != 0, false, false, false, w0, w1);
    double acc = carry_own + shup(carry_ne) + ta + w0 * tb;
    const double he = w1 * tb;  // H-edge (2I+1, 2J) → (I+1, J)
    acc += shup(he);
    // odd row 2J+1: V-edge (a) and centre (b)
    row(2 * J + 1, ta, tb, A, Bc);
    w[0] = wn[0]; w[1] = wn[1]; w[2] = wn[2]; w[3] = wn[3];
    W4(J + 1, wn);
    edge_w(A, false, opdep != 0, false, false, false, w0, w1);
    const double se = w[1] * tb;
    acc += w0 * ta + w[0] * tb + shup(se);
    if (outI) rcb[(int64_t)J * gc.n0 + I] = is_dir(bc, mc, I, J) ? 0.0 : acc;
    carry_own = w1 * ta + w[2] * tb;
    carry_ne = w[3] * tb;
  }
  cpa_wait<0>();
}

// ---- level 0 through a cp.async ring ----------------------------------------------------------------
// The register-marching level-0 sweeps above prefetch one row of loads in registers; at 128
// registers that leaves too few bytes in flight (long-scoreboard bound at 2.7–3.7 TB/s). These
// variants stage each warp's rows (64 columns of k and r, plus the prolongation's z₁ and pw for
// the up sweep) in a shared-memory ring with cp.async, in the warp layout of the coarse kernels,
// and read k/r pairs back from it as often as needed: only the derived row state stays in
// registers. The fp32 centre weights of the up sweep occupy 64 doubles (4 × 32 floats) at L0R_PW.
enum { L0R_K = 0, L0R_R = 64, L0R_ZC0 = 128, L0R_ZC1 = 161, L0R_PW = 194 };
constexpr int L0R_WORDS_UP = 258, L0R_WORDS_DN = 128;
__device__ __forceinline__ double l0r_pw(const double* S, int lane, int q) {
  return (double)reinterpret_cast<const float*>(S + L0R_PW)[q * 32 + lane];
}
constexpr int L0R_RING = 5;
// Warps (strips) per CTA of the ring sweeps (A/B knobs; the other march kernels use MW). One-warp
// CTAs let the SM refill a warp slot as soon as that warp's strip is done, instead of holding it
// until the slowest of four finishes (end-of-kernel barrier stalls were 14–19% of the samples of
// the 4-warp up sweep). Config 4 per step: smooth_up 37.6 → 31.6 ms, restrict 23.8 → 20.4 ms,
// coarse up 20.6 → 19.3 ms (2048² solve); the coarse down sweep is slower with one warp
// (16.0 → 21.4 ms) and keeps four.
constexpr int SUR_W = 1;
constexpr int RR_W = 1;  // level-0 ring restriction
constexpr size_t L0R_SMEM_UP = sizeof(double) * L0R_RING * SUR_W * L0R_WORDS_UP;  // 51.5 KB at 4 warps
constexpr size_t L0R_SMEM_DN = sizeof(double) * L0R_RING * RR_W * L0R_WORDS_DN;  // 20.5 KB

// stage the raw edge weights (fp32 E then N, 64 + 64 floats in the 64 doubles at L0R_K) and r of fine
// row y (columns x0 … x0+63) into S; off-grid values are zero
__device__ __forceinline__ void l0_issue_kr(double* S, const float* eb, const float* nb, const double* rb, int x0,
                                            int lane, int y, int n0) {
  const bool yok = (unsigned)y < (unsigned)n0;
  const int c0 = x0 + lane, c1 = c0 + 32;
  const bool ok0 = yok && (unsigned)c0 < (unsigned)n0, ok1 = yok && (unsigned)c1 < (unsigned)n0;
  const int64_t i0 = (int64_t)y * n0 + c0;
  float* SF = reinterpret_cast<float*>(S + L0R_K);
  cpa4(SF + lane, eb + i0, ok0);
  cpa4(SF + 32 + lane, eb + i0 + 32, ok1);
  cpa4(SF + 64 + lane, nb + i0, ok0);
  cpa4(SF + 96 + lane, nb + i0 + 32, ok1);
  cpa8(S + L0R_R + lane, rb + i0, ok0);
  cpa8(S + L0R_R + 32 + lane, rb + i0 + 32, ok1);
}
__device__ __forceinline__ Pair l0_pair(const double* S, int k, int lane) {
  const double2 v = *reinterpret_cast<const double2*>(S + k + 2 * lane);
  return Pair{v.x, v.y};
}
// raw E and N of the lane's column pair in a staged row
__device__ __forceinline__ void l0_edges(const double* S, int lane, Pair& E, Pair& N) {
  const float* SF = reinterpret_cast<const float*>(S + L0R_K);
  const float2 e = *reinterpret_cast<const float2*>(SF + 2 * lane);
  const float2 n = *reinterpret_cast<const float2*>(SF + 64 + 2 * lane);
  E = Pair{(double)e.x, (double)e.y};
  N = Pair{(double)n.x, (double)n.y};
}

template <bool INT>
__device__ __forceinline__ void restrict_ring_body(Geo g, Geo gc, int bc, const float* __restrict__ e0,
                                                   const float* __restrict__ n0e,
                                                   const double* __restrict__ r, PW4 pw, double* __restrict__ rc,
                                                   int b, int I, bool outI, int J0, int J1, int lane, double* wring) {
  const int m = g.m, n0 = g.n0, mc = gc.m;
  const int xa = 2 * I, x0 = xa - 2 * lane;
  const int64_t off = (int64_t)b * g.N;
  const double* rb = r + off;
  const float *eb = e0 + off, *nb = n0e + off;
  const int ys = 2 * J0 - 1;
  const int ylast = 2 * J1 + 1;  // ingest rows end at 2J1+1
  auto slot = [&](int q) { return wring + (size_t)((unsigned)(q - (ys - 3)) % L0R_RING) * (RR_W * L0R_WORDS_DN); };
  auto issue = [&](int q) {
    if (q <= ylast) l0_issue_kr(slot(q), eb, nb, rb, x0, lane, q, n0);
    cpa_commit();
  };
  for (int j = 0; j < L0R_RING; ++j) issue(ys - 3 + j);
  const Pair zero{0.0, 0.0};
  Pair N1, E1 = zero, N2 = zero, E2 = zero, N3 = zero;
  double zr2 = 0.0, zr1 = 0.0, rbl1 = 0.0;
  Sten sb1{1.0, 0.0, 0.0, 0.0, 0.0};
  Pair zp3 = zero, zp2 = zero;
  cpa_wait<2>();  // rows ys−3 … ys−1
  __syncwarp();
  {
    Pair Ed;
    l0_edges(slot(ys - 3), lane, Ed, N1);  // row ys−3: its N only
  }
  auto ingest = [&](int q) {
    cpa_wait<2>();  // rows ≤ q+1
    __syncwarp();
    Pair E, N;
    l0_edges(slot(q), lane, E, N);
    const Pair r0 = l0_pair(slot(q), L0R_R, lane);
    __syncwarp();
    issue(q + 4);  // into the slot of row q−1
    const Sten2 st = sten_pair<INT>(E, N, N1, xa, q, m, bc);
    const bool ra = RED_IS_A(q);
    const double zr0 = (ra ? r0.a : r0.b) * rcp64s(ra ? st.a.d : st.b.d);
    const bool ra1 = !ra;
    const double zr1_e = shdn(zr1), zr1_w = shup(zr1);
    const double zbl = (rbl1 - (sb1.e * (ra1 ? zr1_e : zr1) + sb1.w * (ra1 ? zr1 : zr1_w) + sb1.n * zr0 +
                                sb1.s * zr2)) * rcp64s(sb1.d);
    const Pair zp1 = ra1 ? Pair{zr1, zbl} : Pair{zbl, zr1};
    const double t = ra ? red_resid<INT, true>(E2, N2, N3, zp3, zp2, zp1, xa, q - 2, m, bc)
                        : red_resid<INT, false>(E2, N2, N3, zp3, zp2, zp1, xa, q - 2, m, bc);
    N3 = N2; E2 = E1; N2 = N1; E1 = E; N1 = N;
    zr2 = zr1; zr1 = zr0;
    sb1 = ra ? st.b : st.a;
    rbl1 = ra ? r0.b : r0.a;
    zp3 = zp2; zp2 = zp1;
    return t;
  };
  ingest(ys - 2);
  ingest(ys - 1);
  ingest(ys);
  ingest(ys + 1);
  const int mcl = m / 2;
  const int64_t cb0 = (int64_t)b * mcl * mcl;
  // fp32 weights stay fp32 in registers until their use (a conversion right after the load would
  // wait on it there and expose the load latency the row-pair prefetch is meant to hide)
  auto W4 = [&](int Jc, float w[4]) {
    const bool ok = I >= 0 && I < mcl && Jc >= 0 && Jc < mcl;
    const int64_t cell = cb0 + (int64_t)Jc * mcl + I;
    w[0] = ok ? __ldg(pw.w0 + cell) : 0.0f;
    w[1] = ok ? __ldg(pw.w1 + cell) : 0.0f;
    w[2] = ok ? __ldg(pw.w2 + cell) : 0.0f;
    w[3] = ok ? __ldg(pw.w3 + cell) : 0.0f;
  };
  float wc[4], wn[4];
  W4(J0 - 1, wc);
  W4(J0, wn);
  const double t_first = ingest(ys + 2);  // (xb, 2J0−1)
  double a_nw = t_first * wc[2], a_ne = t_first * wc[3];
  double* rcb = rc + (int64_t)b * gc.N;
  for (int J = J0; J < J1; ++J) {
    wc[0] = wn[0]; wc[1] = wn[1]; wc[2] = wn[2]; wc[3] = wn[3];
    W4(J + 1, wn);
    const double t_even = ingest(2 * J + 2);  // (xa, 2J)
    const double t = ingest(2 * J + 3);       // (xb, 2J+1)
    const double a_sw = t * wc[0], a_se = t * wc[1];
    const double v = t_even + a_sw + shup(a_se) + a_nw + shup(a_ne);
    if (outI) rcb[(int64_t)J * gc.n0 + I] = is_dir(bc, mc, I, J) ? 0.0 : v;
    a_nw = t * wc[2];
    a_ne = t * wc[3];
  }
  cpa_wait<0>();
}

__global__ void __launch_bounds__(32 * RR_W, 4 * 4 / RR_W) restrict_ring_kernel(Geo g, Geo gc, int bc, const float* __restrict__ e0,
                                                              const float* __restrict__ n0e,
                                                              const double* __restrict__ r, PW4 pw,
                                                              double* __restrict__ rc, const int* flags) {
  const int b = blockIdx.z;
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;
  extern __shared__ __align__(16) double l0ring[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = blockIdx.x * RR_W + warp;
  const int I = strip * 30 - 1 + lane;
  const bool outI = lane >= 1 && lane < 31 && I <= gc.m;
  const int lyc = coarse_rows_per_warp(gc.m);
  const int J0 = blockIdx.y * lyc, J1 = min(J0 + lyc, gc.n0);
  const bool interior = strip * 60 - 2 >= 2 && strip * 60 + 61 <= g.m - 2 && 2 * J0 - 6 >= 1 &&
                        2 * J1 + 4 <= g.m - 1;
  double* wring = l0ring + warp * L0R_WORDS_DN;
  if (interior) restrict_ring_body<true>(g, gc, bc, e0, n0e, r, pw, rc, b, I, outI, J0, J1, lane, wring);
  else restrict_ring_body<false>(g, gc, bc, e0, n0e, r, pw, rc, b, I, outI, J0, J1, lane, wring);
}

template <bool INT>
__device__ __forceinline__ double2 smooth_up_ring_body(Geo g, Geo gc, int bc, const float* __restrict__ e0,
                                                       const float* __restrict__ n0e,
                                                       const double* __restrict__ r, z_t* __restrict__ z_out,
                                                       const double* __restrict__ zc, PW4 pw, const PairCtx& c,
                                                       double* wring) {
  PAIR_UNPACK

  const int lane = c.lane, x0 = xa - 2 * lane;
  const double *rb = r + off, *zcb = zc + (int64_t)b * gc.N;
  const float *eb = e0 + off, *nb = n0e + off;
  const int nc0 = gc.n0;
  const int I0 = x0 >> 1;
  const int mcl = m / 2;
  const int64_t cb0 = (int64_t)b * mcl * mcl;
  const int ylast = y1 + 2;
  auto slot = [&](int q) { return wring + (size_t)((unsigned)(q - (y0 - 3)) % L0R_RING) * (SUR_W * L0R_WORDS_UP); };
  auto issue = [&](int q) {
    if (q <= ylast) {
      double* S = slot(q);
      l0_issue_kr(S, eb, nb, rb, x0, lane, q, n0);
      // prolongation inputs of row q's red node: z₁ rows q>>1 (and +1 on odd rows), columns
      // I0 … I0+32; centre weights of the odd rows' cells
      const int Jc = q >> 1, ci = I0 + lane;
      const bool cok = (unsigned)ci < (unsigned)nc0, cok2 = (unsigned)(ci + 32) < (unsigned)nc0;
      const bool j0 = (unsigned)Jc < (unsigned)nc0, j1 = (unsigned)(Jc + 1) < (unsigned)nc0;
      const double* zr0 = zcb + (int64_t)Jc * nc0 + ci;
      cpa8(S + L0R_ZC0 + lane, zr0, j0 && cok);
      if (lane == 0) cpa8(S + L0R_ZC0 + 32, zr0 + 32, j0 && cok2);
      if (q & 1) {
        cpa8(S + L0R_ZC1 + lane, zr0 + nc0, j1 && cok);
        if (lane == 0) cpa8(S + L0R_ZC1 + 32, zr0 + nc0 + 32, j1 && cok2);
        const bool ok = ci >= 0 && ci < mcl && Jc >= 0 && Jc < mcl;
        const int64_t cell = cb0 + (int64_t)Jc * mcl + ci;
        float* SP = reinterpret_cast<float*>(S + L0R_PW);
        cpa4(SP + 0 * 32 + lane, pw.w0 + cell, ok);
        cpa4(SP + 1 * 32 + lane, pw.w1 + cell, ok);
        cpa4(SP + 2 * 32 + lane, pw.w2 + cell, ok);
        cpa4(SP + 3 * 32 + lane, pw.w3 + cell, ok);
      }
    }
    cpa_commit();
  };
  // red value of row y after prolongation: z_red = r/D (pre-smoother from 0) + P z₁
  auto RV = [&](const double* S, int y, Pair rr, Pair E, Pair N, Pair Nm) {
    const double Wa = shup(E.b);
    if (RED_IS_A(y)) {
      const Sten s = mk_sten<INT>(E.a, Wa, N.a, Nm.a, xa, y, m, bc);
      const double c00 = (INT || (unsigned)xa < (unsigned)n0) ? S[L0R_ZC0 + lane] : 0.0;
      return rr.a * rcp64s(s.d) + c00;
    }
    const Sten s = mk_sten<INT>(E.b, E.a, N.b, Nm.b, xb, y, m, bc);
    double p = 0.0;
    if (INT || (unsigned)xb < (unsigned)n0)
      p = l0r_pw(S, lane, 0) * S[L0R_ZC0 + lane] + l0r_pw(S, lane, 1) * S[L0R_ZC0 + lane + 1] +
          l0r_pw(S, lane, 2) * S[L0R_ZC1 + lane] + l0r_pw(S, lane, 3) * S[L0R_ZC1 + lane + 1];
    return rr.b * rcp64s(s.d) + p;
  };
  for (int j = 0; j < L0R_RING; ++j) issue(y0 - 3 + j);  // rows y0−3 … y0+1
  const Pair zero{0.0, 0.0};
  cpa_wait<1>();  // rows y0−3 … y0
  __syncwarp();
  Pair Ed, N3, E2, N2, E1, N1;
  l0_edges(slot(y0 - 3), lane, Ed, N3);
  l0_edges(slot(y0 - 2), lane, E2, N2);
  l0_edges(slot(y0 - 1), lane, E1, N1);
  double qa = RV(slot(y0 - 2), y0 - 2, l0_pair(slot(y0 - 2), L0R_R, lane), E2, N2, N3);
  double qb = RV(slot(y0 - 1), y0 - 1, l0_pair(slot(y0 - 1), L0R_R, lane), E1, N1, N2);
  __syncwarp();
  issue(y0 + 2);  // into the slot of row y0−3 (rows y0−2 … are still read by the loop)
  Pair Nt = N2;
  double zbm = 0.0, zb0 = 0.0;
  Sten sr0{1.0, 0.0, 0.0, 0.0, 0.0};  // stencil of row t's red column
  double rz = 0.0, dc = 0.0;
  // one output row; RA1 = red at column a in row t+1 (static: the loop is unrolled by 2, y0 even)
  auto step = [&](auto RA1, int t) {
    constexpr bool ra1 = decltype(RA1)::value, ra0 = !ra1;
    // rows t … t+3 resident (row t+4 may be in flight)
    cpa_wait<1>();
    __syncwarp();
    const double *S0 = slot(t), *S1 = slot(t + 1), *S2 = slot(t + 2), *S3 = slot(t + 3);
    Pair E2n, N2n;
    l0_edges(S2, lane, E2n, N2n);
    const Pair r0 = l0_pair(S0, L0R_R, lane), r1 = l0_pair(S1, L0R_R, lane);
    // red value of row t+2 (red column a iff row t+2 is even, i.e. as row t)
    double qc;
    {
      const Pair rr = l0_pair(S2, L0R_R, lane);
      const double Wa = shup(E2n.b);
      if constexpr (ra0) {
        const Sten sq = mk_sten<INT>(E2n.a, Wa, N2n.a, N1.a, xa, t + 2, m, bc);
        const double c00 = (INT || (unsigned)xa < (unsigned)n0) ? S2[L0R_ZC0 + lane] : 0.0;
        qc = rr.a * rcp64s(sq.d) + c00;
      } else {
        const Sten sq = mk_sten<INT>(E2n.b, E2n.a, N2n.b, N1.b, xb, t + 2, m, bc);
        double pz = 0.0;
        if (INT || (unsigned)xb < (unsigned)n0)
          pz = l0r_pw(S2, lane, 0) * S2[L0R_ZC0 + lane] + l0r_pw(S2, lane, 1) * S2[L0R_ZC0 + lane + 1] +
               l0r_pw(S2, lane, 2) * S2[L0R_ZC1 + lane] + l0r_pw(S2, lane, 3) * S2[L0R_ZC1 + lane + 1];
        qc = rr.b * rcp64s(sq.d) + pz;
      }
    }
    __syncwarp();
    issue(t + 5);  // into the slot of row t
    const Sten2 st1 = sten_pair<INT>(E1, N1, Nt, xa, t + 1, m, bc);
    const double qb_e = shdn(qb), qb_w = shup(qb);
    const Sten& sb = ra1 ? st1.b : st1.a;
    const double odb = sb.e * (ra1 ? qb_e : qb) + sb.w * (ra1 ? qb : qb_w) + sb.n * qc + sb.s * qa;
    const double zbp1 = ((ra1 ? r1.b : r1.a) - odb) * rcp64s(sb.d);
    const double zb0_e = shdn(zb0), zb0_w = shup(zb0);
    const double s2 = sr0.e * (ra0 ? zb0 : zb0_e) + sr0.w * (ra0 ? zb0_w : zb0) + sr0.n * zbp1 + sr0.s * zbm;
    const double zred = ((ra0 ? r0.a : r0.b) - s2) * rcp64s(sr0.d);
    if (t >= y0) {
      z_t* out = z_out + off + (int64_t)t * n0;
      const double va = ra0 ? zred : zb0, vb = ra0 ? zb0 : zred;
      if (outa) {
        out[xa] = (z_t)va;
        rz = fma(r0.a, va, rz);
      }
      if (outb) {
        out[xb] = (z_t)vb;
        rz = fma(r0.b, vb, rz);
      }
      if (ra0 ? outa : outb) dc = fma(zred - qa, s2, dc);
    }
    qa = qb; qb = qc; Nt = N1; E1 = E2n; N1 = N2n;
    zbm = zb0; zb0 = zbp1;
    sr0 = ra1 ? st1.a : st1.b;
  };
  for (int t = y0 - 2; t < y1; t += 2) {
    step(std::false_type{}, t);
    if (t + 1 < y1) step(std::true_type{}, t + 1);
  }
  cpa_wait<0>();
  return make_double2(rz, dc);
}

// 16 one-warp CTAs per SM (128 registers, no spills): the sweep is bound by dependent fp64 latency at
// 60% issue with 12 warps per SM; 16 gave 3.68 → 3.98 TB/s at 2048² and 3.13 → 3.26 at 1024²
// (profiles/ab_r2/ring_occupancy.txt; 20 CTAs for the restriction spill and lose)
__global__ void __launch_bounds__(32 * SUR_W, 4 * 4 / SUR_W) smooth_up_ring_kernel(Geo g, Geo gc, int bc, const float* __restrict__ e0,
                                                               const float* __restrict__ n0e,
                                                               const double* __restrict__ r,
                                                               z_t* __restrict__ z_out,
                                                               const double* __restrict__ zc, PW4 pw, double* scal,
                                                               int* flags, double2* partial, int maxp,
                                                               unsigned* counter) {
  PAIR_PROLOGUE_W(SUR_W)
  extern __shared__ __align__(16) double l0ring[];
  double* wring = l0ring + (threadIdx.x >> 5) * L0R_WORDS_UP;
  const bool interior3 = interior && c.y1 <= g.m - 3;
  const double2 gd = interior3 ? smooth_up_ring_body<true>(g, gc, bc, e0, n0e, r, z_out, zc, pw, c, wring)
                               : smooth_up_ring_body<false>(g, gc, bc, e0, n0e, r, z_out, zc, pw, c, wring);
  double gamma, dcorr;
  if (reduce2_last(gd.x, gd.y, partial, maxp, counter, b, gamma, dcorr) && threadIdx.x == 0) {
    const double delta = gamma + dcorr;
    const bool first = flags[b * F_NFLAGS + F_ITERS] == 0;
    double beta = first ? 0.0 : gamma / scal[b * S_NSCAL + S_RZ];
    double den = first ? delta : delta - beta * gamma / scal[b * S_NSCAL + S_ALPHA];
    // ⟨p, Ap⟩ = δ − βγ/α_old lies in (0, δ] in exact arithmetic; outside it the recurrence has lost
    // the conjugacy it relies on: restart the direction (p = z, β = 0, α = γ/δ)
    if (!(den > 0.0 && den <= delta * (1.0 + 1e-8))) {
      den = delta;
      beta = 0.0;
    }
    scal[b * S_NSCAL + S_BETA] = beta;
    scal[b * S_NSCAL + S_ALPHA] = gamma / den;
    scal[b * S_NSCAL + S_RZ] = gamma;
  }
}

// device view of the global hierarchy (one level's operator and centre weights)
struct SolverLevelDev {
  const double* C;
  const float *E, *N, *NE, *NW;
  const float* pw[4];
};
struct HierDev {
  SolverLevelDev lev[12];
};

// ---- CTA-resident multigrid (small grids and the V-cycle tail) ----------------------------------------
// One CTA owns one sample; every level's operator, transfer weights and r, z, t live in shared memory.
// Level 0 of the small solver is the 5-point P1 row from k in fp64 (it is the PCG operator); the
// 9-point levels keep the fp32 couplings they are stored with. The V-cycle is the multi-kernel one:
//   - pre-smoother red → black from z = 0;
//   - residual t = r − A z, restricted with Pᵀ;
//   - recursion, then z += P z_c;
//   - post-smoother black → red, into t.
// Each level's output is in its t. These kernels are bound by instruction issue, barriers and
// dependent-latency chains, not by bandwidth (ncu: 1 % of DRAM), so:
//   * everything an iteration would recompute is formed once per solve — the reciprocal diagonals and
//     the edge-node transfer weights (fp32; restriction and prolongation read the same stored value,
//     so the cycle stays symmetric);
//   * the stencil sums are branch-free: every array is preceded (and each level followed) by n0 + 1
//     zeros and the couplings that point outside the grid are stored as exact zeros, so a node reads
//     its eight neighbours unconditionally (a row end reads the neighbouring row's end node through
//     a zero coupling) and never needs its (x, y);
//   * m is even on every level with a coarser one, so n0 is odd and node i is red exactly when i is
//     even: the coloured sweeps run over packed indices;
//   * the red pre-sweep is folded into the black one (z starts at 0, a black node's red neighbours
//     are r/C); a thread owns at most SM_KMAX nodes per level (u of the PCG stays in registers);
//     reductions cost one barrier; the CTA is sized to the grid (7 CTAs per SM at 16², 2 at 32²).
constexpr int SM_KMAX = 3;
constexpr int SM_CSPLIT = 4;  // threads per row of the coarsest solve

struct SLev {
  double *C, *iC;              // diagonal and its reciprocal
  double *E, *N;               // 5-point level 0 of the small solver: fp64 couplings; null on 9-point levels
  float *Ef, *Nf, *NEf, *NWf;  // 9-point levels: couplings as stored
  float *w0, *w1;              // edge nodes: weights to the lower / upper coarse parent
  float* pw[4];                // centre weights of this level's cells
  double *r, *z, *t;
  int m, n0, N_;
  float inv_n0;
};

__device__ __forceinline__ void node_xy(const SLev& L, int i, int& x, int& y) {
  y = __float2int_rz(((float)i + 0.5f) * L.inv_n0);  // exact for the ≤ 33² nodes of these levels
  x = i - y * L.n0;
}

// body(i) for the nodes i < N owned by this thread (i = tid + k·T, k < SM_KMAX; SM_KMAX·T ≥ N)
// (a rolled loop: these kernels are instruction-cache bound — ncu: 33 % of the stall samples were
// "no instruction" with the three-fold unrolled bodies — so code size counts more than loop overhead)
template <class F>
__device__ __forceinline__ void for_nodes(int N, F&& body) {
#pragma unroll 1
  for (int i = threadIdx.x; i < N; i += blockDim.x) body(i);
}
// unrolled variant for the global-memory loads (their latencies overlap across the thread's nodes)
template <class F>
__device__ __forceinline__ void for_nodes_unrolled(int N, F&& body) {
#pragma unroll
  for (int k = 0; k < SM_KMAX; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < N) body(i);
  }
}

// Σ of node i's off-diagonal couplings times v (axis neighbours from va, diagonal ones from vd).
// W, S, SW, SE are the neighbours' E, N, NE, NW. No bounds tests: zero pads and zero outward couplings.
__device__ __forceinline__ double offdiag(const SLev& L, const double* va, const double* vd, int i) {
  const int n0 = L.n0;
  if (L.E) return L.E[i - 1] * va[i - 1] + L.E[i] * va[i + 1] + L.N[i - n0] * va[i - n0] + L.N[i] * va[i + n0];
  double s = L.Ef[i - 1] * va[i - 1] + L.Ef[i] * va[i + 1] + L.Nf[i - n0] * va[i - n0] + L.Nf[i] * va[i + n0];
  s += L.NEf[i - n0 - 1] * vd[i - n0 - 1] + L.NWf[i - n0 + 1] * vd[i - n0 + 1];
  s += L.NWf[i] * vd[i + n0 - 1] + L.NEf[i] * vd[i + n0 + 1];
  return s;
}

// the full row (setup only: transfer weights)
__device__ __forceinline__ S9 row_smem(const SLev& L, int i) {
  S9 r{0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int n0 = L.n0;
  r.c = L.C[i];
  if (L.E) {
    r.e = L.E[i];
    r.n = L.N[i];
    r.w = L.E[i - 1];
    r.s = L.N[i - n0];
  } else {
    r.e = L.Ef[i];
    r.n = L.Nf[i];
    r.ne = L.NEf[i];
    r.nw = L.NWf[i];
    r.w = L.Ef[i - 1];
    r.s = L.Nf[i - n0];
    r.sw = L.NEf[i - n0 - 1];
    r.se = L.NWf[i - n0 + 1];
  }
  return r;
}

// Block sum with one barrier: warp sums → sh[parity][warp] → every thread adds them in warp order
// (deterministic). Consecutive calls alternate the buffer, so no second barrier is needed.
struct BlockSum {
  double (*sh)[32];
  int parity = 0;
  __device__ double operator()(double v) {
    v = warp_sum(v);
    double* s = sh[parity];
    parity ^= 1;
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += s[w];
    return t;
  }
};

// reciprocal diagonals and edge-node transfer weights of levels 0 … nlev−2 (once per solve / call)
__device__ void prepare_levels(const SLev* lev, int nlev, int bc, int opdep) {
  for (int l = 0; l + 1 < nlev; ++l) {
    const SLev& F = lev[l];
    for_nodes(F.N_, [&](int i) {
      int x, y;
      node_xy(F, i, x, y);
      F.iC[i] = rcp64(F.C[i]);
      const bool ox = x & 1, oy = y & 1;
      if (ox == oy) return;
      double a0, a1;
      edge_w(row_smem(F, i), ox, opdep != 0, is_dir(bc, F.m, x, y), false, false, a0, a1);
      F.w0[i] = (float)a0;
      F.w1[i] = (float)a1;
    });
  }
  __syncthreads();
}

// V(1,1) on levels 0..nlev−1 of `lev`: input lev[0].r, output lev[0].t
__device__ void vcycle_smem(const SLev* lev, int nlev, const double* Ainv, int bc) {
  for (int l = 0; l + 1 < nlev; ++l) {
    const SLev& F = lev[l];
    const int n0 = F.n0, m = F.m;
    const int n_red = (F.N_ + 1) / 2, n_black = F.N_ / 2;
    const bool five = F.E != nullptr;
    // red z = r/C; black z = (r − Σ_axis a·z_red)/C with the red neighbours formed in place
    for_nodes(n_red, [&](int j) { F.z[2 * j] = F.r[2 * j] * F.iC[2 * j]; });
    for_nodes(n_black, [&](int j) {
      const int i = 2 * j + 1;
      double s;
      if (five)
        s = F.E[i - 1] * (F.r[i - 1] * F.iC[i - 1]) + F.E[i] * (F.r[i + 1] * F.iC[i + 1]) +
            F.N[i - n0] * (F.r[i - n0] * F.iC[i - n0]) + F.N[i] * (F.r[i + n0] * F.iC[i + n0]);
      else
        s = F.Ef[i - 1] * (F.r[i - 1] * F.iC[i - 1]) + F.Ef[i] * (F.r[i + 1] * F.iC[i + 1]) +
            F.Nf[i - n0] * (F.r[i - n0] * F.iC[i - n0]) + F.Nf[i] * (F.r[i + n0] * F.iC[i + n0]);
      F.z[i] = (F.r[i] - s) * F.iC[i];
    });
    __syncthreads();
    // residual t = r − A z. On a 5-point level the black rows were just solved exactly (their
    // neighbours are all red), so their residual is rounding noise: only the red rows are formed and
    // the restriction below leaves the black (edge-node) terms out.
    if (five)
      for_nodes(n_red, [&](int j) {
        const int i = 2 * j;
        F.t[i] = F.r[i] - (F.C[i] * F.z[i] + offdiag(F, F.z, F.z, i));
      });
    else
      for_nodes(F.N_, [&](int i) { F.t[i] = F.r[i] - (F.C[i] * F.z[i] + offdiag(F, F.z, F.z, i)); });
    __syncthreads();
    const SLev& C = lev[l + 1];
    const int mcl = m / 2;
    for_nodes(C.N_, [&](int ic) {
      int I, J;
      node_xy(C, ic, I, J);
      double acc = 0.0;
      if (!is_dir(bc, C.m, I, J)) {
        const int x = 2 * I, y = 2 * J, i = y * n0 + x;
        acc = F.t[i];
        if (!five) {
          if (x < m) acc += F.w0[i + 1] * F.t[i + 1];
          if (x > 0) acc += F.w1[i - 1] * F.t[i - 1];
          if (y < m) acc += F.w0[i + n0] * F.t[i + n0];
          if (y > 0) acc += F.w1[i - n0] * F.t[i - n0];
        }
        if (I < mcl && J < mcl) acc += F.pw[0][J * mcl + I] * F.t[i + n0 + 1];
        if (I > 0 && J < mcl) acc += F.pw[1][J * mcl + I - 1] * F.t[i + n0 - 1];
        if (I < mcl && J > 0) acc += F.pw[2][(J - 1) * mcl + I] * F.t[i - n0 + 1];
        if (I > 0 && J > 0) acc += F.pw[3][(J - 1) * mcl + I - 1] * F.t[i - n0 - 1];
      }
      C.r[ic] = acc;
    });
    __syncthreads();
  }
  {  // coarsest: t = A⁻¹ r. Every other warp waits for this solve, so its dependent chain is kept short
     // without spending a warp per row: SM_CSPLIT threads per row each sum every SM_CSPLIT-th column
     // (A⁻¹ is symmetric: read by columns, coalesced over the rows; it stays in global memory,
     // L1/L2-resident), the partial sums meet in shared memory.
    const SLev& C = lev[nlev - 1];
    const int nc = C.N_;
    double* part = C.z;  // SM_CSPLIT × nc
    for (int idx = threadIdx.x; idx < SM_CSPLIT * nc; idx += blockDim.x) {
      const int p = idx / nc, i = idx - p * nc;
      double v = 0.0;
      for (int j = p; j < nc; j += SM_CSPLIT) v = fma(__ldg(Ainv + j * nc + i), C.r[j], v);
      part[idx] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      double v = part[i];
#pragma unroll
      for (int p = 1; p < SM_CSPLIT; ++p) v += part[p * nc + i];
      C.t[i] = v;
    }
    __syncthreads();
  }
  for (int l = nlev - 2; l >= 0; --l) {
    const SLev& F = lev[l];
    const SLev& C = lev[l + 1];
    const int mcl = F.m / 2, cn0 = C.n0;
    for_nodes(F.N_, [&](int i) {
      int x, y;
      node_xy(F, i, x, y);
      const int ox = x & 1, oy = y & 1;
      const double* zc = C.t + (y >> 1) * cn0 + (x >> 1);
      double v;
      if (!ox && !oy) {
        v = zc[0];
      } else if (ox && oy) {
        const int cell = (y >> 1) * mcl + (x >> 1);
        v = F.pw[0][cell] * zc[0] + F.pw[1][cell] * zc[1] + F.pw[2][cell] * zc[cn0] + F.pw[3][cell] * zc[cn0 + 1];
      } else {
        v = F.w0[i] * zc[0] + F.w1[i] * zc[ox ? 1 : cn0];
      }
      F.z[i] += v;
    });
    __syncthreads();
    for_nodes(F.N_ / 2, [&](int j) {  // black (odd i): reads z, writes t
      const int i = 2 * j + 1;
      F.t[i] = (F.r[i] - offdiag(F, F.z, F.z, i)) * F.iC[i];
    });
    __syncthreads();
    for_nodes((F.N_ + 1) / 2, [&](int j) {  // red (even i): new black (t) on the axes, old red (z) on the diagonals
      const int i = 2 * j;
      F.t[i] = (F.r[i] - offdiag(F, F.t, F.z, i)) * F.iC[i];
    });
    __syncthreads();
  }
}

// Shared-memory layout of a hierarchy m_top, m_top/2, … (nlev levels); level 0 is 5-point fp64 when
// five_point0. All fp64 arrays first, then the fp32 ones; every array has a zero pad of n0 + 1
// entries in front, every level one behind its last array (the zero-pad / zero-coupling contract of
// offdiag). The coarsest level only holds r, t (its solve is the precomputed inverse).
__host__ __device__ inline void level_counts(int g, bool last, bool p5, int& n64, int& n32) {
  const int N = (g + 1) * (g + 1), mcl = g / 2, pad = g + 2;
  const int a64 = last ? 2 : (p5 ? 7 : 5);      // r, t | z, C, iC | E, N
  const int a32 = last ? 0 : (p5 ? 2 : 6);      // E, N, NE, NW | w0, w1
  n64 = a64 * (N + pad) + pad + (last ? SM_CSPLIT * N : 0);     // + the coarsest solve's partial sums
  n32 = last ? 0 : a32 * (N + pad) + pad + 4 * mcl * mcl;  // + pw
}
__host__ __device__ inline void hier_counts(int m_top, int nlev, bool five_point0, size_t& n64, size_t& n32) {
  n64 = n32 = 0;
  int g = m_top;
  for (int l = 0; l < nlev; ++l, g /= 2) {
    int a, b;
    level_counts(g, l + 1 == nlev, l == 0 && five_point0, a, b);
    n64 += (size_t)a;
    n32 += (size_t)b;
  }
}

// Carve the hierarchy from (zeroed) shared memory: thread 0 fills the level structs (shared), every
// thread gets the first free address.
__device__ double* carve_levels(SLev* lev, double* base, int m_top, int nlev, bool five_point0) {
  size_t n64, n32;
  hier_counts(m_top, nlev, five_point0, n64, n32);
  if (threadIdx.x == 0) {
    double* c64 = base;
    float* c32 = reinterpret_cast<float*>(base + n64);
    int g = m_top;
    for (int l = 0; l < nlev; ++l, g /= 2) {
      const int N = (g + 1) * (g + 1), mcl = g / 2, pad = g + 2;
      auto d = [&] { double* p = c64 + pad; c64 += pad + N; return p; };
      auto f = [&] { float* p = c32 + pad; c32 += pad + N; return p; };
      SLev L{};
      L.m = g;
      L.n0 = g + 1;
      L.N_ = N;
      L.inv_n0 = 1.0f / (float)(g + 1);
      L.r = d();
      L.t = d();
      if (l + 1 == nlev) {
        L.z = c64;  // partial sums of the coarsest solve (SM_CSPLIT × N)
        c64 += SM_CSPLIT * N;
      }
      if (l + 1 < nlev) {
        L.z = d();
        L.C = d();
        L.iC = d();
        if (l == 0 && five_point0) {
          L.E = d();
          L.N = d();
        } else {
          L.Ef = f();
          L.Nf = f();
          L.NEf = f();
          L.NWf = f();
        }
        L.w0 = f();
        L.w1 = f();
        c32 += pad;
        for (int q = 0; q < 4; ++q) {
          L.pw[q] = c32;
          c32 += mcl * mcl;
        }
      }
      c64 += pad;
      lev[l] = L;
    }
  }
  __syncthreads();
  return base + n64 + (n32 + 1) / 2;
}

size_t hier_smem_bytes(int m_top, int nlev, bool five_point0) {
  size_t n64, n32;
  hier_counts(m_top, nlev, five_point0, n64, n32);
  return sizeof(double) * (n64 + (n32 + 1) / 2);
}

constexpr size_t kMaxCtaSmem = 227 * 1024 - 2048;  // dynamic shared memory a CTA-resident hierarchy may take

// threads per CTA: the smallest warp multiple with SM_KMAX·T ≥ (m+1)²
inline int small_threads(int m) {
  const int N = (m + 1) * (m + 1);
  const int t = ((N + SM_KMAX - 1) / SM_KMAX + 31) / 32 * 32;
  return std::min(std::max(t, 64), 1024);
}

__device__ __forceinline__ void zero_smem(double* smem, int n_doubles) {
  for (int i = threadIdx.x; i < n_doubles; i += blockDim.x) smem[i] = 0.0;
  __syncthreads();
}

// Load a stored 9-point level (operator + centre weights) of sample b into shared memory; couplings
// that point outside the grid are stored as zeros (offdiag's contract).
__device__ void load_level(const SLev& L, const SolverLevelDev& G, int b, bool has_coarse) {
  if (!has_coarse) return;  // the coarsest level is solved by its inverse
  const int64_t off = (int64_t)b * L.N_;
  for_nodes_unrolled(L.N_, [&](int i) {
    int x, y;
    node_xy(L, i, x, y);
    const bool xm = x == L.m, ym = y == L.m;
    L.C[i] = __ldg(G.C + off + i);
    L.Ef[i] = xm ? 0.f : __ldg(G.E + off + i);
    L.Nf[i] = ym ? 0.f : __ldg(G.N + off + i);
    L.NEf[i] = (xm || ym) ? 0.f : __ldg(G.NE + off + i);
    L.NWf[i] = (x == 0 || ym) ? 0.f : __ldg(G.NW + off + i);
  });
  const int mcl = L.m / 2;
  const int64_t co = (int64_t)b * mcl * mcl;
  for_nodes_unrolled(mcl * mcl, [&](int i) {
#pragma unroll
    for (int q = 0; q < 4; ++q) L.pw[q][i] = __ldg(G.pw[q] + co + i);
  });
}

// Whole PCG of one sample per CTA (m ≤ 32): level 0 from k, coarse levels + transfers + coarsest
// inverse from the global setup (prow / rap / factor kernels), the same algorithm and stopping
// rule as the multi-kernel path, one launch per batch.
__global__ void __launch_bounds__(1024) small_pcg_kernel(int m0, int nlev, int bc, int opdep, int forcing,
                                                         double fval, double tol, int max_iter_factor,
                                                         const double* __restrict__ kin, HierDev H,
                                                         const double* __restrict__ chol,
                                                         double* __restrict__ uout, int* flags,
                                                         double* scal, int smem_doubles) {
  extern __shared__ double smem[];
  __shared__ double sum_sh[2][32];
  __shared__ SLev lev[6];  // m ≤ 32: at most 32, 16, 8, 4 (or an odd tail)
  BlockSum bsum{sum_sh};
  const int b = blockIdx.x;
  const int N0 = (m0 + 1) * (m0 + 1);
  const double* k0 = kin + (int64_t)b * N0;
  zero_smem(smem, smem_doubles);
  double* p = smem + m0 + 2;  // padded like the level arrays (its back pad is the first level array's front pad)
  carve_levels(lev, p + N0, m0, nlev, true);
  const SLev& L0 = lev[0];
  const int m = m0;
  for_nodes(N0, [&](int i) {  // level-0 5-point rows from k (outward and eliminated couplings are zeros)
    int x, y;
    node_xy(L0, i, x, y);
    const S9 a = row_k(k0, m + 1, 1, m, bc, x, y);
    L0.C[i] = a.c;
    L0.E[i] = a.e;
    L0.N[i] = a.n;
  });
  {
    const int mcl = m / 2;
    for_nodes_unrolled(mcl * mcl, [&](int i) {
#pragma unroll
      for (int q = 0; q < 4; ++q) L0.pw[q][i] = __ldg(H.lev[0].pw[q] + (int64_t)b * mcl * mcl + i);
    });
  }
  for (int l = 1; l < nlev; ++l) load_level(lev[l], H.lev[l], b, l + 1 < nlev);
  const int nc = lev[nlev - 1].N_;
  const double* Ainv = chol + (int64_t)b * 2 * nc * nc + (int64_t)nc * nc;
  __syncthreads();
  prepare_levels(lev, nlev, bc, opdep);
  // PCG init (fem.cpp:335-365): u = lift, r = b − A u; u of this thread's nodes stays in registers
  double ureg[SM_KMAX];
  double bb = 0.0, rr0 = 0.0;
#pragma unroll
  for (int k = 0; k < SM_KMAX; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    ureg[k] = 0.0;
    if (i >= N0) continue;
    int x, y;
    node_xy(L0, i, x, y);
    const double gs = (bc == OSC_BC_FLOWCELL && x == 0) ? 1.0 : 0.0;
    double bi;
    if (is_dir(bc, m, x, y)) {
      bi = gs;
      ureg[k] = gs;
      L0.r[i] = 0.0;
    } else {
      const int tri = 2 * (x < m && y < m) + (x > 0 && y < m) + 2 * (x > 0 && y > 0) + (x < m && y > 0);
      const double h = 1.0 / m;
      bi = forcing ? tri * (fval * (0.5 * h * h) / 3.0) : 0.0;
      if (bc == OSC_BC_FLOWCELL && x == 1) {  // raw coupling to u = 1 at x = 0 (fem.cpp:109-114)
        auto K = [&](int a0, int a1) { return __ldg(k0 + (int64_t)a1 * (m + 1) + a0); };
        const double e = -0.5 * ((y < m ? (K(0, y) + K(1, y) + K(1, y + 1)) / 3.0 : 0.0) +
                                 (y > 0 ? (K(0, y - 1) + K(1, y) + K(0, y)) / 3.0 : 0.0));
        bi -= e * 1.0;
      }
      L0.r[i] = bi;
      rr0 += bi * bi;
    }
    bb += bi * bi;
  }
  const double bnorm = sqrt(bsum(bb));
  double rel = sqrt(bsum(rr0)) / bnorm;
  int it = 0, status = 0;
  const int64_t cap64 = (int64_t)max_iter_factor * N0;
  const int cap = (int)(cap64 < 0x7fffffff ? cap64 : 0x7fffffff);
  if (rel > tol) {
    double rz = 1.0;
    for (;;) {  // one call site of the V-cycle (code size)
      vcycle_smem(lev, nlev, Ainv, bc);
      double rzn = 0.0;
      for_nodes(N0, [&](int i) { rzn += L0.r[i] * L0.t[i]; });
      rzn = bsum(rzn);
      const double beta = it == 0 ? 0.0 : rzn / rz;
      rz = rzn;
      for_nodes(N0, [&](int i) { p[i] = fma(beta, p[i], L0.t[i]); });
      __syncthreads();
      if (it >= cap) {
        status = OSC_ERR_SOLVER;
        break;
      }
      ++it;
      double ap[SM_KMAX];
      double pap = 0.0;
#pragma unroll
      for (int k = 0; k < SM_KMAX; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        ap[k] = 0.0;
        if (i >= N0) continue;
        ap[k] = L0.C[i] * p[i] + offdiag(L0, p, p, i);
        pap += p[i] * ap[k];
      }
      const double alpha = rz / bsum(pap);
      double rr = 0.0;
#pragma unroll
      for (int k = 0; k < SM_KMAX; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        if (i >= N0) continue;
        ureg[k] = fma(alpha, p[i], ureg[k]);
        const double rn = fma(-alpha, ap[k], L0.r[i]);
        L0.r[i] = rn;
        rr += rn * rn;
      }
      rel = sqrt(bsum(rr)) / bnorm;  // barrier: r complete
      if (rel <= tol) break;
      if (!isfinite(rel)) {
        status = OSC_ERR_SOLVER;
        break;
      }
    }
  }
  double* u = uout + (int64_t)b * N0;
#pragma unroll
  for (int k = 0; k < SM_KMAX; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < N0) u[i] = ureg[k];
  }
  if (threadIdx.x == 0) {
    flags[b * F_NFLAGS + F_ACTIVE] = 0;
    flags[b * F_NFLAGS + F_ITERS] = it;
    flags[b * F_NFLAGS + F_STATUS] = status;
    scal[b * S_NSCAL + S_REL] = rel;
    scal[b * S_NSCAL + S_BNORM] = bnorm;
  }
}

size_t small_smem_bytes(int m, int nlev) {
  return sizeof(double) * ((size_t)(m + 1) * (m + 1) + m + 2) + hier_smem_bytes(m, nlev, true);
}

// CTA-resident tail of the V-cycle (levels ls … nlev−1, m_ls ≤ 32) inside large solves: the
// coarsest levels are launch/latency-bound as separate kernels (≈ 20 µs each whatever their size).
__global__ void __launch_bounds__(1024) sub_vcycle_kernel(int m_ls, int nlev, int bc, int opdep, HierDev H,
                                                          const double* __restrict__ r_ls,
                                                          double* __restrict__ z_out,
                                                          const double* __restrict__ chol,
                                                          const int* flags, int smem_doubles) {
  extern __shared__ double smem[];
  __shared__ SLev lev[6];
  const int b = blockIdx.x;
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;
  const int N_ls = (m_ls + 1) * (m_ls + 1);
  zero_smem(smem, smem_doubles);
  carve_levels(lev, smem, m_ls, nlev, false);
  for (int l = 0; l < nlev; ++l) load_level(lev[l], H.lev[l], b, l + 1 < nlev);
  const int nc = lev[nlev - 1].N_;
  const double* Ainv = chol + (int64_t)b * 2 * nc * nc + (int64_t)nc * nc;
  const double* rb = r_ls + (int64_t)b * N_ls;
  for_nodes_unrolled(N_ls, [&](int i) { lev[0].r[i] = rb[i]; });
  __syncthreads();
  prepare_levels(lev, nlev, bc, opdep);
  vcycle_smem(lev, nlev, Ainv, bc);
  double* zb = z_out + (int64_t)b * N_ls;
  for_nodes(N_ls, [&](int i) { zb[i] = lev[0].t[i]; });
}

size_t sub_smem_bytes(int m_ls, int nlev) { return hier_smem_bytes(m_ls, nlev, false); }

__global__ void mark_active_failed_kernel(int B, int* flags) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B && flags[b * F_NFLAGS + F_ACTIVE]) {
    flags[b * F_NFLAGS + F_ACTIVE] = 0;
    flags[b * F_NFLAGS + F_STATUS] = OSC_ERR_SOLVER;
  }
}

// End of one body run of the device-side PCG loop (two iterations): keep looping while a sample of
// the batch is active; the optional hard cap (tests) stops the loop and fails the active samples.
__global__ void pcg_loop_cond_kernel(cudaGraphConditionalHandle h, const int* __restrict__ n_active,
                                     int* __restrict__ loop_runs, long hard_cap, int B, int* flags) {
  __shared__ int go;
  if (threadIdx.x == 0) {
    const int runs = ++loop_runs[0];
    go = n_active[0] > 0 ? 1 : 0;
    if (go && hard_cap >= 0 && 2L * runs >= hard_cap) go = -1;
  }
  __syncthreads();
  if (go < 0)
    for (int b = threadIdx.x; b < B; b += blockDim.x)
      if (flags[b * F_NFLAGS + F_ACTIVE]) {
        flags[b * F_NFLAGS + F_ACTIVE] = 0;
        flags[b * F_NFLAGS + F_STATUS] = OSC_ERR_SOLVER;
      }
  if (threadIdx.x == 0) cudaGraphSetConditional(h, go > 0 ? 1u : 0u);
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

// the running sums re-centred on shifts moved by (dy, dq): no sample is touched
__global__ void level_sums_reshift_kernel(double* sums, double dy, double dq) {
  const double n = sums[0], sy = sums[1], sq = sums[3];
  sums[2] = sums[2] - 2.0 * dy * sy + n * dy * dy;
  sums[1] = sy - n * dy;
  sums[4] = sums[4] - 2.0 * dq * sq + n * dq * dq;
  sums[3] = sq - n * dq;
}

inline int nblocks(int64_t N) { return (int)((N + NT - 1) / NT); }
inline int march_strips(int m) { return (m + 1 + 59) / 60; }  // 60 written columns per warp strip
inline dim3 march_grid(int m, int /*hx*/, int B) {
  const int ly = rows_per_warp(m);
  return dim3((unsigned)((march_strips(m) + MW - 1) / MW), (unsigned)((m + 1 + ly - 1) / ly), (unsigned)B);
}
inline dim3 restrict_grid_w(int mc, int B, int wpb) {
  const int lyc = coarse_rows_per_warp(mc);
  return dim3((unsigned)(((mc + 1 + 29) / 30 + wpb - 1) / wpb), (unsigned)((mc + 1 + lyc - 1) / lyc), (unsigned)B);
}
inline dim3 march_grid_w(int m, int B, int wpb) {
  const int ly = rows_per_warp(m);
  return dim3((unsigned)((march_strips(m) + wpb - 1) / wpb), (unsigned)((m + 1 + ly - 1) / ly), (unsigned)B);
}
inline int64_t tile_parts(int m) {
  const dim3 a = march_grid(m, 1, 1), b = march_grid(m, 2, 1), c = march_grid_w(m, 1, SUR_W),
             d = march_grid_w(m, 1, PU_W);
  return std::max<int64_t>(std::max<int64_t>((int64_t)a.x * a.y, (int64_t)b.x * b.y),
                           std::max<int64_t>((int64_t)c.x * c.y, (int64_t)d.x * d.y));
}

}  // namespace

size_t solver_bytes(int m, int B, int hist_cap) {
  size_t tot = 0;
  int g = m, lev = 0;
  for (;;) {
    const size_t N = (size_t)(g + 1) * (g + 1), mcl = g / 2;
    const bool last = g <= 4 || g % 2 != 0;
    // level 0: u r r2 z z2 p0 p1 (+k by caller); levels ≥ 1: C (fp64), E N NE NW (fp32), r z z2;
    // fp32 centre weights (4 per cell) on every level with a coarser one
    // level 0 also holds the two fp32 raw-edge arrays of the preconditioner sweeps
    tot += N * B * (lev == 0 ? 8 * sizeof(double) + 2 * sizeof(float) : 4 * sizeof(double) + 4 * sizeof(float)) +
           (last ? 0 : 4 * mcl * mcl * B * sizeof(float)) + 7 * 256;
    ++lev;
    if (last) {
      tot += (N > 1089 ? band_doubles(g + 1) : 2 * N * N) * B * sizeof(double);
      if (lev == 1) tot += N * B * (sizeof(double) + 4 * sizeof(float)) + 5 * 256;  // single level: its rows
      break;
    }
    g /= 2;
  }
  tot += (size_t)B * (S_NSCAL * 8 + F_NFLAGS * 4 + 8) + (size_t)B * hist_cap * 8;
  tot += (size_t)B * (tile_parts(m) + (size_t)(m + 1) * (m + 1) / NT + 2) * 16;
  return tot + 16384 * 16;
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
    if (g <= 4 || g % 2 != 0 || nl == 12) break;
    g /= 2;
  }
  w.nlev = nl;
  w.nc = (int)w.lev[nl - 1].N;
  OSC_REQUIRE(w.nc <= 1089 || w.lev[nl - 1].m <= kBandMaxM,
              "solve: coarsest multigrid grid too large (m must be 2^j * c, c <= 128)");
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
    const size_t vb = sizeof(double) * L.N * B, fb = sizeof(float) * L.N * B;
    L.k = nullptr;  // level 0's k is the caller's buffer
    const bool rows = l > 0 || nl == 1;
    L.C = rows ? (double*)take(vb) : nullptr;
    // level 0 of a multilevel solve: the raw fp32 edge weights of the preconditioner sweeps
    L.E = (rows || (l == 0 && nl > 1)) ? (float*)take(fb) : nullptr;
    L.Nw = (rows || (l == 0 && nl > 1)) ? (float*)take(fb) : nullptr;
    L.NE = rows ? (float*)take(fb) : nullptr;
    L.NW = rows ? (float*)take(fb) : nullptr;
    const size_t cb = sizeof(float) * (size_t)(L.m / 2) * (L.m / 2) * B;
    for (int q = 0; q < 4; ++q) L.pw[q] = (l + 1 < nl) ? (float*)take(cb) : nullptr;
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
  w.chol = (double*)take(sizeof(double) * (w.nc > 1089 ? band_doubles(w.lev[nl - 1].m + 1) : 2 * (size_t)w.nc * w.nc) * B);
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

L9 l9_of(const SolverLevel& L) { return L9{L.C, L.E, L.Nw, L.NE, L.NW, L.m, L.m + 1, L.N}; }
PW4 pw_of(const SolverLevel& L) { return PW4{L.pw[0], L.pw[1], L.pw[2], L.pw[3]}; }
HierDev hier_of(const SolverWork& w, int l0) {
  HierDev H{};
  for (int l = l0; l < w.nlev && l - l0 < 12; ++l) {
    const SolverLevel& L = w.lev[l];
    H.lev[l - l0] = SolverLevelDev{L.C, L.E, L.Nw, L.NE, L.NW, {L.pw[0], L.pw[1], L.pw[2], L.pw[3]}};
  }
  return H;
}

// z = A⁻¹ r on the coarsest grid: the explicit inverse (≤ 1089 nodes) or the banded factor
void coarsest_solve(Ctx* ctx, int B, const double* r, double* z) {
  SolverWork& w = ctx->solver;
  KScope ks(ctx, "mg_coarse_solve");
  if (w.nc > 1089) {
    const size_t sm = sizeof(double) * (size_t)w.nc;
    smem_attr(coarse_band_solve_kernel, sm);
    coarse_band_solve_kernel<<<B, 32, sm, ctx->stream>>>(w.lev[w.nlev - 1].m + 1, B, w.chol, r, z, w.flags);
  } else {
    coarse_solve_kernel<<<(B + 3) / 4, 128, 0, ctx->stream>>>(w.nc, B, w.chol, r, z, w.flags);
  }
  OSC_CUDA(cudaGetLastError());
}

// Preconditioner z = M r on level 0 (input w.r_cur, output lev[0].z2): V(1,1) with red-black GS.
// Levels with a coarser level below run ring-staged sweeps: level 0 the restriction (pre-smoother
// recomputed from r) and the up sweep (prolongation + post-smoother, fused with γ = ⟨r, z⟩ and
// δ = ⟨z, Az⟩ of the one-reduction PCG); 9-point levels the fused down sweep (pre-smoother +
// residual + restriction, z never stored) and the up sweep (z recomputed). The first level with
// m ≤ 32 and at least two levels below it runs the rest of the cycle CTA-resident (sub_vcycle).
void vcycle(Ctx* ctx, int bc, int B) {
  SolverWork& w = ctx->solver;
  cudaStream_t st = ctx->stream;
  double2* part = reinterpret_cast<double2*>(w.partial);
  if (w.nlev == 1) {
    coarsest_solve(ctx, B, w.r_cur, w.lev[0].z2);
    KScope ks(ctx, "pcg_dot_rz");
    dot_rz_kernel<<<dim3(nblocks(w.lev[0].N), 1, B), NT, 0, st>>>(geo_of(w.lev[0]), w.r_cur, w.lev[0].z2,
                                                                 w.scal, w.flags, part, w.max_parts, w.counter);
    OSC_CUDA(cudaGetLastError());
    return;
  }
  int ls = w.nlev - 1;
  for (int l = 1; l < w.nlev - 1; ++l)
    if (w.lev[l].m <= 32 && sub_smem_bytes(w.lev[l].m, w.nlev - l) <= kMaxCtaSmem) {
      ls = l;
      break;
    }
  // down
  for (int l = 0; l < ls; ++l) {
    const SolverLevel& L = w.lev[l];
    const SolverLevel& C = w.lev[l + 1];
    if (l == 0) {
      smem_attr(restrict_ring_kernel, L0R_SMEM_DN);
      KScope ks(ctx, "mg_restrict_r.L0");
      restrict_ring_kernel<<<restrict_grid_w(C.m, B, RR_W), 32 * RR_W, L0R_SMEM_DN, st>>>(
          geo_of(L), geo_of(C), bc, L.E, L.Nw, w.r_cur, pw_of(L), C.r, w.flags);
      continue;
    }
    smem_attr(c_down_ring_kernel, DN_RING_SMEM);
    KScope ks(ctx, lvl_name("mg_down", l).c_str());
    c_down_ring_kernel<<<restrict_grid_w(C.m, B, CD_W), 32 * CD_W, DN_RING_SMEM, st>>>(l9_of(L), bc, w.opdep, L.r,
                                                                                      pw_of(L), geo_of(C), C.r,
                                                                                      w.flags);
  }
  if (ls < w.nlev - 1) {
    const SolverLevel& S = w.lev[ls];
    const int nl = w.nlev - ls;
    const size_t sm = sub_smem_bytes(S.m, nl);
    smem_attr(sub_vcycle_kernel, sm);
    KScope ks(ctx, "mg_sub_vcycle");
    sub_vcycle_kernel<<<B, small_threads(S.m), sm, st>>>(S.m, nl, bc, w.opdep, hier_of(w, ls), S.r, S.z2, w.chol,
                                                         w.flags, (int)(sm / sizeof(double)));
  } else {
    const SolverLevel& C = w.lev[w.nlev - 1];
    coarsest_solve(ctx, B, C.r, C.z2);
  }
  // up
  for (int l = ls - 1; l >= 0; --l) {
    const SolverLevel& L = w.lev[l];
    const SolverLevel& C = w.lev[l + 1];
    if (l == 0) {
      smem_attr(smooth_up_ring_kernel, L0R_SMEM_UP);
      KScope ks(ctx, "mg_smooth_up_r.L0");
      smooth_up_ring_kernel<<<march_grid_w(L.m, B, SUR_W), 32 * SUR_W, L0R_SMEM_UP, st>>>(
          geo_of(L), geo_of(C), bc, L.E, L.Nw, w.r_cur, reinterpret_cast<z_t*>(L.z2), C.z2, pw_of(L), w.scal, w.flags, part,
          w.max_parts, w.counter);
      continue;
    }
    smem_attr(c_up_ring_kernel<true>, up_ring_smem<true>());
    KScope ks(ctx, lvl_name("mg_up", l).c_str());
    c_up_ring_kernel<true><<<march_grid_w(L.m, B, CU_W), 32 * CU_W, up_ring_smem<true>(), st>>>(
        l9_of(L), bc, w.opdep, L.r, nullptr, pw_of(L), geo_of(C), C.z2, L.z2, w.flags);
  }
  OSC_CUDA(cudaGetLastError());
}

// Multigrid hierarchy of the batch: transfer weights and coarse operators per coarse_op, and the
// coarsest inverse.
void mg_setup(Ctx* ctx, const osc_problem* prob, int B) {
  SolverWork& w = ctx->solver;
  cudaStream_t st = ctx->stream;
  const int bc = prob->bc, mode = prob->coarse_op;
  const SolverLevel& L0 = w.lev[0];
  const Geo g0 = geo_of(L0);
  if (w.nlev == 1) {
    // single level: the dense factor is built from k directly (exact fp64 rows)
  } else if (mode != OSC_COARSE_REDISCRETIZE) {
    // fused tiled Galerkin setup per level pair (galerkin_tile_kernel)
    smem_attr(galerkin_tile_kernel<true>, galerkin_tile_smem(true));
    smem_attr(galerkin_tile_kernel<false>, galerkin_tile_smem(false));
    for (int l = 0; l + 1 < w.nlev; ++l) {
      const SolverLevel& F = w.lev[l];
      const SolverLevel& C = w.lev[l + 1];
      const dim3 grid((unsigned)((C.m + GT_X) / GT_X), (unsigned)((C.m + GT_Y) / GT_Y), (unsigned)B);
      KScope ks(ctx, l == 0 ? "mg_setup.galerkin.L0" : "mg_setup.galerkin.Lc");
      if (l == 0)
        galerkin_tile_kernel<true><<<grid, GT_THREADS, galerkin_tile_smem(true), st>>>(
            L0.k, L9{nullptr, nullptr, nullptr, nullptr, nullptr, F.m, F.m + 1, F.N}, bc, w.opdep, geo_of(C), C.C,
            C.E, C.Nw, C.NE, C.NW, F.pw[0], F.pw[1], F.pw[2], F.pw[3], L0.E, L0.Nw);
      else
        galerkin_tile_kernel<false><<<grid, GT_THREADS, galerkin_tile_smem(false), st>>>(
            nullptr, l9_of(F), bc, w.opdep, geo_of(C), C.C, C.E, C.Nw, C.NE, C.NW, F.pw[0], F.pw[1], F.pw[2],
            F.pw[3], nullptr, nullptr);
    }
  } else {  // REDISCRETIZE: level-0 rows (5-point) into scratch (u, r, r2 are free until pcg_init)
    {
      KScope ks(ctx, "mg_setup.edges0");
      edges0_kernel<<<dim3(nblocks(L0.N), B), NT, 0, st>>>(g0, L0.k, L0.E, L0.Nw);
    }
    {
      KScope ks(ctx, "mg_setup.rows");
      rows0_kernel<<<dim3(nblocks(L0.N), B), NT, 0, st>>>(g0, bc, L0.k, w.u, reinterpret_cast<float*>(L0.r),
                                                           reinterpret_cast<float*>(w.r2));
    }
    for (int l = 0; l + 1 < w.nlev; ++l) {
      const SolverLevel& F = w.lev[l];
      const SolverLevel& C = w.lev[l + 1];
      const L9 R = l == 0 ? L9{w.u, reinterpret_cast<const float*>(L0.r), reinterpret_cast<const float*>(w.r2),
                               nullptr, nullptr, F.m, F.m + 1, F.N}
                          : l9_of(F);
      {  // P1 transfer weights of level l (centre weights pw; edges are ½)
        KScope ks(ctx, "mg_setup.prow");
        prow_kernel<<<dim3(nblocks(F.N), B), NT, 0, st>>>(R, bc, w.opdep, L0.z, L0.z2, w.p0, w.p1, F.pw[0],
                                                           F.pw[1], F.pw[2], F.pw[3]);
      }
      KScope ks(ctx, "mg_setup.coarse_op");
      rediscretize_kernel<<<dim3(nblocks(C.N), B), NT, 0, st>>>(L0.k, g0, 2 << l, bc, geo_of(C), C.C, C.E, C.Nw,
                                                                C.NE, C.NW);
    }
  }
  KScope ks(ctx, "mg_setup.factor");
  const double* k_exact = w.nlev == 1 ? L0.k : nullptr;
  const SolverLevel& C = w.lev[w.nlev - 1];
  if (w.nc > 1089) {
    const size_t sm = sizeof(double) * (size_t)(C.m + 3) * (C.m + 3);
    smem_attr(coarse_band_factor_kernel, sm);
    coarse_band_factor_kernel<<<B, 32, sm, st>>>(l9_of(C), B, w.chol, k_exact, bc);
  } else if (w.nc <= 32)
    coarse_factor_warp_kernel<<<(B + CF_WARPS - 1) / CF_WARPS, 32 * CF_WARPS, 0, st>>>(l9_of(C), B, w.chol, k_exact, bc);
  else
    coarse_factor_kernel<<<(B + 63) / 64, 64, 0, st>>>(l9_of(C), B, w.chol, k_exact, bc);
  OSC_CUDA(cudaGetLastError());
}

}  // namespace

namespace {
// ---- device-side PCG loop --------------------------------------------------------------------------
// Small grids iterate inside one CUDA graph instead of the host-polled loop: a conditional WHILE node
// whose body is two one-reduction PCG iterations (the r / p ping-pong returns to its start after
// two) followed by pcg_loop_cond_kernel, which keeps the loop going while any sample of the batch is
// active. Samples converge individually as before (every kernel skips inactive samples), so results
// and iteration counts are those of the host loop. Graphs are cached per solve shape and rebuilt
// when a baked-in value (shape, tolerance, buffers) changes. Measured, the host loop was not
// launch-bound even at 64² (the lagged polling keeps the queue full): the device loop is neutral
// (scripts/graph_ab.py), so it is kept to 128², where it removes the host round trips per iteration.
#ifndef OSC_GRAPH_MAX_M
#define OSC_GRAPH_MAX_M 128
#endif
constexpr int kGraphMaxM = OSC_GRAPH_MAX_M;  // A/B (scripts/graph_ab.py): 64² 33.6 vs 33.8 ms, 128² 43.0 vs 43.5 ms per batch; neutral above

void pcg_iteration(Ctx* ctx, const osc_problem* prob, int B, double* r_in, double* r_out, double* p_old,
                   double* p_new) {
  SolverWork& w = ctx->solver;
  SolverLevel& L0 = w.lev[0];
  double2* part = reinterpret_cast<double2*>(w.partial);
  {
    KScope ks(ctx, "pcg_update");
    pcg_update_cg_kernel<<<march_grid_w(L0.m, B, PU_W), 32 * PU_W, 0, ctx->stream>>>(
        geo_of(L0), prob->bc, prob->tol, L0.k, reinterpret_cast<const z_t*>(L0.z2), reinterpret_cast<const p_t*>(p_old),
        reinterpret_cast<p_t*>(p_new), w.u, r_in, r_out, w.scal, w.flags, part, w.max_parts, w.counter, w.n_active,
        w.hist, w.hist_cap);
  }
  w.r_cur = r_out;
  vcycle(ctx, prob->bc, B);
}

void run_pcg_graph(Ctx* ctx, const osc_problem* prob, int B, long hard_cap) {
  SolverWork& w = ctx->solver;
  SolverLevel& L0 = w.lev[0];
  cudaStream_t st = ctx->stream;
  SolverWork::LoopGraph* G = nullptr;
  for (auto& g : w.graphs)
    if (g.m == w.m && g.B == B && g.bc == prob->bc && g.opdep == w.opdep && g.hist_cap == w.hist_cap &&
        g.hard_cap == hard_cap && g.tol == prob->tol && g.k == L0.k && g.mem == w.mem.p &&
        g.mem_bytes == w.mem.bytes)
      G = &g;
  if (!G) {
    if (w.graphs.size() >= 8) {  // evict the least recently used
      auto lru = std::min_element(w.graphs.begin(), w.graphs.end(),
                                  [](const auto& a, const auto& b) { return a.last_use < b.last_use; });
      cudaGraphExecDestroy(lru->exec);
      w.graphs.erase(lru);
    }
    SolverWork::LoopGraph g;
    g.m = w.m;
    g.B = B;
    g.bc = prob->bc;
    g.opdep = w.opdep;
    g.hist_cap = w.hist_cap;
    g.hard_cap = hard_cap;
    g.tol = prob->tol;
    g.k = L0.k;
    g.mem = w.mem.p;
    g.mem_bytes = w.mem.bytes;
    cudaGraph_t graph = nullptr;
    OSC_CUDA(cudaGraphCreate(&graph, 0));
    try {
      cudaGraphConditionalHandle h;
      OSC_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams np = {};
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = h;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      cudaGraphNode_t node;
      OSC_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &np));
      cudaGraph_t body = np.conditional.phGraph_out[0];
      // the kernels launch during capture only as graph nodes: count them once per body run
      const int64_t launches0 = ctx->launches;
      OSC_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      try {
        pcg_iteration(ctx, prob, B, L0.r, w.r2, w.p0, w.p1);
        pcg_iteration(ctx, prob, B, w.r2, L0.r, w.p1, w.p0);
        pcg_loop_cond_kernel<<<1, 256, 0, st>>>(h, w.n_active, w.n_active + 2, hard_cap, B, w.flags);
      } catch (...) {
        cudaGraph_t dummy;
        cudaStreamEndCapture(st, &dummy);
        throw;
      }
      OSC_CUDA(cudaStreamEndCapture(st, &body));
      g.body_launches = (int)(ctx->launches - launches0) + 1;
      ctx->launches = launches0;
      OSC_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
    } catch (...) {
      cudaGraphDestroy(graph);
      throw;
    }
    cudaGraphDestroy(graph);
    w.graphs.push_back(g);
    G = &w.graphs.back();
  }
  G->last_use = ++w.graph_clock;
  w.r_cur = L0.r;  // the body's start state (r in L0.r, previous p in p0)
  OSC_CUDA(cudaMemsetAsync(w.n_active + 2, 0, sizeof(int), st));
  {
    KScope ks(ctx, "pcg_loop_graph", 0);
    OSC_CUDA(cudaGraphLaunch(G->exec, st));
  }
  // body runs of this solve → launch count, read with the results (solver_results synchronises)
  OSC_CUDA(cudaMemcpyAsync(ctx->h_pinned_int + 2, w.n_active + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
  w.pending_body_launches = G->body_launches;
}
}  // namespace

// Solve the batch whose level-0 conductivity sits in ctx->solver.lev[0].k (set by caller).
void solver_run(Ctx* ctx, const osc_problem* prob, int B, const double* uc_guess) {
  SolverWork& w = ctx->solver;
  cudaStream_t st = ctx->stream;
  double2* part = reinterpret_cast<double2*>(w.partial);
  const int bc = prob->bc;
  OSC_REQUIRE(prob->coarse_op == OSC_COARSE_GALERKIN || prob->coarse_op == OSC_COARSE_REDISCRETIZE ||
                  prob->coarse_op == OSC_COARSE_GALERKIN_LINEAR,
              "solve: unknown coarse_op");
  w.opdep = prob->coarse_op == OSC_COARSE_GALERKIN ? 1 : 0;
  struct TagGuard {
    Ctx* c;
    ~TagGuard() { c->tag.clear(); }
  } tg{ctx};
  ctx->tag = std::to_string(w.m);
  SolverLevel& L0 = w.lev[0];
  const Geo g0 = geo_of(L0);
  w.r_cur = L0.r;
  mg_setup(ctx, prob, B);
  if (w.m <= 32 && w.nlev > 1 && w.hist_cap == 0 && small_smem_bytes(w.m, w.nlev) <= kMaxCtaSmem) {
    // whole solve CTA-resident (one CTA per sample, one launch); a kept residual history takes the
    // streaming path below
    const size_t sm = small_smem_bytes(w.m, w.nlev);
    smem_attr(small_pcg_kernel, sm);
    KScope ks(ctx, "small_pcg");
    small_pcg_kernel<<<B, small_threads(w.m), sm, st>>>(w.m, w.nlev, bc, w.opdep, prob->forcing, prob->forcing_value,
                                               prob->tol, prob->max_iter_factor, L0.k, hier_of(w, 0), w.chol,
                                               w.u, w.flags, w.scal, (int)(sm / sizeof(double)));
    OSC_CUDA(cudaGetLastError());
    return;
  }
  OSC_CUDA(cudaMemsetAsync(w.n_active, 0, sizeof(int), st));
  {  // uc_guess: nested iteration, start from the prolonged coarse coupled solution. Large grids form
     // the guess and r0 in a column-pair marching pass (config 4, 2048²: 4.5 → 3.3 ms per 64-sample
     // batch); below m = 1024 the per-node init is faster (256²: 1.4 vs 2.0 ms).
    KScope ks(ctx, "pcg_init");
    if (uc_guess && w.m >= 1024) {
      pcg_init_nested_kernel<<<march_grid(L0.m, 1, B), MT, 0, st>>>(
          g0, bc, prob->forcing, prob->forcing_value, prob->tol, prob->max_iter_factor, L0.k, uc_guess, w.u,
          w.r_cur, w.scal, w.flags, part, w.max_parts, w.counter, w.n_active, w.hist, w.hist_cap);
    } else {
      const dim3 grid((g0.n0 + NT - 1) / NT, (g0.n0 + INIT_RY - 1) / INIT_RY, B);
      pcg_init_kernel<<<grid, NT, 0, st>>>(g0, bc, prob->forcing, prob->forcing_value, prob->tol,
                                           prob->max_iter_factor, L0.k, uc_guess, w.u, w.r_cur, w.scal, w.flags,
                                           part, w.max_parts, w.counter, w.n_active, w.hist, w.hist_cap);
    }
  }
  // optional safety valve (tests): OSC_HARD_ITER_CAP stops the loop early; the samples still active
  // are reported as not converged by solver_results()
  static const long hard_cap = [] {
    const char* e = std::getenv("OSC_HARD_ITER_CAP");
    return e ? std::atol(e) : -1L;
  }();
  double* p_old = w.p0;
  double* p_new = w.p1;
  if (w.nlev > 1) {
    // One-reduction (Chronopoulos–Gear) PCG: pcg_update forms p, u, r and ‖r‖; the V-cycle's up sweep
    // returns γ = ⟨r, z⟩ and δ = ⟨z, Az⟩, hence β and α of the next update.
    vcycle(ctx, bc, B);  // z = M r0; γ0, δ0 → α0
    if (!ctx->profiling && w.m <= kGraphMaxM) {
      // device-side loop: no host polling, no per-kernel launch overhead (launch-bound small grids)
      run_pcg_graph(ctx, prob, B, hard_cap);
      return;
    }
    // Lagged convergence polling: the active count after iteration i is copied to a pinned ring
    // slot behind an event, and the host reads it before launching iteration i + LAG. The device
    // queue never drains while the host polls; iterations launched after the last sample
    // converged exit at once (every kernel skips inactive samples).
    constexpr int LAG = 2;
    int* ring = ctx->h_pinned_int + 4;
    for (int it = 0;; ++it) {
      if (hard_cap >= 0 && it >= hard_cap) {
        mark_active_failed_kernel<<<(B + 255) / 256, 256, 0, st>>>(B, w.flags);
        break;
      }
      if (it >= LAG) {
        const int slot = (it - LAG) & 3;
        OSC_CUDA(cudaEventSynchronize(ctx->ev_poll[slot]));
        if (ring[slot] <= 0) break;
      }
      {
        KScope ks(ctx, "pcg_update");
        double* r_next = (w.r_cur == L0.r) ? w.r2 : L0.r;
        pcg_update_cg_kernel<<<march_grid_w(L0.m, B, PU_W), 32 * PU_W, 0, st>>>(
            g0, bc, prob->tol, L0.k, reinterpret_cast<const z_t*>(L0.z2), reinterpret_cast<const p_t*>(p_old),
            reinterpret_cast<p_t*>(p_new), w.u, w.r_cur, r_next, w.scal, w.flags, part, w.max_parts, w.counter,
            w.n_active, w.hist, w.hist_cap);
        w.r_cur = r_next;
      }
      OSC_CUDA(cudaMemcpyAsync(ring + (it & 3), w.n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
      OSC_CUDA(cudaEventRecord(ctx->ev_poll[it & 3], st));
      vcycle(ctx, bc, B);
      std::swap(p_old, p_new);
    }
    return;
  }
  // a single level (m ≤ 4): classical PCG with the exact coarsest inverse as preconditioner
  vcycle(ctx, bc, B);  // z = M r0, rz = <r0, z>
  for (int it = 0;; ++it) {
    if (hard_cap >= 0 && it >= hard_cap) {
      mark_active_failed_kernel<<<(B + 255) / 256, 256, 0, st>>>(B, w.flags);
      break;
    }
    OSC_CUDA(cudaMemcpyAsync(ctx->h_pinned_int, w.n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
    OSC_CUDA(cudaStreamSynchronize(st));
    if (*ctx->h_pinned_int <= 0) break;
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
                                                              w.counter, w.n_active, w.hist, w.hist_cap, 0);
    }
    w.r_cur = (w.r_cur == L0.r) ? w.r2 : L0.r;
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
  if (w.pending_body_launches) {  // the device-side loop's kernels (body runs × kernels per run)
    ctx->launches += (int64_t)w.pending_body_launches * ctx->h_pinned_int[2];
    w.pending_body_launches = 0;
  }
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

void level_sums_reshift_launch(Ctx* ctx, double* sums_dev, double dy, double dq) {
  KScope ks(ctx, "level_sums");
  level_sums_reshift_kernel<<<1, 1, 0, ctx->stream>>>(sums_dev, dy, dq);
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
