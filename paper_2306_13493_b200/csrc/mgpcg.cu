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

// ---- tiled, fused MG-PCG kernels -------------------------------------------------------------
// Every kernel works on a TX×TY tile of one sample (blockIdx.z) with the fields it needs staged
// in shared memory with a halo, and recomputes the 5-point stencil from the nodal k tile
// (8 B/node of HBM instead of 24 B/node for stored D/E/N).
constexpr int TX = 32, TY = 16;      // fine tile (threads: 32 × 8, two rows each)
constexpr int CXT = 32, CYT = 8;     // coarse tile of the restriction (one node per thread)
constexpr int TT = 256;              // threads per tiled CTA

struct Sten {
  double d, e, w, n, s;  // raw diagonal (1 on Dirichlet rows) and eliminated couplings
};

// Stencil at tile-local (lx, ly) of k tile `kt` (leading dim ld) for global node (gx, gy).
// Bitwise identical to the per-node formulas in the header (same operands, same order),
// so the coupling seen from both ends of an edge is the same double (A stays symmetric).
__device__ __forceinline__ Sten stencil_at(const double* kt, int ld, int lx, int ly, int gx, int gy,
                                           int m, int bc) {
  auto K = [&](int dx, int dy) { return kt[(ly + dy) * ld + lx + dx]; };
  const double k00 = K(0, 0);
  double e = 0.0, w = 0.0, n = 0.0, s = 0.0;
  if (gx < m) e = -0.5 * ((gy < m ? (k00 + K(1, 0) + K(1, 1)) / 3.0 : 0.0) +
                          (gy > 0 ? (K(0, -1) + K(1, 0) + k00) / 3.0 : 0.0));
  if (gx > 0) w = -0.5 * ((gy < m ? (K(-1, 0) + k00 + K(0, 1)) / 3.0 : 0.0) +
                          (gy > 0 ? (K(-1, -1) + k00 + K(-1, 0)) / 3.0 : 0.0));
  if (gy < m) n = -0.5 * ((gx < m ? (k00 + K(1, 1) + K(0, 1)) / 3.0 : 0.0) +
                          (gx > 0 ? (K(-1, 0) + k00 + K(0, 1)) / 3.0 : 0.0));
  if (gy > 0) s = -0.5 * ((gx < m ? (K(0, -1) + K(1, 0) + k00) / 3.0 : 0.0) +
                          (gx > 0 ? (K(-1, -1) + K(0, -1) + k00) / 3.0 : 0.0));
  Sten st;
  if (is_dir(bc, m, gx, gy)) {
    st.d = 1.0;
    st.e = st.w = st.n = st.s = 0.0;
    return st;
  }
  st.d = -(e + w + n + s);
  st.e = is_dir(bc, m, gx + 1, gy) ? 0.0 : e;
  st.w = is_dir(bc, m, gx - 1, gy) ? 0.0 : w;
  st.n = is_dir(bc, m, gx, gy + 1) ? 0.0 : n;
  st.s = is_dir(bc, m, gx, gy - 1) ? 0.0 : s;
  return st;
}

// Stage rows [gy0, gy0+h) × cols [gx0, gx0+wd) of a sample's nodal field into smem with
// cp.async (LDGSTS): every element's copy is in flight at once (no register round trip), and
// out-of-grid elements are zero-filled (src-size 0). Caller: stage_wait() before use.
__device__ __forceinline__ void stage(double* sm, int wd, int h, const double* __restrict__ g,
                                      int gx0, int gy0, int n0) {
  for (int idx = threadIdx.x; idx < wd * h; idx += TT) {
    const int ly = idx / wd, lx = idx - ly * wd;
    const int gx = gx0 + lx, gy = gy0 + ly;
    const bool in = gx >= 0 && gx < n0 && gy >= 0 && gy < n0;
    const double* src = in ? g + (int64_t)gy * n0 + gx : g;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sm + idx);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(in ? 8 : 0)
                 : "memory");
  }
}
__device__ __forceinline__ void stage_wait() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
}

// Raw edge weights of a staged k region (origin (gx0, gy0), wd × h, zero-padded outside the
// grid): es[y][x] couples (x,y)–(x+1,y), ns[y][x] couples (x,y)–(x,y+1). Triangle means use
// the reference's vertex order with ·(1/3) instead of /3 (≤ 1 ulp per coefficient), and each
// edge is formed once, so both rows of A see the same double (A stays symmetric).
__device__ __forceinline__ void build_edges(const double* ks, double* es, double* ns, int wd, int h,
                                            int gx0, int gy0, int m) {
  constexpr double third = 1.0 / 3.0;
  for (int idx = threadIdx.x; idx < wd * h; idx += TT) {
    const int ly = idx / wd, lx = idx - ly * wd;
    const int gx = gx0 + lx, gy = gy0 + ly;
    double e = 0.0, n = 0.0;
    if (lx + 1 < wd && ly > 0 && ly + 1 < h && gx >= 0 && gx < m && gy >= 0 && gy <= m) {
      const double* k = ks + idx;
      const double lo = gy < m ? (k[0] + k[1] + k[wd + 1]) * third : 0.0;       // K_low(x, y)
      const double up = gy > 0 ? (k[-wd] + k[1] + k[0]) * third : 0.0;          // K_up(x, y-1)
      e = -0.5 * (lo + up);
    }
    if (lx > 0 && lx + 1 < wd && ly + 1 < h && gy >= 0 && gy < m && gx >= 0 && gx <= m) {
      const double* k = ks + idx;
      const double up = gx < m ? (k[0] + k[wd + 1] + k[wd]) * third : 0.0;      // K_up(x, y)
      const double lo = gx > 0 ? (k[-1] + k[0] + k[wd]) * third : 0.0;         // K_low(x-1, y)
      n = -0.5 * (up + lo);
    }
    es[idx] = e;
    ns[idx] = n;
  }
}

// 5-point row at local (lx, ly) of an edge region with leading dimension wd.
__device__ __forceinline__ Sten sten_edges(const double* es, const double* ns, int wd, int lx, int ly,
                                           int gx, int gy, int m, int bc) {
  const int c = ly * wd + lx;
  Sten st;
  if (is_dir(bc, m, gx, gy)) {
    st.d = 1.0;
    st.e = st.w = st.n = st.s = 0.0;
    return st;
  }
  const double e = es[c], w = es[c - 1], n = ns[c], s = ns[c - wd];
  st.d = -(e + w + n + s);
  st.e = is_dir(bc, m, gx + 1, gy) ? 0.0 : e;
  st.w = is_dir(bc, m, gx - 1, gy) ? 0.0 : w;
  st.n = is_dir(bc, m, gx, gy + 1) ? 0.0 : n;
  st.s = is_dir(bc, m, gx, gy - 1) ? 0.0 : s;
  return st;
}

#define TILE_PROLOGUE                                                \
  const int b = blockIdx.z;                                          \
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;                       \
  const int m = g.m, n0 = g.n0;                                      \
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;              \
  const int64_t off = (int64_t)b * g.N;                              \
  const int tx = threadIdx.x & 31, ty0 = threadIdx.x >> 5;

// ---- setup: k injection to the next level (fem.cpp:241-244) -----------------------------------------
__global__ void __launch_bounds__(NT) inject_kernel(Geo gf, Geo gc, const double* __restrict__ kf,
                                                    double* __restrict__ kc) {
  const int b = blockIdx.y;
  const int64_t ic = blockIdx.x * (int64_t)NT + threadIdx.x;
  if (ic >= gc.N) return;
  const int J = (int)(ic / gc.n0), I = (int)(ic - (int64_t)J * gc.n0);
  kc[(int64_t)b * gc.N + ic] = kf[(int64_t)b * gf.N + (int64_t)(2 * J) * gf.n0 + 2 * I];
}

// Dense Cholesky of the coarsest operator, one thread per sample (fem.cpp:255-272).
__global__ void coarse_factor_kernel(Geo g, int bc, int B, const double* __restrict__ k,
                                     double* __restrict__ chol) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int n = (int)g.N, n0 = g.n0, m = g.m;
  double* L = chol + (int64_t)b * n * n;
  const double* kb = k + (int64_t)b * n;
  for (int i = 0; i < n * n; ++i) L[i] = 0.0;
  // stencil from a zero-padded 3×3 neighbourhood of k
  for (int i = 0; i < n; ++i) {
    const int gy = i / n0, gx = i - gy * n0;
    double kt[9];
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int x = gx + dx, y = gy + dy;
        kt[(dy + 1) * 3 + dx + 1] = (x >= 0 && x < n0 && y >= 0 && y < n0) ? kb[y * n0 + x] : 0.0;
      }
    const Sten st = stencil_at(kt, 3, 1, 1, gx, gy, m, bc);
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

// ---- PCG: p = z + βp (p = z first), <p, A p> → α  (Ap itself is recomputed where needed) -----------
__global__ void __launch_bounds__(TT) pcg_apply_kernel(Geo g, int bc, const double* __restrict__ k,
                                                       const double* __restrict__ z,
                                                       const double* __restrict__ p_old,
                                                       double* __restrict__ p_new, double* scal,
                                                       int* flags, double2* partial, int maxp,
                                                       unsigned* counter) {
  TILE_PROLOGUE
  constexpr int W1 = TX + 2, H1 = TY + 2;
  __shared__ double ks[H1 * W1], ps[H1 * W1], zs[H1 * W1], es[H1 * W1], ns[H1 * W1];
  const bool first = flags[b * F_NFLAGS + F_FIRST] != 0;
  const double beta = scal[b * S_NSCAL + S_BETA];
  stage(ks, W1, H1, k + off, x0 - 1, y0 - 1, n0);
  stage(zs, W1, H1, z + off, x0 - 1, y0 - 1, n0);
  if (!first) stage(ps, W1, H1, p_old + off, x0 - 1, y0 - 1, n0);
  stage_wait();
  build_edges(ks, es, ns, W1, H1, x0 - 1, y0 - 1, m);
  for (int idx = threadIdx.x; idx < W1 * H1; idx += TT)
    ps[idx] = first ? zs[idx] : fma(beta, ps[idx], zs[idx]);
  __syncthreads();
  double pap = 0.0;
#pragma unroll
  for (int r = 0; r < TY / 8; ++r) {
    const int ly = ty0 + 8 * r, gx = x0 + tx, gy = y0 + ly;
    if (gx < n0 && gy < n0) {
      const int c = (ly + 1) * W1 + tx + 1;
      const Sten st = sten_edges(es, ns, W1, tx + 1, ly + 1, gx, gy, m, bc);
      const double pc = ps[c];
      const double ap = st.d * pc + st.e * ps[c + 1] + st.w * ps[c - 1] + st.n * ps[c + W1] +
                        st.s * ps[c - W1];
      p_new[off + (int64_t)gy * n0 + gx] = pc;
      pap = fma(pc, ap, pap);
    }
  }
  double t0, t1;
  if (reduce2_last(pap, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    scal[b * S_NSCAL + S_ALPHA] = scal[b * S_NSCAL + S_RZ] / t0;
    flags[b * F_NFLAGS + F_FIRST] = 0;
  }
}

// ---- PCG update fused with the level-0 pre-smoother:
//   u += αp, r −= αAp (Ap recomputed from p), ‖r‖ → convergence,
//   then z_red = r/D, z_black = (r − Σ A z_red)/D  (red-black GS from z = 0)
__global__ void __launch_bounds__(TT) pcg_update_down_kernel(
    Geo g, int bc, double tol, const double* __restrict__ k, const double* __restrict__ p,
    double* __restrict__ u, const double* __restrict__ r, double* __restrict__ r_out,
    double* __restrict__ z, double* scal, int* flags,
    double2* partial, int maxp, unsigned* counter, int* n_active, double* hist, int hist_cap) {
  TILE_PROLOGUE
  constexpr int W2 = TX + 4, H2 = TY + 4, W1 = TX + 2, H1 = TY + 2;
  __shared__ double ks[H2 * W2], ps[H2 * W2], rs[H1 * W1], zr[H1 * W1], es[H2 * W2], ns[H2 * W2],
      us[TX * TY];
  const double alpha = scal[b * S_NSCAL + S_ALPHA];
  stage(ks, W2, H2, k + off, x0 - 2, y0 - 2, n0);
  stage(ps, W2, H2, p + off, x0 - 2, y0 - 2, n0);
  stage(rs, W1, H1, r + off, x0 - 1, y0 - 1, n0);
  stage(us, TX, TY, u + off, x0, y0, n0);
  stage_wait();
  build_edges(ks, es, ns, W2, H2, x0 - 2, y0 - 2, m);
  __syncthreads();
  // r_new and z_red = r_new / D on the tile + 1 halo (in place in rs)
  for (int idx = threadIdx.x; idx < W1 * H1; idx += TT) {
    const int ly = idx / W1, lx = idx - ly * W1;
    const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
    double rn = 0.0, zv = 0.0;
    if (gx >= 0 && gx < n0 && gy >= 0 && gy < n0) {
      const int c = (ly + 1) * W2 + lx + 1;
      const Sten st = sten_edges(es, ns, W2, lx + 1, ly + 1, gx, gy, m, bc);
      const double ap = st.d * ps[c] + st.e * ps[c + 1] + st.w * ps[c - 1] + st.n * ps[c + W2] +
                        st.s * ps[c - W2];
      rn = fma(-alpha, ap, rs[idx]);
      if (((gx + gy) & 1) == 0) zv = rn / st.d;
    }
    rs[idx] = rn;
    zr[idx] = zv;
  }
  __syncthreads();
  double rr = 0.0;
#pragma unroll
  for (int q = 0; q < TY / 8; ++q) {
    const int ly = ty0 + 8 * q, gx = x0 + tx, gy = y0 + ly;
    if (gx < n0 && gy < n0) {
      const int c1 = (ly + 1) * W1 + tx + 1;
      const int64_t j = off + (int64_t)gy * n0 + gx;
      const double rn = rs[c1];
      double zv;
      if (((gx + gy) & 1) == 0) {
        zv = zr[c1];
      } else {
        const Sten st = sten_edges(es, ns, W2, tx + 2, ly + 2, gx, gy, m, bc);
        zv = (rn - (st.e * zr[c1 + 1] + st.w * zr[c1 - 1] + st.n * zr[c1 + W1] + st.s * zr[c1 - W1])) / st.d;
      }
      u[j] = fma(alpha, ps[(ly + 2) * W2 + tx + 2], us[ly * TX + tx]);
      r_out[j] = rn;
      z[j] = zv;
      rr = fma(rn, rn, rr);
    }
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

// ---- pre-smoother on coarse levels (and on level 0 for the first V-cycle): red then black -----------
__global__ void __launch_bounds__(TT) smooth_down_kernel(Geo g, int bc, const double* __restrict__ k,
                                                         const double* __restrict__ r,
                                                         double* __restrict__ z, const int* flags) {
  TILE_PROLOGUE
  constexpr int W2 = TX + 4, H2 = TY + 4, W1 = TX + 2, H1 = TY + 2;
  __shared__ double ks[H2 * W2], rs[H1 * W1], zr[H1 * W1], es[H2 * W2], ns[H2 * W2];
  stage(ks, W2, H2, k + off, x0 - 2, y0 - 2, n0);
  stage(rs, W1, H1, r + off, x0 - 1, y0 - 1, n0);
  stage_wait();
  build_edges(ks, es, ns, W2, H2, x0 - 2, y0 - 2, m);
  __syncthreads();
  for (int idx = threadIdx.x; idx < W1 * H1; idx += TT) {
    const int ly = idx / W1, lx = idx - ly * W1;
    const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
    double zv = 0.0;
    if (gx >= 0 && gx < n0 && gy >= 0 && gy < n0 && ((gx + gy) & 1) == 0) {
      const Sten st = sten_edges(es, ns, W2, lx + 1, ly + 1, gx, gy, m, bc);
      zv = rs[idx] / st.d;
    }
    zr[idx] = zv;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < TY / 8; ++q) {
    const int ly = ty0 + 8 * q, gx = x0 + tx, gy = y0 + ly;
    if (gx < n0 && gy < n0) {
      const int c1 = (ly + 1) * W1 + tx + 1;
      double zv;
      if (((gx + gy) & 1) == 0) {
        zv = zr[c1];
      } else {
        const Sten st = sten_edges(es, ns, W2, tx + 2, ly + 2, gx, gy, m, bc);
        zv = (rs[c1] - (st.e * zr[c1 + 1] + st.w * zr[c1 - 1] + st.n * zr[c1 + W1] + st.s * zr[c1 - W1])) / st.d;
      }
      z[off + (int64_t)gy * n0 + gx] = zv;
    }
  }
}

// ---- residual restriction rc = Pᵀ(r − A z) after the red-black pre-smoother (fem.cpp:168-195).
// After the black sweep the residual vanishes on black nodes and equals −Σ A z_black on red
// nodes, so rc(I,J) = t(2I,2J) + ½[t(2I+1,2J+1) + t(2I−1,2J−1)]; zero at coarse Dirichlet nodes.
__global__ void __launch_bounds__(TT) restrict_kernel(Geo g, Geo gc, int bc,
                                                      const double* __restrict__ k,
                                                      const double* __restrict__ z,
                                                      double* __restrict__ rc, const int* flags) {
  const int b = blockIdx.z;
  if (!flags[b * F_NFLAGS + F_ACTIVE]) return;
  const int m = g.m, n0 = g.n0, mc = gc.m;
  const int I0 = blockIdx.x * CXT, J0 = blockIdx.y * CYT;
  constexpr int WR = 2 * CXT + 3, HR = 2 * CYT + 3;
  __shared__ double ks[HR * WR], zs[HR * WR], es[HR * WR], ns[HR * WR];
  const int64_t off = (int64_t)b * g.N;
  const int fx0 = 2 * I0 - 2, fy0 = 2 * J0 - 2;
  stage(ks, WR, HR, k + off, fx0, fy0, n0);
  stage(zs, WR, HR, z + off, fx0, fy0, n0);
  stage_wait();
  build_edges(ks, es, ns, WR, HR, fx0, fy0, m);
  __syncthreads();
  const int I = I0 + (threadIdx.x & 31), J = J0 + (threadIdx.x >> 5);
  if (I > mc || J > mc) return;
  double acc = 0.0;
  if (!is_dir(bc, mc, I, J)) {
    auto t_at = [&](int fx, int fy) {  // residual at a red fine node
      if (fx < 0 || fx > m || fy < 0 || fy > m) return 0.0;
      const int lx = fx - fx0, ly = fy - fy0;
      const Sten st = sten_edges(es, ns, WR, lx, ly, fx, fy, m, bc);
      const int c = ly * WR + lx;
      return -(st.e * zs[c + 1] + st.w * zs[c - 1] + st.n * zs[c + WR] + st.s * zs[c - WR]);
    };
    acc = t_at(2 * I, 2 * J) + 0.5 * (t_at(2 * I + 1, 2 * J + 1) + t_at(2 * I - 1, 2 * J - 1));
  }
  rc[(int64_t)b * gc.N + (int64_t)J * gc.n0 + I] = acc;
}

// ---- prolongation + post-smoother (black then red), on level 0 also <r, z> → β ------------------------
__global__ void __launch_bounds__(TT) smooth_up_kernel(Geo g, Geo gc, int bc,
                                                       const double* __restrict__ k,
                                                       const double* __restrict__ r,
                                                       const double* __restrict__ z,
                                                       double* __restrict__ z_out,
                                                       const double* __restrict__ zc, int finest,
                                                       double* scal, int* flags, double2* partial,
                                                       int maxp, unsigned* counter) {
  TILE_PROLOGUE
  constexpr int W2 = TX + 4, H2 = TY + 4, W1 = TX + 2, H1 = TY + 2;
  constexpr int WC = TX / 2 + 3, HC = TY / 2 + 3;
  __shared__ double ks[H2 * W2], zp[H2 * W2], rs[H1 * W1], zb[H1 * W1], zcs[HC * WC], es[H2 * W2],
      ns[H2 * W2];
  const int cx0 = x0 / 2 - 1, cy0 = y0 / 2 - 1;
  stage(ks, W2, H2, k + off, x0 - 2, y0 - 2, n0);
  stage(zp, W2, H2, z + off, x0 - 2, y0 - 2, n0);
  stage(rs, W1, H1, r + off, x0 - 1, y0 - 1, n0);
  stage(zcs, WC, HC, zc + (int64_t)b * gc.N, cx0, cy0, gc.n0);
  stage_wait();
  build_edges(ks, es, ns, W2, H2, x0 - 2, y0 - 2, m);
  // red nodes of the 2-halo region after prolongation: z_red + P zc (black entries unused)
  for (int idx = threadIdx.x; idx < W2 * H2; idx += TT) {
    const int ly = idx / W2, lx = idx - ly * W2;
    const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
    if (gx >= 0 && gx < n0 && gy >= 0 && gy < n0 && ((gx + gy) & 1) == 0) {
      auto Zc = [&](int I, int J) { return zcs[(J - cy0) * WC + (I - cx0)]; };
      double pz;
      if ((gx & 1) == 0) pz = Zc(gx >> 1, gy >> 1);                                   // even-even
      else pz = 0.5 * (Zc((gx - 1) >> 1, (gy - 1) >> 1) + Zc((gx + 1) >> 1, (gy + 1) >> 1));  // odd-odd
      zp[idx] += pz;
    }
  }
  __syncthreads();
  // black nodes of the 1-halo region: z_b = (r − Σ A z_red)/D
  for (int idx = threadIdx.x; idx < W1 * H1; idx += TT) {
    const int ly = idx / W1, lx = idx - ly * W1;
    const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
    double v = 0.0;
    if (gx >= 0 && gx < n0 && gy >= 0 && gy < n0 && ((gx + gy) & 1) == 1) {
      const Sten st = sten_edges(es, ns, W2, lx + 1, ly + 1, gx, gy, m, bc);
      const int c = (ly + 1) * W2 + lx + 1;
      v = (rs[idx] - (st.e * zp[c + 1] + st.w * zp[c - 1] + st.n * zp[c + W2] + st.s * zp[c - W2])) / st.d;
    }
    zb[idx] = v;
  }
  __syncthreads();
  double rz = 0.0;
#pragma unroll
  for (int q = 0; q < TY / 8; ++q) {
    const int ly = ty0 + 8 * q, gx = x0 + tx, gy = y0 + ly;
    if (gx < n0 && gy < n0) {
      const int c1 = (ly + 1) * W1 + tx + 1;
      double zv;
      if (((gx + gy) & 1) == 0) {
        const Sten st = sten_edges(es, ns, W2, tx + 2, ly + 2, gx, gy, m, bc);
        zv = (rs[c1] - (st.e * zb[c1 + 1] + st.w * zb[c1 - 1] + st.n * zb[c1 + W1] + st.s * zb[c1 - W1])) / st.d;
      } else {
        zv = zb[c1];
      }
      z_out[off + (int64_t)gy * n0 + gx] = zv;
      rz = fma(rs[c1], zv, rz);
    }
  }
  if (!finest) return;
  double t0, t1;
  if (reduce2_last(rz, 0.0, partial, maxp, counter, b, t0, t1) && threadIdx.x == 0) {
    const double old = scal[b * S_NSCAL + S_RZ];
    scal[b * S_NSCAL + S_BETA] = flags[b * F_NFLAGS + F_ITERS] == 0 ? 0.0 : t0 / old;
    scal[b * S_NSCAL + S_RZ] = t0;
  }
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
inline int64_t tile_parts(int m) {
  return (int64_t)((m + 1 + TX - 1) / TX) * ((m + 1 + TY - 1) / TY);
}

}  // namespace

size_t solver_bytes(int m, int B, int hist_cap) {
  size_t tot = 0;
  int g = m, lev = 0;
  for (;;) {
    const size_t N = (size_t)(g + 1) * (g + 1);
    tot += N * B * sizeof(double) * (lev == 0 ? 8 : 4);  // level 0: u r r2 z z2 p0 p1 (+k by caller); else k r z z2
    ++lev;
    if (g <= 4 || g % 2 != 0) { tot += N * N * B * sizeof(double); break; }
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
    L.k = (l > 0) ? (double*)take(vb) : nullptr;  // level 0's k is the caller's buffer
    L.D = L.E = L.Nw = nullptr;                     // stencils are recomputed from k in-tile
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
dim3 tile_grid(const SolverLevel& L, int B) {
  return dim3((unsigned)((L.m + 1 + TX - 1) / TX), (unsigned)((L.m + 1 + TY - 1) / TY), (unsigned)B);
}
dim3 ctile_grid(const SolverLevel& C, int B) {
  return dim3((unsigned)((C.m + 1 + CXT - 1) / CXT), (unsigned)((C.m + 1 + CYT - 1) / CYT), (unsigned)B);
}

// Preconditioner z = M r on level 0. With `fused_down` the level-0 pre-smoother already ran
// inside pcg_update_down (z holds the pre-smoothed correction).
void vcycle(Ctx* ctx, int bc, int B, bool fused_down) {
  SolverWork& w = ctx->solver;
  cudaStream_t st = ctx->stream;
  double2* part = reinterpret_cast<double2*>(w.partial);
  if (w.nlev == 1) {
    {
      KScope ks(ctx, "mg_coarse_solve");
      coarse_solve_kernel<<<(B + 63) / 64, 64, 0, st>>>(w.nc, B, w.chol, w.r_cur, w.lev[0].z2, w.flags);
    }
    KScope ks(ctx, "pcg_dot_rz");
    dot_rz_kernel<<<dim3(nblocks(w.lev[0].N), 1, B), NT, 0, st>>>(geo_of(w.lev[0]), w.r_cur, w.lev[0].z2,
                                                                 w.scal, w.flags, part, w.max_parts, w.counter);
    OSC_CUDA(cudaGetLastError());
    return;
  }
  for (int l = 0; l + 1 < w.nlev; ++l) {
    const SolverLevel& L = w.lev[l];
    const SolverLevel& C = w.lev[l + 1];
    if (l > 0 || !fused_down) {
      KScope ks(ctx, "mg_smooth_down");
      smooth_down_kernel<<<tile_grid(L, B), TT, 0, st>>>(geo_of(L), bc, L.k, l == 0 ? w.r_cur : L.r, L.z, w.flags);
    }
    KScope ks(ctx, "mg_restrict");
    restrict_kernel<<<ctile_grid(C, B), TT, 0, st>>>(geo_of(L), geo_of(C), bc, L.k, L.z, C.r, w.flags);
  }
  {
    const SolverLevel& C = w.lev[w.nlev - 1];
    KScope ks(ctx, "mg_coarse_solve");
    coarse_solve_kernel<<<(B + 63) / 64, 64, 0, st>>>(w.nc, B, w.chol, C.r, C.z2, w.flags);
  }
  for (int l = w.nlev - 2; l >= 0; --l) {
    const SolverLevel& L = w.lev[l];
    const SolverLevel& C = w.lev[l + 1];
    KScope ks(ctx, "mg_smooth_up");
    smooth_up_kernel<<<tile_grid(L, B), TT, 0, st>>>(geo_of(L), geo_of(C), bc, L.k, l == 0 ? w.r_cur : L.r, L.z, L.z2, C.z2,
                                                     l == 0 ? 1 : 0, w.scal, w.flags, part,
                                                     w.max_parts, w.counter);
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
  {  // hierarchy: injected k (fem.cpp:241-244) + coarsest Cholesky (fem.cpp:255-272)
    KScope ks(ctx, "mg_setup", w.nlev);
    for (int l = 0; l + 1 < w.nlev; ++l) {
      const SolverLevel& L = w.lev[l];
      const SolverLevel& C = w.lev[l + 1];
      inject_kernel<<<dim3(nblocks(C.N), B), NT, 0, st>>>(geo_of(L), geo_of(C), L.k, C.k);
    }
    const SolverLevel& C = w.lev[w.nlev - 1];
    coarse_factor_kernel<<<(B + 63) / 64, 64, 0, st>>>(geo_of(C), bc, B, C.k, w.chol);
    OSC_CUDA(cudaGetLastError());
  }
  SolverLevel& L0 = w.lev[0];
  const Geo g0 = geo_of(L0);
  w.r_cur = L0.r;
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
  const bool multilevel = w.nlev > 1;
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
      pcg_apply_kernel<<<tile_grid(L0, B), TT, 0, st>>>(g0, bc, L0.k, L0.z2, p_old, p_new, w.scal, w.flags,
                                                        part, w.max_parts, w.counter);
    }
    {
      KScope ks(ctx, "pcg_update_down");
      double* r_next = (w.r_cur == L0.r) ? w.r2 : L0.r;
      pcg_update_down_kernel<<<tile_grid(L0, B), TT, 0, st>>>(g0, bc, prob->tol, L0.k, p_new, w.u, w.r_cur,
                                                              r_next, L0.z, w.scal, w.flags, part, w.max_parts,
                                                              w.counter, w.n_active, w.hist, w.hist_cap);
    }
    w.r_cur = (w.r_cur == L0.r) ? w.r2 : L0.r;
    // single-level: the "pre-smoothed" z is overwritten by the exact coarse solve
    vcycle(ctx, bc, B, multilevel);
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
