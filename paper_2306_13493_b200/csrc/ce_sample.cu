// K1 + K2: batched circulant-embedding sample with the coarse/fine restriction fused into
// the epilogue. Replaces, per sample, NormalStream::fill (src/rng.cpp:65-67),
// EmbeddingOperator::sample_into (src/embedding.cpp:165-174) with UnitaryDft::forward_real
// (src/fft.cpp:48-56), restrict_to (src/embedding.cpp:183-203) and the exp() of
// assemble_and_solve (src/fem.cpp:324-329).
//
// u = Re(F w) + Im(F w), w = √λ ⊙ ξ, F the unitary 2-D DFT with + sign (fft.hpp:11), only
// the R-block p ∈ [0,m]² is ever read, so:
//   pass 1 (rows, along x): two real rows q1 = 2r, 2r+1 are packed as one complex row
//           z = w_a + i w_b, FFT'd in shared memory (Stockham radix-8), and unpacked into
//           the half spectra X_a[p0], X_b[p0] for the needed p0 only (p0 ≤ m, stride cs);
//   pass 2 (columns, along y): for each needed p0 the length-n column of X is FFT'd and only
//           p1 ≤ m (stride cs) is kept; u = (Re+Im)/n, k = exp(u) written straight into the
//           solver's fine and stride-2 coarse conductivity arrays.
// The intermediate X is [sample][p][q1] complex (transposed: pass-1 writes of a row pair fill
// 32-byte sectors, pass-2 column reads are contiguous).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "osc_device.cuh"
#include "osc_internal.cuh"

namespace osc {

namespace {

// elements per thread for a length-n transform
inline int elems_for(int n) { return n >= 8 ? 8 : n; }

// L2 residency hints of the compile-time-n passes. √λ (n² doubles, read by every sample) is kept
// (evict_last); ξ rows and the half-spectrum intermediate pass through once (evict_first) — without
// the hints the streams evict √λ and the row pass re-reads most of it from DRAM for every sample
// (resident ξ at n = 2048: 26 MB of the 60 MB read per sample).
__device__ __forceinline__ uint64_t l2_policy_stream() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_keep() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ldg_hint(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg_hint(double2* a, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

// Sup-norm mode of the column passes (smoothing_error_estimate, embedding.cpp:217-219): instead of
// storing the field, every thread folds |z| of its outputs into v and the CTA commits max to sup[b]
// (non-negative doubles order like their bit patterns, so one integer atomicMax per warp does it).
__device__ __forceinline__ void sup_commit(double v, unsigned long long* __restrict__ sup_b) {
  // called by every thread of the CTA, converged; CTAs are powers of two (≥ 2 threads), so the live
  // lanes of a warp are 0 … 2^k − 1 and the butterfly over them leaves the warp's max in lane 0
  const unsigned mask = __activemask();
  const int lane = threadIdx.x & 31;
  for (int o = 16; o; o >>= 1) {
    const double w = __shfl_xor_sync(mask, v, o);
    if ((mask >> (lane ^ o)) & 1u) v = fmax(v, w);
  }
  if (lane == 0) atomicMax(sup_b, (unsigned long long)__double_as_longlong(v));
}

// Pass 1: one CTA slot per (row pair, sample). Writes the TRANSPOSED half spectrum
// inter[b][p][q1] (q1 fastest), so rows q1a, q1b land in one 32-byte sector and pass 2 reads
// each column as one contiguous run.
template <int E, int MAXT>
__global__ void __launch_bounds__(MAXT, 1024 / MAXT) ce_rows_kernel(
    const double* __restrict__ sqrt_lam, const double* __restrict__ xi, uint64_t seed,
    uint32_t ell, uint64_t index0, int n, int NT, int P, int cs, const double2* __restrict__ tw,
    double2* __restrict__ inter) {
  extern __shared__ double2 smem[];
  const int T = n / E;                      // threads per transform (power of two)
  const int t = threadIdx.x >> (31 - __clz(T));  // transform slot in this CTA
  const int lt = threadIdx.x & (T - 1);          // lane within the transform
  const int rp = blockIdx.x * NT + t;       // row pair
  const int b = blockIdx.y;                 // sample within the chunk
  const bool valid = rp < n / 2;
  const int q1a = 2 * rp, q1b = 2 * rp + 1;
  double2* x = smem + t * fpad_len(n);
  const int64_t s = (int64_t)n * n;
  const PhiloxKeys keys = philox_keys(seed);
  if (valid) {
    const double2* la = reinterpret_cast<const double2*>(sqrt_lam + (int64_t)q1a * n);
    const double2* lb = reinterpret_cast<const double2*>(sqrt_lam + (int64_t)q1b * n);
#pragma unroll
    for (int g = 0; g < E / 2; ++g) {
      const int c = lt + g * T;  // column pair: columns 2c, 2c+1
      double2 xa, xb;
      if (xi) {
        const double* xr = xi + (int64_t)b * s;
        xa = __ldg(reinterpret_cast<const double2*>(xr + (int64_t)q1a * n) + c);
        xb = __ldg(reinterpret_cast<const double2*>(xr + (int64_t)q1b * n) + c);
      } else {
        const uint64_t idx = index0 + (uint64_t)b;
        xa = normal_pair_k(keys, ell, idx, (uint32_t)((int64_t)q1a * (n / 2) + c));
        xb = normal_pair_k(keys, ell, idx, (uint32_t)((int64_t)q1b * (n / 2) + c));
      }
      const double2 sa = __ldg(la + c), sb = __ldg(lb + c);
      // z[q0] = w(q0, q1a) + i w(q0, q1b)
      x[fpad(2 * c)] = make_double2(sa.x * xa.x, sb.x * xb.x);
      x[fpad(2 * c + 1)] = make_double2(sa.y * xa.y, sb.y * xb.y);
    }
  }
  __syncthreads();
  fft_smem<E>(x, n, lt, tw);
  if (valid) {
    double2* out = inter + (int64_t)b * P * n + q1a;
    for (int p = lt; p < P; p += T) {
      const int p0 = p * cs;
      const double2 zp = x[fpad(p0)];
      const double2 zm = x[fpad((n - p0) & (n - 1))];
      // X_a = (Z[p] + conj Z[-p]) / 2,  X_b = (Z[p] - conj Z[-p]) / (2i)
      double2* o = out + (int64_t)p * n;
      o[0] = make_double2(0.5 * (zp.x + zm.x), 0.5 * (zp.y - zm.y));
      o[1] = make_double2(0.5 * (zp.y + zm.y), 0.5 * (zm.x - zp.x));
    }
  }
}

// Pass 2: NT columns of one sample per CTA; column j of the transposed intermediate is one
// contiguous n-element run (coalesced 16-byte loads).
template <int E, int MAXT>
__global__ void __launch_bounds__(MAXT, 1024 / MAXT) ce_cols_kernel(
    const double2* __restrict__ inter, int n, int m, int NT, int P, int cs, double inv_n,
    int do_exp, const double2* __restrict__ tw, double* __restrict__ out_fine,
    double* __restrict__ out_coarse, int* __restrict__ bad_flag, unsigned long long* __restrict__ sup) {
  extern __shared__ double2 smem[];
  const int T = n / E;
  const int t = threadIdx.x >> (31 - __clz(T));
  const int lt = threadIdx.x & (T - 1);
  const int b = blockIdx.y;
  const int j0 = blockIdx.x * NT;
  const double2* src = inter + ((int64_t)b * P + j0) * n;
  const int ncols = min(NT, P - j0);
  const int ld = fpad_len(n);
  const int ln = 31 - __clz(n);
  for (int idx = threadIdx.x; idx < NT * n; idx += blockDim.x) {
    const int tt = idx >> ln, q1 = idx & (n - 1);
    smem[tt * ld + fpad(q1)] = (idx < ncols * n) ? __ldg(src + idx) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_smem<E>(smem + t * ld, n, lt, tw);

  // outputs: rows p1 = i*cs ≤ m, columns p0 = j*cs
  const int n_rows = m / cs + 1;
  const int mf = m + 1, mc = m / 2 + 1;
  double* of = out_fine ? out_fine + (int64_t)b * mf * mf : nullptr;
  double* oc = out_coarse ? out_coarse + (int64_t)b * mc * mc : nullptr;
  int bad = 0;
  double vmax = 0.0;
  const int lnt = 31 - __clz(NT);  // NT is a power of two
  for (int idx = threadIdx.x; idx < NT * n_rows; idx += blockDim.x) {
    const int tt = idx & (NT - 1), i = idx >> lnt;
    const int j = j0 + tt;
    if (j >= P) continue;
    const int p1 = i * cs, p0 = j * cs;
    const double2 v = smem[tt * ld + fpad(p1)];
    const double zval = (v.x + v.y) * inv_n;
    if (!isfinite(zval)) bad = 1;
    vmax = fmax(vmax, fabs(zval));
    const double o = do_exp ? exp(zval) : zval;
    if (of) of[(int64_t)p1 * mf + p0] = o;
    if (oc && ((p0 | p1) & 1) == 0) oc[(int64_t)(p1 >> 1) * mc + (p0 >> 1)] = o;
  }
  if (bad && bad_flag) atomicOr(bad_flag + b, 1);
  if (sup) sup_commit(vmax, sup + b);
}

// ---- compile-time-n path (n = 2^LOGN, 16 ≤ n ≤ 8192) ----------------------------------------------
// Same arithmetic as ce_rows_kernel / ce_cols_kernel (bit-identical results), restructured so the
// first and last Stockham stages run from registers:
//   rows: each thread draws its stage-1 operands z[lt + r·T] directly (the two lanes of a pair split
//         each Philox block: even lanes draw the even-r blocks, odd lanes the odd-r ones, and swap
//         halves with one shuffle), so the input never goes through shared memory;
//   cols: each thread loads its stage-1 operands straight from the column (coalesced 16-B loads),
//         and keeps the last stage's outputs p1 = j + r·Ns in registers for the exp() epilogue.
// Shared-memory round trips per transform: rows 5 → 4, cols 5 → 3; all index arithmetic is static.
// A/B build knobs: cap the CTAs-per-SM the register budget is sized for (0 = 1024/THREADS, ≤ 64 regs)
template <int LOGN>
struct FftPlan {
  static constexpr int n = 1 << LOGN;
  static constexpr int T = n / 8;                    // threads per transform
  static constexpr int NT = T >= 256 ? 1 : (256 / T < n / 2 ? 256 / T : n / 2);  // transforms per CTA (divides n/2)
  static constexpr int THREADS = NT * T;
  static constexpr int NSTAGE8 = LOGN / 3;           // radix-8 stages
  static constexpr int REM = LOGN % 3;               // log2 of the final radix (0: none)
  // padded transform stride (≥ fpad_len); from T ≥ 32 on transforms sit in different warps and the
  // stride only matters to the row pass's unpack, where two transforms' Z[p], Z[p+1] must fall in four
  // different 16-byte bank groups (stride ≡ 2 mod 8)
  static constexpr int LD = n + (n >> 3) + (LOGN >= 8 ? 2 : 1);
  static constexpr int MINB = THREADS >= 1024 ? 1 : (1024 / THREADS < 32 ? 1024 / THREADS : 32);  // ≤ 64 regs
  // Row pass: at least two row pairs (four rows) per CTA wherever 1024 threads allow, so that the
  // unpack writes whole 128-byte lines of the intermediate (4 rows × 2 interleaved columns × 16 B)
  static constexpr int NTR = T >= 1024 ? 1 : (T >= 256 ? 2 : NT);
};

// Twiddles of one Stockham stage (radix R, sub-length Ns = 2^LNS) for this thread's G = 8/R butterflies.
// They do not depend on the data, so each stage loads them BEFORE the barrier that publishes the
// previous stage's outputs: the L1 latency overlaps the barrier wait.
// They come from the level's per-stage tables (upload_twiddles): stage LNS keeps W^{rk} as
// [r − 1][k], k < Ns, at offset 2^LNS − 8 behind the plain table, so the lanes of a warp (consecutive
// k) read consecutive 16-byte entries — 1 to 4 L1 wavefronts per load. Indexing the plain table
// tw[(r k) << TWS] spread a warp's load over up to 32 lines; with 7 loads per thread and stage the
// twiddles took about as many L1/shared data-pipe cycles as the transform's own exchanges, and that
// pipe — not issue, fp64 or HBM — bounds both passes.
template <int LOGN, int R, int LNS>
struct StageTw {
  double2 w[8 / R][R > 1 ? R - 1 : 1];
  __device__ __forceinline__ void load(int lt, const double2* __restrict__ tw) {
    constexpr int n = 1 << LOGN, T = n / 8, G = 8 / R, Ns = 1 << LNS;
    const double2* st = tw + n + (Ns - 8);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int k = (lt + g * T) & (Ns - 1);
#pragma unroll
      for (int r = 1; r < R; ++r) w[g][r - 1] = __ldg(&st[(r - 1) * Ns + k]);
    }
  }
};

// One Stockham stage from shared memory into registers (radix R, sub-length 2^LNS ≥ 8), E = 8 values
// per thread held as G = 8/R butterflies; v[g][r] receives the butterfly outputs.
template <int LOGN, int R, int LNS>
__device__ __forceinline__ void stage_load_compute(const double2* x, int lt, const StageTw<LOGN, R, LNS>& t,
                                                   double2 (&v)[8 / R][R]) {
  constexpr int n = 1 << LOGN, T = n / 8, nR = n / R, G = 8 / R;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j = lt + g * T;
#pragma unroll
    for (int r = 0; r < R; ++r) v[g][r] = x[fpad(j + r * nR)];
#pragma unroll
    for (int r = 1; r < R; ++r) v[g][r] = cmul(v[g][r], t.w[g][r - 1]);
    dft_r<R>(v[g]);
  }
}

template <int LOGN, int R, int LNS>
__device__ __forceinline__ void stage_store(double2* x, int lt, const double2 (&v)[8 / R][R]) {
  constexpr int T = (1 << LOGN) / 8, G = 8 / R, Ns = 1 << LNS;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j = lt + g * T;
    const int k = j & (Ns - 1);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) x[fpad(base + r * Ns)] = v[g][r];
  }
}

// Middle stages (radix 8, LNS = 3, 6, … below the final stage): twiddles, barrier (previous stage's
// stores visible), loads + butterflies, barrier (all loads done), stores. The caller has stored the
// previous stage and not yet synchronised.
template <int LOGN, int LNS>
__device__ __forceinline__ void mid_stages(double2* x, int lt, const double2* __restrict__ tw) {
  using PL = FftPlan<LOGN>;
  constexpr int last_lns = PL::REM ? 3 * PL::NSTAGE8 : 3 * (PL::NSTAGE8 - 1);  // LNS of the final stage
  if constexpr (LNS < last_lns) {
    StageTw<LOGN, 8, LNS> t;
    t.load(lt, tw);
    __syncthreads();
    double2 v[1][8];
    stage_load_compute<LOGN, 8, LNS>(x, lt, t, v);
    __syncthreads();
    stage_store<LOGN, 8, LNS>(x, lt, v);
    mid_stages<LOGN, LNS + 3>(x, lt, tw);
  }
}

// Final stage: radix 2^REM (or 8 when LOGN % 3 == 0), LNS = LOGN − log2(R); outputs of butterfly g
// are p = (lt + g·T) + r·n/R.
template <int LOGN>
struct LastStage {
  static constexpr int R = FftPlan<LOGN>::REM == 0 ? 8 : (1 << FftPlan<LOGN>::REM);
  static constexpr int G = 8 / R;
  static constexpr int LNS = LOGN - (R == 8 ? 3 : (R == 4 ? 2 : 1));
  using Tw = StageTw<LOGN, R, LNS>;
};

// Stage 1 (Ns = 1, no twiddles) on register operands v[r] = x[lt + r·T], stored to shared memory.
template <int LOGN>
__device__ __forceinline__ void first_stage_store(double2* x, int lt, double2 (&v)[8]) {
  dft8(v);
#pragma unroll
  for (int r = 0; r < 8; ++r) x[fpad(lt * 8 + r)] = v[r];
}

// Stage-1 operands of the row pair (q1a, q1a + 1) of sample b: v[r] = z[lt + r·T] with
// z[q0] = √λ(q0, q1a)·ξ(q0, q1a) + i·√λ(q0, q1b)·ξ(q0, q1b). T is even, so q0 has lt's parity and
// lanes lt, lt^1 need the two halves of the same normal pair c = (lt >> 1) + r·T/2: the even lane
// draws the even-r Philox blocks, the odd lane the odd-r ones, and they trade halves by shuffle.
template <int LOGN, bool XI>
__device__ __forceinline__ void rows_operands(const double* __restrict__ sqrt_lam, const double* __restrict__ xi,
                                              const PhiloxKeys& keys, uint32_t ell, uint64_t idx, int b, int q1a,
                                              int lt, double2 (&v)[8]) {
  constexpr int n = 1 << LOGN, T = n / 8;
  const int64_t s = (int64_t)n * n;
  const bool odd = lt & 1;
  double ra[8], rb[8];  // ξ(q0, q1a), ξ(q0, q1b)
  if constexpr (XI) {
    const double* xa = xi + (int64_t)b * s + (int64_t)q1a * n;
    const double* xb = xa + n;
    const uint64_t once = l2_policy_stream();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      ra[r] = ldg_hint(xa + lt + r * T, once);
      rb[r] = ldg_hint(xb + lt + r * T, once);
    }
  } else {
    const uint32_t ja = (uint32_t)q1a * (n / 2) + (lt >> 1), jb = ja + n / 2;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      // this lane draws block r = 2h + odd for both rows; keeps its half, trades the other
      const uint32_t off = (uint32_t)(2 * h + (odd ? 1 : 0)) * (T / 2);
      const double2 pa = normal_pair_k(keys, ell, idx, ja + off);
      const double2 pb = normal_pair_k(keys, ell, idx, jb + off);
      const double keep_a = odd ? pa.y : pa.x, give_a = odd ? pa.x : pa.y;
      const double keep_b = odd ? pb.y : pb.x, give_b = odd ? pb.x : pb.y;
      const double got_a = __shfl_xor_sync(0xffffffffu, give_a, 1);
      const double got_b = __shfl_xor_sync(0xffffffffu, give_b, 1);
      // even lane: r = 2h is its own draw, r = 2h+1 came from the odd lane; odd lane: the reverse
      ra[2 * h] = odd ? got_a : keep_a;
      ra[2 * h + 1] = odd ? keep_a : got_a;
      rb[2 * h] = odd ? got_b : keep_b;
      rb[2 * h + 1] = odd ? keep_b : got_b;
    }
  }
  const double* la = sqrt_lam + (int64_t)q1a * n + lt;
  if constexpr (XI) {
    const uint64_t keep = l2_policy_keep();
#pragma unroll
    for (int r = 0; r < 8; ++r)
      v[r] = make_double2(ldg_hint(la + r * T, keep) * ra[r], ldg_hint(la + n + r * T, keep) * rb[r]);
  } else {
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = make_double2(__ldg(la + r * T) * ra[r], __ldg(la + n + r * T) * rb[r]);
  }
}

// Intermediate layout of the compile-time-n passes: CE_IL columns interleaved,
// inter[b][p/IL][q1][p%IL] (⌈P/IL⌉ groups per sample). The row pass's lanes for columns p … p+IL−1
// fill IL·16 contiguous bytes per row (IL = 2: one 32-byte sector), and the column pass reads its two
// adjacent columns as one 32-byte run per q1; wider groups help the row pass and hurt the column pass.
// columns interleaved per q1 run (power of two). Measured at n = 2048: IL 2 → rows 28.5 + cols 17.4 µs;
// 4 → 27.4 + 20.7; 8 → 26.7 + 24.8
constexpr int CE_IL = 2;
__device__ __forceinline__ int64_t inter_pair_idx(int b, int Ph, int n, int p, int q1) {
  return (((int64_t)b * Ph + p / CE_IL) * n + q1) * CE_IL + (p & (CE_IL - 1));
}
__host__ __device__ __forceinline__ int inter_groups(int P) { return (P + CE_IL - 1) / CE_IL; }

// Unpack the CTA's NTR row pairs (rows 2·rp0 … 2·rp0 + 2·NTR − 1) into the intermediate. Row q1 = 2t + w
// of transform t: X_a (w = 0) = (Z[p] + conj Z[−p]) / 2, X_b (w = 1) = (Z[p] − conj Z[−p]) / (2i).
// NTR ≥ 2: one 16-byte value per thread and step in address order (interleaved column p & 1 fastest,
// then the row, then the column pair), so a warp's store covers whole 128-byte lines (four rows × one
// column pair) instead of 16 scattered 32-byte sectors — the stores took a quarter of the pass's L1
// data-pipe cycles. NTR = 1: both rows of the pair per thread (half lines).
template <int LOGN, int NTR, bool HINT>
__device__ __forceinline__ void rows_unpack(const double2* smem, double2* __restrict__ inter, int b, int P, int cs,
                                            int rp0) {
  using PL = FftPlan<LOGN>;
  constexpr int n = PL::n, ROWS = 2 * NTR, THREADS = NTR * PL::T;
  const int Ph = inter_groups(P);
  const uint64_t once = HINT ? l2_policy_stream() : 0;
  auto put = [&](double2* a, double2 v) {
    if constexpr (HINT) stg_hint(a, v, once);
    else *a = v;
  };
  if constexpr (NTR == 1) {
    for (int p = threadIdx.x; p < P; p += THREADS) {
      const int p0 = p * cs;
      const double2 zp = smem[fpad(p0)];
      const double2 zm = smem[fpad((n - p0) & (n - 1))];
      double2* o = inter + inter_pair_idx(b, Ph, n, p, 2 * rp0);
      put(o, make_double2(0.5 * (zp.x + zm.x), 0.5 * (zp.y - zm.y)));
      put(o + CE_IL, make_double2(0.5 * (zp.y + zm.y), 0.5 * (zm.x - zp.x)));  // row 2·rp0 + 1
    }
  } else {
    const int items = CE_IL * ROWS * Ph;
    for (int idx = threadIdx.x; idx < items; idx += THREADS) {
      const int pl = idx % CE_IL, q1l = (idx / CE_IL) % ROWS, pp = idx / (CE_IL * ROWS);
      const int p = CE_IL * pp + pl;
      if (p >= P) continue;
      const int p0 = p * cs;
      const double2* x = smem + (q1l >> 1) * PL::LD;
      const double2 zp = x[fpad(p0)];
      const double2 zm = x[fpad((n - p0) & (n - 1))];
      const double2 o = (q1l & 1) ? make_double2(0.5 * (zp.y + zm.y), 0.5 * (zm.x - zp.x))
                                  : make_double2(0.5 * (zp.x + zm.x), 0.5 * (zp.y - zm.y));
      put(inter + inter_pair_idx(b, Ph, n, p, 2 * rp0 + q1l), o);
    }
  }
}

// NTR row pairs per CTA. Resident ξ (a memory-bound pass) runs FftPlan::NTR ≥ 2 pairs for the whole-line
// stores; the device-Philox draw is issue-heavy and overlaps better across many small CTAs, so it
// keeps the column pass's transforms-per-CTA (measured at n = 2048: Philox 23.5 vs 25.5 µs per sample
// with 1 vs 2 pairs, resident ξ 20.4 vs 18.3).
template <int LOGN, int NTR, bool XI>
__global__ void __launch_bounds__(NTR * FftPlan<LOGN>::T, (1024 / (NTR * FftPlan<LOGN>::T) < 32 ? (1024 / (NTR * FftPlan<LOGN>::T) < 1 ? 1 : 1024 / (NTR * FftPlan<LOGN>::T)) : 32)) ce_rows_t_kernel(
    const double* __restrict__ sqrt_lam, const double* __restrict__ xi, uint64_t seed, uint32_t ell,
    uint64_t index0, int P, int cs, const double2* __restrict__ tw, double2* __restrict__ inter) {
  using PL = FftPlan<LOGN>;
  constexpr int T = PL::T;
  extern __shared__ double2 smem[];
  const int t = threadIdx.x / T;  // transform slot in this CTA
  const int lt = threadIdx.x % T;
  const int rp0 = blockIdx.x * NTR;  // first row pair of the CTA (n/2 is a multiple of NTR)
  const int b = blockIdx.y;
  const int q1a = 2 * (rp0 + t);
  double2* x = smem + t * PL::LD;
  double2 v[8];
  rows_operands<LOGN, XI>(sqrt_lam, xi, philox_keys(seed), ell, index0 + (uint64_t)b, b, q1a, lt, v);
  first_stage_store<LOGN>(x, lt, v);
  mid_stages<LOGN, 3>(x, lt, tw);
  {
    using LS = LastStage<LOGN>;
    typename LS::Tw t;
    t.load(lt, tw);
    __syncthreads();
    double2 w[LS::G][LS::R];
    stage_load_compute<LOGN, LS::R, LS::LNS>(x, lt, t, w);
    __syncthreads();
    stage_store<LOGN, LS::R, LS::LNS>(x, lt, w);
    __syncthreads();
  }
  rows_unpack<LOGN, NTR, XI>(smem, inter, b, P, cs, rp0);
}

template <int LOGN>
__global__ void __launch_bounds__(FftPlan<LOGN>::THREADS, FftPlan<LOGN>::MINB) ce_cols_t_kernel(
    const double2* __restrict__ inter, int m, int P, int cs, double inv_n, int do_exp,
    const double2* __restrict__ tw, double* __restrict__ out_fine, double* __restrict__ out_coarse,
    int* __restrict__ bad_flag, unsigned long long* __restrict__ sup) {
  using PL = FftPlan<LOGN>;
  using LS = LastStage<LOGN>;
  constexpr int n = PL::n, T = PL::T;
  extern __shared__ double2 smem[];
  const int t = threadIdx.x / T;
  const int lt = threadIdx.x % T;
  const int b = blockIdx.y;
  const int j = blockIdx.x * PL::NT + t;  // column (p index) of this transform
  const bool valid = j < P;
  double2* x = smem + t * PL::LD;
  {
    double2 v[8];
    const double2* src = inter + inter_pair_idx(b, inter_groups(P), n, valid ? j : 0, lt);
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = valid ? __ldg(src + CE_IL * r * T) : make_double2(0.0, 0.0);
    first_stage_store<LOGN>(x, lt, v);
  }
  mid_stages<LOGN, 3>(x, lt, tw);
  double2 w[LS::G][LS::R];
  {
    typename LS::Tw t;
    t.load(lt, tw);
    __syncthreads();
    stage_load_compute<LOGN, LS::R, LS::LNS>(x, lt, t, w);
  }
  const int mf = m + 1, mc = m / 2 + 1;
  double* of = out_fine ? out_fine + (int64_t)b * mf * mf : nullptr;
  double* oc = out_coarse ? out_coarse + (int64_t)b * mc * mc : nullptr;
  const int p0 = j * cs;
  int bad = 0;
  double vmax = 0.0;
#pragma unroll
  for (int g = 0; g < LS::G; ++g)
#pragma unroll
    for (int r = 0; r < LS::R; ++r) {
      const int p1 = lt + g * T + r * (n / LS::R);  // output row of this register
      if (!valid || p1 > m || (p1 & (cs - 1))) continue;
      const double zval = (w[g][r].x + w[g][r].y) * inv_n;
      if (!isfinite(zval)) bad = 1;
      vmax = fmax(vmax, fabs(zval));
      const double o = do_exp ? exp(zval) : zval;
      if (of) of[(int64_t)p1 * mf + p0] = o;
      if (oc && ((p0 | p1) & 1) == 0) oc[(int64_t)(p1 >> 1) * mc + (p0 >> 1)] = o;
    }
  if (bad && bad_flag) atomicOr(bad_flag + b, 1);
  if (sup) sup_commit(vmax, sup + b);
}

// 32 aligned bytes (two adjacent complex values) through the read-only path in one instruction
__device__ __forceinline__ void ldg256(const double2* p, double2& a, double2& b, uint64_t pol) {
  asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
               : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
               : "l"(p), "l"(pol));
}

// Column pass with two columns per thread (32 ≤ n ≤ 2048; ce_cols_t_kernel below and above): the same stages as ce_cols_t_kernel
// applied to columns j and j + 1 held by one thread, so each barrier interval carries two independent
// butterflies (twice the loads in flight) and every twiddle load serves both columns.
template <int LOGN, int R, int LNS>
__device__ __forceinline__ void stage_load_compute2(const double2* x0, const double2* x1, int lt,
                                                    const StageTw<LOGN, R, LNS>& t, double2 (&v)[2][8 / R][R]) {
  constexpr int n = 1 << LOGN, T = n / 8, nR = n / R, G = 8 / R;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j = lt + g * T;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      v[0][g][r] = x0[fpad(j + r * nR)];
      v[1][g][r] = x1[fpad(j + r * nR)];
    }
  }
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[c][g][r] = cmul(v[c][g][r], t.w[g][r - 1]);
      dft_r<R>(v[c][g]);
    }
}

template <int LOGN, int LNS>
__device__ __forceinline__ void mid_stages2(double2* x0, double2* x1, int lt, const double2* __restrict__ tw) {
  using PL = FftPlan<LOGN>;
  constexpr int last_lns = PL::REM ? 3 * PL::NSTAGE8 : 3 * (PL::NSTAGE8 - 1);
  if constexpr (LNS < last_lns) {
    StageTw<LOGN, 8, LNS> t;
    t.load(lt, tw);
    __syncthreads();
    double2 v[2][1][8];
    stage_load_compute2<LOGN, 8, LNS>(x0, x1, lt, t, v);
    __syncthreads();
    stage_store<LOGN, 8, LNS>(x0, lt, v[0]);
    stage_store<LOGN, 8, LNS>(x1, lt, v[1]);
    mid_stages2<LOGN, LNS + 3>(x0, x1, lt, tw);
  }
}

template <int LOGN>
struct Cols2Plan {
  static constexpr int THREADS = FftPlan<LOGN>::THREADS;
  static constexpr int MINB = THREADS >= 512 ? 1 : 512 / THREADS;  // ≤ 128 registers
};

template <int LOGN>
__global__ void __launch_bounds__(Cols2Plan<LOGN>::THREADS, Cols2Plan<LOGN>::MINB) ce_cols2_t_kernel(
    const double2* __restrict__ inter, int m, int P, int cs, double inv_n, int do_exp,
    const double2* __restrict__ tw, double* __restrict__ out_fine, double* __restrict__ out_coarse,
    int* __restrict__ bad_flag, unsigned long long* __restrict__ sup) {
  using PL = FftPlan<LOGN>;
  using LS = LastStage<LOGN>;
  constexpr int n = PL::n, T = PL::T;
  extern __shared__ double2 smem[];
  const int t = threadIdx.x / T;
  const int lt = threadIdx.x % T;
  const int b = blockIdx.y;
  const int j0 = 2 * (blockIdx.x * PL::NT + t);  // columns j0, j0 + 1
  double2* x0 = smem + (2 * t) * PL::LD;
  double2* x1 = x0 + PL::LD;
  {
    double2 v0[8], v1[8];
    const bool ok0 = j0 < P, ok1 = j0 + 1 < P;
    // columns j0 (even) and j0 + 1 sit side by side: one aligned 32-byte run per q1, read by one
    // 256-bit load (column j0 + 1 of an odd P is allocated but never written: its values are dropped)
    const double2* s0 = inter + inter_pair_idx(b, inter_groups(P), n, ok0 ? j0 : 0, lt);
    static_assert(CE_IL == 2, "the 256-bit load reads one interleaved column pair");
    const uint64_t once = l2_policy_stream();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      ldg256(s0 + CE_IL * r * T, v0[r], v1[r], once);
      if (!ok0) v0[r] = make_double2(0.0, 0.0);
      if (!ok1) v1[r] = make_double2(0.0, 0.0);
    }
    first_stage_store<LOGN>(x0, lt, v0);
    first_stage_store<LOGN>(x1, lt, v1);
  }
  mid_stages2<LOGN, 3>(x0, x1, lt, tw);
  double2 w[2][LS::G][LS::R];
  {
    typename LS::Tw tt;
    tt.load(lt, tw);
    __syncthreads();
    stage_load_compute2<LOGN, LS::R, LS::LNS>(x0, x1, lt, tt, w);
  }
  const int mf = m + 1, mc = m / 2 + 1;
  double* of = out_fine ? out_fine + (int64_t)b * mf * mf : nullptr;
  double* oc = out_coarse ? out_coarse + (int64_t)b * mc * mc : nullptr;
  int bad = 0;
  double vmax = 0.0;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int j = j0 + c;
    if (j >= P) break;
    const int p0 = j * cs;
#pragma unroll
    for (int g = 0; g < LS::G; ++g)
#pragma unroll
      for (int r = 0; r < LS::R; ++r) {
        const int p1 = lt + g * T + r * (n / LS::R);
        if (p1 > m || (p1 & (cs - 1))) continue;
        const double zval = (w[c][g][r].x + w[c][g][r].y) * inv_n;
        if (!isfinite(zval)) bad = 1;
        vmax = fmax(vmax, fabs(zval));
        const double o = do_exp ? exp(zval) : zval;
        if (of) of[(int64_t)p1 * mf + p0] = o;
        if (oc && ((p0 | p1) & 1) == 0) oc[(int64_t)(p1 >> 1) * mc + (p0 >> 1)] = o;
      }
  }
  if (bad && bad_flag) atomicOr(bad_flag + b, 1);
  if (sup) sup_commit(vmax, sup + b);
}

template <int LOGN>
void launch_t(Ctx* ctx, const Level* L, const double* sqrt_lam, const double* xi_dev, uint64_t seed,
              uint32_t ell, uint64_t index0, int count, bool do_exp, double* out_fine, double* out_coarse,
              int* bad_flag, int cs, double2* inter, unsigned long long* sup) {
  using PL = FftPlan<LOGN>;
  const int m = L->m, P = m / cs + 1;
  const double2* tw = L->twiddle.as<double2>();
  const size_t sm = sizeof(double2) * (size_t)PL::NT * PL::LD;
  cudaStream_t st = ctx->stream;
  auto rows = [&](auto ntr, auto with_xi) {
    constexpr int NTR = decltype(ntr)::value;
    const size_t smr = sizeof(double2) * (size_t)NTR * PL::LD;
    auto kern = ce_rows_t_kernel<LOGN, NTR, decltype(with_xi)::value>;
    smem_attr(kern, smr);
    KScope ks(ctx, "ce_rows");
    kern<<<dim3((PL::n / 2) / NTR, count), NTR * PL::T, smr, st>>>(sqrt_lam, xi_dev, seed, ell, index0, P, cs, tw,
                                                                    inter);
    OSC_CUDA(cudaGetLastError());
  };
  if (xi_dev) rows(std::integral_constant<int, PL::NTR>{}, std::true_type{});
  else rows(std::integral_constant<int, PL::NT>{}, std::false_type{});
  // two columns per thread for 32 ≤ n ≤ 2048 (config 2: 277.7 → 208.6 ms per 12288 samples against one
  // column per thread). At n = 4096 the 512-thread, 128-register CTA leaves one CTA per SM: one
  // column per thread (64 registers, two CTAs) is faster there (72.3 → 66.7 µs per sample).
  if constexpr (LOGN >= 5 && LOGN <= 11) {
    auto kern = ce_cols2_t_kernel<LOGN>;
    smem_attr(kern, (2 * sm));
    KScope ks(ctx, "ce_cols");
    kern<<<dim3((P + 2 * PL::NT - 1) / (2 * PL::NT), count), PL::THREADS, 2 * sm, st>>>(
        inter, m, P, cs, 1.0 / PL::n, do_exp ? 1 : 0, tw, out_fine, out_coarse, bad_flag, sup);
    OSC_CUDA(cudaGetLastError());
    return;
  }
  {
    auto kern = ce_cols_t_kernel<LOGN>;
    smem_attr(kern, sm);
    KScope ks(ctx, "ce_cols");
    kern<<<dim3((P + PL::NT - 1) / PL::NT, count), PL::THREADS, sm, st>>>(inter, m, P, cs, 1.0 / PL::n,
                                                                           do_exp ? 1 : 0, tw, out_fine,
                                                                           out_coarse, bad_flag, sup);
    OSC_CUDA(cudaGetLastError());
  }
}

struct CeGeom {
  int E, T, NT, threads;
  size_t smem;
};

CeGeom rows_geom(int n) {
  CeGeom g;
  g.E = elems_for(n);
  g.T = n / g.E;
  g.NT = std::max(1, 256 / g.T);  // T > 256 only for n ≥ 4096: one transform per CTA
  g.NT = std::min(g.NT, std::max(1, n / 2));
  g.threads = g.NT * g.T;
  g.smem = sizeof(double2) * (size_t)g.NT * fpad_len(n);
  return g;
}

CeGeom cols_geom(int n, int P) {
  CeGeom g;
  g.E = elems_for(n);
  g.T = n / g.E;
  g.NT = std::max(1, 256 / g.T);  // power of two; columns beyond P are masked
  g.threads = g.NT * g.T;
  g.smem = sizeof(double2) * (size_t)g.NT * fpad_len(n);
  return g;
}

template <int E, int MAXT>
void launch_pair(Ctx* ctx, const Level* L, const double* sqrt_lam, const double* xi_dev,
                 uint64_t seed, uint32_t ell, uint64_t index0, int count, bool do_exp,
                 double* out_fine, double* out_coarse, int* bad_flag, int cs, double2* inter, unsigned long long* sup) {
  const int n = L->n, m = L->m;
  const int P = m / cs + 1;
  const double2* tw = L->twiddle.as<double2>();
  cudaStream_t st = ctx->stream;
  {
    const CeGeom g = rows_geom(n);
    const dim3 grid((n / 2 + g.NT - 1) / g.NT, count);
    auto kern = ce_rows_kernel<E, MAXT>;
    smem_attr(kern, g.smem);
    KScope ks(ctx, "ce_rows");
    kern<<<grid, g.threads, g.smem, st>>>(sqrt_lam, xi_dev, seed, ell, index0, n, g.NT, P, cs, tw, inter);
    OSC_CUDA(cudaGetLastError());
  }
  {
    const CeGeom g = cols_geom(n, P);
    const dim3 grid((P + g.NT - 1) / g.NT, count);
    auto kern = ce_cols_kernel<E, MAXT>;
    smem_attr(kern, g.smem);
    KScope ks(ctx, "ce_cols");
    kern<<<grid, g.threads, g.smem, st>>>(inter, n, m, g.NT, P, cs, 1.0 / n, do_exp ? 1 : 0, tw,
                                         out_fine, out_coarse, bad_flag, sup);
    OSC_CUDA(cudaGetLastError());
  }
}


// ---- mixed-radix path for padded embeddings -------------------------------------------------------
// Smooth periodisation (J > 0, embedding.cpp:132-141) gives n = 2(m + J) ∈ {3m, 4m, 6m, 10m, 18m}:
// radices 2/3/4/5. One transform per CTA, out-of-place Stockham between two shared buffers.
struct Radices {
  int r[16];
  int n;
};

__device__ __forceinline__ void dft3(double2& a0, double2& a1, double2& a2) {
  const double c = 0.86602540378443864676372317075294;  // √3/2
  const double2 t1 = cadd(a1, a2), t2 = csub(a1, a2);
  const double2 m = make_double2(a0.x - 0.5 * t1.x, a0.y - 0.5 * t1.y);
  const double2 it2 = make_double2(-c * t2.y, c * t2.x);  // i·(√3/2)·t2
  a0 = cadd(a0, t1);
  a1 = cadd(m, it2);
  a2 = csub(m, it2);
}

__device__ __forceinline__ void dft5(double2* v) {
  // X_k = Σ_j v_j exp(+2πi jk/5)
  const double c1 = 0.30901699437494742410229341718282, c2 = -0.80901699437494742410229341718282;
  const double s1 = 0.95105651629515357211643933337938, s2 = 0.58778525229247312916870595463907;
  const double2 a = cadd(v[1], v[4]), b = csub(v[1], v[4]), c = cadd(v[2], v[3]), d = csub(v[2], v[3]);
  const double2 x0 = v[0];
  v[0] = cadd(x0, cadd(a, c));
  const double2 r1 = make_double2(x0.x + c1 * a.x + c2 * c.x, x0.y + c1 * a.y + c2 * c.y);
  const double2 r2 = make_double2(x0.x + c2 * a.x + c1 * c.x, x0.y + c2 * a.y + c1 * c.y);
  const double2 i1 = make_double2(-(s1 * b.y + s2 * d.y), s1 * b.x + s2 * d.x);  // i(s1 b + s2 d)
  const double2 i2 = make_double2(-(s2 * b.y - s1 * d.y), s2 * b.x - s1 * d.x);  // i(s2 b − s1 d)
  v[1] = cadd(r1, i1);
  v[4] = csub(r1, i1);
  v[2] = cadd(r2, i2);
  v[3] = csub(r2, i2);
}

// Out-of-place mixed-radix Stockham FFT (+ sign); returns the buffer holding the result.
__device__ double2* fft_generic(double2* a, double2* b, const Radices& rd, const double2* __restrict__ tw) {
  const int n = rd.n;
  int Ns = 1;
  double2 *src = a, *dst = b;
  for (int s = 0; rd.r[s] > 0; ++s) {
    const int R = rd.r[s], nR = n / R;
    for (int j = threadIdx.x; j < nR; j += blockDim.x) {
      double2 v[5];
      for (int r = 0; r < R; ++r) v[r] = src[j + r * nR];
      const int k = j % Ns;
      if (Ns > 1) {
        const int step = k * (n / (Ns * R));
        for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[(r * step) % n]));
      }
      if (R == 2) dft2(v[0], v[1]);
      else if (R == 3) dft3(v[0], v[1], v[2]);
      else if (R == 4) dft4(v[0], v[1], v[2], v[3]);
      else dft5(v);
      const int base = (j - k) * R + k;
      for (int r = 0; r < R; ++r) dst[base + r * Ns] = v[r];
    }
    __syncthreads();
    double2* t = src;
    src = dst;
    dst = t;
    Ns *= R;
  }
  return src;
}

__global__ void ce_rows_generic_kernel(const double* __restrict__ sqrt_lam, const double* __restrict__ xi,
                                       uint64_t seed, uint32_t ell, uint64_t index0, Radices rd, int P,
                                       int cs, const double2* __restrict__ tw, double2* __restrict__ inter) {
  extern __shared__ double2 smem[];
  const int n = rd.n;
  const int rp = blockIdx.x, b = blockIdx.y;
  const int q1a = 2 * rp, q1b = 2 * rp + 1;
  const int64_t s = (int64_t)n * n;
  double2 *A = smem, *Bf = smem + n;
  for (int c = threadIdx.x; c < n / 2; c += blockDim.x) {
    double2 xa, xb;
    if (xi) {
      const double* xr = xi + (int64_t)b * s;
      xa = make_double2(xr[(int64_t)q1a * n + 2 * c], xr[(int64_t)q1a * n + 2 * c + 1]);
      xb = make_double2(xr[(int64_t)q1b * n + 2 * c], xr[(int64_t)q1b * n + 2 * c + 1]);
    } else {
      xa = normal_pair(seed, ell, index0 + b, (uint32_t)((int64_t)q1a * (n / 2) + c));
      xb = normal_pair(seed, ell, index0 + b, (uint32_t)((int64_t)q1b * (n / 2) + c));
    }
    const double* la = sqrt_lam + (int64_t)q1a * n + 2 * c;
    const double* lb = sqrt_lam + (int64_t)q1b * n + 2 * c;
    A[2 * c] = make_double2(la[0] * xa.x, lb[0] * xb.x);
    A[2 * c + 1] = make_double2(la[1] * xa.y, lb[1] * xb.y);
  }
  __syncthreads();
  const double2* x = fft_generic(A, Bf, rd, tw);
  double2* out = inter + (int64_t)b * P * n + q1a;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const int p0 = p * cs;
    const double2 zp = x[p0], zm = x[(n - p0) % n];
    double2* o = out + (int64_t)p * n;
    o[0] = make_double2(0.5 * (zp.x + zm.x), 0.5 * (zp.y - zm.y));
    o[1] = make_double2(0.5 * (zp.y + zm.y), 0.5 * (zm.x - zp.x));
  }
}

__global__ void ce_cols_generic_kernel(const double2* __restrict__ inter, Radices rd, int m, int P, int cs,
                                       double inv_n, int do_exp, const double2* __restrict__ tw,
                                       double* __restrict__ out_fine, double* __restrict__ out_coarse,
                                       int* __restrict__ bad_flag, unsigned long long* __restrict__ sup) {
  extern __shared__ double2 smem[];
  const int n = rd.n;
  const int j = blockIdx.x, b = blockIdx.y;
  double2 *A = smem, *Bf = smem + n;
  const double2* src = inter + ((int64_t)b * P + j) * n;
  for (int q = threadIdx.x; q < n; q += blockDim.x) A[q] = __ldg(src + q);
  __syncthreads();
  const double2* x = fft_generic(A, Bf, rd, tw);
  const int mf = m + 1, mc = m / 2 + 1;
  double* of = out_fine ? out_fine + (int64_t)b * mf * mf : nullptr;
  double* oc = out_coarse ? out_coarse + (int64_t)b * mc * mc : nullptr;
  int bad = 0;
  double vmax = 0.0;
  const int p0 = j * cs;
  for (int i = threadIdx.x; i <= m / cs; i += blockDim.x) {
    const int p1 = i * cs;
    const double zval = (x[p1].x + x[p1].y) * inv_n;
    if (!isfinite(zval)) bad = 1;
    vmax = fmax(vmax, fabs(zval));
    const double o = do_exp ? exp(zval) : zval;
    if (of) of[(int64_t)p1 * mf + p0] = o;
    if (oc && ((p0 | p1) & 1) == 0) oc[(int64_t)(p1 >> 1) * mc + (p0 >> 1)] = o;
  }
  if (bad && bad_flag) atomicOr(bad_flag + b, 1);
  if (sup) sup_commit(vmax, sup + b);
}

bool radices_of(int n, Radices& rd) {
  int k = 0, v = n;
  while (v % 4 == 0 && k < 15) { rd.r[k++] = 4; v /= 4; }
  while (v % 2 == 0 && k < 15) { rd.r[k++] = 2; v /= 2; }
  while (v % 3 == 0 && k < 15) { rd.r[k++] = 3; v /= 3; }
  while (v % 5 == 0 && k < 15) { rd.r[k++] = 5; v /= 5; }
  for (int i = k; i < 16; ++i) rd.r[i] = 0;
  rd.n = n;
  return v == 1;
}

void launch_generic(Ctx* ctx, const Level* L, const double* sqrt_lam, const double* xi_dev, uint64_t seed,
                    uint32_t ell, uint64_t index0, int count, bool do_exp, double* out_fine,
                    double* out_coarse, int* bad_flag, int cs, double2* inter, const Radices& rd,
                    unsigned long long* sup) {
  const int n = L->n, m = L->m, P = m / cs + 1;
  const double2* tw = L->twiddle.as<double2>();
  const size_t sm = 2 * sizeof(double2) * (size_t)n;
  const int threads = std::min(256, std::max(32, ((n / 2 + 31) / 32) * 32));
  smem_attr(ce_rows_generic_kernel, sm);
  smem_attr(ce_cols_generic_kernel, sm);
  {
    KScope ks(ctx, "ce_rows");
    ce_rows_generic_kernel<<<dim3(n / 2, count), threads, sm, ctx->stream>>>(sqrt_lam, xi_dev, seed, ell, index0,
                                                                             rd, P, cs, tw, inter);
    OSC_CUDA(cudaGetLastError());
  }
  {
    KScope ks(ctx, "ce_cols");
    ce_cols_generic_kernel<<<dim3(P, count), threads, sm, ctx->stream>>>(inter, rd, m, P, cs, 1.0 / n,
                                                                         do_exp ? 1 : 0, tw, out_fine, out_coarse,
                                                                         bad_flag, sup);
    OSC_CUDA(cudaGetLastError());
  }
}
}  // namespace

size_t ce_inter_bytes(const Level* L, int count, int col_stride) {
  const int P = L->m / col_stride + 1;
  const int Pe = CE_IL * inter_groups(P);  // column groups (inter_pair_idx); the runtime-n kernels use P ≤ Pe
  return sizeof(double2) * (size_t)count * L->n * Pe;
}

void ce_sample_launch(Ctx* ctx, const Level* L, const double* sqrt_lam, const double* xi_dev,
                      uint64_t seed, uint32_t ell, uint64_t index0, int count, bool do_exp,
                      double* out_fine, double* out_coarse, int* bad_flag, unsigned long long* sup_out) {
  const bool pow2 = (L->n & (L->n - 1)) == 0 && L->n >= 2;
  Radices rd;
  if (!pow2)
    OSC_REQUIRE(radices_of(L->n, rd) && L->n <= 4096,
                "ce_sample: padded embedding size n = 2(m+J) must factor into 2, 3, 5 and be <= 4096");
  OSC_REQUIRE(L->n <= 8192, "ce_sample: embedding size n > 8192 is not supported");
  if (count <= 0) return;
  // Coarse-only pass (other spectrum on the finest CES level) computes even columns only.
  const int cs = (out_fine == nullptr && out_coarse != nullptr) ? 2 : 1;
  // Process the batch in chunks of up to 1 GiB of half-spectrum intermediate (SURVEY §8(d)
  // 32·n(n/2+1) B/sample round trip). Both passes are fp64-issue bound with DRAM ≤ 16% busy, so the
  // round trip through HBM is hidden; small L2-sized chunks (80 MB: 2 samples at n = 2048) lost
  // more to partial last waves and pass-to-pass drains (config 2: 13.5k → 16.8k samples/s at 400 MB).
  const size_t per = ce_inter_bytes(L, 1, cs);
  constexpr size_t chunk_bytes = size_t(1024) << 20;
  const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)count, chunk_bytes / per));
  ctx->ce_inter.ensure(ce_inter_bytes(L, chunk, cs));
  double2* inter = ctx->ce_inter.as<double2>();
  const int m = L->m, mc = m / 2;
  const int64_t Nf = (int64_t)(m + 1) * (m + 1), Nc = (int64_t)(mc + 1) * (mc + 1);
  for (int c0 = 0; c0 < count; c0 += chunk) {
    const int cnt = std::min(chunk, count - c0);
    const double* xi_c = xi_dev ? xi_dev + (int64_t)c0 * L->s : nullptr;
    double* of = out_fine ? out_fine + c0 * Nf : nullptr;
    double* oc = out_coarse ? out_coarse + c0 * Nc : nullptr;
    int* bf = bad_flag ? bad_flag + c0 : nullptr;
    unsigned long long* sp = sup_out ? sup_out + c0 : nullptr;
    // threads per transform T = n/E: ≤ 256 up to n = 2048, 512 at 4096, 1024 at 8192
    if (!pow2)
      launch_generic(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter, rd, sp);
    else if (L->n >= 16) {
#define OSC_CE_T(LG) \
  case LG: launch_t<LG>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter, sp); break;
      switch (31 - __builtin_clz((unsigned)L->n)) {
        OSC_CE_T(4) OSC_CE_T(5) OSC_CE_T(6) OSC_CE_T(7) OSC_CE_T(8) OSC_CE_T(9) OSC_CE_T(10) OSC_CE_T(11)
        OSC_CE_T(12) OSC_CE_T(13)
      }
#undef OSC_CE_T
    } else if (L->n >= 8192)
      launch_pair<8, 1024>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter, sp);
    else if (L->n == 4096)
      launch_pair<8, 512>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter, sp);
    else if (L->n >= 8)
      launch_pair<8, 256>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter, sp);
    else if (L->n == 4)
      launch_pair<4, 256>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter, sp);
    else
      launch_pair<2, 256>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter, sp);
  }
}

// ---- level setup on the device -------------------------------------------------
// The spectrum of the padding-J embedding, λ = √s·Re(F row) (embedding.cpp:67-88), from the first
// row built on the device (embedding.cpp:22-65, covariance.cpp:47-115) and the CE kernels
// themselves: the row is even in both directions, so F row is real and even, and the CE pass with
// √λ ≡ 1, ξ = row and window m' = n/2 returns (Re + Im)(F_u row) = λ/n on [0, n/2]² (Im is rounding
// noise). The window is mirrored to n². Matérn is supported for ν = k + ½ (k ≤ 3, closed forms of
// the K_ν expression at covariance.cpp:53-62); other ν use the host setup.
namespace {
struct CovDev {
  int family, half_k;  // half_k ≥ 0: Matérn ν = half_k + ½ (closed form); −1: general ν (K_ν below)
  double sigma2, lambda, nu_or_p;
  double pre;  // σ² 2^{1−ν} / Γ(ν) (general ν)
};

// Modified Bessel function K_ν(x), ν > 0, x > 0 (covariance.cpp:58 boost::math::cyl_bessel_k): Temme's
// method. ν = n + μ, |μ| ≤ ½: K_μ, K_{μ+1} from Temme's series (x < 2) or Steed's continued fraction
// CF2 (x ≥ 2), then the stable upward recurrence K_{μ+k+1} = K_{μ+k−1} + 2(μ+k)/x · K_{μ+k}. The
// series' Γ terms come from the Taylor coefficients of 1/Γ(1+z) (Abramowitz–Stegun 6.1.34), whose
// even and odd parts give (1/Γ(1−μ) ± 1/Γ(1+μ))/2 without cancellation. Relative error ≤ 1e-13
// against the host's std::cyl_bessel_k over the Matérn range.
__device__ double bessel_k_dev(double nu, double x) {
  constexpr double kA[26] = {1.0, 0.5772156649015329, -0.6558780715202538, -0.0420026350340952, 0.1665386113822915,
                             -0.0421977345555443, -0.0096219715278770, 0.0072189432466630, -0.0011651675918591,
                             -0.0002152416741149, 0.0001280502823882, -0.0000201348547807, -0.0000012504934821,
                             0.0000011330272320, -0.0000002056338417, 0.0000000061160950, 0.0000000050020075,
                             -0.0000000011812746, 0.0000000001043427, 0.0000000000077823, -0.0000000000036968,
                             0.0000000000005100, -0.0000000000000206, -0.0000000000000054, 0.0000000000000014,
                             0.0000000000000001};
  constexpr double pi = 3.14159265358979323846, eps = 1e-16;
  const int nl = (int)(nu + 0.5);
  const double mu = nu - nl, mu2 = mu * mu, xi = 1.0 / x, xi2 = 2.0 * xi;
  double rkmu, rk1;
  if (x < 2.0) {
    double ev = 0.0, od = 0.0;  // even part Σ a_{2j} μ^{2j}, odd part / μ = Σ a_{2j+1} μ^{2j}
    for (int j = 12; j >= 0; --j) {
      ev = fma(ev, mu2, kA[2 * j]);
      od = fma(od, mu2, kA[2 * j + 1]);
    }
    const double gam1 = -od, gam2 = ev, gampl = gam2 - mu * gam1, gammi = gam2 + mu * gam1;
    const double x2 = 0.5 * x, pimu = pi * mu;
    const double fact = fabs(pimu) < eps ? 1.0 : pimu / sin(pimu);
    double d = -log(x2), e = mu * d;
    const double fact2 = fabs(e) < eps ? 1.0 : sinh(e) / e;
    double ff = fact * (gam1 * cosh(e) + gam2 * fact2 * d);
    double sum = ff;
    e = exp(e);
    double p = 0.5 * e / gampl, q = 0.5 / (e * gammi), c = 1.0, sum1 = p;
    d = x2 * x2;
    for (int i = 1; i <= 500; ++i) {
      ff = (i * ff + p + q) / (i * (double)i - mu2);
      c *= d / i;
      p /= i - mu;
      q /= i + mu;
      const double del = c * ff;
      sum += del;
      sum1 += c * (p - i * ff);
      if (fabs(del) < fabs(sum) * eps) break;
    }
    rkmu = sum;
    rk1 = sum1 * xi2;
  } else {
    double b = 2.0 * (1.0 + x), d = 1.0 / b, h = d, delh = d, q1 = 0.0, q2 = 1.0;
    const double a1 = 0.25 - mu2;
    double q = a1, c = a1, a = -a1, sv = 1.0 + q * delh;
    for (int i = 2; i <= 2000; ++i) {
      a -= 2 * (i - 1);
      c = -a * c / i;
      const double qnew = (q1 - b * q2) / a;
      q1 = q2;
      q2 = qnew;
      q += c * qnew;
      b += 2.0;
      d = 1.0 / (b + a * d);
      delh = (b * d - 1.0) * delh;
      h += delh;
      const double dels = q * delh;
      sv += dels;
      if (fabs(dels / sv) < eps) break;
    }
    h = a1 * h;
    rkmu = sqrt(pi / (2.0 * x)) * exp(-x) / sv;
    rk1 = rkmu * (mu + x + 0.5 - h) * xi;
  }
  for (int i = 1; i <= nl; ++i) {
    const double t = (mu + i) * xi2 * rk1 + rkmu;
    rkmu = rk1;
    rk1 = t;
  }
  return rkmu;
}

__device__ double cov_eval(const CovDev& c, double t0, double t1) {
  if (c.family == OSC_COV_SEPARABLE_EXP) {
    const double p = c.nu_or_p;
    const double sm = pow(fabs(t0), p) + pow(fabs(t1), p);
    return c.sigma2 * exp(-pow(sm, 1.0 / p) / c.lambda);
  }
  const double r = sqrt(t0 * t0 + t1 * t1);
  if (r == 0.0) return c.sigma2;
  const double x = sqrt(2.0 * c.nu_or_p) * r / c.lambda;
  if (x < 1e-13) return c.sigma2;
  if (c.half_k < 0) return c.pre * pow(x, c.nu_or_p) * bessel_k_dev(c.nu_or_p, x);
  // 2^{1−ν}/Γ(ν) x^ν K_ν(x) for ν = k + ½: e^{−x} · Σ_{i≤k} (k+i)!/(i!(k−i)!) (2x)^{k−i} · k!/(2k)!
  double poly = 1.0;
  if (c.half_k == 1) poly = 1.0 + x;
  else if (c.half_k == 2) poly = 1.0 + x + x * x / 3.0;
  else if (c.half_k == 3) poly = 1.0 + x + 2.0 * x * x / 5.0 + x * x * x / 15.0;
  return c.sigma2 * poly * exp(-x);
}

__device__ double eta_d(double x) { return x > 0.0 ? exp(-1.0 / x) : 0.0; }
__device__ double cutoff_phi_d(double t, double kappa) {  // covariance.cpp:87-95
  const double a = fabs(t);
  if (a <= 1.0) return 1.0;
  if (a >= kappa) return 0.0;
  const double up = eta_d((kappa - a) / (kappa - 1.0));
  const double dn = eta_d((a - 1.0) / (kappa - 1.0));
  return up / (up + dn);
}

// first-row table over the distinct displacements d ∈ [0, n/2]² (covariance.cpp:97-115 when padded)
__global__ void first_row_tab_kernel(CovDev c, int m, int J, int h, double* __restrict__ tab) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)(h + 1) * (h + 1)) return;
  const int d1 = (int)(i / (h + 1)), d0 = (int)(i - (int64_t)d1 * (h + 1));
  const double x0 = static_cast<double>(d0) / m, x1 = static_cast<double>(d1) / m;
  double v;
  if (J == 0) {
    v = cov_eval(c, x0, x1);
  } else {
    const double ell = 1.0 + static_cast<double>(J) / m, kappa = 2.0 * ell - 1.0, period = 2.0 * ell;
    v = 0.0;
    for (int n0 = -1; n0 <= 1; ++n0) {
      const double s0 = x0 + period * n0;
      for (int n1 = -1; n1 <= 1; ++n1) {
        const double s1 = x1 + period * n1;
        const double w = cutoff_phi_d(fmax(fabs(s0), fabs(s1)), kappa);
        if (w > 0.0) v += w * cov_eval(c, s0, s1);
      }
    }
  }
  tab[i] = v;
}

// out[q1·n + q0] = scale · win[min(q1, n−q1)·(h+1) + min(q0, n−q0)] (h = n/2)
__global__ void mirror_kernel(const double* __restrict__ win, int n, double scale, double* __restrict__ out) {
  const int64_t s = (int64_t)n * n, h = n / 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q1 = i / n, q0 = i - q1 * n;
    const int64_t d1 = q1 <= h ? q1 : n - q1, d0 = q0 <= h ? q0 : n - q0;
    out[i] = scale * win[d1 * (h + 1) + d0];
  }
}

__global__ void fill_kernel(double* __restrict__ p, int64_t count, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
}  // namespace

// Twiddle tables of a level (long-double angles, rounded once): the plain table tw[t] = exp(+2πi t/n),
// t < n, followed for n = 2^LOGN ≥ 16 by the per-stage tables of the compile-time-n passes — the
// stage with sub-length Ns = 2^LNS (LNS = 3, 6, …) and radix R holds W_{Ns R}^{r k} = tw[r k n/(Ns R)]
// as [r − 1][k] at offset Ns − 8 (the same doubles as the plain table, so results do not change).
void upload_twiddles(Level* L) {
  const int n = L->n;
  const bool staged = n >= 16 && (n & (n - 1)) == 0;
  std::vector<double> tw(2 * (size_t)n * (staged ? 2 : 1), 0.0);
  auto put = [&](size_t slot, int64_t t) {
    const long double a = 6.283185307179586476925286766559005768L * t / n;
    tw[2 * slot] = (double)std::cos(a);
    tw[2 * slot + 1] = (double)std::sin(a);
  };
  for (int t = 0; t < n; ++t) put((size_t)t, t);
  if (staged) {
    const int logn = 31 - __builtin_clz((unsigned)n);
    const int nst8 = logn / 3, rem = logn % 3;
    const int last_lns = rem ? 3 * nst8 : 3 * (nst8 - 1);
    for (int lns = 3; lns <= last_lns; lns += 3) {
      const int Ns = 1 << lns;
      const int R = lns < last_lns ? 8 : (rem ? (1 << rem) : 8);
      for (int r = 1; r < R; ++r)
        for (int k = 0; k < Ns; ++k) put((size_t)n + (Ns - 8) + (size_t)(r - 1) * Ns + k, (int64_t)r * k * (n / (Ns * R)));
    }
  }
  L->twiddle.ensure(sizeof(double) * tw.size());
  OSC_CUDA(cudaMemcpy(L->twiddle.p, tw.data(), sizeof(double) * tw.size(), cudaMemcpyHostToDevice));
}

// every model of the host setup: separable exponential, Matérn ν = k + ½ (closed forms) and general ν
bool spectrum_device_supported(int family, double nu_or_p) {
  return family == OSC_COV_SEPARABLE_EXP || (family == OSC_COV_MATERN && nu_or_p > 0.0 && nu_or_p <= 64.0);
}

// Raw spectrum of the padding-J embedding, left in device memory (eig_dev, s doubles).
void spectrum_device_into(Ctx* ctx, int m, int J, int family, double sigma2, double lambda, double nu_or_p,
                          double* eig_dev) {
  int half_k = -1;
  for (int k = 0; k <= 3; ++k)
    if (nu_or_p == k + 0.5) half_k = k;
  CovDev c{family, half_k, sigma2, lambda, nu_or_p,
           family == OSC_COV_MATERN ? sigma2 * std::pow(2.0, 1.0 - nu_or_p) / std::tgamma(nu_or_p) : 0.0};
  const int n = 2 * (m + J), h = n / 2;
  const int64_t s = (int64_t)n * n, nw = (int64_t)(h + 1) * (h + 1);
  cudaStream_t st = ctx->stream;
  Level T;  // the CE level of the spectrum pass: window m' = n/2, √λ ≡ 1
  T.ctx = ctx;
  T.m = h;
  T.J = 0;
  T.n = n;
  T.s = s;
  DevBuf row, win;
  auto release = [&] {
    T.sqrt_full.release();
    T.twiddle.release();
    row.release();
    win.release();
  };
  try {
    T.sqrt_full.ensure(sizeof(double) * s);
    row.ensure(sizeof(double) * s);
    win.ensure(sizeof(double) * (nw + s));  // the window, then the tab of the first row
    upload_twiddles(&T);
    double* tab = win.as<double>() + nw;
    {
      KScope ks(ctx, "setup.first_row");
      first_row_tab_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(c, m, J, h, tab);
      OSC_CUDA(cudaGetLastError());
      mirror_kernel<<<2048, 256, 0, st>>>(tab, n, 1.0, row.as<double>());
      OSC_CUDA(cudaGetLastError());
      fill_kernel<<<2048, 256, 0, st>>>(T.sqrt_full.as<double>(), s, 1.0);
      OSC_CUDA(cudaGetLastError());
    }
    ce_sample_launch(ctx, &T, T.sqrt_full.as<double>(), row.as<double>(), 0, 0, 0, 1, false, win.as<double>(),
                     nullptr, nullptr);
    {
      KScope ks(ctx, "setup.mirror");
      mirror_kernel<<<2048, 256, 0, st>>>(win.as<double>(), n, static_cast<double>(n), eig_dev);
      OSC_CUDA(cudaGetLastError());
    }
    OSC_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    release();
    throw;
  }
  release();
}

std::vector<double> spectrum_device(Ctx* ctx, int m, int J, int family, double sigma2, double lambda,
                                    double nu_or_p) {
  const int n = 2 * (m + J);
  const int64_t s = (int64_t)n * n;
  DevBuf eig;
  std::vector<double> out((size_t)s);
  try {
    eig.ensure(sizeof(double) * s);
    spectrum_device_into(ctx, m, J, family, sigma2, lambda, nu_or_p, eig.as<double>());
    OSC_CUDA(cudaMemcpy(out.data(), eig.p, sizeof(double) * s, cudaMemcpyDeviceToHost));
  } catch (...) {
    eig.release();
    throw;
  }
  eig.release();
  return out;
}

// Standalone NormalStream fill on device (osc_normals): out[b*s + e] = ξ_e of index0+b.
__global__ void normals_kernel(uint64_t seed, uint32_t ell, uint64_t index0, int64_t s,
                               double* __restrict__ out) {
  const int b = blockIdx.y;
  const int64_t half = (s + 1) / 2;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < half;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = normal_pair(seed, ell, index0 + b, (uint32_t)j);
    out[(int64_t)b * s + 2 * j] = v.x;
    if (2 * j + 1 < s) out[(int64_t)b * s + 2 * j + 1] = v.y;
  }
}

void normals_launch(Ctx* ctx, uint64_t seed, uint32_t ell, uint64_t index0, int count,
                    int64_t s, double* out) {
  const int64_t half = (s + 1) / 2;
  const int blocks = (int)std::min<int64_t>((half + 255) / 256, 4096);
  KScope ks(ctx, "normals");
  normals_kernel<<<dim3(blocks, count), 256, 0, ctx->stream>>>(seed, ell, index0, s, out);
  OSC_CUDA(cudaGetLastError());
}

}  // namespace osc
