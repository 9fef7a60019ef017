// Device helpers: Philox4x32-10 + Box–Muller (bit-compatible with the reference's
// NormalStream, src/rng.cpp:10-67), small-radix DFTs, Stockham FFT stages in shared
// memory, block reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace osc {

// Philox4x32-10 (src/rng.cpp:29-40): M0 = 0xD2511F53, M1 = 0xCD9E8D57, Weyl key bumps.
__device__ __forceinline__ uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Same rounds with a precomputed key schedule (the keys depend only on the seed, so a thread
// that draws many blocks forms them once).
struct PhiloxKeys {
  uint32_t k0[10], k1[10];
};
__device__ __forceinline__ PhiloxKeys philox_keys(uint64_t seed) {
  PhiloxKeys ks;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    ks.k0[r] = k0;
    ks.k1[r] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return ks;
}
__device__ __forceinline__ uint4 philox10k(uint4 c, const PhiloxKeys& ks) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ ks.k0[r], lo1, hi0 ^ c.w ^ ks.k1[r], lo0);
  }
  return c;
}

// Normals 2j, 2j+1 of NormalStream(seed, ell, idx) (src/rng.cpp:42-63): counter
// (j, ell, idx lo, idx hi), key = seed words, 53-bit uniforms, cos first then sin.
__device__ __forceinline__ double2 box_muller(uint4 r);
__device__ __forceinline__ double2 normal_pair(uint64_t seed, uint32_t ell, uint64_t idx,
                                               uint32_t j) {
  return box_muller(philox10(make_uint4(j, ell, (uint32_t)idx, (uint32_t)(idx >> 32)),
                             (uint32_t)seed, (uint32_t)(seed >> 32)));
}
__device__ __forceinline__ double2 normal_pair_k(const PhiloxKeys& ks, uint32_t ell, uint64_t idx,
                                                 uint32_t j) {
  return box_muller(philox10k(make_uint4(j, ell, (uint32_t)idx, (uint32_t)(idx >> 32)), ks));
}
// Box–Muller on the device. The math library's log / sincospi cost ~100 instructions per pair and
// materialise every 64-bit polynomial coefficient with two UMOVs at each use (14% of the CE row
// pass's instruction stream, profiles/r2_ce_rows_opcodes.txt); here the coefficients sit in the
// constant bank, which DFMA reads as a c[][] operand, and the arguments' known ranges drop the
// special-case paths:
//   log(u1), u1 ∈ [2^-54, 1): the classical reduction u1 = 2^k (1 + f), 1 + f ∈ [√½, √2),
//     s = f/(2 + f), log(1+f) = f − ½f² + s(½f² + R(s²)) with R the degree-7 minimax polynomial of
//     the published fdlibm/musl log (≤ 1 ulp);
//   cos/sin(2π u2), u2 ∈ (0, 1): t = 4u2, q = rint(t), r = t − q ∈ [−½, ½] (both exact), then the
//     Taylor series of sin/cos(πr/2) to r^17 / r^18 (truncation < 1e-19) and the quadrant q mod 4.
// The angle is exact (as sincospi), not the rounded 2π·u2 of the reference's std::cos: the normals
// differ from glibc's by a few ulp (≤ 1e-14 relative), fields stay within 1e-10.
static __constant__ double k_bm[] = {
    // log: Lg1..Lg7, ln2_hi, ln2_lo
    6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01, 2.222219843214978396e-01,
    1.818357216161805012e-01, 1.531383769920937332e-01, 1.479819860511658591e-01, 6.93147180369123816490e-01,
    1.90821492927058770002e-10,
    // sin(πr/2) / r: (−1)^k (π/2)^(2k+1) / (2k+1)!, k = 0..8
    1.57079632679489656e+00, -6.45964097506246282e-01, 7.96926262461670476e-02, -4.68175413531868832e-03,
    1.60441184787359829e-04, -3.59884323521208518e-06, 5.69217292196792668e-08, -6.68803510981146768e-10,
    6.06693573110619553e-12,
    // cos(πr/2): (−1)^k (π/2)^(2k) / (2k)!, k = 0..9
    1.0, -1.23370055013616975e+00, 2.53669507901048030e-01, -2.08634807633529609e-02, 9.19260274839426585e-04,
    -2.52020423730606066e-05, 4.71087477881817174e-07, -6.38660308379185209e-09, 6.56596311497947280e-11,
    -5.29440020073462348e-13};

__device__ __forceinline__ double bm_rcp(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = fma(y, fma(-d, y, 1.0), y);
  return fma(y, fma(-d, y, 1.0), y);
}

// log(x) for x ∈ [2^-54, 1) (normal, positive)
__device__ __forceinline__ double bm_log(double x) {
  const int hi = __double2hiint(x), lo = __double2loint(x);
  const int mh = hi & 0x000fffff;
  const bool big = mh >= 0x6a09e;  // mantissa ≥ √2: use (1 + f)/2 and k + 1
  const int k = (hi >> 20) - 1023 + (big ? 1 : 0);
  const double f = __hiloint2double((mh | 0x3ff00000) - (big ? 0x00100000 : 0), lo) - 1.0;
  const double hfsq = 0.5 * f * f;
  const double s = f * bm_rcp(2.0 + f);
  const double z = s * s, w = z * z;
  const double t1 = w * (k_bm[1] + w * (k_bm[3] + w * k_bm[5]));
  const double t2 = z * (k_bm[0] + w * (k_bm[2] + w * (k_bm[4] + w * k_bm[6])));
  const double dk = (double)k;
  return dk * k_bm[7] - ((hfsq - (s * (hfsq + (t2 + t1)) + dk * k_bm[8])) - f);
}

// (cos 2πu, sin 2πu) for u ∈ (0, 1)
__device__ __forceinline__ double2 bm_cossin_2pi(double u) {
  const double t = 4.0 * u;
  const double q = rint(t);
  const double r = t - q;
  const double z = r * r;
  double ps = k_bm[17];
#pragma unroll
  for (int i = 16; i >= 9; --i) ps = fma(ps, z, k_bm[i]);
  ps *= r;
  double pc = k_bm[27];
#pragma unroll
  for (int i = 26; i >= 18; --i) pc = fma(pc, z, k_bm[i]);
  const int qi = (int)q & 3;
  const double cm = (qi & 1) ? ps : pc, sm = (qi & 1) ? pc : ps;
  return make_double2((qi == 1 || qi == 2) ? -cm : cm, qi >= 2 ? -sm : sm);
}

__device__ __forceinline__ double2 box_muller(uint4 r) {
  const double u1 = ((double)((((uint64_t)r.x << 32) | r.y) >> 11) + 0.5) * 0x1p-53;
  const double u2 = ((double)((((uint64_t)r.z << 32) | r.w) >> 11) + 0.5) * 0x1p-53;
  const double mag = sqrt(-2.0 * bm_log(u1));
  const double2 cs = bm_cossin_2pi(u2);
  return make_double2(mag * cs.x, mag * cs.y);
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// multiply by +i
__device__ __forceinline__ double2 cmul_i(double2 a) { return make_double2(-a.y, a.x); }

// In-register DFTs with the + sign (exp(+2πi jk/R)), unnormalised.
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  const double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
  const double2 s13 = cadd(a1, a3), d13 = cmul_i(csub(a1, a3));
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, d13);
  a3 = csub(d02, d13);
}
__device__ __forceinline__ void dft8(double2* v) {
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4(e0, e1, e2, e3);
  dft4(o0, o1, o2, o3);
  const double c = 0.70710678118654752440084436210485;
  o1 = make_double2(c * (o1.x - o1.y), c * (o1.x + o1.y));   // × exp(+iπ/4)
  o2 = cmul_i(o2);                                           // × i
  o3 = make_double2(-c * (o3.x + o3.y), c * (o3.x - o3.y));  // × exp(+3iπ/4)
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
}

template <int R>
__device__ __forceinline__ void dft_r(double2* v) {
  if constexpr (R == 2) dft2(v[0], v[1]);
  else if constexpr (R == 4) dft4(v[0], v[1], v[2], v[3]);
  else dft8(v);
}

// Shared-memory FFT index padding: one spare slot per 8 complex values, so the stride-8 writes of
// the first radix-8 stage (and the strided reads of later stages) spread across banks.
__device__ __forceinline__ int fpad(int i) { return i + (i >> 3); }
__host__ __device__ __forceinline__ int fpad_len(int n) { return n + (n >> 3) + 1; }

// One in-place Stockham stage (radix R, current sub-length Ns) of a length-n transform held
// in shared memory x[0..n), executed by T = n/E threads (lt = local thread id) that each own
// E/R butterflies. tw[t] = exp(+2πi t/n). Caller syncs before and after.
template <int E, int R>
__device__ __forceinline__ void stockham_stage(double2* x, int n, int Ns, int lt,
                                               const double2* __restrict__ tw, int tw_shift) {
  constexpr int G = E / R;
  const int T = n / E;
  const int nR = n / R;
  double2 v[G][R];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j = lt + g * T;
#pragma unroll
    for (int r = 0; r < R; ++r) v[g][r] = x[fpad(j + r * nR)];
    if (Ns > 1) {
      const int k = j & (Ns - 1);
      const int step = k << tw_shift;  // k · n/(Ns·R), all powers of two
#pragma unroll
      for (int r = 1; r < R; ++r) v[g][r] = cmul(v[g][r], __ldg(&tw[r * step]));
    }
    dft_r<R>(v[g]);
  }
  __syncthreads();
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j = lt + g * T;
    const int k = j & (Ns - 1);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) x[fpad(base + r * Ns)] = v[g][r];
  }
}

// Full length-n (power of two, n ≥ E) in-place FFT with + sign: radix-E stages then a
// final stage with the remaining radix. Syncs internally; caller syncs before the call
// (data staged) and after (data consumed).
template <int E>
__device__ __forceinline__ void fft_smem(double2* x, int n, int lt, const double2* __restrict__ tw) {
  constexpr int LE = E == 8 ? 3 : (E == 4 ? 2 : 1);
  const int ln = 31 - __clz(n);  // n is a power of two
  int Ns = 1, lns = 0;
  while (lns + LE <= ln) {
    stockham_stage<E, E>(x, n, Ns, lt, tw, ln - lns - LE);
    __syncthreads();
    Ns <<= LE;
    lns += LE;
  }
  const int rem = ln - lns;  // log2 of the remaining radix
  if constexpr (E >= 4) {
    if (rem == 2) { stockham_stage<E, 4>(x, n, Ns, lt, tw, ln - lns - 2); __syncthreads(); return; }
  }
  if constexpr (E >= 2) {
    if (rem == 1) { stockham_stage<E, 2>(x, n, Ns, lt, tw, ln - lns - 1); __syncthreads(); }
  }
}

// Warp / block sum of doubles (blockDim multiple of 32, ≤ 1024). Result valid in thread 0.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double block_sum(double v, double* sh /* ≥ 32 */) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x * blockDim.y + 31) >> 5;
  v = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
  if (wid == 0) v = warp_sum(v);
  return v;
}

}  // namespace osc
