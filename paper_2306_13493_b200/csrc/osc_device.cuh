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
__device__ __forceinline__ double2 box_muller(uint4 r) {
  const double u1 = ((double)((((uint64_t)r.x << 32) | r.y) >> 11) + 0.5) * 0x1p-53;
  const double u2 = ((double)((((uint64_t)r.z << 32) | r.w) >> 11) + 0.5) * 0x1p-53;
  const double mag = sqrt(-2.0 * log(u1));
  // cos/sin(2π u2) via sincospi(2 u2): the same angle without sincos's Payne–Hanek slow path
  // (differs from glibc's sin(2π·u2) by ≲ 2 ulp; fields stay within 1e-10 of the reference)
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  return make_double2(mag * c, mag * s);
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
