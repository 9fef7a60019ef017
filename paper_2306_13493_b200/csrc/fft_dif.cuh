// Length-n (n = 2^LOGN, 16 ≤ n ≤ 8192) complex FFT with the + sign (fft.hpp:11), T = n/8 threads and 8
// values per thread, as a radix-8 decimation-in-frequency recursion whose exchanges stay inside the
// thread group that owns a sub-transform:
//
//   stage s works on sub-transforms of size M = n/8^s, each held by a group of G = M/8 consecutive
//   threads; thread g of the group holds y[g + (M/8)·r], r < 8. One radix-8 butterfly over r gives
//   the eight size-M/8 sub-transforms k < 8 (input u_k[g] = (Σ_r y[g + (M/8) r] W_8^{kr}) · W_M^{kg}),
//   whose outputs p' land at p = k + 8 p'. The group writes u_k[g] to its own region of the
//   transform's shared buffer (slot k·M/8 + g), synchronises AS A GROUP, and splits into eight
//   subgroups of G/8 threads, one per k.
//
// So only the first exchange spans the whole transform (one CTA-wide or named barrier); from
// G ≤ 32 on the exchanges are warp-local (__syncwarp), and warps drift apart: shared-memory
// traffic, fp64 butterflies and global loads of different warps overlap instead of meeting at
// every stage (the Stockham kernels this replaces ran 6 CTA-wide barriers per 2048-point
// transform at 24–52% issue utilisation). When the remaining size is 2 or 4 the group's threads
// each take 8/M' whole sub-transforms (last radix M'); a remaining size of 1 ends the recursion.
// Output p of the transform = Σ_s k_s 8^s (+ the last radix' index), known statically per register.
//
// NC transforms (columns) per thread share the roles, addresses and twiddles.
#pragma once

#include "osc_device.cuh"

namespace osc {

template <int G, int THREADS>
__device__ __forceinline__ void dif_gsync() {
  if constexpr (G <= 32) {
    __syncwarp();
  } else if constexpr (G == THREADS) {
    __syncthreads();
  } else {  // named barrier per group (ids 1 … THREADS/G ≤ 8)
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)threadIdx.x / G), "n"(G) : "memory");
  }
}

// Sink interface: `out(c, p, v)` receives output p of transform c of this thread.
template <int LOGN, int M, int NC, int THREADS, class Sink>
__device__ __forceinline__ void dif_stage(double2 (&v)[NC][8], double2* (&x)[NC], int rb, int g, int pbase,
                                          const double2* __restrict__ tw, Sink& sink) {
  constexpr int n = 1 << LOGN, Mp = M / 8, pstr = n / M;
  if constexpr (Mp == 1) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      dft8(v[c]);
#pragma unroll
      for (int k = 0; k < 8; ++k) sink(c, pbase + k * pstr, v[c][k]);
    }
  } else {
    double2 w[7];  // W_M^{g k}, shared by the NC transforms
#pragma unroll
    for (int k = 1; k < 8; ++k) w[k - 1] = __ldg(&tw[(g * k) * pstr]);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      dft8(v[c]);
#pragma unroll
      for (int k = 1; k < 8; ++k) v[c][k] = cmul(v[c][k], w[k - 1]);
    }
    // the group's previous reads of its region are done before anyone overwrites it
    if constexpr (M < n) dif_gsync<M / 8, THREADS>();
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[c][fpad(rb + k * Mp + g)] = v[c][k];
    dif_gsync<M / 8, THREADS>();
    if constexpr (Mp >= 8) {
      constexpr int Gn = Mp / 8;
      const int ks = g / Gn, gp = g % Gn;
      const int rbn = rb + ks * Mp;
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int r = 0; r < 8; ++r) v[c][r] = x[c][fpad(rbn + gp + Gn * r)];
      dif_stage<LOGN, Mp, NC, THREADS>(v, x, rbn, gp, pbase + ks * pstr, tw, sink);
    } else {
      // last radix Mp ∈ {2, 4}: the group's Mp threads take 8/Mp whole sub-transforms each (k = g + Mp j)
      constexpr int PER = 8 / Mp;
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          double2 u[Mp];
          const int k = g + Mp * j;
#pragma unroll
          for (int q = 0; q < Mp; ++q) u[q] = x[c][fpad(rb + k * Mp + q)];
          dft_r<Mp>(u);
#pragma unroll
          for (int q = 0; q < Mp; ++q) sink(c, pbase + k * pstr + 8 * pstr * q, u[q]);
        }
    }
  }
}

// Whole transform(s): v[c][r] = input (lt + r·T) of transform c; x[c] = that transform's shared buffer
// (fpad_len(n) slots). lt = thread index within the transform's T threads.
template <int LOGN, int NC, int THREADS, class Sink>
__device__ __forceinline__ void fft_dif(double2 (&v)[NC][8], double2* (&x)[NC], int lt,
                                        const double2* __restrict__ tw, Sink& sink) {
  dif_stage<LOGN, (1 << LOGN), NC, THREADS>(v, x, 0, lt, 0, tw, sink);
}

// Padding of the natural-order buffer the row pass unpacks from: the final outputs of a warp's store
// instruction are p = k₀ + 8k₁ + 64k₂ + … with the digits spread over lanes; these paddings make
// those stores (and the unpack's consecutive reads) bank-conflict-free (searched per size).
template <int LOGN>
__device__ __host__ __forceinline__ constexpr int npad(int a) {
  if constexpr (LOGN == 13) return a + (a >> 3) + (a >> 6) + 2 * (a >> 8);
  else if constexpr (LOGN == 12) return a + (a >> 3) + (a >> 6);
  else if constexpr (LOGN == 11) return a + (a >> 3) + (a >> 5);
  else if constexpr (LOGN == 10) return a + (a >> 3) + 2 * (a >> 5);
  else return a + (a >> 3);
}

}  // namespace osc
