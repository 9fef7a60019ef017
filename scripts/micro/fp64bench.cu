// FP64 vector throughput on this B200: DFMA (and DADD) issue rate with 8 independent chains per
// thread, 148 x 8 CTAs of 256 threads. The CE kernels are fp64-issue bound, so
// this is the denominator of their compute roofline. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <bool ADD>
__global__ void __launch_bounds__(256) fp64_chains(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = ADD ? x[i] + a : fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 0.123456) out[0] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best[2] = {0, 0};
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) fp64_chains<false><<<blocks, threads>>>(out, iters, 0.9999999, 1e-9);
      else fp64_chains<true><<<blocks, threads>>>(out, iters, 1e-9, 0.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters * 16 * 8;  // FMA or ADD instructions (lanes)
      const double rate = ops / (ms * 1e-3);                           // lane-ops/s
      if (rep > 0 && rate > best[mode]) best[mode] = rate;
    }
  }
  printf("{\"sms\": %d, \"dfma_lane_ops_per_s\": %.4e, \"fp64_fma_tflops\": %.2f, \"dadd_lane_ops_per_s\": %.4e, "
         "\"dfma_warp_inst_per_clk_per_sm_at_1965\": %.3f}\n",
         sms, best[0], 2 * best[0] / 1e12, best[1], best[0] / 32 / sms / 1.965e9);
  return 0;
}
