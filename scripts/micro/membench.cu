// HBM micro-benchmark: achievable bandwidth for the read/write mixes of the solver kernels
// (copy 1R1W, apply-like 3R1W, update-like 4R3W, restrict-like 2R), double2 grid-stride.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_1r1w(const double2* a, double2* o, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) o[i] = a[i];
}
__global__ void k_3r1w(const double2* a, const double2* b, const double2* c, double2* o, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i], z = c[i];
    o[i] = make_double2(x.x + y.x * z.x, x.y + y.y * z.y);
  }
}
__global__ void k_4r3w(const double2* a, const double2* b, const double2* c, const double2* d, double2* o1, double2* o2, double2* o3, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i], z = c[i], w = d[i];
    o1[i] = make_double2(x.x + y.x, x.y + y.y);
    o2[i] = make_double2(z.x * w.x, z.y * w.y);
    o3[i] = make_double2(x.x - w.x, x.y - w.y);
  }
}
__global__ void k_2r(const double2* a, const double2* b, double* o, size_t n) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i];
    acc += x.x * y.x + x.y * y.y;
  }
  if (acc == 123.456) o[0] = acc;
}
int main() {
  const size_t N = (size_t)64 * 2049 * 2049;  // doubles per array (cfg4 level 0, B = 64)
  const size_t n2 = N / 2;
  double2* A[7];
  for (int i = 0; i < 7; ++i) { cudaMalloc(&A[i], N * 8); cudaMemset(A[i], 0, N * 8); }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int grid_mul : {4, 8, 16}) {
    const int grid = sms * grid_mul, blk = 256;
    auto run = [&](const char* name, int nr, int nw, auto launch) {
      launch(); cudaDeviceSynchronize();
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("grid %4d  %-6s %7.1f GB/s  (%.3f ms)\n", grid, name, (nr + nw) * N * 8.0 / best / 1e6, best);
    };
    run("1r1w", 1, 1, [&] { k_1r1w<<<grid, blk>>>(A[0], A[1], n2); });
    run("3r1w", 3, 1, [&] { k_3r1w<<<grid, blk>>>(A[0], A[1], A[2], A[3], n2); });
    run("4r3w", 4, 3, [&] { k_4r3w<<<grid, blk>>>(A[0], A[1], A[2], A[3], A[4], A[5], A[6], n2); });
    run("2r", 2, 0, [&] { k_2r<<<grid, blk>>>(A[0], A[1], (double*)A[6], n2); });
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
