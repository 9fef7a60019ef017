// Access-pattern micro-benchmark: row-marching warps (the solver's layout: lane = column pair,
// warp = 64-column strip, CTA = MW strips, LY rows per warp, one row of loads in flight) vs the
// grid-stride stream, for a 3-read/1-write mix over 64 samples of 2049^2 doubles.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int n0 = 2049;
constexpr int B = 64;
template <int MW, int LY, bool PAIR>
__global__ void __launch_bounds__(32 * MW) march(const double* a, const double* b, const double* c, double* o) {
  const int lane = threadIdx.x & 31, strip = blockIdx.x * MW + (threadIdx.x >> 5);
  const int cols = PAIR ? 64 : 32;
  const int x = strip * cols + (PAIR ? 2 * lane : lane);
  const int y0 = blockIdx.y * LY, y1 = min(y0 + LY, n0);
  const size_t off = (size_t)blockIdx.z * n0 * n0;
  auto ld = [&](const double* p, int y, int xx) { return (xx < n0 && y < n0) ? __ldg(p + off + (size_t)y * n0 + xx) : 0.0; };
  double qa = ld(a, y0, x), qb = ld(b, y0, x), qc = ld(c, y0, x);
  double qa2 = PAIR ? ld(a, y0, x + 1) : 0, qb2 = PAIR ? ld(b, y0, x + 1) : 0, qc2 = PAIR ? ld(c, y0, x + 1) : 0;
  for (int y = y0; y < y1; ++y) {
    const double va = qa, vb = qb, vc = qc, va2 = qa2, vb2 = qb2, vc2 = qc2;
    qa = ld(a, y + 1, x); qb = ld(b, y + 1, x); qc = ld(c, y + 1, x);
    if (PAIR) { qa2 = ld(a, y + 1, x + 1); qb2 = ld(b, y + 1, x + 1); qc2 = ld(c, y + 1, x + 1); }
    const double s = va + vb * vc + __shfl_down_sync(0xffffffffu, va, 1);
    if (x < n0) o[off + (size_t)y * n0 + x] = s;
    if (PAIR && x + 1 < n0) o[off + (size_t)y * n0 + x + 1] = va2 + vb2 * vc2;
  }
}
__global__ void stream3(const double* a, const double* b, const double* c, double* o, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    o[i] = a[i] + b[i] * c[i];
}
int main() {
  const size_t N = (size_t)B * n0 * n0;
  double *A, *Bv, *Cv, *O;
  cudaMalloc(&A, N * 8); cudaMalloc(&Bv, N * 8); cudaMalloc(&Cv, N * 8); cudaMalloc(&O, N * 8);
  cudaMemset(A, 0, N * 8); cudaMemset(Bv, 0, N * 8); cudaMemset(Cv, 0, N * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    launch(); cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-28s %7.1f GB/s (%.3f ms) %s\n", name, 4.0 * N * 8 / best / 1e6, best, cudaGetErrorString(cudaGetLastError()));
  };
  run("stream", [&] { stream3<<<148 * 16, 256>>>(A, Bv, Cv, O, N); });
#define M(MW, LY, PAIR) run("march MW=" #MW " LY=" #LY " pair=" #PAIR, [&] { \
    const int cols = PAIR ? 64 : 32; const int strips = (n0 + cols - 1) / cols; \
    march<MW, LY, PAIR><<<dim3((strips + MW - 1) / MW, (n0 + LY - 1) / LY, B), 32 * MW>>>(A, Bv, Cv, O); });
  M(4, 32, true) M(4, 64, true) M(8, 32, true) M(16, 32, true) M(4, 16, true)
  M(4, 32, false) M(8, 32, false) M(16, 32, false) M(32, 32, false) M(8, 64, false)
}
