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

#include "osc_device.cuh"
#include "osc_internal.cuh"

namespace osc {

namespace {

// elements per thread for a length-n transform
inline int elems_for(int n) { return n >= 8 ? 8 : n; }

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
    double* __restrict__ out_coarse, int* __restrict__ bad_flag) {
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
  const int lnt = 31 - __clz(NT);  // NT is a power of two
  for (int idx = threadIdx.x; idx < NT * n_rows; idx += blockDim.x) {
    const int tt = idx & (NT - 1), i = idx >> lnt;
    const int j = j0 + tt;
    if (j >= P) continue;
    const int p1 = i * cs, p0 = j * cs;
    const double2 v = smem[tt * ld + fpad(p1)];
    const double zval = (v.x + v.y) * inv_n;
    if (!isfinite(zval)) bad = 1;
    const double o = do_exp ? exp(zval) : zval;
    if (of) of[(int64_t)p1 * mf + p0] = o;
    if (oc && ((p0 | p1) & 1) == 0) oc[(int64_t)(p1 >> 1) * mc + (p0 >> 1)] = o;
  }
  if (bad && bad_flag) atomicOr(bad_flag + b, 1);
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
                 double* out_fine, double* out_coarse, int* bad_flag, int cs, double2* inter) {
  const int n = L->n, m = L->m;
  const int P = m / cs + 1;
  const double2* tw = L->twiddle.as<double2>();
  cudaStream_t st = ctx->stream;
  {
    const CeGeom g = rows_geom(n);
    const dim3 grid((n / 2 + g.NT - 1) / g.NT, count);
    auto kern = ce_rows_kernel<E, MAXT>;
    OSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
    KScope ks(ctx, "ce_rows");
    kern<<<grid, g.threads, g.smem, st>>>(sqrt_lam, xi_dev, seed, ell, index0, n, g.NT, P, cs, tw, inter);
    OSC_CUDA(cudaGetLastError());
  }
  {
    const CeGeom g = cols_geom(n, P);
    const dim3 grid((P + g.NT - 1) / g.NT, count);
    auto kern = ce_cols_kernel<E, MAXT>;
    OSC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
    KScope ks(ctx, "ce_cols");
    kern<<<grid, g.threads, g.smem, st>>>(inter, n, m, g.NT, P, cs, 1.0 / n, do_exp ? 1 : 0, tw,
                                         out_fine, out_coarse, bad_flag);
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
                                       int* __restrict__ bad_flag) {
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
  const int p0 = j * cs;
  for (int i = threadIdx.x; i <= m / cs; i += blockDim.x) {
    const int p1 = i * cs;
    const double zval = (x[p1].x + x[p1].y) * inv_n;
    if (!isfinite(zval)) bad = 1;
    const double o = do_exp ? exp(zval) : zval;
    if (of) of[(int64_t)p1 * mf + p0] = o;
    if (oc && ((p0 | p1) & 1) == 0) oc[(int64_t)(p1 >> 1) * mc + (p0 >> 1)] = o;
  }
  if (bad && bad_flag) atomicOr(bad_flag + b, 1);
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
                    double* out_coarse, int* bad_flag, int cs, double2* inter, const Radices& rd) {
  const int n = L->n, m = L->m, P = m / cs + 1;
  const double2* tw = L->twiddle.as<double2>();
  const size_t sm = 2 * sizeof(double2) * (size_t)n;
  const int threads = std::min(256, std::max(32, ((n / 2 + 31) / 32) * 32));
  OSC_CUDA(cudaFuncSetAttribute(ce_rows_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  OSC_CUDA(cudaFuncSetAttribute(ce_cols_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
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
                                                                         bad_flag);
    OSC_CUDA(cudaGetLastError());
  }
}
}  // namespace

size_t ce_inter_bytes(const Level* L, int count, int col_stride) {
  const int P = L->m / col_stride + 1;
  return sizeof(double2) * (size_t)count * L->n * P;
}

void ce_sample_launch(Ctx* ctx, const Level* L, const double* sqrt_lam, const double* xi_dev,
                      uint64_t seed, uint32_t ell, uint64_t index0, int count, bool do_exp,
                      double* out_fine, double* out_coarse, int* bad_flag) {
  const bool pow2 = (L->n & (L->n - 1)) == 0 && L->n >= 2;
  Radices rd;
  if (!pow2)
    OSC_REQUIRE(radices_of(L->n, rd) && L->n <= 4096,
                "ce_sample: padded embedding size n = 2(m+J) must factor into 2, 3, 5 and be <= 4096");
  OSC_REQUIRE(L->n <= 8192, "ce_sample: embedding size n > 8192 is not supported");
  if (count <= 0) return;
  // Coarse-only pass (other spectrum on the finest CES level) computes even columns only.
  const int cs = (out_fine == nullptr && out_coarse != nullptr) ? 2 : 1;
  // Process the batch in chunks whose half-spectrum intermediate stays L2-resident between the
  // row and the column pass (≈ 48 MB of the 126 MB L2), so the intermediate round trip
  // (SURVEY §8(d) 32·n(n/2+1) B/sample) is served by L2 instead of HBM.
  const size_t per = ce_inter_bytes(L, 1, cs);
  const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)count, (80u << 20) / per));
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
    // threads per transform T = n/E: ≤ 256 up to n = 2048, 512 at 4096, 1024 at 8192
    if (!pow2)
      launch_generic(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter, rd);
    else if (L->n >= 8192)
      launch_pair<8, 1024>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter);
    else if (L->n == 4096)
      launch_pair<8, 512>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter);
    else if (L->n >= 8)
      launch_pair<8, 256>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter);
    else if (L->n == 4)
      launch_pair<4, 256>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter);
    else
      launch_pair<2, 256>(ctx, L, sqrt_lam, xi_c, seed, ell, index0 + c0, cnt, do_exp, of, oc, bf, cs, inter);
  }
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
