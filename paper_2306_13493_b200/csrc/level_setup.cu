// Level setup that never leaves the device and the OSC1 dump:
//   osc_level_create_device  build_operator + from_parts + truncated (embedding.cpp:90-163): the
//                            spectrum (ce_sample.cu spectrum_device_into), its minimum (the SPD test),
//                            the clamp, √max(λ, 0), the stable descending order and the truncation mask
//                            are all computed in HBM; only the minimum (8 bytes) reaches the host.
//   osc_level_retruncate     EmbeddingOperator::truncated(k) from the resident order.
//   osc_level_eigenvalues    the clamped eigenvalues (for OSC1 dumps / the estimator's k_ℓ rule).
//   osc_smoothing_error      smoothing_error_estimate (embedding.cpp:205-228) as ONE CE pass per sample:
//                            Z − Z̃ is linear in ξ, so it is the CE field of the dropped modes
//                            √λ − √λ̃; the column pass reduces sup|·| in its epilogue (no field is stored).
//   osc_spectrum_save/load   the OSC1 format (embedding.cpp:262-294).
// The order comes from cub::DeviceRadixSort (stable; setup only, not the sample path).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "osc_internal.cuh"

namespace osc {
struct SetupError {
  int code;
  std::string msg;
};
int padding_schedule(int m, int family, double sigma2, double lambda, double nu_or_p, const double* fractions,
                     int n_fractions, double tol_factor, const std::function<double(int)>& attempt_min);
int c_api_error(const std::exception_ptr& ep);

namespace {
constexpr int ST = 256;

// doubles ordered as unsigned keys (negative values flip entirely, the rest set the sign bit)
__device__ __forceinline__ unsigned long long ordered_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
double key_to_double(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double v;
  std::memcpy(&v, &b, sizeof v);
  return v;
}

__global__ void __launch_bounds__(ST) min_key_kernel(const double* __restrict__ eig, int64_t s,
                                                     unsigned long long* __restrict__ out) {
  unsigned long long k = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)ST + threadIdx.x; i < s; i += (int64_t)gridDim.x * ST)
    k = min(k, ordered_key(eig[i]));
  for (int o = 16; o; o >>= 1) k = min(k, __shfl_xor_sync(0xffffffffu, k, o));
  if ((threadIdx.x & 31) == 0) atomicMin(out, k);
}

// build_operator's clamp (embedding.cpp:128-129) and from_parts' √max(λ, 0) (:108-110). −0.0 becomes
// +0.0 so that the radix order below agrees with the comparator a > b (which ties the two zeros).
__global__ void __launch_bounds__(ST) clamp_sqrt_kernel(double* __restrict__ eig, int64_t s,
                                                        double* __restrict__ sqrt_full, unsigned* __restrict__ iota) {
  for (int64_t i = blockIdx.x * (int64_t)ST + threadIdx.x; i < s; i += (int64_t)gridDim.x * ST) {
    double v = eig[i];
    v = v < 0.0 ? 0.0 : v + 0.0;
    eig[i] = v;
    sqrt_full[i] = sqrt(fmax(v, 0.0));
    iota[i] = (unsigned)i;
  }
}

// truncated(k) (embedding.cpp:153-163): the last k entries of the stable descending order are zeroed
__global__ void __launch_bounds__(ST) zero_tail_kernel(const unsigned* __restrict__ perm, int64_t s, int64_t k,
                                                       double* __restrict__ sqrt_trunc) {
  for (int64_t j = s - k + blockIdx.x * (int64_t)ST + threadIdx.x; j < s; j += (int64_t)gridDim.x * ST)
    sqrt_trunc[perm[j]] = 0.0;
}

__global__ void __launch_bounds__(ST) diff_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                  int64_t s, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)ST + threadIdx.x; i < s; i += (int64_t)gridDim.x * ST) out[i] = a[i] - b[i];
}

int grid_for(int64_t s) { return (int)std::min<int64_t>((s + ST - 1) / ST, 148 * 16); }

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return OSC_OK;
  } catch (...) {
    return c_api_error(std::current_exception());
  }
}

void make_truncation(Level* L, int64_t k) {
  Ctx* c = L->ctx;
  OSC_REQUIRE(k >= 0 && k < L->s, "truncated: k must lie in [0, s); at least one mode must survive");
  OSC_REQUIRE(L->perm.p != nullptr || k == 0,
              "osc_level_retruncate: the level holds no device order (create it with osc_level_create_device)");
  L->sqrt_comp.release();
  if (k == 0) {
    L->sqrt_trunc.release();
    L->k_trunc = 0;
    return;
  }
  L->sqrt_trunc.ensure(sizeof(double) * L->s);
  OSC_CUDA(cudaMemcpyAsync(L->sqrt_trunc.p, L->sqrt_full.p, sizeof(double) * L->s, cudaMemcpyDeviceToDevice,
                           c->stream));
  {
    KScope ks(c, "setup.truncate");
    zero_tail_kernel<<<grid_for(k), ST, 0, c->stream>>>(L->perm.as<unsigned>(), L->s, k, L->sqrt_trunc.as<double>());
    OSC_CUDA(cudaGetLastError());
  }
  OSC_CUDA(cudaStreamSynchronize(c->stream));
  L->k_trunc = k;
}
}  // namespace
}  // namespace osc

using namespace osc;

extern "C" {

int osc_level_create_device(osc_ctx* c, int m, int family, double sigma2, double lambda, double nu_or_p,
                            const double* fractions, int n_fractions, double tol_spd_factor, int64_t k_trunc,
                            osc_level** out) {
  return guarded([&] {
    OSC_REQUIRE(c && out, "osc_level_create_device: null argument");
    OSC_REQUIRE(family == OSC_COV_MATERN || family == OSC_COV_SEPARABLE_EXP,
                "osc_level_create_device: unknown covariance family");
    OSC_REQUIRE(spectrum_device_supported(family, nu_or_p),
                "osc_level_create_device: Matern nu must lie in (0, 64] (use osc_build_spectrum)");
    OSC_CUDA(cudaSetDevice(c->device));
    auto* L = new osc_level();
    L->ctx = c;
    L->m = m;
    DevBuf key, sorted_keys, iota, tmp;
    auto drop = [&] {
      key.release();
      sorted_keys.release();
      iota.release();
      tmp.release();
    };
    try {
      key.ensure(sizeof(unsigned long long));
      L->J = padding_schedule(m, family, sigma2, lambda, nu_or_p, fractions, n_fractions, tol_spd_factor, [&](int J) {
        const int n = 2 * (m + J);
        const int64_t s = (int64_t)n * n;
        L->eig.ensure(sizeof(double) * s);
        spectrum_device_into(c, m, J, family, sigma2, lambda, nu_or_p, L->eig.as<double>());
        OSC_CUDA(cudaMemsetAsync(key.p, 0xff, sizeof(unsigned long long), c->stream));
        {
          KScope ks(c, "setup.min");
          min_key_kernel<<<grid_for(s), ST, 0, c->stream>>>(L->eig.as<double>(), s, key.as<unsigned long long>());
          OSC_CUDA(cudaGetLastError());
        }
        unsigned long long k = 0;
        OSC_CUDA(cudaMemcpyAsync(&k, key.p, sizeof k, cudaMemcpyDeviceToHost, c->stream));
        OSC_CUDA(cudaStreamSynchronize(c->stream));
        return key_to_double(k);
      });
      L->n = 2 * (m + L->J);
      L->s = (int64_t)L->n * L->n;
      OSC_REQUIRE(k_trunc >= 0 && k_trunc < L->s,
                  "truncated: k must lie in [0, s); at least one mode must survive");
      const int64_t s = L->s;
      L->sqrt_full.ensure(sizeof(double) * s);
      L->perm.ensure(sizeof(unsigned) * s);
      iota.ensure(sizeof(unsigned) * s);
      sorted_keys.ensure(sizeof(double) * s);
      {
        KScope ks(c, "setup.sqrt");
        clamp_sqrt_kernel<<<grid_for(s), ST, 0, c->stream>>>(L->eig.as<double>(), s, L->sqrt_full.as<double>(),
                                                             iota.as<unsigned>());
        OSC_CUDA(cudaGetLastError());
      }
      // from_parts' stable_sort by a > b (embedding.cpp:105-107): a stable descending radix sort of
      // (λ, index) pairs keeps equal eigenvalues in index order
      size_t tmp_bytes = 0;
      OSC_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, L->eig.as<double>(),
                                                        sorted_keys.as<double>(), iota.as<unsigned>(),
                                                        L->perm.as<unsigned>(), (int)s, 0, 64, c->stream));
      tmp.ensure(tmp_bytes);
      {
        KScope ks(c, "setup.sort");
        OSC_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, tmp_bytes, L->eig.as<double>(),
                                                          sorted_keys.as<double>(), iota.as<unsigned>(),
                                                          L->perm.as<unsigned>(), (int)s, 0, 64, c->stream));
      }
      OSC_CUDA(cudaStreamSynchronize(c->stream));
      make_truncation(L, k_trunc);
      upload_twiddles(L);
    } catch (...) {
      drop();
      for (DevBuf* b : {&L->sqrt_full, &L->sqrt_trunc, &L->twiddle, &L->eig, &L->perm, &L->sqrt_comp}) b->release();
      delete L;
      throw;
    }
    drop();
    *out = L;
  });
}

int osc_level_retruncate(osc_level* L, int64_t k_trunc) {
  return guarded([&] {
    OSC_REQUIRE(L && L->ctx, "osc_level_retruncate: null level");
    OSC_CUDA(cudaSetDevice(L->ctx->device));
    OSC_CUDA(cudaStreamSynchronize(L->ctx->stream));
    make_truncation(L, k_trunc);
  });
}

int osc_level_eigenvalues(osc_level* L, double* out) {
  return guarded([&] {
    OSC_REQUIRE(L && out, "osc_level_eigenvalues: null argument");
    OSC_REQUIRE(L->eig.p != nullptr,
                "osc_level_eigenvalues: the level holds no device eigenvalues (create it with osc_level_create_device)");
    OSC_CUDA(cudaSetDevice(L->ctx->device));
    OSC_CUDA(cudaMemcpyAsync(out, L->eig.p, sizeof(double) * L->s, cudaMemcpyDeviceToHost, L->ctx->stream));
    OSC_CUDA(cudaStreamSynchronize(L->ctx->stream));
  });
}

int osc_smoothing_error(osc_level* L, int n_samples, uint64_t seed, double out[2], double* sup_out) {
  return guarded([&] {
    OSC_REQUIRE(L && out, "osc_smoothing_error: null argument");
    OSC_REQUIRE(n_samples >= 2, "smoothing_error_estimate: need at least 2 samples");
    Ctx* c = L->ctx;
    OSC_CUDA(cudaSetDevice(c->device));
    std::vector<double> sup((size_t)n_samples, 0.0);
    if (L->k_trunc > 0) {
      if (!L->sqrt_comp.p) {
        L->sqrt_comp.ensure(sizeof(double) * L->s);
        KScope ks(c, "setup.comp");
        diff_kernel<<<grid_for(L->s), ST, 0, c->stream>>>(L->sqrt_full.as<double>(), L->sqrt_trunc.as<double>(), L->s,
                                                          L->sqrt_comp.as<double>());
        OSC_CUDA(cudaGetLastError());
      }
      c->out_q.ensure(sizeof(double) * n_samples);
      c->out_i.ensure(sizeof(int) * n_samples);
      OSC_CUDA(cudaMemsetAsync(c->out_q.p, 0, sizeof(double) * n_samples, c->stream));
      OSC_CUDA(cudaMemsetAsync(c->out_i.p, 0, sizeof(int) * n_samples, c->stream));
      // NormalStream(seed, 0, i) (embedding.cpp:214); the fine window only
      ce_sample_launch(c, L, L->sqrt_comp.as<double>(), nullptr, seed, 0, 0, n_samples, false, nullptr, nullptr,
                       c->out_i.as<int>(), c->out_q.as<unsigned long long>());
      std::vector<int> bad((size_t)n_samples);
      OSC_CUDA(cudaMemcpyAsync(sup.data(), c->out_q.p, sizeof(double) * n_samples, cudaMemcpyDeviceToHost, c->stream));
      OSC_CUDA(cudaMemcpyAsync(bad.data(), c->out_i.p, sizeof(int) * n_samples, cudaMemcpyDeviceToHost, c->stream));
      OSC_CUDA(cudaStreamSynchronize(c->stream));
      c->flush_stats();
      for (int b : bad)
        if (b) throw osc::Error(OSC_ERR_NUMERICAL, "sample: non-finite field value");
    }
    double mean = 0.0, m2 = 0.0;  // Welford in index order (embedding.cpp:220-222)
    for (int i = 0; i < n_samples; ++i) {
      const double delta = sup[(size_t)i] - mean;
      mean += delta / (i + 1);
      m2 += delta * (sup[(size_t)i] - mean);
    }
    out[0] = mean;
    out[1] = m2 / (n_samples - 1);
    if (sup_out) std::memcpy(sup_out, sup.data(), sizeof(double) * n_samples);
  });
}

// ---- OSC1 (embedding.cpp:262-294): "OSC1", u32 d, u32 m[d], u32 J[d], u64 s, s little-endian f64 ----
int osc_spectrum_save(const char* path, int m, int J, const double* eigenvalues, int64_t s) {
  return guarded([&] {
    OSC_REQUIRE(path && eigenvalues, "save_spectrum: null argument");
    OSC_REQUIRE(m >= 1 && J >= 0 && s == (int64_t)(2 * (m + J)) * (2 * (m + J)),
                "save_spectrum: eigenvalue count must equal the embedding size");
    FILE* f = std::fopen(path, "wb");
    if (!f) throw osc::Error(OSC_ERR_CONFIG, std::string("save_spectrum: cannot open ") + path);
    auto put = [&](uint64_t v, int bytes) {
      unsigned char b[8];
      for (int i = 0; i < bytes; ++i) b[i] = (unsigned char)(v >> (8 * i));
      return std::fwrite(b, 1, (size_t)bytes, f) == (size_t)bytes;
    };
    bool ok = std::fwrite("OSC1", 1, 4, f) == 4;
    ok = ok && put(2, 4) && put((uint64_t)m, 4) && put((uint64_t)m, 4) && put((uint64_t)J, 4) && put((uint64_t)J, 4) &&
         put((uint64_t)s, 8);
    for (int64_t i = 0; ok && i < s; ++i) {
      uint64_t bits;
      std::memcpy(&bits, eigenvalues + i, 8);
      ok = put(bits, 8);
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw osc::Error(OSC_ERR_CONFIG, std::string("save_spectrum: write failed for ") + path);
  });
}

int osc_spectrum_load(const char* path, int* m_out, int* J_out, int64_t* s_out, double** eig_out) {
  return guarded([&] {
    OSC_REQUIRE(path && m_out && J_out && s_out && eig_out, "load_spectrum: null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw osc::Error(OSC_ERR_CONFIG, std::string("load_spectrum: cannot open ") + path);
    double* buf = nullptr;
    try {
      auto get = [&](int bytes, uint64_t& v) {
        unsigned char b[8];
        if (std::fread(b, 1, (size_t)bytes, f) != (size_t)bytes) return false;
        v = 0;
        for (int i = 0; i < bytes; ++i) v |= (uint64_t)b[i] << (8 * i);
        return true;
      };
      char magic[4];
      if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "OSC1", 4) != 0)
        throw osc::Error(OSC_ERR_CONFIG, std::string("load_spectrum: bad magic in ") + path);
      uint64_t d = 0, m0 = 0, m1 = 0, J0 = 0, J1 = 0, s = 0;
      if (!get(4, d) || d < 1 || d > 2) throw osc::Error(OSC_ERR_CONFIG, "load_spectrum: unsupported dimension");
      OSC_REQUIRE(d == 2, "load_spectrum: only d = 2 is supported by the device path");
      if (!get(4, m0) || !get(4, m1) || !get(4, J0) || !get(4, J1) || !get(8, s) || m0 != m1 || J0 != J1 ||
          s != (2 * (m0 + J0)) * (2 * (m1 + J1)))
        throw osc::Error(OSC_ERR_CONFIG, std::string("load_spectrum: inconsistent header in ") + path);
      buf = static_cast<double*>(std::malloc(sizeof(double) * s));
      if (!buf) throw std::bad_alloc();
      for (uint64_t i = 0; i < s; ++i) {
        uint64_t bits;
        if (!get(8, bits)) throw osc::Error(OSC_ERR_CONFIG, std::string("load_spectrum: truncated file ") + path);
        std::memcpy(buf + i, &bits, 8);
      }
      *m_out = (int)m0;
      *J_out = (int)J0;
      *s_out = (int64_t)s;
      *eig_out = buf;
    } catch (...) {
      std::free(buf);
      std::fclose(f);
      throw;
    }
    std::fclose(f);
  });
}

}  // extern "C"
