// Independent implementation of the FFTW3 subset declared in fftw3.h. FFTW is absent from this
// image; this stands in for it wherever the pristine reference library is compiled: the CPU checker
// oracle/_ref/ and the GPU-routed reference build integration/_build/ (whose only FFT is the
// one-time spectrum setup, build_operator — every sample runs on the GPU).
//
// Algorithm: per-axis 1-D transforms; each 1-D transform is a recursive
// decimation-in-time mixed-radix Cooley-Tukey over the prime factorisation of
// the length (radix p combine is a direct p-point DFT), with an exact twiddle
// table w[t] = exp(sign * 2*pi*i * t / N) evaluated directly (no recurrences),
// so rounding stays at a few ulp for any N.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {
using cd = std::complex<double>;

struct Axis {
  int n = 1;
  std::vector<int> factors;  // prime factors, smallest first
  std::vector<cd> tw;        // tw[t] = exp(sign*2*pi*i*t/n)
};

void factorise(int n, std::vector<int>& f) {
  for (int p = 2; p * p <= n; ++p)
    while (n % p == 0) { f.push_back(p); n /= p; }
  if (n > 1) f.push_back(n);
}

// out[k] = sum_j in[j*stride] * w^(j*k), length n = prod(factors[fi..]);
// twiddle step = N/n so tw[(j*k*step) % N] is the length-n root.
void fft_rec(const cd* in, long stride, cd* out, int n, const Axis& ax, size_t fi, int step,
             std::vector<cd>& scratch_p) {
  if (n == 1) { out[0] = in[0]; return; }
  const int p = ax.factors[fi];
  const int q = n / p;
  // sub-transforms of the p decimated sequences, stored contiguously out[r*q .. r*q+q)
  for (int r = 0; r < p; ++r) fft_rec(in + r * stride, stride * p, out + r * q, q, ax, fi + 1, step * p, scratch_p);
  // combine: X[k + s*q] = sum_r W_n^{r(k+s q)} Y_r[k]
  std::vector<cd> tmp(static_cast<size_t>(n));
  const int N = ax.n;
  for (int k = 0; k < q; ++k) {
    for (int s = 0; s < p; ++s) {
      const int kk = k + s * q;
      cd acc = 0.0;
      for (int r = 0; r < p; ++r) {
        const long e = (static_cast<long>(r) * kk) % n;
        acc += ax.tw[static_cast<size_t>((e * step) % N)] * out[r * q + k];
      }
      tmp[static_cast<size_t>(kk)] = acc;
    }
  }
  std::memcpy(out, tmp.data(), sizeof(cd) * static_cast<size_t>(n));
}
}  // namespace

struct osc_fftw_plan_s {
  int rank;
  std::vector<int> dims;  // row-major: dims[rank-1] fastest
  std::vector<Axis> axes;
  cd* in;
  cd* out;
};

extern "C" {

fftw_complex* fftw_alloc_complex(size_t n) {
  return static_cast<fftw_complex*>(std::malloc(sizeof(fftw_complex) * (n ? n : 1)));
}

void fftw_free(void* p) { std::free(p); }

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned /*flags*/) {
  if (rank < 1) return nullptr;
  auto* pl = new osc_fftw_plan_s;
  pl->rank = rank;
  pl->dims.assign(n, n + rank);
  pl->in = reinterpret_cast<cd*>(in);
  pl->out = reinterpret_cast<cd*>(out);
  for (int a = 0; a < rank; ++a) {
    Axis ax;
    ax.n = n[a];
    if (ax.n < 1) { delete pl; return nullptr; }
    factorise(ax.n, ax.factors);
    ax.tw.resize(static_cast<size_t>(ax.n));
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (int t = 0; t < ax.n; ++t) {
      const long double ang = two_pi * static_cast<long double>(t) / ax.n;
      ax.tw[static_cast<size_t>(t)] =
          cd(static_cast<double>(std::cos(ang)), sign * static_cast<double>(std::sin(ang)));
    }
    pl->axes.push_back(std::move(ax));
  }
  return pl;
}

void fftw_execute(const fftw_plan pl) {
  long total = 1;
  for (int d : pl->dims) total *= d;
  if (pl->out != pl->in) std::memcpy(pl->out, pl->in, sizeof(cd) * static_cast<size_t>(total));
  cd* data = pl->out;
  std::vector<cd> line, res, scratch;
  for (int a = 0; a < pl->rank; ++a) {
    const int n = pl->dims[a];
    long inner = 1;
    for (int b = a + 1; b < pl->rank; ++b) inner *= pl->dims[b];
    const long outer = total / (inner * n);
    line.resize(static_cast<size_t>(n));
    res.resize(static_cast<size_t>(n));
    for (long o = 0; o < outer; ++o) {
      for (long i = 0; i < inner; ++i) {
        cd* base = data + o * n * inner + i;
        for (int j = 0; j < n; ++j) line[static_cast<size_t>(j)] = base[j * inner];
        fft_rec(line.data(), 1, res.data(), n, pl->axes[a], 0, 1, scratch);
        for (int j = 0; j < n; ++j) base[j * inner] = res[static_cast<size_t>(j)];
      }
    }
  }
}

void fftw_destroy_plan(fftw_plan pl) { delete pl; }

}  // extern "C"
