// Host-side level setup (one-time per level, outside the per-sample path):
// covariance kernels, the embedding's first row, its spectrum, the SPD padding schedule.
// Restates, as B200-host C++ (threaded over std::thread), the reference's
//   CovarianceModel::operator()          src/covariance.cpp:47-62
//   cutoff_phi / periodic_eval            src/covariance.cpp:87-115
//   PeriodisationParams::from_padding     src/covariance.cpp:82-85
//   build_first_row                       src/embedding.cpp:22-65
//   spectrum (λ = √s·Re F row, imag check) src/embedding.cpp:67-88
//   build_operator (padding schedule)     src/embedding.cpp:114-151
// The first row is symmetric in each dimension, so only the (n/2+1)² distinct displacements
// are evaluated. The spectrum uses this file's own 2-D FFT (radix-2, direct DFT otherwise).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/oscfield_b200.h"

namespace osc {

struct SetupError {
  int code;
  std::string msg;
};

namespace {

unsigned n_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return std::max(1u, std::min(h == 0 ? 4u : h, 64u));
}

template <typename F>
void parallel_for(int64_t n, F&& f) {
  const unsigned T = n_threads();
  if (n < 64 || T == 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t chunk = (n + T - 1) / T;
  for (unsigned t = 0; t < T; ++t) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&f, lo, hi] {
      for (int64_t i = lo; i < hi; ++i) f(i);
    });
  }
  for (auto& th : pool) th.join();
}

struct Model {
  int family;
  double sigma2, lambda, nu_or_p;
  // covariance.cpp:47-62
  double operator()(double t0, double t1) const {
    if (!std::isfinite(t0) || !std::isfinite(t1))
      throw SetupError{OSC_ERR_CONFIG, "CovarianceModel: non-finite displacement"};
    if (family == OSC_COV_SEPARABLE_EXP) {
      const double p = nu_or_p;
      const double s = std::pow(std::abs(t0), p) + std::pow(std::abs(t1), p);
      return sigma2 * std::exp(-std::pow(s, 1.0 / p) / lambda);
    }
    const double r = std::sqrt(t0 * t0 + t1 * t1);
    if (r == 0.0) return sigma2;
    const double nu = nu_or_p;
    const double x = std::sqrt(2.0 * nu) * r / lambda;
    if (x < 1e-13) return sigma2;
    const double k = std::cyl_bessel_k(nu, x);
    return sigma2 * std::pow(2.0, 1.0 - nu) / std::tgamma(nu) * std::pow(x, nu) * k;
  }
};

double eta(double x) { return x > 0.0 ? std::exp(-1.0 / x) : 0.0; }

double cutoff_phi(double t, double kappa) {  // covariance.cpp:87-95
  const double a = std::abs(t);
  if (a <= 1.0) return 1.0;
  if (a >= kappa) return 0.0;
  const double up = eta((kappa - a) / (kappa - 1.0));
  const double dn = eta((a - 1.0) / (kappa - 1.0));
  return up / (up + dn);
}

double periodic_eval(const Model& mod, double ell, double kappa, double x0, double x1) {
  const double period = 2.0 * ell;  // covariance.cpp:97-115
  double sum = 0.0;
  for (int n0 = -1; n0 <= 1; ++n0) {
    const double s0 = x0 + period * n0;
    for (int n1 = -1; n1 <= 1; ++n1) {
      const double s1 = x1 + period * n1;
      const double sup = std::max(std::abs(s0), std::abs(s1));
      const double w = cutoff_phi(sup, kappa);
      if (w > 0.0) sum += w * mod(s0, s1);
    }
  }
  return sum;
}

// embedding.cpp:22-65 (square grid, J0 = J1 = J)
std::vector<double> first_row(int m, int J, const Model& mod) {
  const int n = 2 * (m + J);
  const int h = n / 2;
  std::vector<double> tab((size_t)(h + 1) * (h + 1));
  const bool padded = J > 0;
  const double ell = 1.0 + static_cast<double>(J) / m;
  const double kappa = 2.0 * ell - 1.0;
  parallel_for(h + 1, [&](int64_t d1) {
    for (int d0 = 0; d0 <= h; ++d0) {
      const double x0 = static_cast<double>(d0) / m, x1 = static_cast<double>(d1) / m;
      tab[(size_t)d1 * (h + 1) + d0] = padded ? periodic_eval(mod, ell, kappa, x0, x1) : mod(x0, x1);
    }
  });
  std::vector<double> row((size_t)n * n);
  parallel_for(n, [&](int64_t q1) {
    const int d1 = (int)std::min<int64_t>(q1, n - q1);
    for (int q0 = 0; q0 < n; ++q0) {
      const int d0 = std::min(q0, n - q0);
      row[(size_t)q1 * n + q0] = tab[(size_t)d1 * (h + 1) + d0];
    }
  });
  return row;
}

using cd = std::complex<double>;

struct Fft1d {
  int n;
  std::vector<cd> tw;  // exp(+2πi t/n)
  explicit Fft1d(int n_) : n(n_), tw((size_t)n_) {
    for (int t = 0; t < n; ++t) {
      const long double a = 6.283185307179586476925286766559005768L * t / n;
      tw[(size_t)t] = cd((double)std::cos(a), (double)std::sin(a));
    }
  }
  void run(cd* x, std::vector<cd>& scratch) const {
    if ((n & (n - 1)) == 0) {
      for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(x[i], x[j]);
      }
      for (int len = 2; len <= n; len <<= 1) {
        const int half = len >> 1, step = n / len;
        for (int s = 0; s < n; s += len)
          for (int k = 0; k < half; ++k) {
            const cd t = x[s + k + half] * tw[(size_t)k * step];
            x[s + k + half] = x[s + k] - t;
            x[s + k] += t;
          }
      }
      return;
    }
    scratch.assign((size_t)n, cd(0.0, 0.0));
    for (int k = 0; k < n; ++k) {
      cd acc(0.0, 0.0);
      for (int j = 0; j < n; ++j) acc += x[j] * tw[(size_t)(((int64_t)j * k) % n)];
      scratch[(size_t)k] = acc;
    }
    std::copy(scratch.begin(), scratch.end(), x);
  }
};

// λ = √s · Re(F row) with F unitary (+ sign); throws on a non-negligible imaginary part
// (embedding.cpp:67-88).
std::vector<double> spectrum(const std::vector<double>& row, int n) {
  const int64_t s = (int64_t)n * n;
  std::vector<cd> a((size_t)s);
  for (int64_t i = 0; i < s; ++i) a[(size_t)i] = cd(row[(size_t)i], 0.0);
  const Fft1d f(n);
  parallel_for(n, [&](int64_t q1) {
    std::vector<cd> scratch;
    f.run(a.data() + q1 * n, scratch);
  });
  parallel_for(n, [&](int64_t q0) {
    std::vector<cd> line((size_t)n), scratch;
    for (int q1 = 0; q1 < n; ++q1) line[(size_t)q1] = a[(size_t)q1 * n + q0];
    f.run(line.data(), scratch);
    for (int q1 = 0; q1 < n; ++q1) a[(size_t)q1 * n + q0] = line[(size_t)q1];
  });
  const double inv = 1.0 / std::sqrt(static_cast<double>(s));
  const double scale = std::sqrt(static_cast<double>(s));
  double max_imag = 0.0;
  std::vector<double> eig((size_t)s);
  for (int64_t i = 0; i < s; ++i) {
    const cd o = a[(size_t)i] * inv;
    eig[(size_t)i] = scale * o.real();
    max_imag = std::max(max_imag, std::abs(scale * o.imag()));
  }
  if (max_imag > 1e-8 * std::abs(row[0])) {
    std::ostringstream os;
    os << "spectrum: imaginary part " << max_imag << " exceeds tolerance; the first row is not symmetric";
    throw SetupError{OSC_ERR_NUMERICAL, os.str()};
  }
  return eig;
}

}  // namespace

// embedding.cpp:114-151; `attempt_spectrum(J)` returns the raw spectrum of the padding-J embedding
// (host: first_row + spectrum below; device: ce_sample.cu spectrum_device).
std::vector<double> build_spectrum_with(int m, int family, double sigma2, double lambda, double nu_or_p,
                                        const double* fractions, int n_fractions, double tol_factor, int* J_out,
                                        const std::function<std::vector<double>(int)>& attempt_spectrum);

std::vector<double> build_spectrum(int m, int family, double sigma2, double lambda, double nu_or_p,
                                   const double* fractions, int n_fractions, double tol_factor,
                                   int* J_out) {
  const Model mod{family, sigma2, lambda, nu_or_p};
  return build_spectrum_with(m, family, sigma2, lambda, nu_or_p, fractions, n_fractions, tol_factor, J_out,
                             [&](int J) { return spectrum(first_row(m, J, mod), 2 * (m + J)); });
}

// The padding schedule of build_operator (embedding.cpp:114-151): J = 0, then ceil(f·m) per fraction,
// until the spectrum's minimum is ≥ −tol. `attempt_min(J)` builds the padding-J spectrum wherever it
// lives (host vector, device buffer) and returns its smallest eigenvalue; the accepted J is returned.
int padding_schedule(int m, int family, double sigma2, double lambda, double nu_or_p, const double* fractions,
                     int n_fractions, double tol_factor, const std::function<double(int)>& attempt_min) {
  if (m < 1) throw SetupError{OSC_ERR_CONFIG, "GridSpec: resolution must be >= 1"};
  if (!(sigma2 > 0.0) || !std::isfinite(sigma2))
    throw SetupError{OSC_ERR_CONFIG, "CovarianceModel: sigma2 must be positive"};
  if (!(lambda > 0.0) || !std::isfinite(lambda))
    throw SetupError{OSC_ERR_CONFIG, "CovarianceModel: lambda must be positive"};
  if (!(nu_or_p > 0.0) || !std::isfinite(nu_or_p))
    throw SetupError{OSC_ERR_CONFIG, family == OSC_COV_MATERN ? "CovarianceModel: nu must be positive"
                                                              : "CovarianceModel: p must be positive"};
  static const double kDefault[5] = {0.5, 1.0, 2.0, 4.0, 8.0};
  if (!fractions) {
    fractions = kDefault;
    n_fractions = 5;
  }
  if (!(tol_factor > 0.0)) tol_factor = 1e-12;
  std::ostringstream tried;
  auto attempt = [&](int J) -> bool {
    const int n = 2 * (m + J);
    if ((int64_t)n * n > (int64_t{1} << 28))
      throw SetupError{OSC_ERR_CONFIG, "build_first_row: embedding size exceeds the addressable limit"};
    const double mn = attempt_min(J);
    const double tol = tol_factor * static_cast<double>((int64_t)n * n) * sigma2;
    tried << " J=" << J << "," << J << " (min eig " << mn << ")";
    return !(mn < -tol);
  };
  int J = 0;
  bool ok = attempt(0);
  for (int i = 0; i < n_fractions && !ok; ++i) {
    J = static_cast<int>(std::ceil(fractions[i] * m));
    ok = attempt(J);
  }
  if (!ok) {
    std::ostringstream os;
    os << "build_operator: no SPD embedding for "
       << (family == OSC_COV_MATERN ? "matern" : "exponential") << "(sigma2=" << sigma2
       << ", lambda=" << lambda << ", " << (family == OSC_COV_MATERN ? "nu=" : "p=") << nu_or_p
       << "); tried" << tried.str();
    throw SetupError{OSC_ERR_EMBEDDING, os.str()};
  }
  return J;
}

std::vector<double> build_spectrum_with(int m, int family, double sigma2, double lambda, double nu_or_p,
                                        const double* fractions, int n_fractions, double tol_factor, int* J_out,
                                        const std::function<std::vector<double>(int)>& attempt_spectrum) {
  std::vector<double> eig;
  *J_out = padding_schedule(m, family, sigma2, lambda, nu_or_p, fractions, n_fractions, tol_factor, [&](int J) {
    eig = attempt_spectrum(J);
    return *std::min_element(eig.begin(), eig.end());
  });
  for (double& v : eig)
    if (v < 0.0) v = 0.0;
  return eig;
}

// Stable descending order (embedding.cpp:105-107) and the truncation mask (:153-163).
void sqrt_spectra(const double* eig, int64_t s, int64_t k_trunc, std::vector<double>& full,
                  std::vector<double>& trunc) {
  full.resize((size_t)s);
  for (int64_t i = 0; i < s; ++i) full[(size_t)i] = std::sqrt(std::max(eig[i], 0.0));
  trunc.clear();
  if (k_trunc <= 0) return;
  std::vector<int64_t> perm((size_t)s);
  for (int64_t i = 0; i < s; ++i) perm[(size_t)i] = i;
  std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return eig[a] > eig[b]; });
  trunc = full;
  for (int64_t j = s - k_trunc; j < s; ++j) trunc[(size_t)perm[(size_t)j]] = 0.0;
}

}  // namespace osc
