// Boost.Math shim — a build dependency of the reference library in this image (oracle/_ref and
// integration/_build). The reference calls
// boost::math::cyl_bessel_k (proj/src/covariance.cpp:3,60; Boost unpinned,
// expected in the gitignored vendor/). Boost is absent from this image; the
// C++17 special function std::cyl_bessel_k (libstdc++) computes the same
// modified Bessel function of the second kind K_nu(x).
#pragma once
#include <cmath>
namespace boost { namespace math {
inline double cyl_bessel_k(double nu, double x) { return std::cyl_bessel_k(nu, x); }
}}  // namespace boost::math
