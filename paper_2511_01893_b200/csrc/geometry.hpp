// Acquisition geometry and the gridding plans, built on the host in double
// and uploaded once per geometry (the reference rebuilds them on every
// operator call, nufft.cpp:109-110, 185-187).
//
// Two spreading kernels evaluate the same operator, the non-uniform DFT of
// operators.cpp:87-200 (the reference's `direct` path):
//   gaussian  the reference's own plan (nufft.cpp:48-103): 24 taps per
//             dimension, tau = pi*12 / (n^2 sigma (sigma - 1/2)); it matches
//             the direct NUDFT to ~3e-12 relative.
//   es        exponential-of-semicircle kernel exp(beta (sqrt(1 - z^2) - 1)),
//             10 taps, beta = 2.30 * 10, same oversampled grid (sigma = 2),
//             deconvolved by its Fourier transform (Gauss-Legendre quadrature):
//             ~2e-9 relative to the direct NUDFT (10x below the complex64
//             rounding of the outputs), with 5.8x fewer taps in two dimensions. Its
//             deconvolution spans 4.8x per dimension instead of the Gaussian's
//             23x, so the complex64 grid rounding is amplified less.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mlrg {

constexpr int kSpread = 12;         // nufft.cpp:12
constexpr int kTaps = 2 * kSpread;  // 24 wrapped grid points per target and dimension (gaussian)
constexpr int kEsTaps = 10;         // es kernel width (grid cells)
constexpr double kEsBeta = 2.30 * kEsTaps;

enum class GridKernel : std::uint8_t { es = 0, gaussian = 1 };
inline int kernel_taps(GridKernel k) { return k == GridKernel::gaussian ? kTaps : kEsTaps; }

struct Shape3 {
  std::int64_t d0 = 0, d1 = 0, d2 = 0;
  std::int64_t count() const { return d0 * d1 * d2; }
  std::int64_t extent(int axis) const { return axis == 0 ? d0 : axis == 1 ? d1 : d2; }
  bool operator==(const Shape3&) const = default;
  std::string str() const {
    return "(" + std::to_string(d0) + ", " + std::to_string(d1) + ", " + std::to_string(d2) + ")";
  }
};

/// Tilted-axis geometry (geometry.hpp:14-46): object (n1, n0, n2), detector
/// stack (n_theta, h, w), tilt phi, thetas = 2 pi t / n_theta.
struct Geometry {
  std::int64_t n1 = 0, n0 = 0, n2 = 0, n_theta = 0, h = 0, w = 0;
  double phi = 0.0;
  std::vector<double> thetas;

  /// geometry.cpp:9-25 + validate (27-50); throws std::invalid_argument.
  static Geometry make(std::int64_t n1, std::int64_t n0, std::int64_t n2, std::int64_t n_theta,
                       std::int64_t h, std::int64_t w, double phi);
  void validate() const;

  Shape3 volume_shape() const { return {n1, n0, n2}; }
  Shape3 mid_shape() const { return {n1, h, n2}; }
  Shape3 projection_shape() const { return {n_theta, h, w}; }
};

/// geometry.cpp:52-75.
struct FrequencyGrids {
  std::vector<double> nu_z, nu_x, nu_y;
};
FrequencyGrids frequency_grids(const Geometry& g);

/// One gridding dimension (nufft.cpp:48-103): oversampled size m (a power of
/// two), per-mode deconvolution and, per target, the first wrapped grid index
/// and the `taps` kernel weights, all in double. The operator is
/// out[t] = pref * sum_a weights[t][a] * FFT(deconv * u)[start[t] + a].
struct DimPlan {
  GridKernel kernel = GridKernel::gaussian;
  int taps = kTaps;
  std::int64_t n = 0, center = 0, m = 0;
  int logm = 0;
  double tau = 0.0, pref = 0.0;      // tau: gaussian only
  std::vector<double> deconv;        // [n]
  std::vector<std::int32_t> start;   // [T] wrapped index of tap 0
  std::vector<double> weights;       // [T * taps]
  std::vector<double> phase_re, phase_im;  // e^{-2 pi i nu center} per target

  static DimPlan make(std::int64_t n_modes, const std::vector<double>& freqs,
                      GridKernel kernel = GridKernel::gaussian);
  /// Wrapped grid slot of mode index i: (i - center) mod m.
  std::int64_t wrap(std::int64_t i) const {
    std::int64_t w = (i - center) % m;
    return w < 0 ? w + m : w;
  }
};

}  // namespace mlrg
