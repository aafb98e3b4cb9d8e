#include "host_io.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <random>
#include <stdexcept>

namespace mlrg {

namespace {

using cd = std::complex<double>;

std::size_t at(const Shape3& s, std::int64_t i, std::int64_t j, std::int64_t k) {
  return static_cast<std::size_t>((i * s.d1 + j) * s.d2 + k);
}

// Five axis-aligned boxes with U(0.25, 1) values (phantom.cpp:28-51). The
// draws use the standard library distributions, so this matches the
// reference bit for bit when built against the same libstdc++.
void boxes(HostArray& a, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> pos(0.05, 0.6), len(0.2, 0.45), val(0.25, 1.0);
  const Shape3 s = a.shape;
  auto lo = [](double f, std::int64_t n) { return std::clamp<std::int64_t>(static_cast<std::int64_t>(f * static_cast<double>(n)), 0, n - 1); };
  auto hi = [](double f, std::int64_t n) { return std::clamp<std::int64_t>(static_cast<std::int64_t>(f * static_cast<double>(n)), 1, n); };
  for (int b = 0; b < 5; ++b) {
    double f[3], l[3];
    for (double& x : f) x = pos(rng);
    for (double& x : l) x = len(rng);
    const double v = val(rng);
    for (std::int64_t i = lo(f[0], s.d0); i < hi(f[0] + l[0], s.d0); ++i)
      for (std::int64_t j = lo(f[1], s.d1); j < hi(f[1] + l[1], s.d1); ++j)
        for (std::int64_t k = lo(f[2], s.d2); k < hi(f[2] + l[2], s.d2); ++k) a.data[at(s, i, j, k)] += v;
  }
}

// Axis-aligned nested ellipsoids (phantom.cpp:59-91).
void ellipsoids(HostArray& a) {
  struct E {
    double a, b, c, x0, y0, z0, v;
  };
  static const E parts[] = {{0.69, 0.92, 0.81, 0.0, 0.0, 0.0, 1.0},
                            {0.6624, 0.874, 0.78, 0.0, -0.0184, 0.0, -0.8},
                            {0.11, 0.31, 0.22, 0.22, 0.0, 0.0, -0.2},
                            {0.16, 0.41, 0.28, -0.22, 0.0, 0.0, -0.2},
                            {0.21, 0.25, 0.41, 0.0, 0.35, -0.15, 0.1},
                            {0.046, 0.046, 0.05, 0.0, 0.1, 0.25, 0.1},
                            {0.046, 0.046, 0.05, 0.0, -0.1, 0.25, 0.1},
                            {0.046, 0.023, 0.05, -0.08, -0.605, 0.0, 0.1},
                            {0.023, 0.023, 0.02, 0.0, -0.606, 0.0, 0.1},
                            {0.023, 0.046, 0.02, 0.06, -0.605, 0.0, 0.1}};
  const Shape3 s = a.shape;
  auto coord = [](std::int64_t q, std::int64_t n) { return 2.0 * (static_cast<double>(q) + 0.5) / static_cast<double>(n) - 1.0; };
  for (std::int64_t i = 0; i < s.d0; ++i)
    for (std::int64_t j = 0; j < s.d1; ++j)
      for (std::int64_t k = 0; k < s.d2; ++k) {
        const double x = coord(i, s.d0), y = coord(j, s.d1), z = coord(k, s.d2);
        double acc = 0.0;
        for (const E& e : parts) {
          const double dx = (x - e.x0) / e.a, dy = (y - e.y0) / e.b, dz = (z - e.z0) / e.c;
          if (dx * dx + dy * dy + dz * dz <= 1.0) acc += e.v;
        }
        a.data[at(s, i, j, k)] = acc;
      }
}

// Gaussian noise and one clamped 3-point box blur per axis (phantom.cpp:93-121).
void smooth_noise(HostArray& a, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> noise(0.0, 1.0);
  for (cd& v : a.data) v = noise(rng);
  const Shape3 s = a.shape;
  decltype(a.data) tmp(a.data.size());
  for (int axis = 0; axis < 3; ++axis) {
    const std::int64_t len = s.extent(axis);
    for (std::int64_t i = 0; i < s.d0; ++i)
      for (std::int64_t j = 0; j < s.d1; ++j)
        for (std::int64_t k = 0; k < s.d2; ++k) {
          std::int64_t c[3] = {i, j, k};
          cd acc = 0.0;
          int cnt = 0;
          for (int off = -1; off <= 1; ++off) {
            const std::int64_t q = c[axis] + off;
            if (q < 0 || q >= len) continue;
            std::int64_t idx[3] = {i, j, k};
            idx[axis] = q;
            acc += a.data[at(s, idx[0], idx[1], idx[2])];
            ++cnt;
          }
          tmp[at(s, i, j, k)] = acc / static_cast<double>(cnt);
        }
    std::swap(a.data, tmp);
  }
}

void put_u64(std::vector<std::uint8_t>& b, std::uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}
std::uint64_t get_u64(const std::uint8_t* p) {
  std::uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(p[i]) << (8 * i);
  return v;
}

}  // namespace

HostArray make_phantom(Shape3 shape, const std::string& kind, std::uint64_t seed) {
  if (shape.d0 < 1 || shape.d1 < 1 || shape.d2 < 1) throw std::invalid_argument("phantom shape extents must be positive");
  HostArray a(shape, 0);
  if (kind == "blocks") boxes(a, seed);
  else if (kind == "shepp3d-like" || kind == "shepp3d") ellipsoids(a);
  else if (kind == "random-smooth") smooth_noise(a, seed);
  else throw std::invalid_argument("unknown phantom kind: " + kind);
  double peak = 0.0;
  for (const cd& v : a.data) peak = std::max(peak, std::abs(v));
  if (peak > 0.0)
    for (cd& v : a.data) v /= peak;
  return a;
}

// LVOL: "LVOL", u8 rank 3, u8 domain, 10 zero bytes, 3 x u64 extents, then
// (re, im) little-endian doubles.
void save_lvol(const std::string& path, const HostArray& a) {
  std::vector<std::uint8_t> b = {'L', 'V', 'O', 'L', 3, a.domain};
  b.resize(16, 0);
  put_u64(b, static_cast<std::uint64_t>(a.shape.d0));
  put_u64(b, static_cast<std::uint64_t>(a.shape.d1));
  put_u64(b, static_cast<std::uint64_t>(a.shape.d2));
  const std::size_t off = b.size();
  b.resize(off + a.data.size() * 16);
  std::memcpy(b.data() + off, a.data.data(), a.data.size() * 16);  // x86-64: little-endian doubles
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw std::runtime_error("cannot open for writing: " + path);
  f.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
  if (!f) throw std::runtime_error("short write: " + path);
}

HostArray load_lvol(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open: " + path);
  const std::vector<std::uint8_t> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  if (b.size() < 40 || std::memcmp(b.data(), "LVOL", 4) != 0)
    throw std::runtime_error("not a volume file (bad magic): " + path);
  if (b[4] != 3) throw std::runtime_error("unsupported rank " + std::to_string(b[4]));
  if (b[5] > 1) throw std::runtime_error("bad domain tag in " + path);
  const Shape3 s{static_cast<std::int64_t>(get_u64(b.data() + 16)), static_cast<std::int64_t>(get_u64(b.data() + 24)),
                 static_cast<std::int64_t>(get_u64(b.data() + 32))};
  if (s.d0 < 0 || s.d1 < 0 || s.d2 < 0 || b.size() - 40 != static_cast<std::size_t>(s.count()) * 16)
    throw std::runtime_error("volume payload size does not match extents: " + path);
  HostArray a(s, b[5]);
  std::memcpy(a.data.data(), b.data() + 40, a.data.size() * 16);
  for (const cd& v : a.data)
    if (!std::isfinite(v.real()) || !std::isfinite(v.imag()))
      throw std::runtime_error("volume contains non-finite values: " + path);
  return a;
}

}  // namespace mlrg
