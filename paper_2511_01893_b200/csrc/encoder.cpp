#include "encoder.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <numbers>
#include <random>
#include <stdexcept>
#include <thread>

namespace mlrg {

const char* op_name(OpId op) {
  switch (op) {
    case OpId::fu1d: return "fu1d";
    case OpId::fu2d: return "fu2d";
    case OpId::fu1d_adj: return "fu1d_adj";
    case OpId::fu2d_adj: return "fu2d_adj";
    case OpId::f2d: return "f2d";
    case OpId::f2d_adj: return "f2d_adj";
  }
  return "unknown";
}

std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

std::uint64_t shape_seed(std::uint64_t seed, Shape3 s) {
  std::uint64_t m = splitmix64(seed ^ static_cast<std::uint64_t>(s.d0));
  m = splitmix64(m ^ static_cast<std::uint64_t>(s.d1));
  return splitmix64(m ^ static_cast<std::uint64_t>(s.d2));
}

namespace {

// Fills out[0..count) with the reference's GaussianStream values times
// `scale`, rounded to float. The mt19937_64 draws are produced sequentially
// (they form one stream); the Box-Muller transform of each (u1, u2) pair is
// independent and runs on all host threads.
void gaussian_fill(std::uint64_t seed, double scale, std::size_t count, float* out) {
  std::mt19937_64 rng(seed);
  const std::size_t pairs = (count + 1) / 2;
  const std::size_t block = std::size_t{1} << 22;  // pairs per block
  std::vector<std::uint64_t> draws(2 * std::min(pairs, block));
  const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  for (std::size_t p0 = 0; p0 < pairs; p0 += block) {
    const std::size_t np = std::min(block, pairs - p0);
    for (std::size_t i = 0; i < 2 * np; ++i) draws[i] = rng();
    auto work = [&](std::size_t a, std::size_t b) {
      for (std::size_t p = a; p < b; ++p) {
        const double u1 = (static_cast<double>(draws[2 * p] >> 11) + 0.5) * 0x1.0p-53;
        const double u2 = (static_cast<double>(draws[2 * p + 1] >> 11) + 0.5) * 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double ang = 2.0 * std::numbers::pi * u2;
        const std::size_t v = 2 * (p0 + p);
        out[v] = static_cast<float>(r * std::cos(ang) * scale);
        if (v + 1 < count) out[v + 1] = static_cast<float>(r * std::sin(ang) * scale);
      }
    };
    if (np < 65536 || nt == 1) {
      work(0, np);
    } else {
      std::vector<std::thread> th;
      for (unsigned t = 0; t < nt; ++t)
        th.emplace_back(work, np * t / nt, np * (t + 1) / nt);
      for (auto& t : th) t.join();
    }
  }
}

}  // namespace

std::vector<float> projection_matrix(Shape3 shape, int key_dim, std::uint64_t seed) {
  const std::size_t cols = static_cast<std::size_t>(2 * shape.count());
  std::vector<float> mat(static_cast<std::size_t>(key_dim) * cols);
  gaussian_fill(shape_seed(seed, shape), 1.0 / std::sqrt(static_cast<double>(key_dim)), mat.size(), mat.data());
  return mat;
}

void slot_mix(float* key, int key_dim, std::uint64_t seed, std::int64_t location, OpId op) {
  std::uint64_t m = splitmix64(seed ^ 0xA5C1E5D1B7F3C9ull);
  m = splitmix64(m ^ static_cast<std::uint64_t>(location));
  m = splitmix64(m ^ static_cast<std::uint64_t>(static_cast<int>(op)));
  std::mt19937_64 rng(m);
  const std::size_t d = static_cast<std::size_t>(key_dim);
  std::vector<std::uint32_t> perm(d);
  for (std::size_t i = 0; i < d; ++i) perm[i] = static_cast<std::uint32_t>(i);
  for (std::size_t i = d; i > 1; --i) {
    const std::size_t j = static_cast<std::size_t>(rng() % i);
    std::swap(perm[i - 1], perm[j]);
  }
  std::vector<float> out(d);
  for (std::size_t i = 0; i < d; ++i) {
    const float sgn = (rng() & 1ull) ? 1.0f : -1.0f;
    out[i] = sgn * key[perm[i]];
  }
  std::copy(out.begin(), out.end(), key);
}

void Encoder::register_shape(Shape3 shape, cudaStream_t s) {
  const std::array<std::int64_t, 3> k{shape.d0, shape.d1, shape.d2};
  if (mats_.count(k)) return;
  const std::size_t n = static_cast<std::size_t>(shape.count());
  const std::vector<float> ref = projection_matrix(shape, key_dim_, seed_);
  std::vector<float> inter(ref.size());
  for (int r = 0; r < key_dim_; ++r) {
    const float* src = ref.data() + static_cast<std::size_t>(r) * 2 * n;
    float* dst = inter.data() + static_cast<std::size_t>(r) * 2 * n;
    for (std::size_t i = 0; i < n; ++i) {
      dst[2 * i] = src[i];
      dst[2 * i + 1] = src[n + i];
    }
  }
  DeviceBuffer<float> buf;
  buf.upload(inter, s);
  MLRG_CUDA(cudaStreamSynchronize(s));
  mats_.emplace(k, std::move(buf));
}

const float* Encoder::device_matrix(Shape3 shape) const {
  const auto it = mats_.find({shape.d0, shape.d1, shape.d2});
  if (it == mats_.end()) throw std::invalid_argument("encoder: shape " + shape.str() + " not registered");
  return it->second.get();
}

}  // namespace mlrg
