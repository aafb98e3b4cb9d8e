#include "encoder.hpp"

#include <algorithm>
#include <array>
#include <cstring>
#include <fstream>
#include <iterator>
#include <cmath>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
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

namespace {
// GaussianStream::next() values (encoder.cpp:29-53) in order, unscaled.
std::vector<double> gaussian_stream(std::uint64_t seed, std::size_t count) {
  std::mt19937_64 rng(seed);
  std::vector<double> out(count);
  for (std::size_t v = 0; v < count; v += 2) {
    const double u1 = (static_cast<double>(rng() >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = (static_cast<double>(rng() >> 11) + 0.5) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * std::numbers::pi * u2;
    out[v] = r * std::cos(ang);
    if (v + 1 < count) out[v + 1] = r * std::sin(ang);  // the spare
  }
  return out;
}
}  // namespace

CnnWeights CnnWeights::init(int key_dim, std::uint64_t seed) {
  CnnWeights w;
  w.key_dim = key_dim;
  const std::size_t n1 = static_cast<std::size_t>(w.c1_out * 2 * w.c1_k * w.c1_k);
  const std::size_t n2 = static_cast<std::size_t>(w.c2_out * w.c1_out * w.c2_k * w.c2_k);
  const std::size_t n3 = static_cast<std::size_t>(key_dim * w.c2_out);
  // one stream for the three tensors; each count is even, so no spare crosses a tensor
  const std::vector<double> g = gaussian_stream(splitmix64(seed ^ 0xC4E1A5ull), n1 + n2 + n3);
  auto fill = [&](std::vector<float>& v, std::size_t off, std::size_t n, double fan_in) {
    const double s = std::sqrt(2.0 / fan_in);
    v.resize(n);
    for (std::size_t i = 0; i < n; ++i) v[i] = static_cast<float>(g[off + i] * s);
  };
  fill(w.c1w, 0, n1, 2.0 * w.c1_k * w.c1_k);
  fill(w.c2w, n1, n2, static_cast<double>(w.c1_out) * w.c2_k * w.c2_k);
  fill(w.fcw, n1 + n2, n3, static_cast<double>(w.c2_out) * 25.0);
  w.c1b.assign(static_cast<std::size_t>(w.c1_out), 0.0f);
  w.c2b.assign(static_cast<std::size_t>(w.c2_out), 0.0f);
  w.fcb.assign(static_cast<std::size_t>(key_dim), 0.0f);
  return w;
}

CnnWeights CnnWeights::load(const std::string& path, int key_dim, std::uint64_t seed) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open: " + path);
  std::vector<unsigned char> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  std::size_t at = 0;
  auto take = [&](void* dst, std::size_t n) {
    if (at + n > b.size()) throw std::runtime_error("weights: truncated file " + path);
    std::memcpy(dst, b.data() + at, n);
    at += n;
  };
  char magic[4];
  take(magic, 4);
  if (std::memcmp(magic, "LENC", 4) != 0) throw std::runtime_error("not a weights file (bad magic): " + path);
  std::uint16_t version = 0;
  take(&version, 2);
  if (version != 1) throw std::runtime_error("unsupported weights version");
  std::uint8_t variant = 0;
  take(&variant, 1);
  if (variant != 1) throw std::invalid_argument("weights file holds a projection encoder, not a cnn");
  std::uint32_t kd = 0, nt = 0;
  take(&kd, 4);
  take(&nt, 4);
  if (nt != 6) throw std::runtime_error("weights: cnn file must hold 6 tensors");
  (void)key_dim;
  CnnWeights w = init(static_cast<int>(kd), seed);
  for (std::vector<float>* t : {&w.c1w, &w.c1b, &w.c2w, &w.c2b, &w.fcw, &w.fcb}) {
    std::uint8_t rank = 0;
    take(&rank, 1);
    std::uint64_t n = 1;
    for (int d = 0; d < rank; ++d) {
      std::uint64_t dim = 0;
      take(&dim, 8);
      n *= dim;
    }
    if (n != t->size()) throw std::runtime_error("weights: unexpected tensor size in " + path);
    take(t->data(), n * sizeof(float));
  }
  return w;
}

Encoder::Encoder(const CnnWeights& w, std::uint64_t seed, cudaStream_t s)
    : key_dim_(w.key_dim), seed_(seed), cnn_(std::make_shared<CnnDevice>()) {
  cnn_->host = w;
  cnn_->c1w.upload(w.c1w, s);
  cnn_->c1b.upload(w.c1b, s);
  cnn_->c2w.upload(w.c2w, s);
  cnn_->c2b.upload(w.c2b, s);
  cnn_->fcw.upload(w.fcw, s);
  cnn_->fcb.upload(w.fcb, s);
  MLRG_CUDA(cudaStreamSynchronize(s));
}

void Encoder::register_shape(Shape3 shape, cudaStream_t s) {
  if (cnn_) return;  // the cnn takes any shape
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
