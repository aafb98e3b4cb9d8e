// Projection key encoder (encoder.hpp:73-118, default Variant::projection).
// The Gaussian matrix per chunk shape is generated on the host from the
// reference's library-independent stream (mt19937_64 + explicit Box-Muller,
// encoder.cpp:32-53), bit-identical to the reference, and kept resident in
// HBM in an interleaved (re, im) column order for the device GEMM.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "device.hpp"
#include "geometry.hpp"

namespace mlrg {

/// encoder.hpp:15-22; numeric values are part of the memo keys.
enum class OpId : std::uint8_t { fu1d = 0, fu2d = 1, fu1d_adj = 2, fu2d_adj = 3, f2d = 4, f2d_adj = 5 };
const char* op_name(OpId op);

std::uint64_t splitmix64(std::uint64_t x);
std::uint64_t shape_seed(std::uint64_t seed, Shape3 s);

/// Reference-layout matrix [key_dim][2n] (encoder.cpp:369-379), host only.
std::vector<float> projection_matrix(Shape3 shape, int key_dim, std::uint64_t seed);

/// encoder.cpp:66-86: signed permutation seeded by (location, op).
void slot_mix(float* key, int key_dim, std::uint64_t seed, std::int64_t location, OpId op);

/// CNN key encoder weights (encoder.hpp:60-90): conv1 2 -> 32 ch 5x5 stride 2,
/// conv2 32 -> 64 ch 3x3 stride 2, global average pool, FC 64 -> key_dim.
struct CnnWeights {
  int c1_out = 32, c1_k = 5, c2_out = 64, c2_k = 3, key_dim = 60;
  std::vector<float> c1w, c1b, c2w, c2b, fcw, fcb;
  /// init_cnn (encoder.cpp:441-470): He-scaled draws from one GaussianStream
  /// seeded splitmix64(seed ^ 0xC4E1A5), biases zero.
  static CnnWeights init(int key_dim, std::uint64_t seed);
  /// Encoder::load_weights (encoder.cpp:636-680): "LENC" v1 file of a cnn encoder.
  static CnnWeights load(const std::string& path, int key_dim, std::uint64_t seed);
};

/// Device copies of the CNN weights (kernels in cnn.cu).
struct CnnDevice {
  CnnWeights host;
  DeviceBuffer<float> c1w, c1b, c2w, c2b, fcw, fcb;
};

class Encoder {
 public:
  Encoder(int key_dim, std::uint64_t seed) : key_dim_(key_dim), seed_(seed) {}
  /// CNN variant (encoder_variant = cnn).
  Encoder(const CnnWeights& w, std::uint64_t seed, cudaStream_t s);
  int key_dim() const { return key_dim_; }
  std::uint64_t seed() const { return seed_; }
  bool cnn() const { return cnn_ != nullptr; }
  const CnnDevice& cnn_device() const { return *cnn_; }

  /// register_shape (encoder.cpp:369-379): builds and uploads once per shape.
  void register_shape(Shape3 shape, cudaStream_t s);
  /// Device matrix [key_dim][2n] with columns (2i, 2i+1) = (Re, Im) weights of x_i.
  const float* device_matrix(Shape3 shape) const;

 private:
  int key_dim_;
  std::uint64_t seed_;
  std::shared_ptr<CnnDevice> cnn_;
  std::map<std::array<std::int64_t, 3>, DeviceBuffer<float>> mats_;
};

}  // namespace mlrg
