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

class Encoder {
 public:
  Encoder(int key_dim, std::uint64_t seed) : key_dim_(key_dim), seed_(seed) {}
  int key_dim() const { return key_dim_; }
  std::uint64_t seed() const { return seed_; }

  /// register_shape (encoder.cpp:369-379): builds and uploads once per shape.
  void register_shape(Shape3 shape, cudaStream_t s);
  /// Device matrix [key_dim][2n] with columns (2i, 2i+1) = (Re, Im) weights of x_i.
  const float* device_matrix(Shape3 shape) const;

 private:
  int key_dim_;
  std::uint64_t seed_;
  std::map<std::array<std::int64_t, 3>, DeviceBuffer<float>> mats_;
};

}  // namespace mlrg
