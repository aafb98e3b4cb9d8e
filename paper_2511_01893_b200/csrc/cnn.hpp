// CNN key encoder kernels (cnn.cu): the reference's encoder_variant = cnn
// (encoder.cpp:95-197) on the device.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device.hpp"
#include "encoder.hpp"
#include "kernels.hpp"

namespace mlrg::ops {

/// Scratch of encode_cnn (grow-only).
struct CnnWork {
  DeviceBuffer<float> act1, act2;
  DeviceBuffer<double> part, scale;
};

/// keys[s][r] (raw, before slot_mix) and norms2[s] = sum |x_s|^2 for `ns`
/// slabs of `shape` starting at starts[] along its axis.
void encode_cnn(const float2* x, SlabGeom shape, const std::int64_t* starts, int ns, const CnnDevice& w, float* keys,
                double* norms2, CnnWork& work, cudaStream_t s);
void encode_cnn(const double2* x, SlabGeom shape, const std::int64_t* starts, int ns, const CnnDevice& w, float* keys,
                double* norms2, CnnWork& work, cudaStream_t s);

}  // namespace mlrg::ops
