// Host-side arrays of the drop-in C API: complex128 row-major volumes with a
// domain tag (array.hpp:38-73), synthetic phantoms (phantom.cpp) and the
// LVOL file format (volume_io.cpp:16-70). Plumbing around the device path.
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include "geometry.hpp"

namespace mlrg {

struct HostArray {
  Shape3 shape;
  std::uint8_t domain = 0;  // 0 = space, 1 = frequency
  std::vector<std::complex<double>> data;
  HostArray() = default;
  HostArray(Shape3 s, std::uint8_t dom)
      : shape(s), domain(dom), data(static_cast<std::size_t>(s.count())) {}
};

/// "blocks", "shepp3d-like" (or "shepp3d") or "random-smooth", normalised to peak 1.
HostArray make_phantom(Shape3 shape, const std::string& kind, std::uint64_t seed);

void save_lvol(const std::string& path, const HostArray& a);
HostArray load_lvol(const std::string& path);

}  // namespace mlrg
