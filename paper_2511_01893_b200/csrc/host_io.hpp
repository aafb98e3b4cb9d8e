// Host-side arrays of the drop-in C API: complex128 row-major volumes with a
// domain tag (array.hpp:38-73), synthetic phantoms (phantom.cpp) and the
// LVOL file format (volume_io.cpp:16-70). Plumbing around the device path.
#pragma once

#include <algorithm>
#include <complex>
#include <memory>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "geometry.hpp"

namespace mlrg {

/// Allocator whose value-less construct() leaves the element uninitialised:
/// result volumes are overwritten by a device copy right away, and zero-filling
/// hundreds of MB first cost more than the copy itself.
template <class T>
struct NoInitAllocator : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAllocator<U>;
  };
  NoInitAllocator() = default;
  template <class U>
  NoInitAllocator(const NoInitAllocator<U>&) noexcept {}
  template <class U>
  void construct(U*) noexcept {}
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};

struct HostArray {
  Shape3 shape;
  std::uint8_t domain = 0;  // 0 = space, 1 = frequency
  std::vector<std::complex<double>, NoInitAllocator<std::complex<double>>> data;
  HostArray() = default;
  /// zero = false leaves the samples uninitialised (the caller fills them)
  HostArray(Shape3 s, std::uint8_t dom, bool zero = true)
      : shape(s), domain(dom), data(static_cast<std::size_t>(s.count())) {
    if (zero) std::fill(data.begin(), data.end(), std::complex<double>(0.0, 0.0));
  }
};

/// "blocks", "shepp3d-like" (or "shepp3d") or "random-smooth", normalised to peak 1.
HostArray make_phantom(Shape3 shape, const std::string& kind, std::uint64_t seed);

void save_lvol(const std::string& path, const HostArray& a);
HostArray load_lvol(const std::string& path);

}  // namespace mlrg
