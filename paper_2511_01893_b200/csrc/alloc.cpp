// Caching allocator behind DeviceBuffer / PinnedBuffer (device.hpp).
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

#include "device.hpp"

namespace mlrg::alloc {

namespace {
constexpr std::size_t kMinCached = 256;  // cudaFree of a small block can stall engine teardown for 100s of ms

struct Cache {
  std::mutex mx;
  std::multimap<std::pair<int, std::size_t>, void*> dev;  // (device, bytes) -> block
  std::multimap<std::size_t, void*> host;
  bool dev_dirty = false;  // a device block was released since the last synchronisation
};
Cache& cache() {
  static Cache* c = new Cache;  // never destroyed: blocks may be released during static teardown
  return *c;
}
int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
}  // namespace

void release_cache() {
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mx);
  if (!c.dev.empty()) cudaDeviceSynchronize();
  for (auto& [k, p] : c.dev) cudaFree(p);
  c.dev.clear();
  for (auto& [k, p] : c.host) cudaFreeHost(p);
  c.host.clear();
  c.dev_dirty = false;
}

std::size_t cached_device_bytes() {
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mx);
  const int d = current_device();
  std::size_t b = 0;
  for (const auto& [k, p] : c.dev)
    if (k.first == d) b += k.second;
  return b;
}

void* device(std::size_t bytes) {
  if (bytes >= kMinCached) {
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mx);
    const int d = current_device();
    auto it = c.dev.lower_bound({d, bytes});
    if (it != c.dev.end() && it->first.first == d && it->first.second <= 2 * bytes) {
      void* p = it->second;
      c.dev.erase(it);
      if (c.dev_dirty) {  // the previous owner's kernels may still run on another stream
        cuda_check(cudaDeviceSynchronize(), "alloc::device (reuse)");
        c.dev_dirty = false;
      }
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    release_cache();
    e = cudaMalloc(&p, bytes);
  }
  cuda_check(e, "cudaMalloc");
  return p;
}

void device_free(void* p, std::size_t bytes) {
  if (!p) return;
  if (bytes < kMinCached) {
    cudaFree(p);
    return;
  }
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mx);
  c.dev.emplace(std::make_pair(current_device(), bytes), p);
  c.dev_dirty = true;
}

void* pinned(std::size_t bytes) {
  if (bytes >= kMinCached) {
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mx);
    auto it = c.host.lower_bound(bytes);
    if (it != c.host.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      c.host.erase(it);
      return p;  // host blocks are only touched by synchronised copies
    }
  }
  void* p = nullptr;
  cuda_check(cudaMallocHost(&p, bytes), "cudaMallocHost");
  return p;
}

void pinned_free(void* p, std::size_t bytes) {
  if (!p) return;
  if (bytes < kMinCached) {
    cudaFreeHost(p);
    return;
  }
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mx);
  c.host.emplace(bytes, p);
}

}  // namespace mlrg::alloc
