// Device plumbing for the host side: CUDA error mapping to exceptions, owning
// device/pinned buffers, and the deterministic two-level reduction buffer.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mlrg {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

/// Launch accounting and opt-in per-kernel CUDA-event timing (bench.py reads
/// both through mlrg_prof_* / mlrg_launch_count).
namespace prof {
void count_launch();
/// Adds n launches (a CUDA graph replay of n captured kernels).
void count_launches(std::uint64_t n);
/// Launches counted so far.
std::uint64_t launches();
bool enabled();
/// Brackets one launch of `name` on `s` with events when profiling is on.
void begin(const char* name, cudaStream_t s);
void end(const char* name, cudaStream_t s);
/// Accumulates a host-side phase's wall time under `name` when profiling is on.
void host_add(const char* name, double ms);
/// Adds the wall time since the previous mark (or HostSpan start) on this
/// thread under `name` (sub-phases of one span).
void host_mark(const char* name);
/// RAII wall timer for host_add.
class HostSpan {
 public:
  explicit HostSpan(const char* name);
  ~HostSpan();
  HostSpan(const HostSpan&) = delete;
  HostSpan& operator=(const HostSpan&) = delete;

 private:
  const char* name_;
  long long t0_;
};
}  // namespace prof

#define MLRG_CUDA(call) ::mlrg::cuda_check((call), #call)

/// Process-wide caching allocator for device and pinned host blocks >= 1 MiB:
/// cudaMalloc maps (and clears) pages at ~30 ms/GiB on B200, which made every
/// drop-in mlr_reconstruct pay seconds of setup. Freed blocks stay mapped and
/// are reused for requests of up to their size (at most 2x larger); a reuse
/// after any release synchronises the device first, so no kernel of a previous
/// owner can still be using the block. On cudaErrorMemoryAllocation the cache
/// is released and the allocation retried.
namespace alloc {
void* device(std::size_t bytes);
void device_free(void* p, std::size_t bytes);
void* pinned(std::size_t bytes);
void pinned_free(void* p, std::size_t bytes);
void release_cache();
/// Device bytes held by the cache (free for this process's next allocations).
std::size_t cached_device_bytes();
}  // namespace alloc
#define MLRG_LAUNCH_CHECK(name) (::mlrg::prof::count_launch(), ::mlrg::cuda_check(cudaGetLastError(), name))

/// Owning device allocation (cudaMalloc), movable, zero-length allowed.
template <class T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) { resize(n); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept
      : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)), cap_(std::exchange(o.cap_, 0)) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
      cap_ = std::exchange(o.cap_, 0);
    }
    return *this;
  }
  /// Grow-only: shrinking keeps the allocation (no release/reallocate churn
  /// when a caller alternates sizes, e.g. per-call scratch of ragged slabs).
  void resize(std::size_t n) {
    if (n <= cap_) {
      n_ = n;
      return;
    }
    release();
    p_ = static_cast<T*>(alloc::device(n * sizeof(T)));
    n_ = cap_ = n;
  }
  void upload(const T* host, std::size_t n, cudaStream_t s) {
    resize(n);
    if (n) MLRG_CUDA(cudaMemcpyAsync(p_, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
  void zero(cudaStream_t s) {
    if (n_) MLRG_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }

 private:
  void release() {
    if (p_) alloc::device_free(p_, cap_ * sizeof(T));
    p_ = nullptr;
    n_ = cap_ = 0;
  }
  T* p_ = nullptr;
  std::size_t n_ = 0, cap_ = 0;
};

/// Owning page-locked host allocation for D2H of small results.
template <class T>
class PinnedBuffer {
 public:
  PinnedBuffer() = default;
  ~PinnedBuffer() {
    if (p_) alloc::pinned_free(p_, n_ * sizeof(T));
  }
  PinnedBuffer(const PinnedBuffer&) = delete;
  PinnedBuffer& operator=(const PinnedBuffer&) = delete;
  PinnedBuffer(PinnedBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  PinnedBuffer& operator=(PinnedBuffer&& o) noexcept {
    if (this != &o) {
      if (p_) alloc::pinned_free(p_, n_ * sizeof(T));
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
    }
    return *this;
  }
  void reserve(std::size_t n) {
    if (n <= n_) return;
    if (p_) alloc::pinned_free(p_, n_ * sizeof(T));
    p_ = nullptr;
    p_ = static_cast<T*>(alloc::pinned(n * sizeof(T)));
    n_ = n;
  }
  T* get() const { return p_; }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

/// Per-CTA partial sums written by the fused kernels; the host adds them in
/// CTA order, so every reduction is deterministic (no float atomics).
class Partials {
 public:
  static constexpr int kMaxSlots = 1 << 20;  // 8 MB: the RSP pass of ~14K planes per rank
  Partials() {
    dev_.resize(static_cast<std::size_t>(kMaxSlots));
    host_.reserve(static_cast<std::size_t>(kMaxSlots));
  }
  double* dev() const { return dev_.get(); }
  /// A [count / nv][nv] table of CTA partials at slot offset `off`.
  struct Range {
    int off, count, nv;
  };
  /// Slot offset for reductions that stay pending across other reducing
  /// kernels (they write from slot 0) until a batched sum() reads them.
  static constexpr int kParked = kMaxSlots / 2;
  /// Column sums of several tables read back with one stream synchronisation
  /// (each table summed in CTA order, as sum() does).
  std::vector<std::vector<double>> sum(const std::vector<Range>& ranges, cudaStream_t s) {
    for (const Range& r : ranges) {
      if (r.off < 0 || r.count < 0 || r.off + r.count > kMaxSlots) throw std::logic_error("Partials: range out of bounds");
      if (r.nv <= 0 || r.count % r.nv) throw std::logic_error("Partials: count is not a multiple of nv");
      if (r.count)
        MLRG_CUDA(cudaMemcpyAsync(host_.get() + r.off, dev_.get() + r.off, static_cast<std::size_t>(r.count) * sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
    }
    MLRG_CUDA(cudaStreamSynchronize(s));
    std::vector<std::vector<double>> out;
    for (const Range& r : ranges) {
      std::vector<double> v(static_cast<std::size_t>(r.nv), 0.0);
      for (int i = 0; i < r.count; ++i) v[static_cast<std::size_t>(i % r.nv)] += host_.get()[r.off + i];
      out.push_back(std::move(v));
    }
    return out;
  }
  /// sum(count, nv, s) in two halves: enqueue the copy of the table (stream
  /// order puts it before any later kernel that reuses the slots), then wait for
  /// that copy alone and sum. Nothing may read host slots [0, count) in between.
  void sum_begin(int count, cudaStream_t s) {
    if (count > kMaxSlots) throw std::logic_error("Partials: too many slots");
    if (!ev_) MLRG_CUDA(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming));
    MLRG_CUDA(cudaMemcpyAsync(host_.get(), dev_.get(), static_cast<std::size_t>(count) * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
    MLRG_CUDA(cudaEventRecord(ev_, s));
  }
  std::vector<double> sum_end(int count, int nv) {
    if (count % nv) throw std::logic_error("Partials: count is not a multiple of nv");
    MLRG_CUDA(cudaEventSynchronize(ev_));
    std::vector<double> out(static_cast<std::size_t>(nv), 0.0);
    for (int i = 0; i < count; ++i) out[static_cast<std::size_t>(i % nv)] += host_.get()[i];
    return out;
  }
  ~Partials() {
    if (ev_) cudaEventDestroy(ev_);
  }
  Partials(const Partials&) = delete;
  Partials& operator=(const Partials&) = delete;
  /// Copies `count` doubles back (synchronising `s`) and returns the column sums
  /// of a [count / nv][nv] table.
  std::vector<double> sum(int count, int nv, cudaStream_t s) {
    if (count > kMaxSlots) throw std::logic_error("Partials: too many slots");
    if (count % nv) throw std::logic_error("Partials: count is not a multiple of nv");
    MLRG_CUDA(cudaMemcpyAsync(host_.get(), dev_.get(), static_cast<std::size_t>(count) * sizeof(double),
                              cudaMemcpyDeviceToHost, s));
    MLRG_CUDA(cudaStreamSynchronize(s));
    std::vector<double> out(static_cast<std::size_t>(nv), 0.0);
    for (int i = 0; i < count; ++i) out[static_cast<std::size_t>(i % nv)] += host_.get()[i];
    return out;
  }

 private:
  DeviceBuffer<double> dev_;
  PinnedBuffer<double> host_;
  cudaEvent_t ev_ = nullptr;
};

/// Number of SMs of the current device (grids are sized in multiples of it).
int sm_count();

}  // namespace mlrg
