#include "cold_tier.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <stdexcept>

#include "device.hpp"

namespace mlrg {

ColdTier::ColdTier(std::string name, int rank, std::size_t chunk_bytes)
    : name_(std::move(name)), rank_(rank), chunk_bytes_(chunk_bytes) {
  if (!name_.empty() && name_[0] != '/') name_ = "/" + name_;
}

ColdTier::~ColdTier() {
  if (pool_thread_.joinable()) pool_thread_.join();
  for (void* p : pool_) cudaFreeHost(p);
  for (auto& [key, c] : chunks_) {
    if (!c.host) continue;
    if (c.shm) {
      cudaHostUnregister(c.host);
      munmap(c.host, c.bytes);
      if (c.owned) shm_unlink(seg_name(key.first, key.second).c_str());
    } else {
      cudaFreeHost(c.host);
    }
  }
}

std::string ColdTier::seg_name(int owner, int c) const {
  return name_ + ".cold." + std::to_string(owner) + "." + std::to_string(c);
}

ColdRef ColdTier::place(int owner, std::size_t bytes) {
  Cursor& k = cur_[owner];
  if (k.chunks == 0 || k.used + bytes > k.last) {
    k.last = std::max(chunk_bytes_, bytes);
    sizes_[{owner, k.chunks}] = k.last;
    ++k.chunks;
    k.used = 0;
  }
  ColdRef r{owner, k.chunks - 1, k.used};
  k.used += bytes;
  k.total += bytes;
  return r;
}

std::size_t ColdTier::bytes_placed(int owner) const {
  const auto it = cur_.find(owner);
  return it == cur_.end() ? 0 : it->second.total;
}

ColdTier::Chunk& ColdTier::chunk(int owner, int c, std::size_t bytes) {
  Chunk& ch = chunks_[{owner, c}];
  if (ch.host) return ch;
  ch.bytes = bytes;
  if (name_.empty()) {
    if (owner != rank_) throw std::logic_error("cold tier: a private tier holds this rank's values only");
    if (bytes == chunk_bytes_) {
      if (pool_thread_.joinable()) pool_thread_.join();
      std::lock_guard<std::mutex> lk(pool_mu_);
      if (!pool_.empty()) {
        ch.host = pool_.back();
        pool_.pop_back();
        return ch;
      }
    }
    MLRG_CUDA(cudaHostAlloc(&ch.host, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    return ch;
  }
  // shared: the owner creates the segment, every other rank maps it (the
  // owner's spill copy is fenced by the flush barrier before any rank reads)
  const std::string seg = seg_name(owner, c);
  const bool own = owner == rank_;
  int fd = -1;
  if (own) {
    shm_unlink(seg.c_str());
    fd = shm_open(seg.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd >= 0 && ftruncate(fd, static_cast<off_t>(bytes)) != 0) {
      close(fd);
      fd = -1;
    }
  } else {
    fd = shm_open(seg.c_str(), O_RDWR, 0600);
  }
  if (fd < 0) throw std::runtime_error("cold tier: shm segment " + seg + ": " + std::strerror(errno));
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) throw std::runtime_error("cold tier: mmap " + seg + ": " + std::strerror(errno));
  const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(p, bytes);
    throw std::runtime_error(std::string("cold tier: cudaHostRegister: ") + cudaGetErrorString(e));
  }
  ch.host = p;
  ch.shm = true;
  ch.owned = own;
  return ch;
}

void ColdTier::prefetch(std::size_t bytes) {
  if (!name_.empty() || pool_thread_.joinable()) return;
  std::size_t have = 0;
  {
    std::lock_guard<std::mutex> lk(pool_mu_);
    have = pool_.size() * chunk_bytes_;
  }
  const auto it = cur_.find(rank_);
  if (it != cur_.end()) have += it->second.last - it->second.used;  // room left in the open chunk
  if (have >= bytes) return;
  const std::size_t n = (bytes - have + chunk_bytes_ - 1) / chunk_bytes_;
  int dev = 0;
  cudaGetDevice(&dev);
  pool_thread_ = std::thread([this, n, dev] {
    cudaSetDevice(dev);
    for (std::size_t i = 0; i < n; ++i) {
      void* p = nullptr;
      if (cudaHostAlloc(&p, chunk_bytes_, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return;  // place() allocates synchronously (and reports) instead
      }
      std::lock_guard<std::mutex> lk(pool_mu_);
      pool_.push_back(p);
    }
  });
}

void* ColdTier::device_ptr(const ColdRef& r) {
  const auto sz = sizes_.find({r.owner, r.chunk});
  if (sz == sizes_.end()) throw std::logic_error("cold tier: unplaced value");
  Chunk& ch = chunk(r.owner, r.chunk, sz->second);
  void* dev = nullptr;
  MLRG_CUDA(cudaHostGetDevicePointer(&dev, ch.host, 0));
  return static_cast<char*>(dev) + r.offset;
}

void ColdTier::copy_in(const ColdRef& r, const void* dev_src, std::size_t bytes, cudaStream_t s) {
  if (r.owner != rank_) throw std::logic_error("cold tier: only the owner spills its values");
  const auto sz = sizes_.find({r.owner, r.chunk});
  Chunk& ch = chunk(r.owner, r.chunk, sz->second);
  MLRG_CUDA(cudaMemcpyAsync(static_cast<char*>(ch.host) + r.offset, dev_src, bytes, cudaMemcpyDeviceToHost, s));
}

// ---- ValueRing ------------------------------------------------------------------------------

std::size_t ValueRing::alloc(std::size_t bytes) {
  bytes = granule(bytes);
  if (bytes > cap_) throw std::logic_error("value ring: a value larger than the arena");
  if (head_ + bytes > cap_) head_ = 0;
  const std::size_t off = head_;
  head_ += bytes;
  return off;
}

void ValueRing::note(std::uint64_t id, std::size_t off, std::size_t bytes) {
  bytes = granule(bytes);
  live_.push_back(Live{id, off, bytes});
  head_ = off + bytes;
}

std::vector<ValueRing::Live> ValueRing::make_room(std::size_t window) {
  std::vector<Live> out;
  if (live_.empty()) return out;
  window = std::min(window, cap_);
  // zone(s) the next window can write
  std::size_t z0 = head_, z1 = std::min(cap_, head_ + window), w1 = 0;
  if (head_ + window > cap_) w1 = window;  // may wrap: [0, window) too
  auto hits = [&](const Live& v) {
    const std::size_t a = v.off, b = v.off + v.bytes;
    return (a < z1 && b > z0) || (w1 && a < w1);
  };
  std::deque<Live> keep;
  for (const Live& v : live_) {
    if (hits(v)) out.push_back(v);
    else keep.push_back(v);
  }
  live_.swap(keep);
  return out;
}

std::size_t ValueRing::live_bytes() const {
  std::size_t s = 0;
  for (const Live& v : live_) s += v.bytes;
  return s;
}

// ---- ColdSpiller ---------------------------------------------------------------------------

ColdSpiller::ColdSpiller(char* arena, std::size_t capacity, std::size_t window, SetPtr set_ptr)
    : arena_(arena), window_(window), ring_(capacity), set_ptr_(std::move(set_ptr)) {
  MLRG_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
  MLRG_CUDA(cudaEventCreateWithFlags(&ev_ready_, cudaEventDisableTiming));
  MLRG_CUDA(cudaEventCreateWithFlags(&ev_copied_, cudaEventDisableTiming));
}

ColdSpiller::~ColdSpiller() {
  if (side_) {
    cudaStreamSynchronize(side_);
    cudaStreamDestroy(side_);
  }
  if (ev_ready_) cudaEventDestroy(ev_ready_);
  if (ev_copied_) cudaEventDestroy(ev_copied_);
}

std::vector<ColdSpiller::Moved> ColdSpiller::copy_out(const std::vector<ValueRing::Live>& v, cudaStream_t s) {
  std::vector<Moved> out;
  out.reserve(v.size());
  for (const ValueRing::Live& x : v) {
    const ColdRef r = cold_.place(0, x.bytes);
    cold_.copy_in(r, arena_ + x.off, x.bytes, s);
    out.push_back(Moved{x.id, cold_.device_ptr(r)});
  }
  spilled_ += static_cast<std::int64_t>(v.size());
  return out;
}

void ColdSpiller::apply(const std::vector<Moved>& m, cudaStream_t s) {
  if (m.empty()) return;
  std::vector<std::uint64_t> ids;
  std::vector<const void*> ptrs;
  for (const Moved& x : m) {
    ids.push_back(x.id);
    ptrs.push_back(x.ptr);
  }
  set_ptr_(ids, ptrs, s);
}

void ColdSpiller::flush(cudaStream_t s) {
  // 1. last flush's copies are done before window k+1 can overwrite their span
  if (!pending_.empty()) {
    MLRG_CUDA(cudaStreamWaitEvent(s, ev_copied_, 0));
    apply(pending_, s);
    pending_.clear();
  }
  // 2. anything left in window k+1's span goes now, in stream order
  apply(copy_out(ring_.make_room(window_), s), s);
  // 3. the span after it starts moving out in the background
  if (ring_.capacity() >= 2 * window_ + window_ / 2 && !ring_.empty()) {
    ValueRing probe = ring_;
    const std::vector<ValueRing::Live> later = probe.make_room(2 * window_);
    if (!later.empty()) {
      ring_ = probe;  // those values leave the live list now; their HBM copies stay valid until step 1
      MLRG_CUDA(cudaEventRecord(ev_ready_, s));
      MLRG_CUDA(cudaStreamWaitEvent(side_, ev_ready_, 0));
      pending_ = copy_out(later, side_);
      MLRG_CUDA(cudaEventRecord(ev_copied_, side_));
    }
  }
}

}  // namespace mlrg
