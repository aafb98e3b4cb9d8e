#include "comm.hpp"

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>

namespace mlrg {

std::vector<std::pair<std::int64_t, std::int64_t>> assign_ranges(std::int64_t n_chunks, int n_workers) {
  if (n_workers <= 0) throw std::invalid_argument("assign: n_workers must be positive");
  std::vector<std::pair<std::int64_t, std::int64_t>> out(static_cast<std::size_t>(n_workers));
  const std::int64_t base = n_chunks / n_workers, extra = n_chunks % n_workers;
  std::int64_t at = 0;
  for (int i = 0; i < n_workers; ++i) {
    const std::int64_t len = base + (i < extra ? 1 : 0);
    out[static_cast<std::size_t>(i)] = {at, at + len};
    at += len;
  }
  return out;
}

namespace {
constexpr std::uint64_t kMagic = 0x6d6c72672d636f6dULL;  // "mlrg-com"
constexpr std::size_t kSlot = std::size_t{1} << 20;        // bytes per rank per bank
constexpr int kMaxWorld = 64;

[[noreturn]] void fail(const std::string& what) { throw std::runtime_error("HostComm: " + what); }
}  // namespace

struct alignas(64) HostComm::Header {
  std::atomic<std::uint64_t> magic;
  std::atomic<int> world;
  std::atomic<int> joined;
  std::atomic<int> abort;
  alignas(64) std::atomic<int> count;
  alignas(64) std::atomic<std::uint64_t> gen;
  alignas(64) std::uint64_t sizes[2][kMaxWorld];
};

std::size_t HostComm::slot_bytes() const { return kSlot; }

unsigned char* HostComm::slot(int bank, int r) const {
  return reinterpret_cast<unsigned char*>(hdr_) + sizeof(Header) +
         (static_cast<std::size_t>(bank) * static_cast<std::size_t>(world_) + static_cast<std::size_t>(r)) * kSlot;
}

HostComm::HostComm(const std::string& name, int rank, int world, double timeout_s)
    : name_(name[0] == '/' ? name : "/" + name), rank_(rank), world_(world) {
  static_assert(std::atomic<std::uint64_t>::is_always_lock_free && std::atomic<int>::is_always_lock_free,
                "shared-memory atomics must be lock-free");
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world) fail("bad rank/world");
  size_ = sizeof(Header) + 2 * static_cast<std::size_t>(world) * kSlot;
  const auto t0 = std::chrono::steady_clock::now();
  auto expired = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s;
  };
  if (rank == 0) {
    shm_unlink(name_.c_str());  // a stale segment of a crashed run
    fd_ = shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd_ < 0) fail("shm_open(create " + name_ + "): " + std::strerror(errno));
    if (ftruncate(fd_, static_cast<off_t>(size_)) != 0) fail(std::string("ftruncate: ") + std::strerror(errno));
  } else {
    while ((fd_ = shm_open(name_.c_str(), O_RDWR, 0600)) < 0) {
      if (expired()) fail("timed out waiting for rank 0 to create " + name_);
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
    struct stat st {};
    while (fstat(fd_, &st) == 0 && static_cast<std::size_t>(st.st_size) < size_) {
      if (expired()) fail("segment " + name_ + " has the wrong size (world mismatch?)");
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
  void* p = mmap(nullptr, size_, PROT_READ | PROT_WRITE, MAP_SHARED, fd_, 0);
  if (p == MAP_FAILED) fail(std::string("mmap: ") + std::strerror(errno));
  hdr_ = static_cast<Header*>(p);
  if (rank == 0) {
    hdr_->world.store(world);
    hdr_->joined.store(0);
    hdr_->abort.store(0);
    hdr_->count.store(0);
    hdr_->gen.store(0);
    hdr_->magic.store(kMagic, std::memory_order_release);
  } else {
    while (hdr_->magic.load(std::memory_order_acquire) != kMagic) {
      if (expired()) fail("timed out waiting for rank 0 to initialise " + name_);
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (hdr_->world.load() != world) fail("world size mismatch with rank 0");
  }
  hdr_->joined.fetch_add(1);
  while (hdr_->joined.load() < world) {
    if (expired()) fail("timed out waiting for all ranks to join " + name_);
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

HostComm::~HostComm() {
  if (!hdr_) return;
  try {
    barrier();  // nobody still reads the segment
  } catch (...) {
  }
  munmap(hdr_, size_);
  if (fd_ >= 0) close(fd_);
  if (rank_ == 0) shm_unlink(name_.c_str());
}

void HostComm::abort() {
  if (hdr_) hdr_->abort.store(1);
}

void HostComm::barrier() {
  if (world_ == 1) return;
  if (hdr_->abort.load(std::memory_order_relaxed)) fail("a peer rank failed");
  const std::uint64_t g = hdr_->gen.load(std::memory_order_acquire);
  if (hdr_->count.fetch_add(1, std::memory_order_acq_rel) + 1 == world_) {
    hdr_->count.store(0, std::memory_order_relaxed);
    hdr_->gen.fetch_add(1, std::memory_order_acq_rel);
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (std::uint64_t spin = 0; hdr_->gen.load(std::memory_order_acquire) == g; ++spin) {
    if (hdr_->abort.load(std::memory_order_relaxed)) fail("a peer rank failed");
    if (spin > 256) sched_yield();
    if ((spin & 0xffff) == 0 && spin &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > 600.0) {
      hdr_->abort.store(1);
      fail("barrier timed out after 600 s");
    }
  }
}

void HostComm::allreduce_sum(double* v, int n) {
  if (world_ == 1 || n <= 0) return;
  if (static_cast<std::size_t>(n) * sizeof(double) > kSlot) fail("allreduce payload too large");
  const int bank = static_cast<int>(epoch_++ & 1);
  std::memcpy(slot(bank, rank_), v, static_cast<std::size_t>(n) * sizeof(double));
  barrier();
  for (int i = 0; i < n; ++i) v[i] = 0.0;
  for (int r = 0; r < world_; ++r) {
    const double* s = reinterpret_cast<const double*>(slot(bank, r));
    for (int i = 0; i < n; ++i) v[i] += s[i];
  }
}

void HostComm::allgather(const void* in, std::size_t bytes, void* out) {
  if (bytes > kSlot) fail("allgather payload too large");
  if (world_ == 1) {
    std::memcpy(out, in, bytes);
    return;
  }
  const int bank = static_cast<int>(epoch_++ & 1);
  std::memcpy(slot(bank, rank_), in, bytes);
  barrier();
  for (int r = 0; r < world_; ++r)
    std::memcpy(static_cast<unsigned char*>(out) + static_cast<std::size_t>(r) * bytes, slot(bank, r), bytes);
}

std::vector<unsigned char> HostComm::allgatherv(const void* in, std::size_t bytes, std::vector<std::size_t>* counts) {
  if (bytes > kSlot) fail("allgatherv payload too large");
  std::vector<unsigned char> out;
  if (counts) counts->assign(static_cast<std::size_t>(world_), 0);
  if (world_ == 1) {
    out.assign(static_cast<const unsigned char*>(in), static_cast<const unsigned char*>(in) + bytes);
    if (counts) (*counts)[0] = bytes;
    return out;
  }
  const int bank = static_cast<int>(epoch_++ & 1);
  std::memcpy(slot(bank, rank_), in, bytes);
  hdr_->sizes[bank][rank_] = bytes;
  barrier();
  for (int r = 0; r < world_; ++r) {
    const std::size_t b = hdr_->sizes[bank][r];
    out.insert(out.end(), slot(bank, r), slot(bank, r) + b);
    if (counts) (*counts)[static_cast<std::size_t>(r)] = b;
  }
  return out;
}

}  // namespace mlrg
