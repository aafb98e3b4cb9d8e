// Two-tier value storage for the memo store (SURVEY.md §7 hard part 6, §8(e)).
//
// The reference's MemoStore is append-only and unbounded (memostore.cpp:112-120):
// every accepted insert stays retrievable for the rest of the solve. At the
// north-star size (configs[3], 1024^3 x 50 iterations on 8 GPUs) that is ~215 GB
// of values per GPU, more than HBM. Here every value is written into a ring
// arena in HBM; before each insert window (one outer iteration between
// flush_inserts calls, memoclient.cpp:302-325) the ring frees the span the
// window can fill by spilling the oldest values that overlap it to pinned host
// memory (the cold tier). A hit on a cold value reads it in place over PCIe
// (the host pages are mapped into the device address space), so the decisions,
// ids and reuse arithmetic are exactly those of an unbounded store; only where
// the bytes live changes.
//
// Sharded runs (one process per GPU): a rank's cold chunks are POSIX
// shared-memory segments registered with CUDA in every process that reads
// them, so a cross-owner hit on a spilled value still resolves to a device
// pointer.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

namespace mlrg {

/// Where a spilled value lives: (owner rank, chunk, byte offset).
struct ColdRef {
  int owner = 0;
  int chunk = -1;
  std::size_t offset = 0;
};

/// Append-only pinned host storage, chunked. `name` empty: process-private
/// (cudaHostAlloc, mapped); otherwise chunk c of rank r is the shared-memory
/// segment "<name>.cold.<r>.<c>", readable by every rank of the job.
class ColdTier {
 public:
  ColdTier(std::string name, int rank, std::size_t chunk_bytes = std::size_t{1} << 30);
  ~ColdTier();
  ColdTier(const ColdTier&) = delete;
  ColdTier& operator=(const ColdTier&) = delete;

  /// Reserves `bytes` for a value of rank `owner` (replicated bookkeeping: every
  /// rank calls this for every spill in the same order and gets the same ref).
  ColdRef place(int owner, std::size_t bytes);
  /// Device-accessible address of a placed value (maps the owner's chunk on first use).
  void* device_ptr(const ColdRef& r);
  /// Enqueues the spill copy of this rank's value (call on the owner only).
  void copy_in(const ColdRef& r, const void* dev_src, std::size_t bytes, cudaStream_t s);
  std::size_t bytes_placed(int owner) const;
  /// Private tier: keep at least `bytes` of pinned chunks allocated ahead of
  /// place(), on a host thread (page pinning costs ~0.1-0.3 s/GB and would
  /// otherwise sit on the flush's critical path).
  void prefetch(std::size_t bytes);

 private:
  struct Chunk {
    void* host = nullptr;
    std::size_t bytes = 0;
    bool shm = false, owned = false;
  };
  struct Cursor {
    int chunks = 0;           // chunks allocated so far
    std::size_t used = 0;     // bytes used in the last chunk
    std::size_t last = 0;     // size of the last chunk
    std::size_t total = 0;
  };
  Chunk& chunk(int owner, int c, std::size_t bytes);
  std::string seg_name(int owner, int c) const;

  std::string name_;
  int rank_;
  std::size_t chunk_bytes_;
  std::map<int, Cursor> cur_;
  std::map<std::pair<int, int>, Chunk> chunks_;
  std::map<std::pair<int, int>, std::size_t> sizes_;  // chunk sizes (replicated)
  // pre-allocated pinned chunks of chunk_bytes_ (private tier)
  std::mutex pool_mu_;
  std::vector<void*> pool_;
  std::thread pool_thread_;
};

/// Bookkeeping of one HBM ring arena (capacity bytes, 256-byte granules).
/// alloc() wraps exactly like k_memo_stage's device allocator: a value that
/// would cross the end starts at offset 0.
class ValueRing {
 public:
  struct Live {
    std::uint64_t id;
    std::size_t off, bytes;
  };
  explicit ValueRing(std::size_t capacity = 0) : cap_(capacity) {}
  void reset(std::size_t capacity) { *this = ValueRing(capacity); }
  std::size_t capacity() const { return cap_; }
  std::size_t head() const { return head_; }
  /// The device allocator's offset after a window (it also advances past
  /// staged values that were never published: an aborted iteration).
  void reset_head(std::size_t head) { head_ = head; }
  static std::size_t granule(std::size_t bytes) { return (bytes + 255) & ~std::size_t{255}; }
  /// Host-side allocation (the host-client and sharded paths).
  std::size_t alloc(std::size_t bytes);
  /// Records a value placed at `off` (the device allocator's choice) and moves
  /// the head past it.
  void note(std::uint64_t id, std::size_t off, std::size_t bytes);
  /// The values that must leave HBM so that the next `window` bytes of
  /// allocations cannot overwrite a live value: everything overlapping
  /// [head, head + window), or [head, cap) and [0, window) when that wraps.
  std::vector<Live> make_room(std::size_t window);
  std::size_t live_bytes() const;
  bool empty() const { return live_.empty(); }

 private:
  std::size_t cap_ = 0, head_ = 0;
  std::deque<Live> live_;  // allocation order
};

/// The spill policy of one process-private ring (the device memo and the
/// host client on one GPU), asynchronous: at the flush that ends window k it
///   1. makes the main stream wait for the copies started at flush k-1 and
///      repoints those values to their cold copies,
///   2. spills (synchronously, on the main stream) whatever still overlaps
///      the span window k+1 can fill,
///   3. starts copying out, on a side stream, the values in the span after
///      it (window k+2's), whose HBM copies stay readable until step 1 of the
///      next flush, so those transfers overlap window k+1's compute.
/// (Pinned cold chunks are allocated when first needed: pinning on a host
/// thread ahead of need stalled the launching thread in the driver.)
class ColdSpiller {
 public:
  /// set_ptr(id, ptr): repoint value `id` (the caller updates its tables, ordered on `s`).
  using SetPtr = std::function<void(const std::vector<std::uint64_t>&, const std::vector<const void*>&, cudaStream_t)>;
  ColdSpiller(char* arena, std::size_t capacity, std::size_t window, SetPtr set_ptr);
  ~ColdSpiller();
  ValueRing& ring() { return ring_; }
  /// At each flush, after the window's values were noted in ring().
  void flush(cudaStream_t s);
  std::int64_t spilled() const { return spilled_; }
  std::size_t spilled_bytes() const { return cold_.bytes_placed(0); }

 private:
  struct Moved {
    std::uint64_t id;
    const void* ptr;
  };
  std::vector<Moved> copy_out(const std::vector<ValueRing::Live>& v, cudaStream_t s);
  void apply(const std::vector<Moved>& m, cudaStream_t s);

  char* arena_;
  std::size_t window_;
  ValueRing ring_;
  ColdTier cold_{"", 0};
  SetPtr set_ptr_;
  cudaStream_t side_ = nullptr;
  cudaEvent_t ev_ready_ = nullptr, ev_copied_ = nullptr;
  std::vector<Moved> pending_;  // copies in flight on side_
  std::int64_t spilled_ = 0;
};

}  // namespace mlrg
