// z-slab sharding of the solver across the GPUs of one node.
//
// Volume-side arrays (u, G, p, psi, lambda, g; (n1, n0, n2)) are split along
// axis 0 and detector-side arrays (r_hat, d_hat; (n_theta, h, w)) along axis 1
// (h), both in whole 16-slabs with the reference's assign() partition
// (scalerun.cpp:14-27), so every memo slab lives on exactly one rank and its
// key is computed there. fu1d produces the mid array (n1, h, n2) plane-sharded;
// fu2d consumes it row-sharded: the exchange between them is an all-to-all
// done by this library's scatter kernel with direct stores into the peers'
// HBM through CUDA IPC mappings (P2P over NVLink/NVSwitch), and fu2d_adj ->
// fu1d_adj is the reverse exchange. The stencils (grad/div, TV) read one
// neighbour plane per side from a halo inbox the neighbour writes into.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "comm.hpp"
#include "geometry.hpp"

namespace mlrg {

struct Shard {
  int rank = 0, world = 1;
  std::shared_ptr<HostComm> comm;
  std::int64_t chunk = 16;
  std::vector<std::pair<std::int64_t, std::int64_t>> planes;  // per rank [a, b) along volume axis 0
  std::vector<std::pair<std::int64_t, std::int64_t>> rows;    // per rank [c, d) along detector axis 1 (h)

  bool sharded() const { return world > 1; }
  std::int64_t a() const { return planes[static_cast<std::size_t>(rank)].first; }
  std::int64_t b() const { return planes[static_cast<std::size_t>(rank)].second; }
  std::int64_t c() const { return rows[static_cast<std::size_t>(rank)].first; }
  std::int64_t d() const { return rows[static_cast<std::size_t>(rank)].second; }
  std::int64_t np() const { return b() - a(); }
  std::int64_t nr() const { return d() - c(); }

  /// The single-process shard (everything local).
  static Shard whole(const Geometry& g, std::int64_t chunk);
  /// Rank `comm->rank()` of `comm->world()`: assign() over the 16-slabs of
  /// each axis; every rank must own at least one slab of each.
  static Shard make(const Geometry& g, std::int64_t chunk, std::shared_ptr<HostComm> comm);
  int owner_of_plane(std::int64_t i) const;
  int owner_of_row(std::int64_t k) const;
};

/// A device allocation of this rank plus the same-role allocation of every
/// peer, mapped through CUDA IPC (collective: every rank constructs it in the
/// same order). at(rank) is the local pointer.
class PeerMemory {
 public:
  PeerMemory(HostComm& comm, void* local);
  ~PeerMemory();
  PeerMemory(const PeerMemory&) = delete;
  PeerMemory& operator=(const PeerMemory&) = delete;
  void* at(int r) const { return ptrs_[static_cast<std::size_t>(r)]; }
  const std::vector<void*>& all() const { return ptrs_; }

 private:
  int rank_;
  std::vector<void*> ptrs_;
};

/// Stream-ordered cross-rank fence: every rank records its interprocess event
/// on its stream, the host barrier only orders the records (no stream
/// synchronisation), then every rank's stream waits on all peers' events. All
/// work enqueued before the fence on any rank happens before all work enqueued
/// after it on every rank (the P2P stores of the producing kernels are visible,
/// and no rank overwrites a buffer a peer is still reading).
class PeerEvents {
 public:
  explicit PeerEvents(HostComm& comm);
  ~PeerEvents();
  PeerEvents(const PeerEvents&) = delete;
  PeerEvents& operator=(const PeerEvents&) = delete;
  void fence(cudaStream_t s);
  /// Every rank drives its own GPU (device UUIDs all distinct). Ranks sharing a
  /// device time-slice: a stream waiting on another process's event then waits
  /// for a context switch (measured 2x slower than a host fence at 256^3, two
  /// ranks on one B200), so the engine uses the event fence only here.
  bool distinct_devices() const { return distinct_; }

 private:
  HostComm& comm_;
  bool distinct_ = true;
  cudaEvent_t mine_ = nullptr;
  std::vector<cudaEvent_t> peers_;
};

namespace ops {

constexpr int kMaxRanks = 64;
struct RankTable {
  int world = 1;
  std::int64_t lo[kMaxRanks], hi[kMaxRanks];  // owned range of the destination axis per rank
  float2* dst[kMaxRanks];                     // each rank's destination array (peer mappings)
};

/// src (np, h, n2) = planes [a, a+np) of the mid array, all detector rows ->
/// dst_s (n1, rows_s, n2) of every rank s (rows_s = hi_s - lo_s).
void scatter_planes_to_rows(const float2* src, std::int64_t np, std::int64_t a, std::int64_t n1, std::int64_t h,
                            std::int64_t n2, const RankTable& t, cudaStream_t s);
/// src (n1, nr, n2) = rows [c, c+nr) of the mid array, all planes ->
/// dst_s (planes_s, h, n2) of every rank s.
void scatter_rows_to_planes(const float2* src, std::int64_t nr, std::int64_t c, std::int64_t n1, std::int64_t h,
                            std::int64_t n2, const RankTable& t, cudaStream_t s);

}  // namespace ops
}  // namespace mlrg
