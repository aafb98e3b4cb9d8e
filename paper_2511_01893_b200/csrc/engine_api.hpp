// Device operator engine: the B200 replacement of the reference's
// OperatorEngine (scalerun.hpp:61-116, scalerun.cpp:168-287). Arrays are full
// device arrays; slabs are views (no split/merge copies). With memoisation on,
// every memoizable application encodes all slabs in one device GEMM, makes
// the reference's decisions on the host, computes the misses in as few
// launches as possible (contiguous miss runs batched), materialises hits from
// the HBM value arena and stages the miss values for the next flush.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "encoder.hpp"
#include "geometry.hpp"
#include "memo.hpp"
#include "cnn.hpp"
#include "cold_tier.hpp"
#include "memo_gpu.hpp"
#include "shard.hpp"
#include "usfft.hpp"

namespace mlrg {

struct EngineConfig {  // scalerun.hpp:27-42
  int workers = 1;                  // accepted for drop-in configs; the device path ignores it
  std::int64_t chunk_extent = 16;
  bool memo_enabled = false;
  bool flush_after_apply = false;
  GridKernel kernel = GridKernel::es;  // B200 extension key `gridding_kernel` (geometry.hpp)
  std::size_t memo_arena_bytes = 0;    // HBM reserved for memo values (sharded: per rank)
  bool device_memo = false;            // lookups on the device (memo_gpu.hpp); set by the assembler
  std::int64_t memo_max_keys = 0;      // device key index capacity
  int memo_window_inserts = 256;       // most values one flush window inserts (per rank when sharded)
};

struct ChunkAudit {  // scalerun.hpp:45-54
  OpId op = OpId::fu1d;
  int axis = 0;
  std::int64_t index = 0, extent = 0;
  MemoOutcome outcome = MemoOutcome::miss;
  float cs = 0.0f;
  int iteration = 0;
  float rel_err = -1.0f;
};

/// Partition axis of each operator's input (scalerun.cpp:29-42).
int chunk_axis_of(OpId op);

/// Sharded mode (a HostComm of world > 1): the volume-side arrays the engine
/// reads and writes are this rank's planes [a, b) (Shard), the detector-side
/// arrays its rows [c, d); fu1d writes the engine-owned mid() block (all
/// planes, rows [c, d)) of every rank and fu2d_adj the mid2() block (planes
/// [a, b), all rows). Memo keys are all-gathered so every rank makes the
/// reference's global decisions (SURVEY.md §8(e) "Memo under sharding").
class Engine {
 public:
  Engine(const Geometry& g, EngineConfig cfg, cudaStream_t s, std::shared_ptr<Encoder> enc = nullptr,
         std::shared_ptr<MemoClient> memo = nullptr, std::shared_ptr<HostComm> comm = nullptr);
  ~Engine();

  const Geometry& geometry() const { return g_; }
  const Shard& shard() const { return shard_; }
  Usfft& usfft() { return usfft_; }
  cudaStream_t stream() const { return s_; }
  MemoClient* memo() const { return memo_.get(); }

  void set_iteration(int it) { iteration_ = it; }
  void flush_inserts();
  /// No memoized call runs from here to the next flush_inserts(): the device
  /// memo reads its log back behind this point, overlapping what is enqueued
  /// in between (the objective). No-op without the device memo.
  void mark_flush_point();
  /// Device-side memo: moves the decisions made so far into audit_log() and the
  /// client's counters without publishing the staged inserts (an aborted
  /// iteration). No-op otherwise.
  void drain_memo_log();
  const std::vector<ChunkAudit>& audit_log() const { return audit_; }
  /// Memo values spilled from the HBM ring to the cold tier so far (count, bytes).
  std::int64_t spilled_values() const;
  std::size_t spilled_bytes() const;
  std::size_t memo_arena_bytes() const { return dmemo_ ? dmemo_->arena_bytes() : arena_cap_; }

  /// Sharded mode: the exchange targets (nullptr when unsharded).
  float2* mid() const { return mid_.get(); }
  float2* mid2() const { return mid2_.get(); }
  /// Sums `v` over the ranks in rank order (no-op unsharded).
  void allreduce(double* v, int n) const;
  /// Sharded: stream-ordered fence across the ranks (PeerEvents; MLRG_FENCE=sync
  /// restores the stream synchronisation + host barrier). No-op unsharded.
  void fence();

  // Full-array applications (scalerun.hpp:77-92).
  // The volume side (fu1d input, fu1d_adj output) is the solver's complex128
  // iterate; complex64 overloads serve the C-ABI and the memo benchmark.
  void fu1d(const double2* u, float2* out, bool memoize = true);
  void fu1d(const float2* u, float2* out, bool memoize = true);
  void fu1d_adj(const float2* v, double2* out, bool memoize = true);
  void fu1d_adj(const float2* v, float2* out, bool memoize = true);
  void fu2d(const float2* v, float2* out, bool memoize = true);
  void fu2d_fused(const float2* v, const float2* d_hat, float2* out, bool memoize = true);
  void fu2d_adj(const float2* p, float2* out, bool memoize = true);
  void f2d(const float2* p, float2* out, bool memoize = true);
  void f2d_adj(const float2* p, float2* out, bool memoize = true);

  /// Non-memoized fu2d whose output is only reduced: {sum |fu2d(v) - sub|^2,
  /// Re<dot, fu2d(v) - sub>} (line search terms admm.cpp:95-102 and the data
  /// term of objective(), admm.cpp:190-195); summed over ranks.
  /// `extra`: partial tables of kernels already enqueued (at Partials::kParked
  /// and up) summed with the same readback, into `extra_out` (summed over ranks).
  std::array<double, 2> fu2d_reduce(const float2* v, const float2* sub, const float2* dot,
                                    const std::vector<Partials::Range>& extra = {},
                                    std::vector<std::vector<double>>* extra_out = nullptr);
  /// fu2d_reduce in two halves: enqueue (returns the partial-slot count), then
  /// read back (with `extra`, as fu2d_reduce) after other host work.
  int fu2d_reduce_begin(const float2* v, const float2* sub, const float2* dot);
  std::array<double, 2> fu2d_reduce_end(int slots, const std::vector<Partials::Range>& extra = {},
                                        std::vector<std::vector<double>>* extra_out = nullptr);

 private:
  void apply(OpId op, bool fused, const void* in, bool in_d, const float2* d_hat, void* out, bool out_d,
             bool memoize);
  void apply_device_memo(OpId op, bool fused, const void* in, bool in_d, const float2* d_hat, void* out, bool out_d);
  void encode_slabs(OpId op, const void* in, bool in_d, int axis, const Shape3& ishape,
                    const std::vector<std::int64_t>& ext, const std::vector<std::int64_t>& starts);
  void take_device_audit(bool publish);
  void compute(OpId op, bool fused, const void* in, bool in_d, const float2* d_hat, void* out, bool out_d,
               std::int64_t start, std::int64_t extent);
  Shape3 in_shape(OpId op) const;   // this rank's input array
  Shape3 out_shape(OpId op) const;  // this rank's output array
  std::int64_t slab0(int axis, OpId op) const;  // global index of this rank's first slab
  void register_shapes();
  void exchange_fence() { fence(); }
  void host_fence();  // stream sync + barrier across ranks (the host reads the results)
  float2* value_slot(int owner, std::int64_t count);
  void spill_values();  // host-path rings: free the next window's span (cold_tier.hpp)

  Geometry g_;
  EngineConfig cfg_;
  cudaStream_t s_;
  Shard shard_;
  Usfft usfft_;
  std::shared_ptr<Encoder> enc_;
  std::shared_ptr<MemoClient> memo_;
  int iteration_ = 0;
  std::vector<ChunkAudit> audit_;
  DeviceBuffer<double> enc_work_, enc_norms_;
  DeviceBuffer<float> enc_keys_;
  PinnedBuffer<float> keys_host_;
  PinnedBuffer<double> norms_host_;
  // sharded mode
  DeviceBuffer<float2> mid_, mid2_, stage1_, stage2_;
  std::unique_ptr<PeerMemory> mid_peers_, mid2_peers_;
  // host-path memo values (the host client on one GPU, every sharded run): one
  // HBM ring arena per rank, bookkeeping replicated on every rank, spills to
  // the cold tier at flush
  DeviceBuffer<char> arena_;
  std::unique_ptr<PeerMemory> arena_peers_;
  std::size_t arena_cap_ = 0, window_bytes_ = 0;
  std::vector<ValueRing> rings_;
  struct Pending {
    int owner;
    std::size_t off, bytes;
  };
  std::vector<Pending> pending_;  // values allocated this window, in staging (= id) order
  std::unique_ptr<ColdTier> cold_;        // sharded: shared segments, synchronous spills
  std::unique_ptr<ColdSpiller> spiller_;  // one rank: asynchronous spills
  std::int64_t spilled_ = 0;
  std::unique_ptr<DeviceMemo> dmemo_;
  std::unique_ptr<PeerEvents> pev_;  // sharded: the stream-ordered fence
  ops::CnnWork cnn_work_;  // encoder_variant = cnn scratch
  bool whole_call_ = false;  // compute() runs a whole unmemoized operator call
};

}  // namespace mlrg
