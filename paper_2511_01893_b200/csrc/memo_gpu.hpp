// Device-side memo lookup (BASELINE north_star: "a reduction kernel plus
// device-side lookup"): the key index, the 1-slot private caches and the
// staging of inserts live in HBM next to the values, so a memoizable operator
// call runs encode -> lookup -> compute (hit slabs skipped inside the kernels)
// -> materialise / stage without a host round trip. The host sees the
// decisions once per outer iteration, at flush_inserts (admm.cpp:251-254),
// where it replays them into its MemoClient/MemoStore mirror (counters, audit,
// IVF training) and uploads the new IVF lists.
//
// Semantics are the reference's, decision for decision:
//   cache probe   memoclient.cpp:177-211 (slot keyed by (location, op) holding
//                 the QUERY key of its last remote hit; float(cs) > tau and
//                 equal value size)
//   store query   memostore.cpp:174-222 (published keys only; flat scan below
//                 train_size, else IVF: centroids ranked by (l2, index), nprobe
//                 lists; best by (l2 in double, lower id); hit iff float(cs) > tau)
//   staging       memoclient.cpp:302-312 (<= insert_queue_cap per flush window,
//                 in call and slab order; the rest dropped)
// Every double operation uses explicit _rn intrinsics in the reference's
// order (no FMA contraction), so distances and similarities are bit-identical
// to the host's.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include <future>

#include "cold_tier.hpp"
#include "device.hpp"
#include "encoder.hpp"
#include "memo.hpp"

namespace mlrg {

/// Per-slab outcome of one device lookup (written by the lookup/stage kernels).
struct DevSlab {
  int outcome;        // 0 miss, 1 remote hit, 2 cache hit
  float cs;
  long long vid;      // value id for hits
  const float2* src;  // hit: stored value
  double scale;       // hit: live norm / stored norm
  float2* dst;        // accepted miss: arena slot for the value
};

/// One logged decision (drained at flush).
struct DevLog {
  int iteration, op, location, outcome;
  float cs;
  int probed;  // a cache slot existed for (location, op)
  int queried; // went to the store
  int staged;  // 1 accepted, 0 dropped, -1 not a miss
};

/// The IVF k-means (kmeans_train + nearest_centroid, memo.cpp) in one GPU CTA on
/// its own stream of `device`; bit-identical to the host. gpu_kmeans_fits: the
/// per-key state and the centroids fit in shared memory.
struct KmeansScratch;  // device buffers and stream, reused across trainings
void gpu_kmeans(const std::vector<std::vector<float>>& keys, int k, std::uint64_t seed, int iters,
                std::vector<std::vector<float>>& cent, std::vector<std::size_t>& nearest, int device,
                KmeansScratch* scratch = nullptr);
bool gpu_kmeans_fits(int nk, int k, int dim);

class DeviceMemo {
 public:
  /// window_inserts: the most values one flush window can insert (the insert
  /// cap, or fewer when the window has fewer lookups). The HBM arena is a ring
  /// (cold_tier.hpp): it must hold one window plus one slab, older values
  /// spill to pinned host memory at flush.
  DeviceMemo(MemoClient& client, int key_dim, std::uint64_t seed, int max_slabs, std::int64_t max_keys,
             std::size_t arena_bytes, int window_inserts, cudaStream_t s);

  /// Per-slab value size (the reference's, scalerun.cpp:196-199) and complex64
  /// element count of `op`'s slabs, set once per operator.
  void set_slabs(OpId op, const std::vector<std::size_t>& value_bytes, const std::vector<std::int64_t>& out_counts,
                 cudaStream_t s);
  /// Looks up the `n` slabs of one call of `op` (keys: raw encoder output
  /// [n][kd], norms2: sum |x|^2 per slab, both device), entirely on the device:
  /// fills slabs() and skip(). No host synchronisation.
  void lookup(OpId op, int n, const float* keys, const double* norms2, int iteration, cudaStream_t s);
  const DevSlab* slabs() const { return slabs_.get(); }
  const unsigned char* skip() const { return skip_.get(); }

  /// Publishes the staged inserts (flush_inserts): replays the logged
  /// decisions into the host client (counters), appends the audit entries,
  /// inserts the staged keys into the host store mirror, re-uploads the IVF
  /// state. Synchronises `s`.
  struct Audit {
    int iteration, op, location, outcome;
    float cs;
  };
  /// publish = false only drains the log (an aborted iteration: the reference
  /// records its decisions but never flushes its inserts).
  void flush(cudaStream_t s, std::vector<Audit>* audit, bool publish = true);
  /// Marks the point of `s` after which no memoized call runs before the next
  /// flush (the objective's unmemoized operators): that flush then reads the
  /// decision log back on its own stream ordered after the mark, so the host's
  /// drain overlaps the work enqueued on `s` after it.
  void mark(cudaStream_t s);
  /// Values spilled to the cold tier so far (count, bytes).
  std::int64_t spilled() const { return spiller_ ? spiller_->spilled() : 0; }
  std::size_t spilled_bytes() const { return spiller_ ? spiller_->spilled_bytes() : 0; }
  std::size_t arena_bytes() const { return arena_bytes_; }

 ~DeviceMemo();

 private:
  void upload_ivf(cudaStream_t s);
  void spill(cudaStream_t s);
  /// Completes a flush whose store update runs on a host thread (the flush
  /// that trains the IVF index: k-means over train_size keys takes ~10 ms of
  /// host time, overlapped with the objective and the next iteration's first
  /// encode); called before anything reads the store or the device IVF state.
  void join(cudaStream_t s);

  cudaStream_t rb_ = nullptr;  // flush readback stream (after a mark)
  cudaEvent_t fp_ = nullptr, rb_done_ = nullptr;
  bool marked_ = false;
  MemoClient& client_;
  int kd_;
  int max_slabs_;
  std::int64_t max_keys_;
  std::size_t arena_bytes_;
  int batch_keys_;  // keys per coalesced store batch (memoclient.cpp:228-246)
  // key index in HBM
  DeviceBuffer<float> keys_;            // [max_keys][kd]
  DeviceBuffer<long long> vbytes_;      // per id
  DeviceBuffer<double> vnorm_;          // per id
  DeviceBuffer<const float2*> vptr_;    // per id
  DeviceBuffer<float> cache_key_;       // [4 ops][max_slabs][kd]
  DeviceBuffer<long long> cache_vid_;   // [4][max_slabs], -1 = empty
  DeviceBuffer<int> mix_perm_;          // [4][max_slabs][kd]
  DeviceBuffer<float> mix_sign_;        // [4][max_slabs][kd]
  DeviceBuffer<float> centroids_;       // [nlist][kd]
  DeviceBuffer<int> cl_ptr_, cl_ids_;   // IVF lists (CSR over ids)
  DeviceBuffer<char> arena_;
  // state: [0] published keys, [1] staged this window, [2] arena offset (bytes),
  // [3] log entries, [4] overflow flag, [5] dropped this window
  DeviceBuffer<long long> state_;
  DeviceBuffer<DevSlab> slabs_;
  DeviceBuffer<unsigned char> skip_;
  DeviceBuffer<long long> slab_vbytes_, slab_counts_;  // [4 ops][max_slabs]
  DeviceBuffer<int> flags_;                            // probed / queried per slab
  DeviceBuffer<float> qkeys_;           // mixed query keys of the current call
  DeviceBuffer<DevLog> log_;
  std::int64_t log_cap_;
  int ncent_ = 0;
  bool trained_ = false;
  PinnedBuffer<long long> h_state_;
  int window_inserts_;
  std::size_t max_slab_bytes_ = 0;  // largest value slab (256-byte granules)
  std::unique_ptr<ColdSpiller> spiller_;  // created with the first slab table
  std::future<void> pending_;             // asynchronous store update (join())
  std::unique_ptr<KmeansScratch> km_;     // the GPU IVF trainer's buffers
  bool pending_spill_ = false;
};

}  // namespace mlrg
