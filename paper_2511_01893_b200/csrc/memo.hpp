// The memoisation database and client, with the reference's exact decision
// semantics. Keys (60 floats) and the index live on
// the host — they are tiny and every decision needs double-precision ranking
// identical to the reference — while the values (operator output slabs, MBs
// each) live in HBM (the engine's ring arena; cold values in mapped pinned
// host memory, cold_tier.hpp) and never round-trip through the host. Replaces:
//   MemoStore   memostore.hpp:12-88, memostore.cpp:17-222
//   MemoClient  memoclient.hpp:21-164, memoclient.cpp:148-350 (local transport)
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <utility>
#include <vector>

#include "device.hpp"
#include "encoder.hpp"

namespace mlrg {

/// A stored operator result: the output slab in HBM (chunk order, complex64),
/// the input norm it was computed from, and the reference's value byte size
/// (8-byte norm header + 16 bytes per complex128 sample, scalerun.cpp:196-199).
struct ValueRef {
  const float2* dev = nullptr;
  std::int64_t count = 0;
  double norm = 0.0;
  std::size_t bytes = 0;
};

struct IvfConfig {  // memostore.hpp:12-20
  int nlist = 64;
  int nprobe = 8;
  int train_size = 1024;
  int kmeans_iters = 20;
  std::uint64_t seed = 7;
};

double cosine_similarity(const float* a, const float* b, int d);
double l2_sq(const float* a, const float* b, int d);
std::vector<std::vector<float>> kmeans_train(const std::vector<std::vector<float>>& keys, int k,
                                             std::uint64_t seed, int iters);

struct QueryOutcome {
  bool found = false, hit = false;
  float cs = 0.0f;
  std::uint64_t id = 0;
};

class MemoStore {
 public:
  /// Trains the IVF index: centroids for `keys` (kmeans_train's exact result)
  /// and each key's nearest final centroid (nearest_centroid's).
  using Trainer = std::function<void(const std::vector<std::vector<float>>& keys, int k, std::uint64_t seed, int iters,
                                     std::vector<std::vector<float>>& centroids, std::vector<std::size_t>& nearest)>;
  explicit MemoStore(IvfConfig cfg = {});
  /// Replaces the host k-means (the device memo trains on the GPU, memo_gpu.cu).
  void set_trainer(Trainer t) { trainer_ = std::move(t); }
  std::uint64_t insert(const std::vector<float>& key, ValueRef value);
  QueryOutcome query(const std::vector<float>& key, float tau, int nprobe = 0) const;
  const ValueRef& value(std::uint64_t id) const { return values_.at(static_cast<std::size_t>(id)); }
  /// A value moved between tiers (cold_tier.hpp): same id, key and bytes.
  void set_value_ptr(std::uint64_t id, const float2* dev) { values_.at(static_cast<std::size_t>(id)).dev = dev; }
  std::uint64_t key_count() const;
  bool trained() const { return trained_; }
  const std::vector<std::vector<float>>& centroids() const { return centroids_; }
  /// Member ids per IVF cluster (insertion order), for the device mirror.
  std::vector<std::vector<std::uint64_t>> cluster_ids() const;
  const IvfConfig& ivf() const { return cfg_; }

 private:
  struct Entry {
    std::vector<float> key;
    std::uint64_t id;
  };
  std::size_t nearest_centroid(const std::vector<float>& key) const;
  void train();

  IvfConfig cfg_;
  Trainer trainer_;
  int key_dim_ = 0;
  bool trained_ = false;
  std::vector<Entry> flat_;
  std::vector<std::vector<float>> centroids_;
  std::vector<std::vector<Entry>> clusters_;
  std::vector<ValueRef> values_;
};

enum class MemoOutcome : std::uint8_t { miss = 0, remote_hit = 1, cache_hit = 2 };

struct MemoDecision {
  MemoOutcome outcome = MemoOutcome::miss;
  float cs = 0.0f;
  std::uint64_t value_id = 0;  // valid for hits
};

struct MemoKey {
  std::vector<float> values;
  std::int64_t location = 0;
  OpId op = OpId::fu1d;
};

struct MemoClientConfig {  // memoclient.hpp:31-39
  float tau = 0.92f;
  int nprobe = 8;
  int timeout_ms = 100;
  std::size_t insert_queue_cap = 256;
  std::size_t coalesce_bytes = 4096;
  bool global_cache = false;
};

struct MemoCounters {  // memoclient.hpp:42-61; miss + remote_hit + cache_hit == lookups
  std::uint64_t lookups = 0, cache_hits = 0, remote_hits = 0, misses = 0;
  std::uint64_t cache_comparisons = 0, cache_probes = 0, timeouts = 0;
  std::uint64_t batches_sent = 0, inserts_enqueued = 0, inserts_sent = 0, inserts_dropped = 0;
};

class MemoClient {
 public:
  MemoClient(MemoClientConfig cfg, std::shared_ptr<MemoStore> store);

  /// memoclient.cpp:220-252 (cache first, then coalesced store queries).
  std::vector<MemoDecision> lookup_batch(const std::vector<MemoKey>& keys,
                                         const std::vector<std::size_t>& value_bytes);
  /// memoclient.cpp:302-312: stages (key, value) unless 256 are already
  /// staged; `make_value` (which copies the slab into the arena) only runs
  /// when the entry is accepted. Returns whether it was staged.
  bool insert_async(const MemoKey& key, const std::function<ValueRef()>& make_value);
  /// memoclient.cpp:314-350: publishes staged inserts in order.
  void flush_inserts();

  const MemoCounters& counters() const { return ctr_; }
  /// The device-side lookup path (memo_gpu.hpp) accounts its decisions here.
  MemoCounters& counters_mut() { return ctr_; }
  const MemoClientConfig& config() const { return cfg_; }
  MemoStore& store() { return *store_; }
  std::size_t cached_slots() const { return cache_.size(); }

 private:
  struct CacheSlot {
    std::vector<float> key;  // the QUERY key of the last remote hit (memoclient.cpp:291)
    std::uint64_t value_id = 0;
  };
  bool cache_probe(const MemoKey& key, std::size_t value_bytes, MemoDecision& out);
  void cache_install(const MemoKey& key, std::uint64_t value_id);
  void send_batch(std::vector<std::size_t>& batch, const std::vector<MemoKey>& keys,
                  const std::vector<std::size_t>& value_bytes, std::vector<MemoDecision>& out);

  MemoClientConfig cfg_;
  std::shared_ptr<MemoStore> store_;
  std::map<std::pair<std::int64_t, std::uint8_t>, CacheSlot> cache_;
  std::vector<std::pair<std::vector<float>, ValueRef>> staged_;
  MemoCounters ctr_;
};

}  // namespace mlrg
