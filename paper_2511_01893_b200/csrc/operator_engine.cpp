#include "engine_api.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "cnn.hpp"
#include "kernels.hpp"

namespace mlrg {

int chunk_axis_of(OpId op) {
  switch (op) {
    case OpId::fu1d:
    case OpId::fu1d_adj: return 0;
    case OpId::fu2d:
    case OpId::fu2d_adj: return 1;
    case OpId::f2d:
    case OpId::f2d_adj: return 0;
  }
  throw std::invalid_argument("chunk_axis_of: unknown operator");
}

namespace {
std::vector<std::int64_t> slab_extents(std::int64_t axis_len, std::int64_t extent) {
  std::vector<std::int64_t> out;
  for (std::int64_t at = 0; at < axis_len; at += extent) out.push_back(std::min(extent, axis_len - at));
  return out;
}
Shape3 with_axis(Shape3 s, int axis, std::int64_t e) {
  (axis == 0 ? s.d0 : axis == 1 ? s.d1 : s.d2) = e;
  return s;
}
}  // namespace

Engine::Engine(const Geometry& g, EngineConfig cfg, cudaStream_t s, std::shared_ptr<Encoder> enc,
               std::shared_ptr<MemoClient> memo, std::shared_ptr<HostComm> comm)
    : g_(g),
      cfg_(cfg),
      s_(s),
      shard_(Shard::make(g, cfg.chunk_extent, std::move(comm))),
      usfft_(g, s, cfg.kernel),
      enc_(std::move(enc)),
      memo_(std::move(memo)) {
  if (cfg_.workers <= 0) throw std::invalid_argument("OperatorEngine: workers must be positive");
  if (cfg_.chunk_extent <= 0) throw std::invalid_argument("OperatorEngine: chunk_extent must be positive");
  if (cfg_.memo_enabled && (!enc_ || !memo_))
    throw std::invalid_argument("OperatorEngine: memoization needs an encoder and a client");
  if (cfg_.memo_enabled) register_shapes();
  if (shard_.sharded()) {
    try {
      pev_ = std::make_unique<PeerEvents>(*shard_.comm);
    } catch (const std::exception&) {
      pev_.reset();  // no interprocess events: host fences (same semantics)
    }
  }
  if (cfg_.memo_enabled && cfg_.device_memo && !shard_.sharded()) {
    // the device-side lookup needs one memo slab per 16-row fu2d batch
    if (cfg_.chunk_extent != Usfft::kRowBatch) throw std::invalid_argument("device memo needs chunk_extent = 16");
    const std::int64_t e = cfg_.chunk_extent;
    const int max_slabs = static_cast<int>(std::max((g_.n1 + e - 1) / e, (g_.h + e - 1) / e));
    dmemo_ = std::make_unique<DeviceMemo>(*memo_, enc_->key_dim(), enc_->seed(), max_slabs,
                                          std::max<std::int64_t>(cfg_.memo_max_keys, 4096), cfg_.memo_arena_bytes,
                                          cfg_.memo_window_inserts, s_);
    for (OpId op : {OpId::fu1d, OpId::fu2d, OpId::fu1d_adj, OpId::fu2d_adj}) {
      const int axis = chunk_axis_of(op);
      const std::vector<std::int64_t> ext = slab_extents(in_shape(op).extent(axis), e);
      std::vector<std::size_t> vb;
      std::vector<std::int64_t> oc;
      for (std::int64_t x : ext) {
        oc.push_back(with_axis(out_shape(op), axis, x).count());
        vb.push_back(8 + static_cast<std::size_t>(oc.back()) * 16);
      }
      dmemo_->set_slabs(op, vb, oc, s_);
    }
  }
  if (shard_.sharded()) {
    HostComm& c = *shard_.comm;
    const std::int64_t np = shard_.np(), nr = shard_.nr();
    mid_.resize(static_cast<std::size_t>(g_.n1 * nr * g_.n2));
    mid2_.resize(static_cast<std::size_t>(np * g_.h * g_.n2));
    stage1_.resize(static_cast<std::size_t>(np * g_.h * g_.n2));
    stage2_.resize(static_cast<std::size_t>(g_.n1 * nr * g_.n2));
    mid_peers_ = std::make_unique<PeerMemory>(c, mid_.get());
    mid2_peers_ = std::make_unique<PeerMemory>(c, mid2_.get());
  }
  if (cfg_.memo_enabled && !dmemo_) {
    // every rank reserves the same capacity (the smallest request), so the
    // replicated per-owner ring offsets agree everywhere
    double cap = static_cast<double>(cfg_.memo_arena_bytes);
    if (shard_.sharded()) {
      std::vector<double> caps(static_cast<std::size_t>(shard_.world));
      shard_.comm->allgather(&cap, sizeof(cap), caps.data());
      cap = *std::min_element(caps.begin(), caps.end());
    }
    arena_cap_ = ValueRing::granule(static_cast<std::size_t>(cap));
    const std::int64_t e = cfg_.chunk_extent;
    const std::int64_t slab = std::max({e * g_.h * g_.n2, e * g_.n0 * g_.n2, g_.n_theta * e * g_.w, g_.n1 * e * g_.n2});
    const std::size_t slab_bytes = ValueRing::granule(static_cast<std::size_t>(slab) * sizeof(float2));
    window_bytes_ = static_cast<std::size_t>(std::max(1, cfg_.memo_window_inserts)) * slab_bytes;
    if (arena_cap_ < window_bytes_ + slab_bytes)  // fail at setup, not mid-solve
      throw std::invalid_argument("memo: value arena of " + std::to_string(arena_cap_) +
                                  " bytes is below one insert window (" + std::to_string(window_bytes_ + slab_bytes) +
                                  " bytes)");
    arena_.resize(arena_cap_);
    if (shard_.sharded()) arena_peers_ = std::make_unique<PeerMemory>(*shard_.comm, arena_.get());
    if (shard_.sharded()) {
      rings_.assign(static_cast<std::size_t>(shard_.world), ValueRing(arena_cap_));
      cold_ = std::make_unique<ColdTier>(shard_.comm->name(), shard_.comm->rank());
    } else {
      spiller_ = std::make_unique<ColdSpiller>(
          arena_.get(), arena_cap_, window_bytes_,
          [this](const std::vector<std::uint64_t>& ids, const std::vector<const void*>& ptrs, cudaStream_t) {
            for (std::size_t i = 0; i < ids.size(); ++i)
              memo_->store().set_value_ptr(ids[i], static_cast<const float2*>(ptrs[i]));
          });
    }
  }
}

Engine::~Engine() = default;

void Engine::allreduce(double* v, int n) const {
  if (shard_.sharded()) shard_.comm->allreduce_sum(v, n);
}

void Engine::host_fence() {
  MLRG_CUDA(cudaStreamSynchronize(s_));
  shard_.comm->barrier();
}

void Engine::fence() {
  if (!shard_.sharded()) return;
  // MLRG_FENCE=sync / =event force either; by default the event fence runs when every
  // rank has its own GPU (PeerEvents::distinct_devices)
  static const int mode = [] {
    const char* e = std::getenv("MLRG_FENCE");
    if (e && std::string(e) == "sync") return 0;
    if (e && std::string(e) == "event") return 1;
    return -1;
  }();
  const bool ev = pev_ && (mode == 1 || (mode == -1 && pev_->distinct_devices()));
  if (!ev) return host_fence();
  pev_->fence(s_);
}

float2* Engine::value_slot(int owner, std::int64_t count) {
  const std::size_t bytes = ValueRing::granule(static_cast<std::size_t>(count) * sizeof(float2));
  // spill_values() freed one window's span at the last flush; a window never inserts more
  ValueRing& ring = spiller_ ? spiller_->ring() : rings_[static_cast<std::size_t>(owner)];
  const std::size_t off = ring.alloc(bytes);
  pending_.push_back(Pending{owner, off, bytes});
  char* base = arena_peers_ ? static_cast<char*>(arena_peers_->at(owner)) : arena_.get();
  return reinterpret_cast<float2*>(base + off);
}

void Engine::spill_values() {
  MemoStore& store = memo_->store();
  // the window's values got ids in staging order at the flush just done
  const std::uint64_t n = store.key_count();
  if (n < pending_.size()) throw std::logic_error("memo: fewer published values than allocated");
  std::uint64_t id = n - pending_.size();
  for (const Pending& p : pending_)
    (spiller_ ? spiller_->ring() : rings_[static_cast<std::size_t>(p.owner)]).note(id++, p.off, p.bytes);
  pending_.clear();
  if (spiller_) {  // one rank: host-side pointers only, the copies are ordered on the engine stream
    spiller_->flush(s_);
    return;
  }
  struct Moved {
    std::uint64_t id;
    ColdRef ref;
  };
  std::vector<Moved> moved;
  const int me = shard_.sharded() ? shard_.comm->rank() : 0;
  for (int r = 0; r < static_cast<int>(rings_.size()); ++r)
    for (const ValueRing::Live& v : rings_[static_cast<std::size_t>(r)].make_room(window_bytes_)) {
      const ColdRef ref = cold_->place(r, v.bytes);
      if (r == me) cold_->copy_in(ref, arena_.get() + v.off, v.bytes, s_);
      moved.push_back(Moved{v.id, ref});
    }
  if (moved.empty()) return;
  prof::HostSpan span("host:memo_spill");
  // the owners' copies (and segments) exist before any rank maps or reads them
  if (shard_.sharded()) host_fence();
  else MLRG_CUDA(cudaStreamSynchronize(s_));
  for (const Moved& m : moved) store.set_value_ptr(m.id, static_cast<const float2*>(cold_->device_ptr(m.ref)));
  spilled_ += static_cast<std::int64_t>(moved.size());
}

std::int64_t Engine::spilled_values() const {
  return dmemo_ ? dmemo_->spilled() : spiller_ ? spiller_->spilled() : spilled_;
}
std::size_t Engine::spilled_bytes() const {
  if (dmemo_) return dmemo_->spilled_bytes();
  if (spiller_) return spiller_->spilled_bytes();
  std::size_t b = 0;
  for (int r = 0; cold_ && r < static_cast<int>(rings_.size()); ++r) b += cold_->bytes_placed(r);
  return b;
}

void Engine::register_shapes() {  // scalerun.cpp:109-124
  const Shape3 vol = g_.volume_shape(), mid = g_.mid_shape(), proj = g_.projection_shape();
  for (std::int64_t e : slab_extents(vol.d0, cfg_.chunk_extent)) {
    enc_->register_shape(with_axis(vol, 0, e), s_);
    enc_->register_shape(with_axis(mid, 0, e), s_);
  }
  for (std::int64_t e : slab_extents(mid.d1, cfg_.chunk_extent)) {
    enc_->register_shape(with_axis(mid, 1, e), s_);
    enc_->register_shape(with_axis(proj, 1, e), s_);
  }
  for (std::int64_t e : slab_extents(proj.d0, cfg_.chunk_extent)) enc_->register_shape(with_axis(proj, 0, e), s_);
}

Shape3 Engine::in_shape(OpId op) const {
  const std::int64_t np = shard_.np(), nr = shard_.nr();
  switch (op) {
    case OpId::fu1d: return {np, g_.n0, g_.n2};
    case OpId::fu1d_adj: return {np, g_.h, g_.n2};
    case OpId::fu2d: return {g_.n1, nr, g_.n2};
    case OpId::fu2d_adj: return {g_.n_theta, nr, g_.w};
    case OpId::f2d:
    case OpId::f2d_adj: return g_.projection_shape();
  }
  throw std::invalid_argument("in_shape: unknown operator");
}

Shape3 Engine::out_shape(OpId op) const {
  const std::int64_t np = shard_.np(), nr = shard_.nr();
  switch (op) {
    case OpId::fu1d: return {np, g_.h, g_.n2};
    case OpId::fu1d_adj: return {np, g_.n0, g_.n2};
    case OpId::fu2d: return {g_.n_theta, nr, g_.w};
    case OpId::fu2d_adj: return {g_.n1, nr, g_.n2};
    case OpId::f2d:
    case OpId::f2d_adj: return g_.projection_shape();
  }
  throw std::invalid_argument("out_shape: unknown operator");
}

std::int64_t Engine::slab0(int axis, OpId op) const {
  if (op == OpId::f2d || op == OpId::f2d_adj) return 0;
  return (axis == 0 ? shard_.a() : shard_.c()) / cfg_.chunk_extent;
}

void Engine::compute(OpId op, bool fused, const void* in, bool in_d, const float2* d_hat, void* out, bool out_d,
                     std::int64_t start, std::int64_t extent) {
  const std::int64_t n0 = g_.n0, n2 = g_.n2, h = g_.h, w = g_.w, nr = shard_.nr();
  if (op != OpId::fu2d_adj) usfft_.forget_class_sums();
  switch (op) {
    case OpId::fu1d:
      if (in_d) usfft_.fu1d(static_cast<const double2*>(in) + start * n0 * n2, static_cast<float2*>(out) + start * h * n2, extent);
      else usfft_.fu1d(static_cast<const float2*>(in) + start * n0 * n2, static_cast<float2*>(out) + start * h * n2, extent);
      return;
    case OpId::fu1d_adj:
      if (out_d) usfft_.fu1d_adj(static_cast<const float2*>(in) + start * h * n2, static_cast<double2*>(out) + start * n0 * n2, extent);
      else usfft_.fu1d_adj(static_cast<const float2*>(in) + start * h * n2, static_cast<float2*>(out) + start * n0 * n2, extent);
      return;
    case OpId::fu2d: {
      Fu2dEpilogue e;
      e.out = static_cast<float2*>(out);
      e.ld_out = nr;
      e.k0_out = start;
      if (fused) {
        e.sub = d_hat;
        e.ld_sub = nr;
        e.k0_sub = start;
        // the whole residual computed in one call: a following fu2d_adj of it
        // reuses the class sums (solver.cpp: r = fu2d(v) - d, then fu2d_adj(r))
        e.class_sums = whole_call_ && start == 0 && extent == nr;
      }
      usfft_.fu2d(static_cast<const float2*>(in), nr, start, extent, e);
      return;
    }
    case OpId::fu2d_adj:
      usfft_.fu2d_adj(static_cast<const float2*>(in), nr, start, extent, static_cast<float2*>(out), nr, start);
      return;
    case OpId::f2d:
    case OpId::f2d_adj:
      usfft_.f2d(static_cast<const float2*>(in) + start * h * w, static_cast<float2*>(out) + start * h * w, extent,
                 op == OpId::f2d_adj);
      return;
  }
}

void Engine::apply(OpId op, bool fused, const void* in, bool in_d, const float2* d_hat, void* out, bool out_d,
                   bool memoize) {
  const int axis = chunk_axis_of(op);
  const Shape3 ishape = in_shape(op), oshape = out_shape(op);
  const std::int64_t len = ishape.extent(axis);
  const bool use_memo = memoize && cfg_.memo_enabled;
  if (!use_memo) {
    whole_call_ = true;
    compute(op, fused, in, in_d, d_hat, out, out_d, 0, len);
    whole_call_ = false;
    return;
  }
  if (shard_.sharded() && (op == OpId::f2d || op == OpId::f2d_adj))
    throw std::invalid_argument("OperatorEngine: f2d is not memoized in sharded mode (pipeline=optimized)");
  if (dmemo_ && op != OpId::f2d && op != OpId::f2d_adj)
    return apply_device_memo(op, fused, in, in_d, d_hat, out, out_d);
  if (dmemo_) throw std::invalid_argument("OperatorEngine: device memo does not memoize f2d (pipeline=optimized)");
  // ---- encode this rank's slabs (one GEMM per distinct slab shape) ----
  const std::vector<std::int64_t> ext = slab_extents(len, cfg_.chunk_extent);
  const int n = static_cast<int>(ext.size());
  const int kd = enc_->key_dim();
  const std::int64_t g0 = slab0(axis, op);  // global location of local slab 0
  keys_host_.reserve(static_cast<std::size_t>(n * kd));
  norms_host_.reserve(static_cast<std::size_t>(n));
  std::vector<std::int64_t> starts(static_cast<std::size_t>(n));
  for (int c = 0; c < n; ++c) starts[static_cast<std::size_t>(c)] = static_cast<std::int64_t>(c) * cfg_.chunk_extent;
  encode_slabs(op, in, in_d, axis, ishape, ext, starts);
  {
    prof::HostSpan span("host:memo_key_sync");
    MLRG_CUDA(cudaMemcpyAsync(keys_host_.get(), enc_keys_.get(), sizeof(float) * n * kd, cudaMemcpyDeviceToHost, s_));
    MLRG_CUDA(cudaMemcpyAsync(norms_host_.get(), enc_norms_.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s_));
    MLRG_CUDA(cudaStreamSynchronize(s_));
  }
  // ---- local keys -> the global key list (slot-mixed with the global location) ----
  std::vector<float> kv(static_cast<std::size_t>(n * kd));
  std::vector<double> nv(static_cast<std::size_t>(n));
  for (int c = 0; c < n; ++c) {
    std::copy(keys_host_.get() + static_cast<std::size_t>(c) * kd, keys_host_.get() + static_cast<std::size_t>(c + 1) * kd,
              kv.begin() + static_cast<std::ptrdiff_t>(c) * kd);
    slot_mix(kv.data() + static_cast<std::size_t>(c) * kd, kd, enc_->seed(), g0 + c, op);
    nv[static_cast<std::size_t>(c)] = std::sqrt(norms_host_.get()[c]);
  }
  const Shape3 gin = op == OpId::fu1d || op == OpId::fu1d_adj ? with_axis(ishape, 0, g_.n1)
                     : op == OpId::fu2d || op == OpId::fu2d_adj ? with_axis(ishape, 1, g_.h)
                                                                : ishape;
  const std::vector<std::int64_t> gext = slab_extents(gin.extent(axis), cfg_.chunk_extent);
  const int N = static_cast<int>(gext.size());
  if (shard_.sharded()) {  // all-gather keys and norms in rank (= slab) order
    std::vector<unsigned char> buf(kv.size() * sizeof(float) + nv.size() * sizeof(double));
    std::memcpy(buf.data(), nv.data(), nv.size() * sizeof(double));
    std::memcpy(buf.data() + nv.size() * sizeof(double), kv.data(), kv.size() * sizeof(float));
    std::vector<std::size_t> counts;
    const std::vector<unsigned char> all = shard_.comm->allgatherv(buf.data(), buf.size(), &counts);
    kv.clear();
    nv.clear();
    std::size_t at = 0;
    for (const std::size_t bytes : counts) {
      const std::size_t m = bytes / (sizeof(double) + sizeof(float) * static_cast<std::size_t>(kd));
      const double* np_ = reinterpret_cast<const double*>(all.data() + at);
      const float* kp = reinterpret_cast<const float*>(all.data() + at + m * sizeof(double));
      nv.insert(nv.end(), np_, np_ + m);
      kv.insert(kv.end(), kp, kp + m * static_cast<std::size_t>(kd));
      at += bytes;
    }
    if (static_cast<int>(nv.size()) != N) throw std::logic_error("sharded memo: global slab count mismatch");
  }
  std::vector<MemoKey> keys(static_cast<std::size_t>(N));
  std::vector<std::size_t> value_bytes(static_cast<std::size_t>(N));
  std::vector<std::int64_t> out_counts(static_cast<std::size_t>(N));
  const Shape3 gout = with_axis(oshape, axis, 1);
  for (int c = 0; c < N; ++c) {
    MemoKey& k = keys[static_cast<std::size_t>(c)];
    k.values.assign(kv.begin() + static_cast<std::ptrdiff_t>(c) * kd, kv.begin() + static_cast<std::ptrdiff_t>(c + 1) * kd);
    k.location = c;
    k.op = op;
    const std::int64_t oc = with_axis(gout, axis, gext[static_cast<std::size_t>(c)]).count();
    out_counts[static_cast<std::size_t>(c)] = oc;
    value_bytes[static_cast<std::size_t>(c)] = 8 + static_cast<std::size_t>(oc) * 16;
  }
  std::vector<MemoDecision> dec;
  {
    prof::HostSpan span("host:memo_lookup");
    dec = memo_->lookup_batch(keys, value_bytes);
  }
  auto local_dec = [&](int c) -> const MemoDecision& { return dec[static_cast<std::size_t>(g0 + c)]; };

  // ---- local misses: computed in contiguous runs (linear fu2d for fused, d_hat after staging) ----
  for (int c0 = 0; c0 < n;) {
    if (local_dec(c0).outcome != MemoOutcome::miss) {
      ++c0;
      continue;
    }
    int c1 = c0;
    std::int64_t extent = 0;
    while (c1 < n && local_dec(c1).outcome == MemoOutcome::miss) extent += ext[static_cast<std::size_t>(c1++)];
    compute(op, false, in, in_d, nullptr, out, out_d, starts[static_cast<std::size_t>(c0)], extent);
    c0 = c1;
  }
  // ---- local hits: value * (live norm / stored norm), minus the live d_hat slab when fused (one launch) ----
  const ops::SlabGeom og{oshape.d0, oshape.d1, oshape.d2, axis, 0, 0};
  auto batch = std::make_unique<ops::SlabBatch>();
  int nb = 0;
  auto flush_hits = [&]() {
    if (out_d) ops::slab_materialize(static_cast<double2*>(out), og, *batch, nb, s_);
    else ops::slab_materialize(static_cast<float2*>(out), og, *batch, nb, fused ? d_hat : nullptr, s_);
    nb = 0;
  };
  for (int c = 0; c < n; ++c) {
    const MemoDecision& d = local_dec(c);
    if (d.outcome == MemoOutcome::miss) continue;
    const ValueRef& v = memo_->store().value(d.value_id);
    const double live = nv[static_cast<std::size_t>(g0 + c)];
    batch->start[nb] = starts[static_cast<std::size_t>(c)];
    batch->extent[nb] = ext[static_cast<std::size_t>(c)];
    batch->value[nb] = v.dev;  // this rank's arena or a peer's (IPC mapping)
    batch->scale[nb] = (v.norm > 0.0 && live > 0.0) ? live / v.norm : 1.0;
    if (++nb == ops::kSlabBatch) flush_hits();
  }
  flush_hits();
  for (int c = 0; c < N; ++c) {
    const MemoDecision& d = dec[static_cast<std::size_t>(c)];
    audit_.push_back(ChunkAudit{op, axis, c, gext[static_cast<std::size_t>(c)], d.outcome, d.cs, iteration_, -1.0f});
  }
  // ---- stage the miss values in global order (the linear part for fused); the
  // owner copies its slabs, then applies d_hat (one launch) ----
  auto flush_stores = [&]() {
    if (out_d) ops::slab_store(static_cast<double2*>(out), og, *batch, nb, s_);
    else ops::slab_store(static_cast<float2*>(out), og, *batch, nb, fused ? d_hat : nullptr, s_);
    nb = 0;
  };
  for (int c = 0; c < N; ++c) {
    if (dec[static_cast<std::size_t>(c)].outcome != MemoOutcome::miss) continue;
    const bool mine = c >= g0 && c < g0 + n;
    const int owner = !shard_.sharded() ? 0
                      : axis == 0       ? shard_.owner_of_plane(c * cfg_.chunk_extent)
                                        : shard_.owner_of_row(c * cfg_.chunk_extent);
    float2* dst = nullptr;
    memo_->insert_async(keys[static_cast<std::size_t>(c)], [&]() {
      prof::HostSpan span("host:memo_alloc");
      ValueRef v;
      v.count = out_counts[static_cast<std::size_t>(c)];
      float2* slot = value_slot(owner, v.count);
      if (mine) dst = slot;
      v.dev = slot;
      v.norm = nv[static_cast<std::size_t>(c)];
      v.bytes = value_bytes[static_cast<std::size_t>(c)];
      return v;
    });
    if (!mine || (!dst && !fused)) continue;  // another rank's slab, or a dropped insert
    batch->start[nb] = starts[static_cast<std::size_t>(c - g0)];
    batch->extent[nb] = ext[static_cast<std::size_t>(c - g0)];
    batch->dst[nb] = dst;
    if (++nb == ops::kSlabBatch) flush_stores();
  }
  flush_stores();
  if (cfg_.flush_after_apply) flush_inserts();
}

void Engine::encode_slabs(OpId /*op*/, const void* in, bool in_d, int axis, const Shape3& ishape,
                          const std::vector<std::int64_t>& ext, const std::vector<std::int64_t>& starts) {
  const int n = static_cast<int>(ext.size());
  const int kd = enc_->key_dim();
  enc_keys_.resize(static_cast<std::size_t>(n * kd));
  enc_norms_.resize(static_cast<std::size_t>(n));
  if (enc_->cnn()) {  // encoder_variant = cnn (cnn.cu), per run of equal slab extents
    for (int c0 = 0; c0 < n;) {
      int c1 = c0;
      while (c1 < n && ext[static_cast<std::size_t>(c1)] == ext[static_cast<std::size_t>(c0)]) ++c1;
      const ops::SlabGeom sg{ishape.d0, ishape.d1, ishape.d2, axis, 0, ext[static_cast<std::size_t>(c0)]};
      float* kdst = enc_keys_.get() + static_cast<std::size_t>(c0) * kd;
      if (in_d)
        ops::encode_cnn(static_cast<const double2*>(in), sg, starts.data() + c0, c1 - c0, enc_->cnn_device(), kdst,
                        enc_norms_.get() + c0, cnn_work_, s_);
      else
        ops::encode_cnn(static_cast<const float2*>(in), sg, starts.data() + c0, c1 - c0, enc_->cnn_device(), kdst,
                        enc_norms_.get() + c0, cnn_work_, s_);
      c0 = c1;
    }
    return;
  }
  for (int c0 = 0; c0 < n;) {  // one GEMM per distinct slab shape
    int c1 = c0;
    while (c1 < n && ext[static_cast<std::size_t>(c1)] == ext[static_cast<std::size_t>(c0)]) ++c1;
    ops::SlabGeom sg{ishape.d0, ishape.d1, ishape.d2, axis, 0, ext[static_cast<std::size_t>(c0)]};
    enc_work_.resize(ops::encode_work_doubles(c1 - c0, kd));
    const float* P = enc_->device_matrix(with_axis(ishape, axis, sg.extent));
    float* kdst = enc_keys_.get() + static_cast<std::size_t>(c0) * kd;
    if (in_d)
      ops::encode(static_cast<const double2*>(in), sg, starts.data() + c0, c1 - c0, P, kd, enc_work_.get(), kdst,
                  enc_norms_.get() + c0, s_);
    else
      ops::encode(static_cast<const float2*>(in), sg, starts.data() + c0, c1 - c0, P, kd, enc_work_.get(), kdst,
                  enc_norms_.get() + c0, s_);
    c0 = c1;
  }
}

void Engine::apply_device_memo(OpId op, bool fused, const void* in, bool in_d, const float2* d_hat, void* out,
                               bool out_d) {
  const int axis = chunk_axis_of(op);
  const Shape3 ishape = in_shape(op), oshape = out_shape(op);
  const std::int64_t len = ishape.extent(axis), e = cfg_.chunk_extent;
  const std::vector<std::int64_t> ext = slab_extents(len, e);
  const int n = static_cast<int>(ext.size());
  std::vector<std::int64_t> starts(static_cast<std::size_t>(n));
  for (int c = 0; c < n; ++c) starts[static_cast<std::size_t>(c)] = static_cast<std::int64_t>(c) * e;
  // encode -> lookup -> compute (hit slabs skip their CTAs) -> hits -> miss values, all enqueued
  encode_slabs(op, in, in_d, axis, ishape, ext, starts);
  dmemo_->lookup(op, n, enc_keys_.get(), enc_norms_.get(), iteration_, s_);
  usfft_.set_skip(dmemo_->skip());
  try {
    compute(op, false, in, in_d, nullptr, out, out_d, 0, len);
  } catch (...) {
    usfft_.set_skip(nullptr);
    throw;
  }
  usfft_.set_skip(nullptr);
  const ops::SlabGeom og{oshape.d0, oshape.d1, oshape.d2, axis, 0, 0};
  if (out_d) ops::dev_finish(static_cast<double2*>(out), og, dmemo_->slabs(), n, e, s_);
  else ops::dev_finish(static_cast<float2*>(out), og, dmemo_->slabs(), n, e, fused ? d_hat : nullptr, s_);
  if (cfg_.flush_after_apply) flush_inserts();
}

void Engine::take_device_audit(bool publish) {
  std::vector<DeviceMemo::Audit> a;
  dmemo_->flush(s_, &a, publish);
  for (const DeviceMemo::Audit& x : a) {
    const OpId op = static_cast<OpId>(x.op);
    const int axis = chunk_axis_of(op);
    const std::int64_t len = in_shape(op).extent(axis), e = cfg_.chunk_extent;
    audit_.push_back(ChunkAudit{op, axis, x.location, std::min(e, len - x.location * e),
                                static_cast<MemoOutcome>(x.outcome), x.cs, x.iteration, -1.0f});
  }
}

void Engine::drain_memo_log() {
  if (dmemo_) take_device_audit(false);
}

void Engine::flush_inserts() {
  prof::HostSpan span("host:memo_flush");
  if (!memo_) return;
  // sharded: a value is read by its first hit only after this flush; the owner's
  // copy must be complete on its stream before any rank publishes the key
  if (shard_.sharded()) host_fence();
  if (dmemo_) return take_device_audit(true);
  memo_->flush_inserts();
  spill_values();
}

void Engine::fu1d(const double2* u, float2* out, bool memoize) {
  if (!shard_.sharded()) return apply(OpId::fu1d, false, u, true, nullptr, out, false, memoize);
  if (out != mid_.get()) throw std::invalid_argument("sharded fu1d: output must be the engine's mid()");
  exchange_fence();  // every rank is done reading its mid block
  if (!(memoize && cfg_.memo_enabled) && shard_.world <= PeerOut::kMax) {
    // fused: k_fu1d stores each detector row straight into its owner's mid block
    PeerOut po;
    po.world = shard_.world;
    po.off = shard_.a();
    for (int r = 0; r < shard_.world; ++r) {
      po.lo[r] = shard_.rows[static_cast<std::size_t>(r)].first;
      po.hi[r] = shard_.rows[static_cast<std::size_t>(r)].second;
      po.dst[r] = static_cast<float2*>(mid_peers_->at(r));
    }
    usfft_.fu1d(u, nullptr, shard_.np(), &po);
    exchange_fence();
    return;
  }
  apply(OpId::fu1d, false, u, true, nullptr, stage1_.get(), false, memoize);
  ops::RankTable t;
  t.world = shard_.world;
  for (int r = 0; r < shard_.world; ++r) {
    t.lo[r] = shard_.rows[static_cast<std::size_t>(r)].first;
    t.hi[r] = shard_.rows[static_cast<std::size_t>(r)].second;
    t.dst[r] = static_cast<float2*>(mid_peers_->at(r));
  }
  ops::scatter_planes_to_rows(stage1_.get(), shard_.np(), shard_.a(), g_.n1, g_.h, g_.n2, t, s_);
  exchange_fence();  // every rank's mid block is complete
}
void Engine::fu1d(const float2* u, float2* out, bool memoize) {
  if (shard_.sharded()) throw std::invalid_argument("sharded fu1d takes the complex128 iterate");
  apply(OpId::fu1d, false, u, false, nullptr, out, false, memoize);
}
void Engine::fu1d_adj(const float2* v, double2* out, bool memoize) {
  apply(OpId::fu1d_adj, false, v, false, nullptr, out, true, memoize);
}
void Engine::fu1d_adj(const float2* v, float2* out, bool memoize) {
  apply(OpId::fu1d_adj, false, v, false, nullptr, out, false, memoize);
}
void Engine::fu2d(const float2* v, float2* out, bool memoize) {
  apply(OpId::fu2d, false, v, false, nullptr, out, false, memoize);
}
void Engine::fu2d_fused(const float2* v, const float2* d_hat, float2* out, bool memoize) {
  apply(OpId::fu2d, true, v, false, d_hat, out, false, memoize);
}
void Engine::fu2d_adj(const float2* p, float2* out, bool memoize) {
  if (!shard_.sharded()) return apply(OpId::fu2d_adj, false, p, false, nullptr, out, false, memoize);
  if (out != mid2_.get()) throw std::invalid_argument("sharded fu2d_adj: output must be the engine's mid2()");
  exchange_fence();
  if (!(memoize && cfg_.memo_enabled) && shard_.world <= PeerOut::kMax) {
    // fused: the row pass stores each plane straight into its owner's mid2 block
    PeerOut po;
    po.world = shard_.world;
    po.off = shard_.c();
    po.h = g_.h;
    for (int r = 0; r < shard_.world; ++r) {
      po.lo[r] = shard_.planes[static_cast<std::size_t>(r)].first;
      po.hi[r] = shard_.planes[static_cast<std::size_t>(r)].second;
      po.dst[r] = static_cast<float2*>(mid2_peers_->at(r));
    }
    usfft_.fu2d_adj(p, shard_.nr(), 0, shard_.nr(), nullptr, 0, 0, &po);
    exchange_fence();
    return;
  }
  apply(OpId::fu2d_adj, false, p, false, nullptr, stage2_.get(), false, memoize);
  ops::RankTable t;
  t.world = shard_.world;
  for (int r = 0; r < shard_.world; ++r) {
    t.lo[r] = shard_.planes[static_cast<std::size_t>(r)].first;
    t.hi[r] = shard_.planes[static_cast<std::size_t>(r)].second;
    t.dst[r] = static_cast<float2*>(mid2_peers_->at(r));
  }
  ops::scatter_rows_to_planes(stage2_.get(), shard_.nr(), shard_.c(), g_.n1, g_.h, g_.n2, t, s_);
  exchange_fence();
}
void Engine::f2d(const float2* p, float2* out, bool memoize) {
  apply(OpId::f2d, false, p, false, nullptr, out, false, memoize);
}
void Engine::f2d_adj(const float2* p, float2* out, bool memoize) {
  apply(OpId::f2d_adj, false, p, false, nullptr, out, false, memoize);
}

int Engine::fu2d_reduce_begin(const float2* v, const float2* sub, const float2* dot) {
  const std::int64_t nr = shard_.nr();
  Fu2dEpilogue e;
  e.sub = sub;
  e.ld_sub = nr;
  e.dot = dot;
  e.ld_dot = nr;
  e.reduce = true;
  return usfft_.fu2d(v, nr, 0, nr, e);
}

std::array<double, 2> Engine::fu2d_reduce_end(int slots, const std::vector<Partials::Range>& extra,
                                              std::vector<std::vector<double>>* extra_out) {
  std::vector<Partials::Range> ranges{{0, slots, 2}};
  ranges.insert(ranges.end(), extra.begin(), extra.end());
  std::vector<std::vector<double>> all = usfft_.partials().sum(ranges, s_);
  for (auto& x : all) allreduce(x.data(), static_cast<int>(x.size()));
  if (extra_out) extra_out->assign(all.begin() + 1, all.end());
  return {all[0][0], all[0][1]};
}

std::array<double, 2> Engine::fu2d_reduce(const float2* v, const float2* sub, const float2* dot,
                                          const std::vector<Partials::Range>& extra,
                                          std::vector<std::vector<double>>* extra_out) {
  return fu2d_reduce_end(fu2d_reduce_begin(v, sub, dot), extra, extra_out);
}

void Engine::mark_flush_point() {
  if (dmemo_) dmemo_->mark(s_);
}

}  // namespace mlrg
