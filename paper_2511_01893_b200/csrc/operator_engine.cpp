#include "engine_api.hpp"

#include <algorithm>
#include <cmath>
#include <memory>
#include <stdexcept>

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
               std::shared_ptr<MemoClient> memo)
    : g_(g), cfg_(cfg), s_(s), usfft_(g, s, cfg.kernel), enc_(std::move(enc)), memo_(std::move(memo)) {
  if (cfg_.workers <= 0) throw std::invalid_argument("OperatorEngine: workers must be positive");
  if (cfg_.chunk_extent <= 0) throw std::invalid_argument("OperatorEngine: chunk_extent must be positive");
  if (cfg_.memo_enabled && (!enc_ || !memo_))
    throw std::invalid_argument("OperatorEngine: memoization needs an encoder and a client");
  if (cfg_.memo_enabled) register_shapes();
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
  switch (op) {
    case OpId::fu1d: return g_.volume_shape();
    case OpId::fu1d_adj: return g_.mid_shape();
    case OpId::fu2d: return g_.mid_shape();
    case OpId::fu2d_adj: return g_.projection_shape();
    case OpId::f2d:
    case OpId::f2d_adj: return g_.projection_shape();
  }
  throw std::invalid_argument("in_shape: unknown operator");
}

Shape3 Engine::out_shape(OpId op) const {
  switch (op) {
    case OpId::fu1d: return g_.mid_shape();
    case OpId::fu1d_adj: return g_.volume_shape();
    case OpId::fu2d: return g_.projection_shape();
    case OpId::fu2d_adj: return g_.mid_shape();
    case OpId::f2d:
    case OpId::f2d_adj: return g_.projection_shape();
  }
  throw std::invalid_argument("out_shape: unknown operator");
}

void Engine::compute(OpId op, bool fused, const void* in, bool in_d, const float2* d_hat, void* out, bool out_d,
                     std::int64_t start, std::int64_t extent) {
  const std::int64_t n0 = g_.n0, n2 = g_.n2, h = g_.h, w = g_.w;
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
      e.ld_out = h;
      e.k0_out = start;
      if (fused) {
        e.sub = d_hat;
        e.ld_sub = h;
        e.k0_sub = start;
      }
      usfft_.fu2d(static_cast<const float2*>(in), h, start, extent, e);
      return;
    }
    case OpId::fu2d_adj:
      usfft_.fu2d_adj(static_cast<const float2*>(in), h, start, extent, static_cast<float2*>(out), h, start);
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
    compute(op, fused, in, in_d, d_hat, out, out_d, 0, len);
    return;
  }
  // ---- encode every slab (one GEMM per distinct slab shape) ----
  const std::vector<std::int64_t> ext = slab_extents(len, cfg_.chunk_extent);
  const int n = static_cast<int>(ext.size());
  const int kd = enc_->key_dim();
  enc_keys_.resize(static_cast<std::size_t>(n * kd));
  enc_norms_.resize(static_cast<std::size_t>(n));
  keys_host_.reserve(static_cast<std::size_t>(n * kd));
  norms_host_.reserve(static_cast<std::size_t>(n));
  std::vector<std::int64_t> starts(static_cast<std::size_t>(n));
  for (int c = 0; c < n; ++c) starts[static_cast<std::size_t>(c)] = static_cast<std::int64_t>(c) * cfg_.chunk_extent;
  for (int c0 = 0; c0 < n;) {
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
  {
    prof::HostSpan span("host:memo_key_sync");
    MLRG_CUDA(cudaMemcpyAsync(keys_host_.get(), enc_keys_.get(), sizeof(float) * n * kd, cudaMemcpyDeviceToHost, s_));
    MLRG_CUDA(cudaMemcpyAsync(norms_host_.get(), enc_norms_.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s_));
    MLRG_CUDA(cudaStreamSynchronize(s_));
  }

  std::vector<MemoKey> keys(static_cast<std::size_t>(n));
  std::vector<std::size_t> value_bytes(static_cast<std::size_t>(n));
  std::vector<double> in_norms(static_cast<std::size_t>(n));
  std::vector<std::int64_t> out_counts(static_cast<std::size_t>(n));
  for (int c = 0; c < n; ++c) {
    MemoKey& k = keys[static_cast<std::size_t>(c)];
    k.values.assign(keys_host_.get() + static_cast<std::size_t>(c) * kd,
                    keys_host_.get() + static_cast<std::size_t>(c + 1) * kd);
    k.location = c;
    k.op = op;
    slot_mix(k.values.data(), kd, enc_->seed(), c, op);
    in_norms[static_cast<std::size_t>(c)] = std::sqrt(norms_host_.get()[c]);
    const std::int64_t oc = with_axis(oshape, axis, ext[static_cast<std::size_t>(c)]).count();
    out_counts[static_cast<std::size_t>(c)] = oc;
    value_bytes[static_cast<std::size_t>(c)] = 8 + static_cast<std::size_t>(oc) * 16;
  }
  std::vector<MemoDecision> dec;
  {
    prof::HostSpan span("host:memo_lookup");
    dec = memo_->lookup_batch(keys, value_bytes);
  }

  // ---- misses: computed in contiguous runs (linear fu2d for fused, d_hat after staging) ----
  for (int c0 = 0; c0 < n;) {
    if (dec[static_cast<std::size_t>(c0)].outcome != MemoOutcome::miss) {
      ++c0;
      continue;
    }
    int c1 = c0;
    std::int64_t extent = 0;
    while (c1 < n && dec[static_cast<std::size_t>(c1)].outcome == MemoOutcome::miss)
      extent += ext[static_cast<std::size_t>(c1++)];
    compute(op, false, in, in_d, nullptr, out, out_d, starts[static_cast<std::size_t>(c0)], extent);
    c0 = c1;
  }
  // ---- hits: value * (live norm / stored norm), minus the live d_hat slab when fused (one launch) ----
  const ops::SlabGeom og{oshape.d0, oshape.d1, oshape.d2, axis, 0, 0};
  auto batch = std::make_unique<ops::SlabBatch>();
  int nb = 0;
  auto flush_hits = [&]() {
    if (out_d) ops::slab_materialize(static_cast<double2*>(out), og, *batch, nb, s_);
    else ops::slab_materialize(static_cast<float2*>(out), og, *batch, nb, fused ? d_hat : nullptr, s_);
    nb = 0;
  };
  for (int c = 0; c < n; ++c) {
    const MemoDecision& d = dec[static_cast<std::size_t>(c)];
    if (d.outcome != MemoOutcome::miss) {
      const ValueRef& v = memo_->store().value(d.value_id);
      const double live = in_norms[static_cast<std::size_t>(c)];
      batch->start[nb] = starts[static_cast<std::size_t>(c)];
      batch->extent[nb] = ext[static_cast<std::size_t>(c)];
      batch->value[nb] = v.dev;
      batch->scale[nb] = (v.norm > 0.0 && live > 0.0) ? live / v.norm : 1.0;
      if (++nb == ops::kSlabBatch) flush_hits();
    }
    audit_.push_back(ChunkAudit{op, axis, c, ext[static_cast<std::size_t>(c)], d.outcome, d.cs, iteration_, -1.0f});
  }
  flush_hits();
  // ---- stage the miss values (the linear part for fused), then apply d_hat (one launch) ----
  auto flush_stores = [&]() {
    if (out_d) ops::slab_store(static_cast<double2*>(out), og, *batch, nb, s_);
    else ops::slab_store(static_cast<float2*>(out), og, *batch, nb, fused ? d_hat : nullptr, s_);
    nb = 0;
  };
  for (int c = 0; c < n; ++c) {
    if (dec[static_cast<std::size_t>(c)].outcome != MemoOutcome::miss) continue;
    float2* dst = nullptr;
    memo_->insert_async(keys[static_cast<std::size_t>(c)], [&]() {
      ValueRef v;
      v.count = out_counts[static_cast<std::size_t>(c)];
      prof::HostSpan span("host:memo_alloc");
      dst = memo_->store().arena().alloc(v.count);
      v.dev = dst;
      v.norm = in_norms[static_cast<std::size_t>(c)];
      v.bytes = value_bytes[static_cast<std::size_t>(c)];
      return v;
    });
    if (!dst && !fused) continue;  // dropped insert, nothing to do for this slab
    batch->start[nb] = starts[static_cast<std::size_t>(c)];
    batch->extent[nb] = ext[static_cast<std::size_t>(c)];
    batch->dst[nb] = dst;
    if (++nb == ops::kSlabBatch) flush_stores();
  }
  flush_stores();
  if (cfg_.flush_after_apply) memo_->flush_inserts();
}

void Engine::flush_inserts() {
  prof::HostSpan span("host:memo_flush");
  if (memo_) memo_->flush_inserts();
}

void Engine::fu1d(const double2* u, float2* out, bool memoize) {
  apply(OpId::fu1d, false, u, true, nullptr, out, false, memoize);
}
void Engine::fu1d(const float2* u, float2* out, bool memoize) {
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
  apply(OpId::fu2d_adj, false, p, false, nullptr, out, false, memoize);
}
void Engine::f2d(const float2* p, float2* out, bool memoize) {
  apply(OpId::f2d, false, p, false, nullptr, out, false, memoize);
}
void Engine::f2d_adj(const float2* p, float2* out, bool memoize) {
  apply(OpId::f2d_adj, false, p, false, nullptr, out, false, memoize);
}

std::array<double, 2> Engine::fu2d_reduce(const float2* v, const float2* sub, const float2* dot) {
  Fu2dEpilogue e;
  e.sub = sub;
  e.ld_sub = g_.h;
  e.dot = dot;
  e.ld_dot = g_.h;
  e.reduce = true;
  const int slots = usfft_.fu2d(v, g_.h, 0, g_.h, e);
  const std::vector<double> r = usfft_.partials().sum(slots, 2, s_);
  return {r[0], r[1]};
}

}  // namespace mlrg
