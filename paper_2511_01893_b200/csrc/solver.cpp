#include "solver.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <iomanip>
#include <memory>
#include <sstream>
#include <utility>

#include "kernels.hpp"
#include "shard.hpp"

namespace mlrg {

void AdmmConfig::validate() const {  // admm.cpp:11-17
  if (!(alpha >= 0.0)) throw std::invalid_argument("admm: alpha must be >= 0");
  if (!(rho0 > 0.0)) throw std::invalid_argument("admm: rho0 must be positive");
  if (n_inner < 1) throw std::invalid_argument("admm: n_inner must be >= 1");
  if (n_outer < 1) throw std::invalid_argument("admm: n_outer must be >= 1");
  if (!(tau > 0.0f && tau <= 1.0f)) throw std::invalid_argument("admm: tau must be in (0, 1]");
}

std::string ReconReport::csv() const {
  std::ostringstream out;
  out << "iteration,loss,E,accuracy,miss,remote_hit,cache_hit,ms_lsp,ms_rsp,ms_update\n";
  out << std::setprecision(12);
  for (const IterationRow& r : rows)
    out << r.iteration << ',' << r.loss << ',' << r.e << ',' << r.accuracy << ',' << r.miss << ',' << r.remote_hit
        << ',' << r.cache_hit << ',' << r.ms_lsp << ',' << r.ms_rsp << ',' << r.ms_update << '\n';
  return out.str();
}

namespace {

/// Device ADMM state (admm.hpp:38-49). lambda is stored scaled: the true
/// multiplier is lam * lam_scale, with lam_scale a power of two, so the
/// residual-balancing rescale (admm.cpp:173-180) is exact and costs no pass.
/// Sharded: volume-side arrays hold this rank's planes [a, b), detector-side
/// arrays its rows [c, d); mid/mid2 are the engine's exchange blocks.
struct State {
  std::int64_t V, P, P0;  // local volume / detector sizes, one axis-0 plane
  DeviceBuffer<double2> u, G, G_prev, p, p_prev;       // volume side, complex128
  DeviceBuffer<double2> psi[3], psi_prev[3], lam[3], g[3];
  DeviceBuffer<double2> ref;                            // accuracy reference (optional)
  DeviceBuffer<float2> mid_own, mid2_own, rhat, dhat, dpred, fu2d_out;  // operator side, complex64
  float2 *mid = nullptr, *mid2 = nullptr;
  // sharded: halo inboxes (written by the neighbours) and their peer mappings
  DeviceBuffer<double2> in_u_lo, in_u_hi, in_g0_lo, in_G_hi, in_pp_hi;
  std::unique_ptr<PeerMemory> pm_u_lo, pm_u_hi, pm_g0_lo, pm_G_hi, pm_pp_hi;
  double rho = 1.0, lam_scale = 1.0;
  bool have_direction = false;
  std::vector<double> inner_losses;

  // ---- ADMM-Offload (AdmmConfig::offload): psi / lambda in pinned host memory ----
  static constexpr std::int64_t kChunk = 16;  // planes per g_init / RSP launch (both modes)
  bool offload = false;
  std::int64_t nchunks = 0;
  PinnedBuffer<double2> h_psi[3], h_psi_new[3], h_lam[3];
  DeviceBuffer<double2> c_psi[2][3], c_psi_new[2][3], c_lam[2][3];
  // offload copies: H2D on `side`, write-back D2H on `side_out`, so chunk k's
  // compute overlaps both chunk k+1's upload and chunk k-1's write-back
  cudaStream_t side = nullptr, side_out = nullptr;
  cudaEvent_t ev_in[2] = {}, ev_done[2] = {}, ev_back[2] = {}, ev_out = nullptr;

  ~State() {
    for (cudaStream_t st : {side, side_out})
      if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
      }
    for (int b = 0; b < 2; ++b)
      for (cudaEvent_t e : {ev_in[b], ev_done[b], ev_back[b]})
        if (e) cudaEventDestroy(e);
    if (ev_out) cudaEventDestroy(ev_out);
  }

  State(const Geometry& geo, const Engine& eng, bool baseline, bool offload_, cudaStream_t s) : offload(offload_) {
    const Shard& sh = eng.shard();
    P0 = geo.n0 * geo.n2;
    V = sh.np() * P0;
    P = geo.n_theta * sh.nr() * geo.w;
    const std::int64_t M = geo.mid_shape().count();
    auto vz = [&](auto& b, std::int64_t n) {
      b.resize(static_cast<std::size_t>(n));
      b.zero(s);
    };
    for (auto* b : {&u, &G, &G_prev, &p, &p_prev}) vz(*b, V);
    for (int c = 0; c < 3; ++c) vz(g[c], V);
    const std::int64_t np = sh.np();
    nchunks = (np + kChunk - 1) / kChunk;
    // the fused RSP pass writes 2 partial slots per CTA per chunk into the fixed
    // Partials table before the host sums them: refuse at setup, not by overrunning it
    if (nchunks * ops::rsp_multiplier_slots() > Partials::kMaxSlots)
      throw std::invalid_argument("solver: " + std::to_string(np) + " planes per rank exceed the RSP partial table (" +
                                  std::to_string(Partials::kMaxSlots / ops::rsp_multiplier_slots() * kChunk) +
                                  " planes); use more ranks");
    if (!offload) {
      for (int c = 0; c < 3; ++c) {
        vz(psi[c], V);
        vz(psi_prev[c], V);
        vz(lam[c], V);
      }
    } else {  // pinned host residency + double-buffered device chunks
      for (int c = 0; c < 3; ++c) {
        for (auto* hb : {&h_psi[c], &h_psi_new[c], &h_lam[c]}) {
          hb->reserve(static_cast<std::size_t>(V));
          std::memset(hb->get(), 0, static_cast<std::size_t>(V) * sizeof(double2));
        }
      }
      const std::int64_t cn = std::min<std::int64_t>(kChunk, np) * P0;
      for (int b = 0; b < 2; ++b)
        for (int c = 0; c < 3; ++c)
          for (auto* db : {&c_psi[b][c], &c_psi_new[b][c], &c_lam[b][c]}) db->resize(static_cast<std::size_t>(cn));
      MLRG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      MLRG_CUDA(cudaStreamCreateWithFlags(&side_out, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b)
        for (cudaEvent_t* e : {&ev_in[b], &ev_done[b], &ev_back[b]})
          MLRG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      MLRG_CUDA(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
    }
    if (sh.sharded()) {
      if (baseline) throw std::invalid_argument("admm: pipeline=baseline runs on one GPU only (sharded: optimized)");
      mid = eng.mid();
      mid2 = eng.mid2();
      for (auto* b : {&in_u_lo, &in_u_hi, &in_g0_lo, &in_G_hi, &in_pp_hi}) vz(*b, P0);
      HostComm& c = *sh.comm;
      MLRG_CUDA(cudaStreamSynchronize(s));
      pm_u_lo = std::make_unique<PeerMemory>(c, in_u_lo.get());
      pm_u_hi = std::make_unique<PeerMemory>(c, in_u_hi.get());
      pm_g0_lo = std::make_unique<PeerMemory>(c, in_g0_lo.get());
      pm_G_hi = std::make_unique<PeerMemory>(c, in_G_hi.get());
      pm_pp_hi = std::make_unique<PeerMemory>(c, in_pp_hi.get());
    } else {
      vz(mid_own, M);
      vz(mid2_own, M);
      mid = mid_own.get();
      mid2 = mid2_own.get();
    }
    vz(rhat, P);
    vz(dhat, P);
    if (baseline) {
      vz(dpred, P);
      vz(fu2d_out, P);
    }
  }
  DField3 f(DeviceBuffer<double2> (&a)[3]) { return DField3{{a[0].get(), a[1].get(), a[2].get()}}; }
};

std::int64_t local_count(const Engine& e) { return e.shard().np() * e.geometry().n0 * e.geometry().n2; }

bool trace_on() {  // MLRG_TRACE=1: per-step solver scalars on stderr (diagnostics)
  static const bool on = [] {
    const char* v = std::getenv("MLRG_TRACE");
    return v && *v && *v != '0';
  }();
  return on;
}

double ms_between(std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}

}  // namespace

struct SolverState : State {
  const float2* d;
  bool has_reference;
  AdmmConfig cfg;
  Engine& eng;
  ReconReport rep;
  MemoCounters prev;
  int outer = 0;
  SolverState(const float2* d_, const AdmmConfig& c, Engine& e, const float2* ref)
      : State(e.geometry(), e, c.pipeline == Pipeline::baseline, c.offload, e.stream()),
        d(d_),
        has_reference(ref != nullptr),
        cfg(c),
        eng(e) {
    if (ref) {  // this rank's planes of the full reference volume
      this->ref.resize(static_cast<std::size_t>(V));
      ops::c64_to_c128(ref + e.shard().a() * P0, this->ref.get(), V, e.stream());
    }
  }

  // ---- halo exchange (sharded): push this rank's boundary planes into the
  // neighbours' inboxes; completion is published by the next fence/allreduce ----
  const Shard& sh() const { return eng.shard(); }
  void push(const double2* plane, const PeerMemory* pm, int to) {
    MLRG_CUDA(cudaMemcpyAsync(pm->at(to), plane, static_cast<std::size_t>(P0) * sizeof(double2), cudaMemcpyDefault,
                              eng.stream()));
  }
  void push_u() {
    if (!sh().sharded()) return;
    const int r = sh().rank;
    if (r > 0) push(u.get(), pm_u_hi.get(), r - 1);
    if (r + 1 < sh().world) push(u.get() + (sh().np() - 1) * P0, pm_u_lo.get(), r + 1);
  }
  void push_g0() {
    if (!sh().sharded() || sh().rank + 1 >= sh().world) return;
    push(g[0].get() + (sh().np() - 1) * P0, pm_g0_lo.get(), sh().rank + 1);
  }
  void push_G_pp() {
    if (!sh().sharded() || sh().rank == 0) return;
    push(G.get(), pm_G_hi.get(), sh().rank - 1);
    push(p_prev.get(), pm_pp_hi.get(), sh().rank - 1);
  }
  // ---- g_init and the fused RSP/multiplier pass, in 16-plane chunks (both modes,
  // so offload on and off launch identical kernels and reduce identically) ----
  std::int64_t chunk_planes(std::int64_t k) const { return std::min(kChunk, sh().np() - k * kChunk); }
  std::size_t chunk_bytes(std::int64_t k) const {
    return static_cast<std::size_t>(chunk_planes(k) * P0) * sizeof(double2);
  }
  void h2d(DeviceBuffer<double2> (&dst)[3], PinnedBuffer<double2> (&src)[3], std::int64_t k) {
    for (int c = 0; c < 3; ++c)
      MLRG_CUDA(cudaMemcpyAsync(dst[c].get(), src[c].get() + k * kChunk * P0, chunk_bytes(k), cudaMemcpyHostToDevice,
                                side));
  }
  void d2h(PinnedBuffer<double2> (&dst)[3], DeviceBuffer<double2> (&src)[3], std::int64_t k) {
    for (int c = 0; c < 3; ++c)
      MLRG_CUDA(cudaMemcpyAsync(dst[c].get() + k * kChunk * P0, src[c].get(), chunk_bytes(k), cudaMemcpyDeviceToHost,
                                side_out));
  }
  static DField3 at(DeviceBuffer<double2> (&a)[3], std::int64_t off) {
    return DField3{{a[0].get() + off, a[1].get() + off, a[2].get() + off}};
  }

  void g_init_chunks(double lc, cudaStream_t s) {  // g = psi - lambda * lc (admm.cpp:64)
    for (std::int64_t k = 0; k < nchunks; ++k) {
      const std::int64_t off = k * kChunk * P0, n = chunk_planes(k) * P0;
      if (!offload) {
        ops::g_init(CDField3(at(psi, off)), CDField3(at(lam, off)), at(g, off), n, lc, s);
        continue;
      }
      const int b = static_cast<int>(k & 1);
      MLRG_CUDA(cudaStreamWaitEvent(side, ev_done[b], 0));  // chunk k-2 is done with buffer b
      h2d(c_psi[b], h_psi, k);
      h2d(c_lam[b], h_lam, k);
      MLRG_CUDA(cudaEventRecord(ev_in[b], side));
      MLRG_CUDA(cudaStreamWaitEvent(s, ev_in[b], 0));
      ops::g_init(CDField3(at(c_psi[b], 0)), CDField3(at(c_lam[b], 0)), at(g, off), n, lc, s);
      MLRG_CUDA(cudaEventRecord(ev_done[b], s));
    }
  }

  /// Returns the partial-slot count written (chunk-major).
  int rsp_chunks(double lc, double thr, double rho_s, double* partials, cudaStream_t s, const Geometry& geo) {
    int slots = 0;
    const ops::Halo rank_halo = halo();
    for (std::int64_t k = 0; k < nchunks; ++k) {
      const std::int64_t off = k * kChunk * P0, np = chunk_planes(k);
      const Dims dk{np, geo.n0, geo.n2};
      ops::Halo hk;  // the plane above the chunk: the next chunk's first, or the rank halo
      hk.u_hi = k + 1 < nchunks ? u.get() + off + np * P0 : rank_halo.u_hi;
      if (!offload) {
        slots += ops::rsp_multiplier(u.get() + off, at(lam, off), CDField3(at(psi, off)), at(psi_prev, off), dk, lc,
                                     thr, rho_s, partials + slots, s, hk);
        continue;
      }
      const int b = static_cast<int>(k & 1);
      // buffer b: chunk k-2's compute is done with c_psi[b] and its write-back has read c_lam[b], c_psi_new[b]
      MLRG_CUDA(cudaStreamWaitEvent(side, ev_done[b], 0));
      if (k >= 2) MLRG_CUDA(cudaStreamWaitEvent(side, ev_back[b], 0));
      h2d(c_psi[b], h_psi, k);
      h2d(c_lam[b], h_lam, k);
      MLRG_CUDA(cudaEventRecord(ev_in[b], side));
      MLRG_CUDA(cudaStreamWaitEvent(s, ev_in[b], 0));
      if (k >= 2) MLRG_CUDA(cudaStreamWaitEvent(s, ev_back[b], 0));  // c_psi_new[b] is free again
      slots += ops::rsp_multiplier(u.get() + off, at(c_lam[b], 0), CDField3(at(c_psi[b], 0)), at(c_psi_new[b], 0), dk,
                                   lc, thr, rho_s, partials + slots, s, hk);
      MLRG_CUDA(cudaEventRecord(ev_done[b], s));
      MLRG_CUDA(cudaStreamWaitEvent(side_out, ev_done[b], 0));
      d2h(h_lam, c_lam[b], k);
      d2h(h_psi_new, c_psi_new[b], k);
      MLRG_CUDA(cudaEventRecord(ev_back[b], side_out));
    }
    if (offload) {  // the host copies are complete before anything reads them
      MLRG_CUDA(cudaEventRecord(ev_out, side_out));
      MLRG_CUDA(cudaStreamWaitEvent(s, ev_out, 0));
    }
    return slots;
  }
  void swap_psi() {  // psi_prev <- old psi; psi <- new
    for (int c = 0; c < 3; ++c) {
      if (offload) std::swap(h_psi[c], h_psi_new[c]);
      else std::swap(psi[c], psi_prev[c]);
    }
  }

  ops::Halo halo() const {
    ops::Halo h;
    if (!sh().sharded()) return h;
    const bool lo = sh().rank > 0, hi = sh().rank + 1 < sh().world;
    if (lo) {
      h.u_lo = in_u_lo.get();
      h.g0_lo = in_g0_lo.get();
    }
    if (hi) {
      h.u_hi = in_u_hi.get();
      h.G_hi = in_G_hi.get();
      h.pp_hi = in_pp_hi.get();
    }
    return h;
  }
};

Solver::Solver(const float2* d, const AdmmConfig& cfg, Engine& eng, const float2* reference) {
  cfg.validate();
  st_ = new SolverState(d, cfg, eng, reference);
  st_->rho = cfg.rho0;
  const Shard& sh = eng.shard();
  if (!sh.sharded()) {
    eng.f2d(d, st_->dhat.get(), false);  // admm.cpp:220
  } else {  // d_hat of the full data, then this rank's rows (n_theta, [c, d), w)
    const Geometry& g = eng.geometry();
    DeviceBuffer<float2> full(static_cast<std::size_t>(g.projection_shape().count()));
    eng.f2d(d, full.get(), false);
    MLRG_CUDA(cudaMemcpy2DAsync(st_->dhat.get(), static_cast<std::size_t>(sh.nr() * g.w) * sizeof(float2),
                                full.get() + sh.c() * g.w, static_cast<std::size_t>(g.h * g.w) * sizeof(float2),
                                static_cast<std::size_t>(sh.nr() * g.w) * sizeof(float2),
                                static_cast<std::size_t>(g.n_theta), cudaMemcpyDeviceToDevice, eng.stream()));
    MLRG_CUDA(cudaStreamSynchronize(eng.stream()));
  }
  st_->prev = eng.memo() ? eng.memo()->counters() : MemoCounters{};
}

Solver::~Solver() { delete st_; }
int Solver::iteration() const { return st_->outer; }
const ReconReport& Solver::report() const { return st_->rep; }
const double2* Solver::u() const { return st_->u.get(); }

bool Solver::step() {
  SolverState& st = *st_;
  if (st.rep.aborted) return false;
  const AdmmConfig& cfg = st.cfg;
  Engine& eng = st.eng;
  const Geometry& geo = eng.geometry();
  cudaStream_t s = eng.stream();
  Partials& part = eng.usfft().partials();
  const Dims dims{eng.shard().np(), geo.n0, geo.n2};  // this rank's planes
  const bool baseline = cfg.pipeline == Pipeline::baseline;
  const float2* d = st.d;
  using clock = std::chrono::steady_clock;
  auto sum = [&](int slots, int nv) {  // CTA partials -> this rank's sums -> summed over ranks
    std::vector<double> v = part.sum(slots, nv, s);
    eng.allreduce(v.data(), nv);
    return v;
  };
  const int outer = st.outer++;
  {
    eng.set_iteration(outer);
    IterationRow row;
    row.iteration = outer;
    int obj_tv_slots = 0, obj_nd_slots = 0, obj_slots = 0;  // the objective's partial tables (enqueued after RSP)
    try {
      const auto t0 = clock::now();
      // ---- LSP (admm.cpp:59-118, 122-152) ----
      st.g_init_chunks(st.lam_scale / st.rho, s);
      st.push_g0();
      st.have_direction = false;
      const std::size_t phase_start = st.inner_losses.size();
      for (int inner = 0; inner < cfg.n_inner; ++inner) {
        // gradient(u): r_hat, loss terms, G
        double rr = 0.0;
        Partials::Range rr_range{Partials::kParked, 0, 2};  // |r_hat|^2, read back with the gradient's terms
        st.push_u();  // published by fu1d's exchange fences
        eng.fu1d(st.u.get(), st.mid);
        if (baseline) {
          eng.fu2d(st.mid, st.fu2d_out.get());
          eng.f2d_adj(st.fu2d_out.get(), st.dpred.get());
          rr = sum(ops::sub_norm(st.dpred.get(), d, st.P, part.dev(), s), 1)[0];
          eng.f2d(st.dpred.get(), st.rhat.get());
        } else {
          eng.fu2d_fused(st.mid, st.dhat.get(), st.rhat.get());
          rr_range.count = ops::norm2_diff(st.rhat.get(), nullptr, st.P, part.dev() + Partials::kParked, s);
        }
        eng.fu2d_adj(st.rhat.get(), st.mid2);
        eng.fu1d_adj(st.mid2, st.G.get());
        const bool hd = st.have_direction;
        const int gu_slots =
            ops::grad_update(st.u.get(), CDField3(st.f(st.g)), st.G.get(), hd ? st.p_prev.get() : nullptr,
                             hd ? st.G_prev.get() : nullptr, dims, st.rho, part.dev(), s, st.halo());
        st.push_G_pp();  // published by the allreduce below
        std::vector<std::vector<double>> sums = part.sum({{0, gu_slots, 3}, rr_range}, s);
        for (auto& x : sums) eng.allreduce(x.data(), static_cast<int>(x.size()));
        const std::vector<double>& gu = sums[0];
        if (!baseline) rr = sums[1][1];
        const double loss = 0.5 * rr + 0.5 * st.rho * gu[0];
        st.inner_losses.push_back(loss);
        const std::size_t n = st.inner_losses.size();
        if (n >= phase_start + 4 && st.inner_losses[n - 1] > 10.0 * st.inner_losses[n - 4]) {
          std::ostringstream msg;
          msg << "inner loss diverged: " << st.inner_losses[n - 4] << " -> " << st.inner_losses[n - 1]
              << " within 3 iterations";
          throw AdmmAbort(msg.str());
        }
        const double normG2 = gu[1];
        double beta = 0.0;
        if (hd && gu[2] > 0.0) beta = normG2 / gu[2];
        auto step_terms = [&](double bt, double& a, double& b) {
          // the direction's terms are read back with fu2d_reduce's (one synchronisation)
          const int dr_slots = ops::direction(st.G.get(), st.p_prev.get(), bt, st.u.get(), CDField3(st.f(st.g)),
                                              st.p.get(), dims, part.dev() + Partials::kParked, s, st.halo());
          eng.fu1d(st.p.get(), st.mid, false);
          std::vector<std::vector<double>> drv;
          const std::array<double, 2> q =
              eng.fu2d_reduce(st.mid, nullptr, st.rhat.get(), {{Partials::kParked, dr_slots, 2}}, &drv);
          const std::vector<double>& dr = drv[0];
          a = q[0] + st.rho * dr[0];
          b = q[1] + st.rho * dr[1];
        };
        double a = 0.0, b = 0.0;
        step_terms(beta, a, b);
        if (b > 0.0) step_terms(0.0, a, b);  // uphill: steepest descent (admm.cpp:103-106)
        if (trace_on())
          std::fprintf(stderr, "mlrg-trace outer %d inner %d loss %.9g normG2 %.9g dy %.9g beta %.9g a %.9g b %.9g\n",
                       outer, inner, loss, normG2, gu[2], beta, a, b);
        if (a > 0.0 && b < 0.0) ops::axpy(st.u.get(), st.p.get(), -b / a, st.V, s);
        std::swap(st.G_prev, st.G);
        std::swap(st.p_prev, st.p);
        st.have_direction = true;
      }
      MLRG_CUDA(cudaStreamSynchronize(s));
      const auto t1 = clock::now();
      // ---- RSP + multiplier/penalty, one fused pass (admm.cpp:154-181) ----
      st.push_u();
      eng.fence();  // sharded: publish the u halos
      // the RSP partials' copy is enqueued now and read after the objective is
      // enqueued behind it (the objective reuses the slots after the copy, in
      // stream order), so the host's readback overlaps the objective's kernels
      const int rsp_slots =
          st.rsp_chunks(st.lam_scale / st.rho, cfg.alpha / st.rho, st.rho / st.lam_scale, part.dev(), s, geo);
      part.sum_begin(rsp_slots, s);
      st.swap_psi();
      eng.mark_flush_point();  // no memoized call from here to the flush
      obj_tv_slots = ops::tv_norm(st.u.get(), dims, part.dev() + Partials::kParked, s, st.halo());
      if (st.has_reference)
        obj_nd_slots = ops::norm2_diff(st.ref.get(), st.u.get(), st.V, part.dev() + Partials::kParked + obj_tv_slots, s);
      eng.fu1d(st.u.get(), st.mid, false);
      obj_slots = eng.fu2d_reduce_begin(st.mid, st.dhat.get(), nullptr);
      std::vector<double> rs = part.sum_end(rsp_slots, 2);
      eng.allreduce(rs.data(), 2);
      const auto t2 = clock::now();
      const double r = std::sqrt(rs[0]);
      const double sres = st.rho * std::sqrt(rs[1]);
      if (!cfg.freeze_rho) {
        if (r > 10.0 * sres) {
          st.rho *= 2.0;
          st.lam_scale *= 0.5;
        } else if (sres > 10.0 * r) {
          st.rho *= 0.5;
          st.lam_scale *= 2.0;
        }
      }
      if (trace_on()) std::fprintf(stderr, "mlrg-trace outer %d rho %.17g r %.17g s %.17g\n", outer, st.rho, r, sres);
      const auto t3 = clock::now();
      row.ms_lsp = ms_between(t0, t1);
      row.ms_rsp = ms_between(t1, t2);
      row.ms_update = ms_between(t2, t3);
    } catch (const AdmmAbort& ex) {
      eng.drain_memo_log();  // the aborted iteration's decisions stay in the audit, unflushed
      st.rep.aborted = true;
      st.rep.abort_reason = ex.what();
      return false;
    }
    // objective (admm.cpp:190-195), not memoized, enqueued above behind the
    // RSP pass; the memo flush (admm.cpp:251-254; no lookup runs in between, so
    // the order does not change a decision) drains the decision log behind the
    // mark while the GPU runs it; TV term and accuracy are read back with the
    // data term
    std::vector<Partials::Range> extra{{Partials::kParked, obj_tv_slots, 1}};
    if (st.has_reference) extra.push_back({Partials::kParked + obj_tv_slots, obj_nd_slots, 2});
    eng.flush_inserts();
    std::vector<std::vector<double>> ex;
    const std::array<double, 2> data = eng.fu2d_reduce_end(obj_slots, extra, &ex);
    const double tv = ex[0][0];
    row.loss = 0.5 * data[0] + cfg.alpha * tv;
    if (st.has_reference) {  // accuracy(reference, u), admm.cpp:183-188
      const std::vector<double>& nd = ex[1];
      if (nd[1] == 0.0) throw std::invalid_argument("accuracy: reference volume has zero norm");
      row.e = std::sqrt(nd[0]) / std::sqrt(nd[1]);
      row.accuracy = 1.0 - row.e;
    }
    if (eng.memo()) {
      const MemoCounters now = eng.memo()->counters();
      row.miss = now.misses - st.prev.misses;
      row.remote_hit = now.remote_hits - st.prev.remote_hits;
      row.cache_hit = now.cache_hits - st.prev.cache_hits;
      st.prev = now;
    }
    st.rep.rows.push_back(row);
  }
  return true;
}

ReconReport reconstruct(const float2* d, const AdmmConfig& cfg, Engine& eng, const float2* reference, float2* u_out) {
  Solver solver(d, cfg, eng, reference);
  for (int outer = 0; outer < cfg.n_outer; ++outer)
    if (!solver.step()) break;
  cudaStream_t s = eng.stream();
  ops::c128_to_c64(solver.u(), u_out, local_count(eng), s);
  MLRG_CUDA(cudaStreamSynchronize(s));
  return solver.report();
}

}  // namespace mlrg
