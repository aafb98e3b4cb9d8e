// C-ABI of the B200 build: the drop-in mlr.h surface (capi.cpp of the
// reference, re-implemented over the device engine) and the device mlrg.h
// surface. All exceptions stop here and become a thread-local message plus
// an MLR_* code (capi.cpp:37-47 error model).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <exception>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "solver.hpp"
#include "config.hpp"
#include "encoder.hpp"
#include "engine_api.hpp"
#include "host_io.hpp"
#include "offload_plan.hpp"
#include "cnn.hpp"
#include "kernels.hpp"
#include "memo.hpp"
#include "mlr.h"
#include "mlrg.h"
#include "usfft.hpp"

struct mlr_config {
  mlrg::RunConfig rc;
};
struct mlr_array {
  mlrg::HostArray a;
};
struct mlr_result {
  mlr_array u;
  mlrg::ReconReport report;
  std::vector<mlrg::ChunkAudit> audit;
};
struct mlr_server {};

struct mlrg_ctx {
  mlrg::Geometry g;
  cudaStream_t s = nullptr;
  bool own_stream = false;
  std::unique_ptr<mlrg::Usfft> usfft;
  mlrg::DeviceBuffer<float2> scratch_mid, scratch_proj;
  ~mlrg_ctx() {
    usfft.reset();
    if (own_stream && s) cudaStreamDestroy(s);
  }
};
struct mlrg_recon {
  mlrg::ReconReport report;
  std::vector<mlrg::ChunkAudit> audit;
  mlrg::MemoCounters counters;
  uint64_t tiers[3] = {0, 0, 0};
};
struct mlrg_solver {
  cudaStream_t own = nullptr;
  std::unique_ptr<mlrg::Engine> eng;
  std::unique_ptr<mlrg::Solver> solver;
  ~mlrg_solver() {
    solver.reset();
    eng.reset();
    if (own) cudaStreamDestroy(own);
  }
};
struct mlrg_comm {
  std::shared_ptr<mlrg::HostComm> c;
};
struct mlrg_memo {
  std::shared_ptr<mlrg::MemoStore> store;
  std::unique_ptr<mlrg::MemoClient> client;
};

namespace {

thread_local std::string t_error;

int code_for(const std::exception& e) {
  return dynamic_cast<const std::invalid_argument*>(&e) != nullptr ? MLR_ERR_CONFIG : MLR_ERR_RUNTIME;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MLR_OK;
  } catch (const std::exception& e) {
    t_error = e.what();
    return code_for(e);
  }
}

template <class T, class F>
T* guarded_ptr(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    t_error = e.what();
    return nullptr;
  }
}

char* dup_text(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  if (out) std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

void need(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

/// Engine assembly per reconstruction (capi.cpp:70-86). Both memo modes use
/// the device-resident store: "distributed" keeps the reference's decision
/// semantics (its transport only adds timeouts) without a TCP memory node.
std::unique_ptr<mlrg::Engine> build_engine(const mlrg::RunConfig& rc, const mlrg::Geometry& g, cudaStream_t s,
                                           std::shared_ptr<mlrg::HostComm> comm = nullptr) {
  mlrg::EngineConfig ec = rc.engine;
  ec.memo_enabled = rc.admm.memoization != mlrg::MemoMode::off;
  if (!ec.memo_enabled) return std::make_unique<mlrg::Engine>(g, ec, s, nullptr, nullptr, std::move(comm));

  auto store = std::make_shared<mlrg::MemoStore>();
  // HBM for the values: a ring arena (cold_tier.hpp) sized for every value the
  // solve can insert (n_outer windows of at most `window` values each, the
  // largest slab each, complex64), capped at 45% of free HBM; older values
  // spill to pinned host memory when the ring would wrap onto them.
  // MLRG_MEMO_ARENA_BYTES overrides the size (tests force spills with it).
  const std::int64_t e = ec.chunk_extent;
  const std::int64_t slab = std::max({e * g.h * g.n2, e * g.n0 * g.n2, g.n_theta * e * g.w, g.n1 * e * g.n2});
  const double slab_bytes = static_cast<double>((slab * static_cast<std::int64_t>(sizeof(float2)) + 255) & ~std::int64_t{255});
  std::size_t free_b = 0, total_b = 0;
  MLRG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  free_b += mlrg::alloc::cached_device_bytes();  // blocks a previous engine returned to the cache
  // lookups per window: every memoizable call of an outer iteration (4 per
  // inner step, 6 with pipeline = baseline) over this rank's slabs
  const int calls = (rc.admm.pipeline == mlrg::Pipeline::baseline ? 6 : 4) * rc.admm.n_inner;
  std::int64_t most = std::max((g.n1 + e - 1) / e, std::max((g.h + e - 1) / e, (g.n_theta + e - 1) / e));
  if (comm && comm->world() > 1) {  // a rank stores only its own slabs' values
    const mlrg::Shard sh = mlrg::Shard::make(g, e, comm);
    most = 0;
    for (int r = 0; r < sh.world; ++r) {
      const auto& pl = sh.planes[static_cast<std::size_t>(r)];
      const auto& rw = sh.rows[static_cast<std::size_t>(r)];
      most = std::max({most, (pl.second - pl.first + e - 1) / e, (rw.second - rw.first + e - 1) / e});
    }
  }
  const std::int64_t window = std::min<std::int64_t>(static_cast<std::int64_t>(rc.memo.insert_queue_cap), calls * most);
  ec.memo_window_inserts = static_cast<int>(std::max<std::int64_t>(window, 1));
  const double floor_b = static_cast<double>(ec.memo_window_inserts + 1) * slab_bytes;
  const double want = static_cast<double>(rc.admm.n_outer) * static_cast<double>(window) * slab_bytes;
  // what the solve still allocates besides the arena: the complex128 state (17
  // local volumes incl. the reference), the complex64 detector-side and exchange
  // arrays (8 local projection / mid arrays), two 16-row grid sets, the encoder
  // matrices (2 distinct slab shapes x key_dim x 2 x slab floats), 2 GiB of tables
  double local = 1.0;
  if (comm && comm->world() > 1) local = 1.0 / comm->world() + 1.0 / (g.n1 / e > 0 ? g.n1 / e : 1);
  const double V = static_cast<double>(g.n1 * g.n0 * g.n2) * local;
  const double P = static_cast<double>(std::max(g.n_theta * g.h * g.w, g.n1 * g.h * g.n2)) * local;
  const double grids = 4.0 * static_cast<double>(4 * g.n1 * g.n2 * 16 * 16);
  const double enc_bytes = 2.0 * rc.encoder.key_dim * 2.0 * static_cast<double>(slab) * sizeof(float);
  const double after = 17.0 * 16.0 * V + 8.0 * 8.0 * P + grids + enc_bytes + 2.0 * (1u << 30);
  const double budget = std::max(0.0, static_cast<double>(free_b) - after) * 0.9;
  std::size_t bytes = static_cast<std::size_t>(std::max(floor_b, std::min(want, budget)));
  if (const char* ov = std::getenv("MLRG_MEMO_ARENA_BYTES")) bytes = static_cast<std::size_t>(std::atoll(ov));
  // one GPU: the lookups run on the device (memo_gpu.hpp) unless the config needs
  // the host client (global cache, baseline pipeline's memoized f2d, other slab
  // sizes) or MLRG_DEVICE_MEMO=0 asks for it
  const char* dm = std::getenv("MLRG_DEVICE_MEMO");
  ec.device_memo = !(comm && comm->world() > 1) && !(dm && *dm == '0') && !rc.memo.global_cache &&
                   rc.admm.pipeline == mlrg::Pipeline::optimized && ec.chunk_extent == 16 && rc.encoder.key_dim <= 64;
  ec.memo_max_keys = std::min<std::int64_t>(
      std::int64_t{1} << 20,
      static_cast<std::int64_t>(rc.admm.n_outer) * static_cast<std::int64_t>(rc.memo.insert_queue_cap) +
          static_cast<std::int64_t>(rc.memo.insert_queue_cap) + 1);
  ec.memo_arena_bytes = bytes;
  auto client = std::make_shared<mlrg::MemoClient>(rc.memo, store);
  std::shared_ptr<mlrg::Encoder> enc;
  if (rc.encoder.variant == mlrg::EncoderConfig::Variant::cnn)  // capi.cpp:56-65: file, else seeded init
    enc = std::make_shared<mlrg::Encoder>(
        rc.encoder_weights.empty() ? mlrg::CnnWeights::init(rc.encoder.key_dim, rc.encoder.seed)
                                   : mlrg::CnnWeights::load(rc.encoder_weights, rc.encoder.key_dim, rc.encoder.seed),
        rc.encoder.seed, s);
  else
    enc = std::make_shared<mlrg::Encoder>(rc.encoder.key_dim, rc.encoder.seed);
  return std::make_unique<mlrg::Engine>(g, ec, s, enc, client, std::move(comm));
}

struct StreamGuard {
  cudaStream_t s = nullptr;
  StreamGuard() { MLRG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~StreamGuard() {
    if (s) cudaStreamDestroy(s);
  }
};

/// Host complex128 -> device complex64 through a ring of pinned blocks: host
/// threads round each block to complex64 while the previous block's DMA runs,
/// so PCIe carries 8 B per element (the device keeps these arrays in complex64;
/// round-to-nearest on the host is the device conversion's rounding).
void upload_c64(const mlrg::HostArray& a, mlrg::DeviceBuffer<float2>& dst, cudaStream_t s) {
  const std::size_t n = a.data.size();
  dst.resize(n);
  constexpr std::size_t kBlock = std::size_t{2} << 20;  // elements (16 MB of complex64)
  constexpr int kRing = 3, kThreads = 8;
  mlrg::PinnedBuffer<float2> ring[kRing];
  cudaEvent_t done[kRing];
  for (int r = 0; r < kRing; ++r) {
    ring[r].reserve(std::min(kBlock, std::max<std::size_t>(n, 1)));
    MLRG_CUDA(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
  }
  std::exception_ptr err;
  try {
    const auto* src = a.data.data();
    for (std::size_t off = 0, i = 0; off < n; off += kBlock, ++i) {
      const int r = static_cast<int>(i % kRing);
      const std::size_t len = std::min(kBlock, n - off);
      if (i >= kRing) MLRG_CUDA(cudaEventSynchronize(done[r]));  // the block's previous copy finished
      float2* buf = ring[r].get();
      const std::size_t per = (len + kThreads - 1) / kThreads;
      std::vector<std::thread> th;
      for (int t = 0; t < kThreads; ++t)
        th.emplace_back([=] {
          for (std::size_t e = std::min(len, t * per), e1 = std::min(len, e + per); e < e1; ++e)
            buf[e] = make_float2(static_cast<float>(src[off + e].real()), static_cast<float>(src[off + e].imag()));
        });
      for (auto& x : th) x.join();
      MLRG_CUDA(cudaMemcpyAsync(dst.get() + off, buf, len * sizeof(float2), cudaMemcpyHostToDevice, s));
      MLRG_CUDA(cudaEventRecord(done[r], s));
    }
    MLRG_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    err = std::current_exception();
    cudaStreamSynchronize(s);
  }
  for (int r = 0; r < kRing; ++r) cudaEventDestroy(done[r]);
  if (err) std::rethrow_exception(err);
}

/// Device -> host copy into pageable memory through a ring of pinned blocks:
/// the copy engine fills block b + 1 while host threads move block b out.
void d2h_staged(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
  constexpr std::size_t kBlock = std::size_t{16} << 20;
  constexpr int kRing = 3, kThreads = 8;
  if (bytes < 2 * kBlock) {
    MLRG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    MLRG_CUDA(cudaStreamSynchronize(s));
    return;
  }
  mlrg::PinnedBuffer<char> ring[kRing];
  cudaEvent_t done[kRing];
  for (int r = 0; r < kRing; ++r) {
    ring[r].reserve(kBlock);
    MLRG_CUDA(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
  }
  const std::size_t nblk = (bytes + kBlock - 1) / kBlock;
  auto issue = [&](std::size_t i) {
    const int r = static_cast<int>(i % kRing);
    const std::size_t off = i * kBlock, len = std::min(kBlock, bytes - off);
    MLRG_CUDA(cudaMemcpyAsync(ring[r].get(), static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s));
    MLRG_CUDA(cudaEventRecord(done[r], s));
  };
  std::exception_ptr err;
  try {
    for (std::size_t i = 0; i < std::min<std::size_t>(kRing, nblk); ++i) issue(i);
    for (std::size_t i = 0; i < nblk; ++i) {
      const int r = static_cast<int>(i % kRing);
      const std::size_t off = i * kBlock, len = std::min(kBlock, bytes - off);
      MLRG_CUDA(cudaEventSynchronize(done[r]));
      const std::size_t per = (len + kThreads - 1) / kThreads;
      std::vector<std::thread> th;
      for (int t = 0; t < kThreads; ++t) {
        const std::size_t lo = std::min(len, t * per), hi = std::min(len, lo + per);
        th.emplace_back([&, lo, hi] { std::memcpy(static_cast<char*>(dst) + off + lo, ring[r].get() + lo, hi - lo); });
      }
      for (auto& x : th) x.join();
      if (i + kRing < nblk) issue(i + kRing);
    }
  } catch (...) {
    err = std::current_exception();
    cudaStreamSynchronize(s);
  }
  for (int r = 0; r < kRing; ++r) cudaEventDestroy(done[r]);
  if (err) std::rethrow_exception(err);
}

void download_c128(const float2* src, mlrg::HostArray& a, cudaStream_t s) {
  const std::size_t n = a.data.size();
  mlrg::DeviceBuffer<double2> tmp(n);
  mlrg::ops::c64_to_c128(src, tmp.get(), static_cast<std::int64_t>(n), s);
  MLRG_CUDA(cudaMemcpyAsync(a.data.data(), tmp.get(), n * sizeof(double2), cudaMemcpyDeviceToHost, s));
  MLRG_CUDA(cudaStreamSynchronize(s));
}

/// forward_L = f2d_adj(fu2d(fu1d(u))) on full device arrays (operators.cpp:301-304).
void forward_L(mlrg::Usfft& op, const float2* u, float2* out, mlrg::DeviceBuffer<float2>& mid,
               mlrg::DeviceBuffer<float2>& proj) {
  const mlrg::Geometry& g = op.geometry();
  mid.resize(static_cast<std::size_t>(g.mid_shape().count()));
  proj.resize(static_cast<std::size_t>(g.projection_shape().count()));
  op.fu1d(u, mid.get(), g.n1);
  mlrg::Fu2dEpilogue e;
  e.out = proj.get();
  e.ld_out = g.h;
  op.fu2d(mid.get(), g.h, 0, g.h, e);
  op.f2d(proj.get(), out, g.n_theta, true);
}

void adjoint_L(mlrg::Usfft& op, const float2* d, float2* out, mlrg::DeviceBuffer<float2>& mid,
               mlrg::DeviceBuffer<float2>& proj) {  // operators.cpp:306-309
  const mlrg::Geometry& g = op.geometry();
  mid.resize(static_cast<std::size_t>(g.mid_shape().count()));
  proj.resize(static_cast<std::size_t>(g.projection_shape().count()));
  op.f2d(d, proj.get(), g.n_theta, false);
  op.fu2d_adj(proj.get(), g.h, 0, g.h, mid.get(), g.h, 0);
  op.fu1d_adj(mid.get(), out, g.n1);
}

void fill_counters(const mlrg::MemoCounters& c, uint64_t out[11]) {
  const uint64_t v[11] = {c.lookups,      c.cache_hits,   c.remote_hits, c.misses,
                          c.cache_comparisons, c.cache_probes, c.timeouts,    c.batches_sent,
                          c.inserts_enqueued,  c.inserts_sent, c.inserts_dropped};
  std::memcpy(out, v, sizeof(v));
}

int64_t copy_audit(const std::vector<mlrg::ChunkAudit>& a, int32_t* meta4, float* cs, int64_t cap) {
  const int64_t n = static_cast<int64_t>(a.size());
  for (int64_t i = 0; i < n && i < cap; ++i) {
    const mlrg::ChunkAudit& e = a[static_cast<std::size_t>(i)];
    if (meta4) {
      meta4[4 * i + 0] = e.iteration;
      meta4[4 * i + 1] = static_cast<int32_t>(e.op);
      meta4[4 * i + 2] = static_cast<int32_t>(e.index);
      meta4[4 * i + 3] = static_cast<int32_t>(e.outcome);
    }
    if (cs) cs[i] = e.cs;
  }
  return n;
}

}  // namespace

extern "C" {

// ============================== mlr.h ==============================

const char* mlr_last_error(void) { return t_error.c_str(); }
void mlr_free(char* text) { std::free(text); }

mlr_config* mlr_config_new(void) {
  return guarded_ptr<mlr_config>([] { return new mlr_config{}; });
}

mlr_config* mlr_config_from_file(const char* path) {
  return guarded_ptr<mlr_config>([&] {
    need(path != nullptr, "config path is null");
    return new mlr_config{mlrg::RunConfig::from_file(path)};
  });
}

int mlr_config_set(mlr_config* cfg, const char* key, const char* value) {
  return guarded([&] {
    need(cfg && key && value, "null argument");
    cfg->rc.set(key, value);
  });
}

char* mlr_config_dump(const mlr_config* cfg) {
  return guarded_ptr<char>([&] {
    need(cfg != nullptr, "null config");
    return dup_text(cfg->rc.str());
  });
}

void mlr_config_free(mlr_config* cfg) { delete cfg; }

mlr_array* mlr_array_load(const char* path) {
  return guarded_ptr<mlr_array>([&] {
    need(path != nullptr, "array path is null");
    return new mlr_array{mlrg::load_lvol(path)};
  });
}

int mlr_array_save(const mlr_array* a, const char* path) {
  try {
    need(a && path, "null argument");
    mlrg::save_lvol(path, a->a);
    return MLR_OK;
  } catch (const std::invalid_argument& e) {
    t_error = e.what();
    return MLR_ERR_CONFIG;
  } catch (const std::exception& e) {
    t_error = e.what();
    return MLR_ERR_IO;
  }
}

int mlr_array_shape(const mlr_array* a, int64_t shape[3]) {
  return guarded([&] {
    need(a && shape, "null argument");
    shape[0] = a->a.shape.d0;
    shape[1] = a->a.shape.d1;
    shape[2] = a->a.shape.d2;
  });
}

const double* mlr_array_data(const mlr_array* a) {
  if (a == nullptr) {
    t_error = "null array";
    return nullptr;
  }
  return reinterpret_cast<const double*>(a->a.data.data());
}

void mlr_array_free(mlr_array* a) { delete a; }

mlr_array* mlr_make_phantom(const char* kind, int64_t d0, int64_t d1, int64_t d2, uint64_t seed) {
  return guarded_ptr<mlr_array>([&] {
    need(kind != nullptr, "phantom kind is null");
    return new mlr_array{mlrg::make_phantom({d0, d1, d2}, kind, seed)};
  });
}

mlr_array* mlr_project(const mlr_config* cfg, const mlr_array* volume) {
  return guarded_ptr<mlr_array>([&] {
    need(cfg && volume, "null argument");
    cfg->rc.validate();
    const mlrg::Geometry g = cfg->rc.make_geometry();
    if (!(volume->a.shape == g.volume_shape()))
      throw std::invalid_argument("volume shape " + volume->a.shape.str() +
                                  " does not match the configured geometry " + g.volume_shape().str());
    StreamGuard sg;
    mlrg::Usfft op(g, sg.s, cfg->rc.engine.kernel);
    mlrg::DeviceBuffer<float2> u, out, mid, proj;
    upload_c64(volume->a, u, sg.s);
    out.resize(static_cast<std::size_t>(g.projection_shape().count()));
    forward_L(op, u.get(), out.get(), mid, proj);
    auto* res = new mlr_array{mlrg::HostArray(g.projection_shape(), 0, /*zero=*/false)};
    download_c128(out.get(), res->a, sg.s);
    return res;
  });
}

mlr_result* mlr_reconstruct(const mlr_config* cfg, const mlr_array* data, const mlr_array* reference) {
  mlrg::prof::HostSpan total("host:e2e_total");
  return guarded_ptr<mlr_result>([&] {
    need(cfg && data, "null argument");
    cfg->rc.validate();
    const mlrg::Geometry g = cfg->rc.make_geometry();
    if (!(data->a.shape == g.projection_shape()))
      throw std::invalid_argument("data shape " + data->a.shape.str() + " does not match the configured geometry " +
                                  g.projection_shape().str());
    if (reference && !(reference->a.shape == g.volume_shape()))
      throw std::invalid_argument("reference shape " + reference->a.shape.str() +
                                  " does not match the configured geometry " + g.volume_shape().str());
    auto res = std::make_unique<mlr_result>();
    // the result volume is allocated and its pages faulted in by host threads
    // while the device iterates (first-touch faults of hundreds of MB otherwise
    // land inside the final device-to-host copy); started once the operator
    // tables are built, so its threads do not compete with the table build
    std::thread prefault;
    auto start_prefault = [&] {
      prefault = std::thread([&res, shape = g.volume_shape()] {
      res->u.a = mlrg::HostArray(shape, 0, /*zero=*/false);
      auto& v = res->u.a.data;
      const std::size_t n = v.size(), nt = 8, per = (n + nt - 1) / nt;
      std::vector<std::thread> th;
      for (std::size_t t = 0; t < nt; ++t)
        th.emplace_back([&v, n, lo = t * per, per] {
          for (std::size_t i = lo; i < std::min(n, lo + per); i += 256) v[i] = {0.0, 0.0};
        });
      for (auto& x : th) x.join();
      });
    };
    struct Joiner {
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } joiner{prefault};
    auto teardown = std::make_unique<mlrg::prof::HostSpan>("host:e2e_teardown_and_rest");
    StreamGuard sg, up;
    std::unique_ptr<mlrg::Engine> eng;
    mlrg::DeviceBuffer<float2> d, ref;
    {
      // the inputs go up on their own stream and thread while this thread
      // builds the operator tables (host work) and the engine
      int dev = 0;
      MLRG_CUDA(cudaGetDevice(&dev));
      std::exception_ptr up_err;
      std::thread uploader([&] {
        try {
          mlrg::prof::HostSpan span("host:e2e_upload");
          MLRG_CUDA(cudaSetDevice(dev));
          upload_c64(data->a, d, up.s);
          if (reference) upload_c64(reference->a, ref, up.s);
        } catch (...) {
          up_err = std::current_exception();
        }
      });
      try {
        mlrg::prof::HostSpan span("host:e2e_engine");
        eng = build_engine(cfg->rc, g, sg.s);
      } catch (...) {
        uploader.join();
        throw;
      }
      uploader.join();
      if (up_err) std::rethrow_exception(up_err);
      start_prefault();
    }
    {
      std::unique_ptr<mlrg::Solver> solver;
      {
        mlrg::prof::HostSpan span("host:e2e_solver_setup");
        solver = std::make_unique<mlrg::Solver>(d.get(), cfg->rc.admm, *eng, reference ? ref.get() : nullptr);
      }
      {
        mlrg::prof::HostSpan span("host:e2e_iterations");
        for (int it = 0; it < cfg->rc.admm.n_outer; ++it)
          if (!solver->step()) break;
      }
      {
        mlrg::prof::HostSpan span("host:e2e_download");
        res->report = solver->report();
        if (prefault.joinable()) prefault.join();
        // the iterate is complex128 on the device: no rounding on the way out
        d2h_staged(res->u.a.data.data(), solver->u(), res->u.a.data.size() * sizeof(double2), sg.s);
      }
      mlrg::prof::HostSpan span("host:e2e_solver_teardown");
      solver.reset();
    }
    res->audit = eng->audit_log();
    {
      mlrg::prof::HostSpan span("host:e2e_engine_teardown");
      eng.reset();
      d = mlrg::DeviceBuffer<float2>();
      ref = mlrg::DeviceBuffer<float2>();
    }
    return res.release();
  });
}

const mlr_array* mlr_result_volume(const mlr_result* r) {
  if (r == nullptr) {
    t_error = "null result";
    return nullptr;
  }
  return &r->u;
}

char* mlr_result_csv(const mlr_result* r) {
  return guarded_ptr<char>([&] {
    need(r != nullptr, "null result");
    return dup_text(r->report.csv());
  });
}

int mlr_result_aborted(const mlr_result* r) { return (r != nullptr && r->report.aborted) ? 1 : 0; }

char* mlr_result_abort_reason(const mlr_result* r) {
  return guarded_ptr<char>([&] {
    need(r != nullptr, "null result");
    return dup_text(r->report.abort_reason);
  });
}

void mlr_result_free(mlr_result* r) { delete r; }

mlr_server* mlr_server_start(const char*, int, int, int, int) {
  t_error = "mlr_server_start: the B200 build keeps the memo store in HBM; no TCP memo node is provided";
  return nullptr;
}
int mlr_server_port(const mlr_server*) {
  t_error = "mlr_server_port: no memo server in the B200 build";
  return -1;
}
void mlr_server_stop(mlr_server* s) { delete s; }

// ADMM-Offload planner (capi.cpp:344-380; offload_plan.cpp)
char* mlr_plan_offload(const char* trace_text, double bandwidth, const char* format) {
  return guarded_ptr<char>([&] {
    need(trace_text != nullptr, "trace text is null");
    return dup_text(mlrg::offload::plan_text(trace_text, bandwidth, format != nullptr ? format : "plan"));
  });
}
char* mlr_lru_baseline(const char* trace_text, double bandwidth, uint64_t budget_bytes) {
  return guarded_ptr<char>([&] {
    need(trace_text != nullptr, "trace text is null");
    return dup_text(mlrg::offload::lru_text(trace_text, bandwidth, budget_bytes));
  });
}
char* mlr_train_encoder(const mlr_config*, const char*, uint64_t, const char*) {
  t_error = "mlr_train_encoder: training the CNN encoder is outside the B200 build's scope "
            "(encoder_variant = cnn runs seeded or LENC-file weights)";
  return nullptr;
}

char* mlr_bench(const mlr_config* cfg) {  // capi.cpp:437-499 on the device engine
  return guarded_ptr<char>([&] {
    need(cfg != nullptr, "null config");
    cfg->rc.validate();
    const mlrg::RunConfig& rc = cfg->rc;
    const mlrg::Geometry g = rc.make_geometry();
    StreamGuard sg;
    mlrg::DeviceBuffer<float2> u, out;
    upload_c64(mlrg::make_phantom(g.volume_shape(), "blocks", 42), u, sg.s);
    out.resize(static_cast<std::size_t>(g.mid_shape().count()));
    using clock = std::chrono::steady_clock;
    auto timed = [&](auto&& fn) {
      const auto t0 = clock::now();
      fn();
      MLRG_CUDA(cudaStreamSynchronize(sg.s));
      return std::chrono::duration<double, std::milli>(clock::now() - t0).count();
    };
    mlrg::EngineConfig off = rc.engine;
    off.memo_enabled = false;
    mlrg::Engine plain(g, off, sg.s);
    const double ms_compute = timed([&] { plain.fu1d(u.get(), out.get()); });
    mlrg::EngineConfig on = rc.engine;
    on.memo_enabled = true;
    {  // one fu1d call per window: a ring of one call's slabs + one
      const std::int64_t e = on.chunk_extent;
      const std::int64_t slab = std::max({e * g.h * g.n2, e * g.n0 * g.n2, g.n_theta * e * g.w, g.n1 * e * g.n2});
      on.memo_window_inserts = static_cast<int>((std::max(g.n1, g.h) + e - 1) / e);
      on.memo_arena_bytes = static_cast<std::size_t>(on.memo_window_inserts + 1) *
                            mlrg::ValueRing::granule(static_cast<std::size_t>(slab) * sizeof(float2));
    }
    auto store = std::make_shared<mlrg::MemoStore>();
    auto enc = std::make_shared<mlrg::Encoder>(rc.encoder.key_dim, rc.encoder.seed);
    auto c_miss = std::make_shared<mlrg::MemoClient>(rc.memo, store);
    mlrg::Engine e_miss(g, on, sg.s, enc, c_miss);
    const double ms_miss = timed([&] { e_miss.fu1d(u.get(), out.get()); });
    e_miss.flush_inserts();
    const mlrg::MemoCounters s_miss = c_miss->counters();
    auto c_hit = std::make_shared<mlrg::MemoClient>(rc.memo, store);
    mlrg::Engine e_hit(g, on, sg.s, enc, c_hit);
    const double ms_remote = timed([&] { e_hit.fu1d(u.get(), out.get()); });
    const mlrg::MemoCounters s_remote = c_hit->counters();
    const double ms_cache = timed([&] { e_hit.fu1d(u.get(), out.get()); });
    const mlrg::MemoCounters s_cache = c_hit->counters();
    std::ostringstream o;
    o << "case,lookups,misses,remote_hits,cache_hits,ms\n"
      << "compute,0,0,0,0," << ms_compute << '\n'
      << "miss," << s_miss.lookups << ',' << s_miss.misses << ',' << s_miss.remote_hits << ',' << s_miss.cache_hits
      << ',' << ms_miss << '\n'
      << "service_hit," << s_remote.lookups << ',' << s_remote.misses << ',' << s_remote.remote_hits << ','
      << s_remote.cache_hits << ',' << ms_remote << '\n'
      << "cache_hit," << (s_cache.lookups - s_remote.lookups) << ',' << (s_cache.misses - s_remote.misses) << ','
      << (s_cache.remote_hits - s_remote.remote_hits) << ',' << (s_cache.cache_hits - s_remote.cache_hits) << ','
      << ms_cache << '\n';
    return dup_text(o.str());
  });
}

// ============================== mlrg.h ==============================

const char* mlrg_last_error(void) { return t_error.c_str(); }
void mlrg_free(char* text) { std::free(text); }
int mlrg_version(void) { return 1; }

mlrg_ctx* mlrg_ctx_create_kernel(int64_t n1, int64_t n0, int64_t n2, int64_t n_theta, int64_t h, int64_t w,
                                 double phi, void* stream, int kernel) {
  return guarded_ptr<mlrg_ctx>([&] {
    need(kernel == 0 || kernel == 1, "kernel must be 0 (es) or 1 (gaussian)");
    auto c = std::make_unique<mlrg_ctx>();
    c->g = mlrg::Geometry::make(n1, n0, n2, n_theta, h, w, phi);
    c->s = static_cast<cudaStream_t>(stream);  // NULL: the legacy default stream
    c->usfft = std::make_unique<mlrg::Usfft>(c->g, c->s, static_cast<mlrg::GridKernel>(kernel));
    return c.release();
  });
}

mlrg_ctx* mlrg_ctx_create(int64_t n1, int64_t n0, int64_t n2, int64_t n_theta, int64_t h, int64_t w, double phi,
                          void* stream) {
  return mlrg_ctx_create_kernel(n1, n0, n2, n_theta, h, w, phi, stream, 0);
}

void mlrg_ctx_destroy(mlrg_ctx* ctx) { delete ctx; }

int mlrg_ctx_stats(mlrg_ctx* ctx, int64_t out[6]) {
  return guarded([&] {
    need(ctx && out, "null argument");
    const mlrg::Usfft::Stats st = ctx->usfft->stats();
    const int64_t v[6] = {st.nclass, st.taps, st.m1, st.m2, st.gather_ctas, st.classes_per_cta};
    std::memcpy(out, v, sizeof(v));
  });
}

int mlrg_sync(mlrg_ctx* ctx) {
  return guarded([&] {
    need(ctx != nullptr, "null context");
    MLRG_CUDA(cudaStreamSynchronize(ctx->s));
  });
}

int mlrg_fu1d(mlrg_ctx* ctx, const void* u, void* out, int64_t d0) {
  return guarded([&] {
    need(ctx && u && out && d0 >= 1, "mlrg_fu1d: bad argument");
    ctx->usfft->fu1d(static_cast<const float2*>(u), static_cast<float2*>(out), d0);
  });
}

int mlrg_fu1d_adj(mlrg_ctx* ctx, const void* v, void* out, int64_t d0) {
  return guarded([&] {
    need(ctx && v && out && d0 >= 1, "mlrg_fu1d_adj: bad argument");
    ctx->usfft->fu1d_adj(static_cast<const float2*>(v), static_cast<float2*>(out), d0);
  });
}

int mlrg_fu2d(mlrg_ctx* ctx, const void* v, const void* d_hat, void* out, int64_t d1) {
  return guarded([&] {
    need(ctx && v && out && d1 >= 1, "mlrg_fu2d: bad argument");
    mlrg::Fu2dEpilogue e;
    e.out = static_cast<float2*>(out);
    e.ld_out = d1;
    e.sub = static_cast<const float2*>(d_hat);
    e.ld_sub = d1;
    ctx->usfft->fu2d(static_cast<const float2*>(v), d1, 0, d1, e);
  });
}

int mlrg_fu2d_adj(mlrg_ctx* ctx, const void* p, void* out, int64_t d1) {
  return guarded([&] {
    need(ctx && p && out && d1 >= 1, "mlrg_fu2d_adj: bad argument");
    ctx->usfft->fu2d_adj(static_cast<const float2*>(p), d1, 0, d1, static_cast<float2*>(out), d1, 0);
  });
}

int mlrg_f2d(mlrg_ctx* ctx, const void* p, void* out, int64_t d0, int adjoint) {
  return guarded([&] {
    need(ctx && p && out && d0 >= 1, "mlrg_f2d: bad argument");
    ctx->usfft->f2d(static_cast<const float2*>(p), static_cast<float2*>(out), d0, adjoint != 0);
  });
}

int mlrg_forward_L(mlrg_ctx* ctx, const void* u, void* out) {
  return guarded([&] {
    need(ctx && u && out, "mlrg_forward_L: bad argument");
    forward_L(*ctx->usfft, static_cast<const float2*>(u), static_cast<float2*>(out), ctx->scratch_mid,
              ctx->scratch_proj);
  });
}

int mlrg_adjoint_L(mlrg_ctx* ctx, const void* d, void* out) {
  return guarded([&] {
    need(ctx && d && out, "mlrg_adjoint_L: bad argument");
    adjoint_L(*ctx->usfft, static_cast<const float2*>(d), static_cast<float2*>(out), ctx->scratch_mid,
              ctx->scratch_proj);
  });
}

int mlrg_grad(mlrg_ctx* ctx, const void* u, void* g0, void* g1, void* g2) {
  return guarded([&] {
    need(ctx && u && g0 && g1 && g2, "mlrg_grad: bad argument");
    mlrg::Field3 f{{static_cast<float2*>(g0), static_cast<float2*>(g1), static_cast<float2*>(g2)}};
    mlrg::ops::grad(static_cast<const float2*>(u), f, {ctx->g.n1, ctx->g.n0, ctx->g.n2}, ctx->s);
  });
}

int mlrg_div(mlrg_ctx* ctx, const void* g0, const void* g1, const void* g2, void* out) {
  return guarded([&] {
    need(ctx && g0 && g1 && g2 && out, "mlrg_div: bad argument");
    mlrg::CField3 f;
    f.c[0] = static_cast<const float2*>(g0);
    f.c[1] = static_cast<const float2*>(g1);
    f.c[2] = static_cast<const float2*>(g2);
    mlrg::ops::div(f, static_cast<float2*>(out), {ctx->g.n1, ctx->g.n0, ctx->g.n2}, ctx->s);
  });
}

int mlrg_cnn_weights(int key_dim, uint64_t seed, float* c1w, float* c2w, float* fcw) {
  return guarded([&] {
    need(c1w && c2w && fcw && key_dim >= 2, "mlrg_cnn_weights: bad argument");
    const mlrg::CnnWeights w = mlrg::CnnWeights::init(key_dim, seed);
    std::memcpy(c1w, w.c1w.data(), w.c1w.size() * sizeof(float));
    std::memcpy(c2w, w.c2w.data(), w.c2w.size() * sizeof(float));
    std::memcpy(fcw, w.fcw.data(), w.fcw.size() * sizeof(float));
  });
}

int mlrg_encode_cnn(mlrg_ctx* ctx, int op, const void* x, int64_t chunk_extent, int key_dim, uint64_t seed,
                    float* keys, double* norms, int64_t n_slabs) {
  return guarded([&] {
    need(ctx && x && keys && norms && op >= 0 && op <= 5 && chunk_extent >= 1, "mlrg_encode_cnn: bad argument");
    const mlrg::OpId oid = static_cast<mlrg::OpId>(op);
    const mlrg::Geometry& g = ctx->g;
    const mlrg::Shape3 in = oid == mlrg::OpId::fu1d ? g.volume_shape()
                            : (oid == mlrg::OpId::fu1d_adj || oid == mlrg::OpId::fu2d) ? g.mid_shape()
                                                                                         : g.projection_shape();
    const int axis = mlrg::chunk_axis_of(oid);
    const int64_t len = in.extent(axis);
    const int64_t ns = (len + chunk_extent - 1) / chunk_extent;
    need(n_slabs == ns, "mlrg_encode_cnn: n_slabs does not match the slab count");
    mlrg::Encoder enc(mlrg::CnnWeights::init(key_dim, seed), seed, ctx->s);
    mlrg::ops::CnnWork work;
    mlrg::DeviceBuffer<float> dkeys(static_cast<std::size_t>(ns * key_dim));
    mlrg::DeviceBuffer<double> dnorm(static_cast<std::size_t>(ns));
    for (int64_t c0 = 0; c0 < ns;) {
      const int64_t e = std::min(chunk_extent, len - c0 * chunk_extent);
      int64_t c1 = c0;
      while (c1 < ns && std::min(chunk_extent, len - c1 * chunk_extent) == e) ++c1;
      std::vector<int64_t> starts;
      for (int64_t c = c0; c < c1; ++c) starts.push_back(c * chunk_extent);
      mlrg::ops::encode_cnn(static_cast<const float2*>(x), {in.d0, in.d1, in.d2, axis, 0, e}, starts.data(),
                            static_cast<int>(c1 - c0), enc.cnn_device(), dkeys.get() + c0 * key_dim, dnorm.get() + c0,
                            work, ctx->s);
      c0 = c1;
    }
    MLRG_CUDA(cudaStreamSynchronize(ctx->s));
    MLRG_CUDA(cudaMemcpy(keys, dkeys.get(), sizeof(float) * ns * key_dim, cudaMemcpyDeviceToHost));
    MLRG_CUDA(cudaMemcpy(norms, dnorm.get(), sizeof(double) * ns, cudaMemcpyDeviceToHost));
    for (int64_t c = 0; c < ns; ++c) norms[c] = std::sqrt(norms[c]);  // keys stay raw (before slot_mix)
  });
}

int mlrg_encode(mlrg_ctx* ctx, int op, const void* x, int64_t chunk_extent, int key_dim, uint64_t seed,
                float* keys, double* norms, int64_t n_slabs) {
  return guarded([&] {
    need(ctx && x && keys && norms && op >= 0 && op <= 5 && chunk_extent >= 1, "mlrg_encode: bad argument");
    const mlrg::OpId oid = static_cast<mlrg::OpId>(op);
    const mlrg::Geometry& g = ctx->g;
    const mlrg::Shape3 in = oid == mlrg::OpId::fu1d ? g.volume_shape()
                            : (oid == mlrg::OpId::fu1d_adj || oid == mlrg::OpId::fu2d) ? g.mid_shape()
                                                                                         : g.projection_shape();
    const int axis = mlrg::chunk_axis_of(oid);
    const int64_t len = in.extent(axis);
    const int64_t ns = (len + chunk_extent - 1) / chunk_extent;
    need(n_slabs == ns, "mlrg_encode: n_slabs does not match the slab count");
    mlrg::Encoder enc(key_dim, seed);
    mlrg::DeviceBuffer<float> dkeys(static_cast<std::size_t>(ns * key_dim));
    mlrg::DeviceBuffer<double> dnorm(static_cast<std::size_t>(ns));
    for (int64_t c0 = 0; c0 < ns;) {
      const int64_t e = std::min(chunk_extent, len - c0 * chunk_extent);
      int64_t c1 = c0;
      while (c1 < ns && std::min(chunk_extent, len - c1 * chunk_extent) == e) ++c1;
      mlrg::Shape3 sh = in;
      (axis == 0 ? sh.d0 : sh.d1) = e;
      enc.register_shape(sh, ctx->s);
      std::vector<int64_t> starts;
      for (int64_t c = c0; c < c1; ++c) starts.push_back(c * chunk_extent);
      mlrg::DeviceBuffer<double> work(mlrg::ops::encode_work_doubles(static_cast<int>(c1 - c0), key_dim));
      mlrg::ops::encode(static_cast<const float2*>(x), {in.d0, in.d1, in.d2, axis, 0, e}, starts.data(),
                        static_cast<int>(c1 - c0), enc.device_matrix(sh), key_dim, work.get(),
                        dkeys.get() + c0 * key_dim, dnorm.get() + c0, ctx->s);
      MLRG_CUDA(cudaStreamSynchronize(ctx->s));
      c0 = c1;
    }
    MLRG_CUDA(cudaMemcpy(keys, dkeys.get(), sizeof(float) * ns * key_dim, cudaMemcpyDeviceToHost));
    MLRG_CUDA(cudaMemcpy(norms, dnorm.get(), sizeof(double) * ns, cudaMemcpyDeviceToHost));
    for (int64_t c = 0; c < ns; ++c) {
      mlrg::slot_mix(keys + c * key_dim, key_dim, seed, c, oid);
      norms[c] = std::sqrt(norms[c]);
    }
  });
}

mlrg_recon* mlrg_reconstruct(const char* config_text, const void* d, const void* reference, void* u_out,
                             void* stream) {
  return guarded_ptr<mlrg_recon>([&] {
    need(config_text && d && u_out, "mlrg_reconstruct: bad argument");
    const mlrg::RunConfig rc = mlrg::RunConfig::from_text(config_text);
    rc.validate();
    const mlrg::Geometry g = rc.make_geometry();
    cudaStream_t s = static_cast<cudaStream_t>(stream);  // NULL: the legacy default stream
    std::unique_ptr<mlrg::Engine> eng = build_engine(rc, g, s);
    auto r = std::make_unique<mlrg_recon>();
    r->report = mlrg::reconstruct(static_cast<const float2*>(d), rc.admm, *eng,
                                  static_cast<const float2*>(reference), static_cast<float2*>(u_out));
    r->audit = eng->audit_log();
    if (eng->memo()) r->counters = eng->memo()->counters();
    r->tiers[0] = eng->memo_arena_bytes();
    r->tiers[1] = static_cast<uint64_t>(eng->spilled_values());
    r->tiers[2] = eng->spilled_bytes();
    return r.release();
  });
}

char* mlrg_recon_csv(const mlrg_recon* r) {
  return guarded_ptr<char>([&] {
    need(r != nullptr, "null result");
    return dup_text(r->report.csv());
  });
}
int mlrg_recon_aborted(const mlrg_recon* r) { return (r && r->report.aborted) ? 1 : 0; }
char* mlrg_recon_abort_reason(const mlrg_recon* r) {
  return guarded_ptr<char>([&] {
    need(r != nullptr, "null result");
    return dup_text(r->report.abort_reason);
  });
}
int64_t mlrg_recon_audit(const mlrg_recon* r, int32_t* meta4, float* cs, int64_t cap) {
  if (!r) return -1;
  return copy_audit(r->audit, meta4, cs, cap);
}
int mlrg_recon_counters(const mlrg_recon* r, uint64_t out[11]) {
  return guarded([&] {
    need(r && out, "null argument");
    fill_counters(r->counters, out);
  });
}
int mlrg_recon_tiers(const mlrg_recon* r, uint64_t out[3]) {
  return guarded([&] {
    need(r && out, "null argument");
    std::copy(r->tiers, r->tiers + 3, out);
  });
}
void mlrg_recon_free(mlrg_recon* r) { delete r; }

mlrg_solver* mlrg_solver_new(const char* config_text, const void* d, const void* reference, void* stream) {
  return mlrg_solver_new_sharded(config_text, d, reference, stream, nullptr);
}

mlrg_solver* mlrg_solver_new_sharded(const char* config_text, const void* d, const void* reference, void* stream,
                                     mlrg_comm* comm) {
  return guarded_ptr<mlrg_solver>([&] {
    need(config_text && d, "mlrg_solver_new: bad argument");
    const mlrg::RunConfig rc = mlrg::RunConfig::from_text(config_text);
    rc.validate();
    const mlrg::Geometry g = rc.make_geometry();
    auto sv = std::make_unique<mlrg_solver>();
    cudaStream_t s = static_cast<cudaStream_t>(stream);  // NULL: the legacy default stream
    sv->eng = build_engine(rc, g, s, comm ? comm->c : nullptr);
    sv->solver = std::make_unique<mlrg::Solver>(static_cast<const float2*>(d), rc.admm, *sv->eng,
                                                static_cast<const float2*>(reference));
    MLRG_CUDA(cudaStreamSynchronize(s));
    return sv.release();
  });
}

int mlrg_solver_shard(const mlrg_solver* s, int64_t out[4]) {
  return guarded([&] {
    need(s && out, "null argument");
    const mlrg::Shard& sh = s->eng->shard();
    out[0] = sh.a();
    out[1] = sh.b();
    out[2] = sh.c();
    out[3] = sh.d();
  });
}

int mlrg_solver_step(mlrg_solver* s, int* aborted) {
  return guarded([&] {
    need(s != nullptr, "null solver");
    bool ok = false;
    try {
      ok = s->solver->step();
    } catch (...) {  // sharded: release the peers blocked in a collective
      if (s->eng->shard().comm) s->eng->shard().comm->abort();
      throw;
    }
    MLRG_CUDA(cudaStreamSynchronize(s->eng->stream()));
    if (aborted) *aborted = ok ? 0 : 1;
  });
}

int mlrg_solver_volume(mlrg_solver* s, void* u_out) {
  return guarded([&] {
    need(s && u_out, "null argument");
    const std::int64_t n = s->eng->shard().np() * s->eng->geometry().n0 * s->eng->geometry().n2;  // this rank's planes
    mlrg::ops::c128_to_c64(s->solver->u(), static_cast<float2*>(u_out), n, s->eng->stream());
    MLRG_CUDA(cudaStreamSynchronize(s->eng->stream()));
  });
}

char* mlrg_solver_csv(const mlrg_solver* s) {
  return guarded_ptr<char>([&] {
    need(s != nullptr, "null solver");
    return dup_text(s->solver->report().csv());
  });
}

int mlrg_solver_counters(const mlrg_solver* s, uint64_t out[11]) {
  return guarded([&] {
    need(s && out, "null argument");
    fill_counters(s->eng->memo() ? s->eng->memo()->counters() : mlrg::MemoCounters{}, out);
  });
}

int mlrg_solver_tiers(const mlrg_solver* s, uint64_t out[3]) {
  return guarded([&] {
    need(s && out, "null argument");
    out[0] = s->eng->memo_arena_bytes();
    out[1] = static_cast<uint64_t>(s->eng->spilled_values());
    out[2] = s->eng->spilled_bytes();
  });
}

int64_t mlrg_solver_audit(const mlrg_solver* s, int32_t* meta4, float* cs, int64_t cap) {
  if (!s) return -1;
  return copy_audit(s->eng->audit_log(), meta4, cs, cap);
}

void mlrg_solver_free(mlrg_solver* s) { delete s; }

int64_t mlrg_result_audit(const struct mlr_result* r, int32_t* meta4, float* cs, int64_t cap) {
  if (!r) return -1;
  return copy_audit(r->audit, meta4, cs, cap);
}

mlrg_memo* mlrg_memo_new(float tau, int nprobe, uint64_t insert_cap, uint64_t coalesce_bytes, int global_cache,
                         int nlist, int train_size) {
  return guarded_ptr<mlrg_memo>([&] {
    mlrg::IvfConfig ic;
    ic.nlist = nlist;
    ic.train_size = train_size;
    ic.nprobe = nprobe;
    mlrg::MemoClientConfig mc;
    mc.tau = tau;
    mc.nprobe = nprobe;
    mc.insert_queue_cap = insert_cap;
    mc.coalesce_bytes = coalesce_bytes;
    mc.global_cache = global_cache != 0;
    auto m = std::make_unique<mlrg_memo>();
    m->store = std::make_shared<mlrg::MemoStore>(ic);
    m->client = std::make_unique<mlrg::MemoClient>(mc, m->store);
    return m.release();
  });
}

void mlrg_memo_free(mlrg_memo* m) { delete m; }

int mlrg_memo_lookup(mlrg_memo* m, int64_t n, int key_dim, const float* keys, const int64_t* locations,
                     const int32_t* ops, const uint64_t* value_bytes, int32_t* outcome, float* cs,
                     uint64_t* value_id) {
  return guarded([&] {
    need(m && keys && locations && ops && value_bytes && outcome && cs && value_id, "null argument");
    std::vector<mlrg::MemoKey> ks(static_cast<std::size_t>(n));
    std::vector<std::size_t> vb(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      ks[static_cast<std::size_t>(i)].values.assign(keys + i * key_dim, keys + (i + 1) * key_dim);
      ks[static_cast<std::size_t>(i)].location = locations[i];
      ks[static_cast<std::size_t>(i)].op = static_cast<mlrg::OpId>(ops[i]);
      vb[static_cast<std::size_t>(i)] = value_bytes[i];
    }
    const std::vector<mlrg::MemoDecision> d = m->client->lookup_batch(ks, vb);
    for (int64_t i = 0; i < n; ++i) {
      outcome[i] = static_cast<int32_t>(d[static_cast<std::size_t>(i)].outcome);
      cs[i] = d[static_cast<std::size_t>(i)].cs;
      value_id[i] = d[static_cast<std::size_t>(i)].value_id;
    }
  });
}

int mlrg_memo_insert(mlrg_memo* m, int key_dim, const float* key, uint64_t value_bytes) {
  try {
    need(m && key, "null argument");
    mlrg::MemoKey k;
    k.values.assign(key, key + key_dim);
    const bool staged = m->client->insert_async(k, [&] {
      mlrg::ValueRef v;
      v.bytes = value_bytes;
      return v;
    });
    return staged ? 1 : 0;
  } catch (const std::exception& e) {
    t_error = e.what();
    return -code_for(e);
  }
}

int mlrg_memo_flush(mlrg_memo* m) {
  return guarded([&] {
    need(m != nullptr, "null memo");
    m->client->flush_inserts();
  });
}

int mlrg_memo_counters(const mlrg_memo* m, uint64_t out[11]) {
  return guarded([&] {
    need(m && out, "null argument");
    fill_counters(m->client->counters(), out);
  });
}

int mlrg_kmeans(const float* keys, int64_t nk, int dim, int k, uint64_t seed, int iters, int on_device,
                float* centroids, int64_t* nearest) {
  return guarded([&] {
    need(keys && centroids && nearest && nk > 0 && dim > 0 && k > 0, "null or empty argument");
    std::vector<std::vector<float>> kv(static_cast<std::size_t>(nk));
    for (int64_t i = 0; i < nk; ++i) kv[static_cast<std::size_t>(i)].assign(keys + i * dim, keys + (i + 1) * dim);
    std::vector<std::vector<float>> cent;
    std::vector<std::size_t> near(static_cast<std::size_t>(nk));
    if (on_device) {
      int dev = 0;
      MLRG_CUDA(cudaGetDevice(&dev));
      need(mlrg::gpu_kmeans_fits(static_cast<int>(nk), k, dim), "kmeans: too many keys for the device trainer");
      mlrg::gpu_kmeans(kv, k, seed, iters, cent, near, dev);
    } else {
      cent = mlrg::kmeans_train(kv, k, seed, iters);
      for (std::size_t i = 0; i < kv.size(); ++i) {
        double best = std::numeric_limits<double>::max();
        for (std::size_t c = 0; c < cent.size(); ++c) {
          const double d = mlrg::l2_sq(kv[i].data(), cent[c].data(), dim);
          if (d < best) {
            best = d;
            near[i] = c;
          }
        }
      }
    }
    for (std::size_t c = 0; c < cent.size(); ++c)
      std::memcpy(centroids + c * static_cast<std::size_t>(dim), cent[c].data(), sizeof(float) * static_cast<std::size_t>(dim));
    for (std::size_t i = 0; i < near.size(); ++i) nearest[i] = static_cast<int64_t>(near[i]);
  });
}

int mlrg_projection_matrix(int64_t d0, int64_t d1, int64_t d2, int key_dim, uint64_t seed, float* out,
                           int64_t count) {
  return guarded([&] {
    need(out != nullptr && count >= 0, "null argument");
    const std::vector<float> m = mlrg::projection_matrix({d0, d1, d2}, key_dim, seed);
    need(count <= static_cast<int64_t>(m.size()), "count exceeds the matrix size");
    std::memcpy(out, m.data(), static_cast<std::size_t>(count) * sizeof(float));
  });
}

int mlrg_slot_mix(float* key, int key_dim, uint64_t seed, int64_t location, int op) {
  return guarded([&] {
    need(key != nullptr, "null key");
    mlrg::slot_mix(key, key_dim, seed, location, static_cast<mlrg::OpId>(op));
  });
}

/* ---- node-local communicator and partition (sharded solver) ---- */

mlrg_comm* mlrg_comm_create(const char* name, int rank, int world, double timeout_s) {
  return guarded_ptr<mlrg_comm>([&] {
    need(name && *name, "mlrg_comm_create: empty name");
    auto c = std::make_unique<mlrg_comm>();
    c->c = std::make_shared<mlrg::HostComm>(name, rank, world, timeout_s > 0 ? timeout_s : 120.0);
    return c.release();
  });
}

void mlrg_comm_free(mlrg_comm* c) { delete c; }

int mlrg_comm_barrier(mlrg_comm* c) {
  return guarded([&] {
    need(c != nullptr, "null comm");
    c->c->barrier();
  });
}

int mlrg_comm_abort(mlrg_comm* c) {
  return guarded([&] {
    need(c != nullptr, "null comm");
    c->c->abort();
  });
}

int mlrg_comm_allreduce(mlrg_comm* c, double* v, int n) {
  return guarded([&] {
    need(c && (v || n == 0), "null argument");
    c->c->allreduce_sum(v, n);
  });
}

int mlrg_comm_allgather(mlrg_comm* c, const void* in, uint64_t bytes, void* out) {
  return guarded([&] {
    need(c && in && out, "null argument");
    c->c->allgather(in, static_cast<std::size_t>(bytes), out);
  });
}

int mlrg_partition(int64_t n1, int64_t h, int64_t chunk, int world, int64_t* out) {
  return guarded([&] {
    need(out != nullptr && world >= 1 && chunk > 0, "mlrg_partition: bad argument");
    mlrg::Geometry g;
    g.n1 = n1;
    g.h = h;
    mlrg::Shard sh = mlrg::Shard::whole(g, chunk);
    if (world > 1) {
      // the same assign() split Shard::make uses, without a communicator
      auto ranges = [&](std::int64_t len) {
        const std::int64_t ns = (len + chunk - 1) / chunk;
        if (ns < world) throw std::invalid_argument("mlrg_partition: fewer slabs than ranks");
        auto r = mlrg::assign_ranges(ns, world);
        for (auto& [lo, hi] : r) {
          lo = std::min(len, lo * chunk);
          hi = std::min(len, hi * chunk);
        }
        return r;
      };
      sh.planes = ranges(n1);
      sh.rows = ranges(h);
    }
    for (int r = 0; r < world; ++r) {
      out[4 * r + 0] = sh.planes[static_cast<std::size_t>(r)].first;
      out[4 * r + 1] = sh.planes[static_cast<std::size_t>(r)].second;
      out[4 * r + 2] = sh.rows[static_cast<std::size_t>(r)].first;
      out[4 * r + 3] = sh.rows[static_cast<std::size_t>(r)].second;
    }
  });
}

}  // extern "C"
