// Golden-fixture generator for the parity tests. TEST INFRASTRUCTURE ONLY:
// it links the unmodified CPU reference (oracle/_ref/libmlr_core.a, built by
// oracle/Makefile from /root/reference/proj/src) and dumps its outputs as .npy
// files. Nothing in the product links or runs this.
//
//   golden_gen ops    <dir> n1 n0 n2 n_theta h w seed   per-operator in/out
//   golden_gen recon  <dir> N n_theta n_outer memo path [workers]
//   golden_gen encoder <dir>                           P prefix + keys
//   golden_gen store  <dir>                            MemoStore KATs
//   golden_gen data   <dir> N n_theta workers random   d (+ phantom) of a large case
//   golden_gen recon_big <dir> N n_theta n_outer memo workers random samples
//
// Inputs that feed a reconstruction are rounded to complex64 first so that
// the fp32 device path and the f64 reference see bit-identical data.
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <unordered_set>
#include <vector>
#include <algorithm>

#include "mlr/admm.hpp"
#include "mlr/config.hpp"
#include "mlr/encoder.hpp"
#include "mlr/memostore.hpp"
#include "mlr/operators.hpp"
#include "mlr/phantom.hpp"
#include "mlr/scalerun.hpp"

using mlr::cplx;

namespace {

template <class T> const char* descr();
template <> const char* descr<cplx>() { return "<c16"; }
template <> const char* descr<std::complex<float>>() { return "<c8"; }
template <> const char* descr<double>() { return "<f8"; }
template <> const char* descr<float>() { return "<f4"; }
template <> const char* descr<std::int32_t>() { return "<i4"; }
template <> const char* descr<std::int64_t>() { return "<i8"; }

template <class T>
void save_npy(const std::string& path, const T* data, std::vector<std::int64_t> shape) {
  std::ostringstream h;
  h << "{'descr': '" << descr<T>() << "', 'fortran_order': False, 'shape': (";
  std::size_t count = 1;
  for (std::size_t i = 0; i < shape.size(); ++i) {
    h << shape[i] << (shape.size() == 1 ? "," : (i + 1 < shape.size() ? ", " : ""));
    count *= static_cast<std::size_t>(shape[i]);
  }
  h << "), }";
  std::string hs = h.str();
  const std::size_t total = 10 + hs.size() + 1;
  hs.append((64 - total % 64) % 64, ' ');
  hs.push_back('\n');
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot write " + path);
  f.write("\x93NUMPY\x01\x00", 8);
  const std::uint16_t hl = static_cast<std::uint16_t>(hs.size());
  f.write(reinterpret_cast<const char*>(&hl), 2);
  f.write(hs.data(), static_cast<std::streamsize>(hs.size()));
  f.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(count * sizeof(T)));
}

void save_arr(const std::string& path, const mlr::Array3& a) {
  const auto s = a.shape();
  save_npy(path, a.data(), {s.d0, s.d1, s.d2});
}

void save_c64(const std::string& path, const mlr::Array3& a) {
  std::vector<std::complex<float>> v(static_cast<std::size_t>(a.size()));
  for (std::size_t i = 0; i < v.size(); ++i)
    v[i] = std::complex<float>(static_cast<float>(a.data()[i].real()),
                               static_cast<float>(a.data()[i].imag()));
  const auto s = a.shape();
  save_npy(path, v.data(), {s.d0, s.d1, s.d2});
}

void save_text(const std::string& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary);
  f << text;
}

mlr::Array3 round_c64(mlr::Array3 a) {
  for (cplx& v : a.flat())
    v = cplx(static_cast<double>(static_cast<float>(v.real())),
             static_cast<double>(static_cast<float>(v.imag())));
  return a;
}

mlr::Array3 random_array(mlr::Shape3 s, mlr::Domain dom, std::mt19937_64& rng) {
  mlr::Array3 a(s, dom);
  for (cplx& v : a.flat()) {
    const double re = (static_cast<double>(rng() >> 11) * 0x1.0p-53) * 2.0 - 1.0;
    const double im = (static_cast<double>(rng() >> 11) * 0x1.0p-53) * 2.0 - 1.0;
    v = cplx(re, im);
  }
  return round_c64(a);
}

int cmd_ops(const std::string& dir, std::int64_t n1, std::int64_t n0, std::int64_t n2,
            std::int64_t nt, std::int64_t h, std::int64_t w, std::uint64_t seed) {
  const mlr::Geometry g = mlr::Geometry::make(n1, n0, n2, nt, h, w, 0.5235987755982988);
  std::mt19937_64 rng(seed);
  const mlr::Array3 u = random_array(g.volume_shape(), mlr::Domain::space, rng);
  const mlr::Array3 mid = random_array(g.mid_shape(), mlr::Domain::space, rng);
  const mlr::Array3 pf = random_array(g.projection_shape(), mlr::Domain::frequency, rng);
  const mlr::Array3 ps = random_array(g.projection_shape(), mlr::Domain::space, rng);
  const mlr::Array3 dh = random_array(g.projection_shape(), mlr::Domain::frequency, rng);
  save_arr(dir + "/in_u.npy", u);
  save_arr(dir + "/in_mid.npy", mid);
  save_arr(dir + "/in_projf.npy", pf);
  save_arr(dir + "/in_projs.npy", ps);
  save_arr(dir + "/in_dhat.npy", dh);
  for (auto path : {mlr::NudftPath::gridding, mlr::NudftPath::direct}) {
    const std::string sfx = path == mlr::NudftPath::gridding ? "_grid" : "_direct";
    save_arr(dir + "/fu1d" + sfx + ".npy", mlr::fu1d(u, g, path));
    save_arr(dir + "/fu1d_adj" + sfx + ".npy", mlr::fu1d_adj(mid, g, path));
    save_arr(dir + "/fu2d" + sfx + ".npy", mlr::fu2d(mid, g, path));
    save_arr(dir + "/fu2d_adj" + sfx + ".npy", mlr::fu2d_adj(pf, g, path));
    save_arr(dir + "/fused" + sfx + ".npy", mlr::fused_sub_fu2d(mid, dh, g, path));
    save_arr(dir + "/forward_L" + sfx + ".npy", mlr::forward_L(u, g, path));
    save_arr(dir + "/adjoint_L" + sfx + ".npy", mlr::adjoint_L(ps, g, path));
  }
  save_arr(dir + "/f2d.npy", mlr::f2d(ps));
  save_arr(dir + "/f2d_adj.npy", mlr::f2d_adj(pf));
  const mlr::GradField gr = mlr::grad(u);
  for (int ax = 0; ax < 3; ++ax) save_arr(dir + "/grad" + std::to_string(ax) + ".npy", gr.comp[ax]);
  mlr::GradField gf;
  for (int ax = 0; ax < 3; ++ax) gf.comp[ax] = random_array(g.volume_shape(), mlr::Domain::space, rng);
  for (int ax = 0; ax < 3; ++ax) save_arr(dir + "/in_g" + std::to_string(ax) + ".npy", gf.comp[ax]);
  save_arr(dir + "/div.npy", mlr::div(gf));
  std::ostringstream geo;
  geo << "n1=" << n1 << "\nn0=" << n0 << "\nn2=" << n2 << "\nn_theta=" << nt << "\nh=" << h
      << "\nw=" << w << "\nphi=0.5235987755982988\nseed=" << seed << "\n";
  save_text(dir + "/geometry.txt", geo.str());
  return 0;
}

int cmd_recon(const std::string& dir, std::int64_t n, std::int64_t nt, int n_outer,
              const std::string& memo, const std::string& path, int workers,
              const std::string& variant = "projection", const std::string& pipeline = "optimized") {
  mlr::RunConfig rc;
  rc.set("n1", std::to_string(n));
  rc.set("n0", std::to_string(n));
  rc.set("n2", std::to_string(n));
  rc.set("n_theta", std::to_string(nt));
  rc.set("h", std::to_string(n));
  rc.set("w", std::to_string(n));
  rc.set("n_outer", std::to_string(n_outer));
  rc.set("memoization", memo);
  rc.set("nudft_path", path);
  rc.set("workers", std::to_string(workers));
  rc.set("encoder_variant", variant);
  rc.set("pipeline", pipeline);
  rc.validate();
  const mlr::Geometry geom = rc.make_geometry();
  const mlr::Volume phantom =
      round_c64(mlr::make_phantom(geom.volume_shape(), mlr::PhantomKind::blocks, 1));
  const mlr::ProjectionSet d = round_c64(mlr::forward_L(phantom, geom, rc.engine.path));
  save_c64(dir + "/phantom.npy", phantom);
  save_c64(dir + "/data.npy", d);

  // Same assembly as capi.cpp build_engine (local memo), plus an observer
  // that records every memoizable input chunk's key in lookup order.
  mlr::EngineConfig ecfg = rc.engine;
  ecfg.memo_enabled = rc.admm.memoization != mlr::MemoMode::off;
  std::shared_ptr<mlr::Encoder> enc;
  std::shared_ptr<mlr::MemoClient> client;
  if (ecfg.memo_enabled) {
    mlr::MemoClientConfig mcfg = rc.memo;
    mcfg.endpoint.clear();
    client = std::make_shared<mlr::MemoClient>(mcfg);
    enc = std::make_shared<mlr::Encoder>(rc.encoder);
  }
  mlr::OperatorEngine eng(geom, ecfg, enc, client);
  std::vector<float> keys;
  std::vector<std::int32_t> key_meta;  // (iteration, op, location)
  std::vector<double> in_norms;
  if (ecfg.memo_enabled) {
    eng.set_chunk_observer([&](mlr::OpId op, const mlr::Chunk& c) {
      const mlr::MemoKey k = enc->encode(c.data, c.location.index, op);
      keys.insert(keys.end(), k.values.begin(), k.values.end());
      key_meta.push_back(c.iteration);
      key_meta.push_back(static_cast<std::int32_t>(op));
      key_meta.push_back(static_cast<std::int32_t>(c.location.index));
      in_norms.push_back(mlr::norm2(c.data));
    });
  }
  mlr::ReconResult res = mlr::reconstruct(d, geom, rc.admm, eng, &phantom);
  save_c64(dir + "/u.npy", res.u);
  save_text(dir + "/report.csv", res.report.csv());
  save_text(dir + "/config.txt", rc.str());
  std::ostringstream ab;
  ab << (res.report.aborted ? 1 : 0) << "\n" << res.report.abort_reason << "\n";
  save_text(dir + "/aborted.txt", ab.str());
  if (ecfg.memo_enabled) {
    const std::vector<mlr::ChunkAudit> audit = eng.audit_log();
    std::vector<std::int32_t> a_int;
    std::vector<float> a_cs;
    for (const auto& e : audit) {
      a_int.push_back(e.iteration);
      a_int.push_back(static_cast<std::int32_t>(e.op));
      a_int.push_back(static_cast<std::int32_t>(e.location.index));
      a_int.push_back(static_cast<std::int32_t>(e.outcome));
      a_cs.push_back(e.cs);
    }
    const std::int64_t na = static_cast<std::int64_t>(audit.size());
    save_npy(dir + "/audit_int.npy", a_int.data(), {na, 4});
    save_npy(dir + "/audit_cs.npy", a_cs.data(), {na});
    const std::int64_t nk = static_cast<std::int64_t>(key_meta.size() / 3);
    save_npy(dir + "/keys.npy", keys.data(), {nk, static_cast<std::int64_t>(rc.encoder.key_dim)});
    save_npy(dir + "/key_meta.npy", key_meta.data(), {nk, 3});
    save_npy(dir + "/in_norms.npy", in_norms.data(), {nk});
    const mlr::MemoCounterSnapshot c = client->counters();
    std::ostringstream cs;
    cs << "lookups=" << c.lookups << "\ncache_hits=" << c.cache_hits
       << "\nremote_hits=" << c.remote_hits << "\nmisses=" << c.misses
       << "\ncache_comparisons=" << c.cache_comparisons << "\ncache_probes=" << c.cache_probes
       << "\nbatches_sent=" << c.batches_sent << "\ninserts_enqueued=" << c.inserts_enqueued
       << "\ninserts_sent=" << c.inserts_sent << "\ninserts_dropped=" << c.inserts_dropped
       << "\n";
    save_text(dir + "/counters.txt", cs.str());
  }
  return 0;
}

// The reconstruction input of the large cases: phantom "blocks" seed 1 and
// d = forward_L(phantom) through the reference's OperatorEngine with `workers`
// threads (scalerun.hpp:55-60: bitwise identical to the unchunked operator),
// both rounded to complex64 like cmd_recon. `random` replaces d by uniform
// values in [-1, 1) from mt19937_64(seed 2511) (random_array), for sizes whose
// dense f2d_adj projector (operators.cpp:39-74) is too slow to rerun.
struct BigInput {
  mlr::Volume phantom;
  mlr::ProjectionSet d;
};

BigInput big_input(const mlr::Geometry& geom, int workers, bool random) {
  BigInput in{round_c64(mlr::make_phantom(geom.volume_shape(), mlr::PhantomKind::blocks, 1)), {}};
  if (random) {
    std::mt19937_64 rng(2511);
    in.d = random_array(geom.projection_shape(), mlr::Domain::space, rng);
    return in;
  }
  mlr::EngineConfig ecfg;
  ecfg.path = mlr::NudftPath::gridding;
  ecfg.workers = workers;
  mlr::OperatorEngine eng(geom, ecfg);
  in.d = round_c64(eng.f2d_adj(eng.fu2d(eng.fu1d(in.phantom, false), false), false));
  return in;
}

mlr::RunConfig big_config(std::int64_t n, std::int64_t nt, int n_outer, const std::string& memo, int workers) {
  mlr::RunConfig rc;
  for (const char* k : {"n1", "n0", "n2", "h", "w"}) rc.set(k, std::to_string(n));
  rc.set("n_theta", std::to_string(nt));
  rc.set("n_outer", std::to_string(n_outer));
  rc.set("memoization", memo);
  rc.set("nudft_path", "gridding");
  rc.set("workers", std::to_string(workers));
  rc.validate();
  return rc;
}

// golden_gen data <dir> N n_theta workers random: writes data.npy (complex64)
// and phantom.npy. The GPU parity tests run this on the box to regenerate the
// exact d of a large fixture instead of committing hundreds of MB.
int cmd_data(const std::string& dir, std::int64_t n, std::int64_t nt, int workers, bool random) {
  const mlr::RunConfig rc = big_config(n, nt, 1, "off", workers);
  const BigInput in = big_input(rc.make_geometry(), workers, random);
  save_c64(dir + "/phantom.npy", in.phantom);
  save_c64(dir + "/data.npy", in.d);
  return 0;
}

// Compact reconstruction fixture for sizes whose full arrays cannot be
// committed (configs[1] 256^3 and the configs[2] 512^3 prefix): the CSV report,
// the audit log and counters, ||u||, a checksum of d, and u at `samples`
// voxel indices drawn from mt19937_64(seed 4242) without replacement
// (Floyd's algorithm, sorted), so the test's rel-L2 on the sample estimates the
// full-volume rel-L2 with ~1/sqrt(samples) relative spread.
int cmd_recon_big(const std::string& dir, std::int64_t n, std::int64_t nt, int n_outer,
                  const std::string& memo, int workers, bool random, std::int64_t samples) {
  const mlr::RunConfig rc = big_config(n, nt, n_outer, memo, workers);
  const mlr::Geometry geom = rc.make_geometry();
  const BigInput in = big_input(geom, workers, random);
  mlr::EngineConfig ecfg = rc.engine;
  ecfg.memo_enabled = rc.admm.memoization != mlr::MemoMode::off;
  std::shared_ptr<mlr::Encoder> enc;
  std::shared_ptr<mlr::MemoClient> client;
  if (ecfg.memo_enabled) {
    mlr::MemoClientConfig mcfg = rc.memo;
    mcfg.endpoint.clear();
    client = std::make_shared<mlr::MemoClient>(mcfg);
    enc = std::make_shared<mlr::Encoder>(rc.encoder);
  }
  mlr::OperatorEngine eng(geom, ecfg, enc, client);
  mlr::ReconResult res = mlr::reconstruct(in.d, geom, rc.admm, eng, random ? nullptr : &in.phantom);
  const std::int64_t total = res.u.size();
  std::vector<std::int64_t> idx;
  {
    std::mt19937_64 rng(4242);
    std::vector<std::int64_t> pick;
    std::unordered_set<std::int64_t> seen;
    for (std::int64_t j = total - samples; j < total; ++j) {
      const std::int64_t t = static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(j + 1));
      if (seen.insert(t).second) pick.push_back(t);
      else { seen.insert(j); pick.push_back(j); }
    }
    std::sort(pick.begin(), pick.end());
    idx = pick;
  }
  std::vector<std::complex<float>> us(idx.size());
  for (std::size_t i = 0; i < idx.size(); ++i) {
    const cplx v = res.u.data()[idx[i]];
    us[i] = std::complex<float>(static_cast<float>(v.real()), static_cast<float>(v.imag()));
  }
  save_npy(dir + "/u_idx.npy", idx.data(), {static_cast<std::int64_t>(idx.size())});
  save_npy(dir + "/u_sample.npy", us.data(), {static_cast<std::int64_t>(us.size())});
  const double unorm = mlr::norm2(res.u), dnorm = mlr::norm2(in.d);
  save_npy(dir + "/u_norm.npy", &unorm, {1});
  save_npy(dir + "/d_norm.npy", &dnorm, {1});
  std::vector<std::complex<float>> dfirst(64);
  const std::size_t stride = static_cast<std::size_t>(in.d.size()) / dfirst.size();
  for (std::size_t i = 0; i < dfirst.size(); ++i)
    dfirst[i] = std::complex<float>(static_cast<float>(in.d.data()[i * stride].real()),
                                    static_cast<float>(in.d.data()[i * stride].imag()));
  save_npy(dir + "/d_probe.npy", dfirst.data(), {64});
  save_text(dir + "/report.csv", res.report.csv());
  save_text(dir + "/config.txt", rc.str());
  std::ostringstream ab;
  ab << (res.report.aborted ? 1 : 0) << "\n" << res.report.abort_reason << "\n"
     << "random_data=" << (random ? 1 : 0) << "\n";
  save_text(dir + "/aborted.txt", ab.str());
  if (ecfg.memo_enabled) {
    const std::vector<mlr::ChunkAudit> audit = eng.audit_log();
    std::vector<std::int32_t> a_int;
    std::vector<float> a_cs;
    for (const auto& e : audit) {
      a_int.push_back(e.iteration);
      a_int.push_back(static_cast<std::int32_t>(e.op));
      a_int.push_back(static_cast<std::int32_t>(e.location.index));
      a_int.push_back(static_cast<std::int32_t>(e.outcome));
      a_cs.push_back(e.cs);
    }
    const std::int64_t na = static_cast<std::int64_t>(audit.size());
    save_npy(dir + "/audit_int.npy", a_int.data(), {na, 4});
    save_npy(dir + "/audit_cs.npy", a_cs.data(), {na});
    const mlr::MemoCounterSnapshot c = client->counters();
    std::ostringstream cs;
    cs << "lookups=" << c.lookups << "\ncache_hits=" << c.cache_hits
       << "\nremote_hits=" << c.remote_hits << "\nmisses=" << c.misses
       << "\ncache_comparisons=" << c.cache_comparisons << "\ncache_probes=" << c.cache_probes
       << "\nbatches_sent=" << c.batches_sent << "\ninserts_enqueued=" << c.inserts_enqueued
       << "\ninserts_sent=" << c.inserts_sent << "\ninserts_dropped=" << c.inserts_dropped
       << "\n";
    save_text(dir + "/counters.txt", cs.str());
  }
  return 0;
}

// Runs the reference outer loop by hand (admm.cpp:226-244 without memo) and
// prints rho, r, s and the inner losses per outer iteration.
int cmd_trace(std::int64_t n, int n_outer) {
  mlr::RunConfig rc;
  for (const char* k : {"n1", "n0", "n2", "n_theta", "h", "w"}) rc.set(k, std::to_string(n));
  rc.set("nudft_path", "gridding");
  rc.set("workers", "8");
  const mlr::Geometry geom = rc.make_geometry();
  const mlr::Volume phantom = round_c64(mlr::make_phantom(geom.volume_shape(), mlr::PhantomKind::blocks, 1));
  const mlr::ProjectionSet d = round_c64(mlr::forward_L(phantom, geom, rc.engine.path));
  mlr::OperatorEngine eng(geom, rc.engine);
  mlr::AdmmState st = mlr::AdmmState::init(geom, rc.admm.rho0);
  const mlr::ProjectionSet d_hat = eng.f2d(d, false);
  for (int outer = 0; outer < n_outer; ++outer) {
    const std::size_t before = st.inner_losses.size();
    mlr::lsp_optimized(st, d_hat, rc.admm, eng);
    mlr::rsp_update(st, rc.admm);
    mlr::multiplier_penalty_update(st, rc.admm);
    std::printf("outer %d rho %.17g r %.17g s %.17g losses", outer, st.rho, st.r, st.s);
    for (std::size_t i = before; i < st.inner_losses.size(); ++i) std::printf(" %.17g", st.inner_losses[i]);
    std::printf("\n");
  }
  return 0;
}

// Sensitivity of the reference itself: reconstruct from d and from d with
// relative Gaussian noise eps, print rel-L2 of the two u per outer iteration.
int cmd_sens(std::int64_t n, int n_outer, double eps, const std::string& memo) {
  mlr::RunConfig rc;
  for (const char* k : {"n1", "n0", "n2", "n_theta", "h", "w"}) rc.set(k, std::to_string(n));
  rc.set("nudft_path", "gridding");
  rc.set("workers", "8");
  rc.set("memoization", memo);
  const mlr::Geometry geom = rc.make_geometry();
  const mlr::Volume phantom = round_c64(mlr::make_phantom(geom.volume_shape(), mlr::PhantomKind::blocks, 1));
  const mlr::ProjectionSet d = round_c64(mlr::forward_L(phantom, geom, rc.engine.path));
  mlr::ProjectionSet dp = d;
  std::mt19937_64 rng(77);
  std::normal_distribution<double> nd(0.0, 1.0);
  const double rms = mlr::norm2(d) / std::sqrt(static_cast<double>(d.size()));
  for (cplx& v : dp.flat()) v += cplx(nd(rng), nd(rng)) * (eps * rms / std::sqrt(2.0));
  for (int k = 1; k <= n_outer; ++k) {
    rc.set("n_outer", std::to_string(k));
    auto run = [&](const mlr::ProjectionSet& dd) {
      mlr::EngineConfig ecfg = rc.engine;
      ecfg.memo_enabled = rc.admm.memoization != mlr::MemoMode::off;
      std::shared_ptr<mlr::Encoder> enc;
      std::shared_ptr<mlr::MemoClient> client;
      if (ecfg.memo_enabled) {
        client = std::make_shared<mlr::MemoClient>(rc.memo);
        enc = std::make_shared<mlr::Encoder>(rc.encoder);
      }
      mlr::OperatorEngine eng(geom, ecfg, enc, client);
      return mlr::reconstruct(dd, geom, rc.admm, eng, &phantom).u;
    };
    const mlr::Volume u0 = run(d), u1 = run(dp);
    std::printf("eps %.1e outer %d rel_u %.3e\n", eps, k, mlr::norm2(mlr::sub(u1, u0)) / mlr::norm2(u0));
    std::fflush(stdout);
  }
  return 0;
}

int cmd_encoder(const std::string& dir) {
  mlr::EncoderConfig ec;  // projection, key_dim 60, seed 1337
  mlr::Encoder enc(ec);
  std::mt19937_64 rng(99);
  const mlr::Shape3 shapes[] = {{16, 16, 16}, {4, 16, 16}, {16, 8, 12}};
  int idx = 0;
  for (const mlr::Shape3& s : shapes) {
    enc.register_shape(s);
    const std::string tag = std::to_string(idx++);
    std::vector<float> keys, raw;
    std::vector<std::int32_t> meta;
    for (int op = 0; op < 4; ++op)
      for (std::int64_t loc = 0; loc < 3; ++loc) {
        const mlr::Array3 x = random_array(s, mlr::Domain::space, rng);
        if (op == 0 && loc == 0) save_arr(dir + "/x" + tag + ".npy", x);
        const mlr::MemoKey k = enc.encode(x, loc, static_cast<mlr::OpId>(op));
        const mlr::MemoKey r = enc.encode_content_only(x, loc, static_cast<mlr::OpId>(op));
        keys.insert(keys.end(), k.values.begin(), k.values.end());
        raw.insert(raw.end(), r.values.begin(), r.values.end());
        meta.push_back(op);
        meta.push_back(static_cast<std::int32_t>(loc));
        save_arr(dir + "/x" + tag + "_op" + std::to_string(op) + "_loc" + std::to_string(loc) +
                     ".npy",
                 x);
      }
    save_npy(dir + "/keys" + tag + ".npy", keys.data(), {12, 60});
    save_npy(dir + "/raw" + tag + ".npy", raw.data(), {12, 60});
    save_npy(dir + "/meta" + tag + ".npy", meta.data(), {12, 2});
  }
  return 0;
}

// CNN encoder (encoder.cpp:95-197, seeded initial weights init_cnn, 441-470):
// the weights, and raw and slot-mixed keys of random chunks of three shapes.
int cmd_cnn(const std::string& dir) {
  mlr::EncoderConfig ec;
  ec.variant = mlr::EncoderConfig::Variant::cnn;
  mlr::Encoder enc(ec);
  const mlr::CnnWeights& w = enc.cnn_weights();
  save_npy(dir + "/c1w.npy", w.c1.w.data(), {static_cast<std::size_t>(w.c1.out_ch), 2, 5, 5});
  save_npy(dir + "/c2w.npy", w.c2.w.data(), {static_cast<std::size_t>(w.c2.out_ch), static_cast<std::size_t>(w.c2.in_ch), 3, 3});
  save_npy(dir + "/fcw.npy", w.fc_w.data(), {60, static_cast<std::size_t>(w.c2.out_ch)});
  std::mt19937_64 rng(77);
  const mlr::Shape3 shapes[] = {{16, 16, 16}, {4, 16, 16}, {16, 8, 12}};
  int idx = 0;
  for (const mlr::Shape3& s : shapes) {
    const std::string tag = std::to_string(idx++);
    std::vector<float> keys, raw;
    std::vector<std::int32_t> meta;
    for (int op = 0; op < 4; ++op) {
      const std::int64_t loc = op;
      const mlr::Array3 x = random_array(s, mlr::Domain::space, rng);
      const mlr::MemoKey k = enc.encode(x, loc, static_cast<mlr::OpId>(op));
      const mlr::MemoKey r = enc.encode_content_only(x, loc, static_cast<mlr::OpId>(op));
      keys.insert(keys.end(), k.values.begin(), k.values.end());
      raw.insert(raw.end(), r.values.begin(), r.values.end());
      meta.push_back(op);
      meta.push_back(static_cast<std::int32_t>(loc));
      save_arr(dir + "/x" + tag + "_op" + std::to_string(op) + ".npy", x);
    }
    save_npy(dir + "/keys" + tag + ".npy", keys.data(), {4, 60});
    save_npy(dir + "/raw" + tag + ".npy", raw.data(), {4, 60});
    save_npy(dir + "/meta" + tag + ".npy", meta.data(), {4, 2});
  }
  return 0;
}

int cmd_store(const std::string& dir) {
  // Small IVF so the clustered regime is exercised with few keys.
  mlr::IvfConfig ic;
  ic.nlist = 4;
  ic.train_size = 32;
  ic.nprobe = 2;
  mlr::MemoStore store(ic);
  std::mt19937_64 rng(5);
  auto rnd_key = [&]() {
    std::vector<float> k(60);
    for (float& v : k) v = static_cast<float>((static_cast<double>(rng() >> 11) * 0x1.0p-53) * 2.0 - 1.0);
    return k;
  };
  std::vector<float> ins, qry, res_cs;
  std::vector<std::int64_t> res_int;  // (phase, found, hit, id)
  std::vector<std::vector<float>> inserted;
  for (int i = 0; i < 48; ++i) {
    // Queries between inserts cover both the flat and the IVF regime.
    if (i % 4 == 0) {
      for (int q = 0; q < 3; ++q) {
        std::vector<float> k = rnd_key();
        if (q == 1 && !inserted.empty()) {
          k = inserted[static_cast<std::size_t>(rng() % inserted.size())];
          for (float& v : k) v *= 1.0001f;
        }
        const mlr::QueryOutcome o = store.query(k, 0.92f, 0);
        qry.insert(qry.end(), k.begin(), k.end());
        res_int.push_back(i);
        res_int.push_back(o.found);
        res_int.push_back(o.hit);
        res_int.push_back(static_cast<std::int64_t>(o.id));
        res_cs.push_back(o.cs);
      }
    }
    std::vector<float> k = rnd_key();
    if (i % 7 == 3) std::fill(k.begin(), k.end(), 0.0f);  // zero keys are legal
    ins.insert(ins.end(), k.begin(), k.end());
    inserted.push_back(k);
    store.insert(k, {static_cast<std::uint8_t>(i)});
  }
  const std::int64_t nq = static_cast<std::int64_t>(res_cs.size());
  save_npy(dir + "/inserted.npy", ins.data(), {48, 60});
  save_npy(dir + "/queries.npy", qry.data(), {nq, 60});
  save_npy(dir + "/q_int.npy", res_int.data(), {nq, 4});
  save_npy(dir + "/q_cs.npy", res_cs.data(), {nq});
  std::vector<float> cent;
  for (const auto& c : store.centroids()) cent.insert(cent.end(), c.begin(), c.end());
  save_npy(dir + "/centroids.npy", cent.data(), {static_cast<std::int64_t>(cent.size() / 60), 60});
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 3) {
      std::fprintf(stderr, "usage: golden_gen ops|recon|encoder|store <dir> ...\n");
      return 2;
    }
    const std::string cmd = argv[1], dir = argv[2];
    auto I = [&](int i) { return static_cast<std::int64_t>(std::stoll(argv[i])); };
    if (cmd == "ops" && argc == 10) return cmd_ops(dir, I(3), I(4), I(5), I(6), I(7), I(8), I(9));
    if (cmd == "recon" && argc >= 8)
      return cmd_recon(dir, I(3), I(4), static_cast<int>(I(5)), argv[6], argv[7],
                       argc > 8 ? static_cast<int>(I(8)) : 1, argc > 9 ? argv[9] : "projection",
                       argc > 10 ? argv[10] : "optimized");
    if (cmd == "encoder") return cmd_encoder(dir);
    if (cmd == "cnn") return cmd_cnn(dir);
    if (cmd == "trace" && argc == 5) return cmd_trace(I(3), static_cast<int>(I(4)));
    if (cmd == "sens" && argc == 7) return cmd_sens(I(3), static_cast<int>(I(4)), std::stod(argv[5]), argv[6]);
    if (cmd == "store") return cmd_store(dir);
    if (cmd == "data" && argc == 7)
      return cmd_data(dir, I(3), I(4), static_cast<int>(I(5)), I(6) != 0);
    if (cmd == "recon_big" && argc == 10)
      return cmd_recon_big(dir, I(3), I(4), static_cast<int>(I(5)), argv[6], static_cast<int>(I(7)),
                           I(8) != 0, I(9));
    std::fprintf(stderr, "bad arguments\n");
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "golden_gen: %s\n", e.what());
    return 1;
  }
}
