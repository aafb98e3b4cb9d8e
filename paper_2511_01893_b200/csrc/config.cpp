#include "config.hpp"

#include <cctype>
#include <initializer_list>
#include <map>
#include <fstream>
#include <sstream>
#include <stdexcept>

namespace mlrg {

namespace {

std::string trim(const std::string& s) {
  std::size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

std::int64_t to_i64(const std::string& key, const std::string& v) {
  try {
    std::size_t pos = 0;
    const std::int64_t out = std::stoll(v, &pos);
    if (pos != v.size()) throw std::invalid_argument("trailing characters");
    return out;
  } catch (const std::exception&) {
    throw std::invalid_argument(key + ": expected an integer, got '" + v + "'");
  }
}

double to_f64(const std::string& key, const std::string& v) {
  try {
    std::size_t pos = 0;
    const double out = std::stod(v, &pos);
    if (pos != v.size()) throw std::invalid_argument("trailing characters");
    return out;
  } catch (const std::exception&) {
    throw std::invalid_argument(key + ": expected a number, got '" + v + "'");
  }
}

bool to_bool(const std::string& key, const std::string& v) {
  if (v == "true" || v == "1" || v == "on") return true;
  if (v == "false" || v == "0" || v == "off") return false;
  throw std::invalid_argument(key + ": expected true/false, got '" + v + "'");
}

int to_int(const std::string& key, const std::string& v) { return static_cast<int>(to_i64(key, v)); }

}  // namespace

std::pair<std::string, std::string> split_key_value(const std::string& line) {
  const std::size_t eq = line.find('=');
  if (eq == std::string::npos) throw std::invalid_argument("expected key=value, got '" + line + "'");
  return {trim(line.substr(0, eq)), trim(line.substr(eq + 1))};
}

namespace {

using Setter = void (*)(RunConfig&, const std::string& key, const std::string& value);

template <class E>
E pick(const std::string& key, const std::string& v, std::initializer_list<std::pair<const char*, E>> opts) {
  std::string names;
  for (const auto& [name, e] : opts) {
    if (v == name) return e;
    names += (names.empty() ? "" : "|") + std::string(name);
  }
  throw std::invalid_argument(key + ": expected " + names + ", got '" + v + "'");
}

// Key table: the reference's key set (config.cpp:60-114), one handler each.
const std::map<std::string, Setter>& setters() {
  static const std::map<std::string, Setter> table = {
      {"n1", [](RunConfig& c, const std::string& k, const std::string& v) { c.n1 = to_i64(k, v); }},
      {"n0", [](RunConfig& c, const std::string& k, const std::string& v) { c.n0 = to_i64(k, v); }},
      {"n2", [](RunConfig& c, const std::string& k, const std::string& v) { c.n2 = to_i64(k, v); }},
      {"n_theta", [](RunConfig& c, const std::string& k, const std::string& v) { c.n_theta = to_i64(k, v); }},
      {"h", [](RunConfig& c, const std::string& k, const std::string& v) { c.h = to_i64(k, v); }},
      {"w", [](RunConfig& c, const std::string& k, const std::string& v) { c.w = to_i64(k, v); }},
      {"phi", [](RunConfig& c, const std::string& k, const std::string& v) { c.phi = to_f64(k, v); }},
      {"alpha", [](RunConfig& c, const std::string& k, const std::string& v) { c.admm.alpha = to_f64(k, v); }},
      {"rho0", [](RunConfig& c, const std::string& k, const std::string& v) { c.admm.rho0 = to_f64(k, v); }},
      {"n_inner", [](RunConfig& c, const std::string& k, const std::string& v) { c.admm.n_inner = to_int(k, v); }},
      {"n_outer", [](RunConfig& c, const std::string& k, const std::string& v) { c.admm.n_outer = to_int(k, v); }},
      {"tau",  // one key drives both the solver and the memo gate
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.memo.tau = c.admm.tau = static_cast<float>(to_f64(k, v));
       }},
      {"pipeline",
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.admm.pipeline = pick<Pipeline>(k, v, {{"baseline", Pipeline::baseline}, {"optimized", Pipeline::optimized}});
       }},
      {"memoization",
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.admm.memoization = pick<MemoMode>(
             k, v, {{"off", MemoMode::off}, {"local", MemoMode::local}, {"distributed", MemoMode::distributed}});
       }},
      {"freeze_rho", [](RunConfig& c, const std::string& k, const std::string& v) { c.admm.freeze_rho = to_bool(k, v); }},
      {"workers", [](RunConfig& c, const std::string& k, const std::string& v) { c.engine.workers = to_int(k, v); }},
      {"chunk_extent",
       [](RunConfig& c, const std::string& k, const std::string& v) { c.engine.chunk_extent = to_i64(k, v); }},
      {"nudft_path",
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.path = pick<NudftPath>(k, v, {{"direct", NudftPath::direct}, {"gridding", NudftPath::gridding}});
       }},
      {"gridding_kernel",  // B200 extension (not a reference key): es (default) | gaussian
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.engine.kernel = pick<GridKernel>(k, v, {{"es", GridKernel::es}, {"gaussian", GridKernel::gaussian}});
       }},
      {"offload",  // B200 extension: off (default) | host -- psi, psi_prev, lambda in pinned host memory
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.admm.offload = pick<bool>(k, v, {{"off", false}, {"host", true}});
       }},
      {"flush_after_apply",
       [](RunConfig& c, const std::string& k, const std::string& v) { c.engine.flush_after_apply = to_bool(k, v); }},
      {"key_dim", [](RunConfig& c, const std::string& k, const std::string& v) { c.encoder.key_dim = to_int(k, v); }},
      {"encoder_variant",
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.encoder.variant = pick<EncoderConfig::Variant>(
             k, v, {{"projection", EncoderConfig::Variant::projection}, {"cnn", EncoderConfig::Variant::cnn}});
       }},
      {"encoder_seed",
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.encoder.seed = static_cast<std::uint64_t>(to_i64(k, v));
       }},
      {"encoder_epochs", [](RunConfig& c, const std::string& k, const std::string& v) { c.encoder.epochs = to_int(k, v); }},
      {"encoder_lr",
       [](RunConfig& c, const std::string& k, const std::string& v) { c.encoder.learning_rate = to_f64(k, v); }},
      {"encoder_pairs",
       [](RunConfig& c, const std::string& k, const std::string& v) { c.encoder.pair_samples = to_int(k, v); }},
      {"encoder_weights", [](RunConfig& c, const std::string&, const std::string& v) { c.encoder_weights = v; }},
      {"memo_endpoint", [](RunConfig& c, const std::string&, const std::string& v) { c.memo_endpoint = v; }},
      {"nprobe", [](RunConfig& c, const std::string& k, const std::string& v) { c.memo.nprobe = to_int(k, v); }},
      {"memo_timeout_ms",
       [](RunConfig& c, const std::string& k, const std::string& v) { c.memo.timeout_ms = to_int(k, v); }},
      {"insert_queue_cap",
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.memo.insert_queue_cap = static_cast<std::size_t>(to_i64(k, v));
       }},
      {"coalesce_bytes",
       [](RunConfig& c, const std::string& k, const std::string& v) {
         c.memo.coalesce_bytes = static_cast<std::size_t>(to_i64(k, v));
       }},
      {"global_cache", [](RunConfig& c, const std::string& k, const std::string& v) { c.memo.global_cache = to_bool(k, v); }},
  };
  return table;
}

}  // namespace

void RunConfig::set(const std::string& key, const std::string& value) {
  const auto it = setters().find(key);
  if (it == setters().end()) throw std::invalid_argument("unknown config key: '" + key + "'");
  it->second(*this, key, value);
}

RunConfig RunConfig::from_text(const std::string& text) {  // config.cpp:116-135
  RunConfig cfg;
  std::istringstream in(text);
  std::string line;
  int line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    const std::size_t hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    line = trim(line);
    if (line.empty()) continue;
    try {
      auto [key, value] = split_key_value(line);
      cfg.set(key, value);
    } catch (const std::invalid_argument& e) {
      throw std::invalid_argument("config line " + std::to_string(line_no) + ": " + e.what());
    }
  }
  return cfg;
}

RunConfig RunConfig::from_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open config file: " + path);
  std::ostringstream buf;
  buf << in.rdbuf();
  return from_text(buf.str());
}

Geometry RunConfig::make_geometry() const { return Geometry::make(n1, n0, n2, n_theta, h, w, phi); }

void RunConfig::validate() const {  // config.cpp:149-158
  if (n1 < 1 || n0 < 1 || n2 < 1 || n_theta < 1 || h < 1 || w < 1)
    throw std::invalid_argument("geometry extents must be positive");
  if (h > n0) throw std::invalid_argument("h must not exceed n0");
  admm.validate();
  if (encoder.key_dim < 1) throw std::invalid_argument("encoder: key_dim must be >= 1");
  if (engine.workers < 1) throw std::invalid_argument("workers must be >= 1");
  if (engine.chunk_extent < 1) throw std::invalid_argument("chunk_extent must be >= 1");
  if (memo.nprobe < 1) throw std::invalid_argument("nprobe must be >= 1");
}

std::string RunConfig::str() const {  // config.cpp:160-189
  std::ostringstream o;
  o << "n1 = " << n1 << "\nn0 = " << n0 << "\nn2 = " << n2 << "\nn_theta = " << n_theta << "\nh = " << h
    << "\nw = " << w << "\nphi = " << phi << "\nalpha = " << admm.alpha << "\nrho0 = " << admm.rho0
    << "\nn_inner = " << admm.n_inner << "\nn_outer = " << admm.n_outer << "\ntau = " << admm.tau
    << "\npipeline = " << (admm.pipeline == Pipeline::baseline ? "baseline" : "optimized") << "\nmemoization = "
    << (admm.memoization == MemoMode::off ? "off" : admm.memoization == MemoMode::local ? "local" : "distributed")
    << "\nfreeze_rho = " << (admm.freeze_rho ? "true" : "false") << "\nworkers = " << engine.workers
    << "\nchunk_extent = " << engine.chunk_extent
    << "\nnudft_path = " << (path == NudftPath::direct ? "direct" : "gridding")
    << "\nflush_after_apply = " << (engine.flush_after_apply ? "true" : "false") << "\nkey_dim = " << encoder.key_dim
    << "\nencoder_variant = " << (encoder.variant == EncoderConfig::Variant::projection ? "projection" : "cnn")
    << "\nencoder_seed = " << encoder.seed << "\nencoder_epochs = " << encoder.epochs
    << "\nencoder_lr = " << encoder.learning_rate << "\nencoder_pairs = " << encoder.pair_samples;
  if (!encoder_weights.empty()) o << "\nencoder_weights = " << encoder_weights;
  if (!memo_endpoint.empty()) o << "\nmemo_endpoint = " << memo_endpoint;
  o << "\nnprobe = " << memo.nprobe << "\nmemo_timeout_ms = " << memo.timeout_ms
    << "\ninsert_queue_cap = " << memo.insert_queue_cap << "\ncoalesce_bytes = " << memo.coalesce_bytes
    << "\nglobal_cache = " << (memo.global_cache ? "true" : "false") << "\n";
  if (engine.kernel == GridKernel::gaussian) o << "gridding_kernel = gaussian\n";
  if (admm.offload) o << "offload = host\n";
  return o.str();
}

}  // namespace mlrg
