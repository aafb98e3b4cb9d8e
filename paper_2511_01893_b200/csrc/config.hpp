// Flat key=value run configuration, key-for-key compatible with the
// reference's RunConfig (config.hpp:16-46, config.cpp:60-189) so existing
// config files and mlr_config_set calls drop in unchanged.
#pragma once

#include <cstdint>
#include <string>
#include <utility>

#include "solver.hpp"
#include "engine_api.hpp"
#include "geometry.hpp"
#include "memo.hpp"

namespace mlrg {

enum class NudftPath : std::uint8_t { direct = 0, gridding = 1 };

struct EncoderConfig {  // encoder.hpp:24-44 (projection variant on the device)
  enum class Variant : std::uint8_t { projection = 0, cnn = 1 };
  int key_dim = 60;
  Variant variant = Variant::projection;
  std::uint64_t seed = 1337;
  int epochs = 20;
  double learning_rate = 1e-3;
  int pair_samples = 200;
};

struct RunConfig {
  std::int64_t n1 = 32, n0 = 32, n2 = 32, n_theta = 32, h = 32, w = 32;
  double phi = 0.5235987755982988;
  AdmmConfig admm;
  EncoderConfig encoder;
  EngineConfig engine;
  NudftPath path = NudftPath::direct;  // accepted; the device always evaluates by gridding
  MemoClientConfig memo;
  std::string memo_endpoint;
  std::string encoder_weights;

  void set(const std::string& key, const std::string& value);
  static RunConfig from_text(const std::string& text);
  static RunConfig from_file(const std::string& path);
  Geometry make_geometry() const;
  void validate() const;
  std::string str() const;
};

std::pair<std::string, std::string> split_key_value(const std::string& line);

}  // namespace mlrg
