// The ADMM outer loop as host C++ driving device kernels: the reference's
// control flow (admm.cpp:59-272) statement for statement, with every array
// statement replaced by a fused device kernel and every scalar kept on the
// host in double.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "device.hpp"
#include "engine_api.hpp"

namespace mlrg {

enum class Pipeline : std::uint8_t { baseline = 0, optimized = 1 };
enum class MemoMode : std::uint8_t { off = 0, local = 1, distributed = 2 };

struct AdmmConfig {  // admm.hpp:19-30
  double alpha = 1e-3;
  double rho0 = 1.0;
  int n_inner = 4;
  int n_outer = 30;
  float tau = 0.92f;
  Pipeline pipeline = Pipeline::optimized;
  MemoMode memoization = MemoMode::off;
  bool freeze_rho = false;
  /// B200 extension (ADMM-Offload): psi, psi_prev and
  /// lambda live in pinned host memory and stream through the device in
  /// 16-plane chunks on a side stream around g_init and the RSP/multiplier pass;
  /// results are bit-identical to offload off.
  bool offload = false;
  void validate() const;
};

struct AdmmAbort : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct IterationRow {  // admm.hpp:51-58
  int iteration = 0;
  double loss = 0.0, e = 0.0, accuracy = 1.0;
  std::uint64_t miss = 0, remote_hit = 0, cache_hit = 0;
  double ms_lsp = 0.0, ms_rsp = 0.0, ms_update = 0.0;
};

struct ReconReport {
  std::vector<IterationRow> rows;
  bool aborted = false;
  std::string abort_reason;
  std::string csv() const;  // admm.cpp:197-206
};

struct SolverState;

/// The outer loop of reconstruct (admm.cpp:208-272) as a steppable object:
/// construction runs the setup (state allocation, d_hat = f2d(d)); each
/// step() runs one outer iteration and appends its report row. Device arrays:
/// `d` (n_theta, h, w) space-domain data, optional `reference` (n1, n0, n2).
class Solver {
 public:
  Solver(const float2* d, const AdmmConfig& cfg, Engine& eng, const float2* reference);
  ~Solver();
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  /// One outer iteration; returns false (and stops) once the solve aborted.
  bool step();
  int iteration() const;
  const ReconReport& report() const;
  const double2* u() const;  // the complex128 iterate (device)

 private:
  SolverState* st_;
};

/// Full solve: n_outer steps, result rounded to complex64 into `u_out` (device).
ReconReport reconstruct(const float2* d, const AdmmConfig& cfg, Engine& eng, const float2* reference, float2* u_out);

}  // namespace mlrg
