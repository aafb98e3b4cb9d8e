// ADMM-Offload planner behind mlr_plan_offload / mlr_lru_baseline (mlr.h;
// reference: offload.hpp:14-152, offload.cpp:1-444, capi.cpp:88-126, 344-380).
//
// A phase trace describes one outer iteration (treated as repeating): the
// phases and their durations, the variables with their sizes and, per phase
// that touches them, the first/last access offsets. The planner enumerates
// per-(variable, idle window) offload/prefetch actions under the paper's
// constraints C1-C4, scores every plan by MT = memory saving / exposed delay
// with a single-channel transfer simulator, and keeps the best; the LRU
// baseline demand-fetches under a byte budget. This is host-side planning:
// its output decides which solver arrays go to pinned host memory
// (`offload = host`, solver.cpp).
#pragma once

#include <map>
#include <string>
#include <vector>

namespace mlrg::offload {

struct Window {  // first/last access offsets within one phase (ms)
  double first = 0.0, last = 0.0;
};

struct Trace {
  std::vector<std::string> phase_name;
  std::vector<double> phase_ms;
  std::vector<std::string> var_name;
  std::vector<double> var_bytes;
  std::vector<bool> var_eligible;
  std::vector<std::map<int, Window>> var_access;  // phase index -> window, ascending phases
  double bytes_per_ms = 3.2e6;                     // one transfer channel

  /// `phase <name> <dur_ms>`, `var <name> <bytes> <0|1>`,
  /// `access <var> <phase> <first_ms> <last_ms>`; '#' comments. Validates.
  static Trace parse(const std::string& text);
  void check() const;  // std::invalid_argument on a malformed trace
  double iteration_ms() const;
  double start_of(int phase) const;
  double resident_bytes() const;
};

/// Idle window of a variable between an accessed phase and the next one
/// (the last wraps into the next iteration); absolute ms from iteration start.
struct Idle {
  int from = -1, to = -1;
  double last_use = 0.0, next_use = 0.0, next_phase_start = 0.0;
  double span() const { return next_use - last_use; }  // MPD
};
std::vector<Idle> idle_windows(const Trace& tr, int var);

struct Action {
  int var = -1, window = -1;
  double offload_at = 0.0, prefetch_at = 0.0;
};

struct Score {
  enum Kind { kUndefined, kFinite, kInfinite } kind = kUndefined;
  double m = 0.0, t = 0.0, mt = 0.0;
};
Score score_of(double m, double t);

struct Simulation {
  double baseline_peak = 0.0, peak = 0.0, exposed_ms = 0.0;
  Score score;
};
Simulation simulate(const std::vector<Action>& plan, const Trace& tr);

struct Best {
  std::vector<Action> plan;
  Simulation sim;
};
Best search(const Trace& tr);

struct Lru {
  bool feasible = true;
  std::string reason;
  double peak = 0.0, exposed_ms = 0.0;
  Score score;
};
Lru lru(const Trace& tr, double budget_bytes);

/// The text mlr_plan_offload / mlr_lru_baseline return (capi.cpp:98-126, 366-374).
std::string plan_text(const std::string& trace_text, double bandwidth, const std::string& format);
std::string lru_text(const std::string& trace_text, double bandwidth, unsigned long long budget_bytes);

}  // namespace mlrg::offload
