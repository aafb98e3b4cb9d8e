#include "offload_plan.hpp"

#include <algorithm>
#include <limits>
#include <set>
#include <sstream>
#include <stdexcept>
#include <utility>

namespace mlrg::offload {

namespace {

[[noreturn]] void bad(const std::string& what) { throw std::invalid_argument(what); }

int find_name(const std::vector<std::string>& names, const std::string& n) {
  const auto it = std::find(names.begin(), names.end(), n);
  return it == names.end() ? -1 : static_cast<int>(it - names.begin());
}

double transfer_ms(const Trace& tr, int var) { return tr.var_bytes[static_cast<std::size_t>(var)] / tr.bytes_per_ms; }

// PlanScore::rank (offload.hpp:111-115): infinite above every finite MT, undefined at 0
double rank_of(const Score& s) {
  if (s.kind == Score::kInfinite) return std::numeric_limits<double>::infinity();
  return s.kind == Score::kFinite ? s.mt : 0.0;
}
bool beats(const Score& a, const Score& b) {  // score_better (offload.cpp:213-216)
  const double ra = rank_of(a), rb = rank_of(b);
  return ra != rb ? ra > rb : a.m > b.m;
}

std::string mt_text(const Score& s) {
  std::ostringstream o;
  if (s.kind == Score::kUndefined) o << "undefined";
  else if (s.kind == Score::kInfinite) o << "inf";
  else o << s.mt;
  return o.str();
}

}  // namespace

// ---- trace (offload.cpp:11-118) ------------------------------------------------------------
double Trace::iteration_ms() const {
  double t = 0.0;
  for (const double d : phase_ms) t += d;
  return t;
}

double Trace::start_of(int phase) const {
  double t = 0.0;
  for (int i = 0; i < phase; ++i) t += phase_ms[static_cast<std::size_t>(i)];
  return t;
}

double Trace::resident_bytes() const {
  double b = 0.0;
  for (const double v : var_bytes) b += v;
  return b;
}

void Trace::check() const {
  if (phase_ms.empty()) bad("trace: no phases");
  if (!(bytes_per_ms > 0.0)) bad("trace: bandwidth must be positive");
  std::set<std::string> seen;
  for (std::size_t p = 0; p < phase_ms.size(); ++p) {
    if (!(phase_ms[p] > 0.0)) bad("trace: phase " + phase_name[p] + " has nonpositive duration");
    if (!seen.insert(phase_name[p]).second) bad("trace: duplicate phase " + phase_name[p]);
  }
  seen.clear();
  for (std::size_t v = 0; v < var_bytes.size(); ++v) {
    const std::string& n = var_name[v];
    if (!(var_bytes[v] > 0.0)) bad("trace: variable " + n + " has nonpositive size");
    if (!seen.insert(n).second) bad("trace: duplicate variable " + n);
    for (const auto& [p, w] : var_access[v]) {
      if (p < 0 || p >= static_cast<int>(phase_ms.size())) bad("trace: access of " + n + " names a missing phase");
      if (!(w.first >= 0.0 && w.first <= w.last && w.last <= phase_ms[static_cast<std::size_t>(p)]))
        bad("trace: access window of " + n + " falls outside its phase");
    }
  }
}

Trace Trace::parse(const std::string& text) {
  Trace tr;
  std::istringstream lines(text);
  std::string line;
  for (int no = 1; std::getline(lines, line); ++no) {
    if (const std::size_t c = line.find('#'); c != std::string::npos) line.erase(c);
    std::istringstream tok(line);
    std::string kind;
    if (!(tok >> kind)) continue;
    const auto error = [no](const std::string& why) { bad("trace line " + std::to_string(no) + ": " + why); };
    if (kind == "phase") {
      std::string name;
      double ms = 0.0;
      if (!(tok >> name >> ms)) error("expected `phase <name> <dur_ms>`");
      tr.phase_name.push_back(name);
      tr.phase_ms.push_back(ms);
    } else if (kind == "var") {
      std::string name;
      double bytes = 0.0;
      int elig = 0;
      if (!(tok >> name >> bytes >> elig)) error("expected `var <name> <bytes> <0|1>`");
      if (elig != 0 && elig != 1) error("eligibility must be 0 or 1");
      tr.var_name.push_back(name);
      tr.var_bytes.push_back(bytes);
      tr.var_eligible.push_back(elig == 1);
      tr.var_access.emplace_back();
    } else if (kind == "access") {
      std::string vn, pn;
      Window w;
      if (!(tok >> vn >> pn >> w.first >> w.last)) error("expected `access <var> <phase> <first_ms> <last_ms>`");
      const int v = find_name(tr.var_name, vn), p = find_name(tr.phase_name, pn);
      if (v < 0) error("unknown variable " + vn);
      if (p < 0) error("unknown phase " + pn);
      if (!tr.var_access[static_cast<std::size_t>(v)].emplace(p, w).second)
        error("duplicate access of " + vn + " in " + pn);
    } else {
      error("unknown record `" + kind + "`");
    }
    std::string extra;
    if (tok >> extra) error("trailing tokens");
  }
  tr.check();
  return tr;
}

// ---- idle windows (offload.cpp:120-141) -----------------------------------------------------
std::vector<Idle> idle_windows(const Trace& tr, int var) {
  const auto& acc = tr.var_access[static_cast<std::size_t>(var)];
  std::vector<Idle> out;
  const double iter = tr.iteration_ms();
  for (auto it = acc.begin(); it != acc.end(); ++it) {
    auto nx = std::next(it);
    const bool wraps = nx == acc.end();
    if (wraps) nx = acc.begin();
    const double shift = wraps ? iter : 0.0;
    Idle g;
    g.from = it->first;
    g.to = nx->first;
    g.last_use = tr.start_of(it->first) + it->second.last;
    g.next_use = tr.start_of(nx->first) + nx->second.first + shift;
    g.next_phase_start = tr.start_of(nx->first) + shift;
    out.push_back(g);
  }
  return out;
}

Score score_of(double m, double t) {  // make_score (offload.cpp:196-211)
  Score s;
  s.m = m;
  s.t = t;
  if (t > 0.0) {
    s.kind = Score::kFinite;
    s.mt = m / t;
  } else if (m > 0.0) {
    s.kind = Score::kInfinite;
    s.mt = std::numeric_limits<double>::infinity();
  }
  return s;
}

// ---- simulator (offload.cpp:218-302) --------------------------------------------------------
// Three back-to-back iterations on one FIFO channel; the middle one is measured.
// Memory drops when an offload completes and returns when a prefetch starts.
Simulation simulate(const std::vector<Action>& plan, const Trace& tr) {
  tr.check();
  for (const Action& a : plan) {  // C1-C3 and structural validity (check_constraints)
    if (a.var < 0 || a.var >= static_cast<int>(tr.var_bytes.size())) bad("simulate: action names a missing variable");
    if (!tr.var_eligible[static_cast<std::size_t>(a.var)]) bad("simulate: variable is not eligible for offloading");
    const std::vector<Idle> w = idle_windows(tr, a.var);
    if (a.window < 0 || a.window >= static_cast<int>(w.size())) bad("simulate: no such access gap");
    const double d = transfer_ms(tr, a.var), span = w[static_cast<std::size_t>(a.window)].span();
    if (a.prefetch_at < a.offload_at + d) bad("simulate: plan violates C1");
    if (!(span > 0.0)) bad("simulate: plan violates C2");
    if (!(d < span)) bad("simulate: plan violates C3");
  }
  const double iter = tr.iteration_ms(), total = tr.resident_bytes();
  Simulation sim;
  sim.baseline_peak = total;

  struct Req {
    double at;
    bool fetch;
    std::size_t act;
    int rep;
  };
  std::vector<Req> reqs;
  for (int rep = 0; rep < 3; ++rep)
    for (std::size_t i = 0; i < plan.size(); ++i) {
      reqs.push_back({rep * iter + plan[i].offload_at, false, i, rep});
      reqs.push_back({rep * iter + plan[i].prefetch_at, true, i, rep});
    }
  std::stable_sort(reqs.begin(), reqs.end(), [](const Req& a, const Req& b) {
    if (a.at != b.at) return a.at < b.at;
    if (a.fetch != b.fetch) return !a.fetch;  // offloads first
    return a.act < b.act;
  });
  std::vector<std::pair<double, double>> delta;  // (time, bytes change)
  std::map<std::pair<std::size_t, int>, double> fetched;
  double free_at = 0.0;
  for (const Req& r : reqs) {
    const int v = plan[r.act].var;
    const double begin = std::max(r.at, free_at), end = begin + transfer_ms(tr, v);
    free_at = end;
    const double b = tr.var_bytes[static_cast<std::size_t>(v)];
    if (r.fetch) {
      delta.emplace_back(begin, b);
      fetched[{r.act, r.rep}] = end;
    } else {
      delta.emplace_back(end, -b);
    }
  }
  std::stable_sort(delta.begin(), delta.end(),
                   [](const std::pair<double, double>& a, const std::pair<double, double>& b) { return a.first < b.first; });
  double level = total, peak = -1.0, t_prev = 0.0;
  for (const auto& [t, d] : delta) {
    if (t_prev < 2.0 * iter && t > iter) peak = std::max(peak, level);
    level += d;
    t_prev = t;
  }
  if (t_prev < 2.0 * iter) peak = std::max(peak, level);
  sim.peak = peak < 0.0 ? total : peak;

  double exposed = 0.0;
  for (std::size_t i = 0; i < plan.size(); ++i) {
    const Idle g = idle_windows(tr, plan[i].var)[static_cast<std::size_t>(plan[i].window)];
    const auto f = fetched.find({i, 1});
    if (f != fetched.end()) exposed += std::max(0.0, f->second - (iter + g.next_phase_start));
  }
  sim.exposed_ms = exposed;
  sim.score = score_of(total > 0.0 ? (total - sim.peak) / total : 0.0, iter > 0.0 ? exposed / iter : 0.0);
  return sim;
}

// ---- exhaustive plan search (offload.cpp:304-357) -------------------------------------------
Best search(const Trace& tr) {
  tr.check();
  // per eligible (variable, idle window) admitted by C2/C3: prefetch right
  // after the offload, or (when later) arriving at the consuming phase start
  std::vector<std::vector<Action>> opts;
  for (int v = 0; v < static_cast<int>(tr.var_bytes.size()); ++v) {
    if (!tr.var_eligible[static_cast<std::size_t>(v)]) continue;
    const double d = transfer_ms(tr, v);
    const std::vector<Idle> ws = idle_windows(tr, v);
    for (int wi = 0; wi < static_cast<int>(ws.size()); ++wi) {
      const Idle& g = ws[static_cast<std::size_t>(wi)];
      if (!(g.span() > 0.0) || !(d < g.span())) continue;
      const Action soon{v, wi, g.last_use, g.last_use + d};
      Action late = soon;
      late.prefetch_at = std::max(soon.prefetch_at, g.next_phase_start - d);
      opts.push_back({soon});
      if (late.prefetch_at != soon.prefetch_at) opts.back().push_back(late);
    }
  }
  Best best;
  best.sim = simulate(best.plan, tr);
  // mixed-radix counter over {none, option 1, option 2}, first window fastest
  std::vector<std::size_t> pick(opts.size(), 0);
  while (true) {
    std::size_t d = 0;
    for (; d < opts.size(); ++d) {
      if (++pick[d] <= opts[d].size()) break;
      pick[d] = 0;
    }
    if (d == opts.size()) break;
    std::vector<Action> plan;
    for (std::size_t s = 0; s < opts.size(); ++s)
      if (pick[s] > 0) plan.push_back(opts[s][pick[s] - 1]);
    Simulation sim = simulate(plan, tr);
    if (beats(sim.score, best.sim.score)) {
      best.plan = std::move(plan);
      best.sim = sim;
    }
  }
  return best;
}

// ---- LRU demand-fetch baseline (offload.cpp:359-442) ----------------------------------------
Lru lru(const Trace& tr, double budget) {
  tr.check();
  Lru res;
  const std::size_t nv = tr.var_bytes.size();
  double pinned = 0.0, biggest = 0.0;
  for (std::size_t v = 0; v < nv; ++v) {
    if (tr.var_eligible[v]) biggest = std::max(biggest, tr.var_bytes[v]);
    else pinned += tr.var_bytes[v];
  }
  if (budget < pinned + biggest) {
    std::ostringstream o;
    o << "budget " << budget << " cannot hold the pinned variables (" << pinned
      << ") plus the largest eligible variable (" << biggest << ")";
    res.feasible = false;
    res.reason = o.str();
    return res;
  }
  struct Touch {
    double at;
    int var, rep;
  };
  std::vector<Touch> touches;
  const double iter = tr.iteration_ms();
  for (int rep = 0; rep < 3; ++rep)
    for (int v = 0; v < static_cast<int>(nv); ++v)
      for (const auto& [p, w] : tr.var_access[static_cast<std::size_t>(v)]) {
        const double base = rep * iter + tr.start_of(p);
        touches.push_back({base + w.first, v, rep});
        if (w.last != w.first) touches.push_back({base + w.last, v, rep});
      }
  std::stable_sort(touches.begin(), touches.end(), [](const Touch& a, const Touch& b) {
    return a.at != b.at ? a.at < b.at : a.var < b.var;
  });
  std::vector<double> seen(nv, -1.0);
  std::vector<char> in(nv, 0);
  for (std::size_t v = 0; v < nv; ++v) in[v] = tr.var_eligible[v] ? 0 : 1;
  double used = pinned, exposed = 0.0, peak = used;
  for (const Touch& e : touches) {
    const std::size_t v = static_cast<std::size_t>(e.var);
    if (!in[v]) {
      while (used + tr.var_bytes[v] > budget) {  // evict the least recently touched
        int out = -1;
        for (std::size_t c = 0; c < nv; ++c)
          if (in[c] && tr.var_eligible[c] && c != v && (out < 0 || seen[c] < seen[static_cast<std::size_t>(out)]))
            out = static_cast<int>(c);
        if (out < 0) break;
        in[static_cast<std::size_t>(out)] = 0;
        used -= tr.var_bytes[static_cast<std::size_t>(out)];
      }
      in[v] = 1;
      used += tr.var_bytes[v];
      if (e.rep == 1) exposed += tr.var_bytes[v] / tr.bytes_per_ms;  // the fetch stalls
    }
    seen[v] = e.at;
    if (e.rep == 1) peak = std::max(peak, used);
  }
  res.peak = peak;
  res.exposed_ms = exposed;
  const double total = tr.resident_bytes();
  res.score = score_of(total > 0.0 ? (total - peak) / total : 0.0, iter > 0.0 ? exposed / iter : 0.0);
  return res;
}

// ---- C-ABI text (capi.cpp:88-126, 344-380) --------------------------------------------------
std::string plan_text(const std::string& trace_text, double bandwidth, const std::string& format) {
  if (format != "plan" && format != "csv") bad("format must be plan or csv, got '" + format + "'");
  Trace tr = Trace::parse(trace_text);
  if (bandwidth > 0.0) tr.bytes_per_ms = bandwidth;
  const Best b = search(tr);
  const bool csv = format == "csv";
  std::ostringstream o;
  o << "# MT = " << mt_text(b.sim.score) << " (M = " << b.sim.score.m << ", T = " << b.sim.score.t << ")\n";
  o << "# peak resident " << b.sim.peak << " of " << b.sim.baseline_peak << " bytes, exposed delay "
    << b.sim.exposed_ms << " ms per iteration of " << tr.iteration_ms() << " ms\n";
  if (csv) o << "var,from_phase,to_phase,offload_start_ms,prefetch_start_ms,mpd_ms,pd_ms\n";
  if (b.plan.empty() && !csv) o << "no beneficial offload found\n";
  for (const Action& a : b.plan) {
    const std::vector<Idle> ws = idle_windows(tr, a.var);
    const Idle& g = ws[static_cast<std::size_t>(a.window)];
    // derive_pd_mpd (offload.cpp:143-154): the first window leaving g.from
    const Idle* f = &g;
    for (const Idle& x : ws)
      if (x.from == g.from) {
        f = &x;
        break;
      }
    const double pd = f->next_use - a.prefetch_at, mpd = f->span();
    const std::string& var = tr.var_name[static_cast<std::size_t>(a.var)];
    const std::string& from = tr.phase_name[static_cast<std::size_t>(g.from)];
    const std::string& to = tr.phase_name[static_cast<std::size_t>(g.to)];
    if (csv)
      o << var << ',' << from << ',' << to << ',' << a.offload_at << ',' << a.prefetch_at << ',' << mpd << ',' << pd
        << '\n';
    else
      o << var << ": offload at " << a.offload_at << " ms after " << from << ", prefetch at " << a.prefetch_at
        << " ms for " << to << " (mpd " << mpd << " ms, pd " << pd << " ms)\n";
  }
  return o.str();
}

std::string lru_text(const std::string& trace_text, double bandwidth, unsigned long long budget_bytes) {
  Trace tr = Trace::parse(trace_text);
  if (bandwidth > 0.0) tr.bytes_per_ms = bandwidth;
  const Lru r = lru(tr, static_cast<double>(budget_bytes));
  std::ostringstream o;
  if (!r.feasible) {
    o << "infeasible: " << r.reason << '\n';
  } else {
    o << "MT = " << mt_text(r.score) << " (M = " << r.score.m << ", T = " << r.score.t << ")\n"
      << "peak resident " << r.peak << " bytes under budget " << budget_bytes << ", exposed delay " << r.exposed_ms
      << " ms per iteration\n";
  }
  return o.str();
}

}  // namespace mlrg::offload
