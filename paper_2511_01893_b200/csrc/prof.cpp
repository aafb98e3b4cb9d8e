// Kernel launch counter and opt-in CUDA-event timers per hot kernel. Events
// are recorded on the launching stream, so a timer measures exactly the
// kernel's device time span even when the host runs ahead.
#include <atomic>
#include <cstdio>
#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "device.hpp"
#include "mlr.h"
#include "mlrg.h"

namespace mlrg::prof {

namespace {
std::atomic<std::uint64_t> g_launches{0};
std::atomic<bool> g_enabled{false};
std::mutex g_mx;
struct Span {
  cudaEvent_t a, b;
  cudaStream_t s;
};
std::map<std::string, std::vector<Span>>& spans() {
  static std::map<std::string, std::vector<Span>> m;
  return m;
}
std::map<std::string, cudaEvent_t>& open_events() {
  static std::map<std::string, cudaEvent_t> m;
  return m;
}
std::map<std::string, std::pair<double, std::int64_t>>& host_spans() {
  static std::map<std::string, std::pair<double, std::int64_t>> m;
  return m;
}
}  // namespace

void host_add(const char* name, double ms) {
  if (!enabled()) return;
  std::lock_guard<std::mutex> lk(g_mx);
  auto& e = host_spans()[name];
  e.first += ms;
  ++e.second;
}

namespace {
thread_local long long t_last_mark = 0;
}
void host_mark(const char* name) {
  if (!enabled()) return;
  const long long t = std::chrono::steady_clock::now().time_since_epoch().count();
  if (t_last_mark)
    host_add(name, static_cast<double>(t - t_last_mark) * 1e3 * std::chrono::steady_clock::period::num /
                       std::chrono::steady_clock::period::den);
  t_last_mark = t;
}
HostSpan::HostSpan(const char* name)
    : name_(name), t0_(enabled() ? std::chrono::steady_clock::now().time_since_epoch().count() : 0) {
  t_last_mark = t0_;
}
HostSpan::~HostSpan() {
  if (!t0_) return;
  const long long t1 = std::chrono::steady_clock::now().time_since_epoch().count();
  host_add(name_, static_cast<double>(t1 - t0_) * 1e3 * std::chrono::steady_clock::period::num /
                      std::chrono::steady_clock::period::den);
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(std::uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
std::uint64_t launches() { return g_launches.load(std::memory_order_relaxed); }
bool enabled() { return g_enabled.load(std::memory_order_relaxed); }

void begin(const char* name, cudaStream_t s) {
  if (!enabled()) return;
  cudaEvent_t e;
  MLRG_CUDA(cudaEventCreate(&e));
  MLRG_CUDA(cudaEventRecord(e, s));
  std::lock_guard<std::mutex> lk(g_mx);
  open_events()[std::string(name) + "@" + std::to_string(reinterpret_cast<std::uintptr_t>(s))] = e;
}

void end(const char* name, cudaStream_t s) {
  if (!enabled()) return;
  cudaEvent_t e;
  MLRG_CUDA(cudaEventCreate(&e));
  MLRG_CUDA(cudaEventRecord(e, s));
  std::lock_guard<std::mutex> lk(g_mx);
  auto it = open_events().find(std::string(name) + "@" + std::to_string(reinterpret_cast<std::uintptr_t>(s)));
  if (it == open_events().end()) return;
  spans()[name].push_back({it->second, e, s});
  open_events().erase(it);
}

}  // namespace mlrg::prof

extern "C" {

uint64_t mlrg_launch_count(void) { return mlrg::prof::g_launches.load(); }

void mlrg_prof_enable(int on) { mlrg::prof::g_enabled.store(on != 0); }

void mlrg_prof_reset(void) {
  std::lock_guard<std::mutex> lk(mlrg::prof::g_mx);
  for (auto& [k, v] : mlrg::prof::spans())
    for (auto& s : v) {
      cudaEventDestroy(s.a);
      cudaEventDestroy(s.b);
    }
  mlrg::prof::spans().clear();
  mlrg::prof::host_spans().clear();
}

int mlrg_prof_dump(const char* path) {
  std::lock_guard<std::mutex> lk(mlrg::prof::g_mx);
  struct Row {
    std::string name;
    const mlrg::prof::Span* sp;
  };
  std::vector<Row> rows;
  for (auto& [k, v] : mlrg::prof::spans())
    for (auto& s : v) rows.push_back({k, &s});
  if (rows.empty()) return 0;
  // reference: the span whose start is earliest
  cudaEvent_t ref = rows[0].sp->a;
  for (auto& r : rows) {
    if (cudaEventSynchronize(r.sp->b) != cudaSuccess) return MLR_ERR_RUNTIME;
    float d = 0.f;
    if (cudaEventElapsedTime(&d, ref, r.sp->a) != cudaSuccess) return MLR_ERR_RUNTIME;
    if (d < 0.f) ref = r.sp->a;
  }
  std::FILE* f = std::fopen(path, "w");
  if (!f) return MLR_ERR_IO;
  for (auto& r : rows) {
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ref, r.sp->a);
    cudaEventElapsedTime(&b, ref, r.sp->b);
    std::fprintf(f, "%s %llu %.4f %.4f\n", r.name.c_str(), static_cast<unsigned long long>(reinterpret_cast<std::uintptr_t>(r.sp->s)), a, b);
  }
  std::fclose(f);
  return 0;
}

int mlrg_prof_query(const char* name, double* total_ms, int64_t* count) {
  std::lock_guard<std::mutex> lk(mlrg::prof::g_mx);
  double tot = 0.0;
  int64_t n = 0;
  auto ht = mlrg::prof::host_spans().find(name ? name : "");
  if (ht != mlrg::prof::host_spans().end()) {  // host-side phase ("host:..."): wall ms
    if (total_ms) *total_ms = ht->second.first;
    if (count) *count = ht->second.second;
    return 0;
  }
  auto it = mlrg::prof::spans().find(name ? name : "");
  if (it != mlrg::prof::spans().end())
    for (auto& s : it->second) {
      if (cudaEventSynchronize(s.b) != cudaSuccess) return MLR_ERR_RUNTIME;
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, s.a, s.b) != cudaSuccess) return MLR_ERR_RUNTIME;
      tot += ms;
      ++n;
    }
  if (total_ms) *total_ms = tot;
  if (count) *count = n;
  return 0;
}

}  // extern "C"
