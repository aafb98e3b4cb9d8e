#include "memo_gpu.hpp"

#include <algorithm>
#include <mutex>
#include <limits>
#include <random>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

namespace mlrg {

namespace {

constexpr int kLookupThreads = 256;
constexpr int kMaxKd = 64;
constexpr int kMaxProbe = 64;
constexpr int kStageThreads = 1024;  // one thread per slab (max_slabs <= 1024)

// memostore.cpp:30-38, in the reference's operation order (no contraction).
__device__ __forceinline__ double l2_sq_d(const float* a, const float* b, int d) {
  double acc = 0.0;
  for (int i = 0; i < d; ++i) {
    const double x = __dsub_rn(static_cast<double>(a[i]), static_cast<double>(b[i]));
    acc = __dadd_rn(acc, __dmul_rn(x, x));
  }
  return acc;
}

// memostore.cpp:17-28.
__device__ __forceinline__ double cosine_d(const float* a, const float* b, int d) {
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (int i = 0; i < d; ++i) {
    const double x = static_cast<double>(a[i]), y = static_cast<double>(b[i]);
    dot = __dadd_rn(dot, __dmul_rn(x, y));
    na = __dadd_rn(na, __dmul_rn(x, x));
    nb = __dadd_rn(nb, __dmul_rn(y, y));
  }
  if (na == 0.0 || nb == 0.0) return 0.0;
  return __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb)));
}

struct Best {
  double d;
  long long id;
};
__device__ __forceinline__ bool better(const Best& a, const Best& b) {  // (l2, lower id)
  return a.id >= 0 && (b.id < 0 || a.d < b.d || (a.d == b.d && a.id < b.id));
}

struct LookupArgs {
  int op, n, kd, nprobe, ncent, trained, max_slabs;
  float tau;
  const float* raw;
  const int* perm;
  const float* sign;
  float* qkeys;
  float* cache_key;
  long long* cache_vid;
  const float* keys;
  const long long* vbytes;
  const long long* slab_vbytes;
  const float* cent;
  const int* cl_ptr;
  const int* cl_ids;
  const long long* state;
  DevSlab* slabs;
  int* probed;
  int* queried;
};

// Candidate j of the store query: flat, key j; trained, entry j of the
// concatenated lists of the probed clusters (base = their starts in cl_ids,
// pre = their prefix sizes).
__device__ __forceinline__ long long candidate(const LookupArgs& a, long long j, int np, const int* base,
                                               const int* pre) {
  if (!a.trained) return j;
  int p = 0;
  while (p + 1 < np && j >= pre[p + 1]) ++p;
  return a.cl_ids[base[p] + (j - pre[p])];
}

// One CTA per slab: cache probe, then (on a cache miss) the store query. The
// query's distances are independent per candidate key, so the CTA spreads the
// candidates over its threads; each distance is still the reference's
// sequential sum, and the (l2, lower id) minimum does not depend on the
// visiting order. The keys the single-thread and per-centroid sums read (the
// cached key, the centroids, the best key) are first staged in shared memory
// by all threads, so no 60-long chain of dependent global loads sits on one
// thread; the candidate scan reads its keys directly, kIlp per thread.
// 4-byte cp.async into shared memory: a thread's staging loads all in flight at once
__device__ __forceinline__ void cp_async4(float* smem, const float* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

constexpr int kChunk = kMaxProbe;   // staged rows (the centroids)
constexpr int kRow = kMaxKd + 1;    // staged row stride (odd: conflict-free column reads)
constexpr int kIlp = 4;             // candidate keys per thread in flight in the distance loop

__global__ void __launch_bounds__(kLookupThreads) k_memo_lookup(LookupArgs a) {
  __shared__ float q[kMaxKd];
  __shared__ float kb[kChunk * kRow];  // staged key rows
  __shared__ Best red[kLookupThreads / 32];
  __shared__ double cd[kMaxProbe];
  __shared__ int probe[kMaxProbe];
  __shared__ int pre[kMaxProbe + 1];
  __shared__ int cbase[kMaxProbe], csize[kMaxProbe];
  __shared__ int done;
  __shared__ long long best_id;
  const int c = blockIdx.x, t = threadIdx.x, kd = a.kd;
  const long long slot = static_cast<long long>(a.op) * a.max_slabs + c;
  const int mix = static_cast<int>(slot) * kd;
  const long long vid = a.cache_vid[slot];
  if (t < kd) {  // slot_mix (encoder.cpp:66-86): tables from the host
    q[t] = a.sign[mix + t] * a.raw[static_cast<long long>(c) * kd + a.perm[mix + t]];
    a.qkeys[static_cast<long long>(c) * kd + t] = q[t];
    if (vid >= 0) kb[t] = a.cache_key[slot * kd + t];
  }
  __syncthreads();
  DevSlab& out = a.slabs[c];
  if (t == 0) {
    done = 0;
    a.probed[c] = vid >= 0;
    a.queried[c] = 0;
    if (vid >= 0) {
      const float cs = static_cast<float>(cosine_d(q, kb, kd));
      if (cs > a.tau && a.vbytes[vid] == a.slab_vbytes[c]) {
        out.outcome = 2;
        out.cs = cs;
        out.vid = vid;
        done = 1;
      }
    }
  }
  __syncthreads();
  if (done) return;
  // ---- store query over the published keys (memostore.cpp:174-222) ----
  long long total = a.state[0];
  int np = 0;
  if (a.trained) {
    // the nprobe clusters with the smallest (l2, index), ascending: the rank of
    // centroid t is the number of centroids ordered before it
    for (int r = t >> 5; r < a.ncent; r += kLookupThreads / 32)  // a warp per centroid row
      for (int i = t & 31; i < kd; i += 32) cp_async4(&kb[r * kRow + i], a.cent + static_cast<long long>(r) * kd + i);
    cp_async_all();
    __syncthreads();
    if (t < a.ncent) cd[t] = l2_sq_d(q, kb + t * kRow, kd);
    __syncthreads();
    np = min(a.nprobe, a.ncent);
    if (t < a.ncent) {
      int rank = 0;
      for (int k = 0; k < a.ncent; ++k) rank += (cd[k] < cd[t] || (cd[k] == cd[t] && k < t)) ? 1 : 0;
      if (rank < np) probe[rank] = t;
    }
    __syncthreads();
    if (t < np) {  // each probed list's start and size (one thread per list)
      cbase[t] = a.cl_ptr[probe[t]];
      csize[t] = a.cl_ptr[probe[t] + 1] - cbase[t];
    }
    __syncthreads();
    if (t == 0) {
      pre[0] = 0;
      for (int p = 0; p < np; ++p) pre[p + 1] = pre[p] + csize[p];
    }
    __syncthreads();
    total = pre[np];
  }
  // candidates straight from global memory, kIlp interleaved per thread (all 256
  // threads busy: at a thousand candidates this beats staging them in rounds)
  Best b{0.0, -1};
  for (long long j0 = t; j0 < total; j0 += static_cast<long long>(kIlp) * kLookupThreads) {
    const float* row[kIlp];
    long long id[kIlp];
    double acc[kIlp];
#pragma unroll
    for (int k = 0; k < kIlp; ++k) {
      const long long j = j0 + static_cast<long long>(k) * kLookupThreads;
      id[k] = j < total ? candidate(a, j, np, cbase, pre) : -1;
      row[k] = a.keys + (id[k] < 0 ? 0 : id[k]) * kd;
      acc[k] = 0.0;
    }
#pragma unroll 8
    for (int i = 0; i < kd; ++i) {  // unrolled: 8 dims x kIlp keys of loads in flight
      const double qi = static_cast<double>(q[i]);
#pragma unroll
      for (int k = 0; k < kIlp; ++k) {
        const double x = __dsub_rn(qi, static_cast<double>(row[k][i]));
        acc[k] = __dadd_rn(acc[k], __dmul_rn(x, x));
      }
    }
#pragma unroll
    for (int k = 0; k < kIlp; ++k) {
      const Best cand{acc[k], id[k]};
      if (better(cand, b)) b = cand;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    Best x;
    x.d = __shfl_xor_sync(0xffffffffu, b.d, o);
    x.id = __shfl_xor_sync(0xffffffffu, b.id, o);
    if (better(x, b)) b = x;
  }
  if ((t & 31) == 0) red[t >> 5] = b;
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < kLookupThreads / 32; ++w)
      if (better(red[w], b)) b = red[w];
    best_id = b.id;
  }
  __syncthreads();
  const long long bid = best_id;
  if (bid >= 0 && t < kd) kb[t] = a.keys[bid * kd + t];
  __syncthreads();
  if (t != 0) return;
  a.queried[c] = 1;
  out.outcome = 0;
  out.cs = 0.0f;
  out.vid = -1;
  if (bid < 0) return;  // empty store: a miss with cs 0
  const float cs = static_cast<float>(cosine_d(q, kb, kd));
  out.cs = cs;
  if (cs > a.tau && a.vbytes[bid] == a.slab_vbytes[c]) {  // memoclient.cpp:284-292
    out.outcome = 1;
    out.vid = bid;
    for (int i = 0; i < kd; ++i) a.cache_key[slot * kd + i] = q[i];  // the QUERY key
    a.cache_vid[slot] = bid;
  }
}

struct StageArgs {
  int n, kd, op, iteration, cap;
  long long arena_bytes, log_cap;
  const float* qkeys;
  const double* norms2;
  const long long* slab_vbytes;
  const long long* slab_counts;
  float* keys;
  long long* vbytes;
  double* vnorm;
  const float2** vptr;
  char* arena;
  long long* state;
  DevSlab* slabs;
  unsigned char* skip;
  const int* probed;
  const int* queried;
  DevLog* log;
};

// One thread per slab: hit sources/scales, insert staging (cap per flush
// window, arena bump allocation) and the decision log, in slab order. The only
// sequential part, the running insert count and arena offset over the misses,
// runs on one thread over shared memory; every global read and write is issued
// by the slab's own thread.
__global__ void __launch_bounds__(kStageThreads) k_memo_stage(StageArgs a) {
  __shared__ long long s_bytes[kStageThreads], s_off[kStageThreads], s_id[kStageThreads];
  __shared__ int s_miss[kStageThreads], s_staged[kStageThreads];
  __shared__ long long st[6];
  const int c = threadIdx.x;
  const bool mine = c < a.n;
  if (c < 6) st[c] = a.state[c];
  DevSlab s{};
  double live = 0.0;
  if (mine) {
    s = a.slabs[c];
    live = __dsqrt_rn(a.norms2[c]);
    s_miss[c] = s.outcome == 0;
    s_bytes[c] = (a.slab_counts[c] * 8 + 255) & ~255LL;
  }
  __syncthreads();
  if (c == 0) {  // memoclient.cpp:302-325: stage up to cap per flush window, in slab order
    // the arena is a ring (cold_tier.hpp ValueRing::alloc): a value that would
    // cross the end starts at 0; the host freed the span this window can fill
    long long nst = st[1], off = st[2], dropped = 0;
    int overflow = 0;
    for (int k = 0; k < a.n; ++k) {
      s_staged[k] = -1;
      if (!s_miss[k]) continue;
      if (nst < a.cap) {
        if (off + s_bytes[k] > a.arena_bytes) off = 0;
        const bool fits = s_bytes[k] <= a.arena_bytes;
        s_staged[k] = 1;
        s_off[k] = fits ? off : -1;
        s_id[k] = st[0] + nst;
        overflow |= fits ? 0 : 1;
        off += fits ? s_bytes[k] : 0;
        ++nst;
      } else {
        s_staged[k] = 0;
        ++dropped;
      }
    }
    a.state[1] = nst;
    a.state[2] = off;
    a.state[3] = st[3] + a.n;
    if (overflow) a.state[4] = 1;  // the host fails the flush
    a.state[5] = st[5] + dropped;
  }
  __syncthreads();
  if (!mine) return;
  const int staged = s_staged[c];
  if (s.outcome != 0) {
    const double stored = a.vnorm[s.vid];
    s.src = a.vptr[s.vid];
    s.scale = (stored > 0.0 && live > 0.0) ? __ddiv_rn(live, stored) : 1.0;
    s.dst = nullptr;
    a.skip[c] = 1;
  } else {
    s.dst = nullptr;
    if (staged == 1) {
      const long long id = s_id[c];
      float2* dst = s_off[c] >= 0 ? reinterpret_cast<float2*>(a.arena + s_off[c]) : nullptr;
      const float* __restrict__ src = a.qkeys + static_cast<long long>(c) * a.kd;
      float* __restrict__ kdst = a.keys + id * a.kd;
      for (int i0 = 0; i0 < a.kd; i0 += 16) {  // 16 loads issued before their stores (the arrays never alias)
        float buf[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i0 + i < a.kd) buf[i] = src[i0 + i];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i0 + i < a.kd) kdst[i0 + i] = buf[i];
      }
      a.vbytes[id] = a.slab_vbytes[c];
      a.vnorm[id] = live;
      a.vptr[id] = dst;
      s.dst = dst;
    }
    s.src = nullptr;
    s.scale = 1.0;
    a.skip[c] = 0;
  }
  a.slabs[c] = s;
  const long long li = st[3] + c;
  if (li < a.log_cap) a.log[li] = DevLog{a.iteration, a.op, c, s.outcome, s.cs, a.probed[c], a.queried[c], staged};
}

}  // namespace

namespace {

// ---- IVF training on the GPU (memostore.cpp:40-108, kmeans_train in memo.cpp) ----
// One CTA: k-means++ seeding with the reference's draws (pre-drawn on the host
// from the same mt19937_64, one per centroid), then the Lloyd iterations and
// the final nearest-centroid assignment. Every distance is the sequential
// double sum over the key's dimensions with explicit _rn arithmetic (no FMA
// contraction), every centroid sum runs over the keys in key order, ties
// resolve to the lower index: the host's results bit for bit.
constexpr int kKmThreads = 1024;

__device__ __forceinline__ double km_l2(const float* __restrict__ a, const float* __restrict__ b, int d) {
  double acc = 0.0;
  for (int i = 0; i < d; ++i) {
    const double x = __dsub_rn(static_cast<double>(a[i]), static_cast<double>(b[i]));
    acc = __dadd_rn(acc, __dmul_rn(x, x));
  }
  return acc;
}

// Seeding (memostore.cpp:50-84) in one CTA: the distance updates run in
// parallel, the total and the cumulative scan on one thread in key order.
__global__ void __launch_bounds__(kKmThreads) k_km_seed(const float* __restrict__ keys, int nk, int dim, int k,
                                                        const unsigned long long* __restrict__ draws,
                                                        float* __restrict__ cent) {
  extern __shared__ double km_smem[];
  double* dist2 = km_smem;  // [nk]
  __shared__ int pick;
  const int tid = threadIdx.x, bd = blockDim.x;
  if (tid == 0) pick = static_cast<int>(draws[0] % static_cast<unsigned long long>(nk));
  for (int i = tid; i < nk; i += bd) dist2[i] = 1.7976931348623157e308;
  __syncthreads();
  for (int c = 0;; ++c) {
    const int p = pick;
    for (int d = tid; d < dim; d += bd) cent[c * dim + d] = keys[static_cast<long long>(p) * dim + d];
    __syncthreads();
    if (c + 1 == k) break;
    for (int i = tid; i < nk; i += bd) {
      const double d = km_l2(keys + static_cast<long long>(i) * dim, cent + c * dim, dim);
      if (d < dist2[i]) dist2[i] = d;
    }
    __syncthreads();
    if (tid == 0) {
      // the sequential sums in key order (bit-identical), 8 values per chunk so the
      // shared-memory loads run ahead of the dependent adds
      double total = 0.0;
      int i = 0;
      for (; i + 8 <= nk; i += 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = dist2[i + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) total = __dadd_rn(total, x[u]);
      }
      for (; i < nk; ++i) total = __dadd_rn(total, dist2[i]);
      int q = 0;
      if (total > 0.0) {
        const double target = __dmul_rn(static_cast<double>(draws[c + 1] >> 11) * 0x1.0p-53, total);
        double run = 0.0;
        q = nk - 1;
        bool found = false;
        for (i = 0; i + 8 <= nk && !found; i += 8) {
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = dist2[i + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            run = __dadd_rn(run, x[u]);
            if (!found && run >= target) {
              q = i + u;
              found = true;
            }
          }
        }
        for (; i < nk && !found; ++i) {
          run = __dadd_rn(run, dist2[i]);
          if (run >= target) {
            q = i;
            found = true;
          }
        }
      } else {
        q = static_cast<int>(draws[c + 1] % static_cast<unsigned long long>(nk));
      }
      pick = q;
    }
    __syncthreads();
  }
}

// Lloyd step 1: every (key, centroid) distance, one thread each.
__global__ void k_km_dist(const float* __restrict__ keys, int nk, int dim, int k, const float* __restrict__ cent,
                          double* __restrict__ dist) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<long long>(nk) * k) return;
  const int i = static_cast<int>(t / k), c = static_cast<int>(t - static_cast<long long>(i) * k);
  dist[t] = km_l2(keys + static_cast<long long>(i) * dim, cent + c * dim, dim);
}
// Lloyd step 2: each key's nearest centroid in centroid order (lower index wins ties).
__global__ void k_km_assign(const double* __restrict__ dist, int nk, int k, int* __restrict__ owner) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nk) return;
  double best = 1.7976931348623157e308;
  int arg = 0;
  for (int c = 0; c < k; ++c) {
    const double d = dist[static_cast<long long>(i) * k + c];
    if (d < best) {
      best = d;
      arg = c;
    }
  }
  owner[i] = arg;
}
// Lloyd step 3: centroid (c, d) = mean of its keys' coordinate d, summed in key order.
__global__ void k_km_update(const float* __restrict__ keys, int nk, int dim, int k, const int* __restrict__ owner,
                            float* __restrict__ cent) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= k * dim) return;
  const int c = o / dim, d = o - c * dim;
  double sum = 0.0;
  int cnt = 0;
  for (int i = 0; i < nk; ++i)
    if (__ldg(owner + i) == c) {
      ++cnt;
      sum = __dadd_rn(sum, static_cast<double>(__ldg(keys + static_cast<long long>(i) * dim + d)));
    }
  if (cnt) cent[o] = __double2float_rn(__ddiv_rn(sum, static_cast<double>(cnt)));  // empty: keep
}

}  // namespace

struct KmeansScratch {
  cudaStream_t s = nullptr;
  DeviceBuffer<float> keys, cent;
  DeviceBuffer<double> dist;
  DeviceBuffer<int> owner;
  DeviceBuffer<unsigned long long> draws;
  ~KmeansScratch() {
    if (s) cudaStreamDestroy(s);
  }
};

void kmeans_seed_attr() {
  static std::once_flag once;
  std::call_once(once, [] {
    MLRG_CUDA(cudaFuncSetAttribute(k_km_seed, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
}

void gpu_kmeans(const std::vector<std::vector<float>>& keys, int k, std::uint64_t seed, int iters,
                std::vector<std::vector<float>>& cent, std::vector<std::size_t>& nearest, int device,
                KmeansScratch* scratch) {
  if (keys.empty()) throw std::invalid_argument("kmeans: no keys");
  MLRG_CUDA(cudaSetDevice(device));  // may run on a host worker thread
  KmeansScratch local;
  KmeansScratch& w = scratch ? *scratch : local;
  if (!w.s) MLRG_CUDA(cudaStreamCreateWithFlags(&w.s, cudaStreamNonBlocking));
  const int nk = static_cast<int>(keys.size()), dim = static_cast<int>(keys.front().size());
  k = std::min(k, nk);
  std::mt19937_64 rng(seed);  // kmeans_train's draws: one for the first centroid, one per further centroid
  std::vector<unsigned long long> draws(static_cast<std::size_t>(k));
  for (auto& d : draws) d = rng();
  std::vector<float> flat(static_cast<std::size_t>(nk) * dim);
  for (int i = 0; i < nk; ++i) std::copy(keys[i].begin(), keys[i].end(), flat.begin() + static_cast<std::ptrdiff_t>(i) * dim);
  kmeans_seed_attr();
  w.keys.upload(flat, w.s);
  w.draws.upload(draws, w.s);
  w.cent.resize(static_cast<std::size_t>(k) * dim);
  w.dist.resize(static_cast<std::size_t>(nk) * k);
  w.owner.resize(static_cast<std::size_t>(nk));
  k_km_seed<<<1, kKmThreads, sizeof(double) * static_cast<std::size_t>(nk), w.s>>>(w.keys.get(), nk, dim, k, w.draws.get(),
                                                                                 w.cent.get());
  MLRG_LAUNCH_CHECK("k_km_seed");
  const long long pairs = static_cast<long long>(nk) * k;
  const unsigned gd = static_cast<unsigned>((pairs + 255) / 256), ga = static_cast<unsigned>((nk + 255) / 256),
                 gu = static_cast<unsigned>((k * dim + 127) / 128);
  for (int it = 0; it <= iters; ++it) {  // iters Lloyd steps, then the final assignment
    k_km_dist<<<gd, 256, 0, w.s>>>(w.keys.get(), nk, dim, k, w.cent.get(), w.dist.get());
    k_km_assign<<<ga, 256, 0, w.s>>>(w.dist.get(), nk, k, w.owner.get());
    if (it < iters) k_km_update<<<gu, 128, 0, w.s>>>(w.keys.get(), nk, dim, k, w.owner.get(), w.cent.get());
  }
  MLRG_LAUNCH_CHECK("k_km_lloyd");
  std::vector<float> hc(static_cast<std::size_t>(k) * dim);
  std::vector<int> hn(static_cast<std::size_t>(nk));
  MLRG_CUDA(cudaMemcpyAsync(hc.data(), w.cent.get(), hc.size() * sizeof(float), cudaMemcpyDeviceToHost, w.s));
  MLRG_CUDA(cudaMemcpyAsync(hn.data(), w.owner.get(), hn.size() * sizeof(int), cudaMemcpyDeviceToHost, w.s));
  MLRG_CUDA(cudaStreamSynchronize(w.s));
  cent.assign(static_cast<std::size_t>(k), std::vector<float>(static_cast<std::size_t>(dim)));
  for (int c = 0; c < k; ++c) std::copy(hc.begin() + static_cast<std::ptrdiff_t>(c) * dim, hc.begin() + static_cast<std::ptrdiff_t>(c + 1) * dim, cent[c].begin());
  nearest.assign(hn.begin(), hn.end());
}

// Setup-time preparation of the trainer (the solve's DeviceMemo constructor):
// its stream, scratch for up to `nk` keys, the seed kernel's shared-memory
// opt-in, and the k-means kernels' modules loaded (lazy loading would load
// them at the first training, inside an iteration), so the training
// iteration makes no driver calls beyond its launches and copies.
void gpu_kmeans_prepare(KmeansScratch* w, int nk, int k, int dim) {
  if (!w->s) MLRG_CUDA(cudaStreamCreateWithFlags(&w->s, cudaStreamNonBlocking));
  k = std::min(k, nk);
  w->keys.resize(static_cast<std::size_t>(nk) * dim);
  w->draws.resize(static_cast<std::size_t>(k));
  w->cent.resize(static_cast<std::size_t>(k) * dim);
  w->dist.resize(static_cast<std::size_t>(nk) * k);
  w->owner.resize(static_cast<std::size_t>(nk));
  cudaFuncAttributes fa{};
  MLRG_CUDA(cudaFuncGetAttributes(&fa, k_km_seed));
  MLRG_CUDA(cudaFuncGetAttributes(&fa, k_km_dist));
  MLRG_CUDA(cudaFuncGetAttributes(&fa, k_km_assign));
  MLRG_CUDA(cudaFuncGetAttributes(&fa, k_km_update));
  kmeans_seed_attr();
}

bool gpu_kmeans_fits(int nk, int k, int dim) {
  return static_cast<std::size_t>(nk) * sizeof(double) <= 200 * 1024 && static_cast<long long>(nk) * k < (1LL << 31) &&
         k * dim > 0;
}

DeviceMemo::DeviceMemo(MemoClient& client, int key_dim, std::uint64_t seed, int max_slabs, std::int64_t max_keys,
                       std::size_t arena_bytes, int window_inserts, cudaStream_t s)
    : client_(client),
      kd_(key_dim),
      max_slabs_(max_slabs),
      max_keys_(max_keys),
      arena_bytes_((arena_bytes + 255) & ~std::size_t{255}),
      log_cap_(std::int64_t{1} << 16) {
  if (kd_ < 1 || kd_ > kMaxKd) throw std::invalid_argument("device memo: key_dim must be in [1, 64]");
  window_inserts_ = std::max(1, window_inserts);
  if (max_slabs_ > kStageThreads) throw std::invalid_argument("device memo: more than 1024 slabs per operator call");
  if (client_.config().global_cache) throw std::invalid_argument("device memo: global_cache is host-only");
  if (client_.store().ivf().nlist > kMaxProbe) throw std::invalid_argument("device memo: nlist must be <= 64");
  {  // the IVF training runs on the GPU (bit-identical to the host k-means)
    int dev = 0;
    MLRG_CUDA(cudaGetDevice(&dev));
    km_ = std::make_unique<KmeansScratch>();
    const IvfConfig& ivf = client_.store().ivf();
    const int nk_max = 2 * ivf.train_size;  // a flush can carry the store past train_size
    if (gpu_kmeans_fits(nk_max, ivf.nlist, kd_)) gpu_kmeans_prepare(km_.get(), nk_max, ivf.nlist, kd_);
    client_.store().set_trainer([dev, this](const std::vector<std::vector<float>>& keys, int k, std::uint64_t seed, int iters,
                                      std::vector<std::vector<float>>& cent, std::vector<std::size_t>& nearest) {
      const int dim = keys.empty() ? 0 : static_cast<int>(keys.front().size());
      if (!gpu_kmeans_fits(static_cast<int>(keys.size()), k, dim)) {
        cent = kmeans_train(keys, k, seed, iters);
        nearest.resize(keys.size());
        for (std::size_t i = 0; i < keys.size(); ++i) {
          double best = std::numeric_limits<double>::max();
          for (std::size_t c = 0; c < cent.size(); ++c) {
            const double d = l2_sq(keys[i].data(), cent[c].data(), dim);
            if (d < best) {
              best = d;
              nearest[i] = c;
            }
          }
        }
        return;
      }
      gpu_kmeans(keys, k, seed, iters, cent, nearest, dev, km_.get());
    });
  }
  const std::size_t per_key = 8 + 4 * static_cast<std::size_t>(kd_);
  batch_keys_ = static_cast<int>((client_.config().coalesce_bytes + per_key - 1) / per_key);
  keys_.resize(static_cast<std::size_t>(max_keys_ * kd_));
  vbytes_.resize(static_cast<std::size_t>(max_keys_));
  vnorm_.resize(static_cast<std::size_t>(max_keys_));
  vptr_.resize(static_cast<std::size_t>(max_keys_));
  const std::size_t slots = 4 * static_cast<std::size_t>(max_slabs_);
  cache_key_.resize(slots * kd_);
  cache_vid_.resize(slots);
  std::vector<long long> neg(slots, -1);
  cache_vid_.upload(neg.data(), neg.size(), s);
  // slot_mix (encoder.cpp:66-86) as gather tables per (op, location)
  std::vector<int> perm(slots * kd_);
  std::vector<float> sign(slots * kd_);
  for (int op = 0; op < 4; ++op)
    for (int loc = 0; loc < max_slabs_; ++loc) {
      const std::size_t base = (static_cast<std::size_t>(op) * max_slabs_ + loc) * kd_;
      // the mix of a one-hot vector e_i is sign_j at j with perm[j] = i; recover both
      std::vector<float> probe(static_cast<std::size_t>(kd_));
      for (int i = 0; i < kd_; ++i) {
        std::fill(probe.begin(), probe.end(), 0.0f);
        probe[static_cast<std::size_t>(i)] = 1.0f;
        slot_mix(probe.data(), kd_, seed, loc, static_cast<OpId>(op));
        for (int j = 0; j < kd_; ++j)
          if (probe[static_cast<std::size_t>(j)] != 0.0f) {
            perm[base + j] = i;
            sign[base + j] = probe[static_cast<std::size_t>(j)];
          }
      }
    }
  mix_perm_.upload(perm, s);
  mix_sign_.upload(sign, s);
  arena_.resize(arena_bytes_);
  state_.resize(6);
  state_.zero(s);
  slabs_.resize(static_cast<std::size_t>(max_slabs_));
  skip_.resize(static_cast<std::size_t>(max_slabs_));
  slab_vbytes_.resize(static_cast<std::size_t>(4 * max_slabs_));
  slab_counts_.resize(static_cast<std::size_t>(4 * max_slabs_));
  flags_.resize(static_cast<std::size_t>(2 * max_slabs_));
  qkeys_.resize(static_cast<std::size_t>(max_slabs_) * kd_);
  log_.resize(static_cast<std::size_t>(log_cap_));
  centroids_.resize(static_cast<std::size_t>(client_.store().ivf().nlist) * kd_);
  cl_ptr_.resize(static_cast<std::size_t>(client_.store().ivf().nlist) + 1);
  cl_ids_.resize(static_cast<std::size_t>(max_keys_));
  h_state_.reserve(6);
  MLRG_CUDA(cudaStreamSynchronize(s));
}

void DeviceMemo::set_slabs(OpId op, const std::vector<std::size_t>& value_bytes,
                           const std::vector<std::int64_t>& out_counts, cudaStream_t s) {
  const int o = static_cast<int>(op);
  if (o > 3 || static_cast<int>(value_bytes.size()) > max_slabs_) throw std::logic_error("device memo: bad slab table");
  std::vector<long long> vb(value_bytes.begin(), value_bytes.end()), oc(out_counts.begin(), out_counts.end());
  for (const std::int64_t c : out_counts)
    max_slab_bytes_ = std::max(max_slab_bytes_, ValueRing::granule(static_cast<std::size_t>(c) * sizeof(float2)));
  // fail at setup, not mid-solve: one window of inserts (+ the wrap of one
  // slab) must fit the ring; everything older can spill to the cold tier
  const std::size_t need = (static_cast<std::size_t>(window_inserts_) + 1) * max_slab_bytes_;
  if (arena_bytes_ < need)
    throw std::invalid_argument("device memo: value arena of " + std::to_string(arena_bytes_) +
                                " bytes is below one insert window (" + std::to_string(need) + " bytes)");
  spiller_ = std::make_unique<ColdSpiller>(
      arena_.get(), arena_bytes_, static_cast<std::size_t>(window_inserts_) * max_slab_bytes_,
      [this](const std::vector<std::uint64_t>& ids, const std::vector<const void*>& ptrs, cudaStream_t st) {
        for (std::size_t i = 0; i < ids.size(); ++i) {  // pageable source: staged before the call returns
          MLRG_CUDA(cudaMemcpyAsync(vptr_.get() + ids[i], &ptrs[i], sizeof(void*), cudaMemcpyHostToDevice, st));
          client_.store().set_value_ptr(ids[i], static_cast<const float2*>(ptrs[i]));
        }
      });
  MLRG_CUDA(cudaMemcpyAsync(slab_vbytes_.get() + o * max_slabs_, vb.data(), vb.size() * sizeof(long long),
                            cudaMemcpyHostToDevice, s));
  MLRG_CUDA(cudaMemcpyAsync(slab_counts_.get() + o * max_slabs_, oc.data(), oc.size() * sizeof(long long),
                            cudaMemcpyHostToDevice, s));
  MLRG_CUDA(cudaStreamSynchronize(s));
}

DeviceMemo::~DeviceMemo() {
  if (pending_.valid()) pending_.wait();
  if (rb_) {
    cudaStreamSynchronize(rb_);
    cudaStreamDestroy(rb_);
  }
  if (fp_) cudaEventDestroy(fp_);
  if (rb_done_) cudaEventDestroy(rb_done_);
}

void DeviceMemo::mark(cudaStream_t s) {
  if (!rb_) {
    MLRG_CUDA(cudaStreamCreateWithFlags(&rb_, cudaStreamNonBlocking));
    MLRG_CUDA(cudaEventCreateWithFlags(&fp_, cudaEventDisableTiming));
    MLRG_CUDA(cudaEventCreateWithFlags(&rb_done_, cudaEventDisableTiming));
  }
  MLRG_CUDA(cudaEventRecord(fp_, s));
  marked_ = true;
}

void DeviceMemo::join(cudaStream_t s) {
  if (!pending_.valid()) return;
  pending_.get();  // rethrows a failure of the store update
  if (pending_spill_) spill(s);
  pending_spill_ = false;
  upload_ivf(s);
}

void DeviceMemo::lookup(OpId op, int n, const float* keys, const double* norms2, int iteration, cudaStream_t s) {
  join(s);
  const int o = static_cast<int>(op);
  if (n > max_slabs_) throw std::logic_error("device memo: too many slabs");
  if (o > 3) throw std::logic_error("device memo: operator not memoizable on the device");
  const long long* svb = slab_vbytes_.get() + o * max_slabs_;
  const long long* scn = slab_counts_.get() + o * max_slabs_;
  LookupArgs la{o, n, kd_, client_.config().nprobe, ncent_, trained_ ? 1 : 0, max_slabs_,
                client_.config().tau, keys, mix_perm_.get(), mix_sign_.get(), qkeys_.get(), cache_key_.get(),
                cache_vid_.get(), keys_.get(), vbytes_.get(), svb, centroids_.get(), cl_ptr_.get(),
                cl_ids_.get(), state_.get(), slabs_.get(), flags_.get(), flags_.get() + max_slabs_};
  prof::begin("k_memo_lookup", s);
  k_memo_lookup<<<n, kLookupThreads, 0, s>>>(la);
  prof::end("k_memo_lookup", s);
  MLRG_LAUNCH_CHECK("k_memo_lookup");
  StageArgs sa{n, kd_, o, iteration, static_cast<int>(client_.config().insert_queue_cap),
               static_cast<long long>(arena_bytes_), log_cap_, qkeys_.get(), norms2, svb, scn, keys_.get(),
               vbytes_.get(), vnorm_.get(), vptr_.get(), arena_.get(), state_.get(), slabs_.get(), skip_.get(),
               la.probed, la.queried, log_.get()};
  prof::begin("k_memo_stage", s);
  k_memo_stage<<<1, static_cast<unsigned>((n + 31) / 32 * 32), 0, s>>>(sa);
  prof::end("k_memo_stage", s);
  MLRG_LAUNCH_CHECK("k_memo_stage");
}

void DeviceMemo::upload_ivf(cudaStream_t s) {
  prof::HostSpan span("host:memo_upload_ivf");
  const MemoStore& st = client_.store();
  if (!st.trained()) return;
  const auto& cents = st.centroids();
  ncent_ = static_cast<int>(cents.size());
  std::vector<float> c(static_cast<std::size_t>(ncent_) * kd_);
  for (int i = 0; i < ncent_; ++i) std::copy(cents[i].begin(), cents[i].end(), c.begin() + static_cast<std::ptrdiff_t>(i) * kd_);
  const auto lists = st.cluster_ids();
  std::vector<int> ptr(lists.size() + 1, 0), ids;
  for (std::size_t i = 0; i < lists.size(); ++i) {
    ptr[i + 1] = ptr[i] + static_cast<int>(lists[i].size());
    for (std::uint64_t id : lists[i]) ids.push_back(static_cast<int>(id));
  }
  MLRG_CUDA(cudaMemcpyAsync(centroids_.get(), c.data(), c.size() * sizeof(float), cudaMemcpyHostToDevice, s));
  MLRG_CUDA(cudaMemcpyAsync(cl_ptr_.get(), ptr.data(), ptr.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  if (!ids.empty())
    MLRG_CUDA(cudaMemcpyAsync(cl_ids_.get(), ids.data(), ids.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  MLRG_CUDA(cudaStreamSynchronize(s));  // the host vectors die here
  trained_ = true;
}

// Frees the ring span the next window can fill (ColdSpiller: the oldest
// values overlapping it move to pinned host memory and their value pointers
// are repointed there, partly in the background); decisions and ids are unaffected.
void DeviceMemo::spill(cudaStream_t s) {
  prof::HostSpan span("host:memo_spill");
  spiller_->ring().reset_head(static_cast<std::size_t>(h_state_.get()[2]));
  spiller_->flush(s);
}

void DeviceMemo::flush(cudaStream_t s, std::vector<Audit>* audit, bool publish) {
  const bool joined = pending_.valid();
  join(s);
  // after a mark (and no join work just enqueued on s), the readback and the
  // state update run on the readback stream behind the mark
  cudaStream_t rs = s;
  if (marked_ && !joined) {
    rs = rb_;
    MLRG_CUDA(cudaStreamWaitEvent(rb_, fp_, 0));
  }
  marked_ = false;
  MLRG_CUDA(cudaMemcpyAsync(h_state_.get(), state_.get(), 6 * sizeof(long long), cudaMemcpyDeviceToHost, rs));
  MLRG_CUDA(cudaStreamSynchronize(rs));
  long long* st = h_state_.get();
  const long long npub = st[0], nstaged = publish ? st[1] : 0, nlog = st[3];
  if (st[4]) throw std::logic_error("device memo: a value larger than the arena (" + std::to_string(arena_bytes_) + " bytes)");
  if (nlog > log_cap_) throw std::runtime_error("device memo: decision log overflow");
  std::vector<DevLog> log(static_cast<std::size_t>(nlog));
  if (nlog) MLRG_CUDA(cudaMemcpyAsync(log.data(), log_.get(), sizeof(DevLog) * nlog, cudaMemcpyDeviceToHost, rs));
  std::vector<float> keys(static_cast<std::size_t>(nstaged) * kd_);
  std::vector<long long> vb(static_cast<std::size_t>(nstaged));
  std::vector<double> vn(static_cast<std::size_t>(nstaged));
  std::vector<const float2*> vp(static_cast<std::size_t>(nstaged));
  if (nstaged) {
    MLRG_CUDA(cudaMemcpyAsync(keys.data(), keys_.get() + npub * kd_, keys.size() * sizeof(float), cudaMemcpyDeviceToHost, rs));
    MLRG_CUDA(cudaMemcpyAsync(vb.data(), vbytes_.get() + npub, vb.size() * sizeof(long long), cudaMemcpyDeviceToHost, rs));
    MLRG_CUDA(cudaMemcpyAsync(vn.data(), vnorm_.get() + npub, vn.size() * sizeof(double), cudaMemcpyDeviceToHost, rs));
    MLRG_CUDA(cudaMemcpyAsync(vp.data(), vptr_.get() + npub, vp.size() * sizeof(void*), cudaMemcpyDeviceToHost, rs));
  }
  MLRG_CUDA(cudaStreamSynchronize(rs));
  // ---- replay the decisions into the client's counters and the audit ----
  MemoCounters& ctr = client_.counters_mut();
  long long queried_in_call = 0;
  for (std::size_t i = 0; i < log.size(); ++i) {
    const DevLog& e = log[i];
    ++ctr.lookups;
    ctr.cache_probes += static_cast<std::uint64_t>(e.probed);
    ctr.cache_comparisons += static_cast<std::uint64_t>(e.probed);
    if (e.outcome == 2) ++ctr.cache_hits;
    else if (e.outcome == 1) ++ctr.remote_hits;
    else ++ctr.misses;
    if (e.staged == 1) ++ctr.inserts_enqueued;
    if (e.staged == 0) ++ctr.inserts_dropped;
    queried_in_call += e.queried;
    const bool call_end = i + 1 == log.size() || log[i + 1].location == 0;
    if (call_end) {  // coalesced store batches of this call (memoclient.cpp:228-246)
      ctr.batches_sent += static_cast<std::uint64_t>((queried_in_call + batch_keys_ - 1) / batch_keys_);
      queried_in_call = 0;
    }
    if (audit) audit->push_back(Audit{e.iteration, e.op, e.location, e.outcome, e.cs});
  }
  // ---- publish: the host mirror gets the staged keys in order (same ids) ----
  MemoStore& store = client_.store();
  const bool was_trained = store.trained();
  const char* arena = arena_.get();
  std::vector<ValueRef> vals(static_cast<std::size_t>(nstaged));
  for (long long i = 0; i < nstaged; ++i) {
    ValueRef& v = vals[static_cast<std::size_t>(i)];
    v.dev = vp[static_cast<std::size_t>(i)];
    spiller_->ring().note(static_cast<std::uint64_t>(npub + i),
                          static_cast<std::size_t>(reinterpret_cast<const char*>(v.dev) - arena),
                          static_cast<std::size_t>(vb[static_cast<std::size_t>(i)] - 8) / 2);
    v.norm = vn[static_cast<std::size_t>(i)];
    v.bytes = static_cast<std::size_t>(vb[static_cast<std::size_t>(i)]);
    v.count = static_cast<std::int64_t>((v.bytes - 8) / 16);
  }
  ctr.inserts_sent += static_cast<std::uint64_t>(nstaged);
  auto insert_all = [this, &store, npub, nstaged, keys = std::move(keys), vals = std::move(vals)]() {
    for (long long i = 0; i < nstaged; ++i) {
      const std::vector<float> k(keys.begin() + i * kd_, keys.begin() + (i + 1) * kd_);
      const std::uint64_t id = store.insert(k, vals[static_cast<std::size_t>(i)]);
      if (static_cast<long long>(id) != npub + i) throw std::logic_error("device memo: id mismatch with the host mirror");
    }
  };
  st[3] = 0;  // the log is drained either way
  if (publish) {
    st[0] = npub + nstaged;
    st[1] = 0;
    st[5] = 0;
  }
  MLRG_CUDA(cudaMemcpyAsync(state_.get(), st, 6 * sizeof(long long), cudaMemcpyHostToDevice, rs));
  if (rs != s) {  // the next lookups on s come after the state update
    MLRG_CUDA(cudaEventRecord(rb_done_, rs));
    MLRG_CUDA(cudaStreamWaitEvent(s, rb_done_, 0));
  }
  MLRG_CUDA(cudaStreamSynchronize(rs));
  if (st[0] > max_keys_ - static_cast<long long>(client_.config().insert_queue_cap))
    throw std::runtime_error("device memo: key index full (" + std::to_string(max_keys_) + " keys)");
  const bool trains = !was_trained && static_cast<long long>(store.key_count()) + nstaged >= store.ivf().train_size;
  if (trains) {
    // the k-means training runs on a host thread while the GPU continues; the
    // spill (it repoints stored values by id) and the IVF upload wait for it (join)
    pending_ = std::async(std::launch::async, std::move(insert_all));
    pending_spill_ = publish;
    return;
  }
  insert_all();
  if (publish) spill(s);
  if (store.trained() && (nstaged > 0 || !was_trained)) upload_ivf(s);
}

}  // namespace mlrg
