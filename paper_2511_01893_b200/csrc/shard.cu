// Sharding plumbing: the partition, CUDA IPC peer mappings, and the all-to-all
// scatter kernels that move the mid array between the plane-sharded (fu1d
// side) and row-sharded (fu2d side) layouts with direct stores into peer HBM.
#include "shard.hpp"

#include <cstring>
#include <stdexcept>
#include <string>

#include "device.hpp"

namespace mlrg {

namespace {
std::vector<std::pair<std::int64_t, std::int64_t>> slab_ranges(std::int64_t len, std::int64_t chunk, int world) {
  const std::int64_t nslabs = (len + chunk - 1) / chunk;
  if (nslabs < world)
    throw std::invalid_argument("shard: " + std::to_string(nslabs) + " slabs of " + std::to_string(chunk) +
                                " cannot give each of " + std::to_string(world) + " ranks one");
  auto r = assign_ranges(nslabs, world);
  for (auto& [lo, hi] : r) {
    lo = std::min(len, lo * chunk);
    hi = std::min(len, hi * chunk);
  }
  return r;
}
}  // namespace

Shard Shard::whole(const Geometry& g, std::int64_t chunk) {
  Shard s;
  s.chunk = chunk;
  s.planes = {{0, g.n1}};
  s.rows = {{0, g.h}};
  return s;
}

Shard Shard::make(const Geometry& g, std::int64_t chunk, std::shared_ptr<HostComm> comm) {
  if (!comm) return whole(g, chunk);
  Shard s;
  s.rank = comm->rank();
  s.world = comm->world();
  s.comm = std::move(comm);
  s.chunk = chunk;
  s.planes = slab_ranges(g.n1, chunk, s.world);
  s.rows = slab_ranges(g.h, chunk, s.world);
  return s;
}

int Shard::owner_of_plane(std::int64_t i) const {
  for (int r = 0; r < world; ++r)
    if (i < planes[static_cast<std::size_t>(r)].second) return r;
  return world - 1;
}

int Shard::owner_of_row(std::int64_t k) const {
  for (int r = 0; r < world; ++r)
    if (k < rows[static_cast<std::size_t>(r)].second) return r;
  return world - 1;
}

PeerMemory::PeerMemory(HostComm& comm, void* local) : rank_(comm.rank()) {
  const int world = comm.world();
  ptrs_.assign(static_cast<std::size_t>(world), nullptr);
  ptrs_[static_cast<std::size_t>(rank_)] = local;
  if (world == 1) return;
  cudaIpcMemHandle_t mine{};
  MLRG_CUDA(cudaIpcGetMemHandle(&mine, local));
  std::vector<cudaIpcMemHandle_t> all(static_cast<std::size_t>(world));
  comm.allgather(&mine, sizeof(mine), all.data());
  for (int r = 0; r < world; ++r) {
    if (r == rank_) continue;
    void* p = nullptr;
    MLRG_CUDA(cudaIpcOpenMemHandle(&p, all[static_cast<std::size_t>(r)], cudaIpcMemLazyEnablePeerAccess));
    ptrs_[static_cast<std::size_t>(r)] = p;
  }
}

PeerMemory::~PeerMemory() {
  for (std::size_t r = 0; r < ptrs_.size(); ++r)
    if (static_cast<int>(r) != rank_ && ptrs_[r]) cudaIpcCloseMemHandle(ptrs_[r]);
}

PeerEvents::PeerEvents(HostComm& comm) : comm_(comm) {
  const int world = comm.world();
  peers_.assign(static_cast<std::size_t>(world), nullptr);
  MLRG_CUDA(cudaEventCreateWithFlags(&mine_, cudaEventDisableTiming | cudaEventInterprocess));
  if (world == 1) return;
  {
    int dev = 0;
    MLRG_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp prop{};
    MLRG_CUDA(cudaGetDeviceProperties(&prop, dev));
    std::vector<cudaUUID_t> ids(static_cast<std::size_t>(world));
    comm.allgather(&prop.uuid, sizeof(cudaUUID_t), ids.data());
    for (int a = 0; a < world; ++a)
      for (int b = a + 1; b < world; ++b)
        if (std::memcmp(&ids[static_cast<std::size_t>(a)], &ids[static_cast<std::size_t>(b)], sizeof(cudaUUID_t)) == 0)
          distinct_ = false;
  }
  cudaIpcEventHandle_t h{};
  MLRG_CUDA(cudaIpcGetEventHandle(&h, mine_));
  std::vector<cudaIpcEventHandle_t> all(static_cast<std::size_t>(world));
  comm.allgather(&h, sizeof(h), all.data());
  for (int r = 0; r < world; ++r)
    if (r != comm.rank()) MLRG_CUDA(cudaIpcOpenEventHandle(&peers_[static_cast<std::size_t>(r)], all[static_cast<std::size_t>(r)]));
}

PeerEvents::~PeerEvents() {
  for (cudaEvent_t e : peers_)
    if (e) cudaEventDestroy(e);
  if (mine_) cudaEventDestroy(mine_);
}

void PeerEvents::fence(cudaStream_t s) {
  MLRG_CUDA(cudaEventRecord(mine_, s));
  comm_.barrier();  // every rank's record is enqueued before anyone waits on it
  for (cudaEvent_t e : peers_)
    if (e) MLRG_CUDA(cudaStreamWaitEvent(s, e, 0));
}

namespace ops {

namespace {

__device__ __forceinline__ int owner(const RankTable& t, long long x) {
  int r = 0;
  while (r + 1 < t.world && x >= t.hi[r]) ++r;
  return r;
}

// One CTA row-copy per (source row): a row is the n2 contiguous samples of a
// fixed (plane, detector row); the destination row is contiguous too, in the
// owner's array. Vectorised by two complex samples when n2 is even.
template <bool PLANES_TO_ROWS>
__global__ void __launch_bounds__(256) k_scatter(const float2* __restrict__ src, long long nrows_src, long long d1_src,
                                                 long long off, long long h, int n2, RankTable t) {
  for (long long row = blockIdx.x * static_cast<long long>(blockDim.y) + threadIdx.y; row < nrows_src;
       row += static_cast<long long>(gridDim.x) * blockDim.y) {
    const long long i = row / d1_src, kk = row - i * d1_src;  // source (axis-0 index, axis-1 index)
    long long drow;
    int r;
    if (PLANES_TO_ROWS) {  // src (np, h, n2): i local plane, kk global row
      r = owner(t, kk);
      drow = (off + i) * (t.hi[r] - t.lo[r]) + (kk - t.lo[r]);
    } else {  // src (n1, nr, n2): i global plane, kk local row
      r = owner(t, i);
      drow = (i - t.lo[r]) * h + off + kk;
    }
    const float2* s = src + row * n2;
    float2* d = t.dst[r] + drow * n2;
    if ((n2 & 1) == 0) {
      const float4* s4 = reinterpret_cast<const float4*>(s);
      float4* d4 = reinterpret_cast<float4*>(d);
      for (int j = threadIdx.x; j < n2 / 2; j += blockDim.x) d4[j] = s4[j];
    } else {
      for (int j = threadIdx.x; j < n2; j += blockDim.x) d[j] = s[j];
    }
  }
}

dim3 scatter_block(std::int64_t n2) {
  const int tx = n2 >= 256 ? 128 : n2 >= 64 ? 32 : 16;
  return dim3(static_cast<unsigned>(tx), static_cast<unsigned>(256 / tx));
}

}  // namespace

void scatter_planes_to_rows(const float2* src, std::int64_t np, std::int64_t a, std::int64_t n1, std::int64_t h,
                            std::int64_t n2, const RankTable& t, cudaStream_t s) {
  (void)n1;
  const long long nrows = np * h;
  if (nrows == 0) return;
  const dim3 blk = scatter_block(n2);
  const unsigned grid = static_cast<unsigned>(std::min<long long>((nrows + blk.y - 1) / blk.y, 16LL * sm_count()));
  prof::begin("k_scatter", s);
  k_scatter<true><<<grid, blk, 0, s>>>(src, nrows, h, a, h, static_cast<int>(n2), t);
  MLRG_LAUNCH_CHECK("k_scatter");
  prof::end("k_scatter", s);
}

void scatter_rows_to_planes(const float2* src, std::int64_t nr, std::int64_t c, std::int64_t n1, std::int64_t h,
                            std::int64_t n2, const RankTable& t, cudaStream_t s) {
  const long long nrows = n1 * nr;
  if (nrows == 0) return;
  const dim3 blk = scatter_block(n2);
  const unsigned grid = static_cast<unsigned>(std::min<long long>((nrows + blk.y - 1) / blk.y, 16LL * sm_count()));
  prof::begin("k_scatter", s);
  k_scatter<false><<<grid, blk, 0, s>>>(src, nrows, nr, c, h, static_cast<int>(n2), t);
  MLRG_LAUNCH_CHECK("k_scatter");
  prof::end("k_scatter", s);
}

}  // namespace ops
}  // namespace mlrg
