// Node-local communicator for the z-slab sharded solver:
// one process per GPU, all on one node. The control plane is a POSIX
// shared-memory segment (barrier, deterministic scalar allreduce, allgather
// of memo keys and CUDA IPC handles); the data plane is device memory of the
// peers mapped through CUDA IPC, written directly by this library's kernels
// (P2P stores over NVLink/NVSwitch on a multi-GPU node; the same code runs
// several ranks on one GPU in the tests).
//
// The reference shards nothing across processes: its OperatorEngine splits
// every apply into 16-slabs over worker threads (scalerun.cpp:14-27, 168-287).
// The sharded build keeps those slabs and that assign() partition, one range
// of slabs per rank.
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace mlrg {

/// assign(n_chunks, n_workers) (scalerun.cpp:14-27): contiguous ranges, the
/// first n_chunks % n_workers ranges one chunk longer.
std::vector<std::pair<std::int64_t, std::int64_t>> assign_ranges(std::int64_t n_chunks, int n_workers);

class HostComm {
 public:
  /// Joins (rank 0 creates) the segment `name`; blocks until all `world`
  /// ranks have joined or `timeout_s` passes (std::runtime_error).
  HostComm(const std::string& name, int rank, int world, double timeout_s = 120.0);
  ~HostComm();
  HostComm(const HostComm&) = delete;
  HostComm& operator=(const HostComm&) = delete;

  int rank() const { return rank_; }
  const std::string& name() const { return name_; }
  int world() const { return world_; }

  void barrier();
  /// Marks the job failed: every rank blocked in (or entering) a collective
  /// throws instead of waiting for this one.
  void abort();
  /// In place: v[i] = sum over ranks (added in rank order, so every rank gets
  /// the bit-identical result).
  void allreduce_sum(double* v, int n);
  /// out[r * bytes .. (r+1) * bytes) = rank r's `in` (bytes <= slot_bytes()).
  void allgather(const void* in, std::size_t bytes, void* out);
  /// Variable-size allgather: returns every rank's bytes, concatenated in
  /// rank order; counts[r] = rank r's byte count.
  std::vector<unsigned char> allgatherv(const void* in, std::size_t bytes, std::vector<std::size_t>* counts);
  std::size_t slot_bytes() const;

 private:
  struct Header;
  unsigned char* slot(int bank, int r) const;
  std::string name_;
  int rank_, world_;
  int fd_ = -1;
  std::size_t size_ = 0;
  Header* hdr_ = nullptr;
  std::uint64_t epoch_ = 0;  // per-rank count of bank uses (all ranks agree)
};

}  // namespace mlrg
