// The laminography USFFT operators on one B200: fu1d / fu1d_adj (1D gridding
// along axis 1 of the volume), fu2d / fu2d_adj (2D gridding per detector
// row), and the centred unitary 2D DFT f2d / f2d_adj. All arrays are device
// complex64 (float2) in the reference's row-major layouts (array.hpp:38-73).
//
// Reference operators replaced (numerically, to fp32 rounding; the spreading
// kernel is selectable, geometry.hpp):
//   nufft::fu1d_gridding      nufft.cpp:107-134
//   nufft::fu1d_adj_gridding  nufft.cpp:136-162
//   nufft::fu2d_gridding      nufft.cpp:183-225  (+ fused_sub_fu2d, operators.cpp:285-299)
//   nufft::fu2d_adj_gridding  nufft.cpp:227-267
//   f2d / f2d_adj             operators.cpp:39-74, 249-259
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "device.hpp"
#include "geometry.hpp"

namespace mlrg {

/// Output stage of fu2d: val = fac * acc - sub; stores val to `out` when set
/// and, when `reduce` is set, accumulates sum |val|^2 and Re<dot, val> into
/// the per-CTA partials (2 doubles per CTA, summed across row batches).
struct Fu2dEpilogue {
  float2* out = nullptr;
  std::int64_t ld_out = 0, k0_out = 0;
  const float2* sub = nullptr;
  std::int64_t ld_sub = 0, k0_sub = 0;
  const float2* dot = nullptr;
  std::int64_t ld_dot = 0, k0_dot = 0;
  bool reduce = false;
  /// Also leave the adjoint's class sums of the (rounded) output in the
  /// operator, so a following fu2d_adj of exactly this output skips its
  /// k_fu2d_adj_prep pass (the solver's r = fu2d(v) - d, then fu2d_adj(r)).
  bool class_sums = false;
};

/// Sharded output of fu1d / fu2d_adj (the fused all-to-all):
/// the producing kernel stores every output row straight into the HBM of the
/// rank that owns it (CUDA IPC mappings, P2P over NVLink), so the exchange
/// overlaps the transform tile by tile. world == 0: plain local output.
struct PeerOut {
  static constexpr int kMax = 8;
  int world = 0;
  std::int64_t lo[kMax] = {}, hi[kMax] = {};  // owned range per rank (rows for fu1d, planes for fu2d_adj)
  float2* dst[kMax] = {};                     // each rank's destination block
  std::int64_t off = 0;  // fu1d: global plane of local plane 0; fu2d_adj: global row of local row 0
  std::int64_t h = 0;    // fu2d_adj: detector rows of the destination blocks
};

class Usfft {
 public:
  static constexpr int kRowBatch = 16;  // detector rows per fu2d grid batch

  Usfft(const Geometry& g, cudaStream_t stream, GridKernel kernel = GridKernel::es);
  ~Usfft();
  Usfft(const Usfft&) = delete;
  Usfft& operator=(const Usfft&) = delete;

  const Geometry& geometry() const { return g_; }
  GridKernel kernel() const { return kernel_; }
  cudaStream_t stream() const { return stream_; }

  /// u: contiguous (d0, n0, n2) -> out (d0, h, n2). The volume side may be
  /// complex128 (the solver's iterate); the transform runs in complex64.
  void fu1d(const float2* u, float2* out, std::int64_t d0);
  void fu1d(const double2* u, float2* out, std::int64_t d0, const PeerOut* peer = nullptr);
  /// v: contiguous (d0, h, n2) -> out (d0, n0, n2).
  void fu1d_adj(const float2* v, float2* out, std::int64_t d0);
  void fu1d_adj(const float2* v, double2* out, std::int64_t d0);

  /// Rows [k0, k0+nk) of an (n1, ld, n2) array -> rows of an (n_theta, ., w)
  /// array via the epilogue. Returns the number of partial doubles written
  /// (2 per gather CTA) when epi.reduce is set, else 0.
  int fu2d(const float2* v, std::int64_t ld, std::int64_t k0, std::int64_t nk, const Fu2dEpilogue& epi);
  /// Plan figures for measurement: fu2d target classes per detector row, kernel
  /// taps per dimension, oversampled grid extents, gather CTAs per row batch.
  struct Stats {
    std::int64_t nclass, taps, m1, m2, gather_ctas, classes_per_cta;
  };
  Stats stats() const;
  /// Rows [k0, k0+nk) of an (n_theta, ld, w) array -> rows [k0_out, k0_out+nk)
  /// of an (n1, ld_out, n2) array.
  void fu2d_adj(const float2* p, std::int64_t ld, std::int64_t k0, std::int64_t nk, float2* out,
                std::int64_t ld_out, std::int64_t k0_out, const PeerOut* peer = nullptr);

  /// Centred unitary 2D DFT of `count` contiguous (h, w) planes.
  void f2d(const float2* p, float2* out, std::int64_t count, bool adjoint);

  Partials& partials() { return partials_; }
  /// Device-side memo: per-16-slab skip flags (a hit slab's CTAs exit at entry)
  /// for the next calls; nullptr clears.
  void set_skip(const unsigned char* flags) { skip_ = flags; }
  /// Drops the class sums a class_sums fu2d left (the output may change next).
  void forget_class_sums() { cls_src_ = nullptr; }
  int reduce_grid() const;  // CTAs of an elementwise reduction kernel

 private:
  template <class TIn>
  void fu1d_t(const TIn* u, float2* out, std::int64_t d0, const PeerOut* peer);
  template <class TOut>
  void fu1d_adj_t(const float2* v, TOut* out, std::int64_t d0);
  void ensure_side();  // second stream + grids for the pipelined row batches
  /// Runs `enqueue` (the kernels of one fu2d / fu2d_adj call) through a CUDA graph
  /// captured for its exact arguments `key` on the call's second occurrence and
  /// replayed from then on (MLRG_GRAPHS=0: plain launches; never while profiling).
  template <class F>
  void graph_run(const std::string& key, F&& enqueue);
  struct Graphs;
  Graphs* graphs_ = nullptr;
  struct Tables;
  Geometry g_;
  cudaStream_t stream_;
  GridKernel kernel_;
  Tables* t_;
  Partials partials_;
  const unsigned char* skip_ = nullptr;
  // class sums of the last class_sums fu2d: its output array and row range
  const float2* cls_src_ = nullptr;
  std::int64_t cls_ld_ = 0, cls_k0_ = 0, cls_nk_ = 0;
};

}  // namespace mlrg
