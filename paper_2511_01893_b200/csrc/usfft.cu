// USFFT operator kernels for sm_100a (see usfft.hpp for the reference map).
//
// Data flow per operator (M = oversampled grid = next_pow2(2n)); every FFT is
// the self-sorting radix-8 Stockham transform of common.cuh, in place in
// shared memory, natural order in and out (no bit reversal):
//   fu1d      one CTA per (volume plane i, 8 columns j): wrapped + deconvolved
//             placement fused into the first pass's loads -> M-point FFT
//             (+1) -> W-tap gather per detector row from the tile -> x pref x
//             phase, stored (or sent to the owning rank's mid array, PeerOut).
//   fu1d_adj  mirror: conj-phase load -> W-tap spread in gather form over a
//             host-built cell -> detector-row CSR (no atomics) -> FFT(-1) ->
//             wrapped read x pref x deconv.
//   fu2d      per batch of 16 detector rows, grid layout [M1][M2 + ghost][16]
//             (row batch innermost, 128 B per grid cell): row FFT pass, column
//             FFT pass (four-step passes for M >= 1024), then the W x W-tap
//             gather, one warp per target class (coincident frequencies share
//             one window sum; class records bulk-copied into shared memory).
//   fu2d_adj  mirror: class values -> spread onto 8x4 cell patches from
//             host-built patch lists (warp pairs, no atomics, split lists
//             summed in slot order) -> column FFT(-1) -> row FFT(-1).
// W = 10 (the default es kernel) or 24 (the reference's Gaussian), geometry.hpp.
// FFT butterflies, twiddles, deconvolution and accumulations run in double;
// the oversampled grids between passes are stored in complex64 (complex128
// for the Gaussian plan's gather/spread grids, see to_g).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <future>
#include <unordered_set>
#include <unordered_map>
#include <cstdlib>
#include <numbers>
#include <type_traits>
#include <thread>
#include <utility>
#include <vector>

#include "common.cuh"
#include "usfft.hpp"

namespace mlrg {

namespace {

constexpr int KB = Usfft::kRowBatch;

// Device-side memo (memo_gpu.hpp): a slab whose lookup hit skips its CTAs.
// Unit u of a launch belongs to slab (base + u) / div.
// Grid element of the fu2d forward gather input and the adjoint spread output:
// complex64 for the es kernel; complex128 for the reference's Gaussian plan,
// whose deconvolution (up to e^pi = 23x per dimension, nufft.cpp:66-70) would
// otherwise amplify the complex64 rounding of exactly these two grids into the
// operator outputs (~4e-7 relative, 17x the output rounding, at 64^3).
template <class TG> __device__ __forceinline__ TG to_g(double2 x);
template <> __device__ __forceinline__ float2 to_g<float2>(double2 x) { return to_f(x); }
template <> __device__ __forceinline__ double2 to_g<double2>(double2 x) { return x; }

struct Skip {
  const unsigned char* f = nullptr;
  int base = 0, div = 1;
};
__device__ __forceinline__ bool skipped(const Skip& s, int unit) { return s.f && s.f[(s.base + unit) / s.div]; }

// minimum resident CTAs per SM for the 256-thread 2D grid FFT passes (register cap)
#ifndef MLRG_FFT_MINB
#define MLRG_FFT_MINB 4
#endif
#ifndef MLRG_GATHER_MINB_G
#define MLRG_GATHER_MINB_G 2  // the 24-tap Gaussian windows
#endif
#ifndef MLRG_GATHER_MINB
#define MLRG_GATHER_MINB 4
#endif

// Complex elements per CTA of the shared-memory FFT passes (double: 16 B each).
// 4096 (64 KB, 8 batch rows of a 512-point line per CTA) measured best at 256^3
// (36.2 vs 35.7 it/s at 2048); MLRG_FFT_ELEMS overrides it for tuning.
std::int64_t fft_elems() {
  static const std::int64_t e = [] {
    const char* v = std::getenv("MLRG_FFT_ELEMS");
    // <= 4096: the 2D passes run up to 512-thread CTAs (m * nb / 8 threads)
    std::int64_t n = v ? std::clamp<std::int64_t>(std::atoll(v), 64, 4096) : std::int64_t{4096};
    while (n & (n - 1)) n &= n - 1;
    return n;
  }();
  return e;
}
// fu2d row batches alternate between two streams (MLRG_FU2D_PIPE=0 disables).
bool pipelined() {
  static const bool on = [] {
    const char* e = std::getenv("MLRG_FU2D_PIPE");
    return !(e && *e == '0');
  }();
  return on;
}
// k-columns per CTA of a 2D-grid FFT pass over length m.
int pass_cols(std::int64_t m) {
  int c = static_cast<int>(std::clamp<std::int64_t>(fft_elems() / m, 1, KB));
  while (c & (c - 1)) c &= c - 1;  // a power of two dividing KB
  return c;
}

// Four-step column passes (k_cols4_*) for an M-point column FFT: by default
// from M = 1024, where the 16-row grid batch (M^2 x 128 B) outgrows L2;
// MLRG_COLS4=0 disables them, MLRG_COLS4=1 uses them from M = 64 (tests).
bool use_cols4(std::int64_t m) {
  static const int mode = [] {
    const char* e = std::getenv("MLRG_COLS4");
    return e ? std::atoi(e) : -1;
  }();
  if (mode == 0) return false;
  return m >= (mode == 1 ? 64 : 1024) && m <= 4096 && (m & (m - 1)) == 0;
}

// ------------------------------------------------------------------------------------------
// fu1d / fu1d_adj
// ------------------------------------------------------------------------------------------
template <class TIn, int W, bool PEER, bool ZP>
__global__ void __launch_bounds__(1024, 1) k_fu1d(const TIn* __restrict__ u, float2* __restrict__ out, int n0, int n2,
                                              int h, int logm, int center, int ncol,
                                              const double* __restrict__ deconv, const int* __restrict__ start,
                                              const double* __restrict__ wts, const double2* __restrict__ fac,
                                              const double2* __restrict__ tw, PeerOut po, Skip sk) {
  if (skipped(sk, blockIdx.y)) return;
  extern __shared__ double2 sd[];
  const int m = 1 << logm, mask = m - 1;
  const int j0 = blockIdx.x * ncol;
  const TIn* ui = u + static_cast<long long>(blockIdx.y) * n0 * n2;
  // grid slot r holds mode (r + center) mod m, deconvolved. Loads are
  // unconditional (clamped address) so a pass issues its 8 back to back.
  auto load = [&](int r, int c) {
    const int mode = (r + center) & mask, j = j0 + c;
    const bool ok = mode < n0 && j < n2;
    const double2 x = to_d(ui[ok ? static_cast<long long>(mode) * n2 + j : 0]);
    const double dc = deconv[ok ? mode : 0];
    return ok ? cscale(x, dc) : make_double2(0.0, 0.0);
  };
  fft_stockham<+1, true, false, ZP>(sd, logm, ncol, ncol, tw, load);
  float2* oi = out + static_cast<long long>(blockIdx.y) * h * n2;
  for (int idx = threadIdx.x; idx < h * ncol; idx += blockDim.x) {
    const int k = idx / ncol, c = idx - k * ncol;
    const int j = j0 + c;
    if (j >= n2) continue;
    const int st = start[k];
    const double* wk = wts + k * W;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int a = 0; a < W; ++a) {
      const double2 g = sd[((st + a) & mask) * ncol + c];
      const double wa = __ldg(wk + a);
      acc.x = fma(g.x, wa, acc.x);
      acc.y = fma(g.y, wa, acc.y);
    }
    float2* dst = oi + static_cast<long long>(k) * n2;
    if constexpr (PEER) {  // fused all-to-all: detector row k goes to the rank that owns it
      int r = 0;
      while (r + 1 < po.world && k >= po.hi[r]) ++r;
      dst = po.dst[r] + ((po.off + blockIdx.y) * (po.hi[r] - po.lo[r]) + (k - po.lo[r])) * n2;
    }
    dst[j] = to_f(cmul(acc, fac[k]));
  }
}

template <class TOut>
__global__ void __launch_bounds__(512, 2) k_fu1d_adj(const float2* __restrict__ v, TOut* __restrict__ out, int n0,
                                                  int n2, int h, int logm, int center, int ncol,
                                                  const double2* __restrict__ cphase,
                                                  const int* __restrict__ cell_ptr, const int* __restrict__ cell_k,
                                                  const double* __restrict__ cell_w,
                                                  const double* __restrict__ pdeconv,
                                                  const double2* __restrict__ tw, Skip sk) {
  if (skipped(sk, blockIdx.y)) return;
  extern __shared__ double2 sd[];
  const int m = 1 << logm, mask = m - 1;
  double2* vt = sd + m * ncol;
  const int j0 = blockIdx.x * ncol;
  const float2* vi = v + static_cast<long long>(blockIdx.y) * h * n2;
  for (int idx = threadIdx.x; idx < h * ncol; idx += blockDim.x) {
    const int k = idx / ncol, c = idx - k * ncol;
    const int j = j0 + c;
    vt[idx] = j < n2 ? cmul(to_d(vi[static_cast<long long>(k) * n2 + j]), cphase[k]) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < m * ncol; idx += blockDim.x) {
    const int l = idx / ncol, c = idx - l * ncol;
    double2 acc = make_double2(0.0, 0.0);
    const int e0 = cell_ptr[l], e1 = cell_ptr[l + 1];
    // the first kSpread1 entries unrolled (their list loads issue together), the rest in order
    constexpr int kSpread1 = 8;
#pragma unroll
    for (int i = 0; i < kSpread1; ++i) {
      const int e = e0 + i;
      if (e < e1) {
        const double2 x = vt[cell_k[e] * ncol + c];
        const double wv = __ldg(cell_w + e);
        acc.x = fma(x.x, wv, acc.x);
        acc.y = fma(x.y, wv, acc.y);
      }
    }
    for (int e = e0 + kSpread1; e < e1; ++e) {
      const double2 x = vt[cell_k[e] * ncol + c];
      const double wv = __ldg(cell_w + e);
      acc.x = fma(x.x, wv, acc.x);
      acc.y = fma(x.y, wv, acc.y);
    }
    sd[idx] = acc;
  }
  __syncthreads();
  TOut* oi = out + static_cast<long long>(blockIdx.y) * n0 * n2;
  auto store = [&](int slot, int c, double2 x) {
    const int mode = (slot + center) & mask, j = j0 + c;
    if (mode >= n0 || j >= n2) return;
    const double2 r = cscale(x, pdeconv[mode]);
    TOut& o = oi[static_cast<long long>(mode) * n2 + j];
    o.x = static_cast<decltype(o.x)>(r.x);
    o.y = static_cast<decltype(o.y)>(r.y);
  };
  fft_stockham<-1, false, true>(sd, logm, ncol, ncol, tw, NoLoad(), store);
}

// ------------------------------------------------------------------------------------------
// fu2d forward: row pass, column pass, gather
// ------------------------------------------------------------------------------------------
// S[i][c'][KB]: row FFT of v[i, k0+kk, :] * dx[i] * dy[:] placed at wrapped slots.
// TS (with the four-step column passes): S[i][KB][c'] instead, so the stores of
// a CTA holding 1-2 batch rows of a long row are contiguous.
template <bool ZP, bool TS>
__global__ void __launch_bounds__(512, MLRG_FFT_MINB / 2) k_fu2d_rows(const float2* __restrict__ v, long long ld, long long k0, int nk,
                                                   int n2, int logm2, int center2, int ks_n,
                                                   const double* __restrict__ dx, const double* __restrict__ dy,
                                                   const double2* __restrict__ tw2, float2* __restrict__ S, Skip sk) {
  if (skipped(sk, 0)) return;
  extern __shared__ double2 sd[];
  const int m2 = 1 << logm2, mask2 = m2 - 1, sm = ks_n;
  const int i = blockIdx.y, ks = blockIdx.x * ks_n;  // ks groups of one line adjacent in launch order
  const double di = dx[i];
  auto load = [&](int r, int kk) {
    const int j = (r + center2) & mask2;
    const bool ok = j < n2 && ks + kk < nk;
    const double2 x = to_d(v[ok ? (static_cast<long long>(i) * ld + k0 + ks + kk) * n2 + j : 0]);
    const double f = di * dy[ok ? j : 0];
    return ok ? cscale(x, f) : make_double2(0.0, 0.0);
  };
  float2* Si = S + static_cast<long long>(i) * m2 * KB + (TS ? static_cast<long long>(ks) * m2 : ks);
  auto store = [&](int r, int kk, double2 x) {
    Si[TS ? static_cast<long long>(kk) * m2 + r : static_cast<long long>(r) * KB + kk] = to_f(x);
  };
  fft_stockham<+1, true, true, ZP>(sd, logm2, ks_n, sm, tw2, load, store);
}

// G[r'][c'][KB]: column FFT over the n1 non-zero wrapped rows of S.
// The grid rows are ldg >= M2 + ghost cells long: columns [0, ghost) are
// repeated at [M2, M2 + ghost) so the gather's windows never wrap.
template <bool ZP, class TG>
__global__ void __launch_bounds__(512, MLRG_FFT_MINB / 2) k_fu2d_cols(const float2* __restrict__ S, int n1, int logm1, int center1,
                                                   int logm2, int ks_n, const double2* __restrict__ tw1,
                                                   TG* __restrict__ G, int ldg, int ghost, Skip sk) {
  if (skipped(sk, 0)) return;
  extern __shared__ double2 sd[];
  const int m1 = 1 << logm1, mask1 = m1 - 1, m2 = 1 << logm2;
  const int c = blockIdx.y, ks = blockIdx.x * ks_n;  // ks groups of one line adjacent in launch order
  auto load = [&](int r, int kk) {
    const int i = (r + center1) & mask1;
    const bool ok = i < n1;
    const double2 x = to_d(S[(static_cast<long long>(ok ? i : 0) * m2 + c) * KB + ks + kk]);
    return ok ? x : make_double2(0.0, 0.0);
  };
  const bool dup = c < ghost;
  auto store = [&](int r, int kk, double2 x) {
    TG* g = G + (static_cast<long long>(r) * ldg + c) * KB + ks + kk;
    g[0] = to_g<TG>(x);
    if (dup) g[static_cast<long long>(m2) * KB] = to_g<TG>(x);
  };
  fft_stockham<+1, true, true, ZP>(sd, logm1, ks_n, ks_n, tw1, load, store);
}

struct GatherOut {
  float2* out;
  long long ld_out, k0_out;
  const float2* sub;
  long long ld_sub, k0_sub;
  const float2* dot;
  long long ld_dot, k0_dot;
  int reduce;
  double2* cls;          // non-null: the adjoint's class sums of the stored output ([C][KB], complex64 values widened)
  const double2* cfac;   // the members' conjugate phases (k_fu2d_adj_prep's factors)
};

// ---- gather: one warp per target class ---------------------------------------------------
// A class is a set of detector samples with the same frequency (the tilted
// geometry samples every frequency twice: (theta, q) and (theta + pi, w - q)
// coincide, and q = w/2 is the origin for every angle): its 2D sum is
// computed once and multiplied by each member's phase (Usfft::Tables).
// Lane l owns batch row l % 16 and the window columns of parity l / 16, so a
// half warp reads one 128 B grid cell (16 rows x complex64) per tap: every
// load is a full coalesced line, no tap is wasted and no lane idles. Per
// window row the warp reads W/2 cells per half warp, widens them, sums them
// against the column weights (double) and adds the row weight times that
// sum, which is the reference's order of summation (inner over columns,
// outer over rows, nufft.cpp:205-216). Targets are processed in a spatially
// sorted order, a contiguous range per CTA, so the warps of a CTA share their
// windows' cells in L1.
//   * The CTA's class records (window origin, weights, members and phases:
//     ClassRec, one contiguous block) arrive in shared memory through one
//     bulk-copy (TMA engine, cp.async.bulk) on an mbarrier, so no class waits
//     on a global load of its own parameters.
//   * The forward grid carries `ghost` replicated columns past M2 (written by
//     the column pass), so no window wraps horizontally: one row address per
//     window row, the W/2 cells at immediate offsets.
//   * Rows stream through a 2-deep register ring that runs across class
//     boundaries: the next class's first row is in flight while the current
//     class's last row is summed.
constexpr int kGatherWarps = 8;
constexpr std::size_t kClassMax = 4;

template <int W>
struct ClassRec {
  int r0, c0, nmem, first;  // window origin (row, column), member count, first member index
  int tq[kClassMax];        // members: packed (t << 16 | q)
  double2 fac[kClassMax];   // members' pref x phase
  double w1[W], w2[W];      // row and column kernel weights
};
static_assert(sizeof(ClassRec<10>) % 16 == 0 && sizeof(ClassRec<24>) % 16 == 0, "bulk-copy granularity");

// MLRG_WIDE_GRID=1: complex128 grids for the ES kernel too (experiment)
bool wide_grids_env() {
  static const bool v = [] {
    const char* e = std::getenv("MLRG_WIDE_GRID");
    return e && std::atoi(e) != 0;
  }();
  return v;
}

// gather prefetch depth: rows in flight ahead of the row being summed
#ifndef MLRG_GATHER_D
#define MLRG_GATHER_D 1
#endif
constexpr int gather_depth(int W) { return W == 10 ? MLRG_GATHER_D : 1; }

// classes per gather CTA (MLRG_GATHER_PER_CTA overrides, for tuning)
int gather_per_cta() {
  static const int v = [] {
    const char* e = std::getenv("MLRG_GATHER_PER_CTA");
    return e ? std::max(8, std::atoi(e)) : 16;
  }();
  return v;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

// One thread: arm `bar` for `bytes` and bulk-copy [src, src + bytes) into smem
// (cp.async.bulk, completes on the mbarrier's transaction count).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// The class's window sum, shared by its members: each member's sample is the
// sum times its own phase (minus its d_hat value when fused), stored as
// complex64; optional class sums for the adjoint and the residual's
// reductions (operators.cpp:285-299).
template <int W>
__device__ __forceinline__ void gather_epilogue(double2 acc, const ClassRec<W>& R, int s, const GatherOut& eo, int w,
                                                int nk, int kk, int ph, double (&red)[2]) {
  acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
  acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
  if (ph == 0 && eo.cls && kk >= nk) eo.cls[static_cast<long long>(s) * KB + kk] = make_double2(0.0, 0.0);
  if (ph == 0 && kk < nk) {
    // every detector sample of the class gets the shared sum times its own phase
    double2 cs = make_double2(0.0, 0.0);
    for (int e = 0; e < R.nmem; ++e) {
      const int tq = R.tq[e];
      const int t = tq >> 16, q = tq & 0xffff;
      double2 val = cmul(acc, R.fac[e]);
      if (eo.sub) val = csub(val, to_d(eo.sub[(t * eo.ld_sub + eo.k0_sub + kk) * w + q]));
      const float2 stored = to_f(val);
      if (eo.out) eo.out[(t * eo.ld_out + eo.k0_out + kk) * w + q] = stored;
      if (eo.cls) cs = cadd(cs, cmul(to_d(stored), eo.cfac[R.first + e]));  // k_fu2d_adj_prep's sum, member order
      if (eo.reduce) {
        red[0] += val.x * val.x + val.y * val.y;
        if (eo.dot) {
          const float2 d = eo.dot[(t * eo.ld_dot + eo.k0_dot + kk) * w + q];
          red[1] += static_cast<double>(d.x) * val.x + static_cast<double>(d.y) * val.y;
        }
      }
    }
    if (eo.cls) eo.cls[static_cast<long long>(s) * KB + kk] = to_d(to_f(cs));
  }
}

__device__ __forceinline__ void gather_finish(double (&red)[2], double* red_scratch, const GatherOut& eo,
                                              double* __restrict__ partials, int accumulate) {
  if (eo.reduce) {
    block_sum<2>(red, red_scratch);
    if (threadIdx.x == 0) {
      double* p = partials + 2 * blockIdx.x;
      if (accumulate) {
        p[0] += red[0];
        p[1] += red[1];
      } else {
        p[0] = red[0];
        p[1] = red[1];
      }
    }
  }
}

// (the 24-tap Gaussian windows: 2 CTAs/SM, 128 registers)
template <int W, class TG>
__global__ void __launch_bounds__(32 * kGatherWarps, W == kEsTaps ? (sizeof(TG) == 8 ? MLRG_GATHER_MINB : 3) : MLRG_GATHER_MINB_G) k_fu2d_gather(
    const TG* __restrict__ G, int T, int w, int logm1, int ldg, int nk, const ClassRec<W>* __restrict__ recs,
    GatherOut eo, int per_cta, double* __restrict__ partials, int accumulate, Skip sk) {
  if (skipped(sk, 0)) return;
  constexpr int WH = W / 2;
  // rows in flight ahead of the one summed; the ring runs across classes, so
  // its period D + 1 must divide W
  constexpr int D = gather_depth(W);
  static_assert(W % (D + 1) == 0, "the cross-class row ring period must divide W");
  extern __shared__ __align__(16) unsigned char gather_smem[];
  __shared__ unsigned long long bar;
  __shared__ double red_scratch[kGatherWarps * 2];
  const ClassRec<W>* rec = reinterpret_cast<const ClassRec<W>*>(gather_smem);
  const int s0 = blockIdx.x * per_cta, s_end = min(T, s0 + per_cta);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    bulk_load(gather_smem, recs + s0, static_cast<unsigned>((s_end - s0) * sizeof(ClassRec<W>)), &bar);
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, kk = lane & 15, ph = lane >> 4;
  const int mask1 = (1 << logm1) - 1;
  const unsigned rs = static_cast<unsigned>(ldg) * KB * static_cast<unsigned>(sizeof(TG));  // bytes per grid row
  constexpr int CB = 2 * KB * static_cast<int>(sizeof(TG));  // bytes between a lane's window columns
  double red[2] = {0.0, 0.0};
  mbar_wait(&bar, 0);
  const char* gbase = reinterpret_cast<const char*>(G + ph * KB + kk);
  auto col_base = [&](int s) { return gbase + static_cast<long long>(rec[s - s0].c0) * KB * sizeof(TG); };
  auto row = [&](const char* cb, int r) { return cb + static_cast<unsigned>(r & mask1) * rs; };
  TG buf[D + 1][WH];
  int s = s0 + warp;
  if (s < s_end) {  // prime the ring with the first class's first D rows
    const char* cb0 = col_base(s);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const char* gr = row(cb0, rec[s - s0].r0 + a);
#pragma unroll
      for (int j = 0; j < WH; ++j) buf[a][j] = __ldg(reinterpret_cast<const TG*>(gr + j * CB));
    }
  }
  for (; s < s_end; s += kGatherWarps) {
    const ClassRec<W>& R = rec[s - s0];
    const int sn = s + kGatherWarps < s_end ? s + kGatherWarps : s;  // the next class (or a harmless reload)
    const char* cb = col_base(s);
    const char* cbn = col_base(sn);
    const int r0 = R.r0, r0n = rec[sn - s0].r0;
    double w2l[WH];  // this lane's column weights (window columns 2 j + ph)
#pragma unroll
    for (int j = 0; j < WH; ++j) w2l[j] = R.w2[2 * j + ph];
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int a = 0; a < W; ++a) {
      {  // row a + D of this class, or row a + D - W of the next
        const char* gr = a + D < W ? row(cb, r0 + a + D) : row(cbn, r0n + a + D - W);
#pragma unroll
        for (int j = 0; j < WH; ++j) buf[(a + D) % (D + 1)][j] = __ldg(reinterpret_cast<const TG*>(gr + j * CB));
      }
      double2 racc = make_double2(0.0, 0.0);
      auto tap = [&](auto jc) {
        constexpr int j = decltype(jc)::value;
        const TG v = buf[a % (D + 1)][j];
        racc.x = fma(w2l[j], static_cast<double>(v.x), racc.x);
        racc.y = fma(w2l[j], static_cast<double>(v.y), racc.y);
      };
      [&]<int... J>(std::integer_sequence<int, J...>) { (tap(std::integral_constant<int, J>{}), ...); }(
          std::make_integer_sequence<int, WH>{});
      const double wa = R.w1[a];
      acc.x = fma(wa, racc.x, acc.x);
      acc.y = fma(wa, racc.y, acc.y);
    }
    gather_epilogue(acc, R, s, eo, w, nk, kk, ph, red);
  }
  gather_finish(red, red_scratch, eo, partials, accumulate);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- warp-cooperative spread (adjoint) -----------------------------------------------------
// One warp pair owns an 8x4 patch of grid cells and the 16 batch rows (warp
// half h: rows 8h..8h+7) and walks the host-built list of targets whose window
// touches the patch, kSpreadChunk targets per chunk, one chunk ahead. Per
// target the pair stages the 32 cell weights w1[row] * w2[col] of this patch
// (zero outside the window; the double product of nufft.cpp:250-256) and each
// warp cp.asyncs its half of the 16 values (complex64 values the producers
// store widened to double, so no conversion pass sits in the chunk loop).
// A lane owns 4 cells x 2 batch rows (register blocking): per target it reads
// two 16-byte weight pairs and two double2 values (4 shared wavefronts per
// warp) for 16 DFMA, where a lane-per-cell layout needs 10 wavefronts (8 value
// broadcasts + 2 weights) and a DMUL for the same 16 DFMA. Every (cell, row)
// sum runs in target order in double exactly as before (cells near nu = 0
// receive thousands of terms). Patches are processed heaviest first.
constexpr int kPatchR = 8, kPatchC = 4;
constexpr int KH = KB / 2;
constexpr int kSpreadChunk = 16;

constexpr int kWgtStride = 34;  // doubles per target row: 16-byte aligned, conflict-free STS.128 / LDS.128

struct SpreadShared {
  double wgt[2][2][kSpreadChunk][kWgtStride];    // [pair][buf][target][cell]
  double2 vals[4][2][kSpreadChunk][KH];          // per warp, double-buffered half values
  int last[2];                                   // per pair: this item completes its split patch
};

__device__ __forceinline__ void pair_sync(int pair) {
  asm volatile("bar.sync %0, 64;\n" ::"r"(pair + 1));
}

// A work item is (patch, a sub-range of its target list): lists longer than
// kSplit (the cells around nu = 0) are split over several warp pairs. Each
// writes its double partials to its slot; the pair that completes the patch
// (an atomic count per split group) sums all of the group's slots in slot
// order (deterministic, whoever finishes last) and writes the grid.
struct SpreadItem {
  int patch, e0, e1, slot;  // slot < 0: write the grid directly
  int grp;                  // split group (index into the (patch, first slot, slots) table)
};
constexpr int kSplit = 256;

// Chunk staging, software-pipelined so that no global load latency sits in
// front of the arithmetic: a chunk's list entries are loaded two chunks ahead,
// its weights one chunk ahead (in registers, turned into products after the
// current chunk's arithmetic), its values by cp.async one chunk ahead. Pair
// lane pl = part * 16 + j owns target j of a chunk: the weights of patch rows
// 2*part, 2*part+1 (cells 8*part .. 8*part+7, four 16-byte stores); each warp
// cp.asyncs its half of the values (four 16-byte pieces per lane).
// A list entry is (target, a0 | b0 << 16): the target's window offsets of the
// patch origin, (pr0 - r0[t]) mod m1 and (pc0 - c0[t]) mod m2, host-computed.
// (Measured and not kept: 8 lanes per target loading one weight row each and
// exchanging column weights by shuffle -- fewer cache lines per load, but the
// shuffles cost as many L1 data-pipe wavefronts as they save.)
struct SpreadW {
  double r[2], c[kPatchC];
  bool ok;
};

__device__ __forceinline__ int2 spread_entry(const int2* __restrict__ lst, int e, int e1, int lane) {
  const int j = lane & (kSpreadChunk - 1);
  return e + j < e1 ? lst[e + j] : make_int2(-1, 0);
}

template <int W>
__device__ __forceinline__ SpreadW spread_weights(int2 en, int part, int mask1, int mask2,
                                                  const double* __restrict__ w1, const double* __restrict__ w2) {
  SpreadW w;
  w.ok = en.x >= 0;
  const int a0 = (en.y & 0xffff) + 2 * part, b0 = en.y >> 16;
  const double* wr = w1 + static_cast<long long>(en.x) * W;
  const double* wc = w2 + static_cast<long long>(en.x) * W;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int a = (a0 + i) & mask1;
    w.r[i] = w.ok && a < W ? wr[a] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < kPatchC; ++q) {
    const int b = (b0 + q) & mask2;
    w.c[q] = w.ok && b < W ? wc[b] : 0.0;
  }
  return w;
}

__device__ __forceinline__ void spread_values(SpreadShared& sh, int2 en, int half, int warp, int buf,
                                              const double2* __restrict__ val, int lane) {
  if (en.x >= 0) {
    const int j = lane & (kSpreadChunk - 1), q0 = (lane >> 4) * (KH / 2);
    const double2* v = val + static_cast<long long>(en.x) * KB + half * KH;
#pragma unroll
    for (int q = q0; q < q0 + KH / 2; ++q) cp_async16(&sh.vals[warp][buf][j][q], v + q);
  }
  cp_async_commit();
}

__device__ __forceinline__ void spread_store_weights(SpreadShared& sh, const SpreadW& w, int pair, int buf, int part,
                                                     int lane) {
  if (!w.ok) return;
  double2* dst = reinterpret_cast<double2*>(&sh.wgt[pair][buf][lane & (kSpreadChunk - 1)][8 * part]);
#pragma unroll
  for (int i = 0; i < 2; ++i) {  // the double product w1 * w2 (nufft.cpp:250-256)
    dst[2 * i] = make_double2(w.r[i] * w.c[0], w.r[i] * w.c[1]);
    dst[2 * i + 1] = make_double2(w.r[i] * w.c[2], w.r[i] * w.c[3]);
  }
}

template <int W, class TG>
__global__ void __launch_bounds__(128, 4) k_fu2d_adj_spread(const double2* __restrict__ val, int logm1, int logm2,
                                                         int nitems, const SpreadItem* __restrict__ items,
                                                         const int2* __restrict__ lst, const double* __restrict__ w1,
                                                         const double* __restrict__ w2, TG* __restrict__ G,
                                                         double2* __restrict__ partial, const int4* __restrict__ split,
                                                         int* __restrict__ split_cnt, Skip sk) {
  if (skipped(sk, 0)) return;
  extern __shared__ float4 dyn_smem[];
  SpreadShared& sh = *reinterpret_cast<SpreadShared*>(dyn_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, pair = warp >> 1, half = warp & 1;
  const int pi = blockIdx.x * 2 + pair;
  if (pi >= nitems) return;  // both warps of the pair leave together
  const int m2 = 1 << logm2, mask1 = (1 << logm1) - 1, mask2 = m2 - 1;
  const SpreadItem it = items[pi];
  const int npc = m2 / kPatchC;
  const int pr0 = (it.patch / npc) * kPatchR, pc0 = (it.patch % npc) * kPatchC;
  // this lane: cells 2g, 2g+1, 16+2g, 17+2g (cell = row * 4 + col) and batch rows kb, kb+1
  const int g = lane & 7, kb = half * KH + 2 * (lane >> 3);
  double2 acc[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = make_double2(0.0, 0.0);
  const int part = half * 2 + (lane >> 4);  // staging role
  const int e0 = it.e0, e1 = it.e1;
  {
    const int2 en0 = spread_entry(lst, e0, e1, lane);
    spread_values(sh, en0, half, warp, 0, val, lane);
    spread_store_weights(sh, spread_weights<W>(en0, part, mask1, mask2, w1, w2), pair, 0, part, lane);
  }
  int2 en = spread_entry(lst, e0 + kSpreadChunk, e1, lane);  // the next chunk's entries
  for (int e = e0, chunk = 0; e < e1; e += kSpreadChunk, ++chunk) {
    const int buf = chunk & 1;
    pair_sync(pair);  // weights of this chunk visible; the other buffer is free
    const SpreadW wn = spread_weights<W>(en, part, mask1, mask2, w1, w2);  // lands during the arithmetic
    spread_values(sh, en, half, warp, buf ^ 1, val, lane);
    en = spread_entry(lst, e + 2 * kSpreadChunk, e1, lane);
    cp_async_wait<1>();  // this chunk's values (the next chunk's group may be pending)
    __syncwarp();
    const int n = min(kSpreadChunk, e1 - e);
    const double* wrow = &sh.wgt[pair][buf][0][0];
#pragma unroll 2
    for (int j = 0; j < n; ++j) {
      const double2 wa = *reinterpret_cast<const double2*>(wrow + j * kWgtStride + 2 * g);
      const double2 wb = *reinterpret_cast<const double2*>(wrow + j * kWgtStride + 16 + 2 * g);
      const double2 x0 = sh.vals[warp][buf][j][kb - half * KH], x1 = sh.vals[warp][buf][j][kb - half * KH + 1];
      const double w[4] = {wa.x, wa.y, wb.x, wb.y};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[c][0].x = fma(w[c], x0.x, acc[c][0].x);
        acc[c][0].y = fma(w[c], x0.y, acc[c][0].y);
        acc[c][1].x = fma(w[c], x1.x, acc[c][1].x);
        acc[c][1].y = fma(w[c], x1.y, acc[c][1].y);
      }
    }
    spread_store_weights(sh, wn, pair, buf ^ 1, part, lane);
  }
  const int cells[4] = {2 * g, 2 * g + 1, 16 + 2 * g, 17 + 2 * g};
  if (it.slot >= 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double2* pp = partial + (static_cast<long long>(it.slot) * 32 + cells[c]) * KB + kb;
      pp[0] = acc[c][0];
      pp[1] = acc[c][1];
    }
    __threadfence();  // this pair's partials are visible before its arrival is counted
    pair_sync(pair);
    const int4 sp = split[it.grp];  // (patch, first slot, slots, -)
    if (half == 0 && lane == 0) sh.last[pair] = atomicAdd(split_cnt + it.grp, 1) == sp.z - 1;
    pair_sync(pair);
    if (!sh.last[pair]) return;
    __threadfence();
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = make_double2(0.0, 0.0);
    for (int q = 0; q < sp.z; ++q) {  // slot order
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double2* src = partial + (static_cast<long long>(sp.y + q) * 32 + cells[c]) * KB + kb;
        acc[c][0] = cadd(acc[c][0], __ldcg(src));
        acc[c][1] = cadd(acc[c][1], __ldcg(src + 1));
      }
    }
    if (half == 0 && lane == 0) split_cnt[it.grp] = 0;  // ready for the next launch
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int r = pr0 + cells[c] / kPatchC, col = pc0 + cells[c] % kPatchC;
    const long long o = (static_cast<long long>(r) * m2 + col) * KB + kb;
    if constexpr (std::is_same_v<TG, double2>) {
      G[o] = acc[c][0];
      G[o + 1] = acc[c][1];
    } else {
      const float2 lo = to_f(acc[c][0]), hi = to_f(acc[c][1]);
      *reinterpret_cast<float4*>(G + o) = make_float4(lo.x, lo.y, hi.x, hi.y);
    }
  }
}

// ------------------------------------------------------------------------------------------
// fu2d adjoint: prep, column pass, row pass (the spread is above)
// ------------------------------------------------------------------------------------------
// val[c][kk] = sum over the members e of class c of p[t_e, k0+kk, q_e] *
// conj(phase_e), in member order (deterministic); zero for kk >= nk.
__global__ void __launch_bounds__(256) k_fu2d_adj_prep(const float2* __restrict__ p, long long ld, long long k0,
                                                       int nk, int C, int w, const int* __restrict__ m_first,
                                                       const int* __restrict__ m_tidx,
                                                       const double2* __restrict__ m_cfac, double2* __restrict__ val, Skip sk) {
  if (skipped(sk, 0)) return;
  const int kk = threadIdx.x & (KB - 1);
  const int c = blockIdx.x * (blockDim.x / KB) + threadIdx.x / KB;
  if (c >= C) return;
  double2 acc = make_double2(0.0, 0.0);
  if (kk < nk)
    for (int e = m_first[c], e1 = m_first[c + 1]; e < e1; ++e) {
      const int tq = m_tidx[e];
      const int t = tq >> 16, q = tq & 0xffff;  // packed (Usfft::Tables)
      acc = cadd(acc, cmul(to_d(p[(t * ld + k0 + kk) * w + q]), m_cfac[e]));
    }
  val[static_cast<long long>(c) * KB + kk] = to_d(to_f(acc));  // complex64 values, stored widened for the spread
}

// Column FFT(-1) over natural rows; keep only the n1 rows that map to modes.
template <class TG>
__global__ void __launch_bounds__(512, MLRG_FFT_MINB / 2) k_fu2d_adj_cols(const TG* __restrict__ G, int n1, int logm1, int center1,
                                                       int logm2, int ks_n, const double2* __restrict__ tw1,
                                                       float2* __restrict__ S, Skip sk) {
  if (skipped(sk, 0)) return;
  extern __shared__ double2 sd[];
  const int m1 = 1 << logm1, mask1 = m1 - 1, m2 = 1 << logm2;
  const int c = blockIdx.y, ks = blockIdx.x * ks_n;  // ks groups of one line adjacent in launch order
  auto load = [&](int r, int kk) { return to_d(G[(static_cast<long long>(r) * m2 + c) * KB + ks + kk]); };
  auto store = [&](int slot, int kk, double2 x) {  // keep the n1 slots that map to modes
    const int i = (slot + center1) & mask1;
    if (i < n1) S[(static_cast<long long>(i) * m2 + c) * KB + ks + kk] = to_f(x);
  };
  fft_stockham<-1, true, true>(sd, logm1, ks_n, ks_n, tw1, load, store);
}

// ---- four-step column passes (grids beyond L2) --------------------------------------------
// From M = 1024 the one-pass column kernels hold only 1-2 of a cell's 16 batch
// rows per CTA (an M-point double column is M x 16 B of shared memory), so
// every CTA touches 8-16 B of each 128 B cell; once the grid no longer fits L2
// those partial-line accesses dominate the iteration. With M = A * B the
// column FFT is X[ka + A kb] = sum_b W_B^{b kb} W_M^{b ka} sum_a x[a B + b] W_A^{a ka}:
// pass 1 takes the A-point FFTs over rows b, B + b, ... for one b and writes
// Y[b A + ka] times the twiddle, pass 2 the B-point FFTs over rows ka, A + ka, ...
// A CTA of either pass holds kCols4 grid columns x all 16 batch rows, a
// contiguous 512 B block of every grid row it touches, so all traffic is in
// whole lines at the cost of one more trip through the grid.
#ifndef MLRG_COLS4_W
#define MLRG_COLS4_W 4
#endif
constexpr int kCols4 = MLRG_COLS4_W;
constexpr int kCols4Lanes = kCols4 * KB;

// The block of a grid row a CTA owns: lane l is (column c0 + l / KB, batch row
// l % KB), at offset l in the [c][KB] layout; with the transposed S layout
// ([KB][c], TS) lane l is (c0 + l % kCols4, l / kCols4) instead, so both the
// S side and the grid side of the pass move whole 32 B sectors.
__device__ __forceinline__ int cols4_off(int l, bool ts) { return ts ? (l % kCols4) * KB + l / kCols4 : l; }
__device__ __forceinline__ long long cols4_ts(int row, int c0, int l, int m2) {
  return (static_cast<long long>(row) * KB + l / kCols4) * m2 + c0 + l % kCols4;
}

// FROM_S: the input rows are the S rows of the n1 wrapped slots (forward);
// otherwise all M natural rows (adjoint). TS: S in the transposed layout.
template <int SIGN, bool FROM_S, bool TS>
__global__ void __launch_bounds__(512, 2) k_cols4_pass1(const float2* __restrict__ in, int n1, int logm1, int center1,
                                                        int logA, int logm2, const double2* __restrict__ twA,
                                                        const double2* __restrict__ twM, float2* __restrict__ Y, Skip sk) {
  if (skipped(sk, 0)) return;
  extern __shared__ double2 sd[];
  const int mask1 = (1 << logm1) - 1, m2 = 1 << logm2, logB = logm1 - logA;
  const int b = blockIdx.x, c0 = blockIdx.y * kCols4;
  // this CTA's inter-pass twiddles W_M^(b ka), ka < A, staged behind the tile
  // before the first pass (its closing barrier publishes them), so the last
  // pass's products do not wait on global loads
  double2* twb = sd + (kCols4Lanes << logA);
  for (int ka = threadIdx.x; ka < (1 << logA); ka += blockDim.x) {
    double2 w = twM[b * ka];  // b * ka < M
    if (SIGN < 0) w.y = -w.y;
    twb[ka] = w;
  }
  auto load = [&](int a, int l) {
    const int r = (a << logB) + b;  // one row per warp: the branch is uniform
    int i = r;
    if constexpr (FROM_S) {
      i = (r + center1) & mask1;
      if (i >= n1) return make_double2(0.0, 0.0);
      if constexpr (TS) return to_d(in[cols4_ts(i, c0, l, m2)]);
    }
    return to_d(in[(static_cast<long long>(i) * m2 + c0) * KB + l]);
  };
  auto store = [&](int ka, int l, double2 x) {
    const double2 w = twb[ka];
    Y[(static_cast<long long>((b << logA) + ka) * m2 + c0) * KB + cols4_off(l, FROM_S && TS)] = to_f(cmul(x, w));
  };
  fft_stockham<SIGN, true, true>(sd, logA, kCols4Lanes, kCols4Lanes, twA, load, store);
}

// TO_S: keep the n1 output slots that map to modes, at their S rows (adjoint);
// otherwise all M rows in natural order (forward). TS: S in the transposed layout.
// (forward: `out` is the gather's grid, rows ldo cells long with `ghost`
// repeated columns, as k_fu2d_cols writes it)
template <int SIGN, bool TO_S, bool TS>
__global__ void __launch_bounds__(512, 2) k_cols4_pass2(const float2* __restrict__ Y, int n1, int logm1, int center1,
                                                        int logA, int logm2, const double2* __restrict__ twB,
                                                        float2* __restrict__ out, int ldo, int ghost, Skip sk) {
  if (skipped(sk, 0)) return;
  extern __shared__ double2 sd[];
  const int mask1 = (1 << logm1) - 1, m2 = 1 << logm2, logB = logm1 - logA;
  const int ka = blockIdx.x, c0 = blockIdx.y * kCols4;
  constexpr bool T = TO_S && TS;
  auto load = [&](int bb, int l) {
    return to_d(Y[(static_cast<long long>((bb << logA) + ka) * m2 + c0) * KB + cols4_off(l, T)]);
  };
  auto store = [&](int kb, int l, double2 x) {
    int r = ka + (kb << logA);
    if constexpr (TO_S) {
      r = (r + center1) & mask1;
      if (r >= n1) return;
    }
    if constexpr (T) {
      out[cols4_ts(r, c0, l, m2)] = to_f(x);
    } else {
      float2* o = out + (static_cast<long long>(r) * ldo + c0) * KB + l;
      o[0] = to_f(x);
      if (c0 + l / KB < ghost) o[static_cast<long long>(m2) * KB] = to_f(x);
    }
  };
  fft_stockham<SIGN, true, true>(sd, logB, kCols4Lanes, kCols4Lanes, twB, load, store);
}

// Row FFT(-1) and the final deconvolution into out[i, k0_out+kk, j].
template <bool PEER, bool TS>
__global__ void __launch_bounds__(512, MLRG_FFT_MINB / 2) k_fu2d_adj_rows(const float2* __restrict__ S, int nk, int n2, int logm2,
                                                       int center2, int ks_n, const double* __restrict__ pdx,
                                                       const double* __restrict__ dy, const double2* __restrict__ tw2,
                                                       float2* __restrict__ out, long long ld_out,
                                                       long long k0_out, PeerOut po, Skip sk) {
  if (skipped(sk, 0)) return;
  extern __shared__ double2 sd[];
  const int m2 = 1 << logm2, mask2 = m2 - 1, sm = ks_n + 1;
  const int i = blockIdx.y, ks = blockIdx.x * ks_n;  // ks groups of one line adjacent in launch order
  const float2* Si = S + static_cast<long long>(i) * m2 * KB + (TS ? static_cast<long long>(ks) * m2 : ks);
  const double pi = pdx[i];
  // plane i of the output: local, or (fused all-to-all) in the HBM of the rank owning plane i
  float2* oplane = out + static_cast<long long>(i) * ld_out * n2;
  if constexpr (PEER) {
    int r = 0;
    while (r + 1 < po.world && i >= po.hi[r]) ++r;
    oplane = po.dst[r] + (i - po.lo[r]) * po.h * n2;
    k0_out += po.off;
  }
  auto load = [&](int c, int kk) {
    return to_d(Si[TS ? static_cast<long long>(kk) * m2 + c : static_cast<long long>(c) * KB + kk]);
  };
  auto store = [&](int slot, int kk, double2 x) {
    const int j = (slot + center2) & mask2;
    if (j < n2 && ks + kk < nk) oplane[(k0_out + ks + kk) * n2 + j] = to_f(cscale(x, pi * dy[j]));
  };
  fft_stockham<-1, true, true>(sd, logm2, ks_n, sm, tw2, load, store);
}

// ------------------------------------------------------------------------------------------
// f2d: centred unitary 2D DFT. Power-of-two planes use two FFT passes with the
// (-1)^(k+m+N/2) checkerboard; other sizes fall back to dense DFT passes with
// the host-built centred matrix (both on the device).
// ------------------------------------------------------------------------------------------
// FFT along the contiguous axis of `rows` rows of length m (one CTA per ncol rows).
template <int SIGN>
__global__ void __launch_bounds__(512) k_center_fft_rows(const float2* __restrict__ in, float2* __restrict__ out,
                                                         long long rows, int logm, int ncol, double scale,
                                                         const double2* __restrict__ tw) {
  extern __shared__ double2 sd[];
  const int m = 1 << logm, sm = ncol + 1;
  const long long r0 = static_cast<long long>(blockIdx.x) * ncol;
  auto load = [&](int n, int c) {
    const bool ok = r0 + c < rows;
    const double2 x = to_d(in[ok ? (r0 + c) * m + n : 0]);
    return !ok ? make_double2(0.0, 0.0) : (n & 1) ? make_double2(-x.x, -x.y) : x;
  };
  auto store = [&](int k, int c, double2 x) {
    if (r0 + c >= rows) return;
    const double sg = ((k + (m >> 1)) & 1) ? -scale : scale;
    out[(r0 + c) * m + k] = to_f(cscale(x, sg));
  };
  fft_stockham<SIGN, true, true>(sd, logm, ncol, sm, tw, load, store);
}

// FFT along the middle axis of [outer][m][inner] (one CTA per outer x ncol inner).
template <int SIGN>
__global__ void __launch_bounds__(512) k_center_fft_cols(const float2* in, float2* out, int inner, int logm, int ncol,
                                                         double scale, const double2* __restrict__ tw) {
  extern __shared__ double2 sd[];
  const int m = 1 << logm;
  const long long o = blockIdx.y;
  const int c0 = blockIdx.x * ncol;
  const float2* io = in + o * m * inner;
  float2* oo = out + o * m * inner;
  auto load = [&](int n, int c) {
    const bool ok = c0 + c < inner;
    const double2 x = to_d(io[ok ? static_cast<long long>(n) * inner + c0 + c : 0]);
    return !ok ? make_double2(0.0, 0.0) : (n & 1) ? make_double2(-x.x, -x.y) : x;
  };
  auto store = [&](int k, int c, double2 x) {  // in place is safe: all loads precede the first store
    if (c0 + c >= inner) return;
    const double sg = ((k + (m >> 1)) & 1) ? -scale : scale;
    oo[static_cast<long long>(k) * inner + c0 + c] = to_f(cscale(x, sg));
  };
  fft_stockham<SIGN, true, true>(sd, logm, ncol, ncol, tw, load, store);
}

// out[o, k, in] = sum_m W[k, m] x[o, m, in] (dense centred DFT along the middle axis).
__global__ void k_dense_dft(const float2* __restrict__ in, float2* __restrict__ out, long long outer, int m,
                            int inner, const double2* __restrict__ W) {
  const long long total = outer * m * inner;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e % inner);
    const long long rest = e / inner;
    const int k = static_cast<int>(rest % m);
    const long long o = rest / m;
    const float2* io = in + o * m * inner + c;
    double2 acc = make_double2(0.0, 0.0);
    for (int n = 0; n < m; ++n) acc = cadd(acc, cmul(to_d(io[static_cast<long long>(n) * inner]), W[k * m + n]));
    out[e] = to_f(acc);
  }
}

// e^{2 pi i k/m} for k < m (the Stockham passes index the full circle).
std::vector<double2> twiddles(std::int64_t m) {
  std::vector<double2> t(static_cast<std::size_t>(std::max<std::int64_t>(m, 1)));
  for (std::int64_t k = 0; k < m; ++k) {
    const double a = 2.0 * std::numbers::pi * static_cast<double>(k) / static_cast<double>(m);
    t[static_cast<std::size_t>(k)] = make_double2(std::cos(a), std::sin(a));
  }
  return t;
}

bool is_pow2(std::int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
// A length-n signal placed at the centred slots of an m = 2n grid: the input of
// slots [m/4, 3m/4) is zero (the ZP first pass of fft_stockham skips it).
bool zero_padded(const DimPlan& p) { return p.m == 2 * p.n && 2 * p.center == p.n; }
int ilog2(std::int64_t n) {
  int l = 0;
  while ((std::int64_t{1} << l) < n) ++l;
  return l;
}


template <class K>
void allow_big_smem(K kernel) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

}  // namespace

int sm_count() {
  static int n = [] {
    int dev = 0, c = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return 148;
    return c;
  }();
  return n;
}

struct Usfft::Tables {
  // fu1d
  DimPlan pz;
  int z_ncol = 0, z_ncol_adj = 0;
  DeviceBuffer<double> z_deconv, z_pdeconv;
  DeviceBuffer<double> z_w, z_cell_w;
  DeviceBuffer<int> z_start, z_cell_ptr, z_cell_k;
  DeviceBuffer<double2> z_fac, z_cphase, z_tw;
  // fu2d
  DimPlan px, py;
  DeviceBuffer<double> x_deconv, x_pdeconv, y_deconv;
  // target classes (coincident frequencies), spatially sorted: window origin
  // and weights per class, member lists with each member's phase factors
  int nclass = 0;
  int gather_per = 16;  // classes per gather CTA (whole waves of resident CTAs)
  int ghost = 0, ldg = 0;  // forward grid: repeated columns and row length (cells)
  DeviceBuffer<unsigned char> recs;  // ClassRec<W>[C]
  DeviceBuffer<int> m_first, m_tidx;
  DeviceBuffer<double> t_w1, t_w2;  // [C][W]
  DeviceBuffer<double2> m_fac, m_cfac, x_tw, y_tw;
  DeviceBuffer<float2> S, Gd;  // scratch: row pass, grid
  DeviceBuffer<double2> val;   // adjoint class values (complex64 values, widened)
  DeviceBuffer<double2> cls;        // class sums left by a class_sums fu2d, [batch][C][KB]
  // fu2d runs its row batches on two streams (the second set of grids and
  // partial slots belongs to the side stream) so one batch's gather overlaps the
  // next batch's FFT passes
  // stream j > 0 of the K-stream pipeline owns sides[j - 1] and these buffers
  struct Lane {
    cudaStream_t s = nullptr;
    cudaEvent_t ev_join = nullptr;
    DeviceBuffer<float2> S, Gd;
    DeviceBuffer<double2> val;
    DeviceBuffer<double2> partial;
    DeviceBuffer<int> split_cnt;
  };
  std::vector<std::unique_ptr<Lane>> sides;
  // four-step column passes: M = A * B, A = 2^logA
  bool cols4 = false;
  bool wide = false;  // Gd holds complex128 (the Gaussian plan's grids, see to_g)
  int logA = 0;
  DeviceBuffer<double2> a_tw, b_tw;
  cudaEvent_t ev_fork = nullptr;
  // warp-cooperative spread: 8x4 cell patches -> targets, heaviest patch first
  int nitems = 0, nsplit = 0;
  DeviceBuffer<int2> patch_t;  // (class, a0 | b0 << 16) per patch list entry
  DeviceBuffer<SpreadItem> items;
  DeviceBuffer<int4> split;
  DeviceBuffer<double2> partial;
  DeviceBuffer<int> split_cnt;  // arrivals per split group (zero between launches)
  // f2d
  bool f2d_fft = false;
  DeviceBuffer<double2> h_tw, w_tw, Wh, Ww, Whc, Wwc;
  DeviceBuffer<float2> f2d_tmp;
};

namespace {
// Table uploads of the constructor through pinned staging blocks (the caching
// allocator's): the host never waits on a pageable copy queued behind the
// drop-in's concurrent input upload; one synchronisation when the tables are done.
class Stager {
 public:
  explicit Stager(cudaStream_t s) : s_(s) {}
  ~Stager() {
    cudaStreamSynchronize(s_);
    for (auto& b : blocks_) alloc::pinned_free(b.first, b.second);
  }
  Stager(const Stager&) = delete;
  Stager& operator=(const Stager&) = delete;
  template <class T>
  void up(DeviceBuffer<T>& d, const T* src, std::size_t n) {
    d.resize(n);
    if (!n) return;
    const std::size_t bytes = n * sizeof(T);
    void* h = alloc::pinned(bytes);
    blocks_.emplace_back(h, bytes);
    std::memcpy(h, src, bytes);
    MLRG_CUDA(cudaMemcpyAsync(d.get(), h, bytes, cudaMemcpyHostToDevice, s_));
  }
  template <class T>
  void up(DeviceBuffer<T>& d, const std::vector<T>& v) {
    up(d, v.data(), v.size());
  }

 private:
  cudaStream_t s_;
  std::vector<std::pair<void*, std::size_t>> blocks_;
};
}  // namespace

Usfft::Usfft(const Geometry& g, cudaStream_t stream, GridKernel kernel)
    : g_(g), stream_(stream), kernel_(kernel), t_(new Tables) {
  Stager stg(stream_);
  prof::HostSpan span("host:usfft_tables");
  Tables& t = *t_;
  const FrequencyGrids fg = frequency_grids(g_);
  if (g_.w > 0xffff || g_.n_theta > 0x7fff)  // packed (t, q) member indices of the fu2d classes
    throw std::invalid_argument("fu2d: w must be < 65536 and n_theta < 32768");
  // ---- fu1d plan (nufft.cpp:109-110) ----
  // the two fu2d plans (the largest host tables) build on worker threads while the
  // fu1d plan and its tables are made here
  auto fx = std::async(std::launch::async, [&] { return DimPlan::make(g_.n1, fg.nu_x, kernel_); });
  auto fy = std::async(std::launch::async, [&] { return DimPlan::make(g_.n2, fg.nu_y, kernel_); });
  t.pz = DimPlan::make(g_.n0, fg.nu_z, kernel_);
  const int W = t.pz.taps;
  const DimPlan& pz = t.pz;
  t.z_ncol = static_cast<int>(std::clamp<std::int64_t>(fft_elems() / pz.m, 1, 64));
  t.z_ncol_adj = t.z_ncol;
  // fu1d: 8 columns per CTA (512 threads at m = 512, 1024 at m = 1024) make every global row
  // segment a full 128 B line and every shared-memory phase one grid row
  // (conflict-free taps); fu1d_adj keeps the smaller tile (its spread stage
  // holds h extra rows per column).
  t.z_ncol = static_cast<int>(std::clamp<std::int64_t>(pz.m >= 1024 ? 8192 / pz.m : 4096 / pz.m, 1, 64));
  if (const char* e = std::getenv("MLRG_FU1D_NCOL"))  // tuning override (threads = ncol * m / 8 <= 1024)
    t.z_ncol = static_cast<int>(std::clamp<std::int64_t>(std::atoll(e), 1, std::max<std::int64_t>(1, 8192 / pz.m)));
  t.z_ncol = static_cast<int>(std::min<std::int64_t>(t.z_ncol, g_.n2));
  if (const char* e = std::getenv("MLRG_FU1D_ADJ_NCOL"))  // tuning override (threads = ncol * m / 8 <= 512)
    t.z_ncol_adj = static_cast<int>(std::clamp<std::int64_t>(std::atoll(e), 1, std::max<std::int64_t>(1, 4096 / pz.m)));
  t.z_ncol_adj = static_cast<int>(std::min<std::int64_t>(t.z_ncol_adj, g_.n2));
  stg.up(t.z_deconv, pz.deconv);
  std::vector<double> pdec(pz.deconv.size());
  for (std::size_t i = 0; i < pdec.size(); ++i) pdec[i] = pz.pref * pz.deconv[i];
  stg.up(t.z_pdeconv, pdec);
  stg.up(t.z_start, std::vector<int>(pz.start.begin(), pz.start.end()));
  stg.up(t.z_w, pz.weights);
  std::vector<double2> fac(static_cast<std::size_t>(g_.h)), cph(static_cast<std::size_t>(g_.h));
  for (std::size_t k = 0; k < fac.size(); ++k) {
    fac[k] = make_double2(pz.pref * pz.phase_re[k], pz.pref * pz.phase_im[k]);
    cph[k] = make_double2(pz.phase_re[k], -pz.phase_im[k]);
  }
  stg.up(t.z_fac, fac);
  stg.up(t.z_cphase, cph);
  {  // cell -> (target, weight) CSR for the scatter-free adjoint, targets ascending
    std::vector<int> cnt(static_cast<std::size_t>(pz.m + 1), 0);
    for (std::int64_t k = 0; k < g_.h; ++k)
      for (int a = 0; a < W; ++a) cnt[static_cast<std::size_t>((pz.start[k] + a) % pz.m) + 1]++;
    for (std::size_t l = 1; l < cnt.size(); ++l) cnt[l] += cnt[l - 1];
    std::vector<int> ck(static_cast<std::size_t>(cnt.back())), pos(cnt.begin(), cnt.end() - 1);
    std::vector<double> cw(ck.size());
    for (std::int64_t k = 0; k < g_.h; ++k)
      for (int a = 0; a < W; ++a) {
        const std::size_t l = static_cast<std::size_t>((pz.start[k] + a) % pz.m);
        ck[static_cast<std::size_t>(pos[l])] = static_cast<int>(k);
        cw[static_cast<std::size_t>(pos[l]++)] = pz.weights[static_cast<std::size_t>(k * W + a)];
      }
    stg.up(t.z_cell_ptr, cnt);
    stg.up(t.z_cell_k, ck);
    stg.up(t.z_cell_w, cw);
  }
  stg.up(t.z_tw, twiddles(pz.m));

  prof::host_mark("host:usfft_fu1d_plan");
  // ---- fu2d plans (nufft.cpp:185-187) ----
  t.px = fx.get();
  t.py = fy.get();
  prof::host_mark("host:usfft_fu2d_dimplans");
  // the 2D grid passes hold one M-point double column per CTA (M x 16 B of shared memory,
  // M / 8 threads) and the four-step column passes split M = A B up to 4096: n1, n2 <= 2048
  // (configs[4]'s 2048^3)
  if (t.px.m > 4096 || t.py.m > 4096)
    throw std::invalid_argument("fu2d: n1 and n2 up to 2048 are supported");
  const std::size_t WS = static_cast<std::size_t>(W);
  const DimPlan &px = t.px, &py = t.py;
  const std::size_t T = fg.nu_x.size();
  stg.up(t.x_deconv, px.deconv);
  stg.up(t.y_deconv, py.deconv);
  std::vector<double> pdx(px.deconv.size());
  for (std::size_t i = 0; i < pdx.size(); ++i) pdx[i] = px.pref * py.pref * px.deconv[i];
  stg.up(t.x_pdeconv, pdx);
  std::vector<double2> tf(T), tcf(T);
  for (std::size_t q = 0; q < T; ++q) {
    const std::complex<double> ph = std::complex<double>(px.phase_re[q], px.phase_im[q]) *
                                    std::complex<double>(py.phase_re[q], py.phase_im[q]);
    const std::complex<double> f = (px.pref * py.pref) * ph;
    tf[q] = make_double2(f.real(), f.imag());
    tcf[q] = make_double2(ph.real(), -ph.imag());
  }
  prof::host_mark("host:usfft_fu2d_plans");
  // Classes of coincident targets: equal window origins and kernel weights
  // within 1e-13 (the duplicates differ only by the rounding of cos/sin of
  // theta and theta + pi), at most kClassMax members (the n_theta samples of
  // the origin would otherwise serialise one warp), ordered by 16 x 16 bins
  // of the window origin.
  std::vector<int> order(T);
  for (std::size_t q = 0; q < T; ++q) order[q] = static_cast<int>(q);
  std::vector<std::uint64_t> key(T);
  for (std::size_t q = 0; q < T; ++q) {
    const std::uint64_t r = static_cast<std::uint64_t>(px.start[q]), c = static_cast<std::uint64_t>(py.start[q]);
    key[q] = ((r / 16) << 48) | ((c / 16) << 32) | (r << 16) | c;
  }
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return key[static_cast<std::size_t>(a)] < key[static_cast<std::size_t>(b)]; });
  prof::host_mark("host:usfft_class_sort");
  auto same_weights = [&](std::size_t a, std::size_t b) {
    for (std::size_t k = 0; k < WS; ++k)
      if (std::abs(px.weights[a * WS + k] - px.weights[b * WS + k]) > 1e-13 ||
          std::abs(py.weights[a * WS + k] - py.weights[b * WS + k]) > 1e-13)
        return false;
    return true;
  };
  std::vector<int> rep_of;                   // class representative (lowest target index)
  std::vector<std::vector<int>> members;
  {
    // runs of equal keys are independent (a class never spans two runs): host
    // threads group contiguous ranges of runs, concatenated in order (the
    // sequential scan's class order)
    const int nth = static_cast<int>(std::min<std::size_t>(T / 4096 + 1, std::max(1u, std::min(16u, std::thread::hardware_concurrency()))));
    std::vector<std::size_t> cut(static_cast<std::size_t>(nth) + 1, T);
    cut[0] = 0;
    for (int w = 1; w < nth; ++w) {
      std::size_t j = std::max(cut[static_cast<std::size_t>(w) - 1], T * static_cast<std::size_t>(w) / static_cast<std::size_t>(nth));
      while (j > 0 && j < T && key[static_cast<std::size_t>(order[j])] == key[static_cast<std::size_t>(order[j - 1])]) ++j;
      cut[static_cast<std::size_t>(w)] = j;
    }
    std::vector<std::vector<int>> reps(static_cast<std::size_t>(nth));
    std::vector<std::vector<std::vector<int>>> mems(static_cast<std::size_t>(nth));
    auto group = [&](int w) {
      std::vector<int>& rp = reps[static_cast<std::size_t>(w)];
      std::vector<std::vector<int>>& mb = mems[static_cast<std::size_t>(w)];
      for (std::size_t i = cut[static_cast<std::size_t>(w)]; i < cut[static_cast<std::size_t>(w) + 1];) {
        std::size_t j = i;
        while (j < T && key[static_cast<std::size_t>(order[j])] == key[static_cast<std::size_t>(order[i])]) ++j;
        std::vector<int> run(order.begin() + static_cast<std::ptrdiff_t>(i), order.begin() + static_cast<std::ptrdiff_t>(j));
        std::sort(run.begin(), run.end());
        const std::size_t first_class = mb.size();
        for (const int q : run) {
          std::size_t c = first_class;
          while (c < mb.size() && (mb[c].size() >= kClassMax ||
                                   !same_weights(static_cast<std::size_t>(rp[c]), static_cast<std::size_t>(q))))
            ++c;
          if (c == mb.size()) {
            rp.push_back(q);
            mb.emplace_back();
          }
          mb[c].push_back(q);
        }
        i = j;
      }
    };
    std::vector<std::thread> th;
    for (int w = 1; w < nth; ++w) th.emplace_back(group, w);
    group(0);
    for (auto& x : th) x.join();
    for (int w = 0; w < nth; ++w) {
      rep_of.insert(rep_of.end(), reps[static_cast<std::size_t>(w)].begin(), reps[static_cast<std::size_t>(w)].end());
      for (auto& m : mems[static_cast<std::size_t>(w)]) members.push_back(std::move(m));
    }
  }
  const std::size_t C = members.size();
  t.nclass = static_cast<int>(C);
  prof::host_mark("host:usfft_class_group");
  {
    std::vector<int> r0(C), c0(C), mfirst(C + 1, 0);
    std::vector<double> w1(C * WS), w2(C * WS);
    for (std::size_t c = 0; c < C; ++c) mfirst[c + 1] = mfirst[c] + static_cast<int>(members[c].size());
    std::vector<int> mtidx(static_cast<std::size_t>(mfirst[C]));
    std::vector<double2> mfac(mtidx.size()), mcfac(mtidx.size());
    const int nthc = static_cast<int>(std::min<std::size_t>(C / 2048 + 1, std::max(1u, std::min(16u, std::thread::hardware_concurrency()))));
    auto par_classes = [&](auto&& fn) {  // contiguous class ranges on host threads
      std::vector<std::thread> th;
      const std::size_t per = (C + static_cast<std::size_t>(nthc) - 1) / static_cast<std::size_t>(nthc);
      for (int w = 1; w < nthc; ++w)
        th.emplace_back([&, w] {
          for (std::size_t c = w * per; c < std::min(C, (w + 1) * per); ++c) fn(c);
        });
      for (std::size_t c = 0; c < std::min(C, per); ++c) fn(c);
      for (auto& x : th) x.join();
    };
    par_classes([&](std::size_t c) {
      const std::size_t q = static_cast<std::size_t>(rep_of[c]);
      r0[c] = px.start[q];
      c0[c] = py.start[q];
      std::copy_n(px.weights.begin() + static_cast<std::ptrdiff_t>(q * WS), WS,
                  w1.begin() + static_cast<std::ptrdiff_t>(c * WS));
      std::copy_n(py.weights.begin() + static_cast<std::ptrdiff_t>(q * WS), WS,
                  w2.begin() + static_cast<std::ptrdiff_t>(c * WS));
      std::size_t k = static_cast<std::size_t>(mfirst[c]);
      for (const int e : members[c]) {
        mtidx[k] = static_cast<int>((e / g_.w) << 16 | (e % g_.w));  // packed (t, q)
        mfac[k] = tf[static_cast<std::size_t>(e)];
        mcfac[k] = tcf[static_cast<std::size_t>(e)];
        ++k;
      }
    });
    prof::host_mark("host:usfft_class_tables");
    stg.up(t.t_w1, w1);
    stg.up(t.t_w2, w2);
    stg.up(t.m_first, mfirst);
    stg.up(t.m_tidx, mtidx);
    stg.up(t.m_fac, mfac);
    stg.up(t.m_cfac, mcfac);
    prof::host_mark("host:usfft_class_uploads");
    // the gather's per-class records (bulk-copied into shared memory per CTA)
    auto build = [&](auto tag) {
      using Rec = decltype(tag);
      constexpr int RW = sizeof(Rec::w1) / sizeof(double);
      std::vector<Rec> rv(C);
      par_classes([&](std::size_t c) {
        Rec& r = rv[c];
        std::memset(&r, 0, sizeof(Rec));
        r.r0 = r0[c];
        r.c0 = c0[c];
        r.first = mfirst[c];
        r.nmem = mfirst[c + 1] - mfirst[c];
        for (int e = 0; e < r.nmem; ++e) {
          r.tq[e] = mtidx[static_cast<std::size_t>(mfirst[c] + e)];
          r.fac[e] = mfac[static_cast<std::size_t>(mfirst[c] + e)];
        }
        std::copy_n(w1.begin() + static_cast<std::ptrdiff_t>(c * RW), RW, r.w1);
        std::copy_n(w2.begin() + static_cast<std::ptrdiff_t>(c * RW), RW, r.w2);
      });
      stg.up(t.recs, reinterpret_cast<const unsigned char*>(rv.data()), rv.size() * sizeof(Rec));
    };
    if (W == kEsTaps) build(ClassRec<kEsTaps>{});
    else build(ClassRec<kTaps>{});
  }
  prof::host_mark("host:usfft_classes");
  {  // spread patches: 8x4 cells -> targets whose W x W window touches them (targets ascending)
    const std::int64_t npr = px.m / kPatchR, npc = py.m / kPatchC;
    const int npatch = static_cast<int>(npr * npc);
    // patches touched by a class's W x W window (dedup within the class): its
    // distinct patch rows and columns (in first-touch order), then their product
    // in the row-major order of the full W x W scan
    auto patches_of = [&](std::size_t c, std::vector<std::int64_t>& prs, std::vector<std::int64_t>& pcs,
                          std::vector<int>& touched) {
      const std::size_t q = static_cast<std::size_t>(rep_of[c]);
      prs.clear();
      pcs.clear();
      for (int a = 0; a < W; ++a) {
        const std::int64_t pr = ((px.start[q] + a) % px.m + px.m) % px.m / kPatchR;
        if (std::find(prs.begin(), prs.end(), pr) == prs.end()) prs.push_back(pr);
        const std::int64_t pc = ((py.start[q] + a) % py.m + py.m) % py.m / kPatchC;
        if (std::find(pcs.begin(), pcs.end(), pc) == pcs.end()) pcs.push_back(pc);
      }
      touched.clear();
      for (const std::int64_t pr : prs)
        for (const std::int64_t pc : pcs) touched.push_back(static_cast<int>(pr * npc + pc));
    };
    // CSR patch -> classes, classes ascending within a patch: host threads own
    // contiguous class ranges, count per patch, then fill from per-thread offsets
    // (thread 0's classes first), which is the sequential order
    constexpr int kHostThreads = 8;
    const std::size_t per = (C + kHostThreads - 1) / kHostThreads;
    std::vector<std::vector<int>> tcnt(kHostThreads, std::vector<int>(static_cast<std::size_t>(npatch), 0));
    std::vector<int> cnt(static_cast<std::size_t>(npatch + 1), 0);
    std::vector<int2> lst;
    auto run = [&](auto&& body) {
      std::vector<std::thread> th;
      for (int w = 0; w < kHostThreads; ++w)
        th.emplace_back([&, w] {
          std::vector<std::int64_t> prs, pcs;
          std::vector<int> touched;
          for (std::size_t c = w * per; c < std::min(C, (w + 1) * per); ++c) {
            patches_of(c, prs, pcs, touched);
            body(w, c, touched);
          }
        });
      for (auto& x : th) x.join();
    };
    run([&](int w, std::size_t, const std::vector<int>& touched) {
      for (const int p : touched) ++tcnt[static_cast<std::size_t>(w)][static_cast<std::size_t>(p)];
    });
    for (int p = 0; p < npatch; ++p) {
      int tot = 0;
      for (int w = 0; w < kHostThreads; ++w) tot += tcnt[static_cast<std::size_t>(w)][static_cast<std::size_t>(p)];
      cnt[static_cast<std::size_t>(p) + 1] = cnt[static_cast<std::size_t>(p)] + tot;
    }
    lst.resize(static_cast<std::size_t>(cnt.back()));
    for (int p = 0; p < npatch; ++p) {  // tcnt becomes each thread's fill position
      int at = cnt[static_cast<std::size_t>(p)];
      for (int w = 0; w < kHostThreads; ++w) {
        const int n = tcnt[static_cast<std::size_t>(w)][static_cast<std::size_t>(p)];
        tcnt[static_cast<std::size_t>(w)][static_cast<std::size_t>(p)] = at;
        at += n;
      }
    }
    run([&](int w, std::size_t c, const std::vector<int>& touched) {
      const std::size_t q = static_cast<std::size_t>(rep_of[c]);
      for (const int p : touched) {  // the window offsets of the patch origin (the kernel's a0, b0)
        const std::int64_t a0 = ((p / npc * kPatchR - px.start[q]) % px.m + px.m) % px.m;
        const std::int64_t b0 = ((p % npc * kPatchC - py.start[q]) % py.m + py.m) % py.m;
        lst[static_cast<std::size_t>(tcnt[static_cast<std::size_t>(w)][static_cast<std::size_t>(p)]++)] =
            make_int2(static_cast<int>(c), static_cast<int>(a0 | b0 << 16));
      }
    });
    std::vector<int> porder(static_cast<std::size_t>(npatch));
    for (int p = 0; p < npatch; ++p) porder[static_cast<std::size_t>(p)] = p;
    std::stable_sort(porder.begin(), porder.end(), [&](int a, int b) {
      return cnt[static_cast<std::size_t>(a) + 1] - cnt[static_cast<std::size_t>(a)] >
             cnt[static_cast<std::size_t>(b) + 1] - cnt[static_cast<std::size_t>(b)];
    });
    std::vector<SpreadItem> items;
    std::vector<int4> split;
    int slots = 0;
    for (const int p : porder) {  // heaviest first
      const int e0 = cnt[static_cast<std::size_t>(p)], e1 = cnt[static_cast<std::size_t>(p) + 1];
      if (e1 - e0 <= kSplit) {
        items.push_back(SpreadItem{p, e0, e1, -1, -1});
        continue;
      }
      const int first = slots;
      const int grp = static_cast<int>(split.size());
      for (int e = e0; e < e1; e += kSplit) items.push_back(SpreadItem{p, e, std::min(e1, e + kSplit), slots++, grp});
      split.push_back(make_int4(p, first, slots - first, 0));
    }
    t.nitems = static_cast<int>(items.size());
    t.nsplit = static_cast<int>(split.size());
    stg.up(t.items, items);
    stg.up(t.split, split);
    t.partial.resize(static_cast<std::size_t>(std::max(slots, 1)) * 32 * KB);
    t.split_cnt.resize(static_cast<std::size_t>(std::max(t.nsplit, 1)));
    t.split_cnt.zero(stream_);
    stg.up(t.patch_t, lst);
  }
  stg.up(t.x_tw, twiddles(px.m));
  stg.up(t.y_tw, twiddles(py.m));
  t.cols4 = use_cols4(px.m);
  if (t.cols4) {
    t.logA = px.logm / 2;
    stg.up(t.a_tw, twiddles(std::int64_t{1} << t.logA));
    stg.up(t.b_tw, twiddles(std::int64_t{1} << (px.logm - t.logA)));
  }
  prof::host_mark("host:usfft_patches");
  t.wide = (kernel_ == GridKernel::gaussian || wide_grids_env()) && !t.cols4;
  t.ghost = (W - 1 + 7) & ~7;
  t.ldg = static_cast<int>(py.m) + t.ghost;
  t.S.resize(static_cast<std::size_t>(px.m * t.ldg * KB));
  t.Gd.resize(static_cast<std::size_t>(px.m * t.ldg * KB) * (t.wide ? 2 : 1));
  t.val.resize(C * KB);
  {  // classes per gather CTA: ~gather_per_cta(), rounded so the grid is whole waves
    int nb = 0;
    const std::size_t rb = static_cast<std::size_t>(gather_per_cta()) *
                           (W == kEsTaps ? sizeof(ClassRec<kEsTaps>) : sizeof(ClassRec<kTaps>));
    if (t.wide && W == kEsTaps) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fu2d_gather<kEsTaps, double2>, 32 * kGatherWarps, rb);
    else if (t.wide) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fu2d_gather<kTaps, double2>, 32 * kGatherWarps, rb);
    else if (W == kEsTaps) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fu2d_gather<kEsTaps, float2>, 32 * kGatherWarps, rb);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fu2d_gather<kTaps, float2>, 32 * kGatherWarps, rb);
    const std::int64_t slots = std::max(1, nb) * static_cast<std::int64_t>(sm_count());
    const std::int64_t per = gather_per_cta();
    const std::int64_t waves = std::max<std::int64_t>(1, (static_cast<std::int64_t>(C) + per * slots - 1) / (per * slots));
    t.gather_per = static_cast<int>(std::max<std::int64_t>(1, (static_cast<std::int64_t>(C) + waves * slots - 1) / (waves * slots)));
    if (std::getenv("MLRG_GATHER_PER_CTA")) t.gather_per = static_cast<int>(per);
  }

  // ---- f2d (operators.cpp:20-74) ----
  t.f2d_fft = is_pow2(g_.h) && is_pow2(g_.w) && g_.h >= 8 && g_.w >= 8;
  if (t.f2d_fft) {
    stg.up(t.h_tw, twiddles(g_.h));
    stg.up(t.w_tw, twiddles(g_.w));
  } else {
    auto mat = [](std::int64_t n, bool conj) {
      std::vector<double2> W(static_cast<std::size_t>(n * n));
      const double c = static_cast<double>(n) / 2.0, sc = 1.0 / std::sqrt(static_cast<double>(n));
      for (std::int64_t k = 0; k < n; ++k)
        for (std::int64_t m = 0; m < n; ++m) {
          const std::complex<double> z = std::polar(
              sc, -2.0 * std::numbers::pi * (static_cast<double>(k) - c) * (static_cast<double>(m) - c) /
                      static_cast<double>(n));
          W[static_cast<std::size_t>(k * n + m)] = make_double2(z.real(), conj ? -z.imag() : z.imag());
        }
      return W;
    };
    stg.up(t.Wh, mat(g_.h, false));
    stg.up(t.Ww, mat(g_.w, false));
    stg.up(t.Whc, mat(g_.h, true));
    stg.up(t.Wwc, mat(g_.w, true));
  }
  MLRG_CUDA(cudaStreamSynchronize(stream_));
  static bool smem_set = [] {
    allow_big_smem(k_fu1d<float2, kEsTaps, false, false>);
    allow_big_smem(k_fu1d<double2, kEsTaps, false, false>);
    allow_big_smem(k_fu1d<double2, kEsTaps, true, false>);
    allow_big_smem(k_fu1d<float2, kTaps, false, false>);
    allow_big_smem(k_fu1d<double2, kTaps, false, false>);
    allow_big_smem(k_fu1d<double2, kTaps, true, false>);
    allow_big_smem(k_fu1d<float2, kEsTaps, false, true>);
    allow_big_smem(k_fu1d<double2, kEsTaps, false, true>);
    allow_big_smem(k_fu1d<double2, kEsTaps, true, true>);
    allow_big_smem(k_fu1d<float2, kTaps, false, true>);
    allow_big_smem(k_fu1d<double2, kTaps, false, true>);
    allow_big_smem(k_fu1d<double2, kTaps, true, true>);
    allow_big_smem(k_fu1d_adj<float2>);
    allow_big_smem(k_fu1d_adj<double2>);
    allow_big_smem(k_fu2d_rows<false, false>);
    allow_big_smem(k_fu2d_rows<true, false>);
    allow_big_smem(k_fu2d_rows<false, true>);
    allow_big_smem(k_fu2d_rows<true, true>);
    allow_big_smem(k_fu2d_adj_spread<kEsTaps, float2>);
    allow_big_smem(k_fu2d_adj_spread<kTaps, float2>);
    allow_big_smem(k_fu2d_adj_spread<kTaps, double2>);
    allow_big_smem(k_fu2d_adj_spread<kEsTaps, double2>);
    allow_big_smem(k_fu2d_cols<false, float2>);
    allow_big_smem(k_fu2d_cols<true, float2>);
    allow_big_smem(k_fu2d_cols<false, double2>);
    allow_big_smem(k_fu2d_cols<true, double2>);
    allow_big_smem(k_fu2d_adj_cols<float2>);
    allow_big_smem(k_fu2d_adj_cols<double2>);
    allow_big_smem(k_cols4_pass1<+1, true, true>);
    allow_big_smem(k_cols4_pass1<-1, false, true>);
    allow_big_smem(k_cols4_pass2<+1, false, true>);
    allow_big_smem(k_cols4_pass2<-1, true, true>);
    allow_big_smem(k_fu2d_adj_rows<false, false>);
    allow_big_smem(k_fu2d_adj_rows<true, false>);
    allow_big_smem(k_fu2d_adj_rows<false, true>);
    allow_big_smem(k_fu2d_adj_rows<true, true>);
    allow_big_smem(k_center_fft_rows<+1>);
    allow_big_smem(k_center_fft_rows<-1>);
    allow_big_smem(k_center_fft_cols<+1>);
    allow_big_smem(k_center_fft_cols<-1>);
    return true;
  }();
  (void)smem_set;
}

// streams of the fu2d / fu2d_adj row-batch pipeline (MLRG_FU2D_STREAMS, default 2;
// MLRG_FU2D_PIPE=0: one)
int pipe_streams() {
  static const int k = [] {
    if (!pipelined()) return 1;
    const char* e = std::getenv("MLRG_FU2D_STREAMS");
    return e ? std::clamp(std::atoi(e), 1, 8) : 2;
  }();
  return k;
}

// CUDA graphs of the fu2d / fu2d_adj kernel sequences (one per distinct call):
// 3 kernels per 16-row batch on K streams make a call 48+ launches at 256^3,
// launch-bound at the small configs[0] volume.
bool graphs_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("MLRG_GRAPHS");
    return !(e && *e == '0');
  }();
  return v;
}

struct GraphKey {
  std::string s;
  template <class T>
  GraphKey& add(const T& x) {
    static_assert(std::is_trivially_copyable_v<T>);
    s.append(reinterpret_cast<const char*>(&x), sizeof(T));
    return *this;
  }
  GraphKey& add(const char* tag) {
    s.append(tag);
    s.push_back('\0');
    return *this;
  }
};

struct Usfft::Graphs {
  struct Entry {
    cudaGraphExec_t exec = nullptr;
    std::uint64_t launches = 0;
  };
  std::unordered_map<std::string, Entry> exec;
  std::unordered_set<std::string> seen;
  cudaStream_t capture = nullptr;  // the engine stream may be the legacy default stream (not capturable)
  ~Graphs() {
    for (auto& [k, e] : exec)
      if (e.exec) cudaGraphExecDestroy(e.exec);
    if (capture) cudaStreamDestroy(capture);
  }
};

template <class F>
void Usfft::graph_run(const std::string& key, F&& enqueue) {
  if (!graphs_enabled() || prof::enabled()) return enqueue();
  if (!graphs_) graphs_ = new Graphs;
  auto it = graphs_->exec.find(key);
  if (it != graphs_->exec.end()) {
    MLRG_CUDA(cudaGraphLaunch(it->second.exec, stream_));
    prof::count_launches(it->second.launches);
    return;
  }
  // first call: buffers and side streams get made; a bounded cache (the solver makes
  // a handful of distinct calls; callers cycling through many arrays launch plainly)
  constexpr std::size_t kMaxGraphs = 64;
  if (graphs_->seen.size() > 4096) graphs_->seen.clear();
  if (graphs_->exec.size() >= kMaxGraphs || graphs_->seen.insert(key).second) return enqueue();
  if (!graphs_->capture) MLRG_CUDA(cudaStreamCreateWithFlags(&graphs_->capture, cudaStreamNonBlocking));
  const std::uint64_t n0 = prof::launches();
  cudaGraph_t g = nullptr;
  // capture on a private stream standing in for the engine stream (the kernels'
  // order and the side streams' fork/join are the same), replay on the engine stream
  const cudaStream_t engine = stream_;
  stream_ = graphs_->capture;
  MLRG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue();
  } catch (...) {
    cudaStreamEndCapture(stream_, &g);
    stream_ = engine;
    if (g) cudaGraphDestroy(g);
    throw;
  }
  const cudaError_t ce = cudaStreamEndCapture(stream_, &g);
  stream_ = engine;
  MLRG_CUDA(ce);
  Graphs::Entry e;
  e.launches = prof::launches() - n0;
  prof::count_launches(0);
  MLRG_CUDA(cudaGraphInstantiate(&e.exec, g, 0));
  MLRG_CUDA(cudaGraphDestroy(g));
  MLRG_CUDA(cudaGraphLaunch(e.exec, stream_));
  graphs_->exec.emplace(key, e);
}

void Usfft::ensure_side() {
  Tables& t = *t_;
  if (!t.ev_fork) MLRG_CUDA(cudaEventCreateWithFlags(&t.ev_fork, cudaEventDisableTiming));
  while (static_cast<int>(t.sides.size()) + 1 < pipe_streams()) {
    auto l = std::make_unique<Tables::Lane>();
    MLRG_CUDA(cudaStreamCreateWithFlags(&l->s, cudaStreamNonBlocking));
    MLRG_CUDA(cudaEventCreateWithFlags(&l->ev_join, cudaEventDisableTiming));
    l->S.resize(t.S.size());
    l->Gd.resize(t.Gd.size());
    t.sides.push_back(std::move(l));
  }
}

Usfft::~Usfft() {
  delete graphs_;
  for (auto& l : t_->sides) {
    cudaStreamSynchronize(l->s);
    cudaStreamDestroy(l->s);
    cudaEventDestroy(l->ev_join);
  }
  if (t_->ev_fork) cudaEventDestroy(t_->ev_fork);
  delete t_;
}

int Usfft::reduce_grid() const { return 4 * sm_count(); }

template <class TIn>
void Usfft::fu1d_t(const TIn* u, float2* out, std::int64_t d0, const PeerOut* peer) {
  if (d0 <= 0) return;
  const Tables& t = *t_;
  const int ncol = t.z_ncol;
  const dim3 grid(static_cast<unsigned>((g_.n2 + ncol - 1) / ncol), static_cast<unsigned>(d0));
  const std::size_t smem = static_cast<std::size_t>(t.pz.m * ncol) * sizeof(double2);
  prof::begin("k_fu1d", stream_);
  const bool zp = zero_padded(t.pz);
  auto pick = [&](auto es, auto ga) { return t.pz.taps == kEsTaps ? es : ga; };
  auto kern = zp ? pick(k_fu1d<TIn, kEsTaps, false, true>, k_fu1d<TIn, kTaps, false, true>)
                 : pick(k_fu1d<TIn, kEsTaps, false, false>, k_fu1d<TIn, kTaps, false, false>);
  if constexpr (std::is_same_v<TIn, double2>)
    if (peer)
      kern = zp ? pick(k_fu1d<TIn, kEsTaps, true, true>, k_fu1d<TIn, kTaps, true, true>)
                : pick(k_fu1d<TIn, kEsTaps, true, false>, k_fu1d<TIn, kTaps, true, false>);
  kern<<<grid, static_cast<unsigned>(ncol * t.pz.m / 8), smem, stream_>>>(u, out, static_cast<int>(g_.n0), static_cast<int>(g_.n2),
                                     static_cast<int>(g_.h), t.pz.logm, static_cast<int>(t.pz.center), ncol,
                                     t.z_deconv.get(), t.z_start.get(), t.z_w.get(), t.z_fac.get(), t.z_tw.get(),
                                     peer ? *peer : PeerOut{}, Skip{skip_, 0, 16});
  MLRG_LAUNCH_CHECK("k_fu1d");
  prof::end("k_fu1d", stream_);
}

template <class TOut>
void Usfft::fu1d_adj_t(const float2* v, TOut* out, std::int64_t d0) {
  if (d0 <= 0) return;
  const Tables& t = *t_;
  const int ncol = t.z_ncol_adj;
  const dim3 grid(static_cast<unsigned>((g_.n2 + ncol - 1) / ncol), static_cast<unsigned>(d0));
  const std::size_t smem = static_cast<std::size_t>((t.pz.m + g_.h) * ncol) * sizeof(double2);
  prof::begin("k_fu1d_adj", stream_);
  k_fu1d_adj<TOut><<<grid, static_cast<unsigned>(ncol * t.pz.m / 8), smem, stream_>>>(v, out, static_cast<int>(g_.n0), static_cast<int>(g_.n2),
                                                 static_cast<int>(g_.h), t.pz.logm, static_cast<int>(t.pz.center),
                                                 ncol, t.z_cphase.get(), t.z_cell_ptr.get(), t.z_cell_k.get(),
                                                 t.z_cell_w.get(), t.z_pdeconv.get(), t.z_tw.get(),
                                                 Skip{skip_, 0, 16});
  MLRG_LAUNCH_CHECK("k_fu1d_adj");
  prof::end("k_fu1d_adj", stream_);
}

void Usfft::fu1d(const float2* u, float2* out, std::int64_t d0) { fu1d_t(u, out, d0, nullptr); }
void Usfft::fu1d(const double2* u, float2* out, std::int64_t d0, const PeerOut* peer) { fu1d_t(u, out, d0, peer); }
void Usfft::fu1d_adj(const float2* v, float2* out, std::int64_t d0) { fu1d_adj_t(v, out, d0); }
void Usfft::fu1d_adj(const float2* v, double2* out, std::int64_t d0) { fu1d_adj_t(v, out, d0); }

int Usfft::fu2d(const float2* v, std::int64_t ld, std::int64_t k0, std::int64_t nk, const Fu2dEpilogue& epi) {
  const Tables& t = *t_;
  const int ks1 = pass_cols(t.px.m), ks2 = pass_cols(t.py.m);
  const int per_cta = t.gather_per;
  const int ggrid = (t.nclass + per_cta - 1) / per_cta;
  Tables& tm = *t_;
  // class sums for a following fu2d_adj of this output (memo skip flags would
  // leave batches uncomputed: not with them)
  const bool cls = epi.class_sums && epi.out && !skip_ && nk > 0;
  cls_src_ = cls ? epi.out : nullptr;
  if (cls) {
    tm.cls.resize(static_cast<std::size_t>((nk + KB - 1) / KB) * static_cast<std::size_t>(t.nclass) * KB);
    cls_ld_ = epi.ld_out;
    cls_k0_ = epi.k0_out;
    cls_nk_ = nk;
  }
  // K streams take the row batches round robin (stream j: batches j, j + K, ...)
  const int K = static_cast<int>(std::min<std::int64_t>(pipe_streams(), (nk + KB - 1) / KB));
  const bool pipe = K > 1;
  auto enqueue = [&] {
  if (pipe) {
    ensure_side();
    MLRG_CUDA(cudaEventRecord(tm.ev_fork, stream_));  // inputs and partial slots ready
    for (int j = 1; j < K; ++j) MLRG_CUDA(cudaStreamWaitEvent(tm.sides[static_cast<std::size_t>(j - 1)]->s, tm.ev_fork, 0));
  }
  int bi = 0;
  for (std::int64_t b = 0; b < nk; b += KB, ++bi) {
    const int nb = static_cast<int>(std::min<std::int64_t>(KB, nk - b));
    const int lane = pipe ? bi % K : 0;
    Tables::Lane* L = lane ? tm.sides[static_cast<std::size_t>(lane - 1)].get() : nullptr;
    cudaStream_t s = L ? L->s : stream_;
    float2* S = L ? L->S.get() : t.S.get();
    float2* Gd = L ? L->Gd.get() : t.Gd.get();
    const Skip sk{skip_, static_cast<int>((k0 + b) / KB), 1};
    prof::begin("k_fu2d_rows", s);
    auto rows = zero_padded(t.py) ? (t.cols4 ? k_fu2d_rows<true, true> : k_fu2d_rows<true, false>)
                                  : (t.cols4 ? k_fu2d_rows<false, true> : k_fu2d_rows<false, false>);
    rows<<<dim3(KB / ks2, static_cast<unsigned>(g_.n1)), static_cast<unsigned>(ks2 * t.py.m / 8),
                  static_cast<std::size_t>(t.py.m * (ks2 + 1)) * sizeof(double2), s>>>(
        v, ld, k0 + b, nb, static_cast<int>(g_.n2), t.py.logm, static_cast<int>(t.py.center), ks2, t.x_deconv.get(),
        t.y_deconv.get(), t.y_tw.get(), S, sk);
    MLRG_LAUNCH_CHECK("k_fu2d_rows");
    prof::end("k_fu2d_rows", s);
    prof::begin("k_fu2d_cols", s);
    const float2* G = Gd;
    if (t.cols4) {  // S -> Gd (intermediate) -> S (the grid, all M1 rows)
      const int A = 1 << t.logA, B = t.px.m >> t.logA;
      const unsigned nc = static_cast<unsigned>(t.py.m / kCols4);
      k_cols4_pass1<+1, true, true><<<dim3(B, nc), kCols4Lanes * A / 8, static_cast<std::size_t>(A * (kCols4Lanes + 1)) * sizeof(double2), s>>>(
          S, static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center), t.logA, t.py.logm, t.a_tw.get(),
          t.x_tw.get(), Gd, sk);
      MLRG_LAUNCH_CHECK("k_cols4_pass1");
      k_cols4_pass2<+1, false, true><<<dim3(A, nc), kCols4Lanes * B / 8, static_cast<std::size_t>(B * kCols4Lanes) * sizeof(double2), s>>>(
          Gd, static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center), t.logA, t.py.logm, t.b_tw.get(), S,
          t.ldg, t.ghost, sk);
      MLRG_LAUNCH_CHECK("k_cols4_pass2");
      G = S;
    } else if (t.wide) {
      (zero_padded(t.px) ? k_fu2d_cols<true, double2> : k_fu2d_cols<false, double2>)<<<dim3(KB / ks1, static_cast<unsigned>(t.py.m)), static_cast<unsigned>(ks1 * t.px.m / 8),
                    static_cast<std::size_t>(t.px.m * ks1) * sizeof(double2), s>>>(
          S, static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center), t.py.logm, ks1, t.x_tw.get(),
          reinterpret_cast<double2*>(Gd), t.ldg, t.ghost, sk);
      MLRG_LAUNCH_CHECK("k_fu2d_cols");
    } else {
      (zero_padded(t.px) ? k_fu2d_cols<true, float2> : k_fu2d_cols<false, float2>)<<<dim3(KB / ks1, static_cast<unsigned>(t.py.m)), static_cast<unsigned>(ks1 * t.px.m / 8),
                    static_cast<std::size_t>(t.px.m * ks1) * sizeof(double2), s>>>(
          S, static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center), t.py.logm, ks1, t.x_tw.get(), Gd,
          t.ldg, t.ghost, sk);
      MLRG_LAUNCH_CHECK("k_fu2d_cols");
    }
    prof::end("k_fu2d_cols", s);
    GatherOut eo{epi.out, epi.ld_out, epi.k0_out + b, epi.sub, epi.ld_sub, epi.k0_sub + b,
                 epi.dot, epi.ld_dot, epi.k0_dot + b, epi.reduce ? 1 : 0,
                 cls ? tm.cls.get() + static_cast<long long>(bi) * t.nclass * KB : nullptr, t.m_cfac.get()};
    prof::begin("k_fu2d_gather", s);
    // each stream accumulates into its own partial slots (stream j: [2 j ggrid, 2 (j + 1) ggrid))
    auto launch_gather = [&](auto kern, auto grid_ptr, auto rec_tag) {
      using Rec = decltype(rec_tag);
      kern<<<ggrid, 32 * kGatherWarps, static_cast<std::size_t>(per_cta) * sizeof(Rec), s>>>(
          grid_ptr, t.nclass, static_cast<int>(g_.w), t.px.logm, t.ldg, nb, reinterpret_cast<const Rec*>(t.recs.get()),
          eo, per_cta, partials_.dev() + 2 * lane * ggrid, bi >= K ? 1 : 0, sk);
    };
    if (t.wide && t.px.taps == kEsTaps) launch_gather(k_fu2d_gather<kEsTaps, double2>, reinterpret_cast<const double2*>(G), ClassRec<kEsTaps>{});
    else if (t.wide) launch_gather(k_fu2d_gather<kTaps, double2>, reinterpret_cast<const double2*>(G), ClassRec<kTaps>{});
    else if (t.px.taps == kEsTaps) launch_gather(k_fu2d_gather<kEsTaps, float2>, G, ClassRec<kEsTaps>{});
    else launch_gather(k_fu2d_gather<kTaps, float2>, G, ClassRec<kTaps>{});
    MLRG_LAUNCH_CHECK("k_fu2d_gather");
    prof::end("k_fu2d_gather", s);
  }
  if (pipe)
    for (int j = 1; j < K; ++j) {
      Tables::Lane& l = *tm.sides[static_cast<std::size_t>(j - 1)];
      MLRG_CUDA(cudaEventRecord(l.ev_join, l.s));
      MLRG_CUDA(cudaStreamWaitEvent(stream_, l.ev_join, 0));
    }
  };
  GraphKey key;
  key.add("fu2d").add(v).add(ld).add(k0).add(nk).add(epi.out).add(epi.ld_out).add(epi.k0_out).add(epi.sub)
      .add(epi.ld_sub).add(epi.k0_sub).add(epi.dot).add(epi.ld_dot).add(epi.k0_dot).add(epi.reduce).add(cls)
      .add(skip_).add(K).add(tm.cls.get());
  graph_run(key.s, enqueue);
  return epi.reduce && nk > 0 ? 2 * K * ggrid : 0;
}

Usfft::Stats Usfft::stats() const {
  const Tables& t = *t_;
  const std::int64_t per = t.gather_per;
  return {t.nclass, t.px.taps, t.px.m, t.py.m, (t.nclass + per - 1) / per, per};
}

void Usfft::fu2d_adj(const float2* p, std::int64_t ld, std::int64_t k0, std::int64_t nk, float2* out,
                     std::int64_t ld_out, std::int64_t k0_out, const PeerOut* peer) {
  const Tables& t = *t_;
  const int ks1 = pass_cols(t.px.m), ks2 = pass_cols(t.py.m);
  Tables& tm = *t_;
  // p is exactly the output a class_sums fu2d just produced: its class sums replace the prep pass
  const bool use_cls = cls_src_ && p == cls_src_ && ld == cls_ld_ && k0 == cls_k0_ && nk == cls_nk_ && !skip_;
  cls_src_ = nullptr;
  // row batches round robin over K streams, as in fu2d
  const int K = static_cast<int>(std::min<std::int64_t>(pipe_streams(), (nk + KB - 1) / KB));
  const bool pipe = K > 1;
  auto enqueue = [&] {
  if (pipe) {
    ensure_side();
    for (auto& l : tm.sides)
      if (l->val.size() != tm.val.size()) {
        l->val.resize(tm.val.size());
        l->partial.resize(tm.partial.size());
        l->split_cnt.resize(tm.split_cnt.size());
        l->split_cnt.zero(stream_);
      }
    MLRG_CUDA(cudaEventRecord(tm.ev_fork, stream_));
    for (int j = 1; j < K; ++j) MLRG_CUDA(cudaStreamWaitEvent(tm.sides[static_cast<std::size_t>(j - 1)]->s, tm.ev_fork, 0));
  }
  int bi = 0;
  for (std::int64_t b = 0; b < nk; b += KB, ++bi) {
    const int nb = static_cast<int>(std::min<std::int64_t>(KB, nk - b));
    const int lane = pipe ? bi % K : 0;
    Tables::Lane* L = lane ? tm.sides[static_cast<std::size_t>(lane - 1)].get() : nullptr;
    cudaStream_t s = L ? L->s : stream_;
    float2* S = L ? L->S.get() : t.S.get();
    float2* Gd = L ? L->Gd.get() : t.Gd.get();
    double2* val = use_cls ? tm.cls.get() + static_cast<long long>(bi) * t.nclass * KB : L ? L->val.get() : t.val.get();
    double2* partial = L ? L->partial.get() : t.partial.get();
    int* split_cnt = L ? L->split_cnt.get() : tm.split_cnt.get();
    const Skip sk{skip_, static_cast<int>((k0 + b) / KB), 1};
    if (!use_cls) {
    prof::begin("k_fu2d_adj_prep", s);
    k_fu2d_adj_prep<<<static_cast<unsigned>((t.nclass + 15) / 16), 256, 0, s>>>(
        p, ld, k0 + b, nb, t.nclass, static_cast<int>(g_.w), t.m_first.get(), t.m_tidx.get(), t.m_cfac.get(), val,
        sk);
    MLRG_LAUNCH_CHECK("k_fu2d_adj_prep");
    prof::end("k_fu2d_adj_prep", s);
    }
    prof::begin("k_fu2d_adj_spread", s);
    auto spread = t.px.taps == kEsTaps ? k_fu2d_adj_spread<kEsTaps, float2> : k_fu2d_adj_spread<kTaps, float2>;
    if (t.wide)
      (t.px.taps == kEsTaps ? k_fu2d_adj_spread<kEsTaps, double2> : k_fu2d_adj_spread<kTaps, double2>)<<<(t.nitems + 1) / 2, 128, sizeof(SpreadShared), s>>>(
          val, t.px.logm, t.py.logm, t.nitems, t.items.get(), t.patch_t.get(),
          t.t_w1.get(), t.t_w2.get(), reinterpret_cast<double2*>(Gd), partial, t.split.get(), split_cnt, sk);
    else
      spread<<<(t.nitems + 1) / 2, 128, sizeof(SpreadShared), s>>>(val, t.px.logm, t.py.logm, t.nitems, t.items.get(),
                                                                 t.patch_t.get(), t.t_w1.get(), t.t_w2.get(), Gd, partial, t.split.get(),
                                                                 split_cnt, sk);
    MLRG_LAUNCH_CHECK("k_fu2d_adj_spread");
    prof::end("k_fu2d_adj_spread", s);
    prof::begin("k_fu2d_adj_cols", s);
    const float2* Sc = S;
    if (t.cols4) {  // Gd -> S (intermediate) -> Gd (rows of the n1 mode slots)
      const int A = 1 << t.logA, B = t.px.m >> t.logA;
      const unsigned nc = static_cast<unsigned>(t.py.m / kCols4);
      k_cols4_pass1<-1, false, true><<<dim3(B, nc), kCols4Lanes * A / 8, static_cast<std::size_t>(A * (kCols4Lanes + 1)) * sizeof(double2), s>>>(
          Gd, static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center), t.logA, t.py.logm, t.a_tw.get(),
          t.x_tw.get(), S, sk);
      MLRG_LAUNCH_CHECK("k_cols4_pass1");
      k_cols4_pass2<-1, true, true><<<dim3(A, nc), kCols4Lanes * B / 8, static_cast<std::size_t>(B * kCols4Lanes) * sizeof(double2), s>>>(
          S, static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center), t.logA, t.py.logm, t.b_tw.get(), Gd,
          static_cast<int>(t.py.m), 0, sk);
      MLRG_LAUNCH_CHECK("k_cols4_pass2");
      Sc = Gd;
    } else if (t.wide) {
      k_fu2d_adj_cols<double2><<<dim3(KB / ks1, static_cast<unsigned>(t.py.m)), static_cast<unsigned>(ks1 * t.px.m / 8),
                                 static_cast<std::size_t>(t.px.m * ks1) * sizeof(double2), s>>>(
          reinterpret_cast<const double2*>(Gd), static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center),
          t.py.logm, ks1, t.x_tw.get(), S, sk);
      MLRG_LAUNCH_CHECK("k_fu2d_adj_cols");
    } else {
      k_fu2d_adj_cols<float2><<<dim3(KB / ks1, static_cast<unsigned>(t.py.m)), static_cast<unsigned>(ks1 * t.px.m / 8),
                                static_cast<std::size_t>(t.px.m * ks1) * sizeof(double2), s>>>(
          Gd, static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center), t.py.logm, ks1, t.x_tw.get(), S, sk);
      MLRG_LAUNCH_CHECK("k_fu2d_adj_cols");
    }
    prof::end("k_fu2d_adj_cols", s);
    prof::begin("k_fu2d_adj_rows", s);
    auto arows = peer ? (t.cols4 ? k_fu2d_adj_rows<true, true> : k_fu2d_adj_rows<true, false>)
                      : (t.cols4 ? k_fu2d_adj_rows<false, true> : k_fu2d_adj_rows<false, false>);
    arows<<<dim3(KB / ks2, static_cast<unsigned>(g_.n1)),
                                                              static_cast<unsigned>(ks2 * t.py.m / 8),
                                                              static_cast<std::size_t>(t.py.m * (ks2 + 1)) *
                                                                  sizeof(double2),
                                                              s>>>(
        Sc, nb, static_cast<int>(g_.n2), t.py.logm, static_cast<int>(t.py.center), ks2, t.x_pdeconv.get(),
        t.y_deconv.get(), t.y_tw.get(), out, ld_out, k0_out + b, peer ? *peer : PeerOut{}, sk);
    MLRG_LAUNCH_CHECK("k_fu2d_adj_rows");
    prof::end("k_fu2d_adj_rows", s);
  }
  if (pipe)
    for (int j = 1; j < K; ++j) {
      Tables::Lane& l = *tm.sides[static_cast<std::size_t>(j - 1)];
      MLRG_CUDA(cudaEventRecord(l.ev_join, l.s));
      MLRG_CUDA(cudaStreamWaitEvent(stream_, l.ev_join, 0));
    }
  };
  if (peer) return enqueue();  // sharded: fenced exchanges, plain launches
  GraphKey key;
  key.add("fu2d_adj").add(p).add(ld).add(k0).add(nk).add(out).add(ld_out).add(k0_out).add(use_cls).add(skip_).add(K)
      .add(tm.cls.get());
  graph_run(key.s, enqueue);
}

void Usfft::f2d(const float2* p, float2* out, std::int64_t count, bool adjoint) {
  cls_src_ = nullptr;
  if (count <= 0) return;
  Tables& t = *t_;
  const std::int64_t h = g_.h, w = g_.w;
  if (t.f2d_fft) {
    // rows (along w) into out, then columns (along h) in place
    const int lw = ilog2(w), lh = ilog2(h);
    const int ncr = static_cast<int>(std::clamp<std::int64_t>(fft_elems() / w, 1, 64));
    const std::int64_t rows = count * h;
    const std::size_t smr = static_cast<std::size_t>(w * (ncr + 1)) * sizeof(double2);
    const double sw = 1.0 / std::sqrt(static_cast<double>(w)), sh = 1.0 / std::sqrt(static_cast<double>(h));
    const unsigned gr = static_cast<unsigned>((rows + ncr - 1) / ncr);
    const unsigned tr = static_cast<unsigned>(ncr * w / 8);
    if (adjoint) k_center_fft_rows<+1><<<gr, tr, smr, stream_>>>(p, out, rows, lw, ncr, sw, t.w_tw.get());
    else k_center_fft_rows<-1><<<gr, tr, smr, stream_>>>(p, out, rows, lw, ncr, sw, t.w_tw.get());
    MLRG_LAUNCH_CHECK("k_center_fft_rows");
    const int ncc = static_cast<int>(std::clamp<std::int64_t>(fft_elems() / h, 1, std::min<std::int64_t>(64, w)));
    const dim3 gc(static_cast<unsigned>((w + ncc - 1) / ncc), static_cast<unsigned>(count));
    const std::size_t smc = static_cast<std::size_t>(h * ncc) * sizeof(double2);
    const unsigned tc = static_cast<unsigned>(ncc * h / 8);
    if (adjoint)
      k_center_fft_cols<+1><<<gc, tc, smc, stream_>>>(out, out, static_cast<int>(w), lh, ncc, sh, t.h_tw.get());
    else
      k_center_fft_cols<-1><<<gc, tc, smc, stream_>>>(out, out, static_cast<int>(w), lh, ncc, sh, t.h_tw.get());
    MLRG_LAUNCH_CHECK("k_center_fft_cols");
    return;
  }
  t.f2d_tmp.resize(static_cast<std::size_t>(count * h * w));
  const int blocks = 4 * sm_count();
  // along w: treat as [count*h][w][1]; along h: [count][h][w]
  k_dense_dft<<<blocks, 256, 0, stream_>>>(p, t.f2d_tmp.get(), count * h, static_cast<int>(w), 1,
                                           adjoint ? t.Wwc.get() : t.Ww.get());
  MLRG_LAUNCH_CHECK("k_dense_dft");
  k_dense_dft<<<blocks, 256, 0, stream_>>>(t.f2d_tmp.get(), out, count, static_cast<int>(h), static_cast<int>(w),
                                           adjoint ? t.Whc.get() : t.Wh.get());
  MLRG_LAUNCH_CHECK("k_dense_dft");
}

}  // namespace mlrg
