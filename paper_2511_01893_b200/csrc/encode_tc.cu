// Projection-encoder keys on the 5th-generation tensor cores (tcgen05 + TMEM,
// P staged by TMA): keys[s][r] = sum_k P[r][k] X[s][k] (encoder.cpp:405-422,
// P in the interleaved (re, im) column order of encoder.hpp), split-K over one
// persistent CTA per SM.
//
// The GEMM is M = 60 key rows x N = 16 slabs x K = 2n (n complex elements per
// slab), HBM-bound on streaming P (60 x 2n floats, 503 MB per call at 256^3)
// once per operator call. Precision follows the reference's double
// accumulation closely enough that the memo decisions (cosine > tau) are the
// reference's: every product runs as a two-term TF32 split and every 128
// columns of fp32 tensor-core sums are added into double registers.
//
//   * A producer warp stages each 128-column step: the raw fp32 P tile (128
//     columns x 64 rows; rows >= kd are the box's zero fill) by TMA
//     (cp.async.bulk.tensor, SWIZZLE_128B), and every slab's 64 complex
//     elements of the step by cp.async, both completing on one mbarrier, 4
//     steps deep (3 for complex128 input).
//   * Eight converter warps split each P element into hi = P with the low 13
//     mantissa bits cleared (exact TF32) and lo = P - hi and write them to
//     TMEM as the MMA's A operand, stacked: rows 0..63 = P_hi, 64..127 = P_lo
//     (tcgen05.st; warp w owns TMEM lanes 32 (w % 4) ..). They split the slab
//     columns the same way into a K-major B operand [X_hi; X_lo] (canonical
//     no-swizzle core-matrix layout in shared memory) and keep sum |x|^2.
//   * One thread issues, per 8 columns, D += [P_hi; P_lo] [X_hi; X_lo]^T
//     (tcgen05.mma kind::tf32, M = 128, N = 32, A from TMEM): D row r holds
//     P_hi X_hi | P_hi X_lo and row r + 64 P_lo X_hi | P_lo X_lo. Even and odd
//     8-column steps accumulate into two D tiles; D is double-buffered.
//   * Four of the converter warps read each step's D (tcgen05.ld) into double
//     accumulators two steps later (fp32 over 128 columns, double across
//     steps, as the reference accumulates in double), and at the end add rows
//     r and r + 64 and write the CTA's [slab][kd + 1] partial tile
//     (k_encode_reduce sums the CTAs in a fixed order).
//
// Measured (256^3, 16 slabs of 16 x 256 x 256, complex64): 140 us per call
// vs 151 us for the mma.sync kernel (637 MB: 4.6 TB/s). The step period is set
// by the tensor core: 16 M128 x N32 x K8 tf32 MMAs take ~1.3K cycles (~80
// cycles each at this small N), the converters ~1.1K cycles per step.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <map>
#include <mutex>
#include <stdexcept>
#include <tuple>

#include "device.hpp"
#include "kernels.hpp"

namespace mlrg::ops {

namespace {

constexpr int kStageCols = 128;                 // P / X columns per pipeline stage
constexpr int kBoxCols = 32;                    // TMA box width (128 B, one swizzle atom row)
constexpr int kBoxes = kStageCols / kBoxCols;   // TMA loads per stage
constexpr int kPRows = 64;                      // TMA box height (key rows, zero-filled past kd)
constexpr int kBoxBytes = kBoxCols * kPRows * 4;
constexpr int kPBytes = kBoxes * kBoxBytes;   // 32 KB of raw P per stage
constexpr int kSlabs = 16;                      // MMA N
constexpr int kBRows = 2 * kSlabs;              // B = [X_hi; X_lo] stacked along N: MMA N = 32
constexpr int kBBytes = kStageCols * kBRows * 4;  // one B operand per buffer: 16 KB
constexpr int kConvWarps = 8;
constexpr int kThreads = (kConvWarps + 2) * 32;  // + TMA producer warp + MMA warp
constexpr int kTmemCols = 512;
constexpr int kDCol = 0;     // D[b][chain] at columns 64 b + 32 chain
constexpr int kACol = 128;   // A[b] at columns 128 + 128 b
constexpr int kSmemB = 2 * kBBytes;
constexpr int kSmemTail = 256 + (64 + 16) * kSlabs * 8;  // barriers + reduction scratch

// Per element type: a stage is the raw P tile plus each slab's 64 complex
// elements of the stage (one bulk copy per slab, rows padded by 16 B so the
// converters' reads are conflict-free), 1 KB aligned for the swizzled P boxes.
template <class TX>
struct StageCfg {
  static constexpr int kXBytes = (kStageCols / 2) * static_cast<int>(sizeof(TX));
  static constexpr int kXStride = kXBytes + 16;
  static constexpr int kBytes = (kPBytes + kSlabs * kXStride + 1023) / 1024 * 1024;
  static constexpr int kStages = sizeof(TX) == 8 ? 4 : 3;
  static constexpr int kSmem = kStages * kBytes + kSmemB + 1024 + kSmemTail;
};
static_assert(StageCfg<float2>::kSmem <= 227 * 1024 && StageCfg<double2>::kSmem <= 227 * 1024, "stage ring fits");

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// K-major, no-swizzle shared-memory matrix descriptor: core matrices of 8 rows
// x 16 B; LBO = byte distance between the two K-adjacent core matrices of one
// MMA, SBO = between 8-row groups (tcgen05 descriptor version 1).
__device__ __forceinline__ std::uint64_t smem_desc(unsigned addr, unsigned lbo, unsigned sbo) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((addr >> 4) & 0x3FFFu);
  d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<std::uint64_t>(1) << 46;
  return d;
}
// kind::tf32 instruction descriptor: F32 accumulator, TF32 A and B, both
// K-major, N = 32, M = 128.
constexpr std::uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kBRows >> 3) << 17) | ((128 >> 4) << 24);

__device__ __forceinline__ void mma_tf32_ts(unsigned d_tmem, unsigned a_tmem, std::uint64_t b_desc, unsigned acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(kIdesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}
__device__ __forceinline__ void mma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}

__device__ __forceinline__ unsigned tf32_hi(unsigned bits) { return bits & 0xFFFFE000u; }

// 32 consecutive TMEM columns of this warp's lanes <- 32 registers per thread
__device__ __forceinline__ void tmem_st32(unsigned taddr, const unsigned (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(unsigned taddr, float (&v)[32]) {
  unsigned r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

struct TcSlabs {
  long long start[kSlabs];
};

// Launch requirement (encode_tc_supported): every slab's 64-element stage
// chunk is one contiguous run of the input (axis-0 slabs always; axis-1 slabs
// when extent * d2 is a multiple of 64 and d2 is even) and n is a multiple of 64.
//
// Warps: 0..7 converters (warp w: TMEM lanes 32 (w % 4) .., TMA boxes 2 (w / 4)
// and 2 (w / 4) + 1 of each stage; warps 0..3 also run the D epilogue),
// 8 = producer (lane 0: the P boxes by TMA; all lanes: the X chunks by
// cp.async, tracked by the same mbarrier), 9 = MMA issuer + TMEM owner.
template <class TX>
__global__ void __launch_bounds__(kThreads, 1)
    k_encode_tc(const __grid_constant__ CUtensorMap pmap, const TX* __restrict__ x, SlabGeom g, TcSlabs sl, int ns,
                long long n, int kd, int nstages, double* __restrict__ part) {
  using C = StageCfg<TX>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  unsigned char* ring = smem;                          // [stage]{P boxes (swizzled) | X rows [slab][kXStride]}
  unsigned char* bop = smem + C::kStages * C::kBytes;  // [buf][kq][32 rows: X_hi 0..15, X_lo 16..31][16 B]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(bop + kSmemB);
  unsigned long long* tma_full = bars;                  // [kStages]
  unsigned long long* raw_free = bars + C::kStages;     // [kStages]
  unsigned long long* a_ready = bars + 2 * C::kStages;  // [2]
  unsigned long long* mma_done = a_ready + 2;           // [2]
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(mma_done + 2);
  double* red = reinterpret_cast<double*>(bop + kSmemB + 256);  // [64][16] + norms [16][16]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA's stages blockIdx.x + k gridDim.x: at any moment the CTAs stream
  // neighbouring column ranges of every P row (DRAM page locality)
  const int nst = (nstages - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x);
  auto stage_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x); };
  constexpr int kConv = kConvWarps * 32;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&tma_full[i], 1);
      mbar_init(&raw_free[i], kConv);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_ready[i], kConv);
      mbar_init(&mma_done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == kConvWarps + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const unsigned tmem = *tmem_slot;

  if (warp == kConvWarps) {
    // ---------------- producer ----------------
    if (lane == 0) asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&pmap)) : "memory");
    constexpr int kPieces = C::kXBytes / 16;  // 16 B pieces per slab chunk (32 or 64)
    for (int k = 0; k < nst; ++k) {
      const int st = k % C::kStages, use = k / C::kStages;
      if (use > 0) mbar_wait(&raw_free[st], (use - 1) & 1);
      unsigned char* sp = ring + st * C::kBytes;
      const int col0 = stage_of(k) * kStageCols;
      // X: every slab's chunk starts at the same in-slab element ce (one division per stage)
      const long long ce = static_cast<long long>(col0) >> 1;
      long long rel = ce, smul = g.d1 * g.d2;
      if (g.axis != 0) {
        const long long per = g.extent * g.d2, i = ce / per;
        rel = i * g.d1 * g.d2 + (ce - i * per);
        smul = g.d2;
      }
      for (int q = 0; q < ns; ++q) {
        const unsigned char* src = reinterpret_cast<const unsigned char*>(x + (sl.start[q] * smul + rel));
#pragma unroll
        for (int j = lane; j < kPieces; j += 32) {
          const unsigned dst = su32(sp + kPBytes + q * C::kXStride + j * 16);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + j * 16) : "memory");
        }
      }
      // the barrier tracks this lane's copies (pending count +1 now, -1 when they land)
      asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(su32(&tma_full[st])) : "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_expect_tx(&tma_full[st], static_cast<unsigned>(kPBytes));
        for (int q = 0; q < kBoxes; ++q) tma_load_2d(sp + q * kBoxBytes, &pmap, col0 + q * kBoxCols, 0, &tma_full[st]);
      }
    }
  } else if (warp == kConvWarps + 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      for (int k = 0; k < nst; ++k) {
        const int b = k & 1;
        mbar_wait(&a_ready[b], (k >> 1) & 1);
        fence_after();
        const unsigned d = tmem + kDCol + 64 * b;
        const unsigned a0 = tmem + kACol + 128 * b;
        // K = 8 columns = two 16 B core matrices along K (LBO = 32 rows x 16 B); 8-row groups at
        // SBO = 128 B; step j starts 1 KB further (+64 in the descriptor's address field); even /
        // odd k-steps accumulate into two independent D tiles
        const std::uint64_t bdesc = smem_desc(su32(bop + b * kBBytes), 512, 128);
        mma_tf32_ts(d, a0, bdesc, 0u);
        mma_tf32_ts(d + 32, a0 + 8, bdesc + 64, 0u);
#pragma unroll
        for (int j = 2; j < kStageCols / 8; ++j) mma_tf32_ts(d + 32 * (j & 1), a0 + 8 * j, bdesc + 64 * j, 1u);
        mma_commit(&mma_done[b]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- converter / epilogue warps ----------------
    const int sub = warp & 3;                  // TMEM lanes 32 sub .. 32 sub + 31
    const int half = warp >> 2;                // boxes 2 half, 2 half + 1
    const int arow = 32 * sub + lane;          // A row = TMEM lane
    const int prow = arow & 63;                // P row it carries (hi for arow < 64, lo above)
    const bool is_lo = arow >= 64;
    const unsigned t_lane = static_cast<unsigned>(32 * sub) << 16;
    // X: this thread's slab and two K chunks (4 floats = 2 complex elements each)
    const int xs = (lane & 7) + 8 * (warp & 1);
    const int kq0 = (lane >> 3) + 4 * (warp >> 1);  // chunks kq0 + 16 i, i < 2
    const bool xs_ok = xs < ns;
    double acc[kSlabs];
#pragma unroll
    for (int i = 0; i < kSlabs; ++i) acc[i] = 0.0;
    double nrm = 0.0;
    auto epilogue = [&](int k) {  // D of stage k -> double accumulators (warps 0..3)
      const int b = k & 1;
      mbar_wait(&mma_done[b], (k >> 1) & 1);
      fence_after();
      if (half) return;  // warps 4..7 only wait (A[b] / B[b] reuse)
      float v[2][32];
      tmem_ld32(tmem + t_lane + kDCol + 64 * b, v[0]);
      tmem_ld32(tmem + t_lane + kDCol + 64 * b + 32, v[1]);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < kSlabs; ++i)  // columns i (A X_hi) and 16 + i (A X_lo) of both chains
        acc[i] += static_cast<double>((v[0][i] + v[1][i]) + (v[0][kSlabs + i] + v[1][kSlabs + i]));
    };
    for (int k = 0; k < nst; ++k) {
      const int b = k & 1, st = k % C::kStages;
      if (k >= 2) epilogue(k - 2);  // also frees A[b] / B[b] (their MMAs are done)
      mbar_wait(&tma_full[st], (k / C::kStages) & 1);
      const unsigned char* sp = ring + st * C::kBytes;
      // ---- A: P rows from the swizzled TMA tile -> hi or lo -> TMEM ----
      const unsigned char* tile = sp + prow * 128;
#pragma unroll
      for (int qq = 0; qq < kBoxes / 2; ++qq) {
        const int q = 2 * half + qq;
        unsigned v[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 w = *reinterpret_cast<const uint4*>(tile + q * kBoxBytes + ((c ^ (prow & 7)) << 4));
          v[4 * c + 0] = w.x;
          v[4 * c + 1] = w.y;
          v[4 * c + 2] = w.z;
          v[4 * c + 3] = w.w;
        }
        if (is_lo) {  // warp-uniform
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) - __uint_as_float(tf32_hi(v[j])));
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = tf32_hi(v[j]);
        }
        tmem_st32(tmem + t_lane + kACol + 128 * b + 32 * q, v);
      }
      // ---- B: this stage's slab columns -> X_hi / X_lo (K-major core matrices) ----
      float4 xv[2];
      const unsigned char* xr = sp + kPBytes + xs * C::kXStride;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int kq = kq0 + 16 * i;
        if (!xs_ok) {
          xv[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else if constexpr (sizeof(TX) == 8) {
          xv[i] = *reinterpret_cast<const float4*>(xr + kq * 16);
        } else {
          const double2 a = *reinterpret_cast<const double2*>(xr + kq * 32);
          const double2 c = *reinterpret_cast<const double2*>(xr + kq * 32 + 16);
          xv[i] = make_float4(static_cast<float>(a.x), static_cast<float>(a.y), static_cast<float>(c.x),
                              static_cast<float>(c.y));
        }
      }
      mbar_arrive(&raw_free[st]);
      unsigned char* bh = bop + b * kBBytes;  // rows 0..15: X_hi, rows 16..31: X_lo
      float fn = 0.f;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float4 f = xv[i];
        fn = fmaf(f.w, f.w, fmaf(f.z, f.z, fmaf(f.y, f.y, fmaf(f.x, f.x, fn))));
        const uint4 h = make_uint4(tf32_hi(__float_as_uint(f.x)), tf32_hi(__float_as_uint(f.y)),
                                   tf32_hi(__float_as_uint(f.z)), tf32_hi(__float_as_uint(f.w)));
        const float4 l = make_float4(f.x - __uint_as_float(h.x), f.y - __uint_as_float(h.y), f.z - __uint_as_float(h.z),
                                     f.w - __uint_as_float(h.w));
        const int off = (kq0 + 16 * i) * (kBRows * 16) + xs * 16;
        *reinterpret_cast<uint4*>(bh + off) = h;
        *reinterpret_cast<float4*>(bh + off + kSlabs * 16) = l;
      }
      nrm += static_cast<double>(fn);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      fence_before();
      mbar_arrive(&a_ready[b]);
    }
    for (int k = nst > 2 ? nst - 2 : 0; k < nst; ++k) epilogue(k);
    // ---- CTA partial tile: key row r = D row r (P_hi X) + D row r + 64 (P_lo X); norms ----
    asm volatile("bar.sync 1, %0;\n" ::"n"(kConv) : "memory");
    if (is_lo && !half)
#pragma unroll
      for (int i = 0; i < kSlabs; ++i) red[prow * kSlabs + i] = acc[i];
    double* rn = red + 64 * kSlabs;  // [slab][16 contributors]
    rn[xs * 16 + (lane >> 3) + 4 * (warp >> 1)] = nrm;
    asm volatile("bar.sync 1, %0;\n" ::"n"(kConv) : "memory");
    double* pb = part + static_cast<long long>(blockIdx.x) * ns * (kd + 1);
    if (!is_lo && !half && prow < kd)
#pragma unroll
      for (int i = 0; i < kSlabs; ++i)
        if (i < ns) pb[i * (kd + 1) + prow] = acc[i] + red[prow * kSlabs + i];
    if (threadIdx.x < ns) {
      double s = 0.0;
      for (int c = 0; c < 16; ++c) s += rn[threadIdx.x * 16 + c];
      pb[threadIdx.x * (kd + 1) + kd] = s;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == kConvWarps + 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols) : "memory");
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_tiled_fn() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

// one tensor map per (P, K, kd): P is uploaded once per slab shape
const CUtensorMap& p_map(const float* P, long long K, int kd) {
  static std::mutex mx;
  static std::map<std::tuple<const float*, long long, int>, CUtensorMap> maps;
  std::lock_guard<std::mutex> lk(mx);
  auto key = std::make_tuple(P, K, kd);
  auto it = maps.find(key);
  if (it != maps.end()) return it->second;
  EncodeTiled fn = encode_tiled_fn();
  if (!fn) throw std::runtime_error("encode_tc: cuTensorMapEncodeTiled unavailable");
  CUtensorMap m{};
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(kd)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 4};
  const cuuint32_t box[2] = {kBoxCols, kPRows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(P), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("encode_tc: cuTensorMapEncodeTiled failed");
  return maps.emplace(key, m).first->second;
}

template <class TX>
void launch(const TX* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd, int grid,
            double* work, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    MLRG_CUDA(cudaFuncSetAttribute(k_encode_tc<TX>, cudaFuncAttributeMaxDynamicSharedMemorySize, StageCfg<TX>::kSmem));
    attr = true;
  }
  const long long n = shape.count();
  const long long K = 2 * n;
  TcSlabs sl{};
  for (int q = 0; q < ns; ++q) sl.start[q] = starts[q];
  const int nstages = static_cast<int>((K + kStageCols - 1) / kStageCols);
  k_encode_tc<TX><<<grid, kThreads, StageCfg<TX>::kSmem, s>>>(p_map(P, K, kd), x, shape, sl, ns, n, kd, nstages, work);
  MLRG_LAUNCH_CHECK("k_encode_tc");
}

}  // namespace

bool encode_tc_supported(SlabGeom shape, const float* P, int kd, int ns) {
  const long long n = shape.count(), K = 2 * n;
  const bool runs = shape.axis == 0 || ((shape.extent * shape.d2) % (kStageCols / 2) == 0 && shape.d2 % 2 == 0);
  return kd <= 60 && ns <= kSlabs && n % (kStageCols / 2) == 0 && runs &&
         reinterpret_cast<std::uintptr_t>(P) % 16 == 0 && K / kStageCols >= 2 * sm_count() &&
         encode_tiled_fn() != nullptr;
}
int encode_tc_grid() { return sm_count(); }

void encode_tc(const float2* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
               double* work, cudaStream_t s) {
  launch(x, shape, starts, ns, P, kd, encode_tc_grid(), work, s);
}
void encode_tc(const double2* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
               double* work, cudaStream_t s) {
  launch(x, shape, starts, ns, P, kd, encode_tc_grid(), work, s);
}

}  // namespace mlrg::ops
