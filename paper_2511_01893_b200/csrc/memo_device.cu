// Memo-layer kernels: the projection encoder as one split-K skinny GEMM per
// operator call (every slab of the call shares the Gaussian matrix P, so P is
// streamed from HBM once per call), and the slab copy kernels that
// materialise hits and capture miss values (scalerun.cpp:86-105, 250-283).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "device.hpp"
#include "kernels.hpp"
#include "memo_gpu.hpp"

namespace mlrg::ops {

namespace {

constexpr int kMaxSlabs = 64;
constexpr int kRows = 64;    // key rows padded (key_dim <= 64)

struct SlabList {
  long long start[kMaxSlabs];
};

// Split-K skinny GEMM keys[s][r] = sum_k P[r][k] X[s][k] over K = 2n for up
// to 16 slabs per launch, with P in the reference's row layout but interleaved
// columns (column 2i weights Re x_i, 2i+1 weights Im x_i; the reference's row
// is [re block | im block], encoder.cpp:414-419). The GEMM is HBM-bound on
// streaming P (60 x 2n floats) once per call.
//
// Every warp owns 32-column chunks of K (grid-stride over warps) and stages
// them in warp-private double-buffered shared memory: P by cp.async (60 rows x
// 128 B), x through registers (converted to float once). Lane (sg, rg) holds a
// 4-slab x 8-row register tile (rows rg, rg+8, ..., rg+56): per pair of K
// columns 2 LDS.128 (x) + 8 LDS.64 (P) feed 64 FMAs. Products are summed in
// float within a chunk and in double across chunks (the reference accumulates
// in double, encoder.cpp:416-420); slot kd of each slab carries sum |x|^2.
#ifndef MLRG_ENC_MINB
#define MLRG_ENC_MINB 2
#endif
constexpr int kEncWarps = 4;
#ifndef MLRG_TC_FLUSH
#define MLRG_TC_FLUSH 2
#endif
constexpr int kTcFlush = MLRG_TC_FLUSH;  // chunks (of 32 columns) summed in fp32 before the double add
constexpr int kPStride = 36;  // floats per staged P row: 16 B aligned, conflict-free LDS.64 across rg
constexpr int kXStride = 34;  // floats per staged slab row: conflict-free STS.64 / LDS.64
struct EncStage {
  float x[16][kXStride];     // [slab][column kk]
  float p[kRows][kPStride];  // [row][column kk]
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}

// TC: the chunk products run on the tensor cores (mma.sync m16n8k8 TF32 with the
// 3xTF32 split a = a_hi + a_lo, products a_hi b_hi + a_hi b_lo + a_lo b_hi, ~2^-21
// relative per product, fp32 accumulation within the 32-column chunk like the
// FFMA path), which removes the FMA/shared-load issue limit of the skinny GEMM.
__device__ __forceinline__ void tf32_split(float v, unsigned& hi, unsigned& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(v));
  const float r = v - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <class TX, bool TC>
__global__ void __launch_bounds__(kEncWarps * 32, MLRG_ENC_MINB) k_encode(const TX* __restrict__ x, SlabGeom g, SlabList sl, int ns,
                                                           const float* __restrict__ P, long long n, int kd,
                                                           bool p_vec, double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char enc_smem[];
  EncStage(*stage)[2] = reinterpret_cast<EncStage(*)[2]>(enc_smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sg = lane >> 3, rg = lane & 7;
  EncStage* st = stage[warp];
  // rows >= kd stay zero in both buffers
  for (int e = lane; e < 2 * (kRows - kd) * kPStride; e += 32) {
    const int b = e / ((kRows - kd) * kPStride), r = e % ((kRows - kd) * kPStride);
    st[b].p[kd + r / kPStride][r % kPStride] = 0.f;
  }
  const long long K = 2 * n;
  const long long nchunks = (K + 31) / 32;
  const long long gw = static_cast<long long>(blockIdx.x) * kEncWarps + warp;
  const long long W = static_cast<long long>(gridDim.x) * kEncWarps;
  // x staging: lane owns complex element e = lane & 15 of slabs (lane >> 4) + 2j
  const int xe = lane & 15, xs0 = lane >> 4;
  float2 xr[8];
  // element ce of slab `start` sits at base(ce) + start * smul: axis 0 slabs
  // are contiguous; axis 1 slabs are runs of extent * d2 (32-bit division: slab
  // sizes stay below 2^31), decomposed once per chunk for all the lane's slabs
  const unsigned per = static_cast<unsigned>(g.extent * g.d2), d2 = static_cast<unsigned>(g.d2);
  const long long smul = g.axis == 0 ? g.d1 * g.d2 : g.d2;
  auto load_x = [&](long long ch) {
    const long long ce = ch * 16 + xe;
    long long base = ce;
    if (g.axis != 0) {
      const unsigned c = static_cast<unsigned>(ce), i = c / per, rem = c - i * per, kl = rem / d2;
      base = (static_cast<long long>(i) * g.d1 + kl) * g.d2 + (rem - kl * d2);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int sidx = xs0 + 2 * j;
      xr[j] = make_float2(0.f, 0.f);
      if (sidx < ns && ce < n) {
        const TX v = x[base + sl.start[sidx] * smul];
        xr[j] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
      }
    }
  };
  auto store_x = [&](EncStage& b) {  // (re, im) of element xe = columns (2 xe, 2 xe + 1)
#pragma unroll
    for (int j = 0; j < 8; ++j) *reinterpret_cast<float2*>(&b.x[xs0 + 2 * j][2 * xe]) = xr[j];
  };
  auto load_p = [&](EncStage& b, long long ch) {
    const long long k0 = ch * 32;
    if (p_vec) {  // 8 x 16 B per row: lane (r0, q) copies columns 4q.. of rows r0, r0 + 4, ...
      const int q = lane & 7;
      const long long k = k0 + 4 * q;
      const int bytes = k >= K ? 0 : static_cast<int>(min(16LL, (K - k) * 4));
      const float* src = P + (bytes ? k : 0);
      for (int r = lane >> 3; r < kd; r += 4)
        cp_async16z(&b.p[r][4 * q], src + (bytes ? static_cast<long long>(r) * K : 0), bytes);
    } else {
      const long long k = k0 + lane;
      const int bytes = k < K ? 4 : 0;
      for (int r = 0; r < kd; ++r) cp_async4(&b.p[r][lane], P + (bytes ? static_cast<long long>(r) * K + k : 0), bytes);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  // FFMA path: lane (sg, rg) owns slabs 4 sg + a x rows 8 i + rg; TC path: lane
  // (gq, tq) owns the mma C fragments, rows 16 mt + gq (+8) x slabs 8 nt + 2 tq (+1)
  double acc[4][8], nrm[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    nrm[a] = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[a][i] = 0.0;
  }
  const int gq = lane >> 2, tq = lane & 3;
  float tc_c[4][2][4], tc_fn[2] = {0.f, 0.f};  // TC: fp32 chunk-group partials
  int tc_n = 0;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) tc_c[mt][nt][i] = 0.f;
  int buf = 0;
  if (gw < nchunks) {
    load_p(st[0], gw);
    load_x(gw);
    store_x(st[0]);
  }
  for (long long ch = gw; ch < nchunks; ch += W) {
    const bool more = ch + W < nchunks;
    if (more) {
      load_p(st[buf ^ 1], ch + W);
      load_x(ch + W);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncwarp();
    const EncStage& b = st[buf];
    if constexpr (TC) {
      auto& c = tc_c;
      auto& fn = tc_fn;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int k0 = 8 * ks;
        unsigned bh[2][2], bl[2][2];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const float b0 = b.x[8 * nt + gq][k0 + tq], b1 = b.x[8 * nt + gq][k0 + tq + 4];
          fn[nt] = fmaf(b1, b1, fmaf(b0, b0, fn[nt]));
          tf32_split(b0, bh[nt][0], bl[nt][0]);
          tf32_split(b1, bh[nt][1], bl[nt][1]);
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const float av[4] = {b.p[16 * mt + gq][k0 + tq], b.p[16 * mt + gq + 8][k0 + tq],
                               b.p[16 * mt + gq][k0 + tq + 4], b.p[16 * mt + gq + 8][k0 + tq + 4]};
          unsigned ah[4], al[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) tf32_split(av[i], ah[i], al[i]);
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            mma_tf32(c[mt][nt], al, bh[nt]);
            mma_tf32(c[mt][nt], ah, bl[nt]);
            mma_tf32(c[mt][nt], ah, bh[nt]);
          }
        }
      }
      // fp32 over kTcFlush chunks, then double
      if (++tc_n == kTcFlush || !more) {
        tc_n = 0;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              acc[mt][nt * 4 + i] += c[mt][nt][i];
              c[mt][nt][i] = 0.f;
            }
        nrm[0] += fn[0];
        nrm[1] += fn[1];
        fn[0] = fn[1] = 0.f;
      }
    } else {
      float fa[4][8], fn[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        fn[a] = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) fa[a][i] = 0.f;
      }
#pragma unroll 4
      for (int kk = 0; kk < 32; kk += 2) {
        float xa0[4], xa1[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const float2 xv = *reinterpret_cast<const float2*>(&b.x[4 * sg + a][kk]);
          xa0[a] = xv.x;
          xa1[a] = xv.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 pv = *reinterpret_cast<const float2*>(&b.p[8 * i + rg][kk]);
#pragma unroll
          for (int a = 0; a < 4; ++a) fa[a][i] = fmaf(pv.y, xa1[a], fmaf(pv.x, xa0[a], fa[a][i]));
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) fn[a] = fmaf(xa1[a], xa1[a], fmaf(xa0[a], xa0[a], fn[a]));
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        nrm[a] += fn[a];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[a][i] += fa[a][i];
      }
    }
    __syncwarp();
    if (more) store_x(st[buf ^ 1]);
    buf ^= 1;
  }
  // CTA reduction over warps (fixed order) into the partial tile [block][slab][kd + 1]
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  double* red = reinterpret_cast<double*>(enc_smem);  // [warp][16][kRows + 1]
  constexpr int kRS = kRows + 1;
  if constexpr (TC) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = 16 * mt + gq + (i >= 2 ? 8 : 0), slab = 8 * nt + 2 * tq + (i & 1);
          red[(warp * 16 + slab) * kRS + row] = acc[mt][nt * 4 + i];
        }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {  // |x|^2: the 4 lanes of a quad hold one slab's columns
      double v = nrm[nt];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      if (tq == 0) red[(warp * 16 + 8 * nt + gq) * kRS + kRows] = v;
    }
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
      for (int i = 0; i < 8; ++i) red[(warp * 16 + 4 * sg + a) * kRS + 8 * i + rg] = acc[a][i];
      if (rg == 0) red[(warp * 16 + 4 * sg + a) * kRS + kRows] = nrm[a];
    }
  }
  __syncthreads();
  double* pb = part + static_cast<long long>(blockIdx.x) * ns * (kd + 1);
  for (int e = threadIdx.x; e < ns * (kd + 1); e += blockDim.x) {
    const int slab = e / (kd + 1), r = e - slab * (kd + 1);
    const int col = r < kd ? r : kRows;
    double v = 0.0;
    for (int w = 0; w < kEncWarps; ++w) v += red[(w * 16 + slab) * kRS + col];
    pb[e] = v;
  }
}

// One warp per output value: lanes stride over the CTA partials, then a fixed
// shuffle tree (deterministic).
__global__ void k_encode_reduce(const double* __restrict__ part, int nblocks, int ns, int kd,
                                float* __restrict__ keys, double* __restrict__ norms2) {
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int per = ns * (kd + 1);
  if (e >= per) return;
  double s = 0.0;
  for (int b = lane; b < nblocks; b += 32) s += part[static_cast<long long>(b) * per + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane != 0) return;
  const int slab = e / (kd + 1), r = e - slab * (kd + 1);
  if (r < kd) keys[slab * kd + r] = static_cast<float>(s);
  else norms2[slab] = s;
}

// Slab copies between full arrays and the value arena, batched: blockIdx.y
// selects the slab of the list, blockIdx.x strides over its elements.
// A slab is `runs` contiguous runs of `run_len` elements in the full array
// (axis 0: extent planes; axis 1: one run of extent*d2 per index of axis 0),
// stored back to back in the value.
constexpr long long kSeg = 4096;  // elements per block iteration
struct SlabRuns {
  long long runs, run_len, first, stride;  // run r starts at first + r * stride
};
__device__ __forceinline__ SlabRuns slab_runs(const SlabGeom& g, long long start, long long extent) {
  if (g.axis == 0) return {extent, g.d1 * g.d2, start * g.d1 * g.d2, g.d1 * g.d2};
  return {g.d0, extent * g.d2, start * g.d2, g.d1 * g.d2};
}

// Slab copies between full arrays and the value arena, batched: blockIdx.y
// selects the slab of the list; warps stride over (run, element) pairs.
template <class TO>
__global__ void __launch_bounds__(256) k_slab_materialize(TO* __restrict__ out, SlabGeom g, SlabBatch b,
                                                          const float2* __restrict__ sub) {
  const int q = blockIdx.y;
  const SlabRuns sr = slab_runs(g, b.start[q], b.extent[q]);
  const float2* __restrict__ value = b.value[q];
  const double scale = b.scale[q];
  const long long segs = (sr.run_len + kSeg - 1) / kSeg;
  for (long long t = blockIdx.x; t < sr.runs * segs; t += gridDim.x) {
    const long long r = t / segs, e0 = (t - r * segs) * kSeg;
    const long long o0 = sr.first + r * sr.stride, v0 = r * sr.run_len;
    const long long e1 = min(sr.run_len, e0 + kSeg);
    for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const long long o = o0 + e;
      const float2 v = value[v0 + e];
      double re = v.x * scale, im = v.y * scale;
      if (sub) {
        const float2 sv = sub[o];
        re -= sv.x;
        im -= sv.y;
      }
      TO res;
      res.x = static_cast<decltype(res.x)>(re);
      res.y = static_cast<decltype(res.y)>(im);
      out[o] = res;
    }
  }
}

// value = out[slab] and, when `sub` is set, out[slab] -= sub[slab] afterwards
// (the fused op stores the linear part and keeps out = fu2d(v) - d_hat).
template <class TO>
__global__ void __launch_bounds__(256) k_slab_store(TO* __restrict__ out, SlabGeom g, SlabBatch b,
                                                    const float2* __restrict__ sub) {
  const int q = blockIdx.y;
  const SlabRuns sr = slab_runs(g, b.start[q], b.extent[q]);
  float2* __restrict__ value = b.dst[q];
  const long long segs = (sr.run_len + kSeg - 1) / kSeg;
  for (long long t = blockIdx.x; t < sr.runs * segs; t += gridDim.x) {
    const long long r = t / segs, e0 = (t - r * segs) * kSeg;
    const long long o0 = sr.first + r * sr.stride, v0 = r * sr.run_len;
    const long long e1 = min(sr.run_len, e0 + kSeg);
    for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const long long o = o0 + e;
      const TO v = out[o];
      if (value) value[v0 + e] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
      if constexpr (sizeof(TO) == sizeof(float2)) {
        if (sub) out[o] = csub(v, sub[o]);
      }
    }
  }
}

__device__ __forceinline__ long long slab_len(const SlabGeom& g) { return g.axis == 0 ? g.d0 : g.d1; }

// Each thread moves kPer elements of a kSeg segment in groups of kInFlight:
// the group's loads first, then its arithmetic and stores.
constexpr int kCopyThreads = 256;
constexpr int kPer = static_cast<int>(kSeg) / kCopyThreads;
constexpr int kInFlight = 4;

// hit slab: its value (x scale, - sub) into the output
template <class TO>
__device__ __forceinline__ void dev_materialize_slab(TO* __restrict__ out, SlabGeom g, const DevSlab& d,
                                                     long long chunk, const float2* __restrict__ sub) {
  const long long start = blockIdx.y * chunk;
  const SlabRuns sr = slab_runs(g, start, min(chunk, slab_len(g) - start));
  const float2* __restrict__ value = d.src;
  const long long segs = (sr.run_len + kSeg - 1) / kSeg;
  for (long long t = blockIdx.x; t < sr.runs * segs; t += gridDim.x) {
    const long long r = t / segs, e0 = (t - r * segs) * kSeg;
    const long long o0 = sr.first + r * sr.stride + e0, v0 = r * sr.run_len + e0;
    const int cnt = static_cast<int>(min(kSeg, sr.run_len - e0));
    for (int i0 = 0; i0 < kPer; i0 += kInFlight) {
      float2 v[kInFlight], sv[kInFlight];
#pragma unroll
      for (int i = 0; i < kInFlight; ++i) {
        const int e = (i0 + i) * kCopyThreads + threadIdx.x;
        v[i] = e < cnt ? value[v0 + e] : make_float2(0.f, 0.f);
        sv[i] = sub && e < cnt ? sub[o0 + e] : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < kInFlight; ++i) {
        const int e = (i0 + i) * kCopyThreads + threadIdx.x;
        if (e >= cnt) continue;
        double re = v[i].x * d.scale, im = v[i].y * d.scale;
        if (sub) {
          re -= sv[i].x;
          im -= sv[i].y;
        }
        TO res;
        res.x = static_cast<decltype(res.x)>(re);
        res.y = static_cast<decltype(res.y)>(im);
        out[o0 + e] = res;
      }
    }
  }
}

// miss slab: the computed output into its arena slot (complex64), then - sub
template <class TO>
__device__ __forceinline__ void dev_store_slab(TO* __restrict__ out, SlabGeom g, const DevSlab& d, long long chunk,
                                               const float2* __restrict__ sub) {
  const long long start = blockIdx.y * chunk;
  const SlabRuns sr = slab_runs(g, start, min(chunk, slab_len(g) - start));
  float2* __restrict__ value = d.dst;
  if (!value && !sub) return;
  const long long segs = (sr.run_len + kSeg - 1) / kSeg;
  for (long long t = blockIdx.x; t < sr.runs * segs; t += gridDim.x) {
    const long long r = t / segs, e0 = (t - r * segs) * kSeg;
    const long long o0 = sr.first + r * sr.stride + e0, v0 = r * sr.run_len + e0;
    const int cnt = static_cast<int>(min(kSeg, sr.run_len - e0));
    for (int i0 = 0; i0 < kPer; i0 += kInFlight) {
      TO v[kInFlight];
#pragma unroll
      for (int i = 0; i < kInFlight; ++i) {
        const int e = (i0 + i) * kCopyThreads + threadIdx.x;
        if (e < cnt) v[i] = out[o0 + e];
      }
#pragma unroll
      for (int i = 0; i < kInFlight; ++i) {
        const int e = (i0 + i) * kCopyThreads + threadIdx.x;
        if (e >= cnt) continue;
        if (value) value[v0 + e] = make_float2(static_cast<float>(v[i].x), static_cast<float>(v[i].y));
        if constexpr (sizeof(TO) == sizeof(float2)) {
          if (sub) out[o0 + e] = csub(v[i], sub[o0 + e]);
        }
      }
    }
  }
}

// One launch per memoized call finishes every slab: hits are materialized,
// accepted misses stored into the value arena (one grid, so the hit and miss
// slabs' copies share the waves instead of running as two launches).
template <class TO>
__global__ void __launch_bounds__(kCopyThreads, 4) k_dev_finish(TO* __restrict__ out, SlabGeom g,
                                                                const DevSlab* __restrict__ slabs, long long chunk,
                                                                const float2* __restrict__ sub) {
  const DevSlab d = slabs[blockIdx.y];
  if (d.outcome != 0) dev_materialize_slab(out, g, d, chunk, sub);
  else dev_store_slab(out, g, d, chunk, sub);
}

int enc_blocks() { return 2 * sm_count(); }
constexpr int kEncSlabs = 16;  // slabs per launch (one 4 x 8 register tile per lane)

}  // namespace

std::size_t encode_work_doubles(int ns, int kd) {
  return static_cast<std::size_t>(enc_blocks()) * static_cast<std::size_t>(std::min(ns, kEncSlabs)) *
         static_cast<std::size_t>(kd + 1);
}

namespace {
template <class TX>
void encode_impl(const TX* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
                 double* work, float* keys, double* norms2, cudaStream_t s) {
  if (kd > kRows - 1) throw std::invalid_argument("encode: key_dim must be < 64");
  const long long n = shape.count();
  constexpr std::size_t smem = sizeof(EncStage) * 2 * kEncWarps;
  static_assert(smem >= sizeof(double) * kEncWarps * 16 * (kRows + 1), "reduction scratch must fit");
  static bool attr = false;
  if (!attr) {
    MLRG_CUDA(cudaFuncSetAttribute(k_encode<float2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    MLRG_CUDA(cudaFuncSetAttribute(k_encode<double2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    MLRG_CUDA(cudaFuncSetAttribute(k_encode<float2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    MLRG_CUDA(cudaFuncSetAttribute(k_encode<double2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const bool p_vec = (2 * n) % 4 == 0 && reinterpret_cast<std::uintptr_t>(P) % 16 == 0;
  for (int b = 0; b < ns; b += kEncSlabs) {
    const int nb = std::min(kEncSlabs, ns - b);
    SlabList sl{};
    for (int q = 0; q < nb; ++q) sl.start[q] = starts[b + q];
    int blocks = enc_blocks();
    prof::begin("k_encode", s);
    // MLRG_ENCODE_TC: unset / "tcgen05" = the tcgen05 kernel where supported, "mma" = the
    // mma.sync TF32 kernel, "0" = the FFMA path
    static const int mode = [] {
      const char* e = std::getenv("MLRG_ENCODE_TC");
      if (e && *e == '0') return 0;
      if (e && std::string(e) == "mma") return 1;
      return 2;
    }();
    if (mode == 2 && encode_tc_supported(shape, P, kd, nb)) {
      blocks = encode_tc_grid();
      encode_tc(x, shape, starts + b, nb, P, kd, work, s);
    } else if (mode >= 1) {
      k_encode<TX, true><<<blocks, kEncWarps * 32, smem, s>>>(x, shape, sl, nb, P, n, kd, p_vec, work);
    } else {
      k_encode<TX, false><<<blocks, kEncWarps * 32, smem, s>>>(x, shape, sl, nb, P, n, kd, p_vec, work);
    }
    MLRG_LAUNCH_CHECK("k_encode");
    prof::end("k_encode", s);
    const int per = nb * (kd + 1);
    prof::begin("k_encode_reduce", s);
    k_encode_reduce<<<(per * 32 + 255) / 256, 256, 0, s>>>(work, blocks, nb, kd, keys + b * kd, norms2 + b);
    prof::end("k_encode_reduce", s);
    MLRG_LAUNCH_CHECK("k_encode_reduce");
  }
}
}  // namespace

void encode(const float2* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
            double* work, float* keys, double* norms2, cudaStream_t s) {
  encode_impl(x, shape, starts, ns, P, kd, work, keys, norms2, s);
}

void encode(const double2* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
            double* work, float* keys, double* norms2, cudaStream_t s) {
  encode_impl(x, shape, starts, ns, P, kd, work, keys, norms2, s);
}

namespace {
dim3 batch_grid(int nb) {
  return dim3(static_cast<unsigned>(std::max(1, 8 * sm_count() / std::max(nb, 1))), static_cast<unsigned>(nb));
}
template <class TO>
void materialize_impl(TO* out, SlabGeom g, const SlabBatch& b, int nb, const float2* sub, cudaStream_t s) {
  if (nb <= 0) return;
  if (nb > kSlabBatch) throw std::logic_error("slab batch too large");
  k_slab_materialize<TO><<<batch_grid(nb), 256, 0, s>>>(out, g, b, sub);
  MLRG_LAUNCH_CHECK("k_slab_materialize");
}
template <class TO>
void store_impl(TO* out, SlabGeom g, const SlabBatch& b, int nb, const float2* sub, cudaStream_t s) {
  if (nb <= 0) return;
  if (nb > kSlabBatch) throw std::logic_error("slab batch too large");
  k_slab_store<TO><<<batch_grid(nb), 256, 0, s>>>(out, g, b, sub);
  MLRG_LAUNCH_CHECK("k_slab_store");
}
}  // namespace

void dev_finish(float2* out, SlabGeom g, const DevSlab* slabs, int n, std::int64_t chunk, const float2* sub,
                cudaStream_t s) {
  if (n <= 0) return;
  prof::begin("k_dev_finish", s);
  k_dev_finish<float2><<<batch_grid(n), kCopyThreads, 0, s>>>(out, g, slabs, chunk, sub);
  prof::end("k_dev_finish", s);
  MLRG_LAUNCH_CHECK("k_dev_finish");
}
void dev_finish(double2* out, SlabGeom g, const DevSlab* slabs, int n, std::int64_t chunk, cudaStream_t s) {
  if (n <= 0) return;
  prof::begin("k_dev_finish", s);
  k_dev_finish<double2><<<batch_grid(n), kCopyThreads, 0, s>>>(out, g, slabs, chunk, nullptr);
  prof::end("k_dev_finish", s);
  MLRG_LAUNCH_CHECK("k_dev_finish");
}

void slab_materialize(float2* out, SlabGeom g, const SlabBatch& b, int nb, const float2* sub, cudaStream_t s) {
  materialize_impl(out, g, b, nb, sub, s);
}
void slab_materialize(double2* out, SlabGeom g, const SlabBatch& b, int nb, cudaStream_t s) {
  materialize_impl(out, g, b, nb, static_cast<const float2*>(nullptr), s);
}
void slab_store(float2* out, SlabGeom g, const SlabBatch& b, int nb, const float2* sub, cudaStream_t s) {
  store_impl(out, g, b, nb, sub, s);
}
void slab_store(double2* out, SlabGeom g, const SlabBatch& b, int nb, cudaStream_t s) {
  store_impl(out, g, b, nb, static_cast<const float2*>(nullptr), s);
}

}  // namespace mlrg::ops
