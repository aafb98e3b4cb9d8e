// Memo-layer kernels: the projection encoder as one split-K skinny GEMM per
// operator call (every slab of the call shares the Gaussian matrix P, so P is
// streamed from HBM once per call), and the slab copy kernels that
// materialise hits and capture miss values (scalerun.cpp:86-105, 250-283).
#include <algorithm>

#include "common.cuh"
#include "device.hpp"
#include "kernels.hpp"

namespace mlrg::ops {

namespace {

constexpr int kEncThreads = 256;
constexpr int kChunk = 32;   // K elements per smem stage
constexpr int kMaxSlabs = 64;
constexpr int kRows = 64;    // key rows padded (key_dim <= 64)

struct SlabList {
  long long start[kMaxSlabs];
};

__device__ __forceinline__ long long slab_offset(const SlabGeom& g, long long start, long long ce) {
  if (g.axis == 0) return start * g.d1 * g.d2 + ce;
  const long long per = g.extent * g.d2;
  const long long i = ce / per;
  const long long rem = ce - i * per;
  const long long kl = rem / g.d2;
  return (i * g.d1 + start + kl) * g.d2 + (rem - kl * g.d2);
}

// Split-K GEMM keys[s][r] = sum_k P[r][k] X[s][k] over K = 2n, with P stored
// interleaved on the device (column 2i weights Re x_i, 2i+1 weights Im x_i;
// the reference's row layout is [re block | im block], encoder.cpp:414-419).
// Thread (ty, tx) owns slabs {ty + 16 q} x rows {tx + 16 p}
// (q < SG, p < 4); each CTA walks K chunks grid-stride and writes its double
// partial tile. The first row slot past kd accumulates |x|^2.
template <int SG, class TX>
__global__ void __launch_bounds__(kEncThreads) k_encode(const TX* __restrict__ x, SlabGeom g, SlabList sl, int ns,
                                                        const float* __restrict__ P, long long n, int kd,
                                                        double* __restrict__ part) {
  __shared__ float xs[kChunk][16 * SG + 1];
  __shared__ float ps[kChunk][kRows + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[SG][4];
  double nrm_acc[SG];
#pragma unroll
  for (int q = 0; q < SG; ++q) {
    nrm_acc[q] = 0.0;
#pragma unroll
    for (int p = 0; p < 4; ++p) acc[q][p] = 0.0;
  }
  const long long K = 2 * n;
  const long long nchunks = (K + kChunk - 1) / kChunk;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long k0 = ch * kChunk;
    for (int e = threadIdx.x; e < (kChunk / 2) * 16 * SG; e += blockDim.x) {
      const int s = e / (kChunk / 2), ee = e - s * (kChunk / 2);
      const long long ce = k0 / 2 + ee;
      float xr = 0.f, xi = 0.f;
      if (s < ns && ce < n) {
        const TX xv = x[slab_offset(g, sl.start[s], ce)];
        xr = static_cast<float>(xv.x);
        xi = static_cast<float>(xv.y);
      }
      xs[2 * ee][s] = xr;
      xs[2 * ee + 1][s] = xi;
    }
    for (int e = threadIdx.x; e < kChunk * kRows; e += blockDim.x) {
      const int r = e / kChunk, kk = e - r * kChunk;
      const long long k = k0 + kk;
      ps[kk][r] = (r < kd && k < K) ? P[static_cast<long long>(r) * K + k] : 0.f;
    }
    __syncthreads();
    float fa[SG][4];
    float fn[SG];
#pragma unroll
    for (int q = 0; q < SG; ++q) {
      fn[q] = 0.f;
#pragma unroll
      for (int p = 0; p < 4; ++p) fa[q][p] = 0.f;
    }
#pragma unroll 4
    for (int kk = 0; kk < kChunk; ++kk) {
      float xv[SG], pv[4];
#pragma unroll
      for (int q = 0; q < SG; ++q) xv[q] = xs[kk][ty + 16 * q];
#pragma unroll
      for (int p = 0; p < 4; ++p) pv[p] = ps[kk][tx + 16 * p];
#pragma unroll
      for (int q = 0; q < SG; ++q) {
#pragma unroll
        for (int p = 0; p < 4; ++p) fa[q][p] = fmaf(pv[p], xv[q], fa[q][p]);
        fn[q] = fmaf(xv[q], xv[q], fn[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < SG; ++q) {
      nrm_acc[q] += fn[q];
#pragma unroll
      for (int p = 0; p < 4; ++p) acc[q][p] += fa[q][p];
    }
    __syncthreads();
  }
  // partial tile layout: [block][slab][kd + 1]
  double* pb = part + static_cast<long long>(blockIdx.x) * ns * (kd + 1);
#pragma unroll
  for (int q = 0; q < SG; ++q) {
    const int s = ty + 16 * q;
    if (s >= ns) continue;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int r = tx + 16 * p;
      if (r < kd) pb[s * (kd + 1) + r] = acc[q][p];
    }
    if (tx == 0) pb[s * (kd + 1) + kd] = nrm_acc[q];
  }
}

__global__ void k_encode_reduce(const double* __restrict__ part, int nblocks, int ns, int kd,
                                float* __restrict__ keys, double* __restrict__ norms2) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int per = ns * (kd + 1);
  if (e >= per) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += part[static_cast<long long>(b) * per + e];
  const int slab = e / (kd + 1), r = e - slab * (kd + 1);
  if (r < kd) keys[slab * kd + r] = static_cast<float>(s);
  else norms2[slab] = s;
}

template <class TO>
__global__ void k_slab_materialize(TO* __restrict__ out, SlabGeom g, const float2* __restrict__ value, double scale,
                                   const float2* __restrict__ sub) {
  const long long n = g.count();
  for (long long ce = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; ce < n;
       ce += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long o = slab_offset(g, g.start, ce);
    const float2 v = value[ce];
    double re = v.x * scale, im = v.y * scale;
    if (sub) {
      re -= sub[o].x;
      im -= sub[o].y;
    }
    out[o].x = static_cast<decltype(out[o].x)>(re);
    out[o].y = static_cast<decltype(out[o].y)>(im);
  }
}

template <class TO>
__global__ void k_slab_store(const TO* __restrict__ out, SlabGeom g, float2* __restrict__ value) {
  const long long n = g.count();
  for (long long ce = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; ce < n;
       ce += static_cast<long long>(gridDim.x) * blockDim.x) {
    const TO v = out[slab_offset(g, g.start, ce)];
    value[ce] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
  }
}

__global__ void k_slab_sub(float2* __restrict__ out, SlabGeom g, const float2* __restrict__ sub) {
  const long long n = g.count();
  for (long long ce = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; ce < n;
       ce += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long o = slab_offset(g, g.start, ce);
    out[o] = csub(out[o], sub[o]);
  }
}

int enc_blocks() { return 2 * sm_count(); }

}  // namespace

std::size_t encode_work_doubles(int ns, int kd) {
  return static_cast<std::size_t>(enc_blocks()) * static_cast<std::size_t>(std::min(ns, kMaxSlabs)) *
         static_cast<std::size_t>(kd + 1);
}

namespace {
template <class TX>
void encode_impl(const TX* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
                 double* work, float* keys, double* norms2, cudaStream_t s) {
  if (kd > kRows - 1) throw std::invalid_argument("encode: key_dim must be < 64");
  const long long n = shape.count();
  for (int b = 0; b < ns; b += kMaxSlabs) {
    const int nb = std::min(kMaxSlabs, ns - b);
    SlabList sl{};
    for (int q = 0; q < nb; ++q) sl.start[q] = starts[b + q];
    const int blocks = enc_blocks();
    prof::begin("k_encode", s);
    if (nb <= 16) k_encode<1, TX><<<blocks, kEncThreads, 0, s>>>(x, shape, sl, nb, P, n, kd, work);
    else if (nb <= 32) k_encode<2, TX><<<blocks, kEncThreads, 0, s>>>(x, shape, sl, nb, P, n, kd, work);
    else k_encode<4, TX><<<blocks, kEncThreads, 0, s>>>(x, shape, sl, nb, P, n, kd, work);
    MLRG_LAUNCH_CHECK("k_encode");
    prof::end("k_encode", s);
    const int per = nb * (kd + 1);
    k_encode_reduce<<<(per + 255) / 256, 256, 0, s>>>(work, blocks, nb, kd, keys + b * kd, norms2 + b);
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

void slab_materialize(float2* out, SlabGeom g, const float2* value, double scale, const float2* sub, cudaStream_t s) {
  k_slab_materialize<float2><<<2 * sm_count(), 256, 0, s>>>(out, g, value, scale, sub);
  MLRG_LAUNCH_CHECK("k_slab_materialize");
}

void slab_materialize(double2* out, SlabGeom g, const float2* value, double scale, cudaStream_t s) {
  k_slab_materialize<double2><<<2 * sm_count(), 256, 0, s>>>(out, g, value, scale, nullptr);
  MLRG_LAUNCH_CHECK("k_slab_materialize");
}

void slab_store(const float2* out, SlabGeom g, float2* value, cudaStream_t s) {
  k_slab_store<float2><<<2 * sm_count(), 256, 0, s>>>(out, g, value);
  MLRG_LAUNCH_CHECK("k_slab_store");
}

void slab_store(const double2* out, SlabGeom g, float2* value, cudaStream_t s) {
  k_slab_store<double2><<<2 * sm_count(), 256, 0, s>>>(out, g, value);
  MLRG_LAUNCH_CHECK("k_slab_store");
}

void slab_sub(float2* out, SlabGeom g, const float2* sub, cudaStream_t s) {
  k_slab_sub<<<2 * sm_count(), 256, 0, s>>>(out, g, sub);
  MLRG_LAUNCH_CHECK("k_slab_sub");
}

}  // namespace mlrg::ops
