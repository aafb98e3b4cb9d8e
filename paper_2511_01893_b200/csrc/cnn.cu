// CNN key encoder on the device (encoder_variant = cnn; encoder.cpp:95-197):
// per slab, the chunk (rows = the chunk's (axis 0, axis 1) pairs, columns =
// axis 2) is normalised by its RMS into two float planes (re, im), then
// conv1 (2 -> 32, 5x5, stride 2, pad 2) + ReLU, conv2 (32 -> 64, 3x3, stride 2,
// pad 1) + ReLU, global average pool and FC -> key_dim. Every output of the
// convolutions and the FC accumulates in double, bias first, then over (input
// channel, ky, kx) in the reference's order with explicit _rn arithmetic (no
// contraction), and rounds to float like the reference's FeatureMap. The
// RMS and the pool are deterministic two-level reductions.
#include <algorithm>

#include "cnn.hpp"
#include "common.cuh"

namespace mlrg::ops {

namespace {

constexpr int kParts = 64;  // CTAs per slab for the RMS and pool reductions
constexpr int kMaxSlabs = 64;
struct SlabList {
  long long start[kMaxSlabs];
};

__device__ __forceinline__ long long chunk_offset(const SlabGeom& g, long long start, long long ce) {
  if (g.axis == 0) return start * g.d1 * g.d2 + ce;
  const long long per = g.extent * g.d2;
  const long long i = ce / per, rem = ce - i * per, kl = rem / g.d2;
  return (i * g.d1 + start + kl) * g.d2 + (rem - kl * g.d2);
}

// partial sums of |x|^2 per (slab, part)
template <class TX>
__global__ void __launch_bounds__(256) k_cnn_sq(const TX* __restrict__ x, SlabGeom g, SlabList sl, long long n,
                                                double* __restrict__ part) {
  const int slab = blockIdx.y;
  double v[1] = {0.0};
  for (long long ce = blockIdx.x * 256LL + threadIdx.x; ce < n; ce += 256LL * gridDim.x) {
    const TX a = x[chunk_offset(g, sl.start[slab], ce)];
    v[0] += static_cast<double>(a.x) * a.x + static_cast<double>(a.y) * a.y;
  }
  __shared__ double scratch[8];
  block_sum<1>(v, scratch);
  if (threadIdx.x == 0) part[slab * kParts + blockIdx.x] = v[0];
}

__global__ void k_cnn_sq_final(const double* __restrict__ part, int ns, long long n, double* __restrict__ norms2,
                               double* __restrict__ scale) {
  const int slab = threadIdx.x;
  if (slab >= ns) return;
  double s = 0.0;
  for (int p = 0; p < kParts; ++p) s += part[slab * kParts + p];
  norms2[slab] = s;
  const double rms = sqrt(s / static_cast<double>(n > 0 ? n : 1));  // cnn_input, encoder.cpp:96-111
  scale[slab] = rms > 0.0 ? 1.0 / rms : 0.0;
}

// conv1 + ReLU: one thread per (slab, y2, x2) for all output channels; the
// 2 x 5 x 5 input patch (rounded to float as cnn_input does) stays in registers.
template <class TX>
__global__ void __launch_bounds__(128) k_cnn_conv1(const TX* __restrict__ x, SlabGeom g, SlabList sl,
                                                   const double* __restrict__ scale, int H, int W, int H1, int W1,
                                                   const float* __restrict__ w, const float* __restrict__ b,
                                                   int cout, float* __restrict__ act1) {
  constexpr int K = 5, PAD = 2;
  const int slab = blockIdx.y;
  const long long pos = blockIdx.x * 128LL + threadIdx.x;
  if (pos >= static_cast<long long>(H1) * W1) return;
  const int y2 = static_cast<int>(pos / W1), x2 = static_cast<int>(pos - static_cast<long long>(y2) * W1);
  const double sc = scale[slab];
  float in[2][K][K];
  bool ok[K][K];
#pragma unroll
  for (int ky = 0; ky < K; ++ky)
#pragma unroll
    for (int kx = 0; kx < K; ++kx) {
      const int iy = 2 * y2 + ky - PAD, ix = 2 * x2 + kx - PAD;
      ok[ky][kx] = iy >= 0 && iy < H && ix >= 0 && ix < W;
      in[0][ky][kx] = in[1][ky][kx] = 0.f;
      if (ok[ky][kx]) {
        const TX a = x[chunk_offset(g, sl.start[slab], static_cast<long long>(iy) * W + ix)];
        in[0][ky][kx] = static_cast<float>(__dmul_rn(static_cast<double>(a.x), sc));
        in[1][ky][kx] = static_cast<float>(__dmul_rn(static_cast<double>(a.y), sc));
      }
    }
  float* out = act1 + static_cast<long long>(slab) * cout * H1 * W1 + pos;
  for (int o = 0; o < cout; ++o) {
    double acc = b[o];
    const float* wo = w + o * 2 * K * K;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int ky = 0; ky < K; ++ky)
#pragma unroll
        for (int kx = 0; kx < K; ++kx)
          if (ok[ky][kx])
            acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(wo[(c * K + ky) * K + kx]),
                                           static_cast<double>(in[c][ky][kx])));
    const float v = static_cast<float>(acc);
    out[static_cast<long long>(o) * H1 * W1] = v > 0.f ? v : 0.f;
  }
}

// conv2 + ReLU: one thread per (slab, y2, x2, group of 8 output channels).
constexpr int kOG = 8;
__global__ void __launch_bounds__(128) k_cnn_conv2(const float* __restrict__ act1, int cin, int H1, int W1, int H2,
                                                   int W2, const float* __restrict__ w, const float* __restrict__ b,
                                                   int cout, float* __restrict__ act2) {
  constexpr int K = 3, PAD = 1;
  const int slab = blockIdx.z, og = blockIdx.y;
  const long long pos = blockIdx.x * 128LL + threadIdx.x;
  if (pos >= static_cast<long long>(H2) * W2) return;
  const int y2 = static_cast<int>(pos / W2), x2 = static_cast<int>(pos - static_cast<long long>(y2) * W2);
  const float* in = act1 + static_cast<long long>(slab) * cin * H1 * W1;
  double acc[kOG];
#pragma unroll
  for (int q = 0; q < kOG; ++q) acc[q] = b[og * kOG + q];
  for (int c = 0; c < cin; ++c) {
    const float* ic = in + static_cast<long long>(c) * H1 * W1;
#pragma unroll
    for (int ky = 0; ky < K; ++ky) {
      const int iy = 2 * y2 + ky - PAD;
      if (iy < 0 || iy >= H1) continue;
#pragma unroll
      for (int kx = 0; kx < K; ++kx) {
        const int ix = 2 * x2 + kx - PAD;
        if (ix < 0 || ix >= W1) continue;
        const double v = static_cast<double>(ic[static_cast<long long>(iy) * W1 + ix]);
#pragma unroll
        for (int q = 0; q < kOG; ++q)
          acc[q] = __dadd_rn(acc[q], __dmul_rn(static_cast<double>(w[(((og * kOG + q) * cin + c) * K + ky) * K + kx]), v));
      }
    }
  }
  float* out = act2 + static_cast<long long>(slab) * cout * H2 * W2 + pos;
#pragma unroll
  for (int q = 0; q < kOG; ++q) {
    const float v = static_cast<float>(acc[q]);
    out[static_cast<long long>(og * kOG + q) * H2 * W2] = v > 0.f ? v : 0.f;
  }
}

// global average pool partials per (slab, channel, part)
__global__ void __launch_bounds__(256) k_cnn_pool(const float* __restrict__ act2, int cout, long long hw,
                                                  double* __restrict__ part) {
  const int slab = blockIdx.z, c = blockIdx.y;
  const float* a = act2 + (static_cast<long long>(slab) * cout + c) * hw;
  double v[1] = {0.0};
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < hw; e += 256LL * gridDim.x) v[0] += a[e];
  __shared__ double scratch[8];
  block_sum<1>(v, scratch);
  if (threadIdx.x == 0) part[(static_cast<long long>(slab) * cout + c) * kParts + blockIdx.x] = v[0];
}

// pool + FC per slab (one CTA): z[r] = fc_b[r] + sum_c fc_w[r][c] * gap[c]
__global__ void k_cnn_head(const double* __restrict__ part, int cout, long long hw, const float* __restrict__ fw,
                           const float* __restrict__ fb, int kd, float* __restrict__ keys) {
  const int slab = blockIdx.x;
  __shared__ double gap[256];
  const double inv_hw = 1.0 / static_cast<double>(hw);
  for (int c = threadIdx.x; c < cout; c += blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < kParts; ++p) s += part[(static_cast<long long>(slab) * cout + c) * kParts + p];
    gap[c] = __dmul_rn(s, inv_hw);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < kd; r += blockDim.x) {
    double acc = fb[r];
    for (int c = 0; c < cout; ++c)
      acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(fw[r * cout + c]), gap[c]));
    keys[static_cast<long long>(slab) * kd + r] = static_cast<float>(acc);
  }
}

template <class TX>
void encode_cnn_impl(const TX* x, SlabGeom g, const std::int64_t* starts, int ns, const CnnDevice& w, float* keys,
                     double* norms2, CnnWork& work, cudaStream_t s) {
  const CnnWeights& h = w.host;
  const long long n = g.count();
  const int H = static_cast<int>(g.axis == 0 ? g.extent * g.d1 : g.d0 * g.extent), W = static_cast<int>(g.d2);
  const int H1 = (H - 1) / 2 + 1, W1 = (W - 1) / 2 + 1, H2 = (H1 - 1) / 2 + 1, W2 = (W1 - 1) / 2 + 1;
  // slabs in groups bounded to ~4 GB of activations
  const long long per_slab = static_cast<long long>(h.c1_out) * H1 * W1 + static_cast<long long>(h.c2_out) * H2 * W2;
  const int grp = static_cast<int>(std::clamp<long long>((1LL << 30) / std::max(per_slab, 1LL), 1, kMaxSlabs));
  for (int b0 = 0; b0 < ns; b0 += grp) {
    const int nb = std::min(grp, ns - b0);
    SlabList sl{};
    for (int q = 0; q < nb; ++q) sl.start[q] = starts[b0 + q];
    work.act1.resize(static_cast<std::size_t>(nb) * h.c1_out * H1 * W1);
    work.act2.resize(static_cast<std::size_t>(nb) * h.c2_out * H2 * W2);
    work.part.resize(static_cast<std::size_t>(nb) * (h.c2_out + 2) * kParts);
    work.scale.resize(static_cast<std::size_t>(nb));
    k_cnn_sq<TX><<<dim3(kParts, nb), 256, 0, s>>>(x, g, sl, n, work.part.get());
    MLRG_LAUNCH_CHECK("k_cnn_sq");
    k_cnn_sq_final<<<1, 64, 0, s>>>(work.part.get(), nb, n, norms2 + b0, work.scale.get());
    MLRG_LAUNCH_CHECK("k_cnn_sq_final");
    const long long p1 = static_cast<long long>(H1) * W1, p2 = static_cast<long long>(H2) * W2;
    k_cnn_conv1<TX><<<dim3(static_cast<unsigned>((p1 + 127) / 128), nb), 128, 0, s>>>(
        x, g, sl, work.scale.get(), H, W, H1, W1, w.c1w.get(), w.c1b.get(), h.c1_out, work.act1.get());
    MLRG_LAUNCH_CHECK("k_cnn_conv1");
    k_cnn_conv2<<<dim3(static_cast<unsigned>((p2 + 127) / 128), h.c2_out / kOG, nb), 128, 0, s>>>(
        work.act1.get(), h.c1_out, H1, W1, H2, W2, w.c2w.get(), w.c2b.get(), h.c2_out, work.act2.get());
    MLRG_LAUNCH_CHECK("k_cnn_conv2");
    k_cnn_pool<<<dim3(kParts, h.c2_out, nb), 256, 0, s>>>(work.act2.get(), h.c2_out, p2, work.part.get());
    MLRG_LAUNCH_CHECK("k_cnn_pool");
    k_cnn_head<<<nb, 128, 0, s>>>(work.part.get(), h.c2_out, p2, w.fcw.get(), w.fcb.get(), h.key_dim,
                                  keys + static_cast<long long>(b0) * h.key_dim);
    MLRG_LAUNCH_CHECK("k_cnn_head");
  }
}

}  // namespace

void encode_cnn(const float2* x, SlabGeom shape, const std::int64_t* starts, int ns, const CnnDevice& w, float* keys,
                double* norms2, CnnWork& work, cudaStream_t s) {
  encode_cnn_impl(x, shape, starts, ns, w, keys, norms2, work, s);
}
void encode_cnn(const double2* x, SlabGeom shape, const std::int64_t* starts, int ns, const CnnDevice& w, float* keys,
                double* norms2, CnnWork& work, cudaStream_t s) {
  encode_cnn_impl(x, shape, starts, ns, w, keys, norms2, work, s);
}

}  // namespace mlrg::ops
