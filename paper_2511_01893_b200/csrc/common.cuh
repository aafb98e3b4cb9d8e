// Shared device helpers for the sm_100a kernels: complex arithmetic on
// float2/double2, block reductions and the shared-memory Stockham FFT.
//
// Precision: the transforms store their big intermediates (oversampled
// grids) in complex64 but compute every FFT butterfly, twiddle and long
// accumulation in double. The reference solve is sensitive to operator
// noise (a 1e-6 relative perturbation of every operator output moves the
// 64^3 iterate by 2.7e-4 after ten iterations), so the operators must stay
// within a few complex64 ulps of the reference, which fp32 butterflies and
// fp32 accumulations over thousands of terms do not.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mlrg {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// multiply by +i (SIGN>0) or -i (SIGN<0)
template <int SIGN, class T>
__device__ __forceinline__ T cmul_i(T a) {
  T r;
  if (SIGN > 0) {
    r.x = -a.y;
    r.y = a.x;
  } else {
    r.x = a.y;
    r.y = -a.x;
  }
  return r;
}

__device__ __forceinline__ double2 to_d(float2 a) { return make_double2(a.x, a.y); }
__device__ __forceinline__ double2 to_d(double2 a) { return a; }
__device__ __forceinline__ float2 to_f(double2 a) { return make_float2(static_cast<float>(a.x), static_cast<float>(a.y)); }

// Sum of NV doubles across the block; result valid in thread 0. `scratch`
// needs blockDim.x/32 * NV doubles of shared memory.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[warp * NV + i] = v[i];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += scratch[w * NV + i];
      v[i] = s;
    }
  }
  __syncthreads();
}

// ---- batched Stockham FFT over a shared-memory tile ------------------------------------
// The tile holds nb independent columns of length m = 2^logm: element (row,
// b) at s[row * ld + b]. The transform is in place and self-sorting (natural
// order in and out): X[k] = sum_j x[j] e^{SIGN 2 pi i jk/m}. It runs one
// radix-2 or radix-4 pass (logm % 3 != 0) followed by radix-8 passes, each
// thread owning 8 elements per pass in registers, so a 512-point column
// costs three passes and six block barriers. The block must have exactly
// nb * m / 8 threads (m >= 8); thread t works on column b = t % nb and
// butterfly group g = t / nb. `tw` holds e^{+2 pi i k/m} for k < m.
template <int SIGN>
__device__ __forceinline__ void fft4_reg(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3);
  const double2 d13 = cmul_i<SIGN>(csub(a1, a3));
  a0 = cadd(s02, s13);
  a1 = cadd(d02, d13);
  a2 = csub(s02, s13);
  a3 = csub(d02, d13);
}

template <int SIGN>
__device__ __forceinline__ void fft8_reg(double2* v) {
  fft4_reg<SIGN>(v[0], v[2], v[4], v[6]);  // E[k] at v[2k]
  fft4_reg<SIGN>(v[1], v[3], v[5], v[7]);  // O[k] at v[2k+1]
  constexpr double c = 0.70710678118654752440;
  const double2 o1 = v[3], o3 = v[7];
  // w8 = c (1 + SIGN i), w8^2 = SIGN i, w8^3 = c (-1 + SIGN i)
  const double2 t1 = make_double2(c * (o1.x - SIGN * o1.y), c * (o1.y + SIGN * o1.x));
  const double2 t2 = cmul_i<SIGN>(v[5]);
  const double2 t3 = make_double2(c * (-o3.x - SIGN * o3.y), c * (-o3.y + SIGN * o3.x));
  const double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], o0 = v[1];
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, t1);
  v[5] = csub(e1, t1);
  v[2] = cadd(e2, t2);
  v[6] = csub(e2, t2);
  v[3] = cadd(e3, t3);
  v[7] = csub(e3, t3);
}

template <int R, int SIGN>
__device__ __forceinline__ void fft_reg(double2* v) {
  if constexpr (R == 8) {
    fft8_reg<SIGN>(v);
  } else if constexpr (R == 4) {
    fft4_reg<SIGN>(v[0], v[1], v[2], v[3]);
  } else {
    const double2 a = v[0];
    v[0] = cadd(a, v[1]);
    v[1] = csub(a, v[1]);
  }
}

// One pass. GIN: the pass reads its inputs through load(row, b) (global
// memory, the transform's first pass) instead of the tile; GOUT: it writes
// through store(row, b, value) (the last pass) instead of the tile.
// ZP (zero-padded input, first pass only): the input of slots [m/4, 3m/4) is
// known to be zero (a length-n signal centred in m = 2n slots: fu1d, the fu2d
// row and column passes), so a radix-8 first pass never loads its inputs
// r = 2..5 (rows [m/4, 3m/4) for stride m/8).
template <int R, int LOGR, int SIGN, bool GIN, bool GOUT, bool ZP, class Load, class Store>
__device__ __forceinline__ void stockham_pass(double2* s, int ld, int b, int g, int logm, int logns,
                                              const double2* __restrict__ tw, const Load& load, const Store& store) {
  constexpr int PER = 8 / R;
  const int m8 = 1 << (logm - 3), stride = 1 << (logm - LOGR), ns = 1 << logns;
  double2 v[8];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int gg = g + q * m8;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = gg + r * stride;
      if constexpr (GIN && ZP && R == 8) {
        if (r >= 2 && r < 6) v[q * R + r] = make_double2(0.0, 0.0);
        else v[q * R + r] = load(row, b);
      } else if constexpr (GIN) {
        v[q * R + r] = load(row, b);
      } else {
        v[q * R + r] = s[row * ld + b];
      }
    }
  }
  if constexpr (!GIN || GOUT) __syncthreads();  // in place: every read precedes any write
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int gg = g + q * m8;
    const int k = gg & (ns - 1);
    if (logns > 0) {
      const int step = k << (logm - logns - LOGR);  // k m / (ns R)
      // w^r for r < R from the table entries w, w^2, w^4 and products (the
      // twiddle loads share the L1/shared-memory pipe with the data, which
      // bounds these passes; the products are exact to a few double ulps)
      double2 w[8];
      w[1] = tw[step];
      if constexpr (R >= 4) {
        w[2] = tw[2 * step];
        w[3] = cmul(w[1], w[2]);
      }
      if constexpr (R == 8) {
        w[4] = tw[4 * step];
        w[5] = cmul(w[4], w[1]);
        w[6] = cmul(w[4], w[2]);
        w[7] = cmul(w[4], w[3]);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) {
        if (SIGN < 0) w[r].y = -w[r].y;
        v[q * R + r] = cmul(v[q * R + r], w[r]);
      }
    }
    fft_reg<R, SIGN>(v + q * R);
    const int base = ((gg >> logns) << (logns + LOGR)) + k;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = base + (r << logns);
      if constexpr (GOUT) store(row, b, v[q * R + r]);
      else s[row * ld + b] = v[q * R + r];
    }
  }
  if constexpr (!GOUT) __syncthreads();
}

struct NoLoad {
  __device__ double2 operator()(int, int) const { return make_double2(0.0, 0.0); }
};
struct NoStore {
  __device__ void operator()(int, int, double2) const {}
};

// Full transform. With GIN the tile's initial contents are ignored and the
// first pass reads load(row, b) for row < m (natural input order); with GOUT
// the last pass hands X[row] of column b to store(row, b, X) and the tile is
// left as scratch; otherwise the tile holds the input / output.
template <int SIGN, bool GIN, bool GOUT, bool ZP, class Load, class Store>
__device__ __forceinline__ void fft_stockham_impl(double2* s, int logm, int nb, int ld, const double2* __restrict__ tw,
                                                  const Load& load, const Store& store) {
  const int b = threadIdx.x % nb, g = threadIdx.x / nb;
  const int npass = (logm + 2) / 3;
  int logns = 0, p = 0;
  if (logm % 3 == 1) {
    if (npass == 1) stockham_pass<2, 1, SIGN, GIN, GOUT, false>(s, ld, b, g, logm, 0, tw, load, store);
    else stockham_pass<2, 1, SIGN, GIN, false, false>(s, ld, b, g, logm, 0, tw, load, store);
    logns = 1;
    p = 1;
  } else if (logm % 3 == 2) {
    if (npass == 1) stockham_pass<4, 2, SIGN, GIN, GOUT, false>(s, ld, b, g, logm, 0, tw, load, store);
    else stockham_pass<4, 2, SIGN, GIN, false, false>(s, ld, b, g, logm, 0, tw, load, store);
    logns = 2;
    p = 1;
  }
  for (; logns < logm; logns += 3, ++p) {
    const bool first = p == 0, last = p == npass - 1;
    if (first && last) stockham_pass<8, 3, SIGN, GIN, GOUT, ZP>(s, ld, b, g, logm, logns, tw, load, store);
    else if (first) stockham_pass<8, 3, SIGN, GIN, false, ZP>(s, ld, b, g, logm, logns, tw, load, store);
    else if (last) stockham_pass<8, 3, SIGN, false, GOUT, false>(s, ld, b, g, logm, logns, tw, load, store);
    else stockham_pass<8, 3, SIGN, false, false, false>(s, ld, b, g, logm, logns, tw, load, store);
  }
}

// The transform with the common shapes' (logm, nb, ld) as literals, so the
// inlined passes' index arithmetic (strides, masks, the column / butterfly
// split of threadIdx) folds into immediates: 256^3 and 512^3 run 512- and
// 1024-point transforms over 4 or 8 columns per CTA. Other shapes take the
// general path.
template <int SIGN, bool GIN = false, bool GOUT = false, bool ZP = false, class Load = NoLoad, class Store = NoStore>
__device__ __forceinline__ void fft_stockham(double2* s, int logm, int nb, int ld, const double2* __restrict__ tw,
                                             const Load& load = Load(), const Store& store = Store()) {
#ifndef MLRG_FFT_GENERIC_ONLY
#define MLRG_FFT_CASE(L, N)                                                                      \
  if (logm == L && nb == N) {                                                                    \
    if (ld == N) return fft_stockham_impl<SIGN, GIN, GOUT, ZP>(s, L, N, N, tw, load, store);     \
    if (ld == N + 1) return fft_stockham_impl<SIGN, GIN, GOUT, ZP>(s, L, N, N + 1, tw, load, store); \
  }
  MLRG_FFT_CASE(9, 8)
  MLRG_FFT_CASE(10, 4)
  MLRG_FFT_CASE(10, 8)
#undef MLRG_FFT_CASE
#endif
  fft_stockham_impl<SIGN, GIN, GOUT, ZP>(s, logm, nb, ld, tw, load, store);
}

}  // namespace mlrg
