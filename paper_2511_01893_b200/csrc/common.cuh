// Shared device helpers for the sm_100a kernels: complex arithmetic on
// float2/double2, bit reversal for the in-place FFTs, block reductions and the
// shared-memory FFT cores.
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

// Position of frequency k inside a length-2^logm DIF output (bit-reversed order).
__device__ __forceinline__ int brev(int k, int logm) {
  return static_cast<int>(__brev(static_cast<unsigned>(k)) >> (32 - logm));
}

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

// In-place radix-4/radix-2 decimation-in-frequency FFT over shared memory.
// Element (m, c) of the batch lives at s[m * sm + c]; the natural-order input
// is replaced by its unnormalised transform X[k] = sum_m x[m] e^{SIGN 2 pi i mk/M}
// stored at position brev(k). `tw` holds e^{+2 pi i k/M} for k < M/2.
// Lanes run along c first, so rows stay contiguous across a warp.
template <int SIGN, class T>
__device__ void fft_dif(T* s, int logm, int ncols, int sm, const T* __restrict__ tw) {
  const int m = 1 << logm;
  int span = m;  // current sub-transform size
  while (span >= 4) {
    const int l = span >> 2;
    const int tws1 = m / span;         // w_{4L}^j -> tw[j * m/(4L)]
    const int tws2 = (m << 1) / span;  // w_{2L}^j -> tw[j * m/(2L)]
    const int nbf = (m >> 2) * ncols;
    for (int idx = threadIdx.x; idx < nbf; idx += blockDim.x) {
      const int c = idx % ncols, bf = idx / ncols;
      const int j = bf % l, base = (bf / l) * span + j;
      T* p = s + base * sm + c;
      const T a0 = p[0], a1 = p[l * sm], a2 = p[2 * l * sm], a3 = p[3 * l * sm];
      T w4 = tw[j * tws1];
      T w2 = tw[j * tws2];
      if (SIGN < 0) {
        w4.y = -w4.y;
        w2.y = -w2.y;
      }
      const T y0 = cadd(a0, a2), y1 = cadd(a1, a3);
      const T y2 = cmul(csub(a0, a2), w4);
      const T y3 = cmul(cmul_i<SIGN>(csub(a1, a3)), w4);  // w_{4L}^{j+L} = w_{4L}^j * (SIGN i)
      p[0] = cadd(y0, y1);
      p[l * sm] = cmul(csub(y0, y1), w2);
      p[2 * l * sm] = cadd(y2, y3);
      p[3 * l * sm] = cmul(csub(y2, y3), w2);
    }
    __syncthreads();
    span = l;
  }
  if (span == 2) {
    const int nbf = (m >> 1) * ncols;
    for (int idx = threadIdx.x; idx < nbf; idx += blockDim.x) {
      const int c = idx % ncols, bf = idx / ncols;
      T* p = s + (bf * 2) * sm + c;
      const T a0 = p[0], a1 = p[sm];
      p[0] = cadd(a0, a1);
      p[sm] = csub(a0, a1);
    }
    __syncthreads();
  }
}

// In-place radix-2/radix-4 decimation-in-time FFT over shared memory: the
// input sits at bit-reversed positions (x[m] at brev(m)), the output X[k] is
// left in natural order. Same layout and twiddle table as fft_dif.
template <int SIGN, class T>
__device__ void fft_dit(T* s, int logm, int ncols, int sm, const T* __restrict__ tw) {
  const int m = 1 << logm;
  int l = 1;  // size of the sub-transforms being combined
  if (logm & 1) {
    const int nbf = (m >> 1) * ncols;
    for (int idx = threadIdx.x; idx < nbf; idx += blockDim.x) {
      const int c = idx % ncols, bf = idx / ncols;
      T* p = s + (bf * 2) * sm + c;
      const T a0 = p[0], a1 = p[sm];
      p[0] = cadd(a0, a1);
      p[sm] = csub(a0, a1);
    }
    __syncthreads();
    l = 2;
  }
  for (; l < m; l <<= 2) {
    const int span = l << 2;
    const int tws2 = (m << 1) / span;  // w_{2L}^j
    const int tws4 = m / span;         // w_{4L}^j
    const int nbf = (m >> 2) * ncols;
    for (int idx = threadIdx.x; idx < nbf; idx += blockDim.x) {
      const int c = idx % ncols, bf = idx / ncols;
      const int j = bf % l, base = (bf / l) * span + j;
      T* p = s + base * sm + c;
      T t = tw[j * tws2];
      T u = tw[j * tws4];
      if (SIGN < 0) {
        t.y = -t.y;
        u.y = -u.y;
      }
      const T a0 = p[0], a1 = cmul(p[l * sm], t), a2 = p[2 * l * sm], a3 = cmul(p[3 * l * sm], t);
      const T y0 = cadd(a0, a1), y1 = csub(a0, a1), y2 = cadd(a2, a3), y3 = csub(a2, a3);
      const T uy2 = cmul(y2, u), uy3 = cmul_i<SIGN>(cmul(y3, u));
      p[0] = cadd(y0, uy2);
      p[2 * l * sm] = csub(y0, uy2);
      p[l * sm] = cadd(y1, uy3);
      p[3 * l * sm] = csub(y1, uy3);
    }
    __syncthreads();
  }
}

}  // namespace mlrg
