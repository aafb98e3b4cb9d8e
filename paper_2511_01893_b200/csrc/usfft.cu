// USFFT operator kernels for sm_100a (see usfft.hpp for the reference map).
//
// Data flow per operator (M = oversampled grid = next_pow2(2n)):
//   fu1d      one CTA per (volume row i, tile of C columns j): wrapped +
//             deconvolved placement -> in-smem DIF FFT (bit-reversed output)
//             -> 24-tap gather read straight from the bit-reversed positions.
//   fu1d_adj  mirror: conj-phase load -> 24-tap spread in gather form over a
//             host-built cell->target CSR (no atomics) -> DIF FFT(-1) -> read.
//   fu2d      per batch of 16 detector rows, grid layout [M1][M2][16] (row
//             batch innermost, 128 B per grid cell): row FFT pass, column FFT
//             pass (both DIF, indices stay bit-reversed), then a warp-cooperative
//             576-tap gather per target with weights amortised over the 16 rows.
//   fu2d_adj  mirror: targets listed per 8x4 cell patch (host CSR) -> each cell
//             gathers its targets (no atomics) -> column DIF(-1) -> row DIT(-1).
// FFT butterflies, twiddles, deconvolution and accumulations run in double;
// the oversampled grids between passes are stored in complex64 (common.cuh).
#include <algorithm>
#include <cmath>
#include <complex>
#include <numbers>
#include <vector>

#include "common.cuh"
#include "usfft.hpp"

namespace mlrg {

namespace {

constexpr int KB = Usfft::kRowBatch;

// k-columns per CTA of a 2D-grid FFT pass over length m (double smem <= ~140 KB).
int pass_cols(std::int64_t m) { return static_cast<int>(std::clamp<std::int64_t>(8192 / m, 2, KB)); }

// ------------------------------------------------------------------------------------------
// fu1d / fu1d_adj
// ------------------------------------------------------------------------------------------
template <class TIn>
__global__ void __launch_bounds__(256) k_fu1d(const TIn* __restrict__ u, float2* __restrict__ out, int n0, int n2,
                                              int h, int logm, int center, int ncol,
                                              const double* __restrict__ deconv, const int* __restrict__ start,
                                              const float* __restrict__ wts, const double2* __restrict__ fac,
                                              const double2* __restrict__ tw) {
  extern __shared__ double2 sd[];
  const int m = 1 << logm, mask = m - 1;
  const int j0 = blockIdx.x * ncol;
  const TIn* ui = u + static_cast<long long>(blockIdx.y) * n0 * n2;
  for (int idx = threadIdx.x; idx < m * ncol; idx += blockDim.x) {
    const int r = idx / ncol, c = idx - r * ncol;
    const int mode = (r + center) & mask;  // grid slot r holds mode (r + center) mod m
    const int j = j0 + c;
    double2 v = make_double2(0.0, 0.0);
    if (mode < n0 && j < n2) v = cscale(to_d(ui[static_cast<long long>(mode) * n2 + j]), deconv[mode]);
    sd[idx] = v;
  }
  __syncthreads();
  fft_dif<+1>(sd, logm, ncol, ncol, tw);
  float2* oi = out + static_cast<long long>(blockIdx.y) * h * n2;
  for (int idx = threadIdx.x; idx < h * ncol; idx += blockDim.x) {
    const int k = idx / ncol, c = idx - k * ncol;
    const int j = j0 + c;
    if (j >= n2) continue;
    const int st = start[k];
    const float* wk = wts + k * kTaps;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int a = 0; a < kTaps; ++a) {
      const double2 g = sd[brev((st + a) & mask, logm) * ncol + c];
      const double wa = __ldg(wk + a);
      acc.x = fma(g.x, wa, acc.x);
      acc.y = fma(g.y, wa, acc.y);
    }
    oi[static_cast<long long>(k) * n2 + j] = to_f(cmul(acc, fac[k]));
  }
}

template <class TOut>
__global__ void __launch_bounds__(256) k_fu1d_adj(const float2* __restrict__ v, TOut* __restrict__ out, int n0,
                                                  int n2, int h, int logm, int center, int ncol,
                                                  const double2* __restrict__ cphase,
                                                  const int* __restrict__ cell_ptr, const int* __restrict__ cell_k,
                                                  const float* __restrict__ cell_w,
                                                  const double* __restrict__ pdeconv,
                                                  const double2* __restrict__ tw) {
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
    const int e1 = cell_ptr[l + 1];
    for (int e = cell_ptr[l]; e < e1; ++e) {
      const double2 x = vt[cell_k[e] * ncol + c];
      const double wv = __ldg(cell_w + e);
      acc.x = fma(x.x, wv, acc.x);
      acc.y = fma(x.y, wv, acc.y);
    }
    sd[idx] = acc;
  }
  __syncthreads();
  fft_dif<-1>(sd, logm, ncol, ncol, tw);
  TOut* oi = out + static_cast<long long>(blockIdx.y) * n0 * n2;
  for (int idx = threadIdx.x; idx < n0 * ncol; idx += blockDim.x) {
    const int mode = idx / ncol, c = idx - mode * ncol;
    const int j = j0 + c;
    if (j >= n2) continue;
    const int slot = (mode - center) & mask;
    const double2 r = cscale(sd[brev(slot, logm) * ncol + c], pdeconv[mode]);
    TOut& o = oi[static_cast<long long>(mode) * n2 + j];
    o.x = static_cast<decltype(o.x)>(r.x);
    o.y = static_cast<decltype(o.y)>(r.y);
  }
}

// ------------------------------------------------------------------------------------------
// fu2d forward: row pass, column pass, gather
// ------------------------------------------------------------------------------------------
// S[i][c'][KB]: row FFT of v[i, k0+kk, :] * dx[i] * dy[:] placed at wrapped slots.
__global__ void __launch_bounds__(256) k_fu2d_rows(const float2* __restrict__ v, long long ld, long long k0, int nk,
                                                   int n2, int logm2, int center2, int ks_n,
                                                   const double* __restrict__ dx, const double* __restrict__ dy,
                                                   const double2* __restrict__ tw2, float2* __restrict__ S) {
  extern __shared__ double2 sd[];
  const int m2 = 1 << logm2, mask2 = m2 - 1, sm = ks_n + 1;
  const int i = blockIdx.x, ks = blockIdx.y * ks_n;
  const double di = dx[i];
  for (int idx = threadIdx.x; idx < m2 * ks_n; idx += blockDim.x) {
    const int kk = idx / m2, r = idx - kk * m2;
    const int j = (r + center2) & mask2;
    double2 val = make_double2(0.0, 0.0);
    if (j < n2 && ks + kk < nk)
      val = cscale(to_d(v[(static_cast<long long>(i) * ld + k0 + ks + kk) * n2 + j]), di * dy[j]);
    sd[r * sm + kk] = val;
  }
  __syncthreads();
  fft_dif<+1>(sd, logm2, ks_n, sm, tw2);
  float2* Si = S + static_cast<long long>(i) * m2 * KB + ks;
  for (int idx = threadIdx.x; idx < m2 * ks_n; idx += blockDim.x) {
    const int r = idx / ks_n, kk = idx - r * ks_n;
    Si[static_cast<long long>(r) * KB + kk] = to_f(sd[r * sm + kk]);
  }
}

// G[r'][c'][KB]: column FFT over the n1 non-zero wrapped rows of S.
__global__ void __launch_bounds__(256) k_fu2d_cols(const float2* __restrict__ S, int n1, int logm1, int center1,
                                                   int logm2, int ks_n, const double2* __restrict__ tw1,
                                                   float2* __restrict__ G) {
  extern __shared__ double2 sd[];
  const int m1 = 1 << logm1, mask1 = m1 - 1, m2 = 1 << logm2;
  const int c = blockIdx.x, ks = blockIdx.y * ks_n;
  for (int idx = threadIdx.x; idx < m1 * ks_n; idx += blockDim.x) {
    const int r = idx / ks_n, kk = idx - r * ks_n;
    const int i = (r + center1) & mask1;
    sd[idx] = i < n1 ? to_d(S[(static_cast<long long>(i) * m2 + c) * KB + ks + kk]) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_dif<+1>(sd, logm1, ks_n, ks_n, tw1);
  for (int idx = threadIdx.x; idx < m1 * ks_n; idx += blockDim.x) {
    const int r = idx / ks_n, kk = idx - r * ks_n;
    G[(static_cast<long long>(r) * m2 + c) * KB + ks + kk] = to_f(sd[idx]);
  }
}

struct GatherOut {
  float2* out;
  long long ld_out, k0_out;
  const float2* sub;
  long long ld_sub, k0_sub;
  const float2* dot;
  long long ld_dot, k0_dot;
  int reduce;
};


// ---- warp-cooperative gather -------------------------------------------------------------
// Targets are binned by window origin (kBox x kBox cells) and cut into groups
// of <= 32 (host, once per geometry). One
// warp owns one group and walks the union of the group's 24x24 windows row by
// row: the warp stages the row's grid cells (128 B each: 16 detector rows)
// into shared memory with cp.async, double-buffered one row ahead, then every
// lane reads the SAME cell (a broadcast) and weights it for its own target
// (zero outside its window). Per cell a warp issues 8 broadcast loads and 32
// FMA per lane instead of 32 scattered 128 B loads.
struct GatherGroup {
  int first, count, r0, c0, nr, nc;  // sorted-target range, union window origin and extent
};

constexpr int kGroupWarps = 4;
constexpr int kWStride = kTaps + 1;  // padded smem weight rows (odd stride: no bank conflicts)
constexpr int kBox = 12;             // group bounding box (cells) -> union window <= 37 x 37
constexpr int kUnionMax = kTaps + kBox + 1;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct GatherSmem {
  float4 row[2][kUnionMax][KB / 2];  // two staged union rows (complex64), 128 B per cell
  double2 rowd[kUnionMax][KB];       // the row being consumed, widened once per warp
  float w1[32][kWStride];
  float w2[32][kWStride];
};

__device__ __forceinline__ void stage_row(GatherSmem& sm, int buf, const float2* __restrict__ G, long long rbase,
                                          int c0, int c_lo, int c_hi, int mask2, int logm2, int lane) {
  for (int idx = c_lo * (KB / 2) + lane; idx < c_hi * (KB / 2); idx += 32) {
    const int cell = idx / (KB / 2), part = idx - cell * (KB / 2);
    const float2* src = G + (rbase + brev((c0 + cell) & mask2, logm2)) * KB + 2 * part;
    cp_async16(&sm.row[buf][cell][part], src);
  }
  cp_async_commit();
}

// Columns [c_lo, c_hi) that some lane needs in union row rr (empty: c_lo >= c_hi).
__device__ __forceinline__ int2 row_span(int rr, int dr, int dc) {
  const bool on = rr - dr >= 0 && rr - dr < kTaps;
  return make_int2(__reduce_min_sync(0xffffffffu, on ? dc : 1 << 20),
                   __reduce_max_sync(0xffffffffu, on ? dc + kTaps : -1));
}

__global__ void __launch_bounds__(32 * kGroupWarps) k_fu2d_gather_warp(
    const float2* __restrict__ G, int ngroups, const GatherGroup* __restrict__ groups, int w, int logm1, int logm2,
    int nk, const int* __restrict__ g_tidx, const int* __restrict__ g_dr, const int* __restrict__ g_dc,
    const float* __restrict__ g_w1, const float* __restrict__ g_w2, const double2* __restrict__ g_fac,
    GatherOut eo, double* __restrict__ partials, int accumulate) {
  extern __shared__ float4 dyn_smem[];
  __shared__ double red_scratch[kGroupWarps * 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  GatherSmem& sm = reinterpret_cast<GatherSmem*>(dyn_smem)[warp];
  const int gi = blockIdx.x * kGroupWarps + warp;
  const int mask1 = (1 << logm1) - 1, mask2 = (1 << logm2) - 1, m2 = 1 << logm2;
  double red[2] = {0.0, 0.0};
  if (gi < ngroups) {
    const GatherGroup gr = groups[gi];
    const bool live = lane < gr.count;
    const int st = gr.first + lane;
    const int dr = live ? g_dr[st] : -1000, dc = live ? g_dc[st] : -1000;
    int2 span = row_span(0, dr, dc);
    stage_row(sm, 0, G, static_cast<long long>(brev(gr.r0 & mask1, logm1)) * m2, gr.c0, span.x, span.y, mask2,
              logm2, lane);
    for (int a = 0; a < kTaps; ++a) {
      sm.w1[lane][a] = live ? g_w1[static_cast<long long>(st) * kTaps + a] : 0.f;
      sm.w2[lane][a] = live ? g_w2[static_cast<long long>(st) * kTaps + a] : 0.f;
    }
    double2 acc[KB];
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) acc[kk] = make_double2(0.0, 0.0);
    for (int rr = 0; rr < gr.nr; ++rr) {
      const int2 cur = span;
      if (rr + 1 < gr.nr) {
        span = row_span(rr + 1, dr, dc);
        stage_row(sm, (rr + 1) & 1, G, static_cast<long long>(brev((gr.r0 + rr + 1) & mask1, logm1)) * m2, gr.c0,
                  span.x, span.y, mask2, logm2, lane);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      // widen the staged row once per warp (not once per lane)
      for (int idx = cur.x * (KB / 2) + lane; idx < cur.y * (KB / 2); idx += 32) {
        const int cell = idx / (KB / 2), part = idx - cell * (KB / 2);
        const float4 g = sm.row[rr & 1][cell][part];
        sm.rowd[cell][2 * part] = make_double2(g.x, g.y);
        sm.rowd[cell][2 * part + 1] = make_double2(g.z, g.w);
      }
      __syncwarp();
      const int a = rr - dr;
      const bool row_on = a >= 0 && a < kTaps;
      double2 inner[KB];
#pragma unroll
      for (int kk = 0; kk < KB; ++kk) inner[kk] = make_double2(0.0, 0.0);
      for (int cc = cur.x; cc < cur.y; ++cc) {
        const int b = cc - dc;
        const double wv = (row_on && b >= 0 && b < kTaps) ? static_cast<double>(sm.w2[lane][b]) : 0.0;
        const double2* gp = sm.rowd[cc];
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) {
          const double2 g = gp[kk];
          inner[kk].x = fma(wv, g.x, inner[kk].x);
          inner[kk].y = fma(wv, g.y, inner[kk].y);
        }
      }
      const double w1 = row_on ? static_cast<double>(sm.w1[lane][a]) : 0.0;
#pragma unroll
      for (int kk = 0; kk < KB; ++kk) {
        acc[kk].x = fma(w1, inner[kk].x, acc[kk].x);
        acc[kk].y = fma(w1, inner[kk].y, acc[kk].y);
      }
      __syncwarp();  // row buffers are refilled by the next iterations
    }
    if (live) {
      const int tq = g_tidx[st];
      const int t = tq / w, q = tq - (tq / w) * w;
      const double2 f = g_fac[st];
#pragma unroll
      for (int kk = 0; kk < KB; ++kk) {
        if (kk >= nk) break;
        double2 val = cmul(acc[kk], f);
        if (eo.sub) val = csub(val, to_d(eo.sub[(t * eo.ld_sub + eo.k0_sub + kk) * w + q]));
        if (eo.out) eo.out[(t * eo.ld_out + eo.k0_out + kk) * w + q] = to_f(val);
        if (eo.reduce) {
          red[0] += val.x * val.x + val.y * val.y;
          if (eo.dot) {
            const float2 d = eo.dot[(t * eo.ld_dot + eo.k0_dot + kk) * w + q];
            red[1] += static_cast<double>(d.x) * val.x + static_cast<double>(d.y) * val.y;
          }
        }
      }
    }
  }
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

// ---- warp-cooperative spread (adjoint) -----------------------------------------------------
// One warp owns an 8x4 patch of grid cells (lane = cell) and walks the host-built
// list of targets whose window touches the patch, 32 targets per chunk: each
// lane stages one target's window origin, weight rows and 16 values into
// shared memory with cp.async (double-buffered one chunk ahead), the warp
// widens the values to double once, then consumes the chunk target by target:
// the values are a broadcast read and each lane adds its own weight. All sums
// run in double (cells near nu = 0 receive thousands of terms). Patches are
// processed heaviest first.
constexpr int kPatchR = 8, kPatchC = 4;

struct SpreadSmem {
  float4 val[2][32][KB / 2];
  double2 vald[32][KB];
  float w1[2][32][kTaps];
  float w2[2][32][kTaps];
  int r0[2][32], c0[2][32];
};

__device__ __forceinline__ void stage_targets(SpreadSmem& sm, int buf, int e, int e1,
                                              const int* __restrict__ patch_t, const int* __restrict__ r0,
                                              const int* __restrict__ c0, const float* __restrict__ w1,
                                              const float* __restrict__ w2, const float2* __restrict__ val,
                                              int lane) {
  if (e + lane < e1) {
    const int t = patch_t[e + lane];
    sm.r0[buf][lane] = r0[t];
    sm.c0[buf][lane] = c0[t];
    const float4* a = reinterpret_cast<const float4*>(w1 + static_cast<long long>(t) * kTaps);
    const float4* b = reinterpret_cast<const float4*>(w2 + static_cast<long long>(t) * kTaps);
    const float4* v = reinterpret_cast<const float4*>(val + static_cast<long long>(t) * KB);
#pragma unroll
    for (int q = 0; q < kTaps / 4; ++q) {
      cp_async16(&sm.w1[buf][lane][4 * q], a + q);
      cp_async16(&sm.w2[buf][lane][4 * q], b + q);
    }
#pragma unroll
    for (int q = 0; q < KB / 2; ++q) cp_async16(&sm.val[buf][lane][q], v + q);
  }
  cp_async_commit();
}

// A work item is (patch, a sub-range of its target list): lists longer than
// kSplit (the cells around nu = 0) are split over several warps whose double
// partials are summed in item order by k_fu2d_adj_spread_reduce.
struct SpreadItem {
  int patch, e0, e1, slot;  // slot < 0: write the grid directly
};
constexpr int kSplit = 256;

__global__ void __launch_bounds__(32 * kGroupWarps) k_fu2d_adj_spread_warp(
    const float2* __restrict__ val, int logm1, int logm2, int nitems, const SpreadItem* __restrict__ items,
    const int* __restrict__ patch_t, const int* __restrict__ r0, const int* __restrict__ c0,
    const float* __restrict__ w1, const float* __restrict__ w2, float2* __restrict__ G,
    double2* __restrict__ partial) {
  extern __shared__ float4 dyn_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SpreadSmem& sm = reinterpret_cast<SpreadSmem*>(dyn_smem)[warp];
  const int pi = blockIdx.x * kGroupWarps + warp;
  if (pi >= nitems) return;
  const int m2 = 1 << logm2, mask1 = (1 << logm1) - 1, mask2 = m2 - 1;
  const SpreadItem it = items[pi];
  const int patch = it.patch;
  const int npc = m2 / kPatchC;
  const int r = (patch / npc) * kPatchR + lane / kPatchC, c = (patch % npc) * kPatchC + lane % kPatchC;
  double2 acc[KB];
#pragma unroll
  for (int kk = 0; kk < KB; ++kk) acc[kk] = make_double2(0.0, 0.0);
  const int e0 = it.e0, e1 = it.e1;
  if (e0 < e1) stage_targets(sm, 0, e0, e1, patch_t, r0, c0, w1, w2, val, lane);
  for (int e = e0, chunk = 0; e < e1; e += 32, ++chunk) {
    const int buf = chunk & 1;
    if (e + 32 < e1) {
      stage_targets(sm, buf ^ 1, e + 32, e1, patch_t, r0, c0, w1, w2, val, lane);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const int n = min(32, e1 - e);
    for (int idx = lane; idx < n * (KB / 2); idx += 32) {  // widen once per warp
      const int j = idx / (KB / 2), part = idx - j * (KB / 2);
      const float4 x = sm.val[buf][j][part];
      sm.vald[j][2 * part] = make_double2(x.x, x.y);
      sm.vald[j][2 * part + 1] = make_double2(x.z, x.w);
    }
    __syncwarp();
    for (int j = 0; j < n; ++j) {
      const int a = (r - sm.r0[buf][j]) & mask1, b = (c - sm.c0[buf][j]) & mask2;
      const double wgt = (a < kTaps && b < kTaps) ? static_cast<double>(sm.w1[buf][j][min(a, kTaps - 1)]) *
                                                        static_cast<double>(sm.w2[buf][j][min(b, kTaps - 1)])
                                                  : 0.0;
      const double2* vp = sm.vald[j];
#pragma unroll
      for (int kk = 0; kk < KB; ++kk) {
        const double2 x = vp[kk];
        acc[kk].x = fma(wgt, x.x, acc[kk].x);
        acc[kk].y = fma(wgt, x.y, acc[kk].y);
      }
    }
    __syncwarp();  // this buffer is refilled by the prefetch two chunks ahead
  }
  if (it.slot >= 0) {
    double2* pp = partial + (static_cast<long long>(it.slot) * 32 + lane) * KB;
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) pp[kk] = acc[kk];
    return;
  }
  float4* gp = reinterpret_cast<float4*>(G + (static_cast<long long>(r) * m2 + c) * KB);
#pragma unroll
  for (int q = 0; q < KB / 2; ++q) {
    const float2 lo = to_f(acc[2 * q]), hi = to_f(acc[2 * q + 1]);
    gp[q] = make_float4(lo.x, lo.y, hi.x, hi.y);
  }
}

// Sums the split patches' partials in item order (deterministic) into the grid.
__global__ void __launch_bounds__(32 * kGroupWarps) k_fu2d_adj_spread_reduce(
    int nsplit, const int4* __restrict__ split, int logm2, const double2* __restrict__ partial,
    float2* __restrict__ G) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int si = blockIdx.x * kGroupWarps + warp;
  if (si >= nsplit) return;
  const int4 sp = split[si];  // (patch, first slot, slot count, -)
  const int m2 = 1 << logm2, npc = m2 / kPatchC;
  const int r = (sp.x / npc) * kPatchR + lane / kPatchC, c = (sp.x % npc) * kPatchC + lane % kPatchC;
  float2* gp = G + (static_cast<long long>(r) * m2 + c) * KB;
#pragma unroll
  for (int kk = 0; kk < KB; ++kk) {
    double2 a = make_double2(0.0, 0.0);
    for (int q = 0; q < sp.z; ++q) a = cadd(a, partial[(static_cast<long long>(sp.y + q) * 32 + lane) * KB + kk]);
    gp[kk] = to_f(a);
  }
}

// ------------------------------------------------------------------------------------------
// fu2d adjoint: prep, column pass, row pass (the spread is above)
// ------------------------------------------------------------------------------------------
// val[t][KB] = p[t_, k0+kk, q_] * conj(phase product), zero for kk >= nk.
__global__ void __launch_bounds__(256) k_fu2d_adj_prep(const float2* __restrict__ p, long long ld, long long k0,
                                                       int nk, int T, int w, const double2* __restrict__ cfac,
                                                       float2* __restrict__ val) {
  __shared__ float2 tile[32][KB + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
  const int t = blockIdx.x * 32 + tx;
  for (int kk = ty; kk < KB; kk += 8) {
    float2 x = make_float2(0.f, 0.f);
    if (t < T && kk < nk) {
      const int ta = t / w, q = t - ta * w;
      x = to_f(cmul(to_d(p[(ta * ld + k0 + kk) * w + q]), cfac[t]));
    }
    tile[tx][kk] = x;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * KB; e += blockDim.x) {
    const int tt = e / KB, kk = e - tt * KB;
    const long long tg = static_cast<long long>(blockIdx.x) * 32 + tt;
    if (tg < T) val[tg * KB + kk] = tile[tt][kk];
  }
}

// Column FFT(-1) over natural rows; keep only the n1 rows that map to modes.
__global__ void __launch_bounds__(256) k_fu2d_adj_cols(const float2* __restrict__ G, int n1, int logm1, int center1,
                                                       int logm2, int ks_n, const double2* __restrict__ tw1,
                                                       float2* __restrict__ S) {
  extern __shared__ double2 sd[];
  const int m1 = 1 << logm1, mask1 = m1 - 1, m2 = 1 << logm2;
  const int c = blockIdx.x, ks = blockIdx.y * ks_n;
  for (int idx = threadIdx.x; idx < m1 * ks_n; idx += blockDim.x) {
    const int r = idx / ks_n, kk = idx - r * ks_n;
    sd[idx] = to_d(G[(static_cast<long long>(r) * m2 + c) * KB + ks + kk]);
  }
  __syncthreads();
  fft_dif<-1>(sd, logm1, ks_n, ks_n, tw1);
  for (int idx = threadIdx.x; idx < n1 * ks_n; idx += blockDim.x) {
    const int i = idx / ks_n, kk = idx - i * ks_n;
    const int slot = (i - center1) & mask1;
    S[(static_cast<long long>(i) * m2 + c) * KB + ks + kk] = to_f(sd[brev(slot, logm1) * ks_n + kk]);
  }
}

// Row FFT(-1) (DIT from bit-reversed placement, natural output) and the
// final deconvolution into out[i, k0_out+kk, j].
__global__ void __launch_bounds__(256) k_fu2d_adj_rows(const float2* __restrict__ S, int nk, int n2, int logm2,
                                                       int center2, int ks_n, const double* __restrict__ pdx,
                                                       const double* __restrict__ dy, const double2* __restrict__ tw2,
                                                       float2* __restrict__ out, long long ld_out,
                                                       long long k0_out) {
  extern __shared__ double2 sd[];
  const int m2 = 1 << logm2, mask2 = m2 - 1, sm = ks_n + 1;
  const int i = blockIdx.x, ks = blockIdx.y * ks_n;
  const float2* Si = S + static_cast<long long>(i) * m2 * KB + ks;
  for (int idx = threadIdx.x; idx < m2 * ks_n; idx += blockDim.x) {
    const int c = idx / ks_n, kk = idx - c * ks_n;
    sd[brev(c, logm2) * sm + kk] = to_d(Si[static_cast<long long>(c) * KB + kk]);
  }
  __syncthreads();
  fft_dit<-1>(sd, logm2, ks_n, sm, tw2);
  const double pi = pdx[i];
  for (int idx = threadIdx.x; idx < ks_n * n2; idx += blockDim.x) {
    const int kk = idx / n2, j = idx - kk * n2;
    if (ks + kk >= nk) continue;
    const int slot = (j - center2) & mask2;
    out[(static_cast<long long>(i) * ld_out + k0_out + ks + kk) * n2 + j] = to_f(cscale(sd[slot * sm + kk], pi * dy[j]));
  }
}

// ------------------------------------------------------------------------------------------
// f2d: centred unitary 2D DFT. Power-of-two planes use two FFT passes with the
// (-1)^(k+m+N/2) checkerboard; other sizes fall back to dense DFT passes with
// the host-built centred matrix (both on the device).
// ------------------------------------------------------------------------------------------
// FFT along the contiguous axis of `rows` rows of length m (one CTA per ncol rows).
template <int SIGN>
__global__ void __launch_bounds__(256) k_center_fft_rows(const float2* __restrict__ in, float2* __restrict__ out,
                                                         long long rows, int logm, int ncol, double scale,
                                                         const double2* __restrict__ tw) {
  extern __shared__ double2 sd[];
  const int m = 1 << logm, sm = ncol + 1;
  const long long r0 = static_cast<long long>(blockIdx.x) * ncol;
  for (int idx = threadIdx.x; idx < m * ncol; idx += blockDim.x) {
    const int c = idx / m, n = idx - c * m;
    double2 x = make_double2(0.0, 0.0);
    if (r0 + c < rows) {
      x = to_d(in[(r0 + c) * m + n]);
      if (n & 1) x = make_double2(-x.x, -x.y);
    }
    sd[n * sm + c] = x;
  }
  __syncthreads();
  fft_dif<SIGN>(sd, logm, ncol, sm, tw);
  for (int idx = threadIdx.x; idx < m * ncol; idx += blockDim.x) {
    const int c = idx / m, k = idx - c * m;
    if (r0 + c >= rows) continue;
    const double sg = ((k + (m >> 1)) & 1) ? -scale : scale;
    out[(r0 + c) * m + k] = to_f(cscale(sd[brev(k, logm) * sm + c], sg));
  }
}

// FFT along the middle axis of [outer][m][inner] (one CTA per outer x ncol inner).
template <int SIGN>
__global__ void __launch_bounds__(256) k_center_fft_cols(const float2* in, float2* out, int inner, int logm, int ncol,
                                                         double scale, const double2* __restrict__ tw) {
  extern __shared__ double2 sd[];
  const int m = 1 << logm;
  const long long o = blockIdx.y;
  const int c0 = blockIdx.x * ncol;
  const float2* io = in + o * m * inner;
  for (int idx = threadIdx.x; idx < m * ncol; idx += blockDim.x) {
    const int n = idx / ncol, c = idx - n * ncol;
    double2 x = make_double2(0.0, 0.0);
    if (c0 + c < inner) {
      x = to_d(io[static_cast<long long>(n) * inner + c0 + c]);
      if (n & 1) x = make_double2(-x.x, -x.y);
    }
    sd[idx] = x;
  }
  __syncthreads();
  fft_dif<SIGN>(sd, logm, ncol, ncol, tw);
  float2* oo = out + o * m * inner;
  for (int idx = threadIdx.x; idx < m * ncol; idx += blockDim.x) {
    const int k = idx / ncol, c = idx - k * ncol;
    if (c0 + c >= inner) continue;
    const double sg = ((k + (m >> 1)) & 1) ? -scale : scale;
    oo[static_cast<long long>(k) * inner + c0 + c] = to_f(cscale(sd[brev(k, logm) * ncol + c], sg));
  }
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

std::vector<double2> twiddles(std::int64_t m) {
  std::vector<double2> t(static_cast<std::size_t>(std::max<std::int64_t>(m / 2, 1)));
  for (std::int64_t k = 0; k < m / 2; ++k) {
    const double a = 2.0 * std::numbers::pi * static_cast<double>(k) / static_cast<double>(m);
    t[static_cast<std::size_t>(k)] = make_double2(std::cos(a), std::sin(a));
  }
  return t;
}

bool is_pow2(std::int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
int ilog2(std::int64_t n) {
  int l = 0;
  while ((std::int64_t{1} << l) < n) ++l;
  return l;
}

std::vector<float> to_float(const std::vector<double>& v) { return {v.begin(), v.end()}; }

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
  int z_ncol = 0;
  DeviceBuffer<double> z_deconv, z_pdeconv;
  DeviceBuffer<float> z_w, z_cell_w;
  DeviceBuffer<int> z_start, z_cell_ptr, z_cell_k;
  DeviceBuffer<double2> z_fac, z_cphase, z_tw;
  // fu2d
  DimPlan px, py;
  DeviceBuffer<double> x_deconv, x_pdeconv, y_deconv;
  DeviceBuffer<float> t_w1, t_w2;
  DeviceBuffer<int> t_r0, t_c0;
  DeviceBuffer<double2> t_fac, t_cfac, x_tw, y_tw;
  DeviceBuffer<float2> S, Gd, val;  // scratch: row pass, grid, adjoint values
  // warp-cooperative gather: Morton-sorted target groups
  int ngroups = 0;
  DeviceBuffer<GatherGroup> groups;
  DeviceBuffer<int> g_tidx, g_dr, g_dc;
  DeviceBuffer<float> g_w1, g_w2;
  DeviceBuffer<double2> g_fac;
  // warp-cooperative spread: 8x4 cell patches -> targets, heaviest patch first
  int nitems = 0, nsplit = 0;
  DeviceBuffer<int> patch_t;
  DeviceBuffer<SpreadItem> items;
  DeviceBuffer<int4> split;
  DeviceBuffer<double2> partial;
  // f2d
  bool f2d_fft = false;
  DeviceBuffer<double2> h_tw, w_tw, Wh, Ww, Whc, Wwc;
  DeviceBuffer<float2> f2d_tmp;
};

Usfft::Usfft(const Geometry& g, cudaStream_t stream) : g_(g), stream_(stream), t_(new Tables) {
  Tables& t = *t_;
  const FrequencyGrids fg = frequency_grids(g_);
  // ---- fu1d plan (nufft.cpp:109-110) ----
  t.pz = DimPlan::make(g_.n0, fg.nu_z);
  const DimPlan& pz = t.pz;
  t.z_ncol = static_cast<int>(std::clamp<std::int64_t>(4096 / pz.m, 1, 64));
  t.z_ncol = static_cast<int>(std::min<std::int64_t>(t.z_ncol, g_.n2));
  t.z_deconv.upload(pz.deconv, stream_);
  std::vector<double> pdec(pz.deconv.size());
  for (std::size_t i = 0; i < pdec.size(); ++i) pdec[i] = pz.pref * pz.deconv[i];
  t.z_pdeconv.upload(pdec, stream_);
  t.z_start.upload(std::vector<int>(pz.start.begin(), pz.start.end()), stream_);
  t.z_w.upload(to_float(pz.weights), stream_);
  std::vector<double2> fac(static_cast<std::size_t>(g_.h)), cph(static_cast<std::size_t>(g_.h));
  for (std::size_t k = 0; k < fac.size(); ++k) {
    fac[k] = make_double2(pz.pref * pz.phase_re[k], pz.pref * pz.phase_im[k]);
    cph[k] = make_double2(pz.phase_re[k], -pz.phase_im[k]);
  }
  t.z_fac.upload(fac, stream_);
  t.z_cphase.upload(cph, stream_);
  {  // cell -> (target, weight) CSR for the scatter-free adjoint, targets ascending
    std::vector<int> cnt(static_cast<std::size_t>(pz.m + 1), 0);
    for (std::int64_t k = 0; k < g_.h; ++k)
      for (int a = 0; a < kTaps; ++a) cnt[static_cast<std::size_t>((pz.start[k] + a) % pz.m) + 1]++;
    for (std::size_t l = 1; l < cnt.size(); ++l) cnt[l] += cnt[l - 1];
    std::vector<int> ck(static_cast<std::size_t>(cnt.back())), pos(cnt.begin(), cnt.end() - 1);
    std::vector<float> cw(ck.size());
    for (std::int64_t k = 0; k < g_.h; ++k)
      for (int a = 0; a < kTaps; ++a) {
        const std::size_t l = static_cast<std::size_t>((pz.start[k] + a) % pz.m);
        ck[static_cast<std::size_t>(pos[l])] = static_cast<int>(k);
        cw[static_cast<std::size_t>(pos[l]++)] = static_cast<float>(pz.weights[k * kTaps + a]);
      }
    t.z_cell_ptr.upload(cnt, stream_);
    t.z_cell_k.upload(ck, stream_);
    t.z_cell_w.upload(cw, stream_);
  }
  t.z_tw.upload(twiddles(pz.m), stream_);

  // ---- fu2d plans (nufft.cpp:185-187) ----
  t.px = DimPlan::make(g_.n1, fg.nu_x);
  t.py = DimPlan::make(g_.n2, fg.nu_y);
  const DimPlan &px = t.px, &py = t.py;
  const std::size_t T = fg.nu_x.size();
  t.x_deconv.upload(px.deconv, stream_);
  t.y_deconv.upload(py.deconv, stream_);
  std::vector<double> pdx(px.deconv.size());
  for (std::size_t i = 0; i < pdx.size(); ++i) pdx[i] = px.pref * py.pref * px.deconv[i];
  t.x_pdeconv.upload(pdx, stream_);
  t.t_r0.upload(std::vector<int>(px.start.begin(), px.start.end()), stream_);
  t.t_c0.upload(std::vector<int>(py.start.begin(), py.start.end()), stream_);
  const std::vector<float> w1f = to_float(px.weights), w2f = to_float(py.weights);
  t.t_w1.upload(w1f, stream_);
  t.t_w2.upload(w2f, stream_);
  std::vector<double2> tf(T), tcf(T);
  for (std::size_t q = 0; q < T; ++q) {
    const std::complex<double> ph = std::complex<double>(px.phase_re[q], px.phase_im[q]) *
                                    std::complex<double>(py.phase_re[q], py.phase_im[q]);
    const std::complex<double> f = (px.pref * py.pref) * ph;
    tf[q] = make_double2(f.real(), f.imag());
    tcf[q] = make_double2(ph.real(), -ph.imag());
  }
  t.t_fac.upload(tf, stream_);
  t.t_cfac.upload(tcf, stream_);
  {  // gather groups: <= 32 targets from one kBox x kBox bin of window origins
    std::vector<int> order(T);
    for (std::size_t q = 0; q < T; ++q) order[q] = static_cast<int>(q);
    // fixed kBox x kBox bins of the window origin (2.6M vs 3.3M union cells per
    // 256^3 launch compared with Morton runs), row-major inside a bin
    std::vector<std::uint64_t> key(T);
    for (std::size_t q = 0; q < T; ++q) {
      const std::uint64_t r = static_cast<std::uint64_t>(px.start[q]), c = static_cast<std::uint64_t>(py.start[q]);
      key[q] = ((r / kBox) << 48) | ((c / kBox) << 32) | (r << 16) | c;
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key[static_cast<std::size_t>(a)] < key[static_cast<std::size_t>(b)]; });
    std::vector<GatherGroup> grp;
    std::vector<int> tidx(T), dr(T), dc(T);
    std::vector<float> gw1(T * kTaps), gw2(T * kTaps);
    std::vector<double2> gfac(T);
    std::size_t i = 0;
    while (i < T) {
      const std::size_t first = i;
      int rmin = px.start[static_cast<std::size_t>(order[i])], rmax = rmin;
      int cmin = py.start[static_cast<std::size_t>(order[i])], cmax = cmin;
      ++i;
      while (i < T && i - first < 32) {
        const int r = px.start[static_cast<std::size_t>(order[i])], c = py.start[static_cast<std::size_t>(order[i])];
        if ((key[static_cast<std::size_t>(order[i])] >> 32) != (key[static_cast<std::size_t>(order[first])] >> 32)) break;
        if (std::max(rmax, r) - std::min(rmin, r) > kBox || std::max(cmax, c) - std::min(cmin, c) > kBox) break;
        rmin = std::min(rmin, r), rmax = std::max(rmax, r), cmin = std::min(cmin, c), cmax = std::max(cmax, c);
        ++i;
      }
      grp.push_back(GatherGroup{static_cast<int>(first), static_cast<int>(i - first), rmin, cmin,
                                rmax - rmin + kTaps, cmax - cmin + kTaps});
      for (std::size_t s = first; s < i; ++s) {
        const std::size_t q = static_cast<std::size_t>(order[s]);
        tidx[s] = static_cast<int>(q);
        dr[s] = px.start[q] - rmin;
        dc[s] = py.start[q] - cmin;
        std::copy_n(w1f.begin() + static_cast<std::ptrdiff_t>(q * kTaps), kTaps,
                    gw1.begin() + static_cast<std::ptrdiff_t>(s * kTaps));
        std::copy_n(w2f.begin() + static_cast<std::ptrdiff_t>(q * kTaps), kTaps,
                    gw2.begin() + static_cast<std::ptrdiff_t>(s * kTaps));
        gfac[s] = tf[q];
      }
    }
    t.ngroups = static_cast<int>(grp.size());
    t.groups.upload(grp, stream_);
    t.g_tidx.upload(tidx, stream_);
    t.g_dr.upload(dr, stream_);
    t.g_dc.upload(dc, stream_);
    t.g_w1.upload(gw1, stream_);
    t.g_w2.upload(gw2, stream_);
    t.g_fac.upload(gfac, stream_);
  }
  {  // spread patches: 8x4 cells -> targets whose 24x24 window touches them (targets ascending)
    const std::int64_t npr = px.m / kPatchR, npc = py.m / kPatchC;
    const int npatch = static_cast<int>(npr * npc);
    auto cover = [&](std::int32_t st, std::int64_t m, int edge, int* out) {
      int n = 0;
      for (int a = 0; a < kTaps; ++a) {
        const int p = static_cast<int>(((st + a) % m) / edge);
        bool seen = false;
        for (int e = 0; e < n; ++e) seen |= out[e] == p;
        if (!seen) out[n++] = p;
      }
      return n;
    };
    std::vector<int> cnt(static_cast<std::size_t>(npatch + 1), 0), lst;
    int pr[kTaps], pc[kTaps];
    for (int pass = 0; pass < 2; ++pass) {
      std::vector<int> pos;
      if (pass == 1) {
        for (std::size_t l = 1; l < cnt.size(); ++l) cnt[l] += cnt[l - 1];
        pos.assign(cnt.begin(), cnt.end() - 1);
        lst.resize(static_cast<std::size_t>(cnt.back()));
      }
      for (std::size_t q = 0; q < T; ++q) {
        const int nr = cover(px.start[q], px.m, kPatchR, pr), nc = cover(py.start[q], py.m, kPatchC, pc);
        for (int a = 0; a < nr; ++a)
          for (int b = 0; b < nc; ++b) {
            const std::size_t p = static_cast<std::size_t>(pr[a] * npc + pc[b]);
            if (pass == 0) cnt[p + 1]++;
            else lst[static_cast<std::size_t>(pos[p]++)] = static_cast<int>(q);
          }
      }
    }
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
        items.push_back(SpreadItem{p, e0, e1, -1});
        continue;
      }
      const int first = slots;
      for (int e = e0; e < e1; e += kSplit) items.push_back(SpreadItem{p, e, std::min(e1, e + kSplit), slots++});
      split.push_back(make_int4(p, first, slots - first, 0));
    }
    t.nitems = static_cast<int>(items.size());
    t.nsplit = static_cast<int>(split.size());
    t.items.upload(items, stream_);
    t.split.upload(split, stream_);
    t.partial.resize(static_cast<std::size_t>(std::max(slots, 1)) * 32 * KB);
    t.patch_t.upload(lst, stream_);
  }
  t.x_tw.upload(twiddles(px.m), stream_);
  t.y_tw.upload(twiddles(py.m), stream_);
  t.S.resize(static_cast<std::size_t>(px.m * py.m * KB));
  t.Gd.resize(static_cast<std::size_t>(px.m * py.m * KB));
  t.val.resize(T * KB);

  // ---- f2d (operators.cpp:20-74) ----
  t.f2d_fft = is_pow2(g_.h) && is_pow2(g_.w) && g_.h >= 4 && g_.w >= 4;
  if (t.f2d_fft) {
    t.h_tw.upload(twiddles(g_.h), stream_);
    t.w_tw.upload(twiddles(g_.w), stream_);
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
    t.Wh.upload(mat(g_.h, false), stream_);
    t.Ww.upload(mat(g_.w, false), stream_);
    t.Whc.upload(mat(g_.h, true), stream_);
    t.Wwc.upload(mat(g_.w, true), stream_);
  }
  MLRG_CUDA(cudaStreamSynchronize(stream_));
  static bool smem_set = [] {
    allow_big_smem(k_fu1d<float2>);
    allow_big_smem(k_fu1d<double2>);
    allow_big_smem(k_fu1d_adj<float2>);
    allow_big_smem(k_fu1d_adj<double2>);
    allow_big_smem(k_fu2d_rows);
    allow_big_smem(k_fu2d_gather_warp);
    allow_big_smem(k_fu2d_adj_spread_warp);
    allow_big_smem(k_fu2d_cols);
    allow_big_smem(k_fu2d_adj_cols);
    allow_big_smem(k_fu2d_adj_rows);
    allow_big_smem(k_center_fft_rows<+1>);
    allow_big_smem(k_center_fft_rows<-1>);
    allow_big_smem(k_center_fft_cols<+1>);
    allow_big_smem(k_center_fft_cols<-1>);
    return true;
  }();
  (void)smem_set;
}

Usfft::~Usfft() { delete t_; }

int Usfft::reduce_grid() const { return 4 * sm_count(); }

template <class TIn>
void Usfft::fu1d_t(const TIn* u, float2* out, std::int64_t d0) {
  if (d0 <= 0) return;
  const Tables& t = *t_;
  const int ncol = t.z_ncol;
  const dim3 grid(static_cast<unsigned>((g_.n2 + ncol - 1) / ncol), static_cast<unsigned>(d0));
  const std::size_t smem = static_cast<std::size_t>(t.pz.m * ncol) * sizeof(double2);
  prof::begin("k_fu1d", stream_);
  k_fu1d<TIn><<<grid, 256, smem, stream_>>>(u, out, static_cast<int>(g_.n0), static_cast<int>(g_.n2),
                                            static_cast<int>(g_.h), t.pz.logm, static_cast<int>(t.pz.center), ncol,
                                            t.z_deconv.get(), t.z_start.get(), t.z_w.get(), t.z_fac.get(),
                                            t.z_tw.get());
  MLRG_LAUNCH_CHECK("k_fu1d");
  prof::end("k_fu1d", stream_);
}

template <class TOut>
void Usfft::fu1d_adj_t(const float2* v, TOut* out, std::int64_t d0) {
  if (d0 <= 0) return;
  const Tables& t = *t_;
  const int ncol = t.z_ncol;
  const dim3 grid(static_cast<unsigned>((g_.n2 + ncol - 1) / ncol), static_cast<unsigned>(d0));
  const std::size_t smem = static_cast<std::size_t>((t.pz.m + g_.h) * ncol) * sizeof(double2);
  prof::begin("k_fu1d_adj", stream_);
  k_fu1d_adj<TOut><<<grid, 256, smem, stream_>>>(v, out, static_cast<int>(g_.n0), static_cast<int>(g_.n2),
                                                 static_cast<int>(g_.h), t.pz.logm, static_cast<int>(t.pz.center),
                                                 ncol, t.z_cphase.get(), t.z_cell_ptr.get(), t.z_cell_k.get(),
                                                 t.z_cell_w.get(), t.z_pdeconv.get(), t.z_tw.get());
  MLRG_LAUNCH_CHECK("k_fu1d_adj");
  prof::end("k_fu1d_adj", stream_);
}

void Usfft::fu1d(const float2* u, float2* out, std::int64_t d0) { fu1d_t(u, out, d0); }
void Usfft::fu1d(const double2* u, float2* out, std::int64_t d0) { fu1d_t(u, out, d0); }
void Usfft::fu1d_adj(const float2* v, float2* out, std::int64_t d0) { fu1d_adj_t(v, out, d0); }
void Usfft::fu1d_adj(const float2* v, double2* out, std::int64_t d0) { fu1d_adj_t(v, out, d0); }

int Usfft::fu2d(const float2* v, std::int64_t ld, std::int64_t k0, std::int64_t nk, const Fu2dEpilogue& epi) {
  const Tables& t = *t_;
  const std::int64_t T = g_.n_theta * g_.w;
  const int ks1 = pass_cols(t.px.m), ks2 = pass_cols(t.py.m);
  const int ggrid = (t.ngroups + kGroupWarps - 1) / kGroupWarps;
  for (std::int64_t b = 0; b < nk; b += KB) {
    const int nb = static_cast<int>(std::min<std::int64_t>(KB, nk - b));
    prof::begin("k_fu2d_rows", stream_);
    k_fu2d_rows<<<dim3(static_cast<unsigned>(g_.n1), KB / ks2), 256,
                  static_cast<std::size_t>(t.py.m * (ks2 + 1)) * sizeof(double2), stream_>>>(
        v, ld, k0 + b, nb, static_cast<int>(g_.n2), t.py.logm, static_cast<int>(t.py.center), ks2, t.x_deconv.get(),
        t.y_deconv.get(), t.y_tw.get(), t.S.get());
    MLRG_LAUNCH_CHECK("k_fu2d_rows");
    prof::end("k_fu2d_rows", stream_);
    prof::begin("k_fu2d_cols", stream_);
    k_fu2d_cols<<<dim3(static_cast<unsigned>(t.py.m), KB / ks1), 256,
                  static_cast<std::size_t>(t.px.m * ks1) * sizeof(double2), stream_>>>(
        t.S.get(), static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center), t.py.logm, ks1, t.x_tw.get(),
        t.Gd.get());
    MLRG_LAUNCH_CHECK("k_fu2d_cols");
    prof::end("k_fu2d_cols", stream_);
    GatherOut eo{epi.out, epi.ld_out, epi.k0_out + b, epi.sub, epi.ld_sub, epi.k0_sub + b,
                 epi.dot, epi.ld_dot, epi.k0_dot + b, epi.reduce ? 1 : 0};
    prof::begin("k_fu2d_gather", stream_);
    k_fu2d_gather_warp<<<ggrid, 32 * kGroupWarps, kGroupWarps * sizeof(GatherSmem), stream_>>>(
        t.Gd.get(), t.ngroups, t.groups.get(), static_cast<int>(g_.w), t.px.logm, t.py.logm, nb, t.g_tidx.get(),
        t.g_dr.get(), t.g_dc.get(), t.g_w1.get(), t.g_w2.get(), t.g_fac.get(), eo, partials_.dev(), b > 0 ? 1 : 0);
    MLRG_LAUNCH_CHECK("k_fu2d_gather");
    prof::end("k_fu2d_gather", stream_);
  }
  return epi.reduce && nk > 0 ? 2 * ggrid : 0;
}

void Usfft::fu2d_adj(const float2* p, std::int64_t ld, std::int64_t k0, std::int64_t nk, float2* out,
                     std::int64_t ld_out, std::int64_t k0_out) {
  const Tables& t = *t_;
  const std::int64_t T = g_.n_theta * g_.w;
  const int ks1 = pass_cols(t.px.m), ks2 = pass_cols(t.py.m);
  for (std::int64_t b = 0; b < nk; b += KB) {
    const int nb = static_cast<int>(std::min<std::int64_t>(KB, nk - b));
    prof::begin("k_fu2d_adj_prep", stream_);
    k_fu2d_adj_prep<<<static_cast<unsigned>((T + 31) / 32), 256, 0, stream_>>>(
        p, ld, k0 + b, nb, static_cast<int>(T), static_cast<int>(g_.w), t.t_cfac.get(), t.val.get());
    MLRG_LAUNCH_CHECK("k_fu2d_adj_prep");
    prof::end("k_fu2d_adj_prep", stream_);
    prof::begin("k_fu2d_adj_spread", stream_);
    k_fu2d_adj_spread_warp<<<(t.nitems + kGroupWarps - 1) / kGroupWarps, 32 * kGroupWarps,
                             kGroupWarps * sizeof(SpreadSmem), stream_>>>(
        t.val.get(), t.px.logm, t.py.logm, t.nitems, t.items.get(), t.patch_t.get(), t.t_r0.get(), t.t_c0.get(),
        t.t_w1.get(), t.t_w2.get(), t.Gd.get(), t.partial.get());
    MLRG_LAUNCH_CHECK("k_fu2d_adj_spread");
    if (t.nsplit > 0) {
      k_fu2d_adj_spread_reduce<<<(t.nsplit + kGroupWarps - 1) / kGroupWarps, 32 * kGroupWarps, 0, stream_>>>(
          t.nsplit, t.split.get(), t.py.logm, t.partial.get(), t.Gd.get());
      MLRG_LAUNCH_CHECK("k_fu2d_adj_spread_reduce");
    }
    prof::end("k_fu2d_adj_spread", stream_);
    prof::begin("k_fu2d_adj_cols", stream_);
    k_fu2d_adj_cols<<<dim3(static_cast<unsigned>(t.py.m), KB / ks1), 256,
                      static_cast<std::size_t>(t.px.m * ks1) * sizeof(double2), stream_>>>(
        t.Gd.get(), static_cast<int>(g_.n1), t.px.logm, static_cast<int>(t.px.center), t.py.logm, ks1,
        t.x_tw.get(), t.S.get());
    MLRG_LAUNCH_CHECK("k_fu2d_adj_cols");
    prof::end("k_fu2d_adj_cols", stream_);
    prof::begin("k_fu2d_adj_rows", stream_);
    k_fu2d_adj_rows<<<dim3(static_cast<unsigned>(g_.n1), KB / ks2), 256,
                      static_cast<std::size_t>(t.py.m * (ks2 + 1)) * sizeof(double2), stream_>>>(
        t.S.get(), nb, static_cast<int>(g_.n2), t.py.logm, static_cast<int>(t.py.center), ks2, t.x_pdeconv.get(),
        t.y_deconv.get(), t.y_tw.get(), out, ld_out, k0_out + b);
    MLRG_LAUNCH_CHECK("k_fu2d_adj_rows");
    prof::end("k_fu2d_adj_rows", stream_);
  }
}

void Usfft::f2d(const float2* p, float2* out, std::int64_t count, bool adjoint) {
  if (count <= 0) return;
  Tables& t = *t_;
  const std::int64_t h = g_.h, w = g_.w;
  if (t.f2d_fft) {
    // rows (along w) into out, then columns (along h) in place
    const int lw = ilog2(w), lh = ilog2(h);
    const int ncr = static_cast<int>(std::clamp<std::int64_t>(4096 / w, 1, 64));
    const std::int64_t rows = count * h;
    const std::size_t smr = static_cast<std::size_t>(w * (ncr + 1)) * sizeof(double2);
    const double sw = 1.0 / std::sqrt(static_cast<double>(w)), sh = 1.0 / std::sqrt(static_cast<double>(h));
    const unsigned gr = static_cast<unsigned>((rows + ncr - 1) / ncr);
    if (adjoint) k_center_fft_rows<+1><<<gr, 256, smr, stream_>>>(p, out, rows, lw, ncr, sw, t.w_tw.get());
    else k_center_fft_rows<-1><<<gr, 256, smr, stream_>>>(p, out, rows, lw, ncr, sw, t.w_tw.get());
    MLRG_LAUNCH_CHECK("k_center_fft_rows");
    const int ncc = static_cast<int>(std::clamp<std::int64_t>(4096 / h, 1, std::min<std::int64_t>(64, w)));
    const dim3 gc(static_cast<unsigned>((w + ncc - 1) / ncc), static_cast<unsigned>(count));
    const std::size_t smc = static_cast<std::size_t>(h * ncc) * sizeof(double2);
    if (adjoint)
      k_center_fft_cols<+1><<<gc, 256, smc, stream_>>>(out, out, static_cast<int>(w), lh, ncc, sh, t.h_tw.get());
    else
      k_center_fft_cols<-1><<<gc, 256, smc, stream_>>>(out, out, static_cast<int>(w), lh, ncc, sh, t.h_tw.get());
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
