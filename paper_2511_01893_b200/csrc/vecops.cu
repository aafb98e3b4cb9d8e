// Fused, HBM-bound ADMM kernels (admm.cpp:59-195 restated on the device).
// Each stencil kernel walks rows (i, m) of the (n1, n0, n2) volume with the
// threads of a CTA along j, recomputes grad(u) - g from u and g where the
// reference materialises GradFields, and reduces in double per CTA. The
// volume-side state is complex128 (see kernels.hpp).
#include <cmath>

#include "common.cuh"
#include "device.hpp"
#include "kernels.hpp"

namespace mlrg::ops {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double2 dadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 dsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 dscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 dfma(double s, double2 x, double2 y) {  // s*x + y
  return make_double2(fma(s, x.x, y.x), fma(s, x.y, y.y));
}
__device__ __forceinline__ double dnrm(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double dredot(double2 a, double2 b) { return a.x * b.x + a.y * b.y; }  // Re(a conj b)
__device__ __forceinline__ double fnrm(float2 a) {
  return static_cast<double>(a.x) * a.x + static_cast<double>(a.y) * a.y;
}
__device__ __forceinline__ double2 zero2() { return make_double2(0.0, 0.0); }

int row_bx(std::int64_t n2) {
  int bx = 32;
  while (bx < 256 && bx < n2) bx <<= 1;
  return bx;
}

int grid_blocks() { return 4 * sm_count(); }

struct DevDims {
  int n1, n0, n2, bx;
  long long s0, s1;  // strides of axes 0 and 1
};

DevDims dev_dims(Dims d) {
  return {static_cast<int>(d.n1), static_cast<int>(d.n0), static_cast<int>(d.n2), row_bx(d.n2), d.n0 * d.n2, d.n2};
}

// Iterates every voxel; `body(idx, i, m, j)` per voxel.
template <class F>
__device__ __forceinline__ void for_voxels(const DevDims& d, F&& body) {
  const int tx = threadIdx.x % d.bx, ty = threadIdx.x / d.bx, rows_per = blockDim.x / d.bx;
  const long long nrows = static_cast<long long>(d.n1) * d.n0;
  for (long long row = static_cast<long long>(blockIdx.x) * rows_per + ty; row < nrows;
       row += static_cast<long long>(gridDim.x) * rows_per) {
    const int i = static_cast<int>(row / d.n0), m = static_cast<int>(row - static_cast<long long>(i) * d.n0);
    const long long base = row * d.n2;
    for (int j = tx; j < d.n2; j += d.bx) body(base + j, i, m, j);
  }
}

#define GRID_STRIDE(e, n)                                                                 \
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < (n); \
       e += static_cast<long long>(gridDim.x) * blockDim.x)

template <int NV>
__device__ __forceinline__ void write_partials(double (&v)[NV], double* partials) {
  __shared__ double scratch[(kThreads / 32) * NV];
  block_sum<NV>(v, scratch);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[blockIdx.x * NV + k] = v[k];
}

__global__ void __launch_bounds__(kThreads) k_g_init(CDField3 psi, CDField3 lam, DField3 g, long long n, double lc) {
  GRID_STRIDE(e, n) {
#pragma unroll
    for (int c = 0; c < 3; ++c) g.c[c][e] = dsub(psi.c[c][e], dscale(lam.c[c][e], lc));
  }
}

// Axis-0 neighbours across the shard boundary: plane i+1 / i-1 of the local
// range, else the halo plane (pl = offset within a plane), else absent.
__device__ __forceinline__ bool has_fwd(int i, int n1, const double2* hi) { return i + 1 < n1 || hi != nullptr; }
__device__ __forceinline__ bool has_bwd(int i, const double2* lo) { return i > 0 || lo != nullptr; }
__device__ __forceinline__ double2 fwd0(const double2* __restrict__ a, const double2* __restrict__ hi, int i, int n1,
                                        long long idx, long long s0, long long pl) {
  return i + 1 < n1 ? a[idx + s0] : hi[pl];
}
__device__ __forceinline__ double2 bwd0(const double2* __restrict__ a, const double2* __restrict__ lo, int i,
                                        long long idx, long long s0, long long pl) {
  return i > 0 ? a[idx - s0] : lo[pl];
}

// One voxel of k_grad_update; EDGE: plane 0 or n1-1 of this rank (axis-0
// neighbours from the halo planes or absent), else the interior fast path.
template <bool EDGE>
__device__ __forceinline__ void grad_update_voxel(const double2* __restrict__ u, const CDField3& g,
                                                  double2* __restrict__ G, const double2* __restrict__ p_prev,
                                                  const double2* __restrict__ G_prev, const DevDims& d, double rho,
                                                  const Halo& hl, long long idx, int i, int m, int j,
                                                  double (&red)[3]) {
  const int pos[3] = {i, m, j};
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  const long long pl = static_cast<long long>(m) * d.n2 + j;
  const double2 u0 = u[idx];
  double2 dv = zero2();
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const bool fwd = EDGE && ax == 0 ? has_fwd(i, d.n1, hl.u_hi) : pos[ax] + 1 < len[ax];
    double2 un = zero2();
    if (fwd) un = EDGE && ax == 0 ? fwd0(u, hl.u_hi, i, d.n1, idx, st[0], pl) : u[idx + st[ax]];
    const double2 gu = fwd ? dsub(un, u0) : zero2();
    const double2 gd = dsub(gu, g.c[ax][idx]);  // (grad u - g)_ax at idx
    red[0] += dnrm(gd);
    if (fwd) dv = dadd(dv, gd);
    const bool bwd = EDGE && ax == 0 ? has_bwd(i, hl.u_lo) : pos[ax] > 0;
    if (bwd) {
      const double2 ub = EDGE && ax == 0 ? bwd0(u, hl.u_lo, i, idx, st[0], pl) : u[idx - st[ax]];
      const double2 gb = EDGE && ax == 0 ? bwd0(g.c[0], hl.g0_lo, i, idx, st[0], pl) : g.c[ax][idx - st[ax]];
      dv = dsub(dv, dsub(dsub(u0, ub), gb));
    }
  }
  const double2 Gn = dfma(-rho, dv, G[idx]);
  G[idx] = Gn;
  red[1] += dnrm(Gn);
  if (p_prev) red[2] += dredot(p_prev[idx], dsub(Gn, G_prev[idx]));
}

__global__ void __launch_bounds__(kThreads) k_grad_update(const double2* __restrict__ u, CDField3 g,
                                                          double2* __restrict__ G,
                                                          const double2* __restrict__ p_prev,
                                                          const double2* __restrict__ G_prev, DevDims d,
                                                          double rho, double* __restrict__ partials, Halo hl) {
  double red[3] = {0.0, 0.0, 0.0};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    if (i > 0 && i + 1 < d.n1) grad_update_voxel<false>(u, g, G, p_prev, G_prev, d, rho, hl, idx, i, m, j, red);
    else grad_update_voxel<true>(u, g, G, p_prev, G_prev, d, rho, hl, idx, i, m, j, red);
  });
  write_partials<3>(red, partials);
}

__device__ __forceinline__ double2 dir_at(const double2* __restrict__ G, const double2* __restrict__ pp,
                                          double beta, long long e) {
  const double2 g = G[e];
  if (beta == 0.0) return make_double2(-g.x, -g.y);
  return dfma(beta, pp[e], make_double2(-g.x, -g.y));
}

__global__ void __launch_bounds__(kThreads) k_direction(const double2* __restrict__ G,
                                                        const double2* __restrict__ p_prev, double beta,
                                                        const double2* __restrict__ u, CDField3 g,
                                                        double2* __restrict__ p, DevDims d,
                                                        double* __restrict__ partials, Halo hl) {
  double red[2] = {0.0, 0.0};
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    const int pos[3] = {i, m, j};
    const long long pl = static_cast<long long>(m) * d.n2 + j;
    const double2 p0 = dir_at(G, p_prev, beta, idx);
    p[idx] = p0;
    const double2 u0 = u[idx];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const bool fwd = ax == 0 ? has_fwd(i, d.n1, hl.u_hi) : pos[ax] + 1 < len[ax];
      double2 pn = zero2(), un = zero2();
      if (fwd) {
        if (ax == 0 && i + 1 >= d.n1) {
          pn = dir_at(hl.G_hi, hl.pp_hi, beta, pl);
          un = hl.u_hi[pl];
        } else {
          pn = dir_at(G, p_prev, beta, idx + st[ax]);
          un = u[idx + st[ax]];
        }
      }
      const double2 gp = fwd ? dsub(pn, p0) : zero2();
      const double2 gu = fwd ? dsub(un, u0) : zero2();
      const double2 gd = dsub(gu, g.c[ax][idx]);
      red[0] += dnrm(gp);
      red[1] += dredot(gd, gp);
    }
  });
  write_partials<2>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_axpy(double2* __restrict__ y, const double2* __restrict__ x, double a,
                                                   long long n) {
  GRID_STRIDE(e, n) y[e] = dfma(a, x[e], y[e]);
}

__global__ void __launch_bounds__(kThreads) k_rsp_multiplier(const double2* __restrict__ u, DField3 lam,
                                                             CDField3 psi_old, DField3 psi_new, DevDims d,
                                                             double lc, double thr, double rho_s,
                                                             double* __restrict__ partials, Halo hl) {
  double red[2] = {0.0, 0.0};
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    const int pos[3] = {i, m, j};
    const double2 u0 = u[idx];
    double2 gu[3], z[3], l[3];
    double msq = 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (ax == 0)
        gu[ax] = has_fwd(i, d.n1, hl.u_hi)
                     ? dsub(fwd0(u, hl.u_hi, i, d.n1, idx, st[0], static_cast<long long>(m) * d.n2 + j), u0)
                     : zero2();
      else
        gu[ax] = pos[ax] + 1 < len[ax] ? dsub(u[idx + st[ax]], u0) : zero2();
      l[ax] = lam.c[ax][idx];
      z[ax] = dadd(gu[ax], dscale(l[ax], lc));
      msq += dnrm(z[ax]);
    }
    const double mg = sqrt(msq);
    const double sc = mg > 0.0 ? fmax(mg - thr, 0.0) / mg : 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const double2 ps = dscale(z[ax], sc);
      const double2 df = dsub(gu[ax], ps);
      red[0] += dnrm(df);
      red[1] += dnrm(dsub(ps, psi_old.c[ax][idx]));
      psi_new.c[ax][idx] = ps;
      lam.c[ax][idx] = dfma(rho_s, df, l[ax]);
    }
  });
  write_partials<2>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_tv(const double2* __restrict__ u, DevDims d,
                                                 double* __restrict__ partials, Halo hl) {
  double red[1] = {0.0};
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    const int pos[3] = {i, m, j};
    const double2 u0 = u[idx];
    double acc = 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (ax == 0) {
        if (has_fwd(i, d.n1, hl.u_hi))
          acc += dnrm(dsub(fwd0(u, hl.u_hi, i, d.n1, idx, st[0], static_cast<long long>(m) * d.n2 + j), u0));
      } else if (pos[ax] + 1 < len[ax]) {
        acc += dnrm(dsub(u[idx + st[ax]], u0));
      }
    }
    red[0] += sqrt(acc);
  });
  write_partials<1>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_norm2_diff_f(const float2* __restrict__ a, const float2* __restrict__ b,
                                                           long long n, double* __restrict__ partials) {
  double red[2] = {0.0, 0.0};
  GRID_STRIDE(e, n) {
    const float2 av = a[e];
    red[1] += fnrm(av);
    if (b) {
      const float2 bv = b[e];
      const double dx = static_cast<double>(av.x) - bv.x, dy = static_cast<double>(av.y) - bv.y;
      red[0] += dx * dx + dy * dy;
    }
  }
  write_partials<2>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_norm2_diff_d(const double2* __restrict__ a,
                                                           const double2* __restrict__ b, long long n,
                                                           double* __restrict__ partials) {
  double red[2] = {0.0, 0.0};
  GRID_STRIDE(e, n) {
    const double2 av = a[e];
    red[1] += dnrm(av);
    if (b) red[0] += dnrm(dsub(av, b[e]));
  }
  write_partials<2>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_sub_norm(float2* __restrict__ a, const float2* __restrict__ b,
                                                       long long n, double* __restrict__ partials) {
  double red[1] = {0.0};
  GRID_STRIDE(e, n) {
    const float2 r = csub(a[e], b[e]);
    a[e] = r;
    red[0] += fnrm(r);
  }
  write_partials<1>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_grad(const float2* __restrict__ u, Field3 out, DevDims d) {
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    const int pos[3] = {i, m, j};
    const float2 u0 = u[idx];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
      out.c[ax][idx] = pos[ax] + 1 < len[ax] ? csub(u[idx + st[ax]], u0) : make_float2(0.f, 0.f);
  });
}

__global__ void __launch_bounds__(kThreads) k_div(CField3 g, float2* __restrict__ out, DevDims d) {
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    const int pos[3] = {i, m, j};
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      float2 v = make_float2(0.f, 0.f);
      if (pos[ax] + 1 < len[ax]) v = cadd(v, g.c[ax][idx]);
      if (pos[ax] > 0) v = csub(v, g.c[ax][idx - st[ax]]);
      acc = cadd(acc, v);
    }
    out[idx] = acc;
  });
}

__global__ void k_c128_to_c64(const double2* __restrict__ in, float2* __restrict__ out, long long n) {
  GRID_STRIDE(e, n) {
    const double2 v = in[e];
    out[e] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
  }
}

__global__ void k_c64_to_c128(const float2* __restrict__ in, double2* __restrict__ out, long long n) {
  GRID_STRIDE(e, n) {
    const float2 v = in[e];
    out[e] = make_double2(v.x, v.y);
  }
}

}  // namespace

void g_init(CDField3 psi, CDField3 lam, DField3 g, std::int64_t n, double lc, cudaStream_t s) {
  prof::begin("k_g_init", s);
  k_g_init<<<grid_blocks(), kThreads, 0, s>>>(psi, lam, g, n, lc);
  MLRG_LAUNCH_CHECK("k_g_init");
  prof::end("k_g_init", s);
}

int grad_update(const double2* u, CDField3 g, double2* G, const double2* p_prev, const double2* G_prev, Dims d,
                double rho, double* partials, cudaStream_t s, const Halo& halo) {
  prof::begin("k_grad_update", s);
  k_grad_update<<<grid_blocks(), kThreads, 0, s>>>(u, g, G, p_prev, G_prev, dev_dims(d), rho, partials, halo);
  MLRG_LAUNCH_CHECK("k_grad_update");
  prof::end("k_grad_update", s);
  return 3 * grid_blocks();
}

int direction(const double2* G, const double2* p_prev, double beta, const double2* u, CDField3 g, double2* p,
              Dims d, double* partials, cudaStream_t s, const Halo& halo) {
  prof::begin("k_direction", s);
  k_direction<<<grid_blocks(), kThreads, 0, s>>>(G, p_prev, beta, u, g, p, dev_dims(d), partials, halo);
  MLRG_LAUNCH_CHECK("k_direction");
  prof::end("k_direction", s);
  return 2 * grid_blocks();
}

void axpy(double2* y, const double2* x, double a, std::int64_t n, cudaStream_t s) {
  prof::begin("k_axpy", s);
  k_axpy<<<grid_blocks(), kThreads, 0, s>>>(y, x, a, n);
  MLRG_LAUNCH_CHECK("k_axpy");
  prof::end("k_axpy", s);
}

int rsp_multiplier_slots() { return 2 * grid_blocks(); }

int rsp_multiplier(const double2* u, DField3 lam, CDField3 psi_old, DField3 psi_new, Dims d, double lc, double thr,
                   double rho_over_scale, double* partials, cudaStream_t s, const Halo& halo) {
  prof::begin("k_rsp_multiplier", s);
  k_rsp_multiplier<<<grid_blocks(), kThreads, 0, s>>>(u, lam, psi_old, psi_new, dev_dims(d), lc, thr,
                                                      rho_over_scale, partials, halo);
  MLRG_LAUNCH_CHECK("k_rsp_multiplier");
  prof::end("k_rsp_multiplier", s);
  return 2 * grid_blocks();
}

int tv_norm(const double2* u, Dims d, double* partials, cudaStream_t s, const Halo& halo) {
  k_tv<<<grid_blocks(), kThreads, 0, s>>>(u, dev_dims(d), partials, halo);
  MLRG_LAUNCH_CHECK("k_tv");
  return grid_blocks();
}

int norm2_diff(const float2* a, const float2* b, std::int64_t n, double* partials, cudaStream_t s) {
  k_norm2_diff_f<<<grid_blocks(), kThreads, 0, s>>>(a, b, n, partials);
  MLRG_LAUNCH_CHECK("k_norm2_diff_f");
  return 2 * grid_blocks();
}

int norm2_diff(const double2* a, const double2* b, std::int64_t n, double* partials, cudaStream_t s) {
  k_norm2_diff_d<<<grid_blocks(), kThreads, 0, s>>>(a, b, n, partials);
  MLRG_LAUNCH_CHECK("k_norm2_diff_d");
  return 2 * grid_blocks();
}

int sub_norm(float2* a, const float2* b, std::int64_t n, double* partials, cudaStream_t s) {
  k_sub_norm<<<grid_blocks(), kThreads, 0, s>>>(a, b, n, partials);
  MLRG_LAUNCH_CHECK("k_sub_norm");
  return grid_blocks();
}

void grad(const float2* u, Field3 out, Dims d, cudaStream_t s) {
  k_grad<<<grid_blocks(), kThreads, 0, s>>>(u, out, dev_dims(d));
  MLRG_LAUNCH_CHECK("k_grad");
}

void div(CField3 g, float2* out, Dims d, cudaStream_t s) {
  k_div<<<grid_blocks(), kThreads, 0, s>>>(g, out, dev_dims(d));
  MLRG_LAUNCH_CHECK("k_div");
}

void c128_to_c64(const double2* in, float2* out, std::int64_t n, cudaStream_t s) {
  k_c128_to_c64<<<grid_blocks(), kThreads, 0, s>>>(in, out, n);
  MLRG_LAUNCH_CHECK("k_c128_to_c64");
}

void c64_to_c128(const float2* in, double2* out, std::int64_t n, cudaStream_t s) {
  k_c64_to_c128<<<grid_blocks(), kThreads, 0, s>>>(in, out, n);
  MLRG_LAUNCH_CHECK("k_c64_to_c128");
}

}  // namespace mlrg::ops
