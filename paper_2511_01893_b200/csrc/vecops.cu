// Fused, HBM-bound ADMM kernels (admm.cpp:59-195 restated on the device).
// Each stencil kernel walks rows (i, m) of the (n1, n0, n2) volume with the
// threads of a CTA along j, recomputes grad(u) - g from u and g where the
// reference materialises GradFields, and reduces in double per CTA.
#include <cmath>

#include "common.cuh"
#include "device.hpp"
#include "kernels.hpp"

namespace mlrg::ops {

namespace {

constexpr int kThreads = 256;

struct RowWalk {
  int bx, rows_per;  // threads along j, rows per CTA iteration
};

RowWalk row_walk(std::int64_t n2) {
  int bx = 32;
  while (bx < 256 && bx < n2) bx <<= 1;
  return {bx, kThreads / bx};
}

int grid_blocks() { return 4 * sm_count(); }

struct DevDims {
  int n1, n0, n2, bx;
  long long s0, s1;  // strides of axes 0 and 1
};

DevDims dev_dims(Dims d) {
  return {static_cast<int>(d.n1), static_cast<int>(d.n0), static_cast<int>(d.n2), row_walk(d.n2).bx,
          d.n0 * d.n2, d.n2};
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

__device__ __forceinline__ double nrm(float2 a) {
  return static_cast<double>(a.x) * a.x + static_cast<double>(a.y) * a.y;
}
__device__ __forceinline__ double redot(float2 a, float2 b) {  // Re(a * conj(b))
  return static_cast<double>(a.x) * b.x + static_cast<double>(a.y) * b.y;
}

template <int NV>
__device__ __forceinline__ void write_partials(double (&v)[NV], double* partials) {
  __shared__ double scratch[(kThreads / 32) * NV];
  block_sum<NV>(v, scratch);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[blockIdx.x * NV + k] = v[k];
}

__global__ void __launch_bounds__(kThreads) k_g_init(const float2* __restrict__ p0, const float2* __restrict__ p1,
                                                     const float2* __restrict__ p2, const float2* __restrict__ l0,
                                                     const float2* __restrict__ l1, const float2* __restrict__ l2,
                                                     float2* __restrict__ g0, float2* __restrict__ g1,
                                                     float2* __restrict__ g2, long long n, float lc) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    g0[e] = csub(p0[e], cscale(l0[e], lc));
    g1[e] = csub(p1[e], cscale(l1[e], lc));
    g2[e] = csub(p2[e], cscale(l2[e], lc));
  }
}

__global__ void __launch_bounds__(kThreads) k_grad_update(const float2* __restrict__ u, CField3 g,
                                                          float2* __restrict__ G,
                                                          const float2* __restrict__ p_prev,
                                                          const float2* __restrict__ G_prev, DevDims d,
                                                          float rho, double* __restrict__ partials) {
  double red[3] = {0.0, 0.0, 0.0};
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    const int pos[3] = {i, m, j};
    const float2 u0 = u[idx];
    float2 dv = make_float2(0.f, 0.f);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const bool fwd = pos[ax] + 1 < len[ax];
      const float2 gu = fwd ? csub(u[idx + st[ax]], u0) : make_float2(0.f, 0.f);
      const float2 gd = csub(gu, g.c[ax][idx]);  // (grad u - g)_ax at idx
      red[0] += nrm(gd);
      if (fwd) dv = cadd(dv, gd);
      if (pos[ax] > 0) {  // neighbour's component, always an interior difference
        const float2 gdm = csub(csub(u0, u[idx - st[ax]]), g.c[ax][idx - st[ax]]);
        dv = csub(dv, gdm);
      }
    }
    const float2 Gn = make_float2(fmaf(-rho, dv.x, G[idx].x), fmaf(-rho, dv.y, G[idx].y));
    G[idx] = Gn;
    red[1] += nrm(Gn);
    if (p_prev) red[2] += redot(p_prev[idx], csub(Gn, G_prev[idx]));
  });
  write_partials<3>(red, partials);
}

__device__ __forceinline__ float2 dir_at(const float2* __restrict__ G, const float2* __restrict__ pp, float beta,
                                         long long e) {
  const float2 g = G[e];
  if (beta == 0.f) return make_float2(-g.x, -g.y);
  const float2 p = pp[e];
  return make_float2(fmaf(beta, p.x, -g.x), fmaf(beta, p.y, -g.y));
}

__global__ void __launch_bounds__(kThreads) k_direction(const float2* __restrict__ G,
                                                        const float2* __restrict__ p_prev, float beta,
                                                        const float2* __restrict__ u, CField3 g,
                                                        float2* __restrict__ p, DevDims d,
                                                        double* __restrict__ partials) {
  double red[2] = {0.0, 0.0};
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    const int pos[3] = {i, m, j};
    const float2 p0 = dir_at(G, p_prev, beta, idx);
    p[idx] = p0;
    const float2 u0 = u[idx];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const bool fwd = pos[ax] + 1 < len[ax];
      const float2 gp = fwd ? csub(dir_at(G, p_prev, beta, idx + st[ax]), p0) : make_float2(0.f, 0.f);
      const float2 gu = fwd ? csub(u[idx + st[ax]], u0) : make_float2(0.f, 0.f);
      const float2 gd = csub(gu, g.c[ax][idx]);
      red[0] += nrm(gp);
      red[1] += redot(gd, gp);
    }
  });
  write_partials<2>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_axpy(float2* __restrict__ y, const float2* __restrict__ x, float a,
                                                   long long n) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float2 xv = x[e];
    float2 yv = y[e];
    yv.x = fmaf(a, xv.x, yv.x);
    yv.y = fmaf(a, xv.y, yv.y);
    y[e] = yv;
  }
}

__global__ void __launch_bounds__(kThreads) k_scale(float2* __restrict__ y, const float2* __restrict__ x, float a,
                                                    long long n) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    y[e] = cscale(x[e], a);
}

__global__ void __launch_bounds__(kThreads) k_rsp_multiplier(const float2* __restrict__ u, Field3 lam,
                                                             CField3 psi_old, Field3 psi_new, DevDims d,
                                                             float lc, float thr, float rho_s,
                                                             double* __restrict__ partials) {
  double red[2] = {0.0, 0.0};
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    const int pos[3] = {i, m, j};
    const float2 u0 = u[idx];
    float2 gu[3], z[3], l[3];
    float msq = 0.f;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      gu[ax] = pos[ax] + 1 < len[ax] ? csub(u[idx + st[ax]], u0) : make_float2(0.f, 0.f);
      l[ax] = lam.c[ax][idx];
      z[ax] = cadd(gu[ax], cscale(l[ax], lc));
      msq = fmaf(z[ax].x, z[ax].x, fmaf(z[ax].y, z[ax].y, msq));
    }
    const float mg = sqrtf(msq);
    const float sc = mg > 0.f ? fmaxf(mg - thr, 0.f) / mg : 0.f;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const float2 ps = cscale(z[ax], sc);
      const float2 df = csub(gu[ax], ps);
      red[0] += nrm(df);
      red[1] += nrm(csub(ps, psi_old.c[ax][idx]));
      psi_new.c[ax][idx] = ps;
      lam.c[ax][idx] = make_float2(fmaf(rho_s, df.x, l[ax].x), fmaf(rho_s, df.y, l[ax].y));
    }
  });
  write_partials<2>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_tv(const float2* __restrict__ u, DevDims d,
                                                 double* __restrict__ partials) {
  double red[1] = {0.0};
  const int len[3] = {d.n1, d.n0, d.n2};
  const long long st[3] = {d.s0, d.s1, 1};
  for_voxels(d, [&](long long idx, int i, int m, int j) {
    const int pos[3] = {i, m, j};
    const float2 u0 = u[idx];
    double acc = 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
      if (pos[ax] + 1 < len[ax]) acc += nrm(csub(u[idx + st[ax]], u0));
    red[0] += sqrt(acc);
  });
  write_partials<1>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_norm2_diff(const float2* __restrict__ a, const float2* __restrict__ b,
                                                         long long n, double* __restrict__ partials) {
  double red[2] = {0.0, 0.0};
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float2 av = a[e];
    red[1] += nrm(av);
    if (b) red[0] += nrm(csub(av, b[e]));
  }
  write_partials<2>(red, partials);
}

__global__ void __launch_bounds__(kThreads) k_sub_norm(float2* __restrict__ a, const float2* __restrict__ b,
                                                       long long n, double* __restrict__ partials) {
  double red[1] = {0.0};
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float2 r = csub(a[e], b[e]);
    a[e] = r;
    red[0] += nrm(r);
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
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double2 v = in[e];
    out[e] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
  }
}

__global__ void k_c64_to_c128(const float2* __restrict__ in, double2* __restrict__ out, long long n) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float2 v = in[e];
    out[e] = make_double2(v.x, v.y);
  }
}

}  // namespace

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

int sub_norm(float2* a, const float2* b, std::int64_t n, double* partials, cudaStream_t s) {
  k_sub_norm<<<grid_blocks(), kThreads, 0, s>>>(a, b, n, partials);
  MLRG_LAUNCH_CHECK("k_sub_norm");
  return grid_blocks();
}

void g_init(CField3 psi, CField3 lam, Field3 g, std::int64_t n, float lc, cudaStream_t s) {
  k_g_init<<<grid_blocks(), kThreads, 0, s>>>(psi.c[0], psi.c[1], psi.c[2], lam.c[0], lam.c[1], lam.c[2], g.c[0],
                                              g.c[1], g.c[2], n, lc);
  MLRG_LAUNCH_CHECK("k_g_init");
}

int grad_update(const float2* u, CField3 g, float2* G, const float2* p_prev, const float2* G_prev, Dims d,
                float rho, double* partials, cudaStream_t s) {
  k_grad_update<<<grid_blocks(), kThreads, 0, s>>>(u, g, G, p_prev, G_prev, dev_dims(d), rho, partials);
  MLRG_LAUNCH_CHECK("k_grad_update");
  return 3 * grid_blocks();
}

int direction(const float2* G, const float2* p_prev, float beta, const float2* u, CField3 g, float2* p, Dims d,
              double* partials, cudaStream_t s) {
  k_direction<<<grid_blocks(), kThreads, 0, s>>>(G, p_prev, beta, u, g, p, dev_dims(d), partials);
  MLRG_LAUNCH_CHECK("k_direction");
  return 2 * grid_blocks();
}

void axpy(float2* y, const float2* x, float a, std::int64_t n, cudaStream_t s) {
  k_axpy<<<grid_blocks(), kThreads, 0, s>>>(y, x, a, n);
  MLRG_LAUNCH_CHECK("k_axpy");
}

void scale(float2* y, const float2* x, float a, std::int64_t n, cudaStream_t s) {
  k_scale<<<grid_blocks(), kThreads, 0, s>>>(y, x, a, n);
  MLRG_LAUNCH_CHECK("k_scale");
}

int rsp_multiplier(const float2* u, Field3 lam, CField3 psi_old, Field3 psi_new, Dims d, float lc, float thr,
                   float rho_over_scale, double* partials, cudaStream_t s) {
  k_rsp_multiplier<<<grid_blocks(), kThreads, 0, s>>>(u, lam, psi_old, psi_new, dev_dims(d), lc, thr,
                                                      rho_over_scale, partials);
  MLRG_LAUNCH_CHECK("k_rsp_multiplier");
  return 2 * grid_blocks();
}

int tv_norm(const float2* u, Dims d, double* partials, cudaStream_t s) {
  k_tv<<<grid_blocks(), kThreads, 0, s>>>(u, dev_dims(d), partials);
  MLRG_LAUNCH_CHECK("k_tv");
  return grid_blocks();
}

int norm2_diff(const float2* a, const float2* b, std::int64_t n, double* partials, cudaStream_t s) {
  k_norm2_diff<<<grid_blocks(), kThreads, 0, s>>>(a, b, n, partials);
  MLRG_LAUNCH_CHECK("k_norm2_diff");
  return 2 * grid_blocks();
}

}  // namespace mlrg::ops
