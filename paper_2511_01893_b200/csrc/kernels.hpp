// Host launchers for the fused ADMM kernels (vecops.cu) and the memo-layer
// kernels (memo_kernels.cu). Every reduction writes nv doubles per CTA into
// `partials`; the launcher returns the number of doubles written so the host
// sums them in CTA order (deterministic, no float atomics).
//
// Precision split: the USFFT operators compute in complex64, but the ADMM
// iterate and its multipliers (u, G, p, psi, lambda, g; the volume side) are
// complex128. Differences such as grad(u) and grad(u) - psi + lambda/rho
// cancel leading digits; in complex64 storage that cancellation alone moved
// the 64^3 reference trajectory by 1e-3 after ten iterations.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#ifdef __CUDACC__
#define MLRG_HD __host__ __device__
#else
#define MLRG_HD
#endif

namespace mlrg {

struct DevSlab;  // memo_gpu.hpp

/// Volume extents for the stencil kernels (row-major (n1, n0, n2)).
struct Dims {
  std::int64_t n1 = 0, n0 = 0, n2 = 0;
  std::int64_t count() const { return n1 * n0 * n2; }
};

/// Three-component field (GradField, operators.hpp:17-30), one plane per axis.
template <class T>
struct Field3T {
  T* c[3] = {nullptr, nullptr, nullptr};
};
template <class T>
struct CField3T {
  const T* c[3] = {nullptr, nullptr, nullptr};
  CField3T() = default;
  CField3T(const Field3T<T>& f) : c{f.c[0], f.c[1], f.c[2]} {}
};
using Field3 = Field3T<float2>;
using CField3 = CField3T<float2>;
using DField3 = Field3T<double2>;
using CDField3 = CField3T<double2>;

namespace ops {

/// Neighbour planes of this rank's axis-0 range in sharded mode (SURVEY.md
/// §8(e)): plane a-1 ("lo") and plane b ("hi") of the global volume, each
/// (n0, n2). Null = the global boundary (or unsharded).
struct Halo {
  const double2* u_lo = nullptr;
  const double2* u_hi = nullptr;
  const double2* g0_lo = nullptr;  // axis-0 component of g at plane a-1
  const double2* G_hi = nullptr;
  const double2* pp_hi = nullptr;  // p_prev at plane b
};

/// g = psi - lambda * lc (admm.cpp:64 with the lazy lambda scale folded in lc).
void g_init(CDField3 psi, CDField3 lam, DField3 g, std::int64_t n, double lc, cudaStream_t s);

/// G -= rho * div(grad(u) - g) (admm.cpp:144-147) with partials
/// [|grad u - g|^2, |G|^2, Re<p_prev, G - G_prev>] (the last one only when
/// p_prev/G_prev are non-null).
int grad_update(const double2* u, CDField3 g, double2* G, const double2* p_prev, const double2* G_prev, Dims d,
                double rho, double* partials, cudaStream_t s, const Halo& halo = {});

/// p = -G + beta * p_prev (admm.cpp:86-93) with partials
/// [|grad p|^2, Re<grad u - g, grad p>] (admm.cpp:95-102).
int direction(const double2* G, const double2* p_prev, double beta, const double2* u, CDField3 g, double2* p,
              Dims d, double* partials, cudaStream_t s, const Halo& halo = {});

/// y += a * x (admm.cpp:108-110).
void axpy(double2* y, const double2* x, double a, std::int64_t n, cudaStream_t s);

/// Fused rsp_update + multiplier update (admm.cpp:154-181):
/// psi_new = shrink(grad u + lam*lc, thr); lam += rho_over_lam_scale * (grad u - psi_new).
/// Partials [|grad u - psi_new|^2, |psi_new - psi_old|^2].
/// Partial slots one rsp_multiplier launch writes.
int rsp_multiplier_slots();
int rsp_multiplier(const double2* u, DField3 lam, CDField3 psi_old, DField3 psi_new, Dims d, double lc, double thr,
                   double rho_over_scale, double* partials, cudaStream_t s, const Halo& halo = {});

/// Isotropic TV: partials [sum sqrt(sum_c |grad_c u|^2)] (admm.cpp:39-46).
int tv_norm(const double2* u, Dims d, double* partials, cudaStream_t s, const Halo& halo = {});

/// Partials [|a - b|^2, |a|^2] (b may be null).
int norm2_diff(const float2* a, const float2* b, std::int64_t n, double* partials, cudaStream_t s);
int norm2_diff(const double2* a, const double2* b, std::int64_t n, double* partials, cudaStream_t s);

/// a -= b with partials [|a - b|^2] (resid = d_pred - d, admm.cpp:126-128).
int sub_norm(float2* a, const float2* b, std::int64_t n, double* partials, cudaStream_t s);

/// Forward differences (operators.cpp:311-328) and the negative-adjoint
/// divergence (operators.cpp:330-352), materialised (tests and the C-ABI).
void grad(const float2* u, Field3 out, Dims d, cudaStream_t s);
void div(CField3 g, float2* out, Dims d, cudaStream_t s);

/// complex128 <-> complex64 conversion on the device.
void c128_to_c64(const double2* in, float2* out, std::int64_t n, cudaStream_t s);
void c64_to_c128(const float2* in, double2* out, std::int64_t n, cudaStream_t s);

// ---- memo layer ----

/// A chunk of a full row-major array (split_chunks, array.cpp:30-63): slab
/// `start..start+extent` along axis 0 or 1.
struct SlabGeom {
  std::int64_t d0 = 0, d1 = 0, d2 = 0;
  int axis = 0;
  std::int64_t start = 0, extent = 0;
  MLRG_HD std::int64_t count() const { return axis == 0 ? extent * d1 * d2 : d0 * extent * d2; }
};

/// keys[s][r] = sum_i P[r][i] Re x_s[i] + P[r][n+i] Im x_s[i] for `ns` slabs of
/// one shape (encoder.cpp:405-422), float keys; norms2[s] = sum |x_s|^2 (double).
/// `starts` lists each slab's start along the split axis; `work` needs
/// encode_work_doubles(ns, kd) doubles.
void encode(const float2* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
            double* work, float* keys, double* norms2, cudaStream_t s);
void encode(const double2* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
            double* work, float* keys, double* norms2, cudaStream_t s);
std::size_t encode_work_doubles(int ns, int kd);
/// The same GEMM on the tcgen05 tensor cores (encode_tc.cu): one launch of at
/// most 16 slabs writing encode_tc_grid() CTA partial tiles [slab][kd + 1] into
/// `work` (summed by the k_encode_reduce pass). Supported when kd <= 60, 2n is
/// a multiple of 4 and K = 2n spans at least two 128-column stages per SM.
bool encode_tc_supported(SlabGeom shape, const float* P, int kd, int ns);
int encode_tc_grid();
void encode_tc(const float2* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
               double* work, cudaStream_t s);
void encode_tc(const double2* x, SlabGeom shape, const std::int64_t* starts, int ns, const float* P, int kd,
               double* work, cudaStream_t s);

/// A list of slabs of one SlabGeom (start/extent per entry) for the batched
/// copies: hits read `value[q]` scaled by `scale[q]`, stores write `dst[q]`.
constexpr int kSlabBatch = 64;
struct SlabBatch {
  std::int64_t start[kSlabBatch];
  std::int64_t extent[kSlabBatch];
  const float2* value[kSlabBatch];
  float2* dst[kSlabBatch];
  double scale[kSlabBatch];
};

/// out[slab_q] = value_q * scale_q - sub[slab_q] for every listed slab (sub may
/// be null) (scalerun.cpp:250-255).
void slab_materialize(float2* out, SlabGeom g, const SlabBatch& b, int nb, const float2* sub, cudaStream_t s);
void slab_materialize(double2* out, SlabGeom g, const SlabBatch& b, int nb, cudaStream_t s);
/// dst_q = out[slab_q] (contiguous chunk order, complex64; dst_q may be null)
/// and then out[slab_q] -= sub[slab_q] when sub is set (scalerun.cpp:276-283).
void slab_store(float2* out, SlabGeom g, const SlabBatch& b, int nb, const float2* sub, cudaStream_t s);
void slab_store(double2* out, SlabGeom g, const SlabBatch& b, int nb, cudaStream_t s);

/// Device-side memo: the same copies driven by the per-slab decisions in HBM
/// (slab c = [c * chunk, ...) along g.axis): hits get value * scale (- sub),
/// misses are copied to their arena slot (when accepted) and then get out -= sub.
/// One launch (k_dev_finish) per call.
void dev_finish(float2* out, SlabGeom g, const DevSlab* slabs, int n, std::int64_t chunk, const float2* sub,
                cudaStream_t s);
void dev_finish(double2* out, SlabGeom g, const DevSlab* slabs, int n, std::int64_t chunk, cudaStream_t s);

}  // namespace ops
}  // namespace mlrg
