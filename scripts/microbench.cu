// Issue-rate microbenchmarks behind the kernel design notes in DESIGN.md:
// FP64 FMA, FP32 FMA, and float->double conversion (F2F.F64.F32) throughput
// on one B200. Build and run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench.cu && /tmp/mb
#include <cuda_runtime.h>

#include <cstdio>

template <class T>
__global__ void k_fma(T* out, T a, T b, int iters) {
  T x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = x[i] * a + b;
  T s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// per element: 1 FFMA (fresh float), 1 F2F.F64.F32, 1 DFMA
__global__ void k_cvt(double* out, float a, float b, double c, int iters) {
  float f[8];
  double d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = threadIdx.x + i, d[i] = 0.0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      f[i] = fmaf(f[i], a, b);
      d[i] = fma(static_cast<double>(f[i]), c, d[i]);
    }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d = nullptr;
  cudaMalloc(&d, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  const double elems = 8.0 * iters * blocks * threads;
  float ms = 0.f;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_fma<double><<<blocks, threads>>>(d, 0.999, 1e-3, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("fp64 fma          : %.1f TFLOP/s (%.1f Gop/s)\n", 2 * elems / ms / 1e9, elems / ms / 1e6);
    cudaEventRecord(e0);
    k_fma<float><<<blocks, threads>>>(reinterpret_cast<float*>(d), 0.999f, 1e-3f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("fp32 fma          : %.1f TFLOP/s\n", 2 * elems / ms / 1e9);
    cudaEventRecord(e0);
    k_cvt<<<blocks, threads>>>(d, 0.999f, 1e-3f, 1.0001, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("ffma+f2f+dfma     : %.1f G elem/s (per SM per clk at 1.965 GHz: %.1f)\n", elems / ms / 1e6,
                elems / ms / 1e6 / sms / 1.965);
  }
  return 0;
}
