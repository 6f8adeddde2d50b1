// k_peak.cu -- FP64 peak microbenchmarks (the roofline denominator for the
// FP64-bound phases; MEASURED_PEAKS.json carries no FP64 figure).
#include <cuda_runtime.h>

#include "../../include/fdhelm_c.h"

namespace {
__global__ void k_peak_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}
__global__ void k_peak_dfma(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}
}  // namespace

extern "C" double fdh_fp64_peak_tflops(int kind) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, 1024 * sizeof(double)) != cudaSuccess) return 0.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 2, threads = 512, iters = 20000;
  double best = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    float ms = 0.f;
    double fl = 0.0;
    if (kind == 0) {
      k_peak_dmma<<<blocks, threads>>>(out, 64);
      cudaEventRecord(e0);
      k_peak_dmma<<<blocks, threads>>>(out, iters / 4);
      cudaEventRecord(e1);
      fl = 2.0 * 8 * 8 * 4 * 8 * (iters / 4) * (double)blocks * (threads / 32);
    } else {
      k_peak_dfma<<<blocks, threads>>>(out, 64, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      k_peak_dfma<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      fl = 2.0 * 16 * iters * (double)blocks * threads;
    }
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms > 0) best = fl / (ms * 1e-3) / 1e12 > best ? fl / (ms * 1e-3) / 1e12 : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}
