// DMMA issue-pattern microbenchmark: the inner step of k_m2l_gemm without
// global memory.  Per k-step a warp loads NT B fragments from shared memory and
// issues 4 x NT DMMAs (4 m-tiles) into 4 x NT independent accumulators; CTAs of
// 128 threads, resident CTAs per SM set through the dynamic smem size.
// Prints FP64 TFLOP/s per (NT, CTAs/SM, DADD-per-B) variant.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int NT, bool SUM>
__global__ void __launch_bounds__(128) k(double* out, int iters) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 4096; i += 128) sm[i] = 1e-3 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double a[4] = {1e-3 * lane, 2e-3, 3e-3, 4e-3};
  double c[4][NT][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) c[m][n][0] = c[m][n][1] = 0.0;
  const double* B = sm + (lane >> 2) * 36 + (lane & 3);
  for (int it = 0; it < iters; ++it) {
    const int ko = (it & 31) * 8;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double b[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        b[n] = B[n * 8 * 36 + ko + 4 * h];
        if (SUM) b[n] += B[n * 8 * 36 + ko + 4 * h + 512];
      }
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma(c[m][n], a[m], b[n]);
    }
  }
  double s = 0;
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) s += c[m][n][0] + c[m][n][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int NT, bool SUM>
void run(int sms, double* out, int cps) {
  const int smem = (228 * 1024) / cps - 2048;
  cudaFuncSetAttribute(k<NT, SUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int blocks = sms * cps * 8, iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<NT, SUM><<<blocks, 128, smem>>>(out, 10);
  cudaEventRecord(e0);
  k<NT, SUM><<<blocks, 128, smem>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 512.0 * 2 * 4 * NT * (double)iters * blocks * 4;
  printf("NT=%d sum=%d ctas/SM=%d: %.2f TFLOP/s  (%s)\n", NT, (int)SUM, cps, fl / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  for (int cps : {1, 2, 3, 4}) {
    run<1, false>(sms, out, cps);
    run<2, false>(sms, out, cps);
    run<2, true>(sms, out, cps);
    run<4, false>(sms, out, cps);
  }
  return 0;
}
