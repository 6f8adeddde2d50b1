// Does DMMA (FP64 tensor pipe) run concurrently with DFMA (FP64 ALU pipe)?
// Warp-specialised mix: warps with (warp % den) < num issue DFMA chains, the
// others DMMA chains; reports the combined FP64 rate.  Also an interleaved mix
// inside one warp.  Used to decide whether the M2L can split its flops.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dfma_body(double (&x)[16], int iters, double a, double b) {
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
}
__device__ __forceinline__ void dmma_body(double (&c)[8][2], int iters, double a, double b) {
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
}

// role: 0 = DFMA, 1 = DMMA (per warp); it_f / it_m iterations
__global__ void mix_kernel(double* out, int num, int den, int it_f, int it_m) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp % den < num) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
    dfma_body(x, it_f, 1.0000001, 1e-9);
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
  } else {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    dmma_body(c, it_m, threadIdx.x * 1e-3, 1.0 - threadIdx.x * 1e-4);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  }
  if (s == 12345.0) out[threadIdx.x] = s;
}

// one warp interleaves: per iteration 8 DMMA + R x 16 DFMA
template <int R>
__global__ void inter_kernel(double* out, int iters) {
  double x[16];
  double c[8][2];
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        x[2 * i] = fma(x[2 * i], 1.0000001, 1e-9);
        x[2 * i + 1] = fma(x[2 * i + 1], 1.0000001, 1e-9);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int threads = 512, blocks = sms * 2;
  const int W = threads / 32;
  // flop per warp-iteration: DFMA 16 * 2 * 32 = 1024, DMMA 8 * 512 = 4096
  struct Mix { int num, den; };
  for (Mix m : {Mix{0, 1}, Mix{1, 1}, Mix{1, 2}, Mix{1, 4}, Mix{1, 8}, Mix{3, 4}}) {
    for (int ratio : {1, 2, 4, 8}) {  // DFMA iterations per DMMA iteration
      const int it_m = 4000, it_f = it_m * ratio;
      mix_kernel<<<blocks, threads>>>(out, m.num, m.den, 10, 10);
      cudaEventRecord(e0);
      mix_kernel<<<blocks, threads>>>(out, m.num, m.den, it_f, it_m);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      int nf = 0, nm = 0;
      for (int w = 0; w < W; ++w) (w % m.den < m.num ? nf : nm)++;
      const double ff = 1024.0 * it_f * nf * (double)blocks, fm = 4096.0 * it_m * nm * (double)blocks;
      printf("warp-mix dfma_warps=%d/%d ratio=%d: DFMA %.2f + DMMA %.2f = %.2f TFLOP/s (%.3f ms)\n", nf, W, ratio,
             ff / ms / 1e9, fm / ms / 1e9, (ff + fm) / ms / 1e9, ms);
      if (m.num == 0 || m.num == m.den) break;
    }
  }
  const int iters = 4000;
#define INTER(R)                                                                                         \
  inter_kernel<R><<<blocks, threads>>>(out, 10);                                                         \
  cudaEventRecord(e0);                                                                                   \
  inter_kernel<R><<<blocks, threads>>>(out, iters);                                                      \
  cudaEventRecord(e1);                                                                                   \
  cudaEventSynchronize(e1);                                                                              \
  cudaEventElapsedTime(&ms, e0, e1);                                                                     \
  {                                                                                                      \
    const double fm = 4096.0 * iters * W * (double)blocks, ff = 1024.0 * R * iters * W * (double)blocks; \
    printf("interleaved R=%d: DFMA %.2f + DMMA %.2f = %.2f TFLOP/s\n", R, ff / ms / 1e9, fm / ms / 1e9,  \
           (ff + fm) / ms / 1e9);                                                                        \
  }
  INTER(1) INTER(2) INTER(4)
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
