// FP64 peak microbenchmarks (DFMA chain and DMMA mma.sync) used as the roofline
// denominator for the FP64-bound phases (M2L, P2P). MEASURED_PEAKS.json has no FP64
// figure, so bench.py / DESIGN.md quote these numbers.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
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

__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k16_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 + i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
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
  for (int threads : {256, 512, 1024}) {
    for (int cps : {1, 2, 4}) {
      int blocks = sms * cps;
      int iters = 20000;
      dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * iters * (double)blocks * threads;
      printf("DFMA threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
      dmma_m8n8k4_kernel<<<blocks, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma_m8n8k4_kernel<<<blocks, threads>>>(out, iters / 4);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 8 * 8 * 4 * 8 * (iters / 4) * (double)blocks * (threads / 32);
      printf("DMMA m8n8k4 threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
      dmma_m16n8k16_kernel<<<blocks, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma_m16n8k16_kernel<<<blocks, threads>>>(out, iters / 16);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 16 * 8 * 16 * 4 * (iters / 16) * (double)blocks * (threads / 32);
      printf("DMMA m16n8k16 threads=%d blocks=%d: %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
