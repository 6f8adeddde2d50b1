// DMMA throughput probe: operand-pattern variants of mma.sync.m8n8k4.f64
// (what the M2L GEMM inner loop can reach on sm_100a).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int V>
__global__ void probe(double* out, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 1e-4;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double a[4], b[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { a[i] = lane * 1e-3 + i; b[i] = 1.0 - lane * 1e-4 + i; }
  for (int it = 0; it < iters; ++it) {
    if (V == 3 || V == 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = sm[(it * 64 + i * 32 + lane) & 4095]; b[i] = sm[(it * 64 + 2048 + i * 32 + lane) & 4095]; }
    }
    if (V == 1 || V == 3) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], a[mt], b[nt]);
    } else {
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) dmma(acc[mt][nt], a[mt], b[nt]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int V>
void run(const char* name, int threads, int cps) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8192);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * cps, iters = 4000;
  probe<V><<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  probe<V><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 8 * 8 * 4 * 16 * (double)iters * blocks * (threads / 32);
  printf("%-28s threads=%4d ctas/sm=%d : %.2f TFLOP/s\n", name, threads, cps, fl / ms / 1e9);
  cudaFree(out);
}

int main() {
  for (int t : {128, 256}) for (int c : {1, 2, 3, 4}) {
    run<1>("regs, mt-outer (a reuse)", t, c);
    run<2>("regs, nt-outer (b reuse)", t, c);
    run<3>("lds, mt-outer", t, c);
    run<4>("lds, nt-outer", t, c);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
