// k_peak.cu -- peak microbenchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry: FP64 (DMMA / DFMA) and the int8 tcgen05
// tensor core (k_m2l_i8).
#include <cuda_runtime.h>
#include <stdint.h>

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
// int8 tcgen05: one CTA per SM, one thread issues back-to-back M=128 N=256 K=32
// MMAs on SMEM-resident operands (constant-offset descriptors, as k_m2l_i8)
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_peak_i8(int iters, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned long long bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (128 + 256) * 32; i += blockDim.x) sm[i] = (unsigned char)(i * 37);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t td = tbase;
  if (threadIdx.x == 0) {
    auto desc = [](uint32_t a) {
      return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | ((uint64_t)1 << 46);
    };
    const uint64_t da = desc(su32(sm)), db = desc(su32(sm + 128 * 32));
    const uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(td),
                     "l"(da), "l"(db), "r"(id), "r"((it | u) > 0 ? 1 : 0));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
                 "@!P1 bra W_%=;\n\t}\n" ::"r"(su32(&bar)));
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(td));
}
}  // namespace

// kind 0: burst (best of three ~1 ms runs from idle clocks); kind 1: sustained -- the
// same kernel back to back for ~3 s, the rate over the last ~0.6 s (the int8 MMAs run
// into the board power limit within about a second; a kernel inside a long step sees
// this peak, not the burst one)
extern "C" double fdh_tensor_peak_tops(int kind) {
  if (kind != 0 && kind != 1) return 0.0;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long* cyc = nullptr;
  if (cudaMalloc(&cyc, sizeof(long long) * sms) != cudaSuccess) return 0.0;
  const int smem = (128 + 256) * 32;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  const int iters = 4000;
  if (kind == 1) {
    const double ops = 2.0 * 128 * 256 * 32 * 8.0 * iters * sms;
    k_peak_i8<<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(e0);
    k_peak_i8<<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms1 = 0.f;
    cudaEventElapsedTime(&ms1, e0, e1);
    const int warm = ms1 > 0 ? (int)(2400.0 / ms1) : 1000, meas = ms1 > 0 ? (int)(600.0 / ms1) + 1 : 300;
    for (int i = 0; i < warm; ++i) k_peak_i8<<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(e0);
    for (int i = 0; i < meas; ++i) k_peak_i8<<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(cyc);
    return (cudaGetLastError() == cudaSuccess && ms > 0) ? ops * meas / (ms * 1e-3) / 1e12 : 0.0;
  }
  for (int rep = 0; rep < 3; ++rep) {
    k_peak_i8<<<sms, 128, smem>>>(16, cyc);
    cudaEventRecord(e0);
    k_peak_i8<<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * 128 * 256 * 32 * 8.0 * iters * sms;
    if (ms > 0 && ops / (ms * 1e-3) / 1e12 > best) best = ops / (ms * 1e-3) / 1e12;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(cyc);
  return cudaGetLastError() == cudaSuccess ? best : 0.0;
}

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
