// tcgen05 kind::i8 throughput vs N and for the digit-stage MMA pattern of k_m2l_i8
// (operands resident in shared memory: the upper bound of the M2L's tensor-pipe use,
// independent of L2).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_nsweep tools/umma_i8_nsweep.cu
//   mode 0: back-to-back M=128 N=n K=32 MMAs, one A and one B tile
//   mode 1: the stage pattern of KS digits, NC columns per digit: W digit i times the
//           stacked B digits 0..KS-1-i (N = (KS-i) NC, split in equal parts <= 256)
//   mode 2: mode 1 while a second warp streams `copy_kb` KB per stage from global
//           memory into a shared-memory ring with cp.async.bulk (the W / B loads)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint32_t idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t td, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(td), "l"(da), "l"(db), "r"(id),
               "r"(acc));
}
__device__ __forceinline__ void wait_bar(unsigned long long* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@!P1 bra W_%=;\n\t}\n" ::"r"(su32(bar)), "r"(ph));
}

__device__ int g_random = 0;  // 1: pseudo-random operand bytes (hash), 0: the (i * 37) ramp
template <int KS, int NC>
__global__ void k_pat(int mode, int n, int iters, int copy_bytes, const unsigned char* src, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned long long bar, cbar[4];
  __shared__ uint32_t tbase;
  constexpr int A_BYTES = KS * 4096, B_BYTES = KS * NC * 32;
  for (int i = threadIdx.x; i < A_BYTES + B_BYTES; i += blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u + blockIdx.x * 40503u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    sm[i] = g_random ? (unsigned char)(h >> 11) : (unsigned char)(i * 37);
  }
  unsigned char* ring = sm + ((A_BYTES + B_BYTES + 1023) & ~1023);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbar[s])));
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t td = tbase;
  if (threadIdx.x == 0) {
    const uint64_t da = desc(su32(sm)), db = desc(su32(sm + A_BYTES));
    const long long t0 = clock64();
    if (mode == 0) {
      const uint32_t id = idesc(n);
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) mma(td, da, db, id, (it | u) > 0);
      }
    } else {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < KS; ++i) {
          const int ncol = (KS - i) * NC;
          const int nsp = (ncol + 255) / 256;
          const int part = ((ncol / nsp + 31) / 32) * 32;
#pragma unroll
          for (int p0 = 0; p0 < ncol;) {
            const int np = ncol - p0 < part ? ncol - p0 : part;
            mma(td + i * NC + p0, da + (uint64_t)((i * 4096) >> 4), db + (uint64_t)((p0 * 32) >> 4), idesc(np),
                (it | i) > 0);
            p0 += np;
          }
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    wait_bar(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 32 && mode == 2) {
    // stream copy_bytes per stage into a 4-slot ring (nobody reads it)
    const unsigned char* g = src + (size_t)blockIdx.x * copy_bytes * 4;
    for (int it = 0; it < iters; ++it) {
      const int s = it & 3;
      if (it >= 4) wait_bar(&cbar[s], ((it >> 2) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&cbar[s])), "r"(copy_bytes)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(ring + (size_t)s * copy_bytes)),
                   "l"(g + (size_t)s * copy_bytes), "r"(copy_bytes), "r"(su32(&cbar[s]))
                   : "memory");
    }
    for (int it = iters < 4 ? 0 : iters - 4; it < iters; ++it) wait_bar(&cbar[it & 3], (it >> 2) & 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(td));
}

template <int KS, int NC>
double run(int mode, int n, int copy_bytes, int sms, const unsigned char* src, long long* cyc, double* ms_out) {
  auto kern = k_pat<KS, NC>;
  const int smem = ((KS * 4096 + KS * NC * 32 + 1023) & ~1023) + 4 * copy_bytes + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  double best = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    kern<<<sms, 64, smem>>>(mode, n, 16, copy_bytes, src, cyc);
    cudaEventRecord(e0);
    kern<<<sms, 64, smem>>>(mode, n, iters, copy_bytes, src, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    double cols = mode == 0 ? 8.0 * n : (double)KS * (KS + 1) / 2 * NC;
    const double ops = 2.0 * 128 * cols * 32 * iters * sms;
    const double t = ops / (ms * 1e-3) / 1e12;
    if (t > best) { best = t; *ms_out = ms; }
  }
  if (cudaGetLastError() != cudaSuccess) printf("CUDA error\n");
  return best;
}

// the stage pattern held for `secs` seconds; rate over the last 20 % (power-limited clocks)
template <int KS, int NC>
double run_sustained(double secs, int sms, const unsigned char* src, long long* cyc, int random) {
  auto kern = k_pat<KS, NC>;
  const int smem = ((KS * 4096 + KS * NC * 32 + 1023) & ~1023) + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemcpyToSymbol(g_random, &random, sizeof(int));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  kern<<<sms, 64, smem>>>(1, 0, iters, 0, src, cyc);
  cudaEventRecord(e0);
  kern<<<sms, 64, smem>>>(1, 0, iters, 0, src, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms1 = 0.f;
  cudaEventElapsedTime(&ms1, e0, e1);
  const int warm = (int)(secs * 800.0 / ms1), meas = (int)(secs * 200.0 / ms1) + 1;
  for (int i = 0; i < warm; ++i) kern<<<sms, 64, smem>>>(1, 0, iters, 0, src, cyc);
  cudaEventRecord(e0);
  for (int i = 0; i < meas; ++i) kern<<<sms, 64, smem>>>(1, 0, iters, 0, src, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  int zero = 0;
  cudaMemcpyToSymbol(g_random, &zero, sizeof(int));
  const double cols = (double)KS * (KS + 1) / 2 * NC;
  return 2.0 * 128 * cols * 32 * iters * sms * meas / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, sizeof(long long) * sms);
  unsigned char* src;
  const size_t srcb = (size_t)sms * 4 * 49152;
  cudaMalloc(&src, srcb);
  cudaMemset(src, 1, srcb);
  double ms;
  for (int n : {32, 64, 96, 128, 160, 192, 224, 256}) {
    const double t = run<6, 64>(0, n, 0, sms, src, cyc, &ms);
    printf("{\"mode\": \"single\", \"N\": %d, \"tops\": %.1f}\n", n, t);
  }
  printf("{\"mode\": \"stage 7x64 (7-bit digits)\", \"tops\": %.1f}\n", run<7, 64>(1, 0, 0, sms, src, cyc, &ms));
  printf("{\"mode\": \"stage 6x64\", \"tops\": %.1f}\n", run<6, 64>(1, 0, 0, sms, src, cyc, &ms));
  printf("{\"mode\": \"stage 6x80\", \"tops\": %.1f}\n", run<6, 80>(1, 0, 0, sms, src, cyc, &ms));
  printf("{\"mode\": \"stage 6x32\", \"tops\": %.1f}\n", run<6, 32>(1, 0, 0, sms, src, cyc, &ms));
  for (int kb : {12, 24, 30, 36, 42}) {
    const double t = run<6, 64>(2, 0, kb * 1024, sms, src, cyc, &ms);
    // stage time and implied L2 -> SM rate
    const double stage_us = ms * 1e3 / 4000;
    printf("{\"mode\": \"stage 6x64 + %d KB bulk copy per stage\", \"tops\": %.1f, \"stage_us\": %.3f, \"copy_TBs\": %.2f}\n",
           kb, t, stage_us, kb * 1024.0 * sms / (stage_us * 1e-6) / 1e12);
  }
  for (int kb : {36, 42}) {
    const double t = run<7, 64>(2, 0, kb * 1024, sms, src, cyc, &ms);
    const double stage_us = ms * 1e3 / 4000;
    printf("{\"mode\": \"stage 7x64 + %d KB bulk copy per stage\", \"tops\": %.1f, \"stage_us\": %.3f, \"copy_TBs\": %.2f}\n",
           kb, t, stage_us, kb * 1024.0 * sms / (stage_us * 1e-6) / 1e12);
  }
  for (int rnd : {0, 1}) {
    const double t = run_sustained<6, 64>(4.0, sms, src, cyc, rnd);
    printf("{\"mode\": \"stage 6x64 held 4 s, %s operands\", \"tops_sustained\": %.1f}\n", rnd ? "pseudo-random" : "ramp", t);
  }
  return 0;
}
