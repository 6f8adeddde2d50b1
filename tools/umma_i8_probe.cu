// umma_i8_probe.cu -- tcgen05.mma kind::i8 on sm_100a: descriptor check and throughput.
//
// (1) correctness: D[128 x N] = A[128 x K] * B[N x K]^T (int8 -> int32) on one CTA,
//     K-major SWIZZLE_NONE canonical layout, for both readings of LBO/SBO; prints
//     which one matches the host product.
// (2) throughput: 148 CTAs issue back-to-back MMAs on SMEM-resident operands;
//     reports int8 MAC/clk/SM and TOPS for N = 16 .. 256.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_probe tools/umma_i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);      \
      std::exit(1);                                                                             \
    }                                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
  // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
  return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)            // D = S32
         | (1u << 7)          // A signed
         | (1u << 10)         // B signed
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// element (r, k) of an R x K K-major operand: core matrices of 8 rows x 16 bytes,
// layout [r/8][k/16][r%8][k%16]  -> k-adjacent cores 128 B apart, r-adjacent KB*128.
__host__ __device__ inline int lay(int r, int k, int K) { return ((r >> 3) * (K >> 4) + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15); }

constexpr int M = 128;

__global__ void k_check(const int8_t* A, const int8_t* B, int32_t* D, int N, int K, int swap) {
  extern __shared__ __align__(1024) uint8_t sm[];
  int8_t* sa = (int8_t*)sm;
  int8_t* sb = sa + M * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) sa[lay(i / K, i % K, K)] = A[i];
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) sb[lay(i / K, i % K, K)] = B[i];
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t td = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    const uint32_t kstride = 128, mstride = (K / 16) * 128;
    for (int c = 0; c < K / 32; ++c) {
      const uint32_t off = c * 2 * 128;
      const uint64_t da = swap ? sdesc(a0 + off, mstride, kstride) : sdesc(a0 + off, kstride, mstride);
      const uint64_t db = swap ? sdesc(b0 + off, mstride, kstride) : sdesc(b0 + off, kstride, mstride);
      mma_i8(td, da, db, idesc_i8(M, N), c > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    tmem_ld8(td + ((uint32_t)(w * 32) << 16) + c0, r);
    for (int j = 0; j < 8; ++j) D[(w * 32 + lane) * N + c0 + j] = (int32_t)r[j];
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(td));
}

// throughput: each CTA issues iters x (K/32) MMAs of 128 x N x 32 on resident SMEM
__global__ void k_tput(int N, int K, int iters, int swap, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  int8_t* sa = (int8_t*)sm;
  int8_t* sb = sa + M * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (M + N) * K; i += blockDim.x) sa[i] = (int8_t)((i * 37) & 63) - 32;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t td = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    const uint32_t kstride = 128, mstride = (K / 16) * 128;
    const uint32_t id = idesc_i8(M, N);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int c = 0; c < K / 32; ++c) {
        const uint32_t off = c * 2 * 128;
        const uint64_t da = swap ? sdesc(a0 + off, mstride, kstride) : sdesc(a0 + off, kstride, mstride);
        const uint64_t db = swap ? sdesc(b0 + off, mstride, kstride) : sdesc(b0 + off, kstride, mstride);
        mma_i8(td, da, db, id, (it | c) > 0);
      }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(td));
}


template <int NACC>
__global__ void k_tput2(int N, int K, int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  int8_t* sa = (int8_t*)sm;
  int8_t* sb = sa + M * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (M + N) * K; i += blockDim.x) sa[i] = (int8_t)((i * 37) & 63) - 32;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t td = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    const uint32_t kstride = 128, mstride = (K / 16) * 128;
    const uint32_t id = idesc_i8(M, N);
    uint64_t da[8], db[8];
    for (int c = 0; c < 8; ++c) { da[c] = sdesc(a0 + c * 256, kstride, mstride); db[c] = sdesc(b0 + c * 256, kstride, mstride); }
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int a = 0; a < NACC; ++a) mma_i8(td + a * N, da[c], db[c], id, (it | c) > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(td));
}


// the k_m2l_i8 stage pattern: for digit i, N = (7-i)*NC split at 256, D col = i*NC + p0
__global__ void k_pattern(int NC, int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  int8_t* sa = (int8_t*)sm;              // 7 W digit blocks of 128 x 32
  int8_t* sb = sa + 7 * 4096;            // B: 7*NC rows x 32
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 7 * 4096 + 7 * NC * 32; i += blockDim.x) sa[i] = (int8_t)((i * 37) & 63) - 32;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t td = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    const long long t0 = clock64();
    const uint64_t dA = sdesc(a0, 128, 256), dB = sdesc(b0, 128, 256);
    if (NC == 64) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 7; ++i) {
          constexpr int NCc = 64;
          const int ncol = (7 - i) * NCc;
#pragma unroll
          for (int p0 = 0; p0 < ncol; p0 += 256) {
            const int np = ncol - p0 < 256 ? ncol - p0 : 256;
            mma_i8(td + i * NCc + p0, dA + (uint64_t)(i * 4096 >> 4), dB + (uint64_t)(p0 * 32 >> 4), idesc_i8(128, np), (it | i) > 0);
          }
        }
      }
    } else {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 7; ++i) {
          constexpr int NCc = 32;
          const int ncol = (7 - i) * NCc;
          mma_i8(td + i * NCc, dA + (uint64_t)(i * 4096 >> 4), dB, idesc_i8(128, ncol), (it | i) > 0);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(td));
}

int main() {
  int dev = 0;
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, dev));
  std::printf("device %s, %d SMs\n", pr.name, pr.multiProcessorCount);
  const int K = 256;
  int good_swap = -1;
  for (int N : {16, 32, 64, 224, 256}) {
    std::vector<int8_t> A(M * K), B(N * K);
    srand(N);
    for (auto& v : A) v = (int8_t)(rand() % 255 - 127);
    for (auto& v : B) v = (int8_t)(rand() % 255 - 127);
    std::vector<int32_t> R(M * N, 0);
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        int32_t s = 0;
        for (int k = 0; k < K; ++k) s += (int32_t)A[i * K + k] * (int32_t)B[j * K + k];
        R[i * N + j] = s;
      }
    int8_t *dA, *dB;
    int32_t* dD;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dD, R.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    const size_t sm = (size_t)(M + N) * K;
    CK(cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (int swap = 0; swap < 2; ++swap) {
      CK(cudaMemset(dD, 0, R.size() * 4));
      k_check<<<1, 128, sm>>>(dA, dB, dD, N, K, swap);
      CK(cudaDeviceSynchronize());
      std::vector<int32_t> D(R.size());
      CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
      long bad = 0;
      for (size_t i = 0; i < D.size(); ++i) bad += D[i] != R[i];
      std::printf("check N=%3d K=%d swap=%d: %ld / %zu mismatches (D[0]=%d ref %d)\n", N, K, swap, bad, D.size(), D[0],
                  R[0]);
      if (bad == 0) good_swap = swap;
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  }
  if (good_swap < 0) {
    std::printf("no descriptor variant matched\n");
    return 1;
  }
  long long* dc;
  CK(cudaMalloc(&dc, 4096 * sizeof(long long)));
  const int nsm = pr.multiProcessorCount;
  for (int N : {16, 32, 64, 96, 128, 160, 224, 256}) {
    const int iters = 2000;
    const size_t sm = (size_t)(M + N) * K;
    CK(cudaFuncSetAttribute(k_tput, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_tput<<<nsm, 128, sm>>>(N, K, 10, good_swap, dc);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_tput<<<nsm, 128, sm>>>(N, K, iters, good_swap, dc);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(nsm);
    CK(cudaMemcpy(c.data(), dc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (auto v : c) mx = v > mx ? v : mx;
    const double macs = (double)M * N * K * iters;
    std::printf("tput N=%3d: %.1f MAC/clk/SM, %.0f TOPS (event %.3f ms)\n", N, macs / (double)mx,
                2.0 * macs * nsm / (ms * 1e-3) / 1e12, ms);
  }

  for (int nacc : {1, 2, 4}) for (int N : {16, 32, 64, 128}) {
    if (nacc * N > 512) continue;
    const int iters = 1000;
    const size_t sm = (size_t)(M + N) * K;
    auto f = nacc == 1 ? k_tput2<1> : (nacc == 2 ? k_tput2<2> : k_tput2<4>);
    CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    f<<<nsm, 128, sm>>>(N, K, 10, dc);
    CK(cudaDeviceSynchronize());
    f<<<nsm, 128, sm>>>(N, K, iters, dc);
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(nsm);
    CK(cudaMemcpy(c.data(), dc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (auto v : c) mx = v > mx ? v : mx;
    const double macs = (double)M * N * K * iters * nacc;
    std::printf("tput2 nacc=%d N=%3d: %.1f MAC/clk/SM, %.1f clk/MMA\n", nacc, N, macs / (double)mx, (double)mx / (iters * 8.0 * nacc));
  }

  for (int NC : {32, 64}) {
    const int iters = 2000;
    const size_t sm = 7 * 4096 + 7 * NC * 32;
    CK(cudaFuncSetAttribute(k_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_pattern<<<nsm, 128, sm>>>(NC, 10, dc);
    CK(cudaDeviceSynchronize());
    k_pattern<<<nsm, 128, sm>>>(NC, iters, dc);
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(nsm);
    CK(cudaMemcpy(c.data(), dc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (auto v : c) mx = v > mx ? v : mx;
    std::printf("pattern NC=%d: %.1f clk/stage (ideal %d)\n", NC, (double)mx / iters, 28 * NC / 2);
  }
  return 0;
}
