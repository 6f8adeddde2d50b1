// k_m2l_i8.cu -- M2L on the 5th-generation tensor cores (tcgen05.mma kind::i8, sm_100a).
//
// M2L is g~_{t,c} += A_{c,t x s} v~_{s,c} over the admissible
// leaves; per tile of TT target slots and coupling key it is the real GEMM
//
//     C[n x 2TT] = W[n x KP] * B[KP x 2TT],  W = [Re A | Im A],
//     B(:, 2j) = [Re v_j ; -Im v_j],  B(:, 2j+1) = [Im v_j ; Re v_j]      (KP = 2 n_kq)
//
// in complex128.  tcgen05 has no f64 kind, so the FP64 product is computed
// EXACTLY in integers (Ozaki-style fixed-point slicing):
//   * W (per tree level, one power-of-two scale S_W = 2^(eW+1) > 2 max|W|) and the
//     moments v (per (rhs, level), S_V) are rounded to B*KS-bit fixed point and split
//     into KS balanced base-2^B digits (int8), most significant first:
//     x = S * sum_i d_i 2^(-B(i+1)) (+ rounding error <= S 2^(-B KS - 1)).
//     Default KS x B = 6 x 8 (d_i in [-128, 127], 48 bits); 7 x 7 and 7 x 8 compile
//     (kernels.hpp);
//   * the product keeps the digit pairs i + j <= LV - 1 (default LV = 7: 26 of 36
//     pairs; the dropped ones weigh <= 2^(-B(LV+2)) 2^14 relative); pairs of one
//     level L = i + j share the weight 2^(-B(L+2)) and are summed EXACTLY in one
//     int32 TMEM accumulator column block: one MMA per W digit i multiplies W_i by
//     the B digits [B_0 | B_1 | ... | B_min(KS, LV - i) - 1] stacked along N and lands
//     in the level blocks i .. (D column = L * 2TT + target column);
//   * every key of a (tile, key-chunk) item accumulates into the same TMEM
//     columns (the scales are per level, hence per tile), so the int32 sums are
//     exact as long as an item has <= F keys (F from the digit bound, planner);
//   * the epilogue reads TMEM once per item and forms sum_L acc_L 2^(-B(L+2))
//     S_W S_V in FP64 (fixed order); items of a tile are chained in key-chunk
//     order as in k_m2l_gemm (deterministic, no FP atomics).
// Relative l2 error of y ~3e-14 .. 9e-14 on the BASELINE configs (vs 1e-12 allowed,
// north_star): the product is exact, only the 48-bit rounding of W and v and the
// dropped digit pairs remain.
//
// Data movement: the digits of W live in HBM pre-arranged in the UMMA canonical
// K-major layout (core matrices of 8 rows x 16 B, SWIZZLE_NONE), one contiguous
// block per (key, K chunk of 32), moved by ONE cp.async.bulk (TMA engine) per
// pipeline stage onto an mbarrier; the moment digits of the (up to TT) source
// slots of a key are gathered by all threads with 16-byte cp.async.  A single
// thread issues the MMAs (UTCIMMA) and commits them to the stage's "empty"
// mbarrier; NST stages in flight.
#include "kernels.hpp"

#include <algorithm>
#include <cstdlib>

#ifndef FDH_I8_SLEEP_NS
#define FDH_I8_SLEEP_NS 0  // > 0: nanosleep polling in the long mbarrier waits (0: try_wait suspend hint)
#endif
#ifndef FDH_I8_BALANCED
#define FDH_I8_BALANCED 1  // split N > 256 into equal MMAs (0: 256 + rest; tools/gpu_i8_split.sh: ~1 % on config 2)
#endif
#ifndef FDH_I8P_G
#define FDH_I8P_G 1  // k_m2l_i8p: moment-gather stages in flight per warp (beyond the one being issued)
#endif
#ifndef FDH_I8_EXP
#define FDH_I8_EXP 0  // timing experiments: 1 = no B gather, 2 = no W copy, 3 = neither (wrong results)
#endif

namespace fdhelm {

namespace {

constexpr int kKC = 32;               // K bytes per MMA k-step / pipeline stage
constexpr int kCore = 128 * kKC;      // bytes of one 128-row x 32-byte operand block

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// UMMA shared-memory descriptor, K-major SWIZZLE_NONE: LBO = stride between the
// two 16-byte K core matrices (128 B), SBO = stride between 8-row groups (256 B);
// verified on the B200 by tools/umma_i8_probe.cu
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// byte offset of element (row r, k) in a 128 x 32 K-major core-matrix block
__host__ __device__ __forceinline__ int core_off(int r, int k) {
  return ((r >> 3) * 2 + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15);
}
// rows stored per digit of M-block b / per (key, K chunk) in the trimmed layout
__host__ __device__ __forceinline__ int i8_rows_of_block(int n, int b) {
  const int n_pad = (n + 31) / 32 * 32;
  const int r = n_pad - 128 * b;
  return r < 128 ? r : 128;
}
__host__ __device__ __forceinline__ int i8_rows_total(int n) { return (n + 31) / 32 * 32; }
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// long waits (producers ahead of the ring, epilogue warps waiting for an item's MMAs):
// try_wait with a suspend-time hint -- the warp is parked by the hardware until the
// phase completes (no wake-up latency) instead of polling every ~30 ns (NANOSLEEP 128
// returned early: ncu counted 1.6e10 polls per pass, 25 % of all issued instructions,
// each a shared-memory wavefront beside the tensor core's operand reads).
// FDH_I8_SLEEP_NS > 0 restores the nanosleep polling loop.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
#if FDH_I8_SLEEP_NS > 0
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (ok) return;
    __nanosleep(FDH_I8_SLEEP_NS);
  }
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAITS_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(1000000u)
      : "memory");
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// one stage of W digits: one bulk copy when the digit blocks are full (src stride =
// 4096), else KS copies of wdig bytes to the 4096-byte digit slots
template <int KS>
__device__ __forceinline__ void w_stage_g2s(uint8_t* dst, const int8_t* src, int wst_bytes, uint32_t wdig,
                                            uint64_t* bar) {
  mbar_expect_tx(bar, wst_bytes);
  if (wdig == (uint32_t)kCore || wdig * KS != (uint32_t)wst_bytes) {
    bulk_g2s(dst, src, wst_bytes, bar);
  } else {
#pragma unroll
    for (int i = 0; i < KS; ++i) bulk_g2s(dst + i * kCore, src + i * wdig, wdig, bar);
  }
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
// int32 -> double without the conversion unit (I2F.F64 issues at a quarter of the FP64
// rate and bounded the epilogue): the double with high word 0x43300000 and low word
// x ^ 2^31 is 2^52 + 2^31 + x exactly; one subtraction leaves x
__device__ __forceinline__ double i32_to_f64(uint32_t x) {
  return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------- digits
// x -> KS balanced base-128 digits (most significant first) of rint(x / S 2^(7 KS)),
// S = 2^(ex + 1) > 2 |x|.  Exact integer arithmetic after one rounding.
template <int KS>
__device__ __forceinline__ void to_digits(double x, int ex, int8_t (&d)[KS]) {
  constexpr int B = kI8Bits, H = 1 << (B - 1);
  long long X = __double2ll_rn(ldexp(x, B * KS - ex - 1));
#pragma unroll
  for (int i = KS - 1; i > 0; --i) {
    const long long r = ((X + H) & (2 * H - 1)) - H;  // [-H, H-1]
    d[i] = (int8_t)r;
    X = (X - r) >> B;
  }
  d[0] = (int8_t)X;  // |x / S| <= 0.4923 (level_exp) keeps the leading digit inside int8
}
__device__ __forceinline__ int tile_nit_guard(const int32_t* __restrict__ tile_nitem, int tile) {
  return tile_nitem[tile];
}
// exponent of the power-of-two scale S = 2^(ex + 1) of a level with maximum modulus mx.
// 8-bit digits cover [-128, 127] b^-1 + ..., i.e. x / S in [-0.5, 0.498]: the maximum is
// bumped by 2^-6 so that |x / S| <= 0.4923 always has digits (7-bit digits are symmetric)
__device__ __forceinline__ int level_exp(const unsigned long long* lvmax, int l) {
  int ex = 0;
  const double mx = __longlong_as_double((long long)lvmax[l]);
  frexp(kI8Bits == 8 ? mx * 1.015625 : mx, &ex);
  return ex;
}

// per-level max |Re|, |Im| of the coupling matrices (pass 0) and their digits
// (pass 1), in the canonical frame of k_coupling; entries are
// computed exactly as there.
constexpr double kFourPi = 4.0 * 3.14159265358979323846;  // geometry.hpp:11
constexpr int kCplRows = 8;
template <int KS>
__global__ void __launch_bounds__(256) k_coupling_i8(const Consts* __restrict__ C, const double* __restrict__ dirtab,
                                                     int64_t key0, const int32_t* __restrict__ key_level,
                                                     const int64_t* __restrict__ key_d,
                                                     const int32_t* __restrict__ key_dir, int pass,
                                                     unsigned long long* __restrict__ lvmax, int8_t* __restrict__ Wq,
                                                     int n, int nkq, int mb, int gs, int64_t key_base) {
  __shared__ double tn[3][kMaxP], sn[3][kMaxP];
  __shared__ double red[8];
  const int64_t key = key0 + blockIdx.x;
  const int r0 = blockIdx.y * kCplRows;
  const int p = C->p;
  const int l = key_level[key];
  if (threadIdx.x < 3 * p) {
    const int a = threadIdx.x / p, nu = threadIdx.x % p;
    const double side = C->side_t[l][a];
    const int64_t d = key_d[3 * key + a];
    tn[a][nu] = cheb_node(__dmul_rn((double)d, side), __dmul_rn((double)(d + 1), side), C->cheb_cos[nu]);
    sn[a][nu] = cheb_node(0.0, __dmul_rn(1.0, side), C->cheb_cos[nu]);
  }
  const double* c = dir_vec(C, dirtab, l, key_dir[key]);
  const double cv[3] = {c[0], c[1], c[2]};
  const double kappa = C->kappa;
  __syncthreads();
  const int ex = pass ? level_exp(lvmax, l) : 0;
  const int nch = 2 * nkq / kKC;
  extern __shared__ __align__(16) int8_t sbuf[];  // pass 1: [digit][K chunk][256 B]
  if (pass) {
    for (int v = threadIdx.x; v < KS * nch * 16; v += blockDim.x) reinterpret_cast<int4*>(sbuf)[v] = make_int4(0, 0, 0, 0);
    __syncthreads();
  }
  double mx = 0.0;
  // work unit = (source node k, half of the CTA's 8 target rows): the source coordinates
  // stay in registers over 4 rows -- no per-entry index divisions
  const int pp = p * p;
  for (int u = threadIdx.x; u < 2 * n; u += blockDim.x) {
   const int half = u >= n ? 1 : 0, k = u - half * n;
   const double s0 = sn[0][k / pp], s1 = sn[1][(k / p) % p], s2 = sn[2][k % p];
   for (int jr = 4 * half; jr < 4 * half + 4; ++jr) {
    const int j = r0 + jr;
    if (j >= n) break;
    const double d[3] = {__dsub_rn(tn[0][j / pp], s0), __dsub_rn(tn[1][(j / p) % p], s1),
                         __dsub_rn(tn[2][j % p], s2)};
    const double r = sqrt(dot3(d, d));  // geometry.hpp:92-98
    const double ph = __dmul_rn(kappa, __dsub_rn(r, dot3(d, cv)));
    const double w = __ddiv_rn(1.0, __dmul_rn(kFourPi, r));
    double s, co;
    sincos(ph, &s, &co);
    const double re = __dmul_rn(w, co), im = __dmul_rn(w, s);
    if (!pass) {
      mx = fmax(mx, fmax(fabs(re), fabs(im)));
      continue;
    }
    int8_t dr[KS], di[KS];
    to_digits<KS>(re, ex, dr);
    to_digits<KS>(im, ex, di);
    // staged in shared memory: per (digit, K chunk) the 256 bytes of this CTA's
    // 8-row group in the canonical layout (2 K halves x 8 rows x 16 B)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = h ? nkq + k : k;  // K index: [Re A | Im A]
      const int ch = kk / kKC, kin = kk % kKC;
      int8_t* sb = sbuf + ch * 256 + (kin >> 4) * 128 + (j - r0) * 16 + (kin & 15);
#pragma unroll
      for (int i = 0; i < KS; ++i) sb[i * nch * 256] = h ? di[i] : dr[i];
    }
   }
  }
  if (pass) {
    // M-block b belongs to group g = b / gs (gs = 2: blocks {0, 1}, {2}; gs = 1: one
    // block per group); per (key, K chunk) the groups are stored one after the
    // other, digit-major inside a group -- the M-block passes of launch_m2l_i8.
    // gs = 1 (one M-block per pass): the last block stores only its n_pad - 128 (mb - 1)
    // rows per digit (a prefix of the canonical block: 8-row groups of 256 B)
    __syncthreads();
    const int b = r0 >> 7, rr = r0 & 127;
    const int g = b / gs, bg = b % gs, mbg = min(gs, mb - gs * g);
    const int rows_tot = gs == 1 ? i8_rows_total(n) : mb * 128;
    const int dstr = gs == 1 ? i8_rows_of_block(n, b) * kKC : mbg * kCore;  // digit stride
    int8_t* base = Wq + (key - key_base) * nch * (int64_t)(KS * rows_tot * kKC) + (int64_t)(gs * g * KS + bg) * kCore +
                   (rr >> 3) * 256;
    // coalesced: 16 lanes x 16 B per (digit, chunk) group, padding rows / K as zeros
    for (int v = threadIdx.x; v < KS * nch * 16; v += blockDim.x) {
      const int q = v & 15, ic = v >> 4, i = ic / nch, ch = ic - i * nch;
      *reinterpret_cast<int4*>(base + (int64_t)ch * (KS * rows_tot * kKC) + (int64_t)i * dstr + q * 16) =
          *reinterpret_cast<const int4*>(sbuf + ic * 256 + q * 16);
    }
  }
  if (!pass) {
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
      atomicMax(lvmax + l, (unsigned long long)__double_as_longlong(mx));
    }
  }
}

// moments: per-(rhs, level) max (pass 0), then digits of every source slot (pass 1):
// Mq: per (slot, K chunk of 32) one contiguous block of KS x 2 (kb) x 2 (h) x 16 B
// = the pieces a gather warp copies with consecutive lanes; digit i of row h,
// h = 0: [Re v | -Im v], h = 1: [Im v | Re v] (K index kk < n_kq: first half)
__device__ __forceinline__ int64_t mq_off(int64_t slot, int nch, int i, int h, int kk) {
  const int ch = kk / kKC, kin = kk % kKC;
  return (slot * nch + ch) * (int64_t)(kI8Digits * 4 * 16) + ((i * 2 + (kin >> 4)) * 2 + h) * 16 + (kin & 15);
}
__global__ void __launch_bounds__(128) k_mom_max(const double* __restrict__ mom, const int32_t* __restrict__ slot_level,
                                                 int n, int n_pad, unsigned long long* __restrict__ lvmax,
                                                 int64_t nslot1) {
  __shared__ double red[4];
  const int64_t s = blockIdx.x;  // rhs-major slot id (nrhs > 1): level of slot s % nslot1
  const double* g = mom + s * 2 * n_pad;
  double mx = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) mx = fmax(mx, fmax(fabs(g[k]), fabs(g[n_pad + k])));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    mx = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
    // one scale per (rhs, level): a vector of a batch is never rounded against a
    // larger vector's scale (batching must not change results)
    if (mx > 0.0)
      atomicMax(lvmax + (s / nslot1) * kMaxLevels + slot_level[s % nslot1],
                (unsigned long long)__double_as_longlong(mx));
  }
}
template <int KS>
__global__ void __launch_bounds__(128) k_mom_quant(const double* __restrict__ mom,
                                                   const int32_t* __restrict__ slot_level,
                                                   const unsigned long long* __restrict__ lvmax, int n, int n_pad,
                                                   int nkq, int8_t* __restrict__ Mq, int64_t nslot1) {
  const int64_t s = blockIdx.x;
  const double* g = mom + s * 2 * n_pad;
  const int ex = level_exp(lvmax, (int)(s / nslot1) * kMaxLevels + slot_level[s % nslot1]);
  const int kp = 2 * nkq;
  const int nch = kp / kKC;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    int8_t dr[KS], di[KS], dn[KS];
    to_digits<KS>(g[k], ex, dr);
    to_digits<KS>(g[n_pad + k], ex, di);
    to_digits<KS>(-g[n_pad + k], ex, dn);  // -Im v: its own digits (-(-128) is not an int8)
#pragma unroll
    for (int i = 0; i < KS; ++i) {
      Mq[mq_off(s, nch, i, 0, k)] = dr[i];
      Mq[mq_off(s, nch, i, 0, nkq + k)] = dn[i];
      Mq[mq_off(s, nch, i, 1, k)] = di[i];
      Mq[mq_off(s, nch, i, 1, nkq + k)] = dr[i];
    }
  }
}

// The MMAs of one pipeline stage (K = 32): W digit i (M-block b) times the stacked
// B digits j = 0 .. min(KS, LV - i) - 1, into the level blocks i .. (D column =
// L * NC + target column); N > 256 splits into equal parts (multiples of 32).
// In shared memory every W digit block is 4096 bytes apart; a trimmed last M-block
// (fewer than 128 rows stored per digit) is copied digit by digit and its missing rows
// stay zero in shared memory (zeroed once per CTA: zero operands keep the MMA's power
// down; their output rows are never read).
// `first`: the item's first stage overwrites -- every level block by the MMA of
// the first W digit that touches it (level L by i = max(0, L - KS + 1)).
template <int MB, int KS, int LV, int NC>
__device__ __forceinline__ void issue_range(uint32_t tmem, uint64_t dA, uint64_t dB, int i, int b, int c0, int c1,
                                            uint32_t acc) {
  const int ncol = c1 - c0;
  const int nsp = (ncol + 255) / 256;
  const int part = FDH_I8_BALANCED ? ((ncol / nsp + 31) / 32) * 32 : 256;
#pragma unroll
  for (int p0 = c0; p0 < c1;) {
    const int np = c1 - p0 < part ? c1 - p0 : part;
    mma_i8(tmem + b * LV * NC + i * NC + p0, dA + (uint64_t)(((i * MB + b) * kCore) >> 4),
           dB + (uint64_t)((p0 * kKC) >> 4), idesc_i8(np), acc);
    p0 += np;
  }
}
template <int MB, int KS, int LV, int NC, bool FIRST>
__device__ __forceinline__ void issue_stage(uint32_t tmem, uint64_t dA, uint64_t dB) {
#pragma unroll
  for (int i = 0; i < KS; ++i) {
    const int nj = LV - i < KS ? LV - i : KS;  // B digits of W digit i
#pragma unroll
    for (int b = 0; b < MB; ++b) {
      if (!FIRST) {
        issue_range<MB, KS, LV, NC>(tmem, dA, dB, i, b, 0, nj * NC, 1u);
      } else if (i == 0) {
        issue_range<MB, KS, LV, NC>(tmem, dA, dB, i, b, 0, nj * NC, 0u);
      } else if (i + KS - 1 < LV) {  // this digit is the first to touch level i + KS - 1 (j = KS - 1)
        issue_range<MB, KS, LV, NC>(tmem, dA, dB, i, b, 0, (nj - 1) * NC, 1u);
        issue_range<MB, KS, LV, NC>(tmem, dA, dB, i, b, (nj - 1) * NC, nj * NC, 0u);
      } else {
        issue_range<MB, KS, LV, NC>(tmem, dA, dB, i, b, 0, nj * NC, 1u);
      }
    }
  }
}

// ---------------------------------------------------------------- M2L
template <int MB, int TT, int KS, int NST, int NGW>
struct I8Shape {
  static constexpr int THREADS = (2 + NGW) * 32;  // W producer, MMA issuer, NGW gather warps
  static_assert(NGW == 2 || NGW >= 4, "epilogue warps must cover the 4 TMEM lane quarters");
  static constexpr int NC = 2 * TT;                 // real columns per digit block
  static constexpr int LV = kI8Levels;               // levels L = i + j = 0 .. LV-1 kept
  static constexpr int TCOLS = MB * LV * NC;         // TMEM columns used
  static_assert(TCOLS <= 512, "TMEM");
  static constexpr int WST = KS * MB * kCore;        // W bytes per stage
  static constexpr int BST = KS * NC * kKC;          // B bytes per stage
  static constexpr int STAGE = WST + BST;
  static_assert(NST >= 3, "pipeline (gather keeps 2 stages of cp.async in flight)");
};

// dynamic smem: [NST W stages][NST B stages][src table fkeys*TT int32][keys fkeys int32][bars]
//
// Persistent grid: every CTA loops, claiming work items (tile, key chunk) in
// increasing index order from an atomic counter.  The items of a tile are
// chained in that order (item_seq): an item with seq > 0 waits for its tile's
// ticket to reach seq before its epilogue.  The item it waits for has a lower
// index, so it was claimed earlier by a CTA that is already running -- the
// chain always progresses, whatever the dispatch order, co-residency or
// concurrent kernels (no reliance on blockIdx scheduling, no timeout).
// One pass handles MB consecutive 128-row M-blocks starting at blk0.
template <int MB, int TT, int KS, int NST, int NGW, int G>
__global__ void __maxnreg__(128)
    k_m2l_i8(const int32_t* __restrict__ item_tile, const int32_t* __restrict__ item_seq,
             const int64_t* __restrict__ item_k0, const int64_t* __restrict__ item_k1,
             const int32_t* __restrict__ tile_nitem, const int32_t* __restrict__ tile_tslot,
             const int32_t* __restrict__ tile_level, const int32_t* __restrict__ tile_keys,
             const int32_t* __restrict__ tile_src, const uint8_t* __restrict__ tile_cols,
             const uint8_t* __restrict__ tile_cnt, const int8_t* __restrict__ Wq, const int8_t* __restrict__ Mq,
             const unsigned long long* __restrict__ lvmax_w, const unsigned long long* __restrict__ lvmax_v,
             double* __restrict__ tile_acc, int* __restrict__ ticket, double* __restrict__ loc,
             int* __restrict__ counter, int item0, int n_item, int nkq, int n_pad, int fkeys, int mb_tot,
             int blk0, int tick_off, int64_t key_base, int nrhs, double* __restrict__ pair_out, int wkc, int wst_bytes,
             uint32_t dstr16) {
  using S = I8Shape<MB, TT, KS, NST, NGW>;
  constexpr int NC = S::NC;
  constexpr int NT = S::THREADS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* wst = smem;
  uint8_t* bst = smem + NST * S::WST;
  int32_t* srcf = reinterpret_cast<int32_t*>(bst + NST * S::BST);
  int32_t* keys = srcf + fkeys * TT;
  uint64_t* full = reinterpret_cast<uint64_t*>(keys + ((fkeys + 1) & ~1));  // W landed (tx bytes)
  uint64_t* fullb = full + NST;    // B gathered (one arrival per gather warp)
  uint64_t* empty = fullb + NST;   // MMAs of the stage done (tcgen05.commit)
  uint64_t* done = empty + NST;    // all MMAs of the item done
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(done + 1);
  __shared__ int s_item;
  __shared__ double csc[TT];  // S_W S_V of each tile column (its rhs' moment scale)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kp = 2 * nkq, nch = kp / kKC;
  // W ring zeroed once: rows a trimmed M-block does not store stay zero operands
  for (int i = tid * 16; i < NST * S::WST; i += (int)blockDim.x * 16) *reinterpret_cast<int4*>(wst + i) = make_int4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(fullb + s, NGW);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tbase_s;

  // gather lane plan (stage-invariant): work unit = (group of 4 target columns,
  // round of 8 pieces); lane = (column in the group, piece), so every warp
  // instruction reads 4 contiguous 128-byte runs of Mq and writes 4 SMEM wavefronts
  constexpr int RND = (KS * 4 + 7) / 8;  // rounds of 8 pieces per column (pieces: digit, kb, h)
  constexpr int U = (TT / 4) * RND;
  constexpr int UPW = (U + NGW - 1) / NGW;
  int dsto[UPW], gofs[UPW], ccol[UPW];
  if (warp >= 2) {
    const int cl = lane >> 3, p8 = lane & 7;
#pragma unroll
    for (int t = 0; t < UPW; ++t) {
      const int u = (warp - 2) + t * NGW;
      const int cg = u / RND, r = u % RND;
      const int pc = 8 * r + p8;
      const int c = 4 * cg + cl;
      const bool ok = u < U && pc < KS * 4;
      const int h = pc & 1, kb = (pc >> 1) & 1, j = pc >> 2;
      const int n = j * NC + 2 * c + h;
      dsto[t] = ok ? ((n >> 3) * 2 + kb) * 128 + (n & 7) * 16 : -1;
      gofs[t] = pc * 16;
      ccol[t] = ok ? c : 0;
    }
  }
  uint32_t qbase = 0;  // ring stages consumed by the previous items of this CTA
#pragma unroll 1
  for (int it = 0;; ++it) {
    if (tid == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int idx = s_item;
    if (idx >= n_item) break;
    const int item = item0 + idx;
    const int64_t k0 = item_k0[item], k1 = item_k1[item];
    const int nk = (int)(k1 - k0);
    const int tile = item_tile[item];
    // per-item metadata: uncompacted source slot of every (key, target column)
    for (int i = tid; i < nk * TT; i += NT) srcf[i] = -1;
    for (int i = tid; i < nk; i += NT) keys[i] = tile_keys[k0 + i];
    const int lvl = tile_level[tile];
    const int exw = level_exp(lvmax_w, lvl) + 2;
    if (tid < TT) csc[tid] = ldexp(1.0, exw + level_exp(lvmax_v, (tid % nrhs) * kMaxLevels + lvl));
    __syncthreads();
    for (int i = tid; i < nk * TT; i += NT) {
      const int64_t kk = k0 + i / TT;
      const int j = i % TT;
      if (j < tile_cnt[kk]) srcf[(i / TT) * TT + tile_cols[kk * TT + j]] = tile_src[kk * TT + j];
    }
    __syncthreads();

    // warp roles: warp 0 streams W (cp.async.bulk), warp 1 issues the MMAs,
    // warps 2.. gather the moment digits (cp.async); NST stages in a ring whose
    // position continues across items (stage qg = qbase + q)
    const int Q = nk * nch;
    if (warp == 0) {
      // the whole warp walks the ring (no divergent spinning lanes); lane 0 issues
      int kq = 0, ch = 0;
      for (int q = 0; q < Q; ++q) {
        const uint32_t qg = qbase + q;
        const int s = qg % NST;
        if (qg >= NST) mbar_wait_sleep(empty + s, ((qg / NST) - 1) & 1);
        if (lane == 0) {
          if (FDH_I8_EXP & 2) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(full + s)) : "memory");
          } else {
            w_stage_g2s<KS>(wst + s * S::WST,
                            Wq + (((int64_t)keys[kq] - key_base) * nch + ch) * (int64_t)wkc + blk0 * (KS * kCore),
                            wst_bytes, dstr16 * 16u, full + s);
          }
        }
        __syncwarp();
        if (++ch == nch) {
          ch = 0;
          ++kq;
        }
      }
    } else if (warp == 1) {
      const uint64_t dA0 = sdesc(smem_u32(wst)), dB0 = sdesc(smem_u32(bst));
      for (int q = 0; q < Q; ++q) {
        const uint32_t qg = qbase + q;
        const int s = qg % NST;
        const uint32_t ph = (qg / NST) & 1;
        mbar_wait(full + s, ph);
        mbar_wait(fullb + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          // descriptors are linear in the address (14-bit field, addr >> 4): every
          // operand offset below is a compile-time constant added to the stage base
          // (keeps the issuing thread at ~3 instructions per MMA)
          const uint64_t dA = dA0 + (uint64_t)((s * S::WST) >> 4), dB = dB0 + (uint64_t)((s * S::BST) >> 4);
          if (q > 0) issue_stage<MB, KS, S::LV, NC, false>(tmem, dA, dB);
          else issue_stage<MB, KS, S::LV, NC, true>(tmem, dA, dB);
          mma_commit(empty + s);
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(done);
      __syncwarp();
    } else {
      // gather: G groups of cp.async in flight per thread; a stage's arrival on
      // fullb follows its own wait_group + proxy fence
      int kq = 0, ch = 0;
      auto arrive = [&](uint32_t qa) {  // one arrival per warp once all its lanes' pieces landed
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(fullb + qa % NST)) : "memory");
      };
      for (int q = 0; q < Q; ++q) {
        const uint32_t qg = qbase + q;
        const int s = qg % NST;
        if (qg >= NST) mbar_wait_sleep(empty + s, ((qg / NST) - 1) & 1);
        uint8_t* bb = bst + s * S::BST;
        const int32_t* sf = srcf + kq * TT;
        const int8_t* mq = Mq + (int64_t)ch * (KS * 64);
#pragma unroll
        for (int t = 0; t < UPW; ++t) {
          if (dsto[t] < 0 || (FDH_I8_EXP & 1)) continue;
          const int src = sf[ccol[t]];
          if (src >= 0) cp_async16(bb + dsto[t], mq + (int64_t)src * nch * (KS * 64) + gofs[t]);
          else *reinterpret_cast<int4*>(bb + dsto[t]) = make_int4(0, 0, 0, 0);
        }
        cp_async_commit();
        if (q >= G) {
          cp_async_wait<G>();
          arrive(qg - G);
        }
        if (++ch == nch) {
          ch = 0;
          ++kq;
        }
      }
      cp_async_wait<0>();
      for (int qa = Q > G ? Q - G : 0; qa < Q; ++qa) arrive(qbase + qa);
    }
    // all MMAs of the item done
    mbar_wait_sleep(done, it & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- epilogue: levels -> FP64, chained accumulation into the tile
    const int seq = item_seq[item], nit = tile_nitem[tile];
    if (seq > 0) {
      if (tid == 0)
        while (ld_acquire(ticket + tick_off + tile) != seq) __nanosleep(100);
      __syncthreads();
    }
    const bool last = seq == nit - 1;
    double fL[S::LV];  // level weights 2^(-7(L+2)); the power-of-two scale S_W S_V of the
                       // column's rhs is applied after the (exact) level sum
#pragma unroll
    for (int L = 0; L < S::LV; ++L) fL[L] = ldexp(1.0, -kI8Bits * (L + 2));
    double* A = tile_acc + (int64_t)tile * n_pad * NC;
    const int qw = warp & 3;  // TMEM lane quarter of this warp
#pragma unroll 1
    for (int b = 0; b < MB && (NGW == 2 || (warp >= 2 && warp < 6)); ++b) {
      const int row = (blk0 + b) * 128 + qw * 32 + lane;
#pragma unroll 1
      for (int g = 0; g < NC / 8; ++g) {
        uint32_t r[S::LV][8];
#pragma unroll
        for (int L = 0; L < S::LV; ++L)
          tmem_ld8(tmem + ((uint32_t)(qw * 32) << 16) + b * S::LV * NC + L * NC + 8 * g, r[L]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row >= n_pad) continue;
        double v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          double a = 0.0;
#pragma unroll
          for (int L = S::LV - 1; L >= 0; --L) a += i32_to_f64(r[L][e]) * fL[L];
          v[e] = a * csc[(8 * g + e) >> 1];  // exact: a power of two
        }
        double* pa = A + (int64_t)row * NC + 8 * g;
        if (seq > 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] += __ldcg(pa + e);
        }
        if (pair_out) {  // pair mode: one key per item, the pair's values to the output buffer
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int col = 8 * g + e;
            pair_out[((int64_t)idx * TT + (col >> 1)) * 2 * n_pad + (col & 1) * n_pad + row] = v[e];
          }
        } else if (last) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int col = 8 * g + e;
            const int32_t ts = tile_tslot[tile * TT + (col >> 1)];
            if (ts >= 0) loc[(int64_t)ts * 2 * n_pad + (col & 1) * n_pad + row] = v[e];
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) __stcg(pa + e, v[e]);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (!last) {
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release(ticket + tick_off + tile, seq + 1);
    } else {
      __syncthreads();
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    qbase += (uint32_t)Q;
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- M2L, pipelined
// The same work items, digits and arithmetic as k_m2l_i8, with the roles fully
// decoupled by mbarriers so that item boundaries do not drain the pipeline:
//   warp 0      claims items in order (atomic counter), publishes {item} in a
//               2-deep ring (meta_full / meta_empty) and streams W (cp.async.bulk);
//   warp 1      issues the MMAs; before the first MMA of an item it waits until the
//               epilogue warps have read the previous item's TMEM (tfree), after the
//               last it commits tmem_full;
//   warps 2..   gather the moment digits; the source slot of each target column
//   2+NGW-1     is rebuilt per key in registers from the compacted (tile, key) row
//               (warp shuffles), prefetched one key ahead;
//   4 warps     epilogue (TMEM -> FP64 -> chained tile accumulator / locals / pair
//               buffer), the ticket chain as before; its TMEM read overlaps the
//               next item's W / moment loads.
// Forward progress: as k_m2l_i8 (items claimed in increasing order by running CTAs).
template <int MB, int TT, int KS, int NST, int NGW>
__global__ void __maxnreg__(128)
    k_m2l_i8p(const int32_t* __restrict__ item_tile, const int32_t* __restrict__ item_seq,
              const int64_t* __restrict__ item_k0, const int64_t* __restrict__ item_k1,
              const int32_t* __restrict__ tile_nitem, const int32_t* __restrict__ tile_tslot,
              const int32_t* __restrict__ tile_level, const int32_t* __restrict__ tile_keys,
              const int32_t* __restrict__ tile_src, const uint8_t* __restrict__ tile_cols,
              const uint8_t* __restrict__ tile_cnt, const int8_t* __restrict__ Wq, const int8_t* __restrict__ Mq,
              const unsigned long long* __restrict__ lvmax_w, const unsigned long long* __restrict__ lvmax_v,
              double* __restrict__ tile_acc, int* __restrict__ ticket, double* __restrict__ loc,
              int* __restrict__ counter, int item0, int n_item, int nkq, int n_pad, int mb_tot, int blk0,
              int tick_off, int64_t key_base, int nrhs, double* __restrict__ pair_out, int wkc, int wst_bytes,
              uint32_t dstr16) {
  using S = I8Shape<MB, TT, KS, NST, NGW>;
  constexpr int NC = S::NC;
  constexpr int EW0 = 2 + NGW;  // first epilogue warp
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* wst = smem;
  uint8_t* bst = smem + NST * S::WST;
  uint64_t* full = reinterpret_cast<uint64_t*>(bst + NST * S::BST);
  uint64_t* fullb = full + NST;
  uint64_t* empty = fullb + NST;
  uint64_t* meta_full = empty + NST;   // [2]
  uint64_t* meta_empty = meta_full + 2;  // [2]: NGW gather + 1 MMA + 4 epilogue warps
  uint64_t* tmem_full = meta_empty + 2;
  uint64_t* tfree = tmem_full + 1;
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tfree + 1);
  __shared__ int s_idx[2];
  __shared__ double csc[TT];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kp = 2 * nkq, nch = kp / kKC;
  // W ring zeroed once: rows a trimmed M-block does not store stay zero operands
  for (int i = tid * 16; i < NST * S::WST; i += (int)blockDim.x * 16) *reinterpret_cast<int4*>(wst + i) = make_int4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(fullb + s, NGW);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(meta_full + b, 1);
      mbar_init(meta_empty + b, NGW + 1 + 4);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tfree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tbase_s;

  if (warp == 0) {
    // ---------------- producer: claims + W stream
    uint32_t qbase = 0;
    for (int it = 0;; ++it) {
      const int b = it & 1;
      if (it >= 2) mbar_wait_sleep(meta_empty + b, ((it - 2) >> 1) & 1);
      int idx = 0;
      if (lane == 0) {
        idx = atomicAdd(counter, 1);
        s_idx[b] = idx;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(meta_full + b)) : "memory");
      }
      idx = __shfl_sync(0xffffffffu, idx, 0);
      if (idx >= n_item) break;
      const int item = item0 + idx;
      const int64_t k0 = item_k0[item], k1 = item_k1[item];
      const int Q = (int)(k1 - k0) * nch;
      int kq = 0, ch = 0;
      int key = tile_keys[k0];
      for (int q = 0; q < Q; ++q) {
        const uint32_t qg = qbase + q;
        const int s = qg % NST;
        if (qg >= NST) mbar_wait_sleep(empty + s, ((qg / NST) - 1) & 1);
        if (lane == 0) {
          w_stage_g2s<KS>(wst + s * S::WST,
                          Wq + (((int64_t)key - key_base) * nch + ch) * (int64_t)wkc + blk0 * (KS * kCore), wst_bytes,
                          dstr16 * 16u, full + s);
        }
        __syncwarp();
        if (++ch == nch) {
          ch = 0;
          ++kq;
          if (k0 + kq < k1) key = tile_keys[k0 + kq];
        }
      }
      qbase += (uint32_t)Q;
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint64_t dA0 = sdesc(smem_u32(wst)), dB0 = sdesc(smem_u32(bst));
    uint32_t qbase = 0;
    for (int it = 0;; ++it) {
      const int b = it & 1;
      mbar_wait(meta_full + b, (it >> 1) & 1);
      const int idx = s_idx[b];
      if (idx >= n_item) break;
      const int item = item0 + idx;
      const int Q = (int)(item_k1[item] - item_k0[item]) * nch;
      if (it >= 1) mbar_wait(tfree, (it - 1) & 1);  // the epilogue has read the previous item's TMEM
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int q = 0; q < Q; ++q) {
        const uint32_t qg = qbase + q;
        const int s = qg % NST;
        const uint32_t ph = (qg / NST) & 1;
        mbar_wait(full + s, ph);
        mbar_wait(fullb + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint64_t dA = dA0 + (uint64_t)((s * S::WST) >> 4), dB = dB0 + (uint64_t)((s * S::BST) >> 4);
          if (q > 0) issue_stage<MB, KS, S::LV, NC, false>(tmem, dA, dB);
          else issue_stage<MB, KS, S::LV, NC, true>(tmem, dA, dB);
          mma_commit(empty + s);
        }
        __syncwarp();
      }
      if (lane == 0) {
        mma_commit(tmem_full);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(meta_empty + b)) : "memory");
      }
      __syncwarp();
      qbase += (uint32_t)Q;
    }
  } else if (warp < EW0) {
    // ---------------- gather
    constexpr int RND = (KS * 4 + 7) / 8;
    constexpr int U = (TT / 4) * RND;
    constexpr int UPW = (U + NGW - 1) / NGW;
    // cp.async groups (stages) in flight per gather warp beyond the one being issued
    constexpr int G = FDH_I8P_G < NST - 1 ? FDH_I8P_G : NST - 2;
    static_assert(G >= 1, "gather depth");
    int dsto[UPW], gofs[UPW], ccol[UPW];
    {
      const int cl = lane >> 3, p8 = lane & 7;
#pragma unroll
      for (int t = 0; t < UPW; ++t) {
        const int u = (warp - 2) + t * NGW;
        const int cg = u / RND, r = u % RND;
        const int pc = 8 * r + p8;
        const int c = 4 * cg + cl;
        const bool ok = u < U && pc < KS * 4;
        const int h = pc & 1, kb = (pc >> 1) & 1, j = pc >> 2;
        const int n = j * NC + 2 * c + h;
        dsto[t] = ok ? ((n >> 3) * 2 + kb) * 128 + (n & 7) * 16 : -1;
        gofs[t] = pc * 16;
        ccol[t] = ok ? c : 0;
      }
    }
    auto arrive = [&](uint32_t qa) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(fullb + qa % NST)) : "memory");
    };
    // source slot of column `lane` of the compacted (tile, key) row kk (-1: absent)
    auto row_src = [&](int64_t kk, int& col, int& src) {
      const int cnt = tile_cnt[kk];
      col = lane < cnt ? (int)tile_cols[kk * TT + lane] : -1;
      src = lane < cnt ? tile_src[kk * TT + lane] : -1;
    };
    auto expand = [&](int col, int src) {  // lane = column -> its source slot
      int mine = -1;
#pragma unroll 4
      for (int j = 0; j < TT; ++j) {
        const int cj = __shfl_sync(0xffffffffu, col, j), sj = __shfl_sync(0xffffffffu, src, j);
        if (cj == lane) mine = sj;
      }
      return mine;
    };
    uint32_t qbase = 0;
    for (int it = 0;; ++it) {
      const int b = it & 1;
      mbar_wait_sleep(meta_full + b, (it >> 1) & 1);
      const int idx = s_idx[b];
      if (idx >= n_item) break;
      const int item = item0 + idx;
      const int64_t k0 = item_k0[item], k1 = item_k1[item];
      const int Q = (int)(k1 - k0) * nch;
      int ncol, nsrc;
      row_src(k0, ncol, nsrc);
      int srcl = expand(ncol, nsrc);
      if (k0 + 1 < k1) row_src(k0 + 1, ncol, nsrc);  // prefetch the next key's row
      int srcv[UPW];
#pragma unroll
      for (int t = 0; t < UPW; ++t) srcv[t] = __shfl_sync(0xffffffffu, srcl, ccol[t]);
      int kq = 0, ch = 0;
      for (int q = 0; q < Q; ++q) {
        const uint32_t qg = qbase + q;
        const int s = qg % NST;
        if (qg >= NST) mbar_wait_sleep(empty + s, ((qg / NST) - 1) & 1);
        uint8_t* bb = bst + s * S::BST;
        const int8_t* mq = Mq + (int64_t)ch * (KS * 64);
#pragma unroll
        for (int t = 0; t < UPW; ++t) {
          if (dsto[t] < 0) continue;
          if (srcv[t] >= 0) cp_async16(bb + dsto[t], mq + (int64_t)srcv[t] * nch * (KS * 64) + gofs[t]);
          else *reinterpret_cast<int4*>(bb + dsto[t]) = make_int4(0, 0, 0, 0);
        }
        cp_async_commit();
        if (q >= G) {
          cp_async_wait<G>();
          arrive(qg - G);
        }
        if (++ch == nch) {
          ch = 0;
          ++kq;
          if (k0 + kq < k1) {
            srcl = expand(ncol, nsrc);
            if (k0 + kq + 1 < k1) row_src(k0 + kq + 1, ncol, nsrc);
#pragma unroll
            for (int t = 0; t < UPW; ++t) srcv[t] = __shfl_sync(0xffffffffu, srcl, ccol[t]);
          }
        }
      }
      cp_async_wait<0>();
      for (int qa = Q > G ? Q - G : 0; qa < Q; ++qa) arrive(qbase + qa);
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(meta_empty + b)) : "memory");
      qbase += (uint32_t)Q;
    }
  } else {
    // ---------------- epilogue (4 warps, TMEM lane quarter = warp & 3)
    const int qw = warp & 3;
    double fL[S::LV];
#pragma unroll
    for (int L = 0; L < S::LV; ++L) fL[L] = ldexp(1.0, -kI8Bits * (L + 2));
    for (int it = 0;; ++it) {
      const int b = it & 1;
      mbar_wait_sleep(meta_full + b, (it >> 1) & 1);
      const int idx = s_idx[b];
      if (idx >= n_item) break;
      const int item = item0 + idx;
      const int tile = item_tile[item];
      const int seq = item_seq[item], nit = tile_nit_guard(tile_nitem, tile);
      const int lvl = tile_level[tile];
      mbar_wait_sleep(tmem_full, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // csc and the ticket wait among the 4 epilogue warps (named barrier 1)
      if (warp == EW0 && lane < TT)
        csc[lane] = ldexp(1.0, level_exp(lvmax_w, lvl) + 2 + level_exp(lvmax_v, (lane % nrhs) * kMaxLevels + lvl));
      if (seq > 0 && warp == EW0 && lane == 0)
        while (ld_acquire(ticket + tick_off + tile) != seq) __nanosleep(100);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const bool last = seq == nit - 1;
      double* A = tile_acc + (int64_t)tile * n_pad * NC;
#pragma unroll 1
      for (int bb = 0; bb < MB; ++bb) {
        const int row = (blk0 + bb) * 128 + qw * 32 + lane;
#pragma unroll 1
        for (int g = 0; g < NC / 8; ++g) {
          uint32_t r[S::LV][8];
#pragma unroll
          for (int L = 0; L < S::LV; ++L)
            tmem_ld8(tmem + ((uint32_t)(qw * 32) << 16) + bb * S::LV * NC + L * NC + 8 * g, r[L]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (row >= n_pad) continue;
          double v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            double a = 0.0;
#pragma unroll
            for (int L = S::LV - 1; L >= 0; --L) a += i32_to_f64(r[L][e]) * fL[L];
            v[e] = a * csc[(8 * g + e) >> 1];
          }
          if (pair_out) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int col = 8 * g + e;
              pair_out[((int64_t)idx * TT + (col >> 1)) * 2 * n_pad + (col & 1) * n_pad + row] = v[e];
            }
            continue;
          }
          double* pa = A + (int64_t)row * NC + 8 * g;
          if (seq > 0) {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] += __ldcg(pa + e);
          }
          if (last) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int col = 8 * g + e;
              const int32_t ts = tile_tslot[tile * TT + (col >> 1)];
              if (ts >= 0) loc[(int64_t)ts * 2 * n_pad + (col & 1) * n_pad + row] = v[e];
            }
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) __stcg(pa + e, v[e]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      if (!last) __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == EW0 && lane == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(tfree)) : "memory");
        if (!last) st_release(ticket + tick_off + tile, seq + 1);
      }
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(meta_empty + b)) : "memory");
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int MB, int TT, int NST, int NGW>
size_t i8p_smem() {
  using S = I8Shape<MB, TT, kI8Digits, NST, NGW>;
  return (size_t)NST * S::STAGE + (3 * NST + 6) * 8 + 16;
}

inline int m2l_i8_wgroup_of(int mb, int tile) { return (tile == 16 && mb >= 2) ? 2 : 1; }
// W addressing of one pass: bytes per (key, K chunk), bytes per stage, digit stride / 16
struct WPass { int wkc, wst; uint32_t dstr16; };
template <int MB>
WPass wpass(const M2LI8Args& a, int mb_tot, int blk0, bool trimmed) {
  if (!trimmed) return {kI8Digits * mb_tot * kCore, kI8Digits * MB * kCore, (uint32_t)(kCore >> 4)};
  const int rows = std::min(128, a.n_pad - 128 * blk0);  // MB == 1
  return {kI8Digits * a.n_pad * kKC, kI8Digits * rows * kKC, (uint32_t)((rows * kKC) >> 4)};
}

template <int MB, int TT, int NST, int NGW>
void run_i8p(cudaStream_t st, const M2LI8Args& a, int mb_tot, int blk0, int pass) {
  const WPass w = wpass<MB>(a, mb_tot, blk0, m2l_i8_wgroup_of(mb_tot, TT) == 1);
  auto kern = k_m2l_i8p<MB, TT, kI8Digits, NST, NGW>;
  const size_t sm = i8p_smem<MB, TT, NST, NGW>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = std::max(1, std::min(a.n_item, nsm));
  kern<<<grid, (2 + NGW + 4) * 32, sm, st>>>(a.item_tile, a.item_seq, a.item_k0, a.item_k1, a.tile_nitem,
                                            a.tile_tslot, a.tile_level, a.tile_keys, a.tile_src, a.tile_cols,
                                            a.tile_cnt, a.Wq, a.Mq, a.lvmax_w, a.lvmax_v, a.tile_acc, a.ticket, a.loc,
                                            a.counter + pass, a.item0, a.n_item, a.nkq, a.n_pad, mb_tot, blk0,
                                            pass * a.n_tile, a.key_base, a.nrhs, a.pair_out, w.wkc, w.wst, w.dstr16);
}

template <int MB, int TT, int NST, int NGW>
size_t i8_smem(int fkeys) {
  using S = I8Shape<MB, TT, kI8Digits, NST, NGW>;
  return (size_t)NST * S::STAGE + (size_t)fkeys * TT * 4 + (size_t)((fkeys + 1) & ~1) * 4 + (3 * NST + 1) * 8 + 16;
}

template <int MB, int TT, int NST, int NGW, int G>
void run_i8(cudaStream_t st, const M2LI8Args& a, int mb_tot, int blk0, int pass) {
  const WPass w = wpass<MB>(a, mb_tot, blk0, m2l_i8_wgroup_of(mb_tot, TT) == 1);
  using S = I8Shape<MB, TT, kI8Digits, NST, NGW>;
  auto kern = k_m2l_i8<MB, TT, kI8Digits, NST, NGW, G>;
  const size_t sm = i8_smem<MB, TT, NST, NGW>(a.fkeys);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::THREADS, sm);
  const int grid = std::max(1, std::min(a.n_item, nsm * std::max(1, per_sm)));
  kern<<<grid, S::THREADS, sm, st>>>(a.item_tile, a.item_seq, a.item_k0, a.item_k1, a.tile_nitem, a.tile_tslot,
                                     a.tile_level, a.tile_keys, a.tile_src, a.tile_cols, a.tile_cnt, a.Wq, a.Mq,
                                     a.lvmax_w, a.lvmax_v, a.tile_acc, a.ticket, a.loc, a.counter + pass, a.item0,
                                     a.n_item, a.nkq, a.n_pad, a.fkeys, mb_tot, blk0, pass * a.n_tile, a.key_base,
                                     a.nrhs, a.pair_out, w.wkc, w.wst, w.dstr16);
}

}  // namespace

int m2l_i8_supported(int n, int tile) {
  const int mb = (n + 127) / 128;
  return (mb == 1 && tile == 32) || ((mb == 2 || mb == 3) && tile == 16) || (mb >= 2 && tile == 32);
}
int m2l_i8_fkeys(int nkq) {
  // |digit| <= kI8DigitMax: one key adds at most KS * KP * max^2 to a level accumulator
  const int64_t per_key = (int64_t)kI8Digits * 2 * nkq * kI8DigitMax * kI8DigitMax;
  const int64_t f = (int64_t)0x7fffffff / per_key;
  return (int)std::min<int64_t>(256, f);
}
int64_t m2l_i8_wbytes_per_key(int n, int nkq, int tile) {
  const int rows = m2l_i8_wgroup(n, tile) == 1 ? i8_rows_total(n) : (n + 127) / 128 * 128;  // trimmed last M-block
  return (int64_t)kI8Digits * rows * kKC * (2 * nkq / kKC);
}
int64_t m2l_i8_mbytes_per_slot(int nkq) { return (int64_t)kI8Digits * 2 * 2 * nkq; }

void launch_coupling_i8(cudaStream_t st, const Consts* C, const double* dirtab, int64_t key0, int64_t nkeys,
                        const int32_t* key_level, const int64_t* key_d, const int32_t* key_dir, int pass,
                        unsigned long long* lvmax, int8_t* Wq, int n, int nkq, int gs, int64_t key_base) {
  if (nkeys <= 0) return;
  dim3 grid((unsigned)nkeys, (unsigned)((n + kCplRows - 1) / kCplRows));
  const size_t sm = pass ? (size_t)kI8Digits * (2 * nkq / kKC) * 256 : 0;
  // static shared (node tables) counts towards the 48 KB default; the attribute is per
  // device (n_gpus > 1), so it is set on every launch that needs it
  if (sm > 40 * 1024)
    cudaFuncSetAttribute(k_coupling_i8<kI8Digits>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_coupling_i8<kI8Digits><<<grid, 256, sm, st>>>(C, dirtab, key0, key_level, key_d, key_dir, pass, lvmax, Wq, n, nkq,
                                                  (n + 127) / 128, gs, key_base);
}
void launch_mom_quant(cudaStream_t st, const double* mom, const int32_t* slot_level, int64_t nslots, int n, int n_pad,
                      int nkq, unsigned long long* lvmax_v, int8_t* Mq, int nrhs) {
  if (nslots <= 0) return;
  cudaMemsetAsync(lvmax_v, 0, sizeof(unsigned long long) * kMaxLevels * nrhs, st);
  const unsigned nb = (unsigned)(nslots * nrhs);
  k_mom_max<<<nb, 128, 0, st>>>(mom, slot_level, n, n_pad, lvmax_v, nslots);
  k_mom_quant<kI8Digits><<<nb, 128, 0, st>>>(mom, slot_level, lvmax_v, n, n_pad, nkq, Mq, nslots);
}
// pipeline depth: as many K-chunk stages as fit in shared memory beside `reserve`
// bytes (item tables, barriers, static shared), at most 8
constexpr int kSmemMax = 232448;
constexpr int nst_fit(int mb, int tt, int reserve) {
  const int stage = kI8Digits * mb * kCore + kI8Digits * 2 * tt * kKC;
  const int n = (kSmemMax - reserve) / stage;
  return n > 8 ? 8 : (n < 3 ? 3 : n);
}

constexpr int gdepth(int nst) { return FDH_I8P_G < nst - 1 ? FDH_I8P_G : nst - 2; }

int launch_m2l_i8(cudaStream_t st, int n, int tile, const M2LI8Args& a) {
  if (a.n_item <= 0) return 0;
  const int mb = (n + 127) / 128;
  // the pipelined kernel (k_m2l_i8p) for two or more M-blocks and for pair items
  // (measured: config 5 pair mode 964 -> 817 ms, m = 6 hybrid 3337 -> 3176 ms) and
  // k_m2l_i8 for one M-block target tiles (m <= 4: 29.3 vs 32.5 ms on config 2);
  // FDH_I8_PIPE=0 / 1 forces one of them (profiles/r02_m2l_pipe_ab.log)
  static const int pipe_env = [] {
    const char* e = std::getenv("FDH_I8_PIPE");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  const bool pipe = pipe_env >= 0 ? pipe_env == 1 : !(mb == 1 && a.pair_out == nullptr);
  // passes over the item list (m2l_i8_passes): one per M-block group; a.counter
  // holds one zeroed claim counter per pass (and per segment)
  constexpr int kResP = 4096;  // barriers + static shared + alignment (k_m2l_i8p)
  if (pipe) {
    if (mb == 1 && tile == 32) {
      run_i8p<1, 32, nst_fit(1, 32, kResP), 8>(st, a, 1, 0, 0);
    } else if (mb == 2 && tile == 16) {
      run_i8p<2, 16, nst_fit(2, 16, kResP), 8>(st, a, 2, 0, 0);
    } else if (mb == 3 && tile == 16) {
      run_i8p<2, 16, nst_fit(2, 16, kResP), 8>(st, a, 3, 0, 0);
      run_i8p<1, 16, nst_fit(1, 16, kResP), 8>(st, a, 3, 2, 1);
    } else if (mb >= 2 && tile == 32) {
      for (int b = 0; b < mb; ++b) run_i8p<1, 32, nst_fit(1, 32, kResP), 8>(st, a, mb, b, b);
    } else {
      return 1;
    }
    return 0;
  }
  // k_m2l_i8 keeps per-item tables of fkeys x (TT + 1) int32 beside the ring
  constexpr int kFkMax = 256;
  if (a.fkeys > kFkMax) return 1;
  if (mb == 1 && tile == 32) {
    constexpr int R = kResP + kFkMax * 33 * 4;
    if (i8_smem<1, 32, nst_fit(1, 32, kResP + 128 * 33 * 4), 8>(a.fkeys) + 2048 <= (size_t)kSmemMax)
      run_i8<1, 32, nst_fit(1, 32, kResP + 128 * 33 * 4), 8, gdepth(nst_fit(1, 32, kResP + 128 * 33 * 4))>(st, a, 1, 0, 0);
    else
      run_i8<1, 32, nst_fit(1, 32, R), 8, gdepth(nst_fit(1, 32, R))>(st, a, 1, 0, 0);
  } else if (mb == 2 && tile == 16) {
    run_i8<2, 16, nst_fit(2, 16, kResP + kFkMax * 17 * 4), 8, gdepth(nst_fit(2, 16, kResP + kFkMax * 17 * 4))>(st, a, 2, 0, 0);
  } else if (mb == 3 && tile == 16) {
    // 352 rows (m = 6): TMEM holds the levels x 32 columns for two M-blocks only, so
    // the rows run as two M-block groups {0, 1} and {2}, each its own pass over the
    // items with its own ticket chain (same moment gather, disjoint W and rows)
    run_i8<2, 16, nst_fit(2, 16, kResP + kFkMax * 17 * 4), 8, gdepth(nst_fit(2, 16, kResP + kFkMax * 17 * 4))>(st, a, 3, 0, 0);
    run_i8<1, 16, nst_fit(1, 16, kResP + kFkMax * 17 * 4), 8, gdepth(nst_fit(1, 16, kResP + kFkMax * 17 * 4))>(st, a, 3, 2, 1);
  } else if (mb >= 2 && tile == 32) {
    // 32 target columns: one 128-row M-block per pass
    for (int b = 0; b < mb; ++b) {
      if (i8_smem<1, 32, nst_fit(1, 32, kResP + 128 * 33 * 4), 8>(a.fkeys) + 2048 <= (size_t)kSmemMax)
        run_i8<1, 32, nst_fit(1, 32, kResP + 128 * 33 * 4), 8, gdepth(nst_fit(1, 32, kResP + 128 * 33 * 4))>(st, a, mb, b, b);
      else
        run_i8<1, 32, nst_fit(1, 32, kResP + kFkMax * 33 * 4), 8, gdepth(nst_fit(1, 32, kResP + kFkMax * 33 * 4))>(st, a, mb, b, b);
    }
  } else {
    return 1;
  }
  return 0;
}

namespace {
// pair mode: loc[t] += sum of its pairs' outputs of this segment [p0, p1), in pair
// order (cursor[t] advances through the slot's sorted pair list segment by segment)
__global__ void __launch_bounds__(256) k_m2l_reduce(const int64_t* __restrict__ red_ptr,
                                                    const int64_t* __restrict__ red_idx, int64_t* __restrict__ cursor,
                                                    const double* __restrict__ out, int64_t p0, int64_t p1,
                                                    double* __restrict__ loc, int n_pad) {
  const int64_t t = blockIdx.x;
  const int64_t c0 = cursor[t], c1 = red_ptr[t + 1];
  if (c0 >= c1 || red_idx[c0] >= p1) return;
  int64_t ce = c0;  // the slot's pairs in this segment: [c0, ce)
  while (ce < c1 && red_idx[ce] < p1) ++ce;
  // a running sum continued across segments: the same rounding whatever the segment cuts
  for (int r = threadIdx.x; r < 2 * n_pad; r += blockDim.x) {
    double a = loc[t * 2 * n_pad + r];
    for (int64_t c = c0; c < ce; ++c) a += out[(red_idx[c] - p0) * 2 * n_pad + r];
    loc[t * 2 * n_pad + r] = a;
  }
  if (threadIdx.x == 0) cursor[t] = ce;
}
}  // namespace

void launch_m2l_reduce(cudaStream_t st, int64_t nslots, const int64_t* red_ptr, const int64_t* red_idx,
                       int64_t* cursor, const double* out, int64_t p0, int64_t p1, double* loc, int n_pad) {
  if (nslots <= 0) return;
  k_m2l_reduce<<<(unsigned)nslots, 256, 0, st>>>(red_ptr, red_idx, cursor, out, p0, p1, loc, n_pad);
}

namespace {
__global__ void __launch_bounds__(256) k_m2l_add(double* __restrict__ loc, const double* __restrict__ add, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    loc[i] += add[i];
}
}  // namespace
// hybrid mode: locals = target-tile part (assigned by the tiles' last items) + pair part
// (its own running sum): one fixed addition per entry, whatever the segment order
void launch_m2l_add(cudaStream_t st, double* loc, const double* add, int64_t n) {
  if (n <= 0) return;
  k_m2l_add<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(loc, add, n);
}

int m2l_i8_passes(int n, int tile) {
  const int mb = (n + 127) / 128;
  if (tile == 32) return mb;
  return mb > 2 ? 2 : 1;
}
int m2l_i8_wgroup(int n, int tile) { return m2l_i8_wgroup_of((n + 127) / 128, tile); }

}  // namespace fdhelm
