// k_m2l.cu -- coupling matrices and the M2L phase on FP64 DMMA (sm_100a).
//
// M2L: g~_{t,c} += A_{c,t x s} v~_{s,c} for every admissible
// leaf (t,s).  A depends only on the key (level, lattice offset) (PAPER.md:397-399,
// SPEC.md:422-439), so the pairs of a TILE of target slots (same level, direction
// and lattice parity -> nearly identical key lists) form, per key, a real GEMM
//
//     C[n_pad x 2T] += W_key[n_pad x 2 n_k] * B[2 n_k x 2T]   (n_pad = rows, multiple of 32;
//                                                              n_k = K half, multiple of 8)
//     W = [Re A | Im A],  B(:,2j) = [Re v_j ; -Im v_j],  B(:,2j+1) = [Im v_j ; Re v_j]
//
// so that C(:,2j) = Re(A v_j) and C(:,2j+1) = Im(A v_j): the complex product is a
// single real GEMM with 8 n^2 flops per block.  Groups of 8
// targets instead use the 3-multiplication (Gauss) product, 6 n^2 flops:
//     P1 = Re A Re v,  P2 = Im A Im v,  P3 = (Re A + Im A)(Re v + Im v),
//     Re(A v) = P1 - P2,  Im(A v) = P3 - P1 - P2,
// with Re A + Im A stored as a third plane of W.  The FP64 tensor pipe and the
// DFMA pipe share one ~37 TF/s budget on B200 (tools/fp64_mix.cu), so fewer
// issued flops is the only way past it.  It runs on
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), the only FP64 tensor-core path on
// sm_100a (tcgen05 has no f64 kind).  Each warp owns 32 rows x 2T columns in
// registers; A fragments stream from L2 straight into registers (no reuse
// across warps), the gathered moments are staged once per key in shared
// memory (cp.async) and shared by all warps.  Work items (tile, key chunk) run
// chunk-major for L2 reuse of the coupling matrices; the items of a tile are
// chained in chunk order (deterministic, no FP atomics).
#include "kernels.hpp"

#ifndef FDH_KUNROLL
#define FDH_KUNROLL 0
#endif
#ifndef FDH_M2L_TRACE
#define FDH_M2L_TRACE 0
#endif
#ifndef FDH_M2L_MINB
#define FDH_M2L_MINB 0
#endif

namespace fdhelm {

#if FDH_M2L_TRACE
// debug build only: per-phase SM cycles of warp 0 of every M2L CTA
__device__ unsigned long long g_m2l_trace[8];
#define FDH_TR_T(v) const long long v = clock64()
#define FDH_TR_ADD(i, d) \
  if (threadIdx.x == 0) atomicAdd(&g_m2l_trace[i], (unsigned long long)(d))
#else
#define FDH_TR_T(v)
#define FDH_TR_ADD(i, d)
#endif

namespace {

constexpr double kFourPi = 4.0 * 3.14159265358979323846;  // geometry.hpp:11

// ---------------------------------------------------------- coupling gen
// W[key][j][k] = Re f_c(xi_t,j, xi_s,k),  W[key][j][n_k + k] = Im f_c(...),
// W[key][j][2 n_k + k] = Re f_c + Im f_c (the Gauss plane)
// canonical frame: s at the lattice origin, t at offset d.
constexpr int kCplRows = 8;
__global__ void __launch_bounds__(256) k_coupling(const Consts* __restrict__ C, const double* __restrict__ dirtab,
                                                  int64_t key0, const int32_t* __restrict__ key_level,
                                                  const int64_t* __restrict__ key_d, const int32_t* __restrict__ key_dir,
                                                  double* __restrict__ W, int n, int n_pad, int n_k, int64_t wbase) {
  __shared__ double tn[3][kMaxP], sn[3][kMaxP];
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
  const int np = m2l_wplanes(n_pad);
  double* Wk = W + (key - wbase) * n_pad * np * n_k;
  for (int idx = threadIdx.x; idx < kCplRows * n_k; idx += blockDim.x) {
    const int j = r0 + idx / n_k, k = idx % n_k;
    if (j >= n_pad) continue;
    double re = 0.0, im = 0.0;
    if (j < n && k < n) {
      const double d[3] = {__dsub_rn(tn[0][j / (p * p)], sn[0][k / (p * p)]),
                           __dsub_rn(tn[1][(j / p) % p], sn[1][(k / p) % p]),
                           __dsub_rn(tn[2][j % p], sn[2][k % p])};
      const double r = sqrt(dot3(d, d));  // geometry.hpp:92-98
      const double ph = __dmul_rn(kappa, __dsub_rn(r, dot3(d, cv)));
      const double w = __ddiv_rn(1.0, __dmul_rn(kFourPi, r));
      double s, co;
      sincos(ph, &s, &co);
      re = __dmul_rn(w, co);
      im = __dmul_rn(w, s);
    }
    // k-interleaved within blocks of 8 (k = 8b + 4h + q stored at 8b + 2q + h), so
    // that a lane's A fragments of two consecutive k-steps are one 16-byte load
    const int kp = (k & ~7) | ((k & 3) << 1) | ((k >> 2) & 1);
    Wk[(int64_t)j * np * n_k + kp] = re;
    Wk[(int64_t)j * np * n_k + n_k + kp] = im;
    if (np == 3) Wk[(int64_t)j * np * n_k + 2 * n_k + kp] = re + im;  // Gauss plane
  }
}

// ---------------------------------------------------------------- DMMA
__device__ __forceinline__ void dmma8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
template <int NPAD, int NK, int TT>
struct M2LShape {
  static constexpr int K3 = m2l_wplanes(NPAD) * NK;  // W row length: [Re A | Im A (| Re A + Im A)]
  static constexpr int GS = 2 * NPAD;       // moment slot stride in HBM ([Re | Im] planes of NPAD)
  // smem moment column: [Re (NK) | pad | Im (NK) | pad], IMOFF == 8 and MS == 4 (mod 16):
  // both B-fragment patterns (4 columns x Re/Im x 4 k, and 4 columns x 4 k per
  // half-warp) hit 16 distinct 8-byte banks
  static constexpr int IMOFF = NK + ((NK % 16 == 0) ? 8 : 0);
  static constexpr int MS = IMOFF + NK + ((4 - (IMOFF + NK)) % 16 + 16) % 16;
  static_assert(NK % 8 == 0 && IMOFF % 16 == 8 && MS % 16 == 4, "bank-conflict-free B fragments");
  // Gauss product for n_pad <= 128; above, its 1.5x accumulators would cost a
  // resident CTA (n_pad 224: 2 -> 1 CTA/SM), so the real GEMM keeps all 4 n-tiles
  static constexpr bool GAUSS = m2l_gauss(NPAD);
  static_assert(GAUSS || TT == 16, "32-target tiles use the Gauss scheme");
  // rows per warp: 32 (4 m-tiles) for 16-target tiles; 16 (2 m-tiles) for 32-target
  // tiles, which keeps the accumulators at 48 doubles and halves the W (A operand)
  // bytes per DMMA.  Measured on config 2: 32-target tiles (1 CTA/SM) 58.9 ms,
  // 16-target tiles (2 CTAs/SM) 51.9 ms -> only TT = 16 is instantiated
  static constexpr int RW = (TT == 32 || (GAUSS && NPAD > 128)) ? 16 : 32;
  static constexpr int MT = RW / 8;
  static constexpr int THREADS = NPAD / RW * 32;
  static_assert(THREADS % TT == 0, "whole threads per staged column");
  static constexpr int STAGE = TT * MS;     // doubles per smem stage
  // one moment stage: double-buffering (staging key k+1 during key k) measured
  // 10 % slower on config 2 (51.9 -> 58.9 ms at 2 CTAs/SM)
  static constexpr int NBUF = 1;
  static constexpr int SA = 2 * TT;         // smem accumulator row stride (xor-swizzled columns)
  static constexpr int SR = NK;             // accumulator rows: W rows >= n_k are zero padding
  // per-key metadata of the item (key id, cnt, same flag, TT source slots and
  // TT target columns) staged in smem windows of MK keys: the per-key loads
  // are off the critical path (they miss L2: each item reads its slice once)
  static constexpr int MK = (GAUSS || NPAD != 224) ? 64 : 16;  // real-GEMM n_pad 224: keeps 2 CTAs/SM
  static constexpr int META = MK * (4 + 1 + 1 + 5 * TT);  // bytes
  static constexpr size_t SMEM = (size_t)(NBUF * STAGE + SR * SA) * sizeof(double) + (META + 15) / 16 * 16;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(GAUSS || NPAD != 224 || SMEM <= 113 * 1024, "real-GEMM n_pad 224 must keep 2 CTAs/SM");
  // unroll of the k-step-pair loops
  static constexpr int KU = FDH_KUNROLL > 0 ? FDH_KUNROLL : (NPAD <= 128 ? 2 : 1);
  // resident CTAs per SM the register allocation must allow
  static constexpr int MINB = FDH_M2L_MINB > 0 ? FDH_M2L_MINB : (NPAD == 224 && !GAUSS ? 2 : 1);
  static constexpr int NG = GAUSS ? TT / 8 : 1;  // Gauss n-tiles held (1 = unused)
  static constexpr int NO = GAUSS ? 1 : TT / 4;  // real-GEMM n-tiles held
  // A fragments prefetched one k-step pair ahead in registers (Gauss shapes;
  // the n_pad >= 224 shapes have no registers to spare at 2 CTAs/SM)
  static constexpr bool PF = GAUSS;
};

// register accumulators of one warp (RW rows = MT m-tiles):
//   g[p][mt][nt][2]: Gauss products p = P1, P2, P3 of the 8-target n-tiles nt < NG
//   o[mt][nt][2]:    (Re, Im) of the 4-target n-tiles nt < NO of the real GEMM
template <int MT, int NG, int NO>
struct M2LAcc {
  double g[3][MT][NG][2];
  double o[MT][NO][2];
};

// stage the moments of the first ncol compacted columns (cnt valid, rest zero).
// THREADS / TT threads per column: one smem read of the source slot and one
// base address per thread, then a strided run of 16-byte cp.async.  (Bulk copies
// on the TMA engine with an mbarrier measured slower: 52.1-52.4 vs 51.3 ms.)
template <int NPAD, int NK, int TT>
__device__ __forceinline__ void m2l_stage(double* buf, const int32_t* __restrict__ src, int cnt, int ncol,
                                          const double* __restrict__ mom) {
  using S = M2LShape<NPAD, NK, TT>;
  constexpr int CH = NK / 2;             // 16-byte chunks per plane
  constexpr int TPC = S::THREADS / TT;   // threads per column
  const int c = threadIdx.x / TPC, t = threadIdx.x % TPC;
  if (c >= ncol) return;
  double* dst = buf + c * S::MS;
  if (c < cnt) {
    const double* g = mom + (int64_t)src[c] * S::GS;
#pragma unroll 4
    for (int ch = t; ch < 2 * CH; ch += TPC) {
      const int im = ch >= CH, e = 2 * (ch - im * CH);
      cp_async16(dst + (im ? S::IMOFF : 0) + e, g + (im ? NPAD : 0) + e);
    }
  } else {
    for (int ch = t; ch < 2 * CH; ch += TPC) {
      const int im = ch >= CH, e = 2 * (ch - im * CH);
      dst[(im ? S::IMOFF : 0) + e] = 0.0;
      dst[(im ? S::IMOFF : 0) + e + 1] = 0.0;
    }
  }
}
__device__ __forceinline__ int m2l_ncol(M2LSplit sp) { return 8 * sp.a3 + 4 * sp.ao; }

// A fragments of one k-step pair: MT m-tiles x (k-step 2kp, 2kp+1), 16-byte loads
template <int K3, int MT>
__device__ __forceinline__ void m2l_lda(double2 (&a)[MT], const double* __restrict__ p) {
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) a[mt] = __ldg(reinterpret_cast<const double2*>(p + mt * 8 * K3));
}

// DMMAs of one k-step pair of plane PL (0: Re A, 1: Im A, 2: Re A + Im A)
template <int NPAD, int NK, int TT, int A3, int AO, int PL, class Acc>
__device__ __forceinline__ void m2l_step(Acc& acc, const double2 (&a)[M2LShape<NPAD, NK, TT>::MT], const double* Bg,
                                         const double* Bo, int kp, int re_off, int im_off, unsigned long long sgn) {
  using S = M2LShape<NPAD, NK, TT>;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int ko = 8 * kp + 4 * h;
    double bg[A3 > 0 ? A3 : 1], bo[AO > 0 ? AO : 1];
#pragma unroll
    for (int nt = 0; nt < A3; ++nt) {
      const double* q = Bg + nt * 8 * S::MS + ko;
      bg[nt] = PL == 0 ? q[0] : (PL == 1 ? q[S::IMOFF] : q[0] + q[S::IMOFF]);  // P1: Re v, P2: Im v, P3: sum
    }
#pragma unroll
    for (int nt = 0; nt < AO; ++nt) {
      if (PL == 0) bo[nt] = Bo[nt * 4 * S::MS + re_off + ko];
      // -Im by an integer xor of the sign bit (keeps the FP64 pipe for DMMA)
      if (PL == 1) bo[nt] = __longlong_as_double(__double_as_longlong(Bo[nt * 4 * S::MS + im_off + ko]) ^ sgn);
    }
#pragma unroll
    for (int mt = 0; mt < S::MT; ++mt) {
      const double av = h ? a[mt].y : a[mt].x;
#pragma unroll
      for (int nt = 0; nt < A3; ++nt) dmma8x8x4(acc.g[PL][mt][nt], av, bg[nt]);
      if (PL < 2) {
#pragma unroll
        for (int nt = 0; nt < AO; ++nt) dmma8x8x4(acc.o[mt][nt], av, bo[nt]);
      }
    }
  }
}

// One key.  A3 Gauss n-tiles (targets 0 .. 8 A3-1) and AO real-GEMM n-tiles
// (targets 8 A3 .. 8 A3 + 4 AO - 1); the A fragments of the Re / Im planes are
// shared by both schemes.  The A stream is software-pipelined one k-step pair
// ahead when S::PF (a holds the current pair on entry; the planes are contiguous
// in a W row, so the next pair is always 8 doubles on), and the last pair
// prefetches the first pair of the next key (Wn, null at the end of the item).
//   Wk: lane's W row (k-interleaved, see k_coupling) at k offset 2 bk
//   Bg: smem + (lane >> 2) * MS + bk          (Gauss: column = target)
//   Bo: smem + (8 A3 + (lane >> 3)) * MS + bk (real GEMM: column pair per target)
template <int NPAD, int NK, int TT, int A3, int AO, class Acc>
__device__ __forceinline__ void m2l_key(Acc& acc, double2 (&a)[M2LShape<NPAD, NK, TT>::MT],
                                        const double* __restrict__ Wk, const double* __restrict__ Wn, const double* Bg,
                                        const double* Bo, int re_off, int im_off, unsigned long long sgn) {
  using S = M2LShape<NPAD, NK, TT>;
  constexpr int NKP = NK / 8, MT = S::MT;
  constexpr int NPL = A3 > 0 ? 3 : 2;
#pragma unroll
  for (int pl = 0; pl < NPL; ++pl) {
#pragma unroll S::KU
    for (int kp = 0; kp < NKP; ++kp) {
      double2 an[MT];
      if constexpr (S::PF) {
        const double* nx = (pl + 1 < NPL || kp + 1 < NKP) ? Wk + 8 * (pl * NKP + kp + 1) : Wn;
        if (nx) m2l_lda<S::K3, MT>(an, nx);
      } else {
        m2l_lda<S::K3, MT>(a, Wk + 8 * (pl * NKP + kp));
      }
      if (pl == 0) m2l_step<NPAD, NK, TT, A3, AO, 0>(acc, a, Bg, Bo, kp, re_off, im_off, sgn);
      else if (pl == 1) m2l_step<NPAD, NK, TT, A3, AO, 1>(acc, a, Bg, Bo, kp, re_off, im_off, sgn);
      else m2l_step<NPAD, NK, TT, A3, AO, 2>(acc, a, Bg, Bo, kp, re_off, im_off, sgn);
      if constexpr (S::PF) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) a[mt] = an[mt];
      }
    }
  }
}

// dispatch on the split of the key (warp-uniform): only the n-tiles holding columns
template <int NPAD, int NK, int TT, class Acc>
__device__ __forceinline__ void m2l_key_dispatch(M2LSplit sp, Acc& acc, double2 (&a)[M2LShape<NPAD, NK, TT>::MT],
                                                 const double* Wk, const double* Wn, const double* Bg,
                                                 const double* Bo, int re_off, int im_off, unsigned long long sgn) {
  using S = M2LShape<NPAD, NK, TT>;
#define FDH_KEY(A3, AO) m2l_key<NPAD, NK, TT, A3, AO>(acc, a, Wk, Wn, Bg, Bo, re_off, im_off, sgn)
  if constexpr (S::GAUSS) {
    switch (sp.a3 * 2 + sp.ao) {
      case 1: FDH_KEY(0, 1); break;
      case 2: FDH_KEY(1, 0); break;
      case 3: FDH_KEY(1, 1); break;
      case 4: FDH_KEY(2, 0); break;
      default:
        if constexpr (S::NG >= 4) {
          switch (sp.a3 * 2 + sp.ao) {
            case 5: FDH_KEY(2, 1); break;
            case 6: FDH_KEY(3, 0); break;
            case 7: FDH_KEY(3, 1); break;
            default: FDH_KEY(4, 0); break;
          }
        }
        break;
    }
  } else {
    switch (sp.ao) {
      case 1: FDH_KEY(0, 1); break;
      case 2: FDH_KEY(0, 2); break;
      case 3: FDH_KEY(0, 3); break;
      default: FDH_KEY(0, 4); break;
    }
  }
#undef FDH_KEY
}

// add the register tile (compacted columns) into the shared accumulator of the
// tile's target columns; every (row, target) belongs to one lane: no races
template <int NPAD, int NK, int TT, class Acc>
__device__ __forceinline__ void m2l_flush(Acc& acc, double* sacc, const uint8_t* __restrict__ cols, int cnt,
                                          int warp, int lane) {
  using S = M2LShape<NPAD, NK, TT>;
  const M2LSplit sp = m2l_split(cnt, S::GAUSS);
  const int rbase = warp * S::RW + (lane >> 2);
  // Gauss n-tiles: lane holds targets 8 nt + 2 (lane & 3) + e
#pragma unroll
  for (int nt = 0; nt < S::NG; ++nt) {
    if (S::GAUSS && nt < sp.a3) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = nt * 8 + 2 * (lane & 3) + e;
        const int t = j < cnt ? cols[j] : -1;
#pragma unroll
        for (int mt = 0; mt < S::MT; ++mt) {
          const int row = rbase + mt * 8;
          if (t >= 0 && row < S::SR) {
            const double p1 = acc.g[0][mt][nt][e], p2 = acc.g[1][mt][nt][e], p3 = acc.g[2][mt][nt][e];
            double* p = sacc + row * S::SA + 2 * (t ^ (row & (TT - 1)));
            p[0] += p1 - p2;
            p[1] += p3 - (p1 + p2);
          }
          acc.g[0][mt][nt][e] = acc.g[1][mt][nt][e] = acc.g[2][mt][nt][e] = 0.0;
        }
      }
    }
  }
  // real-GEMM n-tiles: lane holds target 8 a3 + 4 nt + (lane & 3), (Re, Im)
#pragma unroll
  for (int nt = 0; nt < S::NO; ++nt) {
    if (nt < sp.ao) {
      const int j = sp.a3 * 8 + nt * 4 + (lane & 3);
      const int t = j < cnt ? cols[j] : -1;
#pragma unroll
      for (int mt = 0; mt < S::MT; ++mt) {
        const int row = rbase + mt * 8;
        if (t >= 0 && row < S::SR) {
          double* p = sacc + row * S::SA + 2 * (t ^ (row & (TT - 1)));
          p[0] += acc.o[mt][nt][0];
          p[1] += acc.o[mt][nt][1];
        }
        acc.o[mt][nt][0] = acc.o[mt][nt][1] = 0.0;
      }
    }
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One work item = (tile, key chunk).  Items run chunk-major (all tiles of
// chunk c before chunk c+1), so the coupling matrices of one chunk are shared
// through L2 by every tile.  Per key, only the target columns that have the key
// are computed: they are compacted to the front (cnt columns -> ceil(cnt/4)
// n-tiles), accumulated in registers over runs of keys with the same column
// map and added into a shared-memory accumulator when the map changes.  The
// items of a tile are chained in chunk order by a ticket (earlier items are
// dispatched first, so the wait is short and cannot deadlock); the last item
// writes the locals.  Summation order is fixed -> bitwise deterministic.
// Each CTA claims its item from an atomic counter when it starts (not by
// blockIdx): an item's predecessor in its tile chain has a lower index, so it
// was claimed by a CTA that is already running -- the chain always progresses,
// whatever the dispatch order or concurrent kernels.
template <int NPAD, int NK, int TT>
__global__ void __launch_bounds__(M2LShape<NPAD, NK, TT>::THREADS, M2LShape<NPAD, NK, TT>::MINB) k_m2l_gemm(const int32_t* __restrict__ item_tile,
                                                   const int32_t* __restrict__ item_seq,
                                                   const int64_t* __restrict__ item_k0,
                                                   const int64_t* __restrict__ item_k1,
                                                   const int32_t* __restrict__ tile_nitem,
                                                   const int32_t* __restrict__ tile_tslot,
                                                   const int32_t* __restrict__ tile_keys,
                                                   const int32_t* __restrict__ tile_src,
                                                   const uint8_t* __restrict__ tile_cols,
                                                   const uint8_t* __restrict__ tile_cnt,
                                                   const uint8_t* __restrict__ tile_same,
                                                   const double* __restrict__ W, const double* __restrict__ mom,
                                                   double* __restrict__ tile_acc, int* __restrict__ ticket,
                                                   double* __restrict__ loc, int* __restrict__ counter, int item0,
                                                   int64_t key_base) {
  using S = M2LShape<NPAD, NK, TT>;
  constexpr int MT = S::MT;
  extern __shared__ __align__(16) double smem[];
  double* sacc = smem + S::NBUF * S::STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int s_item;
  if (threadIdx.x == 0) s_item = atomicAdd(counter, 1);
  __syncthreads();
  const int item = item0 + s_item;
  const int64_t k0 = item_k0[item], k1 = item_k1[item];
  // metadata window [w0, w0 + MK)
  int32_t* m_src = reinterpret_cast<int32_t*>(sacc + S::SR * S::SA);
  int32_t* m_key = m_src + S::MK * TT;
  uint8_t* m_cols = reinterpret_cast<uint8_t*>(m_key + S::MK);
  uint8_t* m_cnt = m_cols + S::MK * TT;
  uint8_t* m_same = m_cnt + S::MK;
  int64_t w0 = k0;
  auto load_meta = [&](int64_t b) {
    const int n = (int)min((int64_t)S::MK, k1 - b);
    for (int i = threadIdx.x; i < n; i += S::THREADS) {
      m_key[i] = tile_keys[b + i];
      m_cnt[i] = tile_cnt[b + i];
      m_same[i] = tile_same[b + i];
    }
    for (int i = threadIdx.x; i < n * TT; i += S::THREADS) {
      m_src[i] = tile_src[b * TT + i];
      m_cols[i] = tile_cols[b * TT + i];
    }
    __syncthreads();
  };
  load_meta(k0);

  for (int i = threadIdx.x; i < S::SR * S::SA; i += S::THREADS) sacc[i] = 0.0;
  M2LAcc<MT, S::NG, S::NO> acc;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
    for (int nt = 0; nt < S::NO; ++nt) acc.o[mt][nt][0] = acc.o[mt][nt][1] = 0.0;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int nt = 0; nt < S::NG; ++nt) acc.g[p][mt][nt][0] = acc.g[p][mt][nt][1] = 0.0;
  }

  // B fragment addressing: lane holds B[k0 + (lane&3)][nt*8 + lane/4]
  //   column col = nt*8 + lane/4 -> source c = nt*4 + lane/8, parity = (lane>>2)&1
  const int bpar = (lane >> 2) & 1;
  const int bcol = lane >> 3;
  const int bk = lane & 3;
  const int re_off = bpar ? S::IMOFF : 0;   // first K half: parity 0 -> Re, 1 -> Im
  const int im_off = bpar ? 0 : S::IMOFF;   // second K half: parity 0 -> -Im, 1 -> Re
  // sign flip of -Im by an integer xor of the sign bit (keeps the FP64 pipe for DMMA)
  const unsigned long long sgn = bpar ? 0ull : 0x8000000000000000ull;

  {
    const int c0 = m_cnt[0];
    m2l_stage<NPAD, NK, TT>(smem, m_src, c0, m2l_ncol(m2l_split(c0, S::GAUSS)), mom);
  }
  cp_async_commit();
  // lane's W row (k-interleaved, offset 2 bk) without the key offset; first A pair of key k0
  const double* __restrict__ Wrow = W + (int64_t)(warp * S::RW + (lane >> 2)) * S::K3 + 2 * bk;
  double2 a[MT];
  if constexpr (S::PF) m2l_lda<S::K3, MT>(a, Wrow + ((int64_t)m_key[0] - key_base) * NPAD * S::K3);
  FDH_TR_T(t_loop);
  for (int64_t kk = k0; kk < k1; ++kk) {
    FDH_TR_T(t0);
    if (kk + 1 < k1 && kk + 1 - w0 >= S::MK) {  // slide the window to [kk - 1, ...)
      __syncthreads();
      w0 = kk - 1;
      load_meta(w0);
    }
    const int j = (int)(kk - w0);
    const int cnt = m_cnt[j];
    cp_async_wait<0>();  // moments of key kk landed (this thread's copies; the barrier covers the rest)
    __syncthreads();
    FDH_TR_T(t1);
    if (kk > k0 && !m_same[j]) m2l_flush<NPAD, NK, TT>(acc, sacc, m_cols + (j - 1) * TT, m_cnt[j - 1], warp, lane);
    FDH_TR_T(t2);
    const double* Bst = smem;
    const double* Bg = Bst + (lane >> 2) * S::MS + bk;
    const M2LSplit sp = m2l_split(cnt, S::GAUSS);
    const double* Bo = Bst + (8 * sp.a3 + bcol) * S::MS + bk;
    const double* __restrict__ Wk = Wrow + ((int64_t)m_key[j] - key_base) * NPAD * S::K3;
    const double* __restrict__ Wn = kk + 1 < k1 ? Wrow + ((int64_t)m_key[j + 1] - key_base) * NPAD * S::K3 : nullptr;
    m2l_key_dispatch<NPAD, NK, TT>(sp, acc, a, Wk, Wn, Bg, Bo, re_off, im_off, sgn);
    FDH_TR_T(t3);
    __syncthreads();
    FDH_TR_T(t4);
    if (kk + 1 < k1) {
      const int cn = m_cnt[j + 1];
      m2l_stage<NPAD, NK, TT>(smem, m_src + (j + 1) * TT, cn, m2l_ncol(m2l_split(cn, S::GAUSS)), mom);
    }
    cp_async_commit();
    FDH_TR_T(t5);
    FDH_TR_ADD(0, t1 - t0);  // wait for the staged moments + barrier
    FDH_TR_ADD(1, t2 - t1);  // flush
    FDH_TR_ADD(2, t3 - t2);  // DMMA key loop
    FDH_TR_ADD(3, t4 - t3);  // end-of-key barrier
    FDH_TR_ADD(4, t5 - t4);  // staging issue
    FDH_TR_ADD(6, 1);        // keys
  }
  FDH_TR_T(t_end);
  FDH_TR_ADD(5, t_end - t_loop);
  FDH_TR_ADD(7, 1);  // items
  m2l_flush<NPAD, NK, TT>(acc, sacc, m_cols + (k1 - 1 - w0) * TT, m_cnt[k1 - 1 - w0], warp, lane);
  __syncthreads();
  // ---- chained accumulation into the tile (chunk order)
  const int tile = item_tile[item], seq = item_seq[item], nit = tile_nitem[tile];
  double* A = tile_acc + (int64_t)tile * NPAD * 2 * TT;
  if (seq > 0) {
    if (threadIdx.x == 0)
      while (ld_acquire(ticket + tile) != seq) __nanosleep(100);
    __syncthreads();
  }
  const bool last = seq == nit - 1;
  for (int idx = threadIdx.x; idx < S::SR * TT; idx += S::THREADS) {  // rows >= n_k of loc stay zero
    const int row = idx / TT, j = idx % TT;
    const int jj = j ^ (row & (TT - 1));
    double2 v = make_double2(sacc[row * S::SA + 2 * jj], sacc[row * S::SA + 2 * jj + 1]);
    double2* pa = reinterpret_cast<double2*>(A + (int64_t)row * 2 * TT + 2 * j);
    if (seq > 0) {
      const double2 o = __ldcg(pa);
      v.x = o.x + v.x;
      v.y = o.y + v.y;
    }
    if (last) {
      const int32_t ts = tile_tslot[tile * TT + j];
      if (ts >= 0) {
        loc[(int64_t)ts * 2 * NPAD + row] = v.x;          // Re(A v)
        loc[(int64_t)ts * 2 * NPAD + NPAD + row] = v.y;   // Im(A v)
      }
    } else {
      __stcg(pa, v);
    }
  }
  if (!last) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(ticket + tile, seq + 1);
  }
}

template <int NPAD, int NK, int TT>
void run_gemm(cudaStream_t st, const M2LArgs& a) {
  using S = M2LShape<NPAD, NK, TT>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_m2l_gemm<NPAD, NK, TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
    attr = true;
  }
  k_m2l_gemm<NPAD, NK, TT><<<a.n_item, S::THREADS, S::SMEM, st>>>(a.item_tile, a.item_seq, a.item_k0, a.item_k1,
                                                              a.tile_nitem, a.tile_tslot, a.tile_keys, a.tile_src,
                                                              a.tile_cols, a.tile_cnt, a.tile_same, a.W, a.mom,
                                                              a.tile_acc, a.ticket, a.loc, a.counter, a.item0,
                                                              a.key_base);
}

}  // namespace

void launch_coupling(cudaStream_t st, const Consts* C, const double* dirtab, int64_t key0, int64_t nkeys,
                     const int32_t* key_level, const int64_t* key_d, const int32_t* key_dir, double* W, int n,
                     int n_pad, int n_k, int64_t wbase) {
  if (nkeys <= 0) return;
  dim3 grid((unsigned)nkeys, (unsigned)((n_pad + kCplRows - 1) / kCplRows));
  k_coupling<<<grid, 256, 0, st>>>(C, dirtab, key0, key_level, key_d, key_dir, W, n, n_pad, n_k, wbase);
}

int launch_m2l_gemm(cudaStream_t st, int n_pad, int n_k, int tile, const M2LArgs& a) {
  if (a.n_item <= 0) return 0;
  if (tile != 16) return 1;
  if (n_pad == 32 && n_k == 8) run_gemm<32, 8, 16>(st, a);
  else if (n_pad == 32 && n_k == 32) run_gemm<32, 32, 16>(st, a);
  else if (n_pad == 64 && n_k == 64) run_gemm<64, 64, 16>(st, a);
  else if (n_pad == 128 && n_k == 128) run_gemm<128, 128, 16>(st, a);
  else if (n_pad == 224 && n_k == 216) run_gemm<224, 216, 16>(st, a);
  else if (n_pad == 352 && n_k == 344) run_gemm<352, 344, 16>(st, a);
  else return 1;
  return 0;
}

}  // namespace fdhelm

#if FDH_M2L_TRACE
extern "C" int fdh_debug_m2l_trace(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, fdhelm::g_m2l_trace, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(fdhelm::g_m2l_trace, z, sizeof(z));
  }
  return 0;
}
#endif
