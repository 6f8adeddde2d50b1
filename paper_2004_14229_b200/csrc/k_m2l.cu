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
// single real GEMM with 8 n^2 flops per block.  It runs on
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

namespace fdhelm {

namespace {

constexpr double kFourPi = 4.0 * 3.14159265358979323846;  // geometry.hpp:11

// ---------------------------------------------------------- coupling gen
// W[key][j][k] = Re f_c(xi_t,j, xi_s,k),  W[key][j][n_k + k] = Im f_c(...)
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
  double* Wk = W + (key - wbase) * n_pad * 2 * n_k;
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
    Wk[(int64_t)j * 2 * n_k + kp] = re;
    Wk[(int64_t)j * 2 * n_k + n_k + kp] = im;
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
  static constexpr int K2 = 2 * NK;         // GEMM K (and W row length)
  static constexpr int GS = 2 * NPAD;       // moment slot stride in HBM ([Re | Im] planes of NPAD)
  static constexpr int MS = 2 * NK + 8 + ((NK & 8) ? 0 : 0);  // smem moment stride (== 8 mod 16)
  static constexpr int IMOFF = NK + 4;      // smem offset of the imaginary plane (== 4 or 12 mod 16)
  static_assert(NK % 8 == 0 && MS % 16 == 8, "bank-conflict-free B fragments");
  static constexpr int NT = 2 * TT / 8;     // 8-column n-tiles per warp
  static constexpr int THREADS = NPAD;      // one warp per 32 rows
  static constexpr int STAGE = TT * MS;     // doubles per smem stage
  static constexpr int NBUF = 1;  // single stage: keeps 3 CTAs/SM with the shared accumulator
  static constexpr int SA = 2 * TT;         // smem accumulator row stride (xor-swizzled columns)
  static constexpr size_t SMEM = (size_t)(NBUF * STAGE + NPAD * SA) * sizeof(double);
  // unroll of the k-step-pair loops: deeper for small tiles (more loads in
  // flight), 1 for n_pad >= 224 where registers limit 2 CTAs/SM (measured)
  static constexpr int KU = FDH_KUNROLL > 0 ? FDH_KUNROLL : (NPAD <= 128 ? 4 : 1);
};

// stage the moments of the first ncol compacted columns (cnt valid, rest zero)
template <int NPAD, int NK, int TT>
__device__ __forceinline__ void m2l_stage(double* buf, const int32_t* __restrict__ src, int cnt, int ncol,
                                          const double* __restrict__ mom) {
  using S = M2LShape<NPAD, NK, TT>;
  constexpr int CH = NK / 2;  // 16-byte chunks per plane
  for (int idx = threadIdx.x; idx < ncol * 2 * CH; idx += S::THREADS) {
    const int c = idx / (2 * CH), ch = idx % (2 * CH);
    const int im = ch >= CH, e = 2 * (ch - im * CH);
    double* dst = buf + c * S::MS + (im ? S::IMOFF : 0) + e;
    if (c < cnt) {
      cp_async16(dst, mom + (int64_t)src[c] * S::GS + (im ? NPAD : 0) + e);
    } else {
      dst[0] = 0.0;
      dst[1] = 0.0;
    }
  }
}

// One key: C[:, n-tiles < NTA] += W_key * B over K = 2 NPAD.
template <int NPAD, int NK, int TT, int NTA>
__device__ __forceinline__ void m2l_key(double (&acc)[4][M2LShape<NPAD, NK, TT>::NT][2], const double* __restrict__ Wk,
                                        const double* Bs, int re_off, int im_off, unsigned long long sgn) {
  using S = M2LShape<NPAD, NK, TT>;
  // W rows are stored k-interleaved in blocks of 8 (k_coupling): the lane's
  // A-fragment values of k-steps 2p and 2p+1 are adjacent -> one 16-byte load.
  // K half 1: columns of Re A against (Re v, Im v)
#pragma unroll S::KU
  for (int kp = 0; kp < NK / 8; ++kp) {
    double2 a[4];
    double b0[NTA], b1[NTA];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) a[mt] = __ldg(reinterpret_cast<const double2*>(Wk + mt * 8 * S::K2 + 8 * kp));
#pragma unroll
    for (int nt = 0; nt < NTA; ++nt) {
      b0[nt] = Bs[nt * 4 * S::MS + re_off + 8 * kp];
      b1[nt] = Bs[nt * 4 * S::MS + re_off + 8 * kp + 4];
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTA; ++nt) dmma8x8x4(acc[mt][nt], a[mt].x, b0[nt]);
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTA; ++nt) dmma8x8x4(acc[mt][nt], a[mt].y, b1[nt]);
  }
  // K half 2: columns of Im A against (-Im v, Re v)
#pragma unroll S::KU
  for (int kp = 0; kp < NK / 8; ++kp) {
    double2 a[4];
    double b0[NTA], b1[NTA];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
      a[mt] = __ldg(reinterpret_cast<const double2*>(Wk + NK + mt * 8 * S::K2 + 8 * kp));
#pragma unroll
    for (int nt = 0; nt < NTA; ++nt) {
      b0[nt] = __longlong_as_double(__double_as_longlong(Bs[nt * 4 * S::MS + im_off + 8 * kp]) ^ sgn);
      b1[nt] = __longlong_as_double(__double_as_longlong(Bs[nt * 4 * S::MS + im_off + 8 * kp + 4]) ^ sgn);
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTA; ++nt) dmma8x8x4(acc[mt][nt], a[mt].x, b0[nt]);
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTA; ++nt) dmma8x8x4(acc[mt][nt], a[mt].y, b1[nt]);
  }
}

// add the register tile (compacted columns) into the shared accumulator of the
// tile's target columns; every (row, target) belongs to one lane: no races
template <int NPAD, int NK, int TT>
__device__ __forceinline__ void m2l_flush(double (&acc)[4][M2LShape<NPAD, NK, TT>::NT][2], double* sacc,
                                          const uint8_t* __restrict__ cols, int cnt, int warp, int lane) {
  using S = M2LShape<NPAD, NK, TT>;
#pragma unroll
  for (int nt = 0; nt < S::NT; ++nt) {
    const int j = nt * 4 + (lane & 3);
    const int t = j < cnt ? cols[j] : -1;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      if (t >= 0) {
        const int row = warp * 32 + mt * 8 + (lane >> 2);
        double* p = sacc + row * S::SA + 2 * (t ^ (row & (TT - 1)));
        p[0] += acc[mt][nt][0];
        p[1] += acc[mt][nt][1];
      }
      acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
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
template <int NPAD, int NK, int TT>
__global__ void __launch_bounds__(NPAD) k_m2l_gemm(const int32_t* __restrict__ item_tile,
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
                                                   double* __restrict__ loc, int* __restrict__ err, int item0,
                                                   int64_t key_base) {
  using S = M2LShape<NPAD, NK, TT>;
  constexpr int NT = S::NT;
  static_assert(NT == 4, "one warp row-block covers 4 n-tiles");
  extern __shared__ __align__(16) double smem[];
  double* sacc = smem + S::NBUF * S::STAGE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = item0 + (int)blockIdx.x;
  const int64_t k0 = item_k0[item], k1 = item_k1[item];

  for (int i = threadIdx.x; i < NPAD * S::SA; i += S::THREADS) sacc[i] = 0.0;
  double acc[4][NT][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

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
    const int c0 = tile_cnt[k0];
    m2l_stage<NPAD, NK, TT>(smem, tile_src + k0 * TT, c0, 4 * ((c0 + 3) >> 2), mom);
  }
  cp_async_commit();
  int stage = 0;
  for (int64_t kk = k0; kk < k1; ++kk) {
    const int cnt = tile_cnt[kk];
    if constexpr (S::NBUF == 2) {
      if (kk + 1 < k1) {
        const int cn = tile_cnt[kk + 1];
        m2l_stage<NPAD, NK, TT>(smem + (stage ^ 1) * S::STAGE, tile_src + (kk + 1) * TT, cn, 4 * ((cn + 3) >> 2), mom);
      }
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kk > k0 && !tile_same[kk]) m2l_flush<NPAD, NK, TT>(acc, sacc, tile_cols + (kk - 1) * TT, tile_cnt[kk - 1], warp,
                                                       lane);
    const double* __restrict__ Wk =
        W + ((int64_t)tile_keys[kk] - key_base) * NPAD * S::K2 + (int64_t)(warp * 32 + (lane >> 2)) * S::K2 + 2 * bk;
    const double* Bs = smem + stage * S::STAGE + bcol * S::MS + bk;
    switch ((cnt + 3) >> 2) {  // warp-uniform: only the n-tiles holding columns
      case 1: m2l_key<NPAD, NK, TT, 1>(acc, Wk, Bs, re_off, im_off, sgn); break;
      case 2: m2l_key<NPAD, NK, TT, 2>(acc, Wk, Bs, re_off, im_off, sgn); break;
      case 3: m2l_key<NPAD, NK, TT, 3>(acc, Wk, Bs, re_off, im_off, sgn); break;
      default: m2l_key<NPAD, NK, TT, 4>(acc, Wk, Bs, re_off, im_off, sgn); break;
    }
    __syncthreads();
    if constexpr (S::NBUF == 2) {
      stage ^= 1;
    } else {
      if (kk + 1 < k1) {
        const int cn = tile_cnt[kk + 1];
        m2l_stage<NPAD, NK, TT>(smem, tile_src + (kk + 1) * TT, cn, 4 * ((cn + 3) >> 2), mom);
      }
      cp_async_commit();
    }
  }
  m2l_flush<NPAD, NK, TT>(acc, sacc, tile_cols + (k1 - 1) * TT, tile_cnt[k1 - 1], warp, lane);
  __syncthreads();
  // ---- chained accumulation into the tile (chunk order)
  const int tile = item_tile[item], seq = item_seq[item], nit = tile_nitem[tile];
  double* A = tile_acc + (int64_t)tile * NPAD * 2 * TT;
  if (seq > 0) {
    if (threadIdx.x == 0) {
      long long spins = 0;
      while (ld_acquire(ticket + tile) != seq) {
        __nanosleep(200);
        if (++spins > (1ll << 26)) {  // > ~10 s: report instead of hanging
          atomicOr(err, 2);
          break;
        }
      }
    }
    __syncthreads();
  }
  const bool last = seq == nit - 1;
  for (int idx = threadIdx.x; idx < NPAD * TT; idx += S::THREADS) {
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
                                                              a.tile_acc, a.ticket, a.loc, a.err, a.item0,
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
