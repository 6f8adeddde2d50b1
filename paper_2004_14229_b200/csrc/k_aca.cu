// k_aca.cu -- ACA-compressed coupling matrices (
// PAPER.md:420-424 "we apply a partially pivoted ACA").
//
// Opt-in, lossy (tolerance eps; eps = 1e-8 agrees with the dense
// matvec to 1e-6): every coupling matrix A_key (n x n complex, the same entries as
// k_coupling / k_coupling_i8, generated on demand from the node geometry, never
// stored) is factorised by partially pivoted ACA into A ~ U W (U n x k, W = V^*
// k x n) with the pinned pivoting: start from row 0, column pivot =
// max-modulus entry of the residual row, next row pivot = max-modulus entry of
// the residual column among unused rows (lowest index on ties), stop when
// |u_k||w_k| <= eps |S_k|_F (incremental Frobenius estimate).  A key whose rank
// would reach n/2 (2 k n >= n^2: no gain) keeps its dense matrix (stored as W with
// U = identity, rank -1).
//   k_aca_factor : one CTA per key; pass 0 ranks only, pass 1 the factors at
//                  their final offsets (the ACA is deterministic, so both passes
//                  pick the same pivots);
//   k_m2l_aca    : the M2L on the factors, g~_t += U (W v~_s) per (tile, key),
//                  FP64, over the same tiles / items / ticket chains as the exact
//                  M2L kernels (deterministic, no FP atomics).
#include "kernels.hpp"

#include <algorithm>
#include <cstdlib>

namespace fdhelm {

namespace {

constexpr double kFourPi = 4.0 * 3.14159265358979323846;  // geometry.hpp:11
constexpr int kAT = 256;                                   // threads per CTA

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct KeyGeo {
  double tn[3][kMaxP], sn[3][kMaxP], c[3], kappa;
  int p;
};

// entry (j, k) of A_key (canonical frame), as k_coupling
__device__ __forceinline__ double2 aca_entry(const KeyGeo& g, int j, int k) {
  const int p = g.p;
  const double d[3] = {__dsub_rn(g.tn[0][j / (p * p)], g.sn[0][k / (p * p)]),
                       __dsub_rn(g.tn[1][(j / p) % p], g.sn[1][(k / p) % p]),
                       __dsub_rn(g.tn[2][j % p], g.sn[2][k % p])};
  const double r = sqrt(dot3(d, d));  // geometry.hpp:92-98
  const double ph = __dmul_rn(g.kappa, __dsub_rn(r, dot3(d, g.c)));
  const double w = __ddiv_rn(1.0, __dmul_rn(kFourPi, r));
  double s, co;
  sincos(ph, &s, &co);
  return make_double2(__dmul_rn(w, co), __dmul_rn(w, s));
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// block-wide argmax of v over i (lowest index on ties); returns (index, value)
__device__ void block_argmax(double v, int i, double* sv, int* si, double& bv, int& bi) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    sv[w] = v;
    si[w] = i;
  }
  __syncthreads();
  bv = sv[0];
  bi = si[0];
  for (int q = 1; q < kAT / 32; ++q)
    if (sv[q] > bv || (sv[q] == bv && si[q] < bi)) {
      bv = sv[q];
      bi = si[q];
    }
}
__device__ double block_sum(double v, double* sv) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int q = 0; q < kAT / 32; ++q) s += sv[q];  // fixed order
  return s;
}

// pass 0: ranks only (factors in the per-CTA scratch); pass 1: factors written at
// uoff / woff.  U: column-major n x k (U[q n + i]); W: row-major k x n (W[q n + c]).
__global__ void __launch_bounds__(kAT) k_aca_factor(const Consts* __restrict__ C, const double* __restrict__ dirtab,
                                                    int64_t key0, const int32_t* __restrict__ key_level,
                                                    const int64_t* __restrict__ key_d,
                                                    const int32_t* __restrict__ key_dir, double eps, int n, int pass,
                                                    int32_t* __restrict__ rank, double2* __restrict__ scratch,
                                                    const int64_t* __restrict__ uoff, const int64_t* __restrict__ woff,
                                                    double2* __restrict__ Uall, double2* __restrict__ Wall) {
  __shared__ KeyGeo g;
  __shared__ double sv[kAT / 32];
  __shared__ int si[kAT / 32];
  extern __shared__ double2 sh[];  // row[n], col[n], used flags as doubles (n)
  double2* row = sh;
  double2* col = sh + n;
  double* used = reinterpret_cast<double*>(sh + 2 * n);
  const int64_t key = key0 + blockIdx.x;
  const int l = key_level[key];
  if (threadIdx.x < 3 * C->p) {
    const int p = C->p, a = threadIdx.x / p, nu = threadIdx.x % p;
    const double side = C->side_t[l][a];
    const int64_t d = key_d[3 * key + a];
    g.tn[a][nu] = cheb_node(__dmul_rn((double)d, side), __dmul_rn((double)(d + 1), side), C->cheb_cos[nu]);
    g.sn[a][nu] = cheb_node(0.0, __dmul_rn(1.0, side), C->cheb_cos[nu]);
  }
  if (threadIdx.x == 0) {
    const double* c = dir_vec(C, dirtab, l, key_dir[key]);
    g.c[0] = c[0];
    g.c[1] = c[1];
    g.c[2] = c[2];
    g.kappa = C->kappa;
    g.p = C->p;
  }
  for (int i = threadIdx.x; i < n; i += kAT) used[i] = 0.0;
  __syncthreads();
  const int kcap = (n + 1) / 2;  // rank kcap: 2 k n >= n^2 -> dense
  if (pass == 1 && rank[key] < 0) {  // dense (from pass 0): W = the matrix rows, U = identity
    double2* W = Wall + woff[key];
    for (int idx = threadIdx.x; idx < n * n; idx += kAT) W[idx] = aca_entry(g, idx / n, idx % n);
    return;
  }
  double2* U = pass == 0 ? scratch + (int64_t)blockIdx.x * n * (n + 1) : Uall + uoff[key];
  double2* W = pass == 0 ? U + (int64_t)kcap * n : Wall + woff[key];
  double s2 = 0.0;
  int ip = 0, k = 0;
  bool dense = false;
  while (true) {
    if (threadIdx.x == 0) used[ip] = 1.0;
    for (int c = threadIdx.x; c < n; c += kAT) {  // residual row ip
      double2 v = aca_entry(g, ip, c);
      for (int q = 0; q < k; ++q) {
        const double2 t = cmul(U[(int64_t)q * n + ip], W[(int64_t)q * n + c]);
        v.x -= t.x;
        v.y -= t.y;
      }
      row[c] = v;
    }
    __syncthreads();
    double bv = -1.0;
    int jp = 0;
    {
      double mv = -1.0;
      int mi = 0x7fffffff;
      for (int c = threadIdx.x; c < n; c += kAT) {
        const double a = hypot(row[c].x, row[c].y);
        if (a > mv) {
          mv = a;
          mi = c;
        }
      }
      block_argmax(mv, mi, sv, si, bv, jp);
    }
    if (bv == 0.0) break;  // residual row vanishes: exact rank k
    if (k == kcap) {
      dense = true;
      break;
    }
    const double2 delta = row[jp];
    const double dd = delta.x * delta.x + delta.y * delta.y;
    __syncthreads();  // every thread has the pivot before the row is rescaled in place
    double pu = 0.0, pw = 0.0;
    for (int i = threadIdx.x; i < n; i += kAT) {  // residual column jp, w = row / delta
      double2 v = aca_entry(g, i, jp);
      for (int q = 0; q < k; ++q) {
        const double2 t = cmul(U[(int64_t)q * n + i], W[(int64_t)q * n + jp]);
        v.x -= t.x;
        v.y -= t.y;
      }
      col[i] = v;
      pu += v.x * v.x + v.y * v.y;
      const double2 r = row[i];  // i < n: the same index range for the row
      const double2 w = make_double2((r.x * delta.x + r.y * delta.y) / dd, (r.y * delta.x - r.x * delta.y) / dd);
      row[i] = w;
      pw += w.x * w.x + w.y * w.y;
    }
    const double nu = block_sum(pu, sv), nw = block_sum(pw, sv);
    // cross terms 2 Re sum_q (u_q^H u)(w_q^H w): one warp per q
    double cr = 0.0;
    for (int q = threadIdx.x >> 5; q < k; q += kAT / 32) {
      double ar = 0, ai = 0, br = 0, bi = 0;
      for (int i = threadIdx.x & 31; i < n; i += 32) {
        const double2 uq = U[(int64_t)q * n + i], u = col[i];
        ar += uq.x * u.x + uq.y * u.y;  // conj(uq) u
        ai += uq.x * u.y - uq.y * u.x;
        const double2 wq = W[(int64_t)q * n + i], w = row[i];
        br += wq.x * w.x + wq.y * w.y;
        bi += wq.x * w.y - wq.y * w.x;
      }
      for (int o = 16; o > 0; o >>= 1) {
        ar += __shfl_xor_sync(0xffffffffu, ar, o);
        ai += __shfl_xor_sync(0xffffffffu, ai, o);
        br += __shfl_xor_sync(0xffffffffu, br, o);
        bi += __shfl_xor_sync(0xffffffffu, bi, o);
      }
      if ((threadIdx.x & 31) == 0) cr += 2.0 * (ar * br - ai * bi);
    }
    const double cross = block_sum((threadIdx.x & 31) == 0 ? cr : 0.0, sv);
    if (k > 0 && sqrt(nu * nw) <= 1e-14 * sqrt(fmax(s2, 0.0))) break;  // round-off cross: exact rank k
    for (int i = threadIdx.x; i < n; i += kAT) {
      U[(int64_t)k * n + i] = col[i];
      W[(int64_t)k * n + i] = row[i];
    }
    ++k;
    s2 += cross + nu * nw;
    __syncthreads();
    if (sqrt(nu * nw) <= eps * sqrt(fmax(s2, 0.0))) break;
    double mv = -1.0;
    int mi = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += kAT) {
      const double a = used[i] != 0.0 ? -1.0 : hypot(col[i].x, col[i].y);
      if (a > mv) {
        mv = a;
        mi = i;
      }
    }
    int inext;
    block_argmax(mv, mi, sv, si, bv, inext);
    if (bv < 0.0) break;
    ip = inext;
    __syncthreads();
  }
  if (2 * k >= n) dense = true;
  if (pass == 0 && threadIdx.x == 0) rank[key] = dense ? -1 : k;
}

// ---------------------------------------------------------------- M2L
// One CTA per claimed work item (tile, key range) of the exact M2L's plan;
// target columns in groups of CG; per key and group: B (n x CG, the gathered
// moments) in shared memory, Z = W B (k x CG) by shared-memory tiles of W, then
// C += U Z in registers (rows j = r0 + RG i, RG = kAT / CG row groups).
template <int CG>
__global__ void __launch_bounds__(kAT) k_m2l_aca(
    const int32_t* __restrict__ item_tile, const int32_t* __restrict__ item_seq, const int64_t* __restrict__ item_k0,
    const int64_t* __restrict__ item_k1, const int32_t* __restrict__ tile_nitem, const int32_t* __restrict__ tile_tslot,
    const int32_t* __restrict__ tile_keys, const int32_t* __restrict__ tile_src, const uint8_t* __restrict__ tile_cols,
    const uint8_t* __restrict__ tile_cnt, const int32_t* __restrict__ rank, const int64_t* __restrict__ uoff,
    const int64_t* __restrict__ woff, const double2* __restrict__ Uall, const double2* __restrict__ Wall,
    const double* __restrict__ mom, double* __restrict__ tile_acc, int* __restrict__ ticket, double* __restrict__ loc,
    int* __restrict__ counter, int n, int n_pad, int TT) {
  constexpr int RG = kAT / CG;  // row groups
  constexpr int KC = 16;        // K chunk of W staged per step
  constexpr int RMAX = CG == 16 ? 14 : 12;  // rows per thread: n <= 224 (CG 16) / 384 (CG 8)
  extern __shared__ double2 sm[];
  double2* Bs = sm;             // [n][CG]
  double2* Ws = Bs + n * CG;    // [n (max rank)][KC]
  double2* Zs = Ws + n * KC;    // [n][CG]
  __shared__ int s_item;
  __shared__ int srcc[32];
  if (threadIdx.x == 0) s_item = atomicAdd(counter, 1);
  __syncthreads();
  const int item = s_item;
  const int tile = item_tile[item];
  const int64_t k0 = item_k0[item], k1 = item_k1[item];
  const int c = threadIdx.x % CG, rg = threadIdx.x / CG;
  const int NC = 2 * TT;
  double* A = tile_acc + (int64_t)tile * n_pad * NC;
  const int seq = item_seq[item], nit = tile_nitem[tile];
  bool waited = false;
  for (int cg0 = 0; cg0 < TT; cg0 += CG) {
    double2 acc[RMAX];
#pragma unroll
    for (int i = 0; i < RMAX; ++i) acc[i] = make_double2(0.0, 0.0);
    for (int64_t kk = k0; kk < k1; ++kk) {
      // uncompacted source slot of each column of this group (-1: absent)
      if (threadIdx.x < CG) srcc[threadIdx.x] = -1;
      __syncthreads();
      if (threadIdx.x < TT) {
        const int j = threadIdx.x;
        if (j < tile_cnt[kk]) {
          const int col = tile_cols[kk * TT + j];
          if (col >= cg0 && col < cg0 + CG) srcc[col - cg0] = tile_src[kk * TT + j];
        }
      }
      __syncthreads();
      bool any = false;
      for (int q = 0; q < CG; ++q) any |= srcc[q] >= 0;
      if (!any) continue;
      for (int idx = threadIdx.x; idx < n * CG; idx += kAT) {
        const int k = idx / CG, cc = idx % CG;
        const int s = srcc[cc];
        Bs[idx] = s >= 0 ? make_double2(mom[(int64_t)s * 2 * n_pad + k], mom[(int64_t)s * 2 * n_pad + n_pad + k])
                         : make_double2(0.0, 0.0);
      }
      const int key = tile_keys[kk];
      const int rk0 = rank[key];
      const bool dense = rk0 < 0;
      const int rk = dense ? n : rk0;
      const double2* Wk = Wall + woff[key];
      // Z = W B: thread (rg, c) rows q = rg + RG i
      double2 z[RMAX];
#pragma unroll
      for (int i = 0; i < RMAX; ++i) z[i] = make_double2(0.0, 0.0);
      for (int kb = 0; kb < n; kb += KC) {
        const int kw = min(KC, n - kb);
        __syncthreads();
        for (int idx = threadIdx.x; idx < rk * KC; idx += kAT) {
          const int q = idx / KC, t = idx % KC;
          Ws[idx] = t < kw ? Wk[(int64_t)q * n + kb + t] : make_double2(0.0, 0.0);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < RMAX; ++i) {
          const int q = rg + RG * i;
          if (q < rk) {
            double2 a = z[i];
            for (int t = 0; t < kw; ++t) {
              const double2 w = Ws[q * KC + t], b = Bs[(kb + t) * CG + c];
              a.x = fma(w.x, b.x, fma(-w.y, b.y, a.x));
              a.y = fma(w.x, b.y, fma(w.y, b.x, a.y));
            }
            z[i] = a;
          }
        }
      }
      if (dense) {  // U = identity: C += Z
#pragma unroll
        for (int i = 0; i < RMAX; ++i) {
          const int q = rg + RG * i;
          if (q < n) {
            acc[i].x += z[i].x;
            acc[i].y += z[i].y;
          }
        }
        continue;
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < RMAX; ++i) {
        const int q = rg + RG * i;
        if (q < rk) Zs[q * CG + c] = z[i];
      }
      __syncthreads();
      // C += U Z: rows j = rg + RG i
      const double2* Uk = Uall + uoff[key];
      for (int q = 0; q < rk; ++q) {
        const double2 zq = Zs[q * CG + c];
#pragma unroll
        for (int i = 0; i < RMAX; ++i) {
          const int j = rg + RG * i;
          if (j < n) {
            const double2 u = Uk[(int64_t)q * n + j];
            acc[i].x = fma(u.x, zq.x, fma(-u.y, zq.y, acc[i].x));
            acc[i].y = fma(u.x, zq.y, fma(u.y, zq.x, acc[i].y));
          }
        }
      }
    }
    // chained accumulation into the tile (item order), as the exact M2L kernels
    if (seq > 0 && !waited) {
      if (threadIdx.x == 0)
        while (ld_acquire_gpu(ticket + tile) != seq) __nanosleep(100);
      __syncthreads();
      waited = true;
    }
    const bool last = seq == nit - 1;
    const int col = cg0 + c;
#pragma unroll
    for (int i = 0; i < RMAX; ++i) {
      const int j = rg + RG * i;
      if (j >= n_pad) continue;
      double2 v = j < n ? acc[i] : make_double2(0.0, 0.0);
      double* pa = A + (int64_t)j * NC + 2 * col;
      if (seq > 0) {
        v.x += __ldcg(pa);
        v.y += __ldcg(pa + 1);
      }
      if (last) {
        const int32_t ts = tile_tslot[tile * TT + col];
        if (ts >= 0) {
          loc[(int64_t)ts * 2 * n_pad + j] = v.x;
          loc[(int64_t)ts * 2 * n_pad + n_pad + j] = v.y;
        }
      } else {
        __stcg(pa, v.x);
        __stcg(pa + 1, v.y);
      }
    }
  }
  if (seq != nit - 1) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(ticket + tile, seq + 1);
  }
}

}  // namespace

void launch_aca_factor(cudaStream_t st, const Consts* C, const double* dirtab, int64_t key0, int64_t nkeys,
                       const int32_t* key_level, const int64_t* key_d, const int32_t* key_dir, double eps, int n,
                       int pass, int32_t* rank, double2* scratch, const int64_t* uoff, const int64_t* woff,
                       double2* Uall, double2* Wall) {
  if (nkeys <= 0) return;
  const size_t sm = (size_t)n * (2 * sizeof(double2) + sizeof(double));
  k_aca_factor<<<(unsigned)nkeys, kAT, sm, st>>>(C, dirtab, key0, key_level, key_d, key_dir, eps, n, pass, rank,
                                                  scratch, uoff, woff, Uall, Wall);
}

int launch_m2l_aca(cudaStream_t st, int n, int n_pad, int tile, const M2LAcaArgs& a) {
  if (a.n_item <= 0) return 0;
  if (n > 384) return 1;
  const int cg = n <= 224 ? 16 : 8;
  const size_t sm = (size_t)n * (cg + 16 + cg) * sizeof(double2);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<a.n_item, kAT, sm, st>>>(a.item_tile, a.item_seq, a.item_k0, a.item_k1, a.tile_nitem, a.tile_tslot,
                                   a.tile_keys, a.tile_src, a.tile_cols, a.tile_cnt, a.rank, a.uoff, a.woff, a.U, a.W,
                                   a.mom, a.tile_acc, a.ticket, a.loc, a.counter, n, n_pad, tile);
  };
  if (cg == 16) go(k_m2l_aca<16>);
  else go(k_m2l_aca<8>);
  return 0;
}

}  // namespace fdhelm
