// kernels.hpp -- host-side launchers of the apply kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "m2l_split.hpp"

namespace fdhelm {

// ---- k_apply.cu
void launch_gather_charges(cudaStream_t st, int64_t ns, const uint32_t* perm, const double2* x, double2* q,
                           double2* q4);
void launch_scatter_y(cudaStream_t st, int64_t nt, const uint32_t* perm, const double2* y_slot, double2* y);
void launch_s2m(cudaStream_t st, const Consts* C, const double* dirtab, int n_entry, const int32_t* slot,
                const int32_t* level, const int32_t* dir, const int64_t* ci, const int64_t* cj, const int64_t* ck,
                const uint32_t* beg, const uint32_t* end, const double* px, const double* py, const double* pz,
                const double2* q, double* mom, int n, int n_pad);
void launch_m2m(cudaStream_t st, const Consts* C, const double* dirtab, int level, int n_entry,
                const int32_t* parent, const int32_t* pdir, const int32_t* cdir, const int32_t* child,
                const int64_t* pc, double* mom, int n, int n_pad);
void launch_l2l(cudaStream_t st, const Consts* C, const double* dirtab, int level, int n_entry,
                const int32_t* child, const int32_t* cdir, const int64_t* cc, const int32_t* ptr,
                const int32_t* pslot, const int32_t* pdir, const int32_t* oct, double* loc, int n, int n_pad);
void launch_l2t(cudaStream_t st, const Consts* C, const double* dirtab, int n_entry, const int32_t* level,
                const int32_t* slot0, const int32_t* nslot, const int64_t* ci, const int64_t* cj,
                const int64_t* ck, const uint32_t* beg, const uint32_t* end, const double* px,
                const double* py, const double* pz, const int32_t* slot_dir, const double* loc,
                const double2* y_near, double2* y_slot, int n, int n_pad);
void launch_p2p(cudaStream_t st, double kappa, int n_entry, const uint32_t* beg, const uint32_t* end,
                const int64_t* ptr, const uint32_t* sbeg, const uint32_t* send, const double* tx,
                const double* ty, const double* tz, const double* sx, const double* sy, const double* sz,
                const double2* q4, const uint32_t* perm_t, const uint32_t* perm_s, int zero_diag,
                double2* y_slot, int* flag, double max_phase, const double2* sctab, int nrhs = 1,
                int64_t qstride = 0, int64_t ystride = 0, int grid = 0);
int p2p_launches(int nrhs);

// ---- k_m2l.cu
void launch_coupling(cudaStream_t st, const Consts* C, const double* dirtab, int64_t key0, int64_t nkeys,
                     const int32_t* key_level, const int64_t* key_d, const int32_t* key_dir, double* W,
                     int n, int n_pad, int n_k, int64_t wbase);
struct M2LArgs {
  int n_item = 0;      // items of this launch: [item0, item0 + n_item)
  int item0 = 0;
  int64_t key_base = 0;  // W holds the keys [key_base, ...) (on-the-fly coupling segments)
  const int32_t *item_tile = nullptr, *item_seq = nullptr;
  const int64_t *item_k0 = nullptr, *item_k1 = nullptr;
  const int32_t *tile_nitem = nullptr, *tile_tslot = nullptr, *tile_keys = nullptr, *tile_src = nullptr;
  const uint8_t *tile_cols = nullptr, *tile_cnt = nullptr, *tile_same = nullptr;
  const double *W = nullptr, *mom = nullptr;
  double* tile_acc = nullptr;
  int* ticket = nullptr;
  double* loc = nullptr;
  int* err = nullptr;
  int* counter = nullptr;  // zeroed item-claim counter (one per launch)
};
// returns 0 on success, nonzero if the n_pad / tile combination is not compiled
int launch_m2l_gemm(cudaStream_t st, int n_pad, int n_k, int tile, const M2LArgs& a);

// ---- k_m2l_i8.cu: M2L on tcgen05 int8 tensor cores (exact fixed-point digit products)
// Fixed-point format of the digit products: kI8Digits balanced digits of kI8Bits bits.
//   6 x 8 (default): base-256 digits in [-128, 127], 48 bits, 21 digit-pair products
//   7 x 7          : base-128 digits in [-64, 64],   49 bits, 28 products (round 1 / early round 2)
//   7 x 8          : 56 bits, 28 products (wider margin at the 7 x 7 cost)
#ifndef FDH_I8_DIGITS
#define FDH_I8_DIGITS 6
#endif
#ifndef FDH_I8_BITS
#define FDH_I8_BITS 8
#endif
// Digit pairs (i, j) with i + j <= kI8Levels - 1 are kept.  Default for 6 x 8: one level
// more than digits (26 products: the five level-6 pairs would otherwise dominate the error,
// ~6x the 48-bit rounding; same operand bytes, one more TMEM level block).
#ifndef FDH_I8_LEVELS
#define FDH_I8_LEVELS (FDH_I8_BITS == 8 && FDH_I8_DIGITS == 6 ? 7 : FDH_I8_DIGITS)
#endif
constexpr int kI8Digits = FDH_I8_DIGITS;
constexpr int kI8Bits = FDH_I8_BITS;
constexpr int kI8Levels = FDH_I8_LEVELS;
static_assert(kI8Levels >= kI8Digits && kI8Levels <= 2 * kI8Digits - 1, "levels");
// digit-pair products kept: sum over W digits i of min(KS, LV - i) B digits
constexpr int i8_products() {
  int s = 0;
  for (int i = 0; i < kI8Digits; ++i) s += (kI8Levels - i < kI8Digits ? kI8Levels - i : kI8Digits);
  return s;
}
static_assert(kI8Bits == 7 || kI8Bits == 8, "int8 digits");
constexpr int kI8DigitMax = 1 << (kI8Bits - 1);  // |digit| <= 64 (7 bits) / 128 (8 bits)
struct M2LI8Args {
  int n_item = 0, item0 = 0;
  const int32_t *item_tile = nullptr, *item_seq = nullptr;
  const int64_t *item_k0 = nullptr, *item_k1 = nullptr;
  const int32_t *tile_nitem = nullptr, *tile_tslot = nullptr, *tile_level = nullptr, *tile_keys = nullptr,
                *tile_src = nullptr;
  const uint8_t *tile_cols = nullptr, *tile_cnt = nullptr;
  const int8_t *Wq = nullptr, *Mq = nullptr;
  const unsigned long long *lvmax_w = nullptr, *lvmax_v = nullptr;
  double* tile_acc = nullptr;
  int* ticket = nullptr;
  double* loc = nullptr;
  int* err = nullptr;
  int nkq = 0, n_pad = 0, fkeys = 0;
  int n_tile = 0;        // ticket chains: one per tile and M-block group (m = 6: 2 groups)
  int64_t key_base = 0;  // first key of the Wq buffer (on-the-fly segments)
  int nrhs = 1;          // moment scales per (rhs, level): lvmax_v[rhs * kMaxLevels + level];
                         // tile column c = (slot, rhs) with rhs = c % nrhs
  int* counter = nullptr;  // zeroed item-claim counters, one per M-block pass (persistent grid)
  double* pair_out = nullptr;  // pair mode: per (item, column) the pair's 2 n_pad values
};
void launch_m2l_reduce(cudaStream_t st, int64_t nslots, const int64_t* red_ptr, const int64_t* red_idx,
                       int64_t* cursor, const double* out, int64_t p0, int64_t p1, double* loc, int n_pad);
void launch_m2l_add(cudaStream_t st, double* loc, const double* add, int64_t n);
int m2l_i8_supported(int n, int tile);
int m2l_i8_fkeys(int nkq);                    // max keys per item (int32 accumulators exact)
int64_t m2l_i8_wbytes_per_key(int n, int nkq, int tile);
int64_t m2l_i8_mbytes_per_slot(int nkq);
// gs: M-blocks per W group (m2l_i8_wgroup)
void launch_coupling_i8(cudaStream_t st, const Consts* C, const double* dirtab, int64_t key0, int64_t nkeys,
                        const int32_t* key_level, const int64_t* key_d, const int32_t* key_dir, int pass,
                        unsigned long long* lvmax, int8_t* Wq, int n, int nkq, int gs, int64_t key_base = 0);
int m2l_i8_passes(int n, int tile);  // M-block passes over the items (= ticket chains / claim counters)
int m2l_i8_wgroup(int n, int tile);  // M-blocks stored together per W group (2: {0,1},{2}; 1: per block)
void launch_mom_quant(cudaStream_t st, const double* mom, const int32_t* slot_level, int64_t nslots, int n, int n_pad,
                      int nkq, unsigned long long* lvmax_v, int8_t* Mq, int nrhs = 1);
int launch_m2l_i8(cudaStream_t st, int n, int tile, const M2LI8Args& a);

// ---- k_aca.cu: ACA-compressed coupling (opt-in, lossy)
struct M2LAcaArgs {
  int n_item = 0;
  const int32_t *item_tile = nullptr, *item_seq = nullptr;
  const int64_t *item_k0 = nullptr, *item_k1 = nullptr;
  const int32_t *tile_nitem = nullptr, *tile_tslot = nullptr, *tile_keys = nullptr, *tile_src = nullptr;
  const uint8_t *tile_cols = nullptr, *tile_cnt = nullptr;
  const int32_t* rank = nullptr;  // per key: ACA rank, -1 = dense (W = A, U = I)
  const int64_t *uoff = nullptr, *woff = nullptr;
  const double2 *U = nullptr, *W = nullptr;
  const double* mom = nullptr;
  double* tile_acc = nullptr;
  int* ticket = nullptr;
  double* loc = nullptr;
  int* counter = nullptr;
};
// pass 0: ranks (scratch: nkeys x n (n + 1) complex); pass 1: factors at uoff / woff
void launch_aca_factor(cudaStream_t st, const Consts* C, const double* dirtab, int64_t key0, int64_t nkeys,
                       const int32_t* key_level, const int64_t* key_d, const int32_t* key_dir, double eps, int n,
                       int pass, int32_t* rank, double2* scratch, const int64_t* uoff, const int64_t* woff,
                       double2* Uall, double2* Wall);
int launch_m2l_aca(cudaStream_t st, int n, int n_pad, int tile, const M2LAcaArgs& a);

// ---- cached near field (k_apply.cu; opt-in, fdh_set_cache)
void launch_p2p_cache_fill(cudaStream_t st, double kappa, int n_entry, const uint32_t* beg, const uint32_t* end,
                           const int64_t* ptr, const uint32_t* sbeg, const uint32_t* send, const double* tx,
                           const double* ty, const double* tz, const double* sx, const double* sy, const double* sz,
                           const uint32_t* diag_slot, int zero_diag, const int64_t* koff, const int64_t* poff,
                           double2* K, uint32_t* spos, int* flag);
void launch_p2p_cached(cudaStream_t st, int n_entry, const uint32_t* beg, const uint32_t* end, const int64_t* koff,
                       const int64_t* poff, const uint32_t* spos, const double2* K, const double2* q, double2* y_slot,
                       int nrhs, int64_t qstride, int64_t ystride);

}  // namespace fdhelm
