// m2l_split.hpp -- shared by the host planner (issued-work accounting) and
// k_m2l_gemm (scheme dispatch).
#pragma once

#ifndef FDH_GAUSS_MAX_NPAD
#define FDH_GAUSS_MAX_NPAD 224
#endif

namespace fdhelm {

#ifdef __CUDACC__
#define FDH_HD __host__ __device__
#else
#define FDH_HD
#endif
// Split of a tile key's cnt compacted target columns between the two DMMA
// schemes of k_m2l_gemm: a3 n-tiles of 8 targets in the 3-multiplication
// (Gauss) complex product (3 real products of K = n_k: cost 3 units) and ao
// n-tiles of 4 targets in the [Re A | Im A] real GEMM (K = 2 n_k: cost 2 units).
// One unit = 16 n_pad n_k flop issued on DMMA.
struct M2LSplit {
  int a3, ao;
};
// the Gauss scheme is used for n_pad <= 128 (k_m2l_gemm: register budget)
FDH_HD constexpr bool m2l_gauss(int n_pad) { return n_pad <= FDH_GAUSS_MAX_NPAD; }
// planes of a coupling matrix row: [Re A | Im A] (+ Re A + Im A for the Gauss shapes)
FDH_HD constexpr int m2l_wplanes(int n_pad) { return m2l_gauss(n_pad) ? 3 : 2; }
FDH_HD inline M2LSplit m2l_split(int cnt, bool gauss) {
  if (!gauss) return {0, (cnt + 3) >> 2};
  const int r = cnt & 7;  // remainder after full 8-target Gauss n-tiles
  return {(cnt >> 3) + (r >= 5 ? 1 : 0), (r >= 1 && r <= 4) ? 1 : 0};
}

}  // namespace fdhelm
