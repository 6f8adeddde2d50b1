// common.cuh -- device-side constants and helpers shared by the apply kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fdhelm {

constexpr int kMaxP = 11;       // m <= 10
constexpr int kMaxLevels = 24;  // tree depth <= 21 (+ margin)

// Per-operator constants, stored once in device memory and passed by pointer.
struct Consts {
  double kappa;
  int m, p, n, n_pad, lhf;
  int zero_diag;
  int pad0;
  double cheb_cos[kMaxP];             // cos((2nu-1) pi / (2p)), host std::cos
  double half[2 * kMaxP * kMaxP];     // half[h][j][k] = L_k^parent(child_h node j)
  double lo_t[3], lo_s[3];            // padded roots
  double side_t[kMaxLevels][3];       // level side lengths
  double side_s[kMaxLevels][3];
  int dir_off[kMaxLevels + 1];        // offsets into the direction-vector table (3 doubles each)
};

// ---- exact FP64 helpers: no FMA contraction, so box / node coordinates are
// bit-identical to the reference's host arithmetic (cluster_tree.cpp:130-139,
// interpolation.cpp:9-20).
__device__ __forceinline__ double box_lo(double root_lo, int64_t c, double side) {
  return __dadd_rn(root_lo, __dmul_rn((double)c, side));
}
__device__ __forceinline__ double box_hi(double root_lo, int64_t c, double side) {
  return __dadd_rn(root_lo, __dmul_rn((double)(c + 1), side));
}
// Chebyshev node nu of (a, b): mid + half * cos_nu.
__device__ __forceinline__ double cheb_node(double a, double b, double cosv) {
  const double mid = __dmul_rn(0.5, __dadd_rn(a, b));
  const double hw = __dmul_rn(0.5, __dsub_rn(b, a));
  return __dadd_rn(mid, __dmul_rn(hw, cosv));
}
// 1D Lagrange cardinals at x (product formula, interpolation.cpp:22-29).
__device__ __forceinline__ void cardinals(const double* nodes, int p, double x, double* out) {
  for (int i = 0; i < p; ++i) {
    double v = 1.0;
    for (int j = 0; j < p; ++j) {
      if (j == i) continue;
      v = __dmul_rn(v, __ddiv_rn(__dsub_rn(x, nodes[j]), __dsub_rn(nodes[i], nodes[j])));
    }
    out[i] = v;
  }
}
__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}

__device__ __forceinline__ const double* dir_vec(const Consts* C, const double* dirtab, int level, int dir) {
  return dirtab + C->dir_off[level] + 3 * dir;
}

}  // namespace fdhelm
