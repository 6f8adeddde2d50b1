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
// Barycentric form of the same cardinals: den[i] = 1 / prod_{j != i}(x_i - x_j)
// once per box (p divisions), then L_i(x) = prefix_i * suffix_i * den[i] with the
// products of (x - x_j) over j < i and j > i: ~4p multiplications per point
// instead of p (p - 1) divisions (the S2M / L2T per-point cost).  Same value as
// cardinals() up to rounding (y tolerance 1e-12; the trees and lists, which must
// be bit-exact, never use it).
__device__ __forceinline__ void cardinal_den(const double* nodes, int p, int i, double* den) {
  double v = 1.0;
  for (int j = 0; j < p; ++j)
    if (j != i) v *= nodes[i] - nodes[j];
  den[i] = 1.0 / v;
}
__device__ __forceinline__ void cardinals_bary(const double* nodes, const double* den, int p, double x, double* out) {
  double d[kMaxP];
  for (int j = 0; j < p; ++j) d[j] = x - nodes[j];
  double pre = 1.0;
  for (int i = 0; i < p; ++i) {
    out[i] = pre * den[i];
    pre *= d[i];
  }
  double suf = 1.0;
  for (int i = p - 1; i >= 0; --i) {
    out[i] *= suf;
    suf *= d[i];
  }
}
__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}

__device__ __forceinline__ const double* dir_vec(const Consts* C, const double* dirtab, int level, int dir) {
  return dirtab + C->dir_off[level] + 3 * dir;
}

}  // namespace fdhelm

namespace fdhelm {
// sin and cos of x with a 3-part Cody-Waite reduction by pi/2 and the FDLIBM
// minimax kernels on [-pi/4, pi/4] (|error| <= ~1 ulp); |x| >= 2^20 * pi/2
// falls back to the CUDA library sincos.  ~22 FP64 ops instead of ~40.
__device__ __forceinline__ void sincos_fast(double x, double* s, double* c) {
  if (fabs(x) >= 1.6e6) {
    sincos(x, s, c);
    return;
  }
  const double k = rint(x * 6.36619772367581382433e-01);  // x * 2/pi
  double y = fma(-k, 1.57079632673412561417e+00, x);       // pio2_1 (33 bits)
  y = fma(-k, 6.07710050630396597660e-11, y);              // pio2_2 (33 bits)
  y = fma(-k, 2.02226624879595063154e-21, y);              // pio2_2t
  const double z = y * y;
  double ps = fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08);
  ps = fma(z, ps, 2.75573137070700676789e-06);
  ps = fma(z, ps, -1.98412698298579493134e-04);
  ps = fma(z, ps, 8.33333333332248946124e-03);
  ps = fma(z, ps, -1.66666666666666324348e-01);
  const double sy = fma(y * z, ps, y);
  double pc = fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09);
  pc = fma(z, pc, -2.75573143513906633035e-07);
  pc = fma(z, pc, 2.48015872894767294178e-05);
  pc = fma(z, pc, -1.38888888888741095749e-03);
  pc = fma(z, pc, 4.16666666666666019037e-02);
  const double cy = fma(z * z, pc, fma(-0.5, z, 1.0));
  const int q = (int)(long long)k & 3;
  const double ss = (q & 1) ? cy : sy;
  const double cc = (q & 1) ? sy : cy;
  *s = (q & 2) ? -ss : ss;
  *c = ((q + 1) & 2) ? -cc : cc;
}
}  // namespace fdhelm

namespace fdhelm {
// Coefficients of sincos_fast in the constant bank: FP64 instructions take
// c[][] operands directly, so the hot loop needs no per-iteration constant
// materialisation (UMOV pairs) -- see k_p2p.
__constant__ double c_trig[18] = {
    6.36619772367581382433e-01,   // 2/pi
    1.57079632673412561417e+00,   // pio2_1
    6.07710050630396597660e-11,   // pio2_2
    2.02226624879595063154e-21,   // pio2_2t
    1.58969099521155010221e-10,  -2.50507602534068634195e-08, 2.75573137070700676789e-06,
    -1.98412698298579493134e-04, 8.33333333332248946124e-03,  -1.66666666666666324348e-01,  // sin
    -1.13596475577881948265e-11, 2.08757232129817482790e-09,  -2.75573143513906633035e-07,
    2.48015872894767294178e-05,  -1.38888888888741095749e-03, 4.16666666666666019037e-02,   // cos
    0.5, 1.0};

// sincos_fast without the large-argument guard: the caller guarantees |x| < 1.6e6.
// k = rint(x 2/pi) via the 1.5*2^52 shifter (one FMA + one add, the quadrant
// from the shifter's low mantissa bits: no FRND / F2I), sign flips by integer xor.
__device__ __forceinline__ void sincos_fast_nc(double x, double* s, double* c) {
  const double shifter = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(x, c_trig[0], shifter);
  const double k = t - shifter;
  const int q = __double2loint(t) & 3;
  double y = fma(-k, c_trig[1], x);
  y = fma(-k, c_trig[2], y);
  y = fma(-k, c_trig[3], y);
  const double z = y * y;
  double ps = fma(z, c_trig[4], c_trig[5]);
  ps = fma(z, ps, c_trig[6]);
  ps = fma(z, ps, c_trig[7]);
  ps = fma(z, ps, c_trig[8]);
  ps = fma(z, ps, c_trig[9]);
  const double sy = fma(y * z, ps, y);
  double pc = fma(z, c_trig[10], c_trig[11]);
  pc = fma(z, pc, c_trig[12]);
  pc = fma(z, pc, c_trig[13]);
  pc = fma(z, pc, c_trig[14]);
  pc = fma(z, pc, c_trig[15]);
  const double cy = fma(z * z, pc, fma(-c_trig[16], z, c_trig[17]));
  const double ss = (q & 1) ? cy : sy;
  const double cc = (q & 1) ? sy : cy;
  const long long sgs = (long long)(q & 2) << 62;        // sin negative in quadrants 2, 3
  const long long sgc = (long long)((q + 1) & 2) << 62;  // cos negative in quadrants 1, 2
  *s = __longlong_as_double(__double_as_longlong(ss) ^ sgs);
  *c = __longlong_as_double(__double_as_longlong(cc) ^ sgc);
}
}  // namespace fdhelm
