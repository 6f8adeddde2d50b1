// fdhelm_b200.hpp -- header-only C++20 host API over the C-ABI (fdhelm_c.h).
//
// Mirrors the reference's C++ vocabulary so that a caller of
//   fdhelm::ClusterTree(std::span<const Point3>, const AxisBox&, int n_max, int depth_cap)
//   (/root/reference/proj/include/fdhelm/cluster_tree.hpp:47) and of the SPEC L4 engine
//   setup(T_T, T_S, ..., kappa, m) / matvec(op, v) / stats(op)
// can switch with a handful of lines.  Errors are re-thrown as
// the reference's exception types: std::invalid_argument (FDH_ERR_ARG, DIM),
// std::domain_error (FDH_ERR_DOMAIN, singular kernel), std::runtime_error (CUDA).
#pragma once
#include <array>
#include <complex>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fdhelm_c.h"

namespace fdhelm_b200 {

using Complex = std::complex<double>;

struct Params {
  double kappa = 1.0;      // WaveNumber (geometry.hpp:38-43), > 0
  int n_max = 64;          // ClusterTree n_max (cluster_tree.hpp:47)
  int m = 4;               // Chebyshev degree, (m+1)^3 nodes per box
  double eta2 = 1.0;       // admissibility constant of (A1)/(A3)
  int l_hf = FDH_LHF_DEFAULT;
  int depth_cap = 30;
  bool zero_diagonal = false;
  int nrhs = 1;            // right-hand sides per device batch (power of two, <= 16)
  int n_gpus = 1;          // > 1: one process drives devices 0..n_gpus-1 (target shards, NCCL reduce of y)
};

inline void check(int rc) {
  if (rc == FDH_OK) return;
  const std::string msg = fdh_last_error();
  switch (rc) {
    case FDH_ERR_ARG:
    case FDH_ERR_DIM: throw std::invalid_argument(msg);
    case FDH_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error("fdhelm_b200: " + msg);
  }
}

namespace detail {
template <class P>
std::vector<double> axis(std::span<const P> pts, int a) {
  std::vector<double> v(pts.size());
  for (size_t i = 0; i < pts.size(); ++i) v[i] = a == 0 ? pts[i].x : (a == 1 ? pts[i].y : pts[i].z);
  return v;
}
}  // namespace detail

class DirectionalOperator {
 public:
  // AoS points with members x, y, z -- e.g. std::span<const fdhelm::Point3>
  // (geometry.hpp:13-20) -- and any box with lower / upper points (AxisBox,
  // geometry.hpp:46-59): the reference's own types work unchanged.
  template <class Pt, class Box>
  DirectionalOperator(std::span<const Pt> targets, std::span<const Pt> sources, const Box& root, const Params& p)
      : DirectionalOperator(detail::axis(targets, 0), detail::axis(targets, 1), detail::axis(targets, 2),
                            detail::axis(sources, 0), detail::axis(sources, 1), detail::axis(sources, 2),
                            std::array<double, 3>{root.lower.x, root.lower.y, root.lower.z}.data(),
                            std::array<double, 3>{root.upper.x, root.upper.y, root.upper.z}.data(), p) {}
  DirectionalOperator(const std::vector<double>& tx, const std::vector<double>& ty, const std::vector<double>& tz,
                      const std::vector<double>& sx, const std::vector<double>& sy, const std::vector<double>& sz,
                      const double* root_lo, const double* root_hi, const Params& p)
      : DirectionalOperator(std::span<const double>(tx), std::span<const double>(ty), std::span<const double>(tz),
                            std::span<const double>(sx), std::span<const double>(sy), std::span<const double>(sz),
                            root_lo, root_hi, p) {}
  // Points as SoA spans (x, y, z) of targets and sources; one shared root box.
  DirectionalOperator(std::span<const double> tx, std::span<const double> ty, std::span<const double> tz,
                      std::span<const double> sx, std::span<const double> sy, std::span<const double> sz,
                      const double root_lo[3], const double root_hi[3], const Params& p)
      : nt_(tx.size()), ns_(sx.size()) {
    if (ty.size() != nt_ || tz.size() != nt_ || sy.size() != ns_ || sz.size() != ns_)
      throw std::invalid_argument("coordinate arrays of one point set differ in length");
    if (p.n_gpus > 1) {
      if (p.nrhs != 1) throw std::invalid_argument("n_gpus > 1 takes one right-hand side per apply");
      check(fdh_create(tx.data(), ty.data(), tz.data(), (int64_t)nt_, sx.data(), sy.data(), sz.data(), (int64_t)ns_,
                       root_lo, root_hi, p.kappa, p.n_max, p.m, p.eta2, p.l_hf, p.depth_cap, p.zero_diagonal ? 1 : 0,
                       p.n_gpus, &op_));
    } else {
      check(fdh_create_multi(tx.data(), ty.data(), tz.data(), (int64_t)nt_, sx.data(), sy.data(), sz.data(),
                             (int64_t)ns_, root_lo, root_hi, p.kappa, p.n_max, p.m, p.eta2, p.l_hf, p.depth_cap,
                             p.zero_diagonal ? 1 : 0, 0, 1, p.nrhs, &op_));
    }
  }
  DirectionalOperator(const DirectionalOperator&) = delete;
  DirectionalOperator& operator=(const DirectionalOperator&) = delete;
  ~DirectionalOperator() { fdh_destroy(op_); }

  // SPEC.md:493-501 matvec: y (N_T) = A x (N_S), original point order.
  void apply(std::span<const Complex> x, std::span<Complex> y) {
    if (x.size() != ns_ || y.size() != nt_) throw std::invalid_argument("matvec: dimension mismatch");
    check(fdh_apply(op_, reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data())));
  }
  std::vector<Complex> apply(std::span<const Complex> x) {
    std::vector<Complex> y(nt_);
    apply(x, y);
    return y;
  }
  // Y = A X for k right-hand sides, X column-major N_S x k
  // (column r = x[r * N_S ...]), Y column-major N_T x k.
  void apply_multi(std::span<const Complex> X, std::span<Complex> Y, int64_t k) {
    if (k < 1 || X.size() != ns_ * (size_t)k || Y.size() != nt_ * (size_t)k)
      throw std::invalid_argument("matvec: dimension mismatch");
    check(fdh_apply_multi(op_, reinterpret_cast<const double*>(X.data()), k, reinterpret_cast<double*>(Y.data())));
  }
  fdh_stats stats() const {
    fdh_stats s{};
    check(fdh_get_stats(op_, &s));
    return s;
  }
  fdh_op* handle() { return op_; }
  // options for repeated applies: ACA-compressed coupling (lossy, SPEC.md:440-448;
  // eps = 0 -> exact) and the cached near-field kernel values
  void set_aca(double eps) { check(fdh_set_aca(op_, eps)); }
  void set_cache_nearfield(bool on) { check(fdh_set_cache(op_, on ? FDH_CACHE_NEARFIELD : 0)); }
  // device-resident apply (x_dev, y_dev: device pointers; errors deferred to sync())
  void apply_device(const Complex* x_dev, Complex* y_dev, void* stream = nullptr) {
    check(fdh_apply_device(op_, reinterpret_cast<const double*>(x_dev), reinterpret_cast<double*>(y_dev), stream));
  }
  void sync() { check(fdh_sync(op_)); }

  // canonical introspection (int64 rows, see fdhelm_c.h): the cluster trees
  // (level, i, j, k, begin, end, leaf), slot -> original index permutations,
  // admissible blocks L+ (level, t ijk, s ijk, direction), inadmissible L-,
  // and the direction sets D / D^ (level, ijk, direction, kind)
  std::vector<int64_t> tree(int which) const { return rows(fdh_export_tree, which, 7); }
  std::vector<int64_t> perm(int which) const { return rows(fdh_export_perm, which, 1); }
  std::vector<int64_t> lplus() const { return rows2(fdh_export_lplus, 8); }
  std::vector<int64_t> lminus() const { return rows2(fdh_export_lminus, 8); }
  std::vector<int64_t> dirsets(int which) const { return rows(fdh_export_dirsets, which, 6); }

 private:
  template <class F>
  std::vector<int64_t> rows(F f, int which, int cols) const {
    const int64_t n = f(op_, which, nullptr);
    std::vector<int64_t> out((size_t)(n * cols));
    if (n > 0) f(op_, which, out.data());
    return out;
  }
  template <class F>
  std::vector<int64_t> rows2(F f, int cols) const {
    const int64_t n = f(op_, nullptr);
    std::vector<int64_t> out((size_t)(n * cols));
    if (n > 0) f(op_, out.data());
    return out;
  }
  size_t nt_, ns_;
  fdh_op* op_ = nullptr;
};

}  // namespace fdhelm_b200
