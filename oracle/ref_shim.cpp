// ref_shim.cpp -- C entry points over the REFERENCE's own C++ (compiled from
// /root/reference/proj/src/{cluster_tree,interpolation}.cpp, unmodified, by
// oracle/Makefile into oracle/_ref/libfdhelm_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the oracle restatement
// (oracle.cpp) against the reference itself, and to generate the golden
// fixtures under tests/golden/.  Never linked by the product.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "fdhelm/cluster_tree.hpp"
#include "fdhelm/geometry.hpp"
#include "fdhelm/interpolation.hpp"

using namespace fdhelm;

namespace {
thread_local std::string g_err;
struct RefTree {
  ClusterTree* t;
};
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ClusterTree(points, root, n_max, depth_cap) (cluster_tree.hpp:47)
void* ref_tree_create(const double* x, const double* y, const double* z, int64_t n, const double lo[3],
                      const double hi[3], int n_max, int depth_cap) {
  try {
    std::vector<Point3> pts(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) pts[i] = {x[i], y[i], z[i]};
    AxisBox root{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
    return new RefTree{new ClusterTree(std::span<const Point3>(pts), root, n_max, depth_cap)};
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_tree_destroy(void* h) {
  auto* r = static_cast<RefTree*>(h);
  delete r->t;
  delete r;
}
int ref_tree_depth(void* h) { return static_cast<RefTree*>(h)->t->depth(); }
int ref_tree_oversized(void* h) { return static_cast<RefTree*>(h)->t->oversized_leaf_count(); }
double ref_tree_level_diameter(void* h, int l) { return static_cast<RefTree*>(h)->t->level_diameter(l); }
// canonical rows: level, i, j, k, begin, end, leaf (level_nodes order = sorted by coord)
int64_t ref_tree_export(void* h, int64_t* out) {
  const ClusterTree& t = *static_cast<RefTree*>(h)->t;
  int64_t r = 0;
  for (int l = 0; l <= t.depth(); ++l)
    for (int32_t id : t.level_nodes(l)) {
      if (out) {
        const ClusterNode& nd = t.node(id);
        int64_t* row = out + 7 * r;
        row[0] = nd.coord.level; row[1] = nd.coord.i; row[2] = nd.coord.j; row[3] = nd.coord.k;
        row[4] = nd.begin; row[5] = nd.end; row[6] = nd.leaf ? 1 : 0;
      }
      ++r;
    }
  return r;
}
int64_t ref_tree_perm(void* h, int64_t* out) {
  const ClusterTree& t = *static_cast<RefTree*>(h)->t;
  if (out)
    for (size_t s = 0; s < t.point_count(); ++s) out[s] = t.original_index(static_cast<uint32_t>(s));
  return static_cast<int64_t>(t.point_count());
}
// box of the node at a coordinate; returns 0 if present (node_at, cpp:141-149)
int ref_tree_box(void* h, int level, int64_t i, int64_t j, int64_t k, double* lo, double* hi) {
  const ClusterTree& t = *static_cast<RefTree*>(h)->t;
  auto id = t.node_at(GridCoord{level, i, j, k});
  if (!id) return -1;
  const AxisBox b = t.box(*id);
  lo[0] = b.lower.x; lo[1] = b.lower.y; lo[2] = b.lower.z;
  hi[0] = b.upper.x; hi[1] = b.upper.y; hi[2] = b.upper.z;
  return 0;
}

int ref_chebyshev_nodes(double a, double b, int m, double* out) {
  try {
    auto v = chebyshev_nodes(a, b, m);
    std::copy(v.begin(), v.end(), out);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
double ref_lagrange_eval(const double* nodes, int n, int idx, double x) {
  return lagrange_eval(std::span<const double>(nodes, static_cast<size_t>(n)), idx, x);
}
// row-major output of the 8 n x n transfer matrices
int ref_transfer_reference(int m, double* out) {
  const TransferRef r = build_transfer_reference(m);
  const int n = tensor_node_count(m);
  for (int o = 0; o < 8; ++o)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) out[(static_cast<size_t>(o) * n + j) * n + k] = r.E[o](j, k);
  return 0;
}
int ref_interp_matrix(const double* px, const double* py, const double* pz, int64_t np, const double lo[3],
                      const double hi[3], const double c[3], double kappa, int m, double* out) {
  std::vector<Point3> pts(static_cast<size_t>(np));
  for (int64_t i = 0; i < np; ++i) pts[i] = {px[i], py[i], pz[i]};
  AxisBox b{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
  const Eigen::MatrixXcd L = build_interp_matrix(std::span<const Point3>(pts), b, {c[0], c[1], c[2]}, kappa, m);
  const int n = tensor_node_count(m);
  for (int64_t j = 0; j < np; ++j)
    for (int k = 0; k < n; ++k) {
      out[2 * (j * n + k)] = L(j, k).real();
      out[2 * (j * n + k) + 1] = L(j, k).imag();
    }
  return 0;
}
int ref_directional_diag(const double lo[3], const double hi[3], const double c[3], const double cc[3],
                         double kappa, int m, double* out) {
  AxisBox b{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
  const Eigen::VectorXcd d = build_directional_diag(b, {c[0], c[1], c[2]}, {cc[0], cc[1], cc[2]}, kappa, m);
  for (int j = 0; j < tensor_node_count(m); ++j) {
    out[2 * j] = d(j).real();
    out[2 * j + 1] = d(j).imag();
  }
  return 0;
}
int ref_kernel(const double d[3], double kappa, double* out2) {
  try {
    const Complex k = kernel_diff({d[0], d[1], d[2]}, kappa);
    out2[0] = k.real();
    out2[1] = k.imag();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
int ref_kernel_directional(const double d[3], const double c[3], double kappa, double* out2) {
  try {
    const Complex k = kernel_directional_diff({d[0], d[1], d[2]}, {c[0], c[1], c[2]}, kappa);
    out2[0] = k.real();
    out2[1] = k.imag();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
double ref_box_distance(const double tlo[3], const double thi[3], const double slo[3], const double shi[3]) {
  AxisBox t{{tlo[0], tlo[1], tlo[2]}, {thi[0], thi[1], thi[2]}};
  AxisBox s{{slo[0], slo[1], slo[2]}, {shi[0], shi[1], shi[2]}};
  return box_distance(t, s);
}
double ref_box_diameter(const double lo[3], const double hi[3]) {
  AxisBox b{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
  return box_diameter(b);
}
}  // extern "C"
