// oracle.cpp -- CPU restatement of the directional multi-level Helmholtz matvec.
//
// TEST INFRASTRUCTURE ONLY (the parity checker).  Loaded by tests/, by
// __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
// leg; the product (paper_2004_14229_b200/) never links or calls it.
//
// Every function cites the reference text it restates.  The reference ships
// C++ for geometry / cluster tree / interpolation only; directions, block tree,
// coupling and the engine exist as PAPER/SPEC text and are restated here with
// the conventions pinned in SURVEY.md Appendix B.
//
// Build: oracle/Makefile (g++ -O2 -fopenmp -ffp-contract=off; no -march so
// that x86-64 baseline code has no FMA, like the reference's default build,
// SURVEY.md App. C).

#include "oracle.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

namespace {

using cplx = std::complex<double>;
constexpr double kPi = 3.141592653589793;                // std::numbers::pi
constexpr double kFourPi = 4.0 * 3.14159265358979323846;  // geometry.hpp:11
constexpr double kRootPad = 1e-12;                        // cluster_tree.cpp:9

thread_local std::string g_err;

struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
// error codes shared with include/fdhelm_c.h
enum { E_ARG = 1, E_DOMAIN = 2, E_DIM = 3, E_UNSUPPORTED = 4 };

// ---------------------------------------------------------------- geometry
// geometry.hpp:27 dot is evaluated left to right: (ax*bx + ay*by) + az*bz.
inline double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double norm3(const double* a) { return std::sqrt(dot3(a, a)); }

// geometry.hpp:80-86 kernel_diff
inline cplx kernel_diff(const double d[3], double kappa) {
  const double r = norm3(d);
  if (r == 0.0) throw Err(E_DOMAIN, "Helmholtz kernel is singular at x == y");
  const double phase = kappa * r;
  const double w = 1.0 / (kFourPi * r);
  return {w * std::cos(phase), w * std::sin(phase)};
}
// geometry.hpp:92-98 kernel_directional_diff
inline cplx kernel_dir_diff(const double d[3], const double c[3], double kappa) {
  const double r = norm3(d);
  if (r == 0.0) throw Err(E_DOMAIN, "Helmholtz kernel is singular at x == y");
  const double phase = kappa * (r - dot3(d, c));
  const double w = 1.0 / (kFourPi * r);
  return {w * std::cos(phase), w * std::sin(phase)};
}

// ----------------------------------------------------------- interpolation
// interpolation.cpp:9-20 chebyshev_nodes
std::vector<double> cheb(double a, double b, int m) {
  if (!(a < b)) throw Err(E_ARG, "chebyshev_nodes: degenerate interval");
  if (m < 0) throw Err(E_ARG, "chebyshev_nodes: negative degree");
  const int n = m + 1;
  const double mid = 0.5 * (a + b), half = 0.5 * (b - a);
  std::vector<double> x(n);
  for (int nu = 1; nu <= n; ++nu) x[nu - 1] = mid + half * std::cos((2.0 * nu - 1.0) * kPi / (2.0 * n));
  return x;
}
// interpolation.cpp:22-29 lagrange_eval (product formula)
double lagr(const double* nodes, int n, int idx, double x) {
  double v = 1.0;
  for (int j = 0; j < n; ++j) {
    if (j == idx) continue;
    v *= (x - nodes[j]) / (nodes[idx] - nodes[j]);
  }
  return v;
}
void cardinals(const std::vector<double>& nodes, double x, double* out) {
  const int n = (int)nodes.size();
  for (int i = 0; i < n; ++i) out[i] = lagr(nodes.data(), n, i, x);
}

struct Box { double lo[3], hi[3]; };

// Tensor grid nodes of a box (interpolation.cpp:31-43): 3 axis node lists.
struct Grid {
  std::vector<double> ax[3];
  Grid(const Box& b, int m) { for (int a = 0; a < 3; ++a) ax[a] = cheb(b.lo[a], b.hi[a], m); }
  void node(int flat, int p, double* out) const {
    out[0] = ax[0][flat / (p * p)];
    out[1] = ax[1][(flat / p) % p];
    out[2] = ax[2][flat % p];
  }
};

// interpolation.cpp:56-87: row j of L_{t,c}: L_k(x_j) * exp(i kappa <x_j, c>)
void interp_row(const Grid& g, int m, const double x[3], const double c[3], double kappa, cplx* row) {
  const int p = m + 1;
  double c1[16], c2[16], c3[16];
  cardinals(g.ax[0], x[0], c1);
  cardinals(g.ax[1], x[1], c2);
  cardinals(g.ax[2], x[2], c3);
  cplx f(1.0, 0.0);
  const bool dir = !(c[0] == 0.0 && c[1] == 0.0 && c[2] == 0.0);
  if (dir) {
    const double ph = kappa * dot3(x, c);
    f = cplx(std::cos(ph), std::sin(ph));
  }
  int flat = 0;
  for (int a = 0; a < p; ++a)
    for (int b = 0; b < p; ++b) {
      const double ab = c1[a] * c2[b];
      for (int cc = 0; cc < p; ++cc) {
        const double l = ab * c3[cc];
        // (l + 0i) * (cos + i sin) == (l*cos, l*sin) bitwise
        row[flat++] = dir ? cplx(l * f.real(), l * f.imag()) : cplx(l, 0.0);
      }
    }
}

// interpolation.cpp:89-119 build_transfer_reference: 8 matrices n x n (row-major)
std::vector<double> transfer_ref(int m) {
  const int p = m + 1, n = p * p * p;
  const std::vector<double> par = cheb(0.0, 1.0, m);
  std::vector<double> half[2];
  for (int h = 0; h < 2; ++h) {
    const std::vector<double> ch = cheb(h == 0 ? 0.0 : 0.5, h == 0 ? 0.5 : 1.0, m);
    half[h].resize(p * p);
    for (int j = 0; j < p; ++j)
      for (int k = 0; k < p; ++k) half[h][j * p + k] = lagr(par.data(), p, k, ch[j]);
  }
  std::vector<double> E((size_t)8 * n * n);
  for (int oct = 0; oct < 8; ++oct) {
    const double* bx = half[(oct >> 2) & 1].data();
    const double* by = half[(oct >> 1) & 1].data();
    const double* bz = half[oct & 1].data();
    double* M = &E[(size_t)oct * n * n];
    for (int j = 0; j < n; ++j) {
      const int j3 = j % p, j2 = (j / p) % p, j1 = j / (p * p);
      for (int k = 0; k < n; ++k) {
        const int k3 = k % p, k2 = (k / p) % p, k1 = k / (p * p);
        M[(size_t)j * n + k] = bx[j1 * p + k1] * by[j2 * p + k2] * bz[j3 * p + k3];
      }
    }
  }
  return E;
}

// interpolation.cpp:121-131 build_directional_diag: exp(i kappa <xi_child, c - c_child>)
void dir_diag(const Box& child, const double c[3], const double cc[3], double kappa, int m, cplx* out) {
  const int p = m + 1, n = p * p * p;
  const Grid g(child, m);
  const double dc[3] = {c[0] - cc[0], c[1] - cc[1], c[2] - cc[2]};
  double xi[3];
  for (int j = 0; j < n; ++j) {
    g.node(j, p, xi);
    const double ph = kappa * dot3(xi, dc);
    out[j] = cplx(std::cos(ph), std::sin(ph));
  }
}

// ------------------------------------------------------------ cluster tree
struct Coord {
  int level;
  int64_t i, j, k;
  bool operator<(const Coord& o) const { return std::tie(level, i, j, k) < std::tie(o.level, o.i, o.j, o.k); }
  bool operator==(const Coord& o) const { return level == o.level && i == o.i && j == o.j && k == o.k; }
};
struct Node {
  Coord c;
  int32_t parent = -1;
  int32_t child[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  uint32_t begin = 0, end = 0;
  bool leaf = true;
  uint32_t count() const { return end - begin; }
};

// Restatement of ClusterTree (cluster_tree.hpp:47-101, cluster_tree.cpp:12-151).
struct Tree {
  std::vector<Node> nodes;
  std::vector<std::vector<int32_t>> levels;  // per level, sorted by Coord
  std::vector<int32_t> leaves;               // by (level, coord)
  std::vector<double> px, py, pz;            // slot order
  std::vector<uint32_t> perm;                // slot -> original index
  Box root;                                  // padded
  std::vector<std::array<double, 3>> side;
  std::vector<double> diam;
  int depth = 0, n_max = 0, cap = 30, oversized = 0;

  void build(const double* x, const double* y, const double* z, int64_t n, const double lo[3],
             const double hi[3], int nmax, int depth_cap) {
    if (n <= 0) throw Err(E_ARG, "cluster tree: empty point set");          // cpp:15
    if (nmax < 1) throw Err(E_ARG, "cluster tree: n_max must be >= 1");     // cpp:16
    if (!(lo[0] < hi[0] && lo[1] < hi[1] && lo[2] < hi[2]))
      throw Err(E_ARG, "cluster tree: invalid root box");                   // cpp:17
    n_max = nmax;
    cap = depth_cap;
    for (int a = 0; a < 3; ++a) {  // cpp:21-24 lower-face padding
      root.lo[a] = lo[a] - kRootPad * (hi[a] - lo[a]);
      root.hi[a] = hi[a];
    }
    px.assign(x, x + n);
    py.assign(y, y + n);
    pz.assign(z, z + n);
    for (int64_t s = 0; s < n; ++s) {  // cpp:25-27 containment (half-open)
      const double p[3] = {px[s], py[s], pz[s]};
      for (int a = 0; a < 3; ++a)
        if (!(p[a] > root.lo[a] && p[a] <= root.hi[a])) throw Err(E_ARG, "cluster tree: point outside root box");
    }
    perm.resize(n);
    for (int64_t s = 0; s < n; ++s) perm[s] = (uint32_t)s;
    side.push_back({root.hi[0] - root.lo[0], root.hi[1] - root.lo[1], root.hi[2] - root.lo[2]});
    diam.push_back(norm3(side[0].data()));
    levels.emplace_back();
    Node r;
    r.c = {0, 0, 0, 0};
    r.begin = 0;
    r.end = (uint32_t)n;
    nodes.push_back(r);
    levels[0].push_back(0);
    refine(0);
    for (auto& lv : levels)
      std::sort(lv.begin(), lv.end(), [&](int32_t a, int32_t b) { return nodes[a].c < nodes[b].c; });
    for (int l = 0; l <= depth; ++l)
      for (int32_t id : levels[l])
        if (nodes[id].leaf) leaves.push_back(id);
  }

  // cluster_tree.cpp:57-128 (recursive, stable octant partition)
  void refine(int32_t id) {
    const int level = nodes[id].c.level;
    if (nodes[id].count() <= (uint32_t)n_max) return;
    if (level >= cap) { ++oversized; return; }
    if ((int)side.size() <= level + 1) {
      const auto& s = side[level];
      side.push_back({0.5 * s[0], 0.5 * s[1], 0.5 * s[2]});
      diam.push_back(norm3(side[level + 1].data()));
      levels.emplace_back();
    }
    const Coord c = nodes[id].c;
    const auto cs = side[level + 1];
    // separate multiply and add, no FMA (compiled with -ffp-contract=off)
    const double mid[3] = {root.lo[0] + (double)(2 * c.i + 1) * cs[0], root.lo[1] + (double)(2 * c.j + 1) * cs[1],
                           root.lo[2] + (double)(2 * c.k + 1) * cs[2]};
    const uint32_t b = nodes[id].begin, e = nodes[id].end;
    std::vector<uint8_t> oct(e - b);
    uint32_t cnt[8] = {0};
    for (uint32_t s = b; s < e; ++s) {
      const int o = 4 * (px[s] > mid[0]) + 2 * (py[s] > mid[1]) + (pz[s] > mid[2]);
      oct[s - b] = (uint8_t)o;
      ++cnt[o];
    }
    uint32_t off[8], cur[8], acc = b;
    for (int o = 0; o < 8; ++o) { off[o] = cur[o] = acc; acc += cnt[o]; }
    std::vector<double> tx(e - b), ty(e - b), tz(e - b);
    std::vector<uint32_t> tp(e - b);
    for (uint32_t s = b; s < e; ++s) {
      const uint32_t d = cur[oct[s - b]]++ - b;
      tx[d] = px[s]; ty[d] = py[s]; tz[d] = pz[s]; tp[d] = perm[s];
    }
    std::copy(tx.begin(), tx.end(), px.begin() + b);
    std::copy(ty.begin(), ty.end(), py.begin() + b);
    std::copy(tz.begin(), tz.end(), pz.begin() + b);
    std::copy(tp.begin(), tp.end(), perm.begin() + b);
    nodes[id].leaf = false;
    depth = std::max(depth, level + 1);
    for (int o = 0; o < 8; ++o) {
      if (cnt[o] == 0) continue;
      Node ch;
      ch.c = {level + 1, 2 * c.i + ((o >> 2) & 1), 2 * c.j + ((o >> 1) & 1), 2 * c.k + (o & 1)};
      ch.parent = id;
      ch.begin = off[o];
      ch.end = off[o] + cnt[o];
      const int32_t cid = (int32_t)nodes.size();
      nodes.push_back(ch);
      nodes[id].child[o] = cid;
      levels[level + 1].push_back(cid);
      refine(cid);
    }
  }

  // cluster_tree.cpp:130-139
  Box box(int32_t id) const {
    const Node& n = nodes[id];
    const auto& s = side[n.c.level];
    Box b;
    const int64_t ij[3] = {n.c.i, n.c.j, n.c.k};
    for (int a = 0; a < 3; ++a) {
      b.lo[a] = root.lo[a] + (double)ij[a] * s[a];
      b.hi[a] = root.lo[a] + (double)(ij[a] + 1) * s[a];
    }
    return b;
  }
};

// ------------------------------------------------------------- directions
// PAPER Alg. 3 (:176-201) and Def. 3 (:205-221); conventions SURVEY.md App. B.2:
//  main faces (-x,+x,-y,+y,-z,+z) = 0..5; children of face j are 4j+q, q = 2*qu+qv
//  with (u,v) the in-face axes in increasing order; closed cells + min-j rule ==
//  first argmax axis, then the lower half whenever the coordinate <= mid.
int num_dirs(int level, int lhf) {
  if (level > lhf) return 1;
  return 6 << (2 * (lhf - level));
}
int dir_map_vec(int level, int lhf, const double v[3]) {
  if (level > lhf) return 0;
  int a = 0;
  double M = std::fabs(v[0]);
  for (int i = 1; i < 3; ++i)
    if (std::fabs(v[i]) > M) { M = std::fabs(v[i]); a = i; }
  if (M == 0.0) return 0;  // dir(0) = 0 (Def. 3)
  const int u = (a == 0) ? 1 : 0, w = (a == 2) ? 1 : 2;
  const double cu = v[u] / M, cw = v[w] / M;  // psi_Q(v) in-face coordinates
  int j = 2 * a + (v[a] > 0.0 ? 1 : 0);
  double ulo = -1.0, uhi = 1.0, wlo = -1.0, whi = 1.0;
  for (int d = 0; d < lhf - level; ++d) {
    const double um = 0.5 * (ulo + uhi), wm = 0.5 * (wlo + whi);
    const int qu = cu > um ? 1 : 0, qw = cw > wm ? 1 : 0;
    if (qu) ulo = um; else uhi = um;
    if (qw) wlo = wm; else whi = wm;
    j = 4 * j + 2 * qu + qw;
  }
  return j;
}
// direction vector c_j^(level): normalized midpoint of face cell j (Alg. 3 lines 5-12)
void dir_vec(int level, int lhf, int idx, double out[3]) {
  out[0] = out[1] = out[2] = 0.0;
  if (level > lhf) return;
  const int d = lhf - level;
  const int j0 = idx >> (2 * d);
  const int a = j0 / 2;
  const int u = (a == 0) ? 1 : 0, w = (a == 2) ? 1 : 2;
  double ulo = -1.0, uhi = 1.0, wlo = -1.0, whi = 1.0;
  for (int k = d - 1; k >= 0; --k) {
    const int q = (idx >> (2 * k)) & 3;
    const double um = 0.5 * (ulo + uhi), wm = 0.5 * (wlo + whi);
    if (q >> 1) ulo = um; else uhi = um;
    if (q & 1) wlo = wm; else whi = wm;
  }
  double p[3];
  p[a] = (j0 & 1) ? 1.0 : -1.0;
  p[u] = 0.5 * (ulo + uhi);
  p[w] = 0.5 * (wlo + whi);
  const double nn = norm3(p);  // geometry.hpp:31-35 normalized
  for (int i = 0; i < 3; ++i) out[i] = (1.0 / nn) * p[i];
}
// parent direction c' = dir_(l+1)(c_j^(l)) = j >> 2 by nesting
inline int parent_dir(int level, int lhf, int j) {
  if (level + 1 > lhf) return 0;
  return j >> 2;
}

// ---------------------------------------------------------------- operator
struct Blk { int32_t t, s; int32_t dir; int32_t key; };

struct Op {
  Tree T, S;
  double kappa = 0, eta2 = 0;
  int m = 0, p = 0, n = 0, lhf = -1, zero_diag = 0;
  double rho[3] = {1, 1, 1};
  bool with_coupling = true;
  std::vector<Blk> lplus;                        // sorted by (t, s)
  std::vector<std::pair<int32_t, int32_t>> lminus;  // (t, s) sorted
  std::map<std::tuple<int, int64_t, int64_t, int64_t>, int32_t> keymap;
  std::vector<std::tuple<int, int64_t, int64_t, int64_t>> keys;
  std::vector<int32_t> key_dir;
  std::vector<cplx> coupling;  // keys x n x n
  // ACA-compressed coupling: per key rank k (0 = kept dense),
  // U (n x k, column-major) and W = V^* (k x n, row-major); A ~ U W
  double aca_eps = 0.0;
  std::vector<int32_t> aca_rank;
  std::vector<std::vector<cplx>> aca_u, aca_w;
  std::vector<double> Eref;    // 8 x n x n
  // per-box direction sets: dirs[node] sorted union; kind bitmask 1=D 2=D^
  std::vector<std::vector<int32_t>> dT, dS;
  std::vector<std::vector<uint8_t>> kT, kS;
  std::vector<int64_t> slotT, slotS;  // first slot of node
  int64_t nslotT = 0, nslotS = 0;
  std::vector<int64_t> lp_ptr, lm_ptr;  // CSR by target node
  int64_t M_D = 0, M_D_zero = 0;
  // sampled-structure mode (orc_create_sampled): the block partition is refined
  // only below target boxes that are ancestors of the sampled leaves, and the
  // coupling matrices are generated per block in the M2L instead of stored
  std::vector<char> need_t;  // empty = every target box
  bool onthefly = false;
  // seconds of the last apply: upward pass, coupling generation (sampled mode),
  // M2L products, L2L + L2T + near field; [4] = coupling matrices generated
  double tim[5] = {0, 0, 0, 0, 0};
  double tim_start = 0.0;
};

bool admissible(const Op& op, int32_t t, int32_t s) {
  // Def. 1 (A1), (A3) with inclusive <=
  const int l = op.T.nodes[t].c.level;
  const double q = std::max(op.T.diam[l], op.S.diam[l]);
  const Box bt = op.T.box(t), bs = op.S.box(s);
  double acc = 0.0;  // geometry.hpp:69-76 box_distance
  for (int a = 0; a < 3; ++a) {
    const double gap = std::max(std::max(bt.lo[a] - bs.hi[a], bs.lo[a] - bt.hi[a]), 0.0);
    acc += gap * gap;
  }
  const double dist = std::sqrt(acc);
  return (q <= op.eta2 * dist) && (op.kappa * q * q <= op.eta2 * dist);
}

// PAPER Alg. 2 RefineBlock (:136-148) + Def. 2 classification (:151-159)
void refine_block(Op& op, int32_t t, int32_t s, std::vector<std::pair<int32_t, int32_t>>& adm) {
  const Node& nt = op.T.nodes[t];
  const Node& ns = op.S.nodes[s];
  const bool adm_ts = admissible(op, t, s);
  if (nt.leaf || ns.leaf) {
    if (adm_ts) adm.push_back({t, s});
    else op.lminus.push_back({t, s});
    return;
  }
  if (!adm_ts) {
    for (int a = 0; a < 8; ++a) {
      if (nt.child[a] < 0 || (!op.need_t.empty() && !op.need_t[nt.child[a]])) continue;
      for (int b = 0; b < 8; ++b) {
        if (ns.child[b] < 0) continue;
        refine_block(op, nt.child[a], ns.child[b], adm);
      }
    }
    return;
  }
  adm.push_back({t, s});
}

void build_structure(Op& op) {
  Tree& T = op.T;
  Tree& S = op.S;
  // ell_hf default rule: max{l <= min(pT,pS): kappa*q_l >= 3}
  if (op.lhf == -2) {
    op.lhf = -1;
    for (int l = 0; l <= std::min(T.depth, S.depth); ++l)
      if (op.kappa * std::max(T.diam[l], S.diam[l]) >= 3.0) op.lhf = l;
  }
  // lattice -> direction vector scale: rho_i = side_i / min side
  const double mn = std::min({T.side[0][0], T.side[0][1], T.side[0][2]});
  for (int a = 0; a < 3; ++a) op.rho[a] = T.side[0][a] / mn;

  std::vector<std::pair<int32_t, int32_t>> adm;
  refine_block(op, 0, 0, adm);
  std::sort(adm.begin(), adm.end());
  std::sort(op.lminus.begin(), op.lminus.end());
  op.lplus.resize(adm.size());
  for (size_t b = 0; b < adm.size(); ++b) {
    const Node& nt = T.nodes[adm[b].first];
    const Node& ns = S.nodes[adm[b].second];
    const int l = nt.c.level;
    const int64_t dx = nt.c.i - ns.c.i, dy = nt.c.j - ns.c.j, dz = nt.c.k - ns.c.k;
    auto key = std::make_tuple(l, dx, dy, dz);
    auto it = op.keymap.find(key);
    int32_t kid;
    if (it == op.keymap.end()) {
      kid = (int32_t)op.keys.size();
      op.keymap.emplace(key, kid);
      op.keys.push_back(key);
      const double v[3] = {dx * op.rho[0], dy * op.rho[1], dz * op.rho[2]};
      op.key_dir.push_back(dir_map_vec(l, op.lhf, v));
    } else {
      kid = it->second;
    }
    op.lplus[b] = {adm[b].first, adm[b].second, op.key_dir[kid], kid};
  }
  // near-field entry count M_D
  op.M_D = 0;
  op.M_D_zero = 0;
  for (auto& b : op.lminus) op.M_D += (int64_t)T.nodes[b.first].count() * S.nodes[b.second].count();

  // Def. 4: D(t) from admissible partners, D^(t) from the parent's D u D^.
  auto sets = [&](Tree& tr, bool is_target, std::vector<std::vector<int32_t>>& dirs,
                  std::vector<std::vector<uint8_t>>& kind) {
    std::vector<std::vector<int32_t>> D(tr.nodes.size()), H(tr.nodes.size());
    for (auto& b : op.lplus) D[is_target ? b.t : b.s].push_back(b.dir);
    for (auto& d : D) { std::sort(d.begin(), d.end()); d.erase(std::unique(d.begin(), d.end()), d.end()); }
    // pre-order by level: parents first
    for (int l = 1; l <= tr.depth; ++l)
      for (int32_t id : tr.levels[l]) {
        const int32_t par = tr.nodes[id].parent;
        std::vector<int32_t> h;
        for (int32_t c : D[par]) h.push_back(parent_dir(l - 1, op.lhf, c));
        for (int32_t c : H[par]) h.push_back(parent_dir(l - 1, op.lhf, c));
        std::sort(h.begin(), h.end());
        h.erase(std::unique(h.begin(), h.end()), h.end());
        H[id] = h;
      }
    dirs.assign(tr.nodes.size(), {});
    kind.assign(tr.nodes.size(), {});
    for (size_t id = 0; id < tr.nodes.size(); ++id) {
      std::vector<int32_t> u = D[id];
      u.insert(u.end(), H[id].begin(), H[id].end());
      std::sort(u.begin(), u.end());
      u.erase(std::unique(u.begin(), u.end()), u.end());
      dirs[id] = u;
      for (int32_t c : u) {
        uint8_t k = 0;
        if (std::binary_search(D[id].begin(), D[id].end(), c)) k |= 1;
        if (std::binary_search(H[id].begin(), H[id].end(), c)) k |= 2;
        kind[id].push_back(k);
      }
    }
  };
  sets(T, true, op.dT, op.kT);
  sets(S, false, op.dS, op.kS);
  auto slots = [](const std::vector<std::vector<int32_t>>& d, std::vector<int64_t>& first, int64_t& tot) {
    first.resize(d.size());
    tot = 0;
    for (size_t i = 0; i < d.size(); ++i) { first[i] = tot; tot += (int64_t)d[i].size(); }
  };
  slots(op.dT, op.slotT, op.nslotT);
  slots(op.dS, op.slotS, op.nslotS);
  // CSR of L+ / L- by target node
  op.lp_ptr.assign(T.nodes.size() + 1, 0);
  for (auto& b : op.lplus) op.lp_ptr[b.t + 1]++;
  for (size_t i = 0; i < T.nodes.size(); ++i) op.lp_ptr[i + 1] += op.lp_ptr[i];
  {
    std::vector<Blk> tmp(op.lplus.size());
    std::vector<int64_t> cur(op.lp_ptr.begin(), op.lp_ptr.end() - 1);
    for (auto& b : op.lplus) tmp[cur[b.t]++] = b;
    op.lplus.swap(tmp);
  }
  op.lm_ptr.assign(T.nodes.size() + 1, 0);
  for (auto& b : op.lminus) op.lm_ptr[b.first + 1]++;
  for (size_t i = 0; i < T.nodes.size(); ++i) op.lm_ptr[i + 1] += op.lm_ptr[i];
  {
    std::vector<std::pair<int32_t, int32_t>> tmp(op.lminus.size());
    std::vector<int64_t> cur(op.lm_ptr.begin(), op.lm_ptr.end() - 1);
    for (auto& b : op.lminus) tmp[cur[b.first]++] = b;
    op.lminus.swap(tmp);
  }
}

// Canonical coupling matrix (App. B.3): s at the lattice origin,
// t at lattice offset (dx,dy,dz); A[j,k] = f_c(xi_t,j, xi_s,k).
void coupling_matrix(int m, double kappa, const double side[3], int64_t dx, int64_t dy, int64_t dz,
                     const double c[3], cplx* A) {
  const int p = m + 1, n = p * p * p;
  Box bs, bt;
  const int64_t d[3] = {dx, dy, dz};
  for (int a = 0; a < 3; ++a) {
    bs.lo[a] = 0.0;
    bs.hi[a] = 1.0 * side[a];
    bt.lo[a] = (double)d[a] * side[a];
    bt.hi[a] = (double)(d[a] + 1) * side[a];
  }
  const Grid gt(bt, m), gs(bs, m);
  double xt[3], xs[3], dd[3];
  for (int j = 0; j < n; ++j) {
    gt.node(j, p, xt);
    for (int k = 0; k < n; ++k) {
      gs.node(k, p, xs);
      for (int a = 0; a < 3; ++a) dd[a] = xt[a] - xs[a];
      A[(size_t)j * n + k] = kernel_dir_diff(dd, c, kappa);
    }
  }
}

void build_coupling(Op& op) {
  op.Eref = transfer_ref(op.m);
  const int n = op.n;
  const size_t nk = op.keys.size();
  op.coupling.assign(nk * (size_t)n * n, cplx(0, 0));
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t k = 0; k < (int64_t)nk; ++k) {
    const auto& key = op.keys[k];
    const int l = std::get<0>(key);
    double c[3];
    dir_vec(l, op.lhf, op.key_dir[k], c);
    coupling_matrix(op.m, op.kappa, op.T.side[l].data(), std::get<1>(key), std::get<2>(key), std::get<3>(key),
                    c, &op.coupling[(size_t)k * n * n]);
  }
}

// SPEC.md:440-448 aca_compress, with the pinned design decisions:
// partially pivoted ACA on the n x n row-major matrix A: start from row 0; the
// column pivot is the max-modulus entry of the residual row (lowest index on
// ties), the next row pivot the max-modulus entry of the residual column among
// the rows not used yet; stop when |u_k| |w_k| <= eps |S_k|_F with the standard
// incremental Frobenius estimate of the accumulated approximation S_k, or at
// max_rank.  Returns the rank k and A ~ U W (U n x k column-major, W = V^* k x n
// row-major), or 0 (keep dense) when 2 k n >= n^2 (no gain).  A zero residual row
// (exact low rank) ends the iteration.
int aca_compress(const cplx* A, int n, double eps, int max_rank, std::vector<cplx>& U, std::vector<cplx>& W) {
  U.clear();
  W.clear();
  std::vector<char> used(n, 0);
  std::vector<cplx> row(n), col(n);
  double s2 = 0.0;  // |S_k|_F^2 estimate
  int ip = 0, k = 0;
  const int kmax = std::min(max_rank, n);
  while (k < kmax) {
    used[ip] = 1;
    for (int c = 0; c < n; ++c) {  // residual row ip
      cplx v = A[(size_t)ip * n + c];
      for (int q = 0; q < k; ++q) v -= U[(size_t)q * n + ip] * W[(size_t)q * n + c];
      row[c] = v;
    }
    int jp = 0;
    double best = -1.0;
    for (int c = 0; c < n; ++c)
      if (std::abs(row[c]) > best) {
        best = std::abs(row[c]);
        jp = c;
      }
    if (best == 0.0) break;  // residual row vanishes: exact rank k
    const cplx delta = row[jp];
    for (int i = 0; i < n; ++i) {  // residual column jp
      cplx v = A[(size_t)i * n + jp];
      for (int q = 0; q < k; ++q) v -= U[(size_t)q * n + i] * W[(size_t)q * n + jp];
      col[i] = v;
    }
    // new cross u w with u = residual column, w = residual row / pivot
    double nu = 0.0, nw = 0.0;
    for (int i = 0; i < n; ++i) nu += std::norm(col[i]);
    std::vector<cplx> w(n);
    for (int c = 0; c < n; ++c) {
      w[c] = row[c] / delta;
      nw += std::norm(w[c]);
    }
    double cross = 0.0;  // 2 Re sum_q <u_q w_q, u w>_F = 2 Re sum_q (u_q^H u)(w_q^H w)
    for (int q = 0; q < k; ++q) {
      cplx a(0, 0), b(0, 0);
      for (int i = 0; i < n; ++i) a += std::conj(U[(size_t)q * n + i]) * col[i];
      for (int c = 0; c < n; ++c) b += std::conj(W[(size_t)q * n + c]) * w[c];
      cross += 2.0 * (a * b).real();
    }
    if (k > 0 && std::sqrt(nu * nw) <= 1e-14 * std::sqrt(std::max(s2, 0.0))) break;  // round-off cross: exact rank k
    U.insert(U.end(), col.begin(), col.end());
    W.insert(W.end(), w.begin(), w.end());
    ++k;
    s2 += cross + nu * nw;
    if (std::sqrt(nu * nw) <= eps * std::sqrt(std::max(s2, 0.0))) break;
    int inext = -1;
    best = -1.0;
    for (int i = 0; i < n; ++i)
      if (!used[i] && std::abs(col[i]) > best) {
        best = std::abs(col[i]);
        inext = i;
      }
    if (inext < 0) break;
    ip = inext;
  }
  if (2 * (int64_t)k * n >= (int64_t)n * n) {  // no gain: keep dense
    U.clear();
    W.clear();
    return 0;
  }
  return k;
}

void build_aca(Op& op) {
  const int n = op.n;
  const size_t nk = op.keys.size();
  op.aca_rank.assign(nk, 0);
  op.aca_u.assign(nk, {});
  op.aca_w.assign(nk, {});
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t k = 0; k < (int64_t)nk; ++k)
    op.aca_rank[k] = aca_compress(&op.coupling[(size_t)k * n * n], n, op.aca_eps, n, op.aca_u[k], op.aca_w[k]);
}

int32_t find_dir(const std::vector<int32_t>& d, int32_t c) {
  auto it = std::lower_bound(d.begin(), d.end(), c);
  if (it == d.end() || *it != c) return -1;
  return (int32_t)(it - d.begin());
}

// Alg. 4.  leaf_mask selects sampled target leaves (nullptr = all).
void apply(Op& op, const double* xin, double* yout, const std::vector<char>* leaf_mask) {
  const Tree& T = op.T;
  const Tree& S = op.S;
  const int n = op.n, m = op.m;
  const double kappa = op.kappa;
  op.tim_start = omp_get_wtime();
  const int64_t NS = (int64_t)S.perm.size();
  std::vector<cplx> v(NS);  // charges in source slot order
  for (int64_t s = 0; s < NS; ++s) v[s] = cplx(xin[2 * (int64_t)S.perm[s]], xin[2 * (int64_t)S.perm[s] + 1]);
  std::vector<cplx> mom((size_t)op.nslotS * n, cplx(0, 0)), loc((size_t)op.nslotT * n, cplx(0, 0));
  const double zero3[3] = {0, 0, 0};

  // (i) S2M: v~_{s,c} = L*_{s,c} v|s
  const int64_t nleafS = (int64_t)S.leaves.size();
#pragma omp parallel
  {
    std::vector<cplx> row(n);
#pragma omp for schedule(dynamic, 8)
    for (int64_t li = 0; li < nleafS; ++li) {
      const int32_t s = S.leaves[li];
      const auto& dirs = op.dS[s];
      if (dirs.empty()) continue;
      const int l = S.nodes[s].c.level;
      const Grid g(S.box(s), m);
      for (size_t di = 0; di < dirs.size(); ++di) {
        double c[3];
        dir_vec(l, op.lhf, dirs[di], c);
        cplx* out = &mom[(size_t)(op.slotS[s] + di) * n];
        for (uint32_t j = S.nodes[s].begin; j < S.nodes[s].end; ++j) {
          const double y[3] = {S.px[j], S.py[j], S.pz[j]};
          interp_row(g, m, y, c, kappa, row.data());
          for (int k = 0; k < n; ++k) out[k] += std::conj(row[k]) * v[j];
        }
      }
    }
  }
  // (ii) M2M, levels p(T_S)-1 .. 0: v~_{s,c} += E*_{s',c} v~_{s',c'}
  for (int l = S.depth - 1; l >= 0; --l) {
    const auto& lv = S.levels[l];
#pragma omp parallel
    {
      std::vector<cplx> dg(n), tmp(n);
#pragma omp for schedule(dynamic, 4)
      for (int64_t bi = 0; bi < (int64_t)lv.size(); ++bi) {
        const int32_t s = lv[bi];
        const Node& ns = S.nodes[s];
        if (ns.leaf) continue;
        const auto& dirs = op.dS[s];
        for (size_t di = 0; di < dirs.size(); ++di) {
          double c[3], cc[3];
          dir_vec(l, op.lhf, dirs[di], c);
          const int cp = parent_dir(l, op.lhf, dirs[di]);
          dir_vec(l + 1, op.lhf, cp, cc);
          cplx* out = &mom[(size_t)(op.slotS[s] + di) * n];
          for (int o = 0; o < 8; ++o) {
            const int32_t ch = ns.child[o];
            if (ch < 0) continue;
            const int32_t cdi = find_dir(op.dS[ch], cp);
            if (cdi < 0) throw Err(E_ARG, "internal: missing child moment");
            const cplx* in = &mom[(size_t)(op.slotS[ch] + cdi) * n];
            dir_diag(S.box(ch), c, cc, kappa, m, dg.data());
            for (int j = 0; j < n; ++j) tmp[j] = std::conj(dg[j]) * in[j];
            const double* E = &op.Eref[(size_t)o * n * n];
            for (int j = 0; j < n; ++j) {
              const cplx tj = tmp[j];
              const double* Ej = E + (size_t)j * n;
              for (int k = 0; k < n; ++k) out[k] += Ej[k] * tj;
            }
          }
        }
      }
    }
  }
  // target boxes needed (sampled mode: sampled leaves and their ancestors)
  std::vector<char> need(T.nodes.size(), 1);
  if (leaf_mask) {
    std::fill(need.begin(), need.end(), 0);
    for (size_t li = 0; li < T.leaves.size(); ++li)
      if ((*leaf_mask)[li])
        for (int32_t id = T.leaves[li]; id >= 0; id = T.nodes[id].parent) need[id] = 1;
  }
  // (iii) M2L: g~_{t,c} += A_{c,t x s} v~_{s,c}; owner computes over t
  const int64_t nT = (int64_t)T.nodes.size();
  const double tm0 = omp_get_wtime();
  op.tim[0] = tm0 - op.tim_start;
  if (op.onthefly) {
    // sampled-structure mode: coupling matrices are generated per key, once per
    // apply for all sampled blocks that use the key (key-major, as a CPU code
    // without room for the 228 GB coupling set of config 4 would run), the
    // products of each block kept and summed per target in block order (the
    // same order as the target-major loop below: deterministic)
    std::vector<std::pair<int32_t, int64_t>> kb;  // (key, block)
    for (int64_t t = 0; t < nT; ++t)
      if (need[t])
        for (int64_t b = op.lp_ptr[t]; b < op.lp_ptr[t + 1]; ++b) kb.push_back({op.lplus[b].key, b});
    std::sort(kb.begin(), kb.end());
    std::vector<int64_t> kstart;
    for (size_t i = 0; i < kb.size(); ++i)
      if (i == 0 || kb[i].first != kb[i - 1].first) kstart.push_back((int64_t)i);
    kstart.push_back((int64_t)kb.size());
    std::unordered_map<int64_t, int64_t> slot_of_block;  // block -> row of prod
    slot_of_block.reserve(kb.size() * 2);
    for (size_t i = 0; i < kb.size(); ++i) slot_of_block[kb[i].second] = (int64_t)i;
    std::vector<cplx> prod(kb.size() * (size_t)n);
    double gen_s = 0.0, mv_s = 0.0;
#pragma omp parallel reduction(+ : gen_s, mv_s)
    {
      std::vector<cplx> A((size_t)n * n);
#pragma omp for schedule(dynamic, 1)
      for (int64_t k = 0; k < (int64_t)kstart.size() - 1; ++k) {
        const double g0 = omp_get_wtime();
        const int32_t key = kb[kstart[k]].first;
        const auto& kk = op.keys[key];
        const int kl = std::get<0>(kk);
        double c[3];
        dir_vec(kl, op.lhf, op.key_dir[key], c);
        coupling_matrix(op.m, op.kappa, op.T.side[kl].data(), std::get<1>(kk), std::get<2>(kk), std::get<3>(kk), c,
                        A.data());
        const double g1 = omp_get_wtime();
        for (int64_t i = kstart[k]; i < kstart[k + 1]; ++i) {
          const Blk& bk = op.lplus[kb[i].second];
          const int32_t sdi = find_dir(op.dS[bk.s], bk.dir);
          const cplx* in = &mom[(size_t)(op.slotS[bk.s] + sdi) * n];
          cplx* out = &prod[(size_t)i * n];
          for (int j = 0; j < n; ++j) {
            cplx acc(0, 0);
            const cplx* Aj = &A[(size_t)j * n];
            for (int q = 0; q < n; ++q) acc += Aj[q] * in[q];
            out[j] = acc;
          }
        }
        gen_s += g1 - g0;
        mv_s += omp_get_wtime() - g1;
      }
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t t = 0; t < nT; ++t) {
      if (!need[t]) continue;
      for (int64_t b = op.lp_ptr[t]; b < op.lp_ptr[t + 1]; ++b) {
        const Blk& bk = op.lplus[b];
        const int32_t tdi = find_dir(op.dT[t], bk.dir);
        cplx* out = &loc[(size_t)(op.slotT[t] + tdi) * n];
        const cplx* pr = &prod[(size_t)slot_of_block[b] * n];
        for (int j = 0; j < n; ++j) out[j] += pr[j];
      }
    }
    const double wall = omp_get_wtime() - tm0;
    op.tim[1] = (gen_s + mv_s) > 0 ? wall * gen_s / (gen_s + mv_s) : 0.0;  // coupling generation share
    op.tim[2] = wall - op.tim[1];
    op.tim[4] = (double)(kstart.size() - 1);
  } else {
#pragma omp parallel
  {
  std::vector<cplx> Abuf(op.onthefly ? (size_t)n * n : 0);
  int32_t Akey = -1;
#pragma omp for schedule(dynamic, 4)
  for (int64_t t = 0; t < nT; ++t) {
    if (!need[t]) continue;
    for (int64_t b = op.lp_ptr[t]; b < op.lp_ptr[t + 1]; ++b) {
      const Blk& bk = op.lplus[b];
      const int32_t tdi = find_dir(op.dT[t], bk.dir), sdi = find_dir(op.dS[bk.s], bk.dir);
      cplx* out = &loc[(size_t)(op.slotT[t] + tdi) * n];
      const cplx* in = &mom[(size_t)(op.slotS[bk.s] + sdi) * n];
      const cplx* A;
      if (op.onthefly) {  // the same deterministic coupling_matrix as build_coupling
        if (bk.key != Akey) {
          const auto& key = op.keys[bk.key];
          const int kl = std::get<0>(key);
          double c[3];
          dir_vec(kl, op.lhf, op.key_dir[bk.key], c);
          coupling_matrix(op.m, op.kappa, op.T.side[kl].data(), std::get<1>(key), std::get<2>(key),
                          std::get<3>(key), c, Abuf.data());
          Akey = bk.key;
        }
        A = Abuf.data();
      } else {
        A = &op.coupling[(size_t)bk.key * n * n];
      }
      if (op.aca_eps > 0.0 && op.aca_rank[bk.key] > 0) {  // A ~ U W: out += U (W in)
        const int rk = op.aca_rank[bk.key];
        const cplx* Uk = op.aca_u[bk.key].data();
        const cplx* Wk = op.aca_w[bk.key].data();
        cplx z[512];
        for (int q = 0; q < rk; ++q) {
          cplx acc(0, 0);
          for (int k = 0; k < n; ++k) acc += Wk[(size_t)q * n + k] * in[k];
          z[q] = acc;
        }
        for (int j = 0; j < n; ++j) {
          cplx acc(0, 0);
          for (int q = 0; q < rk; ++q) acc += Uk[(size_t)q * n + j] * z[q];
          out[j] += acc;
        }
        continue;
      }
      for (int j = 0; j < n; ++j) {
        cplx acc(0, 0);
        const cplx* Aj = A + (size_t)j * n;
        for (int k = 0; k < n; ++k) acc += Aj[k] * in[k];
        out[j] += acc;
      }
    }
  }
  }
    op.tim[1] = 0.0;
    op.tim[2] = omp_get_wtime() - tm0;
    op.tim[4] = 0.0;
  }
  const double tm1 = omp_get_wtime();
  // (iv) L2L, levels 0 .. p(T_T)-1: g~_{t',c'} += E_{t',c} g~_{t,c}
  for (int l = 0; l < T.depth; ++l) {
    const auto& lv = T.levels[l];
#pragma omp parallel
    {
      std::vector<cplx> dg(n), tmp(n);
#pragma omp for schedule(dynamic, 4)
      for (int64_t bi = 0; bi < (int64_t)lv.size(); ++bi) {
        const int32_t t = lv[bi];
        const Node& nt = T.nodes[t];
        if (nt.leaf || !need[t]) continue;
        const auto& dirs = op.dT[t];
        for (size_t di = 0; di < dirs.size(); ++di) {
          double c[3], cc[3];
          dir_vec(l, op.lhf, dirs[di], c);
          const int cp = parent_dir(l, op.lhf, dirs[di]);
          dir_vec(l + 1, op.lhf, cp, cc);
          const cplx* in = &loc[(size_t)(op.slotT[t] + di) * n];
          for (int o = 0; o < 8; ++o) {
            const int32_t ch = nt.child[o];
            if (ch < 0 || !need[ch]) continue;
            const int32_t cdi = find_dir(op.dT[ch], cp);
            if (cdi < 0) throw Err(E_ARG, "internal: missing child local");
            cplx* out = &loc[(size_t)(op.slotT[ch] + cdi) * n];
            dir_diag(T.box(ch), c, cc, kappa, m, dg.data());
            const double* E = &op.Eref[(size_t)o * n * n];
            for (int j = 0; j < n; ++j) {
              cplx acc(0, 0);
              const double* Ej = E + (size_t)j * n;
              for (int k = 0; k < n; ++k) acc += Ej[k] * in[k];
              out[j] += dg[j] * acc;
            }
          }
        }
      }
    }
  }
  // (v) L2T + (vi) near field, per target leaf
  const int64_t nleafT = (int64_t)T.leaves.size();
  int64_t zero_skips = 0;
  int singular = 0;
#pragma omp parallel reduction(+ : zero_skips) reduction(| : singular)
  {
    std::vector<cplx> row(n);
#pragma omp for schedule(dynamic, 8)
    for (int64_t li = 0; li < nleafT; ++li) {
      if (leaf_mask && !(*leaf_mask)[li]) continue;
      const int32_t t = T.leaves[li];
      const Node& nt = T.nodes[t];
      const int l = nt.c.level;
      std::vector<cplx> g(nt.count(), cplx(0, 0));
      const auto& dirs = op.dT[t];
      if (!dirs.empty()) {
        const Grid gr(T.box(t), m);
        for (size_t di = 0; di < dirs.size(); ++di) {
          double c[3];
          dir_vec(l, op.lhf, dirs[di], c);
          const cplx* gl = &loc[(size_t)(op.slotT[t] + di) * n];
          for (uint32_t j = nt.begin; j < nt.end; ++j) {
            const double x[3] = {T.px[j], T.py[j], T.pz[j]};
            interp_row(gr, m, x, c, kappa, row.data());
            cplx acc(0, 0);
            for (int k = 0; k < n; ++k) acc += row[k] * gl[k];
            g[j - nt.begin] += acc;
          }
        }
      }
      // L- blocks whose target is t or an ancestor of t (an inadmissible leaf
      // block (t', s) with s a source leaf can have a non-leaf target t').
      std::vector<int32_t> chain;
      for (int32_t id = t; id >= 0; id = T.nodes[id].parent) chain.push_back(id);
      for (auto it = chain.rbegin(); it != chain.rend(); ++it)
      for (int64_t b = op.lm_ptr[*it]; b < op.lm_ptr[*it + 1]; ++b) {
        const int32_t s = op.lminus[b].second;
        const Node& ns = S.nodes[s];
        for (uint32_t j = nt.begin; j < nt.end; ++j) {
          cplx acc(0, 0);
          for (uint32_t k = ns.begin; k < ns.end; ++k) {
            if (op.zero_diag && T.perm[j] == S.perm[k]) { ++zero_skips; continue; }
            const double d[3] = {T.px[j] - S.px[k], T.py[j] - S.py[k], T.pz[j] - S.pz[k]};
            const double r2 = dot3(d, d);
            if (r2 == 0.0) { singular = 1; continue; }
            acc += kernel_diff(d, kappa) * v[k];
          }
          g[j - nt.begin] += acc;
        }
      }
      for (uint32_t j = nt.begin; j < nt.end; ++j) {
        const int64_t o = T.perm[j];
        yout[2 * o] = g[j - nt.begin].real();
        yout[2 * o + 1] = g[j - nt.begin].imag();
      }
    }
  }
  op.M_D_zero = zero_skips;
  op.tim[3] = omp_get_wtime() - tm1;
  (void)zero3;
  if (singular) throw Err(E_DOMAIN, "Helmholtz kernel is singular at x == y (near field)");
}

// ------------------------------------------------ streaming structure digest
// Order-independent 64-bit digests of the canonical structure (the same row
// layouts as the orc_export_* functions; digest = sum over rows of a splitmix64
// row hash mod 2^64), computed WITHOUT storing the block lists: PAPER Alg. 2
// (RefineBlock, :136-148) is run depth-first from a frontier of block pairs in
// parallel, every L+ / L- block is hashed where it is classified, and D(t) is
// accumulated in per-node direction marks.  Used to pin the structure of the
// configurations whose L+ does not fit in host memory (config 4: 3.47e9 blocks).
inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline uint64_t row_hash(const int64_t* v, int n) {
  uint64_t h = 0x12345678ull;
  for (int i = 0; i < n; ++i) h = mix64(h ^ (uint64_t)v[i]);
  return h;
}

struct DigestAcc {
  uint64_t lp = 0, lm = 0;
  int64_t n_c = 0, n_lm = 0, m_d = 0;
};

struct DigestCtx {
  Op* op;
  std::vector<int64_t> doffT, doffS;                 // first mark of node id
  std::vector<uint8_t> markT, markS;                 // D marks (bit 0), D^ (bit 1)
  std::vector<std::vector<uint64_t>> keybits;        // per level, dense key bitmap (levels <= 8)
  std::vector<int64_t> kext;                         // per level: offsets in (-kext, kext)
};

inline int key_dir_of(const Op& op, int l, int64_t dx, int64_t dy, int64_t dz) {
  const double v[3] = {dx * op.rho[0], dy * op.rho[1], dz * op.rho[2]};
  return dir_map_vec(l, op.lhf, v);
}

void digest_block(DigestCtx& X, DigestAcc& A, int32_t t, int32_t s, std::vector<std::array<int64_t, 4>>& deep) {
  Op& op = *X.op;
  const Node& nt = op.T.nodes[t];
  const Node& ns = op.S.nodes[s];
  const bool adm = admissible(op, t, s);
  const int l = nt.c.level;
  if (nt.leaf || ns.leaf || adm) {
    if (adm) {
      const int64_t dx = nt.c.i - ns.c.i, dy = nt.c.j - ns.c.j, dz = nt.c.k - ns.c.k;
      const int dir = key_dir_of(op, l, dx, dy, dz);
      const int64_t r[8] = {l, nt.c.i, nt.c.j, nt.c.k, ns.c.i, ns.c.j, ns.c.k, dir};
      A.lp += row_hash(r, 8);
      ++A.n_c;
      __atomic_fetch_or(&X.markT[X.doffT[t] + dir], (uint8_t)1, __ATOMIC_RELAXED);
      __atomic_fetch_or(&X.markS[X.doffS[s] + dir], (uint8_t)1, __ATOMIC_RELAXED);
      if (l < (int)X.keybits.size()) {
        const int64_t e = X.kext[l], w = 2 * e + 1;
        const uint64_t bit = (uint64_t)(((dx + e) * w + (dy + e)) * w + (dz + e));
        __atomic_fetch_or(&X.keybits[l][bit >> 6], 1ull << (bit & 63), __ATOMIC_RELAXED);
      } else {
        deep.push_back({l, dx, dy, dz});
      }
    } else {
      const int64_t r[8] = {l, nt.c.i, nt.c.j, nt.c.k, l, ns.c.i, ns.c.j, ns.c.k};
      A.lm += row_hash(r, 8);
      ++A.n_lm;
      A.m_d += (int64_t)nt.count() * ns.count();
    }
    return;
  }
  for (int a = 0; a < 8; ++a) {
    if (nt.child[a] < 0) continue;
    for (int b = 0; b < 8; ++b)
      if (ns.child[b] >= 0) digest_block(X, A, nt.child[a], ns.child[b], deep);
  }
}

void structure_digest_stream(Op& op, uint64_t out[6], int64_t* cnt) {
  Tree& T = op.T;
  Tree& S = op.S;
  if (op.lhf == -2) {  // same rule as build_structure
    op.lhf = -1;
    for (int l = 0; l <= std::min(T.depth, S.depth); ++l)
      if (op.kappa * std::max(T.diam[l], S.diam[l]) >= 3.0) op.lhf = l;
  }
  const double mn = std::min({T.side[0][0], T.side[0][1], T.side[0][2]});
  for (int a = 0; a < 3; ++a) op.rho[a] = T.side[0][a] / mn;
  DigestCtx X;
  X.op = &op;
  auto offs = [&](const Tree& tr, std::vector<int64_t>& off, std::vector<uint8_t>& mark) {
    off.resize(tr.nodes.size() + 1);
    int64_t acc = 0;
    for (size_t id = 0; id < tr.nodes.size(); ++id) {
      off[id] = acc;
      acc += num_dirs(tr.nodes[id].c.level, op.lhf);
    }
    off[tr.nodes.size()] = acc;
    mark.assign(acc, 0);
  };
  offs(T, X.doffT, X.markT);
  offs(S, X.doffS, X.markS);
  const int maxl = std::min(T.depth, S.depth);
  for (int l = 0; l <= std::min(maxl, 8); ++l) {
    const int64_t e = (int64_t)1 << l, w = 2 * e + 1;
    X.kext.push_back(e);
    X.keybits.emplace_back((size_t)((w * w * w + 63) / 64), 0ull);
  }
  // frontier: breadth-first until there are enough independent pairs
  std::vector<std::pair<int32_t, int32_t>> front{{0, 0}};
  DigestAcc A0;
  std::vector<std::array<int64_t, 4>> deep0;
  for (int it = 0; it < 4 && front.size() < 4096; ++it) {
    std::vector<std::pair<int32_t, int32_t>> nxt;
    for (auto [t, s] : front) {
      const Node& nt = T.nodes[t];
      const Node& ns = S.nodes[s];
      if (nt.leaf || ns.leaf || admissible(op, t, s)) {
        digest_block(X, A0, t, s, deep0);  // classified here
        continue;
      }
      for (int a = 0; a < 8; ++a) {
        if (nt.child[a] < 0) continue;
        for (int b = 0; b < 8; ++b)
          if (ns.child[b] >= 0) nxt.push_back({nt.child[a], ns.child[b]});
      }
    }
    front.swap(nxt);
  }
  uint64_t lp = A0.lp, lm = A0.lm;
  int64_t n_c = A0.n_c, n_lm = A0.n_lm, m_d = A0.m_d;
  std::vector<std::array<int64_t, 4>> deep = deep0;
#pragma omp parallel
  {
    DigestAcc A;
    std::vector<std::array<int64_t, 4>> dp;
#pragma omp for schedule(dynamic, 1)
    for (int64_t i = 0; i < (int64_t)front.size(); ++i) digest_block(X, A, front[i].first, front[i].second, dp);
#pragma omp critical
    {
      lp += A.lp;
      lm += A.lm;
      n_c += A.n_c;
      n_lm += A.n_lm;
      m_d += A.m_d;
      deep.insert(deep.end(), dp.begin(), dp.end());
    }
  }
  // N_SC: distinct (level, offset) keys
  int64_t n_sc = 0;
  for (auto& kb : X.keybits)
    for (uint64_t w : kb) n_sc += __builtin_popcountll(w);
  std::sort(deep.begin(), deep.end());
  n_sc += (int64_t)(std::unique(deep.begin(), deep.end()) - deep.begin());
  // D^ (Def. 4): parent's D u D^ mapped to the child level, pre-order by level
  auto hat = [&](Tree& tr, const std::vector<int64_t>& off, std::vector<uint8_t>& mark) {
    for (int l = 1; l <= tr.depth; ++l)
      for (int32_t id : tr.levels[l]) {
        const int32_t par = tr.nodes[id].parent;
        const int npd = num_dirs(l - 1, op.lhf);
        for (int c = 0; c < npd; ++c)
          if (mark[off[par] + c]) mark[off[id] + parent_dir(l - 1, op.lhf, c)] |= 2;
      }
  };
  hat(T, X.doffT, X.markT);
  hat(S, X.doffS, X.markS);
  int64_t slots[2] = {0, 0};
  for (int w = 0; w < 2; ++w) {
    const Tree& tr = w == 0 ? T : S;
    const auto& off = w == 0 ? X.doffT : X.doffS;
    const auto& mark = w == 0 ? X.markT : X.markS;
    uint64_t acc = 0, dacc = 0;
    for (size_t id = 0; id < tr.nodes.size(); ++id) {
      const Node& nd = tr.nodes[id];
      const int64_t r[7] = {nd.c.level, nd.c.i, nd.c.j, nd.c.k, nd.begin, nd.end, nd.leaf ? 1 : 0};
      acc += row_hash(r, 7);
      for (int64_t c = 0; c < off[id + 1] - off[id]; ++c) {
        const uint8_t k = mark[off[id] + c];
        if (!k) continue;
        const int64_t rr[6] = {nd.c.level, nd.c.i, nd.c.j, nd.c.k, c, k};
        dacc += row_hash(rr, 6);
        ++slots[w];
      }
    }
    for (size_t sl = 0; sl < tr.perm.size(); ++sl) {
      const int64_t r[2] = {(int64_t)sl, (int64_t)tr.perm[sl]};
      acc += row_hash(r, 2);
    }
    out[w] = acc;
    out[4 + w] = dacc;
  }
  out[2] = lp;
  out[3] = lm;
  if (cnt) {
    cnt[0] = n_c;
    cnt[1] = n_sc;
    cnt[2] = n_lm;
    cnt[3] = m_d;
    cnt[4] = (int64_t)T.nodes.size();
    cnt[5] = (int64_t)S.nodes.size();
    cnt[6] = slots[0];
    cnt[7] = slots[1];
    cnt[8] = T.depth;
    cnt[9] = S.depth;
    cnt[10] = op.lhf;
  }
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Err& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return E_ARG;
  }
}

}  // namespace

struct orc_op {
  Op op;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}

static int create_impl(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                       const double* sy, const double* sz, int64_t ns, const double lo[3], const double hi[3],
                       double kappa, int n_max, int m, double eta2, int l_hf, int depth_cap, int zero_diagonal,
                       bool coupling, orc_op** out, const int64_t* sample = nullptr, int64_t nsample = 0) {
  *out = nullptr;
  return guard([&] {
    if (!(kappa > 0.0) || !std::isfinite(kappa)) throw Err(E_ARG, "wave number must be positive and finite");
    if (m < 0 || m > 12) throw Err(E_ARG, "interpolation degree out of range");
    if (!(eta2 > 0.0)) throw Err(E_ARG, "eta2 must be positive");
    if (l_hf < -2) throw Err(E_ARG, "l_hf must be >= -1 (or -2 for the default rule)");
    auto* o = new orc_op;
    try {
      Op& op = o->op;
      op.kappa = kappa;
      op.eta2 = eta2;
      op.m = m;
      op.p = m + 1;
      op.n = op.p * op.p * op.p;
      op.lhf = l_hf;
      op.zero_diag = zero_diagonal;
      op.T.build(tx, ty, tz, nt, lo, hi, n_max, depth_cap);
      op.S.build(sx, sy, sz, ns, lo, hi, n_max, depth_cap);
      if (sample) {
        op.need_t.assign(op.T.nodes.size(), 0);
        for (int64_t i = 0; i < nsample; ++i) {
          if (sample[i] < 0 || sample[i] >= (int64_t)op.T.leaves.size()) throw Err(E_ARG, "leaf index out of range");
          for (int32_t id = op.T.leaves[sample[i]]; id >= 0; id = op.T.nodes[id].parent) op.need_t[id] = 1;
        }
        op.need_t[0] = 1;
        op.onthefly = true;
        coupling = false;
      }
      build_structure(op);
      op.with_coupling = coupling;
      if (coupling) build_coupling(op);
      else op.Eref = transfer_ref(op.m);
    } catch (...) {
      delete o;
      throw;
    }
    *out = o;
  });
}

int orc_create(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx, const double* sy,
               const double* sz, int64_t ns, const double lo[3], const double hi[3], double kappa, int n_max, int m,
               double eta2, int l_hf, int depth_cap, int zero_diagonal, orc_op** out) {
  return create_impl(tx, ty, tz, nt, sx, sy, sz, ns, lo, hi, kappa, n_max, m, eta2, l_hf, depth_cap, zero_diagonal,
                     true, out);
}
int orc_create_structure(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                         const double* sy, const double* sz, int64_t ns, const double lo[3], const double hi[3],
                         double kappa, int n_max, int m, double eta2, int l_hf, int depth_cap, int zero_diagonal,
                         orc_op** out) {
  return create_impl(tx, ty, tz, nt, sx, sy, sz, ns, lo, hi, kappa, n_max, m, eta2, l_hf, depth_cap, zero_diagonal,
                     false, out);
}
int orc_create_sampled(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                       const double* sy, const double* sz, int64_t ns, const double lo[3], const double hi[3],
                       double kappa, int n_max, int m, double eta2, int l_hf, int depth_cap, int zero_diagonal,
                       const int64_t* leaf_idx, int64_t nleaf, orc_op** out) {
  return create_impl(tx, ty, tz, nt, sx, sy, sz, ns, lo, hi, kappa, n_max, m, eta2, l_hf, depth_cap, zero_diagonal,
                     false, out, leaf_idx, nleaf);
}
void orc_destroy(orc_op* op) { delete op; }
int orc_structure_digest(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                         const double* sy, const double* sz, int64_t ns, const double lo[3], const double hi[3],
                         double kappa, int n_max, int m_unused, double eta2, int l_hf, int depth_cap,
                         uint64_t* out6, int64_t* counts) {
  return guard([&] {
    if (!(kappa > 0.0) || !std::isfinite(kappa)) throw Err(E_ARG, "wave number must be positive and finite");
    if (!(eta2 > 0.0)) throw Err(E_ARG, "eta2 must be positive");
    if (l_hf < -2) throw Err(E_ARG, "l_hf must be >= -1 (or -2 for the default rule)");
    (void)m_unused;
    Op op;
    op.kappa = kappa;
    op.eta2 = eta2;
    op.lhf = l_hf;
    op.T.build(tx, ty, tz, nt, lo, hi, n_max, depth_cap);
    op.S.build(sx, sy, sz, ns, lo, hi, n_max, depth_cap);
    structure_digest_stream(op, out6, counts);
  });
}

int orc_apply(orc_op* o, const double* x, double* y) {
  return guard([&] {
    if (!o->op.with_coupling) throw Err(E_ARG, "operator built without coupling matrices");
    apply(o->op, x, y, nullptr);
  });
}
int orc_apply_sampled(orc_op* o, const double* x, const int64_t* leaf_idx, int64_t nleaf, double* y) {
  return guard([&] {
    if (!o->op.with_coupling && !o->op.onthefly) throw Err(E_ARG, "operator built without coupling matrices");
    for (int64_t i = 0; i < nleaf && !o->op.need_t.empty(); ++i)
      if (leaf_idx[i] >= 0 && leaf_idx[i] < (int64_t)o->op.T.leaves.size() && !o->op.need_t[o->op.T.leaves[leaf_idx[i]]])
        throw Err(E_ARG, "leaf was not sampled at orc_create_sampled");
    std::vector<char> mask(o->op.T.leaves.size(), 0);
    for (int64_t i = 0; i < nleaf; ++i) {
      if (leaf_idx[i] < 0 || leaf_idx[i] >= (int64_t)mask.size()) throw Err(E_ARG, "leaf index out of range");
      mask[leaf_idx[i]] = 1;
    }
    apply(o->op, x, y, &mask);
  });
}
int orc_set_aca(orc_op* o, double eps) {
  return guard([&] {
    if (!(eps >= 0.0 && eps < 1.0)) throw Err(E_ARG, "ACA tolerance must be in [0, 1)");
    if (eps > 0.0 && !o->op.with_coupling) throw Err(E_ARG, "ACA needs the stored coupling matrices (orc_create)");
    o->op.aca_eps = eps;
    if (eps > 0.0) build_aca(o->op);
  });
}
int64_t orc_aca_ranks(const orc_op* o, int32_t* out) {
  const int64_t nk = (int64_t)o->op.aca_rank.size();
  if (out)
    for (int64_t k = 0; k < nk; ++k) out[k] = o->op.aca_rank[k];
  return nk;
}
int orc_aca_compress(const double* A, int n, double eps, int max_rank, double* U, double* W) {
  std::vector<cplx> u, w;
  const int k = aca_compress(reinterpret_cast<const cplx*>(A), n, eps, max_rank, u, w);
  if (U) std::memcpy(U, u.data(), sizeof(cplx) * u.size());
  if (W) std::memcpy(W, w.data(), sizeof(cplx) * w.size());
  return k;
}
int orc_last_timing(const orc_op* o, double* out5) {
  for (int i = 0; i < 5; ++i) out5[i] = o->op.tim[i];
  return 0;
}
int64_t orc_leaf_count(const orc_op* o, int which) {
  return (int64_t)(which == 0 ? o->op.T : o->op.S).leaves.size();
}
int64_t orc_leaf_points(const orc_op* o, int which, int64_t leaf, int64_t* idx, int64_t cap) {
  const Tree& tr = which == 0 ? o->op.T : o->op.S;
  if (leaf < 0 || leaf >= (int64_t)tr.leaves.size()) return -1;
  const Node& nd = tr.nodes[tr.leaves[leaf]];
  const int64_t cnt = nd.count();
  for (int64_t i = 0; i < cnt && i < cap; ++i) idx[i] = tr.perm[nd.begin + i];
  return cnt;
}

int orc_stats(const orc_op* o, int64_t* out) {
  const Op& op = o->op;
  for (int i = 0; i < ORC_NSTATS; ++i) out[i] = 0;
  out[ORC_N_C] = (int64_t)op.lplus.size();
  out[ORC_N_SC] = (int64_t)op.keys.size();
  out[ORC_M_D] = op.M_D;
  out[ORC_N_LMINUS] = (int64_t)op.lminus.size();
  out[ORC_DEPTH_T] = op.T.depth;
  out[ORC_DEPTH_S] = op.S.depth;
  out[ORC_L_HF] = op.lhf;
  out[ORC_SLOTS_T] = op.nslotT;
  out[ORC_SLOTS_S] = op.nslotS;
  out[ORC_NODES_T] = (int64_t)op.T.nodes.size();
  out[ORC_NODES_S] = (int64_t)op.S.nodes.size();
  out[ORC_M_D_ZERO] = op.M_D_zero;
  // N_LE (Thm. 1 / Remark 1): S2M + M2M + L2L + L2T applications
  int64_t nle = 0;
  for (int w = 0; w < 2; ++w) {
    const Tree& tr = w == 0 ? op.T : op.S;
    const auto& d = w == 0 ? op.dT : op.dS;
    for (size_t id = 0; id < tr.nodes.size(); ++id) {
      const Node& nd = tr.nodes[id];
      if (nd.leaf) {
        nle += (int64_t)d[id].size();
      } else {
        int nch = 0;
        for (int o2 = 0; o2 < 8; ++o2) nch += nd.child[o2] >= 0;
        nle += (int64_t)d[id].size() * nch;
      }
    }
  }
  out[ORC_N_LE] = nle;
  return 0;
}

int64_t orc_export_tree(const orc_op* o, int which, int64_t* out) {
  const Tree& tr = which == 0 ? o->op.T : o->op.S;
  int64_t r = 0;
  for (int l = 0; l <= tr.depth; ++l)
    for (int32_t id : tr.levels[l]) {
      if (out) {
        const Node& nd = tr.nodes[id];
        int64_t* row = out + 7 * r;
        row[0] = nd.c.level; row[1] = nd.c.i; row[2] = nd.c.j; row[3] = nd.c.k;
        row[4] = nd.begin; row[5] = nd.end; row[6] = nd.leaf;
      }
      ++r;
    }
  return r;
}
int64_t orc_export_perm(const orc_op* o, int which, int64_t* out) {
  const Tree& tr = which == 0 ? o->op.T : o->op.S;
  if (out)
    for (size_t i = 0; i < tr.perm.size(); ++i) out[i] = tr.perm[i];
  return (int64_t)tr.perm.size();
}
int64_t orc_export_lplus(const orc_op* o, int64_t* out) {
  const Op& op = o->op;
  const int64_t nb = (int64_t)op.lplus.size();
  if (!out) return nb;
  std::vector<std::array<int64_t, 8>> rows(nb);
  for (int64_t b = 0; b < nb; ++b) {
    const Coord& t = op.T.nodes[op.lplus[b].t].c;
    const Coord& s = op.S.nodes[op.lplus[b].s].c;
    rows[b] = {t.level, t.i, t.j, t.k, s.i, s.j, s.k, op.lplus[b].dir};
  }
  std::sort(rows.begin(), rows.end());
  std::memcpy(out, rows.data(), sizeof(int64_t) * 8 * nb);
  return nb;
}
int64_t orc_export_lminus(const orc_op* o, int64_t* out) {
  const Op& op = o->op;
  const int64_t nb = (int64_t)op.lminus.size();
  if (!out) return nb;
  std::vector<std::array<int64_t, 8>> rows(nb);
  for (int64_t b = 0; b < nb; ++b) {
    const Coord& t = op.T.nodes[op.lminus[b].first].c;
    const Coord& s = op.S.nodes[op.lminus[b].second].c;
    rows[b] = {t.level, t.i, t.j, t.k, s.level, s.i, s.j, s.k};
  }
  std::sort(rows.begin(), rows.end());
  std::memcpy(out, rows.data(), sizeof(int64_t) * 8 * nb);
  return nb;
}
int64_t orc_export_dirsets(const orc_op* o, int which, int64_t* out) {
  const Op& op = o->op;
  const Tree& tr = which == 0 ? op.T : op.S;
  const auto& d = which == 0 ? op.dT : op.dS;
  const auto& k = which == 0 ? op.kT : op.kS;
  int64_t r = 0;
  for (int l = 0; l <= tr.depth; ++l)
    for (int32_t id : tr.levels[l])
      for (size_t i = 0; i < d[id].size(); ++i) {
        if (out) {
          const Coord& c = tr.nodes[id].c;
          int64_t* row = out + 6 * r;
          row[0] = c.level; row[1] = c.i; row[2] = c.j; row[3] = c.k; row[4] = d[id][i]; row[5] = k[id][i];
        }
        ++r;
      }
  return r;
}

int orc_chebyshev_nodes(double a, double b, int m, double* out) {
  return guard([&] {
    auto x = cheb(a, b, m);
    std::copy(x.begin(), x.end(), out);
  });
}
double orc_lagrange_eval(const double* nodes, int n, int idx, double x) { return lagr(nodes, n, idx, x); }
int orc_transfer_reference(int m, double* out) {
  return guard([&] {
    auto E = transfer_ref(m);
    std::copy(E.begin(), E.end(), out);
  });
}
int orc_interp_matrix(const double* px, const double* py, const double* pz, int64_t np, const double lo[3],
                      const double hi[3], const double c[3], double kappa, int m, double* out) {
  return guard([&] {
    Box b;
    for (int a = 0; a < 3; ++a) { b.lo[a] = lo[a]; b.hi[a] = hi[a]; }
    const Grid g(b, m);
    const int p = m + 1, n = p * p * p;
    std::vector<cplx> row(n);
    for (int64_t j = 0; j < np; ++j) {
      const double x[3] = {px[j], py[j], pz[j]};
      interp_row(g, m, x, c, kappa, row.data());
      for (int k = 0; k < n; ++k) {
        out[2 * (j * n + k)] = row[k].real();
        out[2 * (j * n + k) + 1] = row[k].imag();
      }
    }
  });
}
int orc_dir_index(int level, int l_hf, int64_t dx, int64_t dy, int64_t dz, const double rho[3]) {
  const double v[3] = {dx * rho[0], dy * rho[1], dz * rho[2]};
  return dir_map_vec(level, l_hf, v);
}
int orc_dir_map_vector(int level, int l_hf, const double v[3]) { return dir_map_vec(level, l_hf, v); }
int orc_dir_vector(int level, int l_hf, int idx, double* out3) {
  if (level <= l_hf && (idx < 0 || idx >= num_dirs(level, l_hf))) return E_ARG;
  dir_vec(level, l_hf, idx, out3);
  return 0;
}
int orc_coupling_matrix(int m, double kappa, const double side[3], int64_t dx, int64_t dy, int64_t dz,
                        const double c[3], double* out) {
  return guard([&] {
    coupling_matrix(m, kappa, side, dx, dy, dz, c, reinterpret_cast<cplx*>(out));
  });
}
int orc_dense_rows(const double* tx, const double* ty, const double* tz, const int64_t* rows, int64_t nrows,
                   const double* sx, const double* sy, const double* sz, int64_t ns, const double* v, double kappa,
                   int zero_diagonal, double* out) {
  return guard([&] {
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
    for (int64_t r = 0; r < nrows; ++r) {
      const int64_t j = rows[r];
      cplx acc(0, 0);
      for (int64_t k = 0; k < ns; ++k) {
        if (zero_diagonal && k == j) continue;
        const double d[3] = {tx[j] - sx[k], ty[j] - sy[k], tz[j] - sz[k]};
        if (dot3(d, d) == 0.0) { bad = 1; continue; }
        acc += kernel_diff(d, kappa) * cplx(v[2 * k], v[2 * k + 1]);
      }
      out[2 * r] = acc.real();
      out[2 * r + 1] = acc.imag();
    }
    if (bad) throw Err(E_DOMAIN, "Helmholtz kernel is singular at x == y");
  });
}
int orc_kernel(const double d[3], double kappa, double* out2) {
  return guard([&] {
    const cplx k = kernel_diff(d, kappa);
    out2[0] = k.real();
    out2[1] = k.imag();
  });
}

}  // extern "C"
