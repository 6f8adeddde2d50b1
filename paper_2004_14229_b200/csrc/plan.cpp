// plan.cpp -- level-synchronous setup of the directional matvec (see plan.hpp).
//
// Compiled with -ffp-contract=off: the octant and admissibility decisions must
// use the reference's separate FP64 multiply and add (cluster_tree.cpp:73-77,
// geometry.hpp:69-76) to be bit-exact with it.
#include "plan.hpp"
#include "setup_gpu.hpp"

#include <nvtx3/nvToolsExt.h>
#include <omp.h>

#include <algorithm>
#include <parallel/algorithm>
#include <atomic>
#include <memory>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <tuple>
#include <unordered_map>

namespace fdhelm {

namespace {
constexpr double kRootPad = 1e-12;  // cluster_tree.cpp:9
constexpr double kPi = 3.141592653589793;

[[noreturn]] void fail(int code, const std::string& m) { throw PlanError{code, m}; }

inline double norm3(const double* a) { return std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }

// PAPER.md Alg. 1 (cluster_tree.cpp:12-128), level by level: every node of a
// level that holds more than n_max points (and is below the depth cap) is
// split by the stable octant partition; ranges of distinct nodes are disjoint,
// so the nodes of one level are partitioned in parallel.
void build_tree(TreePlan& T, const double* x, const double* y, const double* z, int64_t n, const double lo[3],
                const double hi[3], int nmax, int cap) {
  if (n <= 0) fail(1, "cluster tree: empty point set");
  if (nmax < 1) fail(1, "cluster tree: n_max must be >= 1");
  if (!(lo[0] < hi[0] && lo[1] < hi[1] && lo[2] < hi[2])) fail(1, "cluster tree: invalid root box");
  if (n > (int64_t)UINT32_MAX) fail(4, "cluster tree: more than 2^32-1 points");
  for (int a = 0; a < 3; ++a) {
    T.lo[a] = lo[a] - kRootPad * (hi[a] - lo[a]);
    T.hi[a] = hi[a];
  }
  int bad = 0;
#pragma omp parallel for reduction(| : bad)
  for (int64_t i = 0; i < n; ++i) {
    const bool in = x[i] > T.lo[0] && x[i] <= T.hi[0] && y[i] > T.lo[1] && y[i] <= T.hi[1] && z[i] > T.lo[2] &&
                    z[i] <= T.hi[2];
    if (!in) bad = 1;
  }
  if (bad) fail(1, "cluster tree: point outside root box");
  T.x.assign(x, x + n);
  T.y.assign(y, y + n);
  T.z.assign(z, z + n);
  T.perm.resize(n);
  for (int64_t i = 0; i < n; ++i) T.perm[i] = (uint32_t)i;
  T.side.push_back({T.hi[0] - T.lo[0], T.hi[1] - T.lo[1], T.hi[2] - T.lo[2]});
  T.diam.push_back(norm3(T.side[0].data()));
  T.lv.emplace_back();
  {
    LevelNodes& L0 = T.lv[0];
    L0.ci = {0}; L0.cj = {0}; L0.ck = {0};
    L0.begin = {0}; L0.end = {(uint32_t)n};
    L0.leaf = {1}; L0.parent = {-1};
  }
  T.oversized = 0;
  for (int l = 0;; ++l) {
    LevelNodes& L = T.lv[l];
    const size_t nn = L.size();
    L.child.assign(nn * 8, -1);
    std::vector<int32_t> refine;
    for (size_t i = 0; i < nn; ++i) {
      const uint32_t cnt = L.end[i] - L.begin[i];
      if (cnt <= (uint32_t)nmax) continue;
      if (l >= cap) { ++T.oversized; continue; }
      refine.push_back((int32_t)i);
    }
    if (refine.empty()) { T.depth = l; break; }
    if (l + 1 > 21) fail(4, "cluster tree deeper than 21 levels is not supported by this build");
    const auto& s = T.side[l];
    T.side.push_back({0.5 * s[0], 0.5 * s[1], 0.5 * s[2]});
    T.diam.push_back(norm3(T.side[l + 1].data()));
    const auto cs = T.side[l + 1];
    std::vector<std::array<uint32_t, 8>> cnt(refine.size());
#pragma omp parallel
    {
      std::vector<uint8_t> oct;
      std::vector<double> tx, ty, tz;
      std::vector<uint32_t> tp;
#pragma omp for schedule(dynamic, 16)
      for (int64_t r = 0; r < (int64_t)refine.size(); ++r) {
        const int32_t id = refine[r];
        const uint32_t b = L.begin[id], e = L.end[id];
        // separate multiply then add, as cluster_tree.cpp:75-77 (no FMA)
        const double mx = T.lo[0] + (double)(2 * L.ci[id] + 1) * cs[0];
        const double my = T.lo[1] + (double)(2 * L.cj[id] + 1) * cs[1];
        const double mz = T.lo[2] + (double)(2 * L.ck[id] + 1) * cs[2];
        oct.resize(e - b);
        std::array<uint32_t, 8> c{};
        for (uint32_t i = b; i < e; ++i) {
          const int o = 4 * (T.x[i] > mx) + 2 * (T.y[i] > my) + (T.z[i] > mz);
          oct[i - b] = (uint8_t)o;
          ++c[o];
        }
        std::array<uint32_t, 8> cur;
        uint32_t acc = 0;
        for (int o = 0; o < 8; ++o) { cur[o] = acc; acc += c[o]; }
        tx.resize(e - b); ty.resize(e - b); tz.resize(e - b); tp.resize(e - b);
        for (uint32_t i = b; i < e; ++i) {
          const uint32_t d = cur[oct[i - b]]++;
          tx[d] = T.x[i]; ty[d] = T.y[i]; tz[d] = T.z[i]; tp[d] = T.perm[i];
        }
        std::copy(tx.begin(), tx.end(), T.x.begin() + b);
        std::copy(ty.begin(), ty.end(), T.y.begin() + b);
        std::copy(tz.begin(), tz.end(), T.z.begin() + b);
        std::copy(tp.begin(), tp.end(), T.perm.begin() + b);
        cnt[r] = c;
      }
    }
    LevelNodes N;
    for (size_t r = 0; r < refine.size(); ++r) {
      const int32_t id = refine[r];
      L.leaf[id] = 0;
      uint32_t off = L.begin[id];
      for (int o = 0; o < 8; ++o) {
        if (cnt[r][o] == 0) continue;
        L.child[(size_t)id * 8 + o] = (int32_t)N.ci.size();
        N.ci.push_back(2 * L.ci[id] + ((o >> 2) & 1));
        N.cj.push_back(2 * L.cj[id] + ((o >> 1) & 1));
        N.ck.push_back(2 * L.ck[id] + (o & 1));
        N.begin.push_back(off);
        N.end.push_back(off + cnt[r][o]);
        N.leaf.push_back(1);
        N.parent.push_back(id);
        off += cnt[r][o];
      }
    }
    T.lv.push_back(std::move(N));
  }
}

// Def. 1 (A1)+(A3), inclusive <=; the FP64 operation order of
// box_distance (geometry.hpp:69-76) and ClusterTree::box (cluster_tree.cpp:130-139).
inline bool admissible(const Plan& P, int l, int32_t t, int32_t s) {
  const TreePlan& T = P.T;
  const TreePlan& S = P.S;
  const double q = std::max(T.diam[l], S.diam[l]);
  const int64_t tc[3] = {T.lv[l].ci[t], T.lv[l].cj[t], T.lv[l].ck[t]};
  const int64_t sc[3] = {S.lv[l].ci[s], S.lv[l].cj[s], S.lv[l].ck[s]};
  double acc = 0.0;
  for (int a = 0; a < 3; ++a) {
    const double tlo = T.lo[a] + (double)tc[a] * T.side[l][a];
    const double thi = T.lo[a] + (double)(tc[a] + 1) * T.side[l][a];
    const double slo = S.lo[a] + (double)sc[a] * S.side[l][a];
    const double shi = S.lo[a] + (double)(sc[a] + 1) * S.side[l][a];
    const double gap = std::max(std::max(tlo - shi, slo - thi), 0.0);
    acc += gap * gap;
  }
  const double dist = std::sqrt(acc);
  return (q <= P.prm.eta2 * dist) && (P.prm.kappa * q * q <= P.prm.eta2 * dist);
}

// PAPER.md Alg. 2 as a breadth-first sweep: the children of every inadmissible,
// non-leaf pair of level l form the candidate pairs of level l+1.
void build_blocks(Plan& P) {
  const TreePlan& T = P.T;
  const TreePlan& S = P.S;
  std::vector<std::pair<int32_t, int32_t>> cur{{0, 0}};
  const int maxl = std::min(T.depth, S.depth);
  P.blocks.assign(maxl + 1, {});
  const int nth = omp_get_max_threads();
  for (int l = 0; !cur.empty(); ++l) {
    LevelBlocks& B = P.blocks[l];
    const LevelNodes& LT = T.lv[l];
    const LevelNodes& LS = S.lv[l];
    const int64_t np = (int64_t)cur.size();
    const int nchunk = (int)std::min<int64_t>(np, 4 * nth);
    std::vector<std::vector<int32_t>> lpt(nchunk), lps(nchunk), lmt(nchunk), lms(nchunk);
    std::vector<std::vector<std::pair<int32_t, int32_t>>> nxt(nchunk);
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < nchunk; ++c) {
      const int64_t b = np * c / nchunk, e = np * (c + 1) / nchunk;
      for (int64_t i = b; i < e; ++i) {
        const int32_t t = cur[i].first, s = cur[i].second;
        const bool adm = admissible(P, l, t, s);
        if (LT.leaf[t] || LS.leaf[s]) {
          if (adm) { lpt[c].push_back(t); lps[c].push_back(s); }
          else { lmt[c].push_back(t); lms[c].push_back(s); }
        } else if (!adm) {
          for (int a = 0; a < 8; ++a) {
            const int32_t ta = LT.child[(size_t)t * 8 + a];
            if (ta < 0) continue;
            for (int bb = 0; bb < 8; ++bb) {
              const int32_t sb = LS.child[(size_t)s * 8 + bb];
              if (sb >= 0) nxt[c].push_back({ta, sb});
            }
          }
        } else {
          lpt[c].push_back(t);
          lps[c].push_back(s);
        }
      }
    }
    cur.clear();
    for (int c = 0; c < nchunk; ++c) {
      B.lp_t.insert(B.lp_t.end(), lpt[c].begin(), lpt[c].end());
      B.lp_s.insert(B.lp_s.end(), lps[c].begin(), lps[c].end());
      B.lm_t.insert(B.lm_t.end(), lmt[c].begin(), lmt[c].end());
      B.lm_s.insert(B.lm_s.end(), lms[c].begin(), lms[c].end());
      cur.insert(cur.end(), nxt[c].begin(), nxt[c].end());
    }
    if (!cur.empty() && l + 1 > maxl) fail(1, "internal: block recursion beyond tree depth");
  }
}

// (level, lattice offset) keys, numbered in (level, dx, dy, dz) order; the
// direction of a key is dir_(l)(offset * rho) (Def. 3).
void build_keys(Plan& P) {
  int32_t base = 0;
  for (int l = 0; l < (int)P.blocks.size(); ++l) {
    LevelBlocks& B = P.blocks[l];
    const int64_t nb = (int64_t)B.lp_t.size();
    B.lp_key.assign(nb, -1);
    if (nb == 0) continue;
    const LevelNodes& LT = P.T.lv[l];
    const LevelNodes& LS = P.S.lv[l];
    int64_t mn[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, mx[3] = {INT64_MIN, INT64_MIN, INT64_MIN};
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t d[3] = {LT.ci[B.lp_t[b]] - LS.ci[B.lp_s[b]], LT.cj[B.lp_t[b]] - LS.cj[B.lp_s[b]],
                            LT.ck[B.lp_t[b]] - LS.ck[B.lp_s[b]]};
      for (int a = 0; a < 3; ++a) { mn[a] = std::min(mn[a], d[a]); mx[a] = std::max(mx[a], d[a]); }
    }
    const int64_t ext[3] = {mx[0] - mn[0] + 1, mx[1] - mn[1] + 1, mx[2] - mn[2] + 1};
    const int64_t vol = ext[0] * ext[1] * ext[2];
    auto lin = [&](int64_t b) {
      const int64_t d0 = LT.ci[B.lp_t[b]] - LS.ci[B.lp_s[b]] - mn[0];
      const int64_t d1 = LT.cj[B.lp_t[b]] - LS.cj[B.lp_s[b]] - mn[1];
      const int64_t d2 = LT.ck[B.lp_t[b]] - LS.ck[B.lp_s[b]] - mn[2];
      return (d0 * ext[1] + d1) * ext[2] + d2;
    };
    if (vol <= (int64_t)1 << 27) {
      std::vector<int32_t> tab(vol, -1);
      for (int64_t b = 0; b < nb; ++b) tab[lin(b)] = 0;
      int32_t id = base;
      for (int64_t v = 0; v < vol; ++v)
        if (tab[v] == 0) {
          tab[v] = id++;
          const int64_t d2 = v % ext[2], d1 = (v / ext[2]) % ext[1], d0 = v / (ext[1] * ext[2]);
          P.key_level.push_back(l);
          P.key_dx.push_back(d0 + mn[0]);
          P.key_dy.push_back(d1 + mn[1]);
          P.key_dz.push_back(d2 + mn[2]);
        }
#pragma omp parallel for
      for (int64_t b = 0; b < nb; ++b) B.lp_key[b] = tab[lin(b)];
      base = id;
    } else {
      std::vector<int64_t> u(nb);
      for (int64_t b = 0; b < nb; ++b) u[b] = lin(b);
      std::vector<int64_t> s = u;
      std::sort(s.begin(), s.end());
      s.erase(std::unique(s.begin(), s.end()), s.end());
      for (int64_t v : s) {
        const int64_t d2 = v % ext[2], d1 = (v / ext[2]) % ext[1], d0 = v / (ext[1] * ext[2]);
        P.key_level.push_back(l);
        P.key_dx.push_back(d0 + mn[0]);
        P.key_dy.push_back(d1 + mn[1]);
        P.key_dz.push_back(d2 + mn[2]);
      }
#pragma omp parallel for
      for (int64_t b = 0; b < nb; ++b)
        B.lp_key[b] = base + (int32_t)(std::lower_bound(s.begin(), s.end(), u[b]) - s.begin());
      base += (int32_t)s.size();
    }
  }
  P.n_sc = base;
  P.key_dir.resize(base);
  for (int32_t k = 0; k < base; ++k) {
    const double v[3] = {P.key_dx[k] * P.rho[0], P.key_dy[k] * P.rho[1], P.key_dz[k] * P.rho[2]};
    P.key_dir[k] = dir_map_vec(P.key_level[k], P.lhf, v);
  }
}

// Def. 4: D from admissible partners, D^ from the parent's D u D^; dense slots.
void build_dirsets(Plan& P, TreePlan& T, bool is_target) {
  const int nl = T.depth + 1;
  T.ndir.resize(nl);
  T.kind.assign(nl, {});
  T.slot_of.assign(nl, {});
  for (int l = 0; l < nl; ++l) {
    T.ndir[l] = num_dirs(l, P.lhf);
    T.kind[l].assign(T.lv[l].size() * (size_t)T.ndir[l], 0);
  }
  for (int l = 0; l < (int)P.blocks.size() && l < nl; ++l) {
    const LevelBlocks& B = P.blocks[l];
    const int nd = T.ndir[l];
    const auto& idx = is_target ? B.lp_t : B.lp_s;
    for (size_t b = 0; b < idx.size(); ++b) T.kind[l][(size_t)idx[b] * nd + P.key_dir[B.lp_key[b]]] |= 1;
  }
  for (int l = 1; l < nl; ++l) {
    const int nd = T.ndir[l], npd = T.ndir[l - 1];
    const LevelNodes& L = T.lv[l];
#pragma omp parallel for
    for (int64_t i = 0; i < (int64_t)L.size(); ++i) {
      const int32_t par = L.parent[i];
      for (int c = 0; c < npd; ++c)
        if (T.kind[l - 1][(size_t)par * npd + c]) T.kind[l][(size_t)i * nd + parent_dir(l - 1, P.lhf, c)] |= 2;
    }
  }
  int64_t s = 0;
  T.node_slot_first.clear();
  for (int l = 0; l < nl; ++l) {
    const int nd = T.ndir[l];
    T.slot_of[l].assign(T.kind[l].size(), -1);
    for (size_t i = 0; i < T.lv[l].size(); ++i)
      for (int c = 0; c < nd; ++c)
        if (T.kind[l][i * nd + c]) {
          T.slot_of[l][i * nd + c] = (int32_t)s++;
          T.slot_level.push_back(l);
          T.slot_node.push_back((int32_t)i);
          T.slot_dir.push_back(c);
        }
  }
  T.nslots = s;
}

inline int32_t slot_at(const TreePlan& T, int l, int32_t node, int dir) {
  return T.slot_of[l][(size_t)node * T.ndir[l] + dir];
}

void build_worklists(Plan& P) {
  TreePlan& T = P.T;
  TreePlan& S = P.S;
  const int lhf = P.lhf;
  // ---- S2M over source leaves
  for (int l = 0; l <= S.depth; ++l) {
    const LevelNodes& L = S.lv[l];
    for (size_t i = 0; i < L.size(); ++i) {
      if (!L.leaf[i]) continue;
      for (int c = 0; c < S.ndir[l]; ++c) {
        const int32_t sl = slot_at(S, l, (int32_t)i, c);
        if (sl < 0) continue;
        P.s2m_slot.push_back(sl);
        P.s2m_level.push_back(l);
        P.s2m_dir.push_back(c);
        P.s2m_ci.push_back(L.ci[i]);
        P.s2m_cj.push_back(L.cj[i]);
        P.s2m_ck.push_back(L.ck[i]);
        P.s2m_begin.push_back(L.begin[i]);
        P.s2m_end.push_back(L.end[i]);
      }
    }
  }
  // ---- M2M (parents at level l)
  P.m2m_parent.assign(S.depth + 1, {});
  P.m2m_dir = P.m2m_cdir = P.m2m_child = P.m2m_parent;
  P.m2m_pc.assign(S.depth + 1, {});
  for (int l = 0; l < S.depth; ++l) {
    const LevelNodes& L = S.lv[l];
    for (size_t i = 0; i < L.size(); ++i) {
      if (L.leaf[i]) continue;
      for (int c = 0; c < S.ndir[l]; ++c) {
        const int32_t sl = slot_at(S, l, (int32_t)i, c);
        if (sl < 0) continue;
        const int cp = parent_dir(l, lhf, c);
        P.m2m_parent[l].push_back(sl);
        P.m2m_dir[l].push_back(c);
        P.m2m_cdir[l].push_back(cp);
        P.m2m_pc[l].push_back(L.ci[i]);
        P.m2m_pc[l].push_back(L.cj[i]);
        P.m2m_pc[l].push_back(L.ck[i]);
        for (int o = 0; o < 8; ++o) {
          const int32_t ch = L.child[i * 8 + o];
          int32_t cs = -1;
          if (ch >= 0) {
            cs = slot_at(S, l + 1, ch, cp);
            if (cs < 0) fail(1, "internal: missing child moment slot");
          }
          P.m2m_child[l].push_back(cs);
        }
      }
    }
  }
  // ---- L2L (children at level l+1)
  P.l2l_child.assign(T.depth + 1, {});
  P.l2l_cdir = P.l2l_pslot = P.l2l_pdir = P.l2l_oct = P.l2l_child;
  P.l2l_ptr.assign(T.depth + 1, {0});
  P.l2l_cc.assign(T.depth + 1, {});
  for (int l = 0; l < T.depth; ++l) {
    const LevelNodes& L = T.lv[l + 1];
    const LevelNodes& LP = T.lv[l];
    for (size_t i = 0; i < L.size(); ++i) {
      const int32_t par = L.parent[i];
      const int oct = 4 * (int)(L.ci[i] & 1) + 2 * (int)(L.cj[i] & 1) + (int)(L.ck[i] & 1);
      (void)LP;
      if (!P.t_needed.empty() && !P.t_needed[l + 1][i]) continue;
      for (int cc = 0; cc < T.ndir[l + 1]; ++cc) {
        const int32_t csl = slot_at(T, l + 1, (int32_t)i, cc);
        if (csl < 0) continue;
        int cnt = 0;
        for (int c = 0; c < T.ndir[l]; ++c) {
          const int32_t psl = slot_at(T, l, par, c);
          if (psl < 0 || parent_dir(l, lhf, c) != cc) continue;
          P.l2l_pslot[l].push_back(psl);
          P.l2l_pdir[l].push_back(c);
          P.l2l_oct[l].push_back(oct);
          ++cnt;
        }
        if (cnt == 0) continue;
        P.l2l_child[l].push_back(csl);
        P.l2l_cdir[l].push_back(cc);
        P.l2l_cc[l].push_back(L.ci[i]);
        P.l2l_cc[l].push_back(L.cj[i]);
        P.l2l_cc[l].push_back(L.ck[i]);
        P.l2l_ptr[l].push_back((int32_t)P.l2l_pslot[l].size());
      }
    }
  }
  // ---- L2T + P2P over owned target leaves
  std::vector<std::vector<std::vector<std::pair<uint32_t, uint32_t>>>> near(T.depth + 1);
  for (int l = 0; l <= T.depth; ++l) near[l].assign(T.lv[l].size(), {});
  for (int l = 0; l < (int)P.blocks.size(); ++l) {
    const LevelBlocks& B = P.blocks[l];
    for (size_t b = 0; b < B.lm_t.size(); ++b)
      near[l][B.lm_t[b]].push_back({S.lv[l].begin[B.lm_s[b]], S.lv[l].end[B.lm_s[b]]});
  }
  P.p2p_ptr.assign(1, 0);
  int64_t leaf_id = 0;
  for (int l = 0; l <= T.depth; ++l) {
    const LevelNodes& L = T.lv[l];
    for (size_t i = 0; i < L.size(); ++i) {
      if (!L.leaf[i]) continue;
      const bool own = P.t_leaf_owned.empty() || P.t_leaf_owned[leaf_id];
      ++leaf_id;
      if (!own) continue;
      int32_t s0 = -1, ns = 0;
      for (int c = 0; c < T.ndir[l]; ++c) {
        const int32_t sl = slot_at(T, l, (int32_t)i, c);
        if (sl < 0) continue;
        if (s0 < 0) s0 = sl;
        ++ns;
      }
      P.l2t_level.push_back(l);
      P.l2t_slot0.push_back(s0);
      P.l2t_nslot.push_back(ns);
      P.l2t_ci.push_back(L.ci[i]);
      P.l2t_cj.push_back(L.cj[i]);
      P.l2t_ck.push_back(L.ck[i]);
      P.l2t_begin.push_back(L.begin[i]);
      P.l2t_end.push_back(L.end[i]);
      std::vector<std::pair<uint32_t, uint32_t>> rg;
      int32_t id = (int32_t)i;
      for (int ll = l; ll >= 0; --ll) {
        rg.insert(rg.end(), near[ll][id].begin(), near[ll][id].end());
        id = T.lv[ll].parent[id];
      }
      std::sort(rg.begin(), rg.end());
      for (size_t r = 0; r < rg.size(); ++r) {
        if (!P.p2p_sbeg.empty() && P.p2p_ptr.back() < (int64_t)P.p2p_sbeg.size() && P.p2p_send.back() == rg[r].first) {
          P.p2p_send.back() = rg[r].second;  // merge contiguous ranges
        } else {
          P.p2p_sbeg.push_back(rg[r].first);
          P.p2p_send.push_back(rg[r].second);
        }
      }
      P.p2p_ptr.push_back((int64_t)P.p2p_sbeg.size());
    }
  }
}

// Pair part of the int8 M2L plan (key-major; SURVEY.md 7 "key-major" alternative):
// the (key, target slot, source slot) triples sorted by key, then target slot,
// cut into tiles of TT pairs of one key, one work item per tile (one key: no
// chain), APPENDED to the plan's tiles and items.  The kernel writes each pair's
// n values to an output buffer; k_m2l_reduce adds them to the target slot's
// locals as a running sum in pair order (= key order): deterministic.
// red_ptr / red_idx: per target slot its pair indices (relative to the first
// pair tile: (tile - pair_tile0) * TT + column), increasing.
void append_pair_part(Plan& P, std::vector<std::array<int32_t, 3>>& kts, int TT) {
  __gnu_parallel::sort(kts.begin(), kts.end());  // up to 6e8 triples (config 4 hybrid)
  const int64_t np = (int64_t)kts.size();
  const int64_t tile0 = (int64_t)P.tile_level.size(), item0 = (int64_t)P.item_tile.size();
  P.m2l_pair_tile0 = tile0;
  P.m2l_pair_item0 = item0;
  int64_t ntile = 0;
  for (int64_t b = 0; b < np;) {
    int64_t e = b;
    while (e < np && kts[e][0] == kts[b][0]) ++e;
    ntile += (e - b + TT - 1) / TT;
    b = e;
  }
  const int64_t nt = tile0 + ntile;
  P.tile_level.resize(nt, 0);
  P.tile_dir.resize(nt, 0);
  P.tile_tslot.resize(nt * TT, -1);
  P.tile_nitem.resize(nt, 1);
  const int64_t kbase = (int64_t)P.tile_keys.size();
  P.tile_keys.resize(kbase + ntile, 0);
  P.tile_src.resize((kbase + ntile) * TT, -1);
  P.tile_cols.resize((kbase + ntile) * TT, 0);
  P.tile_cnt.resize(kbase + ntile, 0);
  P.tile_same.resize(kbase + ntile, 0);
  P.tile_kptr.resize(nt + 1, P.tile_kptr.empty() ? 0 : P.tile_kptr.back());
  P.red_ptr.assign(P.T.nslots + 1, 0);
  int64_t tl = tile0, kk = kbase;
  for (int64_t b = 0; b < np;) {
    int64_t e = b;
    while (e < np && kts[e][0] == kts[b][0]) ++e;
    const int32_t key = kts[b][0];
    for (int64_t c0 = b; c0 < e; c0 += TT, ++tl, ++kk) {
      const int cnt = (int)std::min<int64_t>(TT, e - c0);
      P.tile_level[tl] = P.key_level[key];
      P.tile_dir[tl] = P.key_dir[key];
      P.tile_keys[kk] = key;
      P.tile_kptr[tl + 1] = kk + 1;
      P.tile_cnt[kk] = (uint8_t)cnt;
      for (int c = 0; c < cnt; ++c) {
        P.tile_tslot[tl * TT + c] = kts[c0 + c][1];
        P.tile_src[kk * TT + c] = kts[c0 + c][2];
        P.tile_cols[kk * TT + c] = (uint8_t)c;
        ++P.red_ptr[kts[c0 + c][1] + 1];
      }
      P.item_tile.push_back((int32_t)tl);
      P.item_seq.push_back(0);
      P.item_k0.push_back(kk);
      P.item_k1.push_back(kk + 1);
    }
    b = e;
  }
  for (int64_t t = 0; t < P.T.nslots; ++t) P.red_ptr[t + 1] += P.red_ptr[t];
  P.red_idx.assign(np, 0);
  std::vector<int64_t> cur(P.red_ptr.begin(), P.red_ptr.end() - 1);
  for (int64_t t2 = tile0; t2 < nt; ++t2) {
    const int64_t k2 = P.tile_kptr[t2];
    for (int c = 0; c < P.tile_cnt[k2]; ++c) P.red_idx[cur[P.tile_tslot[t2 * TT + c]]++] = (t2 - tile0) * TT + c;
  }
  P.m2l_pair = np > 0;
}

// M2L tiles: target slots grouped by (level, direction, lattice parity) share
// (almost) the same key list; a tile = `tile` such slots, the union of their
// keys, and for every key the source slot of each column (-1 if none).
void build_m2l(Plan& P) {
  auto mts = std::chrono::steady_clock::now();
  const bool mdbg = std::getenv("FDH_DEBUG_SETUP") != nullptr;
#define MTICK(what)                                                                                    \
  do {                                                                                                 \
    const auto now_ = std::chrono::steady_clock::now();                                                \
    if (mdbg) std::fprintf(stderr, "[m2l]   before %-14s %9.1f ms\n", what,                           \
                           std::chrono::duration<double, std::milli>(now_ - mts).count());           \
    mts = now_;                                                                                        \
  } while (0)
  const TreePlan& T = P.T;
  const TreePlan& S = P.S;
  int TT = P.prm.tile;  // < 0: choose 16 or 32 target columns below (int8 M2L, 2-3 M-blocks)
  // multiple right-hand sides: a tile holds TT / R target slots x R rhs; the
  // column of (slot i of the tile, rhs r) is i * R + r and refers to the
  // rhs-major slot id r * nslots + slot (moments / locals stored per rhs)
  const int R = P.prm.nrhs;
  const int tw = TT < 0 ? 16 : TT;  // auto: both candidates (16, 32) are multiples of R <= 16
  if (R < 1 || R > tw || tw % R != 0) throw PlanError{1, "nrhs must divide the M2L tile width " + std::to_string(tw)};
  // pairs (target slot, key, source slot) grouped by target slot: parallel
  // counting pass, prefix, parallel scatter with atomic cursors (the order
  // inside a slot is then fixed by the per-slot sort by key -- keys are unique
  // within a slot, so the result is deterministic)
  int64_t npairs = 0;
  for (auto& B : P.blocks) npairs += (int64_t)B.lp_t.size();
  if (!P.prm.gpu_structure) P.n_c = npairs;  // GPU partition: the full |L+| (shards hold a part)
  std::unique_ptr<std::atomic<int64_t>[]> cnt(new std::atomic<int64_t>[T.nslots + 1]);
  for (int64_t i = 0; i <= T.nslots; ++i) cnt[i].store(0, std::memory_order_relaxed);
  for (int l = 0; l < (int)P.blocks.size(); ++l) {
    const LevelBlocks& B = P.blocks[l];
    const int64_t nb = (int64_t)B.lp_t.size();
#pragma omp parallel for
    for (int64_t b = 0; b < nb; ++b)
      cnt[slot_at(T, l, B.lp_t[b], P.key_dir[B.lp_key[b]]) + 1].fetch_add(1, std::memory_order_relaxed);
  }
  std::vector<int64_t> ptr(T.nslots + 1, 0);
  for (int64_t i = 0; i < T.nslots; ++i) ptr[i + 1] = ptr[i] + cnt[i + 1].load(std::memory_order_relaxed);
  for (int64_t i = 0; i < T.nslots; ++i) cnt[i].store(ptr[i], std::memory_order_relaxed);
  std::unique_ptr<int32_t[]> skb(new int32_t[std::max<int64_t>(1, npairs)]), ssb(new int32_t[std::max<int64_t>(1, npairs)]);
  int32_t* sk = skb.get();
  int32_t* ss = ssb.get();
  for (int l = 0; l < (int)P.blocks.size(); ++l) {
    const LevelBlocks& B = P.blocks[l];
    const int64_t nb = (int64_t)B.lp_t.size();
#pragma omp parallel for
    for (int64_t b = 0; b < nb; ++b) {
      const int d = P.key_dir[B.lp_key[b]];
      const int64_t pos = cnt[slot_at(T, l, B.lp_t[b], d)].fetch_add(1, std::memory_order_relaxed);
      sk[pos] = B.lp_key[b];
      ss[pos] = slot_at(S, l, B.lp_s[b], d);
    }
  }
  MTICK("counting sort");
  // per-slot sort by key: keys are ids inside one level, unique within a slot ->
  // an order-preserving 64-bit pack (key << 32 | source) sorts both at once
#pragma omp parallel
  {
    std::vector<uint64_t> v;
#pragma omp for schedule(dynamic, 64)
    for (int64_t t = 0; t < T.nslots; ++t) {
      const int64_t b = ptr[t], e = ptr[t + 1];
      if (e - b < 2) continue;
      v.resize(e - b);
      for (int64_t i = b; i < e; ++i) v[i - b] = ((uint64_t)(uint32_t)sk[i] << 32) | (uint32_t)ss[i];
      std::sort(v.begin(), v.end());
      for (int64_t i = b; i < e; ++i) {
        sk[i] = (int32_t)(v[i - b] >> 32);
        ss[i] = (int32_t)(uint32_t)v[i - b];
      }
    }
  }
  MTICK("slot sort");
  // group target slots (a shard keeps only the slots of its leaves' ancestor closure)
  std::vector<int32_t> ts;
  for (int64_t t = 0; t < T.nslots; ++t)
    if (ptr[t + 1] > ptr[t] && (P.t_needed.empty() || P.t_needed[T.slot_level[t]][T.slot_node[t]]))
      ts.push_back((int32_t)t);
  auto gkey = [&](int32_t t) {
    const int l = T.slot_level[t];
    const int32_t nd = T.slot_node[t];
    const int par = 4 * (int)(T.lv[l].ci[nd] & 1) + 2 * (int)(T.lv[l].cj[nd] & 1) + (int)(T.lv[l].ck[nd] & 1);
    return ((int64_t)l << 40) | ((int64_t)T.slot_dir[t] << 8) | par;
  };
  std::stable_sort(ts.begin(), ts.end(), [&](int32_t a, int32_t b) { return gkey(a) < gkey(b); });
  std::vector<int32_t> key_lo(64, 0), key_hi(64, 0);
  for (int32_t k = (int32_t)P.key_level.size() - 1; k >= 0; --k) key_lo[P.key_level[k]] = k;
  for (int32_t k = 0; k < (int32_t)P.key_level.size(); ++k) key_hi[P.key_level[k]] = k + 1;
  bool pair_mode = false;
  if (P.prm.m2l_impl == 1) {
    // int8 M2L with 2-3 M-blocks: 16 target columns (one pass over M-blocks {0,1}
    // [+ {2}]) or 32 (one pass per M-block: twice the columns per W byte, the
    // issued rate measured 1.14-1.18x higher, profiles/r02_m2l_sweep_tt_chunk.jsonl)
    // -- but the union of a wider tile's key lists leaves more columns absent
    // (clustered sources: config 5).  Estimated on every 8th 32-wide tile: the
    // tile-keys of it and of its two 16-wide halves; 32 when 32 K32 / 1.16 < 16 K16.
    // When even the better tiling leaves most columns without a key (useful <
    // 0.45: clustered sources), the M2L runs key-major on (target, source) PAIRS
    // instead (pair mode below): every column carries a key.
    const int64_t w32 = 32 / R, w16 = 16 / R;
    // sampled cost of an order `ord` of the slots: tile-keys of the 32- and 16-wide
    // tilings, pairs, and for the 32-wide tiling the full rows / partial pairs of the
    // hybrid split
    struct Smp { int64_t k16 = 0, k32 = 0, pairs = 0, full32 = 0, part32 = 0; };
    auto sample = [&](const std::vector<int32_t>& ord) {
      std::vector<std::pair<int64_t, int64_t>> smp;  // [begin, end) into ord of sampled 32-wide tiles
      for (size_t i = 0; i < ord.size();) {
        size_t j = i;
        const int64_t g = gkey(ord[i]);
        while (j < ord.size() && gkey(ord[j]) == g) ++j;
        int64_t q = 0;
        for (size_t k = i; k < j; k += w32, ++q)
          if ((q & 7) == 0) smp.push_back({(int64_t)k, (int64_t)std::min(j, k + w32)});
        i = j;
      }
      int64_t k16 = 0, k32 = 0, pairs_s = 0, full32 = 0, part32 = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : k16, k32, pairs_s, full32, part32)
      for (int64_t si = 0; si < (int64_t)smp.size(); ++si) {
        const int64_t b = smp[si].first, e = smp[si].second;
        const int l = T.slot_level[ord[b]];
        const int32_t kb = key_lo[l], kr = key_hi[l] - kb;
        thread_local std::vector<uint8_t> mk, ct;
        mk.assign(kr, 0);
        ct.assign(kr, 0);
        for (int64_t i = b; i < e; ++i) {
          const uint8_t bit = (i - b) < w16 ? 1 : 2;
          pairs_s += (ptr[ord[i] + 1] - ptr[ord[i]]) * R;
          for (int64_t q = ptr[ord[i]]; q < ptr[ord[i] + 1]; ++q) {
            mk[sk[q] - kb] |= bit;
            ++ct[sk[q] - kb];
          }
        }
        for (int32_t k = 0; k < kr; ++k) {
          k32 += mk[k] != 0;
          k16 += (mk[k] & 1) + (mk[k] >> 1);
          if (ct[k] == e - b) ++full32;
          else part32 += ct[k] * R;
        }
      }
      return Smp{k16, k32, pairs_s, full32, part32};
    };
    const Smp sm = sample(ts);
    const int64_t k16 = sm.k16, k32 = sm.k32, pairs_s = sm.pairs;
    if (TT < 0) TT = (32.0 * (double)k32 / 1.16 < 16.0 * (double)k16) ? 32 : 16;
    const double useful = (double)pairs_s / std::max(1.0, (double)(TT == 32 ? k32 : k16) * TT);
    const char* pm = std::getenv("FDH_M2L_PAIR");  // 1: force pair mode, 0: never
    pair_mode = R == 1 && (pm ? pm[0] == '1' : useful < 0.45);
    if (pair_mode) TT = 32;
    P.prm.tile = TT;
    if (mdbg)
      std::fprintf(stderr, "[m2l] tile width: sampled tile-keys 16: %lld, 32: %lld, useful %.3f -> %d%s\n",
                   (long long)k16, (long long)k32, useful, TT, pair_mode ? " (pair mode)" : "");
  }
  if (pair_mode) {
    // ---- pair mode (key-major): every (target slot, key, source slot) triple
    std::vector<std::array<int32_t, 3>> kts;
    kts.reserve(npairs);
    for (int32_t t : ts)
      for (int64_t q = ptr[t]; q < ptr[t + 1]; ++q) kts.push_back({sk[q], t, ss[q]});
    P.tile_level.clear();
    P.tile_dir.clear();
    P.tile_tslot.clear();
    P.tile_kptr.assign(1, 0);
    P.tile_keys.clear();
    P.tile_src.clear();
    P.tile_cols.clear();
    P.tile_cnt.clear();
    P.tile_same.clear();
    P.item_tile.clear();
    P.item_seq.clear();
    P.item_k0.clear();
    P.item_k1.clear();
    P.tile_nitem.clear();
    append_pair_part(P, kts, TT);
    P.m2l_chunk = 1;
    P.m2l_units_exec = 0;
    for (int64_t t = 0; t < T.nslots; ++t)
      if (ptr[t + 1] == ptr[t]) P.m2l_zero_slots.push_back((int32_t)t);
    MTICK("pair plan");
    return;
  }
  std::vector<int64_t> tile_first;  // index into ts
  for (size_t i = 0; i < ts.size();) {
    size_t j = i;
    const int64_t g = gkey(ts[i]);
    while (j < ts.size() && gkey(ts[j]) == g) ++j;
    for (size_t k = i; k < j; k += TT / R) tile_first.push_back((int64_t)k);
    i = j;
  }
  tile_first.push_back((int64_t)ts.size());
  const int64_t ntile = (int64_t)tile_first.size() - 1;
  // a tile never spans two groups: clip at group boundaries
  P.tile_level.assign(ntile, 0);
  P.tile_dir.assign(ntile, 0);
  P.tile_tslot.assign(ntile * TT, -1);
  std::vector<std::vector<int32_t>> tkeys(ntile);
  std::vector<int64_t> tcount(ntile);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t tl = 0; tl < ntile; ++tl) {
    int64_t b = tile_first[tl], e = tile_first[tl + 1];
    const int64_t g = gkey(ts[b]);
    int64_t ee = b;
    while (ee < e && gkey(ts[ee]) == g) ++ee;
    e = ee;
    P.tile_level[tl] = T.slot_level[ts[b]];
    P.tile_dir[tl] = T.slot_dir[ts[b]];
    // union of the slots' sorted key lists: dense marks over the level's key range
    const int32_t kb = key_lo[P.tile_level[tl]], kr = key_hi[P.tile_level[tl]] - kb;
    thread_local std::vector<uint8_t> mark;
    mark.assign(kr, 0);
    int64_t nk = 0;
    for (int64_t i = b; i < e; ++i) {
      for (int r = 0; r < R; ++r) P.tile_tslot[tl * TT + (i - b) * R + r] = (int32_t)(ts[i] + r * T.nslots);
      for (int64_t q = ptr[ts[i]]; q < ptr[ts[i] + 1]; ++q) {
        nk += !mark[sk[q] - kb];
        mark[sk[q] - kb] = 1;
      }
    }
    std::vector<int32_t> u;
    u.reserve(nk);
    for (int32_t k = 0; k < kr; ++k)
      if (mark[k]) u.push_back(kb + k);
    tcount[tl] = (int64_t)u.size();
    tkeys[tl] = std::move(u);
  }
  MTICK("tile groups");
  P.tile_kptr.assign(ntile + 1, 0);
  for (int64_t tl = 0; tl < ntile; ++tl) P.tile_kptr[tl + 1] = P.tile_kptr[tl] + tcount[tl];
  const int64_t tot = P.tile_kptr[ntile];
  P.tile_keys.resize(tot);
  P.tile_src.assign(tot * TT, -1);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t tl = 0; tl < ntile; ++tl) {
    const auto& u = tkeys[tl];
    const int64_t base = P.tile_kptr[tl];
    std::copy(u.begin(), u.end(), P.tile_keys.begin() + base);
    if (u.empty()) continue;
    const int32_t kb = u.front();
    std::vector<int32_t> pos(u.back() - kb + 1, -1);  // key -> position in the union
    for (size_t q = 0; q < u.size(); ++q) pos[u[q] - kb] = (int32_t)q;
    for (int c = 0; c < TT; ++c) {
      const int32_t tv = P.tile_tslot[tl * TT + c];
      if (tv < 0) continue;
      const int32_t t = (int32_t)(tv % T.nslots), sr = (int32_t)(tv / T.nslots * S.nslots);
      for (int64_t i = ptr[t]; i < ptr[t + 1]; ++i) P.tile_src[(base + pos[sk[i] - kb]) * TT + c] = ss[i] + sr;
    }
  }
  MTICK("tile src");
  // compact the valid columns of every (tile, key) to the front
  P.tile_cols.assign(tot * TT, 0);
  P.tile_cnt.assign(tot, 0);
  P.tile_same.assign(tot, 0);
  int64_t exec = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : exec)
  for (int64_t tl = 0; tl < ntile; ++tl) {
    for (int64_t i = P.tile_kptr[tl]; i < P.tile_kptr[tl + 1]; ++i) {
      int cnt = 0;
      int32_t src[64];
      uint8_t col[64];
      for (int c = 0; c < TT; ++c)
        if (P.tile_src[i * TT + c] >= 0) {
          src[cnt] = P.tile_src[i * TT + c];
          col[cnt] = (uint8_t)c;
          ++cnt;
        }
      for (int j = 0; j < TT; ++j) {
        P.tile_src[i * TT + j] = j < cnt ? src[j] : -1;
        P.tile_cols[i * TT + j] = j < cnt ? col[j] : 0;
      }
      P.tile_cnt[i] = (uint8_t)cnt;
      if (i > P.tile_kptr[tl] && P.tile_cnt[i - 1] == cnt &&
          std::equal(P.tile_cols.begin() + i * TT, P.tile_cols.begin() + i * TT + cnt,
                     P.tile_cols.begin() + (i - 1) * TT))
        P.tile_same[i] = 1;
      const M2LSplit sp = m2l_split(cnt, m2l_gauss(P.n_pad));
      exec += 3 * sp.a3 + 2 * sp.ao;
    }
  }
  P.m2l_units_exec = exec;
  if (mdbg) {
    int64_t g8 = 0, g16 = 0;
    for (int64_t i = 0; i < tot; ++i) {
      unsigned m8 = 0, m16 = 0;
      for (int j = 0; j < P.tile_cnt[i]; ++j) {
        m8 |= 1u << (P.tile_cols[i * TT + j] / 8);
        m16 |= 1u << (P.tile_cols[i * TT + j] / 16);
      }
      g8 += __builtin_popcount(m8);
      g16 += __builtin_popcount(m16);
    }
    std::fprintf(stderr, "[m2l] present 8-target groups %lld (of %lld), 16-target groups %lld (of %lld)\n", (long long)g8,
                 (long long)(tot * (TT / 8)), (long long)g16, (long long)(tot * std::max(1, TT / 16)));
    int64_t hist[257] = {0};
    for (int64_t i = 0; i < tot; ++i) hist[P.tile_cnt[i]]++;
    std::fprintf(stderr, "[m2l] tiles %lld  tile-keys %lld  units %lld  cnt histogram:", (long long)ntile,
                 (long long)tot, (long long)P.m2l_units_exec);
    for (int c = 1; c <= TT; ++c) std::fprintf(stderr, " %d:%.3f", c, (double)hist[c] / (double)std::max<int64_t>(1, tot));
    std::fprintf(stderr, "\n");
  }
  MTICK("compaction");
  // Hybrid (int8, one rhs): (tile, key) with every valid column present stay in
  // the target tiles; the pairs of the partial ones go to the key-major pair part
  // (appended below) -- no absent column is issued in either part.  Chosen when
  // the issued columns shrink by more than the pair part's lower rate costs.
  std::vector<std::array<int32_t, 3>> hyb;
  if (P.prm.m2l_impl == 1 && R == 1) {
    std::vector<int32_t> nvalid(ntile, 0);
    for (int64_t tl = 0; tl < ntile; ++tl)
      for (int c = 0; c < TT; ++c) nvalid[tl] += P.tile_tslot[tl * TT + c] >= 0;
    // pair-part rate relative to the target tiles: the per-item epilogue and
    // pipeline refill cost ~10 stages of K per item of nch stages (measured:
    // m = 4 0.44, m = 5 0.58, m = 6 0.69 -- profiles/r02_m2l_pair_mode.jsonl, _hybrid.jsonl)
    const double nch = 2.0 * ((P.n + 15) / 16 * 16) / 32.0, rate = nch / (nch + 10.0);
    // a (tile, key) row stays in its target tile when every valid column is present,
    // or when its pairs would cost more in the pair part (cnt / rate) than the full
    // row costs in the tile (TT columns, the absent ones zero)
    auto keep = [&](int64_t i, int64_t tl) {
      return P.tile_cnt[i] == nvalid[tl] || (double)P.tile_cnt[i] >= rate * (double)TT;
    };
    int64_t full_tk = 0, part_pairs = 0;
    for (int64_t tl = 0; tl < ntile; ++tl)
      for (int64_t i = P.tile_kptr[tl]; i < P.tile_kptr[tl + 1]; ++i) {
        if (keep(i, tl)) ++full_tk;
        else part_pairs += P.tile_cnt[i];
      }
    const double c_tile = (double)tot * TT, c_hyb = (double)full_tk * TT + (double)part_pairs / rate;
    const char* hm = std::getenv("FDH_M2L_HYBRID");  // 1: force, 0: never
    const bool hybrid = part_pairs > 0 && (hm ? hm[0] == '1' : c_hyb < 0.95 * c_tile);
    if (mdbg)
      std::fprintf(stderr, "[m2l] hybrid: kept tile-keys %lld of %lld, pairs moved %lld, cost %.3g vs %.3g -> %s\n",
                   (long long)full_tk, (long long)tot, (long long)part_pairs, c_hyb, c_tile, hybrid ? "yes" : "no");
    if (hybrid) {
      hyb.reserve(part_pairs);
      std::vector<int64_t> nk(ntile + 1, 0);
      for (int64_t tl = 0; tl < ntile; ++tl) {
        for (int64_t i = P.tile_kptr[tl]; i < P.tile_kptr[tl + 1]; ++i) {
          if (keep(i, tl)) {
            ++nk[tl + 1];
            continue;
          }
          for (int j = 0; j < P.tile_cnt[i]; ++j)
            hyb.push_back({P.tile_keys[i], P.tile_tslot[tl * TT + P.tile_cols[i * TT + j]], P.tile_src[i * TT + j]});
        }
      }
      for (int64_t tl = 0; tl < ntile; ++tl) nk[tl + 1] += nk[tl];
      int64_t w = 0;  // compact the kept (tile, key) rows in place (order preserved)
      for (int64_t tl = 0; tl < ntile; ++tl)
        for (int64_t i = P.tile_kptr[tl]; i < P.tile_kptr[tl + 1]; ++i) {
          if (!keep(i, tl)) continue;
          if (w != i) {
            P.tile_keys[w] = P.tile_keys[i];
            P.tile_cnt[w] = P.tile_cnt[i];
            P.tile_same[w] = P.tile_same[i];
            std::copy(P.tile_src.begin() + i * TT, P.tile_src.begin() + (i + 1) * TT, P.tile_src.begin() + w * TT);
            std::copy(P.tile_cols.begin() + i * TT, P.tile_cols.begin() + (i + 1) * TT, P.tile_cols.begin() + w * TT);
          }
          ++w;
        }
      P.tile_kptr.assign(nk.begin(), nk.end());
      P.tile_keys.resize(w);
      P.tile_cnt.resize(w);
      P.tile_same.resize(w);
      P.tile_src.resize(w * TT);
      P.tile_cols.resize(w * TT);
    }
  }
  // Work items = (tile, global key chunk), launched chunk-major: the CTAs in
  // flight at any moment all work inside ~one chunk of key ids, so each
  // coupling matrix is read from HBM about once and then served from L2 to
  // every tile that uses it.  Chunk width: ~12 MB of coupling matrices.  The
  // items of one tile are chained in chunk order (item_seq) by the kernel.
  // int8 digits (k_m2l_i8): 7 x ceil(n/128) x 128 x 2 n_kq bytes per key; longer
  // items amortise its per-item TMEM epilogue (config 2: 12 MB 30.2 ms, 24-48 MB 29.1 ms)
  const int nkq = (P.n + 15) / 16 * 16;
  const int64_t wbytes = P.prm.m2l_impl == 1 ? (int64_t)P.prm.i8_digits * ((P.n + 127) / 128) * 128 * 2 * nkq
                                              : (int64_t)P.n_pad * m2l_wplanes(P.n_pad) * P.n_k * 8;
  // int8: 48 MB (profiles/r02_m2l_sweep_tt_chunk.jsonl: 2-3 % faster than 24 MB on configs 3, 5
  // and the m = 6 shape); DMMA: optimum 8-12 MB (profiles/r01_m2l_chunk_sweep.txt)
  int64_t chunk_mb = P.prm.m2l_impl == 1 ? 48 : 12;
  const char* cme = std::getenv("FDH_M2L_CHUNK_MB");  // tuning knob
  if (cme) chunk_mb = std::max(1L, std::atol(cme));
  int64_t cw = std::max<int64_t>(16, (chunk_mb << 20) / wbytes);
  // int8: a chunk wider than the exact-int32 key bound F splits every (tile, chunk) into
  // items of F and (chunk - F) keys; one item per (tile, chunk) measured 11 % faster at
  // m = 5 (chunk 73 -> 48 keys: config 3 M2L 1317 -> 1168 ms) and 6 % at m = 4 (256 -> 85
  // keys: config 2 23.5 -> 22.2 ms); m = 6 has 31 = F keys per 48 MB chunk already
  // (profiles/r02_m2l_chunk_vs_fkeys.jsonl)
  if (!cme && P.prm.m2l_impl == 1 && P.prm.m2l_fkeys > 0) cw = std::min<int64_t>(cw, P.prm.m2l_fkeys);
  P.m2l_chunk = cw;
  std::vector<std::array<int64_t, 4>> items;  // chunk, tile, k0, k1
  const int64_t fk = P.prm.m2l_fkeys > 0 ? P.prm.m2l_fkeys : INT64_MAX;  // k_m2l_i8: exact int32 sums
  for (int64_t tl = 0; tl < ntile; ++tl) {
    int64_t j = P.tile_kptr[tl];
    const int64_t e = P.tile_kptr[tl + 1];
    while (j < e) {
      const int64_t c = P.tile_keys[j] / cw;
      int64_t k = j;
      while (k < e && P.tile_keys[k] / cw == c && k - j < fk) ++k;
      items.push_back({c, tl, j, k});
      j = k;
    }
  }
  std::sort(items.begin(), items.end());
  P.item_tile.resize(items.size());
  P.item_seq.resize(items.size());
  P.item_k0.resize(items.size());
  P.item_k1.resize(items.size());
  P.tile_nitem.assign(ntile, 0);
  for (size_t i = 0; i < items.size(); ++i) {
    const int64_t tl = items[i][1];
    P.item_tile[i] = (int32_t)tl;
    P.item_seq[i] = P.tile_nitem[tl]++;
    P.item_k0[i] = items[i][2];
    P.item_k1[i] = items[i][3];
  }
  MTICK("items");
  // inside every item, order the keys by column map (then key id): runs of keys
  // with the same map accumulate in registers without a flush (k_m2l_gemm)
  {
    const int64_t ni = (int64_t)P.item_tile.size();
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < ni; ++i) {
      const int64_t b = P.item_k0[i], e = P.item_k1[i];
      if (e - b < 2) continue;
      std::vector<int64_t> ord(e - b);
      for (int64_t j = b; j < e; ++j) ord[j - b] = j;
      auto key_of = [&](int64_t j) {
        return std::make_tuple(P.tile_cnt[j],
                               std::string((const char*)&P.tile_cols[j * TT], (size_t)P.tile_cnt[j]),
                               P.tile_keys[j]);
      };
      std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return key_of(x) > key_of(y); });
      std::vector<int32_t> keys(e - b), src((e - b) * TT);
      std::vector<uint8_t> cols((e - b) * TT), cnt(e - b);
      for (int64_t q = 0; q < e - b; ++q) {
        const int64_t j = ord[q];
        keys[q] = P.tile_keys[j];
        cnt[q] = P.tile_cnt[j];
        std::copy(P.tile_src.begin() + j * TT, P.tile_src.begin() + (j + 1) * TT, src.begin() + q * TT);
        std::copy(P.tile_cols.begin() + j * TT, P.tile_cols.begin() + (j + 1) * TT, cols.begin() + q * TT);
      }
      for (int64_t q = 0; q < e - b; ++q) {
        P.tile_keys[b + q] = keys[q];
        P.tile_cnt[b + q] = cnt[q];
        std::copy(src.begin() + q * TT, src.begin() + (q + 1) * TT, P.tile_src.begin() + (b + q) * TT);
        std::copy(cols.begin() + q * TT, cols.begin() + (q + 1) * TT, P.tile_cols.begin() + (b + q) * TT);
      }
      for (int64_t j = b; j < e; ++j)
        P.tile_same[j] = j > b && P.tile_cnt[j - 1] == P.tile_cnt[j] &&
                         std::equal(P.tile_cols.begin() + j * TT, P.tile_cols.begin() + j * TT + P.tile_cnt[j],
                                    P.tile_cols.begin() + (j - 1) * TT);
    }
  }
  MTICK("item map sort");
  if (mdbg) {
    int64_t flushes = 0;
    for (size_t i = 0; i < P.item_k0.size(); ++i)
      for (int64_t j = P.item_k0[i]; j < P.item_k1[i]; ++j) flushes += (j == P.item_k0[i] || !P.tile_same[j]);
    std::fprintf(stderr, "[m2l] items %lld  column-map runs %lld (%.2f keys per run)\n", (long long)P.item_k0.size(),
                 (long long)flushes, (double)tot / (double)std::max<int64_t>(1, flushes));
  }
  if (!hyb.empty()) {
    append_pair_part(P, hyb, TT);
    MTICK("hybrid pairs");
  }
  // target slots with no M2L contribution
  for (int64_t t = 0; t < T.nslots; ++t)
    if (ptr[t + 1] == ptr[t]) P.m2l_zero_slots.push_back((int32_t)t);
  MTICK("end");
#undef MTICK
}

}  // namespace

int num_dirs(int level, int lhf) { return level > lhf ? 1 : (6 << (2 * (lhf - level))); }

// Def. 3 with closed cells and the min-j rule: first argmax
// axis selects the main face (-x,+x,-y,+y,-z,+z); then, per subdivision, the
// lower half whenever the in-face coordinate v_u / M is <= the cell midpoint.
int dir_map_vec(int level, int lhf, const double v[3]) {
  if (level > lhf) return 0;
  int a = 0;
  double M = std::fabs(v[0]);
  for (int i = 1; i < 3; ++i)
    if (std::fabs(v[i]) > M) { M = std::fabs(v[i]); a = i; }
  if (M == 0.0) return 0;
  const int u = (a == 0) ? 1 : 0, w = (a == 2) ? 1 : 2;
  const double cu = v[u] / M, cw = v[w] / M;
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

// Alg. 3: normalized midpoint of the face cell of index idx at level.
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
  const double nn = norm3(p);
  for (int i = 0; i < 3; ++i) out[i] = (1.0 / nn) * p[i];
}

// Ownership of target leaves for sharded runs: leaves in
// Morton order, split into `world` contiguous ranges of equal estimated cost,
// cost(leaf) = sum over the leaf and its ancestors a of
//   (8 n^2 * #L+(a) + 24 * near-field pairs(a)) * points(leaf) / points(a);
// then the ancestor closure of the owned leaves (t_needed).  #L+ per target node
// comes from P.lp_count when the partition was built on the GPU (the L+ lists are
// then compacted to t_needed on the device before they reach the host), else from
// the host lists.
void compute_ownership(Plan& P) {
  const PlanParams& prm = P.prm;
  const TreePlan& T = P.T;
  const int D = T.depth;
  std::vector<std::vector<double>> own(D + 1);
  for (int l = 0; l <= D; ++l) own[l].assign(T.lv[l].size(), 0.0);
  const double fl_m2l = 8.0 * P.n * P.n;
  for (int l = 0; l < (int)P.blocks.size(); ++l) {
    const LevelBlocks& B = P.blocks[l];
    if (l < (int)P.lp_count.size() && !P.lp_count[l].empty()) {
      for (size_t i = 0; i < P.lp_count[l].size(); ++i) own[l][i] += fl_m2l * P.lp_count[l][i];
    } else {
      for (size_t b = 0; b < B.lp_t.size(); ++b) own[l][B.lp_t[b]] += fl_m2l;
    }
    for (size_t b = 0; b < B.lm_t.size(); ++b)
      own[l][B.lm_t[b]] += 24.0 * (double)(T.lv[l].end[B.lm_t[b]] - T.lv[l].begin[B.lm_t[b]]) *
                           (double)(P.S.lv[l].end[B.lm_s[b]] - P.S.lv[l].begin[B.lm_s[b]]);
  }
  // push ancestor cost down by point share: dens[l][i] = cost per point inherited
  std::vector<std::vector<double>> dens(D + 1);
  for (int l = 0; l <= D; ++l) {
    dens[l].assign(T.lv[l].size(), 0.0);
    for (size_t i = 0; i < T.lv[l].size(); ++i) {
      const double pts = (double)(T.lv[l].end[i] - T.lv[l].begin[i]);
      const double inh = l > 0 ? dens[l - 1][T.lv[l].parent[i]] : 0.0;
      dens[l][i] = inh + own[l][i] / pts;
    }
  }
  // Morton key of the leaf's lower corner at the deepest level: 3 bits per level,
  // 128-bit so that any depth up to the cap keeps the spatial order
  struct LeafRef { unsigned __int128 key; int64_t id; double c; };
  std::vector<LeafRef> lr;
  int64_t id = 0;
  for (int l = 0; l <= D; ++l)
    for (size_t i = 0; i < T.lv[l].size(); ++i) {
      if (!T.lv[l].leaf[i]) continue;
      unsigned __int128 k = 0;
      const int64_t ci = T.lv[l].ci[i] << (D - l), cj = T.lv[l].cj[i] << (D - l), ck = T.lv[l].ck[i] << (D - l);
      for (int b = D - 1; b >= 0; --b)
        k = (k << 3) | (unsigned)((((ci >> b) & 1) << 2) | (((cj >> b) & 1) << 1) | ((ck >> b) & 1));
      const double pts = (double)(T.lv[l].end[i] - T.lv[l].begin[i]);
      lr.push_back({k, id++, dens[l][i] * pts + 1.0});
    }
  std::sort(lr.begin(), lr.end(), [](const LeafRef& a, const LeafRef& b) { return a.key < b.key; });
  double tot = 0;
  for (auto& r : lr) tot += r.c;
  P.t_leaf_owned.assign(id, 0);
  P.shard_cost = 0.0;
  double acc = 0;
  for (auto& r : lr) {
    const double mid = acc + 0.5 * r.c;
    const int owner = std::min(prm.world - 1, (int)(mid / tot * prm.world));
    if (owner == prm.rank) {
      P.t_leaf_owned[r.id] = 1;
      P.shard_cost += r.c;
    }
    acc += r.c;
  }
  P.total_cost = tot;
  // ancestor closure of the owned leaves (leaf ids in (level, Morton) order)
  P.t_needed.assign(P.T.depth + 1, {});
  for (int l = 0; l <= P.T.depth; ++l) P.t_needed[l].assign(P.T.lv[l].size(), 0);
  int64_t lid = 0;
  for (int l = 0; l <= P.T.depth; ++l)
    for (size_t i = 0; i < P.T.lv[l].size(); ++i) {
      if (!P.T.lv[l].leaf[i]) continue;
      if (P.t_leaf_owned[lid++]) {
        int32_t nid = (int32_t)i;
        for (int ll = l; ll >= 0 && !P.t_needed[ll][nid]; --ll) {
          P.t_needed[ll][nid] = 1;
          nid = P.T.lv[ll].parent[nid];
          if (nid < 0) break;
        }
      }
    }
}

void build_plan(Plan& P, const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                const double* sy, const double* sz, int64_t ns, const double lo[3], const double hi[3],
                const PlanParams& prm) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!(prm.kappa > 0.0) || !std::isfinite(prm.kappa)) fail(1, "wave number must be positive and finite");
  if (prm.m < 0 || prm.m > 10) fail(1, "interpolation degree must be in [0, 10]");
  if (!(prm.eta2 > 0.0)) fail(1, "eta2 must be positive");
  if (prm.l_hf < -2) fail(1, "l_hf must be >= -1 (or -2 for the default rule)");
  if (prm.depth_cap < 0) fail(1, "depth_cap must be >= 0");
  P.prm = prm;
  P.p = prm.m + 1;
  P.n = P.p * P.p * P.p;
  P.n_pad = (P.n + 31) / 32 * 32;
  P.n_k = (P.n + 7) / 8 * 8;
  const auto t1 = std::chrono::steady_clock::now();
  nvtxRangePushA("fdh:setup:structure");
  if (prm.gpu_structure) {
    // trees, partition, key directions, D / D^ and slots on the device (k_setup.cu)
    gpu_build_structure(P, tx, ty, tz, nt, sx, sy, sz, ns, lo, hi);
  } else {
    build_tree(P.T, tx, ty, tz, nt, lo, hi, prm.n_max, prm.depth_cap);
    build_tree(P.S, sx, sy, sz, ns, lo, hi, prm.n_max, prm.depth_cap);
    // l_hf default
    P.lhf = prm.l_hf;
    if (P.lhf == -2) {
      P.lhf = -1;
      for (int l = 0; l <= std::min(P.T.depth, P.S.depth); ++l)
        if (prm.kappa * std::max(P.T.diam[l], P.S.diam[l]) >= 3.0) P.lhf = l;
    }
    const double mn = std::min({P.T.side[0][0], P.T.side[0][1], P.T.side[0][2]});
    for (int a = 0; a < 3; ++a) P.rho[a] = P.T.side[0][a] / mn;
    build_blocks(P);
    build_keys(P);
    build_dirsets(P, P.T, true);
    build_dirsets(P, P.S, false);
  }
  nvtxRangePop();
  P.structure_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
  // direction vector tables
  const int maxl = std::max(P.T.depth, P.S.depth);
  P.dirvec.assign(maxl + 1, {});
  for (int l = 0; l <= maxl; ++l) {
    const int nd = num_dirs(l, P.lhf);
    P.dirvec[l].resize(3 * nd);
    for (int j = 0; j < nd; ++j) dir_vec(l, P.lhf, j, &P.dirvec[l][3 * j]);
  }
  // interpolation constants (interpolation.cpp:9-20, 89-99)
  P.cheb_cos.resize(P.p);
  for (int nu = 1; nu <= P.p; ++nu) P.cheb_cos[nu - 1] = std::cos((2.0 * nu - 1.0) * kPi / (2.0 * P.p));
  {
    auto nodes = [&](double a, double b) {
      std::vector<double> x(P.p);
      const double mid = 0.5 * (a + b), half = 0.5 * (b - a);
      for (int i = 0; i < P.p; ++i) x[i] = mid + half * P.cheb_cos[i];
      return x;
    };
    const auto par = nodes(0.0, 1.0);
    P.half.assign(2 * P.p * P.p, 0.0);
    for (int h = 0; h < 2; ++h) {
      const auto ch = h == 0 ? nodes(0.0, 0.5) : nodes(0.5, 1.0);
      for (int j = 0; j < P.p; ++j)
        for (int k = 0; k < P.p; ++k) {
          double v = 1.0;
          for (int q = 0; q < P.p; ++q) {
            if (q == k) continue;
            v *= (ch[j] - par[q]) / (par[k] - par[q]);
          }
          P.half[(h * P.p + j) * P.p + k] = v;
        }
    }
  }
  if (prm.world > 1 && P.t_leaf_owned.empty()) compute_ownership(P);
  auto tick = [&](const char* what, std::chrono::steady_clock::time_point& ts) {
    const auto now = std::chrono::steady_clock::now();
    if (std::getenv("FDH_DEBUG_SETUP"))
      std::fprintf(stderr, "[setup] %-12s %9.1f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - ts).count());
    ts = now;
  };
  auto ts = std::chrono::steady_clock::now();
  if (std::getenv("FDH_DEBUG_SETUP"))
    std::fprintf(stderr, "[setup] structure    %9.1f ms\n", P.structure_ms);
  nvtxRangePushA("fdh:setup:worklists");
  build_worklists(P);
  nvtxRangePop();
  tick("worklists", ts);
  nvtxRangePushA("fdh:setup:m2l_tiles");
  build_m2l(P);
  nvtxRangePop();
  tick("m2l tiles", ts);
  // statistics
  for (auto& B : P.blocks) {
    P.n_lminus += (int64_t)B.lm_t.size();
  }
  for (int l = 0; l < (int)P.blocks.size(); ++l) {
    const LevelBlocks& B = P.blocks[l];
    int64_t ext[3] = {0, 0, 0};  // max |lattice offset| per axis over the L- blocks of the level
    for (size_t b = 0; b < B.lm_t.size(); ++b) {
      P.m_d += (int64_t)(P.T.lv[l].end[B.lm_t[b]] - P.T.lv[l].begin[B.lm_t[b]]) *
               (int64_t)(P.S.lv[l].end[B.lm_s[b]] - P.S.lv[l].begin[B.lm_s[b]]);
      ext[0] = std::max(ext[0], (int64_t)std::llabs((long long)(P.T.lv[l].ci[B.lm_t[b]] - P.S.lv[l].ci[B.lm_s[b]])));
      ext[1] = std::max(ext[1], (int64_t)std::llabs((long long)(P.T.lv[l].cj[B.lm_t[b]] - P.S.lv[l].cj[B.lm_s[b]])));
      ext[2] = std::max(ext[2], (int64_t)std::llabs((long long)(P.T.lv[l].ck[B.lm_t[b]] - P.S.lv[l].ck[B.lm_s[b]])));
    }
    if (!B.lm_t.empty()) {  // points of boxes at lattice offset d are at most (|d|+1) sides apart per axis
      double d2 = 0.0;
      for (int a = 0; a < 3; ++a) {
        const double w = (double)(ext[a] + 1) * P.T.side[l][a];
        d2 += w * w;
      }
      P.nf_max_dist = std::max(P.nf_max_dist, 1.0001 * std::sqrt(d2));
    }
  }
  for (int w = 0; w < 2; ++w) {
    const TreePlan& X = w == 0 ? P.T : P.S;
    for (int l = 0; l <= X.depth; ++l) {
      const int nd = X.ndir[l];
      for (size_t i = 0; i < X.lv[l].size(); ++i) {
        int64_t k = 0;
        for (int c = 0; c < nd; ++c) k += X.kind[l][i * nd + c] != 0;
        if (X.lv[l].leaf[i]) {
          P.n_le += k;
        } else {
          int nch = 0;
          for (int o = 0; o < 8; ++o) nch += X.lv[l].child[i * 8 + o] >= 0;
          P.n_le += k * nch;
        }
      }
    }
  }
  P.setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// ------------------------------------------------------------------ exports
namespace {
struct Row7 { int64_t v[7]; };
}

int64_t export_tree(const TreePlan& T, int64_t* rows) {
  int64_t n = 0;
  for (auto& L : T.lv) n += (int64_t)L.size();
  if (!rows) return n;
  std::vector<std::array<int64_t, 7>> r;
  r.reserve(n);
  for (int l = 0; l <= T.depth; ++l) {
    const LevelNodes& L = T.lv[l];
    for (size_t i = 0; i < L.size(); ++i) r.push_back({l, L.ci[i], L.cj[i], L.ck[i], L.begin[i], L.end[i], L.leaf[i]});
  }
  std::sort(r.begin(), r.end());
  std::memcpy(rows, r.data(), sizeof(int64_t) * 7 * n);
  return n;
}
int64_t export_perm(const TreePlan& T, int64_t* out) {
  if (out)
    for (size_t i = 0; i < T.perm.size(); ++i) out[i] = T.perm[i];
  return (int64_t)T.perm.size();
}
int64_t export_lplus(const Plan& P, int64_t* rows) {
  int64_t n = 0;
  for (auto& B : P.blocks) n += (int64_t)B.lp_t.size();
  if (!rows) return n;
  std::vector<std::array<int64_t, 8>> r;
  r.reserve(n);
  for (int l = 0; l < (int)P.blocks.size(); ++l) {
    const LevelBlocks& B = P.blocks[l];
    const LevelNodes& LT = P.T.lv[l];
    const LevelNodes& LS = P.S.lv[l];
    for (size_t b = 0; b < B.lp_t.size(); ++b)
      r.push_back({l, LT.ci[B.lp_t[b]], LT.cj[B.lp_t[b]], LT.ck[B.lp_t[b]], LS.ci[B.lp_s[b]], LS.cj[B.lp_s[b]],
                   LS.ck[B.lp_s[b]], P.key_dir[B.lp_key[b]]});
  }
  std::sort(r.begin(), r.end());
  std::memcpy(rows, r.data(), sizeof(int64_t) * 8 * n);
  return n;
}
int64_t export_lminus(const Plan& P, int64_t* rows) {
  int64_t n = 0;
  for (auto& B : P.blocks) n += (int64_t)B.lm_t.size();
  if (!rows) return n;
  std::vector<std::array<int64_t, 8>> r;
  r.reserve(n);
  for (int l = 0; l < (int)P.blocks.size(); ++l) {
    const LevelBlocks& B = P.blocks[l];
    const LevelNodes& LT = P.T.lv[l];
    const LevelNodes& LS = P.S.lv[l];
    for (size_t b = 0; b < B.lm_t.size(); ++b)
      r.push_back({l, LT.ci[B.lm_t[b]], LT.cj[B.lm_t[b]], LT.ck[B.lm_t[b]], l, LS.ci[B.lm_s[b]], LS.cj[B.lm_s[b]],
                   LS.ck[B.lm_s[b]]});
  }
  std::sort(r.begin(), r.end());
  std::memcpy(rows, r.data(), sizeof(int64_t) * 8 * n);
  return n;
}
// Order-independent 64-bit digests of the canonical exports (sum of splitmix64
// of each row), for configurations whose lists are too large to export
// (config 4: 3.47e9 admissible blocks).  out: T tree, S tree, L+, L-, D/D^ (T), D/D^ (S).
namespace {
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
}  // namespace

void structure_digest(const Plan& P, uint64_t out[6]) {
  for (int i = 0; i < 6; ++i) out[i] = 0;
  for (int w = 0; w < 2; ++w) {
    const TreePlan& T = w == 0 ? P.T : P.S;
    uint64_t acc = 0;
    for (int l = 0; l <= T.depth; ++l) {
      const LevelNodes& L = T.lv[l];
      for (size_t i = 0; i < L.size(); ++i) {
        const int64_t r[7] = {l, L.ci[i], L.cj[i], L.ck[i], L.begin[i], L.end[i], L.leaf[i]};
        acc += row_hash(r, 7);
      }
    }
    for (size_t sl = 0; sl < T.perm.size(); ++sl) {
      const int64_t r[2] = {(int64_t)sl, (int64_t)T.perm[sl]};
      acc += row_hash(r, 2);
    }
    out[w] = acc;
    uint64_t dacc = 0;
    for (int l = 0; l <= T.depth; ++l) {
      const int nd = T.ndir[l];
      const LevelNodes& L = T.lv[l];
      for (size_t i = 0; i < L.size(); ++i)
        for (int c = 0; c < nd; ++c) {
          const uint8_t k = T.kind[l][i * nd + c];
          if (!k) continue;
          const int64_t r[6] = {l, L.ci[i], L.cj[i], L.ck[i], c, k};
          dacc += row_hash(r, 6);
        }
    }
    out[4 + w] = dacc;
  }
  uint64_t lp = 0, lm = 0;
  for (int l = 0; l < (int)P.blocks.size(); ++l) {
    const LevelBlocks& B = P.blocks[l];
    const LevelNodes& LT = P.T.lv[l];
    const LevelNodes& LS = P.S.lv[l];
    uint64_t a = 0;
    // (the digest of the full list is taken on the device when it was built there)
    const int64_t nlp = P.lplus_digest_dev ? 0 : (int64_t)B.lp_t.size();
#pragma omp parallel for reduction(+ : a)
    for (int64_t b = 0; b < nlp; ++b) {
      const int64_t r[8] = {l, LT.ci[B.lp_t[b]], LT.cj[B.lp_t[b]], LT.ck[B.lp_t[b]], LS.ci[B.lp_s[b]], LS.cj[B.lp_s[b]],
                            LS.ck[B.lp_s[b]], P.key_dir[B.lp_key[b]]};
      a += row_hash(r, 8);
    }
    lp += a;
    for (size_t b = 0; b < B.lm_t.size(); ++b) {
      const int64_t r[8] = {l, LT.ci[B.lm_t[b]], LT.cj[B.lm_t[b]], LT.ck[B.lm_t[b]], l, LS.ci[B.lm_s[b]],
                            LS.cj[B.lm_s[b]], LS.ck[B.lm_s[b]]};
      lm += row_hash(r, 8);
    }
  }
  out[2] = P.lplus_digest_dev ? P.lplus_digest : lp;
  out[3] = lm;
}

int64_t export_owned_leaves(const Plan& P, int64_t* rows) {
  int64_t n = (int64_t)P.l2t_level.size();
  if (!rows) return n;
  std::vector<std::array<int64_t, 6>> r(n);
  for (int64_t i = 0; i < n; ++i)
    r[i] = {P.l2t_level[i], P.l2t_ci[i], P.l2t_cj[i], P.l2t_ck[i], P.l2t_begin[i], P.l2t_end[i]};
  std::sort(r.begin(), r.end());
  std::memcpy(rows, r.data(), sizeof(int64_t) * 6 * n);
  return n;
}

int64_t export_dirsets(const Plan& P, int which, int64_t* rows) {
  const TreePlan& T = which == 0 ? P.T : P.S;
  if (!rows) return T.nslots;
  std::vector<std::array<int64_t, 6>> r;
  r.reserve(T.nslots);
  for (int l = 0; l <= T.depth; ++l) {
    const int nd = T.ndir[l];
    const LevelNodes& L = T.lv[l];
    for (size_t i = 0; i < L.size(); ++i)
      for (int c = 0; c < nd; ++c) {
        const uint8_t k = T.kind[l][i * nd + c];
        if (k) r.push_back({l, L.ci[i], L.cj[i], L.ck[i], c, k});
      }
  }
  std::sort(r.begin(), r.end());
  std::memcpy(rows, r.data(), sizeof(int64_t) * 6 * r.size());
  return (int64_t)r.size();
}

}  // namespace fdhelm
