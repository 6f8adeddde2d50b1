// plan.hpp -- host-side setup of the directional matvec.
//
// Builds, level-synchronously (the same data-parallel shape as the CUDA
// kernels of the apply phase, so each stage can move to the device without
// changing its output):
//   * the two uniform box cluster trees (Alg. 1; bit-exact with
//     /root/reference/proj/src/cluster_tree.cpp:12-128),
//   * the block partition L+ / L- (Alg. 2, Def. 1-2),
//   * direction indices per (level, lattice offset) key (Alg. 3, Def. 3),
//   * active / inherited direction sets and dense (box, direction) slots (Def. 4),
//   * the work lists of every apply kernel (S2M, M2M, M2L tiles, L2L, L2T, P2P).
// Nodes of a level are kept in Morton order (the generation order of the
// stable octant partition); canonical (level, i, j, k) order is produced only
// by the export functions.
#pragma once
#include "m2l_split.hpp"
#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace fdhelm {


struct PlanError {
  int code;
  std::string msg;
};

struct PlanParams {
  double kappa = 1.0;
  int n_max = 64;
  int m = 4;
  double eta2 = 1.0;
  int l_hf = -2;
  int depth_cap = 30;
  int zero_diagonal = 0;
  int tile = 16;       // M2L target slots per tile
  int m2l_impl = 0;    // 0: FP64 DMMA (k_m2l_gemm), 1: int8 tcgen05 digits (k_m2l_i8)
  int m2l_fkeys = 0;   // > 0: at most this many keys per M2L work item
  int i8_digits = 7;   // int8 M2L: digits per FP64 value (W bytes per key; set by the C-ABI layer)
  int nrhs = 1;        // right-hand sides per apply: an M2L tile
                       // column is a (target slot, rhs) pair, slot id r * nslots + slot
  int rank = 0, world = 1;
  bool gpu_structure = false;  // trees / partition / directions on the device (k_setup.cu)
};

struct LevelNodes {
  std::vector<int64_t> ci, cj, ck;  // lattice coordinates
  std::vector<uint32_t> begin, end;
  std::vector<uint8_t> leaf;
  std::vector<int32_t> parent;  // index into level-1
  std::vector<int32_t> child;   // 8 per node, index into level+1 or -1 (octant order)
  size_t size() const { return ci.size(); }
};

struct TreePlan {
  double lo[3], hi[3];  // padded root (cluster_tree.cpp:21-24)
  std::vector<std::array<double, 3>> side;
  std::vector<double> diam;
  int depth = 0, oversized = 0;
  std::vector<LevelNodes> lv;
  std::vector<uint32_t> perm;  // slot -> original index
  std::vector<double> x, y, z;  // slot order
  // direction sets / slots
  std::vector<int32_t> ndir;                 // #D^(l)
  std::vector<std::vector<uint8_t>> kind;    // [l][node*nD+dir]: 1 = D, 2 = D^
  std::vector<std::vector<int32_t>> slot_of; // [l][node*nD+dir] -> slot or -1
  int64_t nslots = 0;
  std::vector<int32_t> slot_level, slot_node, slot_dir;
  std::vector<int64_t> node_slot_first;      // per level offsets into a flat array
};

// Per-level block lists (indices into the level node arrays of T / S).
struct LevelBlocks {
  std::vector<int32_t> lp_t, lp_s, lp_key;  // L+
  std::vector<int32_t> lm_t, lm_s;          // L-
};

struct Plan {
  PlanParams prm;
  int p = 0, n = 0, n_pad = 0, n_k = 0, lhf = -1;  // n_pad: GEMM rows (32k), n_k: K half (8k)
  double rho[3] = {1, 1, 1};
  TreePlan T, S;
  std::vector<LevelBlocks> blocks;
  // keys, sorted by (level, dx, dy, dz)
  std::vector<int32_t> key_level, key_dir;
  std::vector<int64_t> key_dx, key_dy, key_dz;
  // direction vectors per level: dirvec[l][3*j + a]
  std::vector<std::vector<double>> dirvec;
  // host constants
  std::vector<double> cheb_cos;      // p values cos((2nu-1)pi/(2p))
  std::vector<double> half;          // 2 x p x p : half[h][j][k] = L_k^par(child_j)

  // ---- apply work lists (flattened, device-ready) ----
  // S2M: one entry per leaf source slot
  std::vector<int32_t> s2m_slot, s2m_level, s2m_dir;
  std::vector<int64_t> s2m_ci, s2m_cj, s2m_ck;
  std::vector<uint32_t> s2m_begin, s2m_end;
  // M2M per level l (parents at l): parent slot, dir pair, 8 child slots
  std::vector<std::vector<int32_t>> m2m_parent, m2m_dir, m2m_cdir, m2m_child;  // child: 8 per entry
  std::vector<std::vector<int64_t>> m2m_pc;  // parent coords (3 per entry)
  // L2L per level l (children at l+1): child slot, child dir, CSR of (parent slot, parent dir, octant)
  std::vector<std::vector<int32_t>> l2l_child, l2l_cdir, l2l_ptr, l2l_pslot, l2l_pdir, l2l_oct;
  std::vector<std::vector<int64_t>> l2l_cc;  // child coords (3 per entry)
  // L2T: one entry per target leaf (owned by this rank)
  std::vector<int32_t> l2t_level, l2t_slot0, l2t_nslot;
  std::vector<int64_t> l2t_ci, l2t_cj, l2t_ck;
  std::vector<uint32_t> l2t_begin, l2t_end;
  // P2P: per target leaf (same order as L2T), CSR of source slot ranges
  std::vector<int64_t> p2p_ptr;
  std::vector<uint32_t> p2p_sbeg, p2p_send;
  // M2L tiles: tile -> (level, dir, T target slots), key list CSR, source table
  std::vector<int32_t> tile_level, tile_dir;
  std::vector<int32_t> tile_tslot;   // tile * T (-1 pad)
  std::vector<int64_t> tile_kptr;    // CSR into tile_keys / tile_src
  std::vector<int32_t> tile_keys;    // key ids
  std::vector<int32_t> tile_src;     // (tile_kptr[i] + kk) * T + j: source slot of compacted column j
  std::vector<uint8_t> tile_cols;    // (tile_kptr[i] + kk) * T + j: target column of compacted column j
  std::vector<uint8_t> tile_cnt;     // per (tile, key): number of target columns that have the key
  std::vector<uint8_t> tile_same;    // per (tile, key): same column map as the previous key of the tile
  // work items (tile, key chunk), chunk-major; item_seq = rank of the item in its tile
  std::vector<int32_t> item_tile, item_seq;
  std::vector<int64_t> item_k0, item_k1;
  std::vector<int32_t> tile_nitem;
  int64_t m2l_chunk = 0;
  // pair mode (int8 M2L, clustered sources): one key per tile, columns = (target,
  // source) pairs; per target slot the pair indices (tile * tile + column) in key order
  bool m2l_pair = false;
  int64_t m2l_pair_tile0 = 0, m2l_pair_item0 = 0;  // first pair tile / item (hybrid: after the target tiles)
  std::vector<int64_t> red_ptr;
  std::vector<int64_t> red_idx;
  // target slots without any M2L contribution (to be zeroed)
  std::vector<int32_t> m2l_zero_slots;
  // rank ownership of targets (all by default)
  std::vector<uint8_t> t_leaf_owned;
  std::vector<std::vector<uint8_t>> t_needed;  // [level][node]: owned leaf or ancestor of one
  double shard_cost = 0.0, total_cost = 0.0;     // estimated flops of this shard / of all targets
  double nf_max_dist = 0.0;  // upper bound of |x_j - y_k| over the near-field pairs
  // GPU partition (k_setup.cu): #L+ per target node per level (shard cost model),
  // the L+ digest of the FULL list (the host keeps only the t_needed part on shards)
  std::vector<std::vector<int32_t>> lp_count;
  uint64_t lplus_digest = 0;
  bool lplus_digest_dev = false;

  // statistics
  int64_t n_c = 0, n_sc = 0, m_d = 0, n_le = 0, n_lminus = 0;
  int64_t m2l_units_exec = 0;  // issued DMMA work in M2LSplit units (16 n_pad n_k flop each)
  double setup_ms = 0.0;
  double structure_ms = 0.0;  // trees + partition + directions + slots
};

// Throws PlanError.
void build_plan(Plan& plan, const double* tx, const double* ty, const double* tz, int64_t nt,
                const double* sx, const double* sy, const double* sz, int64_t ns, const double lo[3],
                const double hi[3], const PlanParams& prm);

int64_t export_tree(const TreePlan& T, int64_t* rows);
int64_t export_perm(const TreePlan& T, int64_t* out);
int64_t export_lplus(const Plan& P, int64_t* rows);
int64_t export_lminus(const Plan& P, int64_t* rows);
int64_t export_dirsets(const Plan& P, int which, int64_t* rows);
int64_t export_owned_leaves(const Plan& P, int64_t* rows);
void structure_digest(const Plan& P, uint64_t out[6]);
// shard ownership (cost-balanced Morton ranges of target leaves) + t_needed
void compute_ownership(Plan& P);

// direction conventions
int num_dirs(int level, int lhf);
int dir_map_vec(int level, int lhf, const double v[3]);
void dir_vec(int level, int lhf, int idx, double out[3]);
inline int parent_dir(int level, int lhf, int j) { return (level + 1 > lhf) ? 0 : (j >> 2); }

}  // namespace fdhelm
