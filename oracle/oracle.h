/*
 * oracle.h -- CPU oracle for the directional multi-level Helmholtz matvec.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker: it may be
 * loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg, never by the product path (paper_2004_14229_b200/).
 *
 * It restates, on the CPU and in plain C++ (OpenMP over targets),
 * the reference's algorithm for the hot path:
 *   Alg. 1 cluster tree          /root/reference/proj/src/cluster_tree.cpp:12-128
 *   Chebyshev interpolation      /root/reference/proj/src/interpolation.cpp:9-131
 *   Alg. 3 / Def. 3 directions
 *   Alg. 2 / Def. 1-2 blocks
 *   Def. 4 direction sets
 *   Eq. 9 coupling (canonical)
 *   Alg. 4 matvec
 *   dense oracle
 * The conventions the reference leaves open are pinned as in SURVEY.md App. B
 * and DESIGN.md section 3.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_op orc_op;

/* Stats layout of orc_stats (int64 array, ORC_NSTATS entries). */
enum {
  ORC_N_C = 0,       /* #L+ (applied coupling matrices)              */
  ORC_N_SC = 1,      /* distinct (level, offset) keys                */
  ORC_M_D = 2,       /* near-field entries sum #t*#s over L-         */
  ORC_N_LE = 3,      /* applied transfer + interpolation matrices    */
  ORC_N_LMINUS = 4,  /* #L- blocks                                   */
  ORC_DEPTH_T = 5,
  ORC_DEPTH_S = 6,
  ORC_L_HF = 7,
  ORC_SLOTS_T = 8,   /* sum over target boxes of |D u D^|            */
  ORC_SLOTS_S = 9,
  ORC_NODES_T = 10,
  ORC_NODES_S = 11,
  ORC_M_D_ZERO = 12, /* skipped diagonal pairs (zero_diagonal)       */
  ORC_NSTATS = 13
};

/* Returns 0 on success; nonzero error code, message via orc_last_error(). */
int orc_create(const double* tx, const double* ty, const double* tz, int64_t nt,
               const double* sx, const double* sy, const double* sz, int64_t ns,
               const double root_lo[3], const double root_hi[3], double kappa, int n_max,
               int m, double eta2, int l_hf, int depth_cap, int zero_diagonal, orc_op** out);
/* Structure only (trees, blocks, directions, stats); no coupling matrices. */
int orc_create_structure(const double* tx, const double* ty, const double* tz, int64_t nt,
                         const double* sx, const double* sy, const double* sz, int64_t ns,
                         const double root_lo[3], const double root_hi[3], double kappa,
                         int n_max, int m, double eta2, int l_hf, int depth_cap,
                         int zero_diagonal, orc_op** out);
/* Sampled-structure operator for sizes whose full L+ / coupling set does not fit
 * in host memory (config 4): trees in full, block partition only below the target
 * boxes on the paths root -> sampled leaf (leaf_idx in canonical leaf order),
 * moments only for the (box, direction) slots those blocks need, coupling
 * matrices generated per block.  orc_apply_sampled with the same leaves gives the
 * same values as a full operator's orc_apply_sampled. */
int orc_create_sampled(const double* tx, const double* ty, const double* tz, int64_t nt,
                       const double* sx, const double* sy, const double* sz, int64_t ns,
                       const double lo[3], const double hi[3], double kappa, int n_max, int m,
                       double eta2, int l_hf, int depth_cap, int zero_diagonal,
                       const int64_t* leaf_idx, int64_t nleaf, orc_op** out);
void orc_destroy(orc_op* op);
/* Streaming structure digest (no block lists stored; config 4 has 3.47e9 L+
 * blocks): both trees, then Alg. 2 depth-first in parallel, hashing every L+ /
 * L- block where it is classified.  out6 = order-independent sums of a
 * splitmix64 row hash over the canonical export rows: [T tree + perm, S tree +
 * perm, L+, L-, D/D^ of T, D/D^ of S] (the layout fdh_structure_digest uses).
 * counts[11] = N_C, N_SC, #L-, M_D, nodes_T, nodes_S, slots_T, slots_S,
 * depth_T, depth_S, l_hf.  m is unused (the structure does not depend on it). */
int orc_structure_digest(const double* tx, const double* ty, const double* tz, int64_t nt,
                         const double* sx, const double* sy, const double* sz, int64_t ns,
                         const double root_lo[3], const double root_hi[3], double kappa, int n_max,
                         int m, double eta2, int l_hf, int depth_cap, uint64_t* out6,
                         int64_t* counts);
const char* orc_last_error(void);
int orc_set_threads(int n);

/* y = A x, complex128 interleaved, both in ORIGINAL point order. */
int orc_apply(orc_op* op, const double* x, double* y);
/* Sampled-target mode: only the target leaves listed (node ids of the target
 * tree in canonical leaf order index, see orc_export_leaves) get M2L/L2L/L2T/P2P.
 * y is written only for the points of those leaves (others left untouched). */
int orc_apply_sampled(orc_op* op, const double* x, const int64_t* leaf_idx, int64_t nleaf,
                      double* y);
/* Number of leaves of a tree (0=targets, 1=sources) and, for leaf i in
 * (level, coord) order, its original point indices. */
int64_t orc_leaf_count(const orc_op* op, int which);
int64_t orc_leaf_points(const orc_op* op, int which, int64_t leaf, int64_t* idx, int64_t cap);

int orc_stats(const orc_op* op, int64_t* out /* ORC_NSTATS */);
/* ACA-compressed coupling: eps > 0 compresses every stored
 * coupling matrix by partially pivoted ACA (A ~ U V^*; dense kept where 2 k n >=
 * n^2) and the M2L applies the factors; eps = 0 restores the dense M2L. */
int orc_set_aca(orc_op* op, double eps);
/* per-key ACA rank (0 = dense); returns the key count */
int64_t orc_aca_ranks(const orc_op* op, int32_t* out);
/* aca_compress on one n x n complex row-major matrix: returns k (0 = dense) and
 * U (n x k complex, column-major), W = V^* (k x n complex, row-major) */
int orc_aca_compress(const double* A, int n, double eps, int max_rank, double* U, double* W);
/* Wall seconds of the last apply: [0] upward pass (S2M + M2M), [1] coupling
 * matrix generation (sampled-structure mode: once per key used), [2] M2L
 * products, [3] L2L + L2T + near field; [4] = coupling matrices generated. */
int orc_last_timing(const orc_op* op, double* out5);

/* Canonical exports.  Each returns the row count; pass
 * out == NULL to query.  Rows are int64 and sorted lexicographically. */
/* tree rows: level, i, j, k, begin, end, leaf                       (7 cols) */
int64_t orc_export_tree(const orc_op* op, int which, int64_t* out);
/* slot -> original index permutation (n entries)                             */
int64_t orc_export_perm(const orc_op* op, int which, int64_t* out);
/* L+ rows: level, ti, tj, tk, si, sj, sk, dir                        (8 cols) */
int64_t orc_export_lplus(const orc_op* op, int64_t* out);
/* L- rows: tlevel, ti, tj, tk, slevel, si, sj, sk                    (8 cols) */
int64_t orc_export_lminus(const orc_op* op, int64_t* out);
/* dirset rows: level, i, j, k, dir, kind (1=D, 2=D^, 3=both)         (6 cols) */
int64_t orc_export_dirsets(const orc_op* op, int which, int64_t* out);

/* --- primitives, exposed for pinning against the reference build --------- */
int orc_chebyshev_nodes(double a, double b, int m, double* out);
double orc_lagrange_eval(const double* nodes, int n, int idx, double x);
/* 8 transfer matrices, n^3 x n^3 each, row-major, out size 8*(m+1)^6 */
int orc_transfer_reference(int m, double* out);
/* directional interp matrix rows x (m+1)^3 complex (interleaved) */
int orc_interp_matrix(const double* px, const double* py, const double* pz, int64_t np,
                      const double lo[3], const double hi[3], const double c[3], double kappa,
                      int m, double* out);
/* direction index of lattice offset (dx,dy,dz) at level (rho = side ratios) */
int orc_dir_index(int level, int l_hf, int64_t dx, int64_t dy, int64_t dz, const double rho[3]);
int orc_dir_vector(int level, int l_hf, int idx, double* out3);
/* psi_Q based dir map of an arbitrary vector (Def. 3) */
int orc_dir_map_vector(int level, int l_hf, const double v[3]);
/* one coupling matrix (n x n complex interleaved) in the canonical frame */
int orc_coupling_matrix(int m, double kappa, const double side[3], int64_t dx, int64_t dy,
                        int64_t dz, const double c[3], double* out);
/* dense oracle rows: y[r] = sum_k f(x_rows[r], y_k) v_k (zero_diag: skip k == row idx) */
int orc_dense_rows(const double* tx, const double* ty, const double* tz, const int64_t* rows,
                   int64_t nrows, const double* sx, const double* sy, const double* sz,
                   int64_t ns, const double* v, double kappa, int zero_diagonal, double* out);
/* helmholtz kernel value (geometry.hpp:80-86 semantics), returns 0 / -1 at r=0 */
int orc_kernel(const double d[3], double kappa, double* out2);

#ifdef __cplusplus
}
#endif
