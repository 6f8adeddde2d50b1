/*
 * fdhelm_c.h -- C-ABI of the B200-native directional Helmholtz matvec.
 *
 * y = A x with A[j,k] = exp(i kappa |x_j - y_k|) / (4 pi |x_j - y_k|), applied by
 * the fast directional multi-level method of PAPER.md Alg. 4 (S2M, M2M, M2L,
 * L2L, L2T + near field) on hand-written CUDA kernels for sm_100a.
 *
 * The reference (/root/reference) has no operator class and no FFI; this
 * boundary is the union of
 *   - ClusterTree(span<const Point3>, const AxisBox& root, int n_max,
 *                 int depth_cap = 30)           proj/include/fdhelm/cluster_tree.hpp:47
 *   - WaveNumber(kappa) (kappa > 0, finite)     proj/include/fdhelm/geometry.hpp:38-43
 *   - the interpolation degree m                proj/include/fdhelm/interpolation.hpp:14-21
 *   - SPEC.md L4 engine: setup(T_T, T_S, BlockTree, DirectionTable, kappa, m)
 *     -> Operator, matvec(op, v) -> g, stats(op)
 *   - block-tree / direction parameters eta2, l_hf
 *   - the zero-diagonal option
 * (see SURVEY.md 8(b) and INTEGRATION.md for the binding a maintainer adds).
 *
 * Conventions: points are SoA float64; charges x and results y are complex128
 * interleaved (re, im) in the caller's ORIGINAL point order.  All
 * inputs are copied at create time; the caller keeps ownership.  No exception
 * crosses this boundary: every call returns an FDH_* code and fdh_last_error()
 * returns the message of the last failure on the calling thread.
 */
#ifndef FDHELM_C_H
#define FDHELM_C_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes (the reference's exception types). */
#define FDH_OK 0
#define FDH_ERR_ARG 1         /* std::invalid_argument: empty set, n_max < 1, invalid root,
                                 point outside root, kappa <= 0, bad degree ... */
#define FDH_ERR_DOMAIN 2      /* std::domain_error: singular kernel (x_j == y_k) in apply */
#define FDH_ERR_DIM 3         /* dimension mismatch */
#define FDH_ERR_UNSUPPORTED 4 /* a configuration this build does not support */
#define FDH_ERR_CUDA 5        /* CUDA runtime failure / no device / extension missing */
#define FDH_ERR_MEMORY 6      /* device allocation failed */

/* l_hf sentinel: choose the largest high-frequency level by the default rule
 * l_hf = max{l <= min(p_T, p_S) : kappa * q_l >= 3}. */
#define FDH_LHF_DEFAULT (-2)

typedef struct fdh_op fdh_op;

/* Phases of Alg. 4, for fdh_stats.phase_ms. */
enum {
  FDH_PHASE_H2D = 0,   /* charges host->device + permutation into slot order */
  FDH_PHASE_S2M = 1,
  FDH_PHASE_M2M = 2,
  FDH_PHASE_M2L = 3,
  FDH_PHASE_L2L = 4,
  FDH_PHASE_L2T = 5,
  FDH_PHASE_P2P = 6,
  FDH_PHASE_D2H = 7,   /* scatter to original order + device->host */
  FDH_NPHASES = 8
};

typedef struct fdh_stats {
  /* RunStats counters (PAPER.md Thms. 1-4, Table 1) */
  int64_t n_le;        /* applied transfer + interpolation matrices          */
  int64_t n_c;         /* |L+|, applied coupling matrices                    */
  int64_t n_sc;        /* distinct (level, lattice offset) coupling keys     */
  int64_t m_d;         /* near-field entries sum_{L-} #t * #s                */
  int64_t n_lminus;    /* |L-|                                               */
  double nf_percent;   /* 100 * m_d / (N_T * N_S)                            */
  int64_t bytes_stored;/* device bytes held by the operator                  */
  int32_t depth_t, depth_s, l_hf, n_pad;
  int64_t slots_t, slots_s, nodes_t, nodes_s;
  /* last apply */
  double phase_ms[FDH_NPHASES]; /* CUDA-event times (when timing enabled)   */
  double apply_ms;              /* whole apply, CUDA events                 */
  double setup_ms;              /* fdh_create wall time                     */
  int64_t gpu_launches;         /* kernels launched by one apply            */
  int64_t m2l_flops_executed;   /* DMMA flops incl. padding / empty columns */
  double m2l_gemm_ms;           /* average M2L GEMM kernel time (timing on)  */
  int64_t timed_applies;        /* applies averaged into phase_ms            */
  int64_t m2l_tiles, m2l_items;  /* M2L target tiles / (tile, key chunk) items */
  int64_t m2l_chunk;            /* key ids per chunk                          */
  double shard_cost, total_cost; /* estimated flops: this shard / all targets */
  double structure_ms;          /* trees + partition + directions + slots     */
  int64_t gpu_structure;        /* 1: built by the k_setup.cu kernels         */
  int64_t w_resident;           /* 1: coupling matrices kept in HBM           */
  int64_t w_segments;           /* else: per-apply generation segments        */
  int64_t m2l_impl;             /* 0: FP64 DMMA (mma.sync), 1: int8 tcgen05 digit products */
  int64_t m2l_i8_ops;           /* int8 tensor ops (2 per MAC) issued by one M2L (impl 1)  */
  int64_t nrhs;                 /* right-hand sides per device apply (fdh_create_multi)    */
  int64_t hbm_bytes[4];         /* algorithmic HBM bytes per rhs of S2M, M2M, L2L, L2T     */
  int64_t graph_replays;        /* applies run as a replay of the captured CUDA graph      */
  double apply_ms_sum;          /* sum of apply_ms over the applies collected since the
                                   last fdh_set_timing (host-path applies: every one)      */
  int64_t applies_collected;
  double aca_eps;               /* ACA tolerance in use (0: exact dense coupling)          */
  double aca_mean_rank;         /* mean ACA rank over the compressed keys                  */
  int64_t aca_bytes;            /* device bytes of the ACA factors                         */
  int64_t aca_dense_keys;       /* keys kept dense (2 k n >= n^2)                          */
  int64_t nf_cache_bytes;       /* device bytes of the cached near-field kernel values     */
  int64_t m2l_pair_mode;        /* 1: int8 M2L key-major on (target, source) pairs         */
  int64_t m2l_i8_digits;        /* int8 M2L: digits per FP64 value ...                     */
  int64_t m2l_i8_bits;          /* ... of this many bits                                   */
  int64_t m2l_i8_products;      /* digit-pair products kept per real MAC (6 x 8 + level 6: 26) */
} fdh_stats;

/* Setup: both cluster trees (Alg. 1), the direction table
 * (Alg. 3), the block tree with L+/L- and D/D^ sets (Alg. 2, Def. 4), the
 * coupling matrices of every (level, offset) key (Eq. 9), device buffers.
 * n_gpus > 1: one process drives devices 0 .. n_gpus-1, device g holding the
 * target-leaf shard g of n_gpus (fdh_create_shard, set up concurrently); an
 * apply broadcasts x from device 0 and reduces y onto device 0 over NCCL
 * (libnccl.so.2 loaded at run time).  fdh_apply_device on such an operator takes
 * device-0 pointers and a device-0 stream; exports describe device 0's shard. */
int fdh_create(const double* tx, const double* ty, const double* tz, int64_t nt,
               const double* sx, const double* sy, const double* sz, int64_t ns,
               const double root_lo[3], const double root_hi[3], double kappa, int n_max, int m,
               double eta2, int l_hf, int depth_cap, int zero_diagonal, int n_gpus,
               fdh_op** out);

/* Same, for rank `rank` of `world` (one process per GPU).  The rank owns a
 * contiguous, cost-balanced Morton range of target leaves; fdh_apply on a shard
 * writes the rows of its targets and zeros elsewhere, so the sum over ranks
 * (an all-reduce of y) is the full product. */
int fdh_create_shard(const double* tx, const double* ty, const double* tz, int64_t nt,
                     const double* sx, const double* sy, const double* sz, int64_t ns,
                     const double root_lo[3], const double root_hi[3], double kappa, int n_max,
                     int m, double eta2, int l_hf, int depth_cap, int zero_diagonal, int rank,
                     int world, fdh_op** out);

/* Same, for nrhs right-hand sides per apply (nrhs a
 * power of two in 1..16).  The M2L tiles then pair (target slot, rhs): one
 * coupling matrix read serves every rhs of a slot, and the near field forms each
 * kernel value once for up to 8 rhs.  fdh_apply_device on such an operator takes
 * nrhs vectors (rhs-major: x_dev[r * N_S + k], y_dev[r * N_T + j]). */
int fdh_create_multi(const double* tx, const double* ty, const double* tz, int64_t nt,
                     const double* sx, const double* sy, const double* sz, int64_t ns,
                     const double root_lo[3], const double root_hi[3], double kappa, int n_max,
                     int m, double eta2, int l_hf, int depth_cap, int zero_diagonal, int rank,
                     int world, int nrhs, fdh_op** out);

/* Host-only setup (trees, blocks, directions, work lists; no device state):
 * for introspection and for testing the planner on machines without a GPU.
 * fdh_apply on such an operator returns FDH_ERR_UNSUPPORTED. */
int fdh_plan_only(const double* tx, const double* ty, const double* tz, int64_t nt,
                  const double* sx, const double* sy, const double* sz, int64_t ns,
                  const double root_lo[3], const double root_hi[3], double kappa, int n_max, int m,
                  double eta2, int l_hf, int depth_cap, int zero_diagonal, int rank, int world,
                  fdh_op** out);

/* matvec: y[N_T] = A x[N_S], host buffers, blocking. */
int fdh_apply(fdh_op* op, const double* x, double* y);
/* k right-hand sides, host buffers, rhs-major (x[r * N_S + k], y[r * N_T + j]),
 * run in device batches of nrhs (fdh_create_multi; a short last batch is padded
 * with zero vectors).  Y = A X with X an N_S x k column-major matrix. */
int fdh_apply_multi(fdh_op* op, const double* x, int64_t k, double* y);
/* Device-resident variant: x_dev / y_dev are device pointers (complex128,
 * original order); enqueued on `stream` (cudaStream_t, NULL = the operator's
 * own stream) and not synchronised.  Errors detected on the device (singular
 * kernel -> FDH_ERR_DOMAIN, as the reference's domain_error) are DEFERRED: they
 * accumulate over device-path applies and are returned by fdh_sync. */
int fdh_apply_device(fdh_op* op, const double* x_dev, double* y_dev, void* stream);
/* ACA-compressed coupling (opt-in and
 * LOSSY): eps > 0 factorises every coupling matrix by partially pivoted ACA on
 * the device (A ~ U V^*, pivoting as SPEC.md:457; a key whose rank would reach
 * n/2 stays dense) and later applies run the M2L on the factors in FP64; results
 * then agree with the exact apply to ~100 eps (eps = 1e-8 -> 1e-6),
 * not to 1e-12.  eps = 0 returns to the exact M2L.  n <= 384 (m <= 6), nrhs = 1;
 * FDH_ERR_MEMORY when the factors do not fit in device memory. */
int fdh_set_aca(fdh_op* op, double eps);
/* Caches for repeated applies (PAPER.md:659, SPEC.md:519
 * "a flag to cache them").  FDH_CACHE_NEARFIELD: the kernel value of every
 * near-field pair (16 B per pair, M_D pairs) is computed once here and later
 * applies stream it instead of recomputing it (exact: the reference's operation
 * order and the library sincos).  FDH_ERR_MEMORY if it does not fit in device
 * memory (configs >= 3), FDH_ERR_DOMAIN for a singular pair.  flags = 0 frees it. */
#define FDH_CACHE_NEARFIELD 1
int fdh_set_cache(fdh_op* op, int flags);
/* Wait for the operator's applies and return (and clear) the deferred device
 * error of the fdh_apply_device calls since the last fdh_sync. */
int fdh_sync(fdh_op* op);
/* The operator's stream (cudaStream_t) for event timing by the caller. */
void* fdh_stream(fdh_op* op);
/* Enable per-phase CUDA-event timing (events recorded between the phases of
 * every apply on its stream -- inside the CUDA graph as event-record nodes, so
 * the timed applies are the same graph replays as untimed ones; fdh_get_stats
 * averages the applies recorded since this call).  Resets the averages and
 * apply_ms_sum. */
int fdh_set_timing(fdh_op* op, int enable);

int fdh_get_stats(const fdh_op* op, fdh_stats* out);

/* Canonical introspection: int64 rows, sorted; out == NULL
 * returns the row count.  Identical layouts to the CPU oracle's exports. */
int64_t fdh_export_tree(const fdh_op* op, int which /*0=T,1=S*/, int64_t* rows /*7 cols*/);
int64_t fdh_export_perm(const fdh_op* op, int which, int64_t* perm);
int64_t fdh_export_lplus(const fdh_op* op, int64_t* rows /*8 cols*/);
int64_t fdh_export_lminus(const fdh_op* op, int64_t* rows /*8 cols*/);
int64_t fdh_export_dirsets(const fdh_op* op, int which, int64_t* rows /*6 cols*/);
/* target leaves owned by this operator (all, or this rank's shard):
 * level, i, j, k, begin, end                                        (6 cols) */
int64_t fdh_export_owned_leaves(const fdh_op* op, int64_t* rows);
/* order-independent 64-bit digests of the canonical exports (sum over rows of a
 * splitmix64 row hash): [T tree+perm, S tree+perm, L+, L-, D/D^ of T, D/D^ of S];
 * compares structures too large to export (config 4). */
int fdh_structure_digest(const fdh_op* op, uint64_t* out6);

void fdh_destroy(fdh_op* op);
const char* fdh_last_error(void);
/* Build identification string (arch, version). */
const char* fdh_version(void);
/* Measured FP64 peak of the current device in TFLOP/s (kind 0: DMMA
 * mma.sync.m8n8k4.f64, 1: DFMA), the roofline denominator of M2L / P2P. */
double fdh_fp64_peak_tflops(int kind);
/* Measured dense tensor peak of the current device in TOPS (kind 0: int8
 * tcgen05.mma kind::i8, M=128 N=256 from shared memory), the roofline
 * denominator of the int8 M2L kernel (k_m2l_i8). */
double fdh_tensor_peak_tops(int kind); /* kind 0: burst (~1 ms), 1: sustained (held ~3 s, power-limited clocks) */

#ifdef __cplusplus
}
#endif
#endif /* FDHELM_C_H */
