// k_setup.cu -- setup on the GPU: cluster trees (Alg. 1), block
// partition (Alg. 2, Def. 1-2), key directions (Alg. 3, Def. 3) and the
// active / inherited direction sets with their dense slots (Def. 4).
//
// Every stage reproduces the host planner (plan.cpp) bit for bit, which in turn
// is bit-exact with the reference's ClusterTree (cluster_tree.cpp:12-128):
//   * tree: level-synchronous stable octant partition.  Octants are decided with
//     the reference's separate FP64 multiply and add (__dmul_rn / __dadd_rn,
//     cluster_tree.cpp:75-77, 86); the stable partition of every refining node is
//     a digit ranking (per-block warp-ballot ranks + a scan over blocks), so the
//     slot order equals the reference's std::stable-style scatter (cpp:98-109);
//     children are created in (parent, octant) = Morton order.
//   * blocks: breadth-first over levels; each candidate pair is classified
//     (A1/A3 with the reference's box_distance operation order) and emits L+,
//     L- or its child pairs at offsets from exclusive scans -> the same list
//     order as the host sweep.
//   * keys: dense offset table per level, numbered by a scan in (dx, dy, dz) order.
//   * D / D^ / slots: byte tables per level, D^ from the parent, slots by a scan.
// All scans are hand-written (block scan + recursive scan of block sums).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>

#include "common.cuh"
#include "plan.hpp"
#include "setup_gpu.hpp"

namespace fdhelm {

namespace {

#define SCK(x)                                                                                            \
  do {                                                                                                    \
    cudaError_t e_ = (x);                                                                                 \
    if (e_ != cudaSuccess) throw PlanError{5, std::string("setup: ") + #x + ": " + cudaGetErrorString(e_)}; \
  } while (0)

constexpr int kScanBlock = 1024;  // elements per scan block (512 threads x 2)

// ------------------------------------------------------------- device buffers
struct Dev {
  std::vector<void*> ptrs;
  ~Dev() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    SCK(cudaMalloc(&p, n * sizeof(T)));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* up(const std::vector<T>& v) {
    T* d = alloc<T>(v.size());
    if (!v.empty()) SCK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  }
  void release(void* p) {
    auto it = std::find(ptrs.begin(), ptrs.end(), p);
    if (it != ptrs.end()) {
      cudaFree(p);
      ptrs.erase(it);
    }
  }
};

template <class T>
std::vector<T> down(const T* d, size_t n) {
  std::vector<T> h(n);
  if (n) SCK(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
  return h;
}

// ------------------------------------------------------------------- scan
// exclusive scan of int64 in place; block sums to `sums`
__global__ void k_scan_block(int64_t* __restrict__ a, int64_t n, int64_t* __restrict__ sums) {
  __shared__ int64_t sh[kScanBlock];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock;
  for (int i = threadIdx.x; i < kScanBlock; i += blockDim.x) sh[i] = base + i < n ? a[base + i] : 0;
  __syncthreads();
  // Hillis-Steele on 1024 elements (10 steps)
  for (int off = 1; off < kScanBlock; off <<= 1) {
    int64_t v[2];
    for (int r = 0; r < 2; ++r) {
      const int i = threadIdx.x + r * blockDim.x;
      v[r] = i >= off ? sh[i - off] : 0;
    }
    __syncthreads();
    for (int r = 0; r < 2; ++r) sh[threadIdx.x + r * blockDim.x] += v[r];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < kScanBlock; i += blockDim.x)
    if (base + i < n) a[base + i] = i == 0 ? 0 : sh[i - 1];  // exclusive
  if (threadIdx.x == 0) sums[blockIdx.x] = sh[kScanBlock - 1];
}
__global__ void k_scan_add(int64_t* __restrict__ a, int64_t n, const int64_t* __restrict__ sums) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] += sums[i / kScanBlock];
}

// exclusive scan; returns the total
int64_t scan_excl(Dev& D, int64_t* a, int64_t n) {
  if (n <= 0) return 0;
  const int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  int64_t* sums = D.alloc<int64_t>((size_t)nb + 1);
  k_scan_block<<<(unsigned)nb, kScanBlock / 2>>>(a, n, sums);
  SCK(cudaGetLastError());
  int64_t tot;
  if (nb > 1) {
    // sums holds the block totals: their scan gives the block offsets and the total
    tot = scan_excl(D, sums, nb);
    k_scan_add<<<(unsigned)((n + 255) / 256), 256>>>(a, n, sums);
    SCK(cudaGetLastError());
  } else {
    tot = down(sums, 1)[0];
  }
  D.release(sums);
  return tot;
}

// ------------------------------------------------------------------- tree
struct DevLevel {
  int64_t n = 0;
  int64_t *ci = nullptr, *cj = nullptr, *ck = nullptr;
  uint32_t *beg = nullptr, *end = nullptr;
  uint8_t* leaf = nullptr;
  int32_t* parent = nullptr;
  int32_t* child = nullptr;  // 8 per node
};

__global__ void k_refine_flags(int64_t nn, const uint32_t* __restrict__ beg, const uint32_t* __restrict__ end,
                               int nmax, int level, int cap, int64_t* __restrict__ refine,
                               unsigned long long* __restrict__ oversized) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  const uint32_t c = end[i] - beg[i];
  const bool r = c > (uint32_t)nmax && level < cap;
  refine[i] = r ? 1 : 0;
  if (c > (uint32_t)nmax && level >= cap) atomicAdd(oversized, 1ull);
}

// octant of every point of a refining node (cluster_tree.cpp:73-89), 0xFF otherwise
__global__ void k_octant(int64_t n, const int32_t* __restrict__ pnode, const int64_t* __restrict__ rflag,
                         const int64_t* __restrict__ ci, const int64_t* __restrict__ cj, const int64_t* __restrict__ ck,
                         const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ z,
                         double lo0, double lo1, double lo2, double cs0, double cs1, double cs2,
                         uint8_t* __restrict__ oct) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t v = pnode[i];
  uint8_t o = 0xFF;
  if (v >= 0 && rflag[v]) {
    const double mx = __dadd_rn(lo0, __dmul_rn((double)(2 * ci[v] + 1), cs0));
    const double my = __dadd_rn(lo1, __dmul_rn((double)(2 * cj[v] + 1), cs1));
    const double mz = __dadd_rn(lo2, __dmul_rn((double)(2 * ck[v] + 1), cs2));
    o = (uint8_t)(4 * (x[i] > mx) + 2 * (y[i] > my) + (z[i] > mz));
  }
  oct[i] = o;
}

// per block of kScanBlock points: in-block rank among equal octants (stable) and
// the per-octant block counts (counts[o * nblk + blk])
__global__ void __launch_bounds__(kScanBlock) k_rank(int64_t n, const uint8_t* __restrict__ oct,
                                                     uint32_t* __restrict__ rank, int64_t* __restrict__ counts,
                                                     int64_t nblk) {
  __shared__ uint32_t wcnt[kScanBlock / 32][8];
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint8_t o = i < n ? oct[i] : 0xFF;
  uint32_t my = 0;
  for (int d = 0; d < 8; ++d) {
    const unsigned b = __ballot_sync(0xffffffffu, o == d);
    if (o == d) my = __popc(b & ((1u << lane) - 1u));
    if (lane == 0) wcnt[warp][d] = __popc(b);
  }
  __syncthreads();
  if (threadIdx.x < 8) {  // exclusive prefix over warps, per octant
    const int d = threadIdx.x;
    uint32_t acc = 0;
    for (int w = 0; w < kScanBlock / 32; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = acc;
      acc += c;
    }
    counts[d * nblk + blockIdx.x] = acc;
  }
  __syncthreads();
  if (i < n && o != 0xFF) rank[i] = my + wcnt[warp][o];
}

// E(o, p) = number of points before position p with octant o
__device__ __forceinline__ int64_t count_before(const uint8_t* __restrict__ oct, const int64_t* __restrict__ bbase,
                                                int64_t nblk, int o, int64_t p, int lane) {
  const int64_t blk = p / kScanBlock;
  int64_t c = blk < nblk ? bbase[o * nblk + blk] : bbase[o * nblk + nblk - 1];
  if (blk >= nblk) return -1;  // not used (p == n handled by caller)
  int64_t loc = 0;
  for (int64_t q = blk * kScanBlock + lane; q < p; q += 32) loc += oct[q] == o;
  for (int s = 16; s; s >>= 1) loc += __shfl_xor_sync(0xffffffffu, loc, s);
  return c + loc;
}

// one warp per refining node: per-octant counts and the octant base E(o, begin)
__global__ void k_node_octants(int64_t nref, const int32_t* __restrict__ ref_nodes, const uint32_t* __restrict__ beg,
                               const uint32_t* __restrict__ end, const uint8_t* __restrict__ oct,
                               const int64_t* __restrict__ bbase, int64_t nblk, int64_t n, int64_t total_o[8],
                               int64_t* __restrict__ cnt, int64_t* __restrict__ obase, int64_t* __restrict__ nchild) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nref) return;
  const int32_t v = ref_nodes[r];
  const int64_t b = beg[v], e = end[v];
  int nc = 0;
  for (int o = 0; o < 8; ++o) {
    const int64_t eb = count_before(oct, bbase, nblk, o, b, lane);
    const int64_t ee = e >= n ? total_o[o] : count_before(oct, bbase, nblk, o, e, lane);
    if (lane == 0) {
      cnt[r * 8 + o] = ee - eb;
      obase[r * 8 + o] = eb;
    }
    nc += (ee - eb) > 0;
  }
  if (lane == 0) nchild[r] = nc;
}

// children of refining node r in octant order (Morton): coords, ranges, links
__global__ void k_make_children(int64_t nref, const int32_t* __restrict__ ref_nodes, const int64_t* __restrict__ ci,
                                const int64_t* __restrict__ cj, const int64_t* __restrict__ ck,
                                const uint32_t* __restrict__ beg, const int64_t* __restrict__ cnt,
                                const int64_t* __restrict__ cbase, int32_t* __restrict__ child, int64_t* __restrict__ nci,
                                int64_t* __restrict__ ncj, int64_t* __restrict__ nck, uint32_t* __restrict__ nbeg,
                                uint32_t* __restrict__ nend, int32_t* __restrict__ npar, uint8_t* __restrict__ leaf,
                                int32_t* __restrict__ coff /* 8 per ref: child index or -1 */,
                                uint32_t* __restrict__ ooff /* 8 per ref: slot offset of octant */) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nref) return;
  const int32_t v = ref_nodes[r];
  leaf[v] = 0;
  int64_t c = cbase[r];
  uint32_t off = beg[v];
  for (int o = 0; o < 8; ++o) {
    const int64_t k = cnt[r * 8 + o];
    ooff[r * 8 + o] = off;
    if (k == 0) {
      coff[r * 8 + o] = -1;
      continue;
    }
    child[(int64_t)v * 8 + o] = (int32_t)c;
    coff[r * 8 + o] = (int32_t)c;
    nci[c] = 2 * ci[v] + ((o >> 2) & 1);
    ncj[c] = 2 * cj[v] + ((o >> 1) & 1);
    nck[c] = 2 * ck[v] + (o & 1);
    nbeg[c] = off;
    nend[c] = off + (uint32_t)k;
    npar[c] = v;
    off += (uint32_t)k;
    ++c;
  }
}

// stable scatter of the points of refining nodes; other points keep their slot
__global__ void k_scatter_points(int64_t n, const int32_t* __restrict__ pnode, const int64_t* __restrict__ refidx,
                                 const int64_t* __restrict__ rflag, const uint8_t* __restrict__ oct,
                                 const uint32_t* __restrict__ rank, const int64_t* __restrict__ bbase, int64_t nblk,
                                 const int64_t* __restrict__ obase, const uint32_t* __restrict__ ooff,
                                 const int32_t* __restrict__ coff, const double* __restrict__ x,
                                 const double* __restrict__ y, const double* __restrict__ z,
                                 const uint32_t* __restrict__ perm, double* __restrict__ x2, double* __restrict__ y2,
                                 double* __restrict__ z2, uint32_t* __restrict__ perm2, int32_t* __restrict__ pnode2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t v = pnode[i];
  int64_t dst = i;
  int32_t nv = -1;
  if (v >= 0 && rflag[v]) {
    const int o = oct[i];
    const int64_t r = refidx[v];
    const int64_t g = bbase[o * nblk + i / kScanBlock] + rank[i];  // E(o, i)
    dst = (int64_t)ooff[r * 8 + o] + (g - obase[r * 8 + o]);
    nv = coff[r * 8 + o];
  }
  x2[dst] = x[i];
  y2[dst] = y[i];
  z2[dst] = z[i];
  perm2[dst] = perm[i];
  pnode2[dst] = nv;
}

__global__ void k_fill_i32(int32_t* a, int64_t n, int32_t v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
__global__ void k_iota_u32(uint32_t* a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = (uint32_t)i;
}
__global__ void k_compact_flags(int64_t nn, const int64_t* __restrict__ rflag, const int64_t* __restrict__ ridx,
                                int32_t* __restrict__ ref_nodes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nn && rflag[i]) ref_nodes[ridx[i]] = (int32_t)i;
}

inline unsigned nblocks(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// Level-synchronous Alg. 1 on the device; fills the host TreePlan like build_tree.
void tree_on_gpu(Dev& D, TreePlan& T, std::vector<DevLevel>& dl, const double* x, const double* y, const double* z,
                 int64_t n, const double lo[3], const double hi[3], int nmax, int cap) {
  if (n <= 0) throw PlanError{1, "cluster tree: empty point set"};
  if (nmax < 1) throw PlanError{1, "cluster tree: n_max must be >= 1"};
  if (!(lo[0] < hi[0] && lo[1] < hi[1] && lo[2] < hi[2])) throw PlanError{1, "cluster tree: invalid root box"};
  if (n > (int64_t)UINT32_MAX) throw PlanError{4, "cluster tree: more than 2^32-1 points"};
  for (int a = 0; a < 3; ++a) {
    T.lo[a] = lo[a] - 1e-12 * (hi[a] - lo[a]);  // cluster_tree.cpp:21-24
    T.hi[a] = hi[a];
  }
  for (int64_t i = 0; i < n; ++i) {
    const bool in = x[i] > T.lo[0] && x[i] <= T.hi[0] && y[i] > T.lo[1] && y[i] <= T.hi[1] && z[i] > T.lo[2] &&
                    z[i] <= T.hi[2];
    if (!in) throw PlanError{1, "cluster tree: point outside root box"};
  }
  double* dx[2] = {D.alloc<double>(n), D.alloc<double>(n)};
  double* dy[2] = {D.alloc<double>(n), D.alloc<double>(n)};
  double* dz[2] = {D.alloc<double>(n), D.alloc<double>(n)};
  uint32_t* dp[2] = {D.alloc<uint32_t>(n), D.alloc<uint32_t>(n)};
  int32_t* pn[2] = {D.alloc<int32_t>(n), D.alloc<int32_t>(n)};
  SCK(cudaMemcpy(dx[0], x, n * 8, cudaMemcpyHostToDevice));
  SCK(cudaMemcpy(dy[0], y, n * 8, cudaMemcpyHostToDevice));
  SCK(cudaMemcpy(dz[0], z, n * 8, cudaMemcpyHostToDevice));
  k_iota_u32<<<nblocks(n), 256>>>(dp[0], n);
  k_fill_i32<<<nblocks(n), 256>>>(pn[0], n, 0);
  uint8_t* oct = D.alloc<uint8_t>(n);
  uint32_t* rank = D.alloc<uint32_t>(n);
  const int64_t nblk = (n + kScanBlock - 1) / kScanBlock;
  int64_t* bcnt = D.alloc<int64_t>(8 * nblk);
  unsigned long long* over = D.alloc<unsigned long long>(1);
  SCK(cudaMemset(over, 0, 8));
  int64_t* total_o = D.alloc<int64_t>(8);
  int cur = 0;

  T.side.assign(1, {T.hi[0] - T.lo[0], T.hi[1] - T.lo[1], T.hi[2] - T.lo[2]});
  auto norm = [](const std::array<double, 3>& s) { return std::sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]); };
  T.diam.assign(1, norm(T.side[0]));
  dl.clear();
  {
    DevLevel L0;
    L0.n = 1;
    L0.ci = D.up(std::vector<int64_t>{0});
    L0.cj = D.up(std::vector<int64_t>{0});
    L0.ck = D.up(std::vector<int64_t>{0});
    L0.beg = D.up(std::vector<uint32_t>{0});
    L0.end = D.up(std::vector<uint32_t>{(uint32_t)n});
    L0.leaf = D.up(std::vector<uint8_t>{1});
    L0.parent = D.up(std::vector<int32_t>{-1});
    dl.push_back(L0);
  }
  for (int l = 0;; ++l) {
    DevLevel& L = dl[l];
    L.child = D.alloc<int32_t>(8 * L.n);
    k_fill_i32<<<nblocks(8 * L.n), 256>>>(L.child, 8 * L.n, -1);
    int64_t* rflag = D.alloc<int64_t>(L.n);
    int64_t* ridx = D.alloc<int64_t>(L.n);
    k_refine_flags<<<nblocks(L.n), 256>>>(L.n, L.beg, L.end, nmax, l, cap, rflag, over);
    SCK(cudaMemcpy(ridx, rflag, L.n * 8, cudaMemcpyDeviceToDevice));
    const int64_t nref = scan_excl(D, ridx, L.n);
    if (nref == 0) {
      T.depth = l;
      break;
    }
    if (l + 1 > 21) throw PlanError{4, "cluster tree deeper than 21 levels is not supported by this build"};
    const auto s = T.side[l];
    T.side.push_back({0.5 * s[0], 0.5 * s[1], 0.5 * s[2]});
    T.diam.push_back(norm(T.side[l + 1]));
    const auto cs = T.side[l + 1];
    int32_t* ref_nodes = D.alloc<int32_t>(nref);
    k_compact_flags<<<nblocks(L.n), 256>>>(L.n, rflag, ridx, ref_nodes);
    k_octant<<<nblocks(n), 256>>>(n, pn[cur], rflag, L.ci, L.cj, L.ck, dx[cur], dy[cur], dz[cur], T.lo[0], T.lo[1],
                                  T.lo[2], cs[0], cs[1], cs[2], oct);
    k_rank<<<(unsigned)nblk, kScanBlock>>>(n, oct, rank, bcnt, nblk);
    // per-octant scan over blocks (bcnt[o*nblk + b]) -> E(o, block start); totals
    std::vector<int64_t> tot(8);
    for (int o = 0; o < 8; ++o) tot[o] = scan_excl(D, bcnt + o * nblk, nblk);
    SCK(cudaMemcpy(total_o, tot.data(), 64, cudaMemcpyHostToDevice));
    int64_t* cnt = D.alloc<int64_t>(8 * nref);
    int64_t* obase = D.alloc<int64_t>(8 * nref);
    int64_t* nchild = D.alloc<int64_t>(nref);
    k_node_octants<<<nblocks(32 * nref), 256>>>(nref, ref_nodes, L.beg, L.end, oct, bcnt, nblk, n, total_o, cnt, obase,
                                                nchild);
    const int64_t nnew = scan_excl(D, nchild, nref);
    DevLevel N;
    N.n = nnew;
    N.ci = D.alloc<int64_t>(nnew);
    N.cj = D.alloc<int64_t>(nnew);
    N.ck = D.alloc<int64_t>(nnew);
    N.beg = D.alloc<uint32_t>(nnew);
    N.end = D.alloc<uint32_t>(nnew);
    N.leaf = D.alloc<uint8_t>(nnew);
    SCK(cudaMemset(N.leaf, 1, nnew));
    N.parent = D.alloc<int32_t>(nnew);
    int32_t* coff = D.alloc<int32_t>(8 * nref);
    uint32_t* ooff = D.alloc<uint32_t>(8 * nref);
    k_make_children<<<nblocks(nref), 256>>>(nref, ref_nodes, L.ci, L.cj, L.ck, L.beg, cnt, nchild, L.child, N.ci, N.cj,
                                            N.ck, N.beg, N.end, N.parent, L.leaf, coff, ooff);
    k_scatter_points<<<nblocks(n), 256>>>(n, pn[cur], ridx, rflag, oct, rank, bcnt, nblk, obase, ooff, coff, dx[cur],
                                          dy[cur], dz[cur], dp[cur], dx[cur ^ 1], dy[cur ^ 1], dz[cur ^ 1], dp[cur ^ 1],
                                          pn[cur ^ 1]);
    SCK(cudaGetLastError());
    cur ^= 1;
    for (void* p : {(void*)rflag, (void*)ref_nodes, (void*)cnt, (void*)obase, (void*)nchild, (void*)coff,
                    (void*)ooff})
      D.release(p);
    // keep ridx for nothing further
    D.release(ridx);
    dl.push_back(N);
  }
  SCK(cudaDeviceSynchronize());
  T.oversized = (int)down(over, 1)[0];
  T.x = down(dx[cur], n);
  T.y = down(dy[cur], n);
  T.z = down(dz[cur], n);
  T.perm = down(dp[cur], n);
  T.lv.assign(T.depth + 1, {});
  for (int l = 0; l <= T.depth; ++l) {
    const DevLevel& L = dl[l];
    LevelNodes& H = T.lv[l];
    H.ci = down(L.ci, L.n);
    H.cj = down(L.cj, L.n);
    H.ck = down(L.ck, L.n);
    H.begin = down(L.beg, L.n);
    H.end = down(L.end, L.n);
    H.leaf = down(L.leaf, L.n);
    H.parent = down(L.parent, L.n);
    H.child = down(L.child, 8 * L.n);
  }
  for (int i = 0; i < 2; ++i) {
    D.release(dx[i]);
    D.release(dy[i]);
    D.release(dz[i]);
    D.release(dp[i]);
    D.release(pn[i]);
  }
  D.release(oct);
  D.release(rank);
  D.release(bcnt);
}

// ------------------------------------------------------------- partition
struct LvlGeo {
  double q, eta2, kappa;
  double tlo[3], slo[3], tside[3], sside[3];
};

// Def. 1 (A1)+(A3) inclusive, box_distance in the reference's operation order
__device__ __forceinline__ bool adm_dev(const LvlGeo& g, int64_t tci, int64_t tcj, int64_t tck, int64_t sci,
                                        int64_t scj, int64_t sck) {
  const int64_t tc[3] = {tci, tcj, tck}, sc[3] = {sci, scj, sck};
  double acc = 0.0;
  for (int a = 0; a < 3; ++a) {
    const double tlo = __dadd_rn(g.tlo[a], __dmul_rn((double)tc[a], g.tside[a]));
    const double thi = __dadd_rn(g.tlo[a], __dmul_rn((double)(tc[a] + 1), g.tside[a]));
    const double slo = __dadd_rn(g.slo[a], __dmul_rn((double)sc[a], g.sside[a]));
    const double shi = __dadd_rn(g.slo[a], __dmul_rn((double)(sc[a] + 1), g.sside[a]));
    const double gap = fmax(fmax(__dsub_rn(tlo, shi), __dsub_rn(slo, thi)), 0.0);
    acc = __dadd_rn(acc, __dmul_rn(gap, gap));
  }
  const double dist = __dsqrt_rn(acc);
  const double rhs = __dmul_rn(g.eta2, dist);
  return (g.q <= rhs) && (__dmul_rn(__dmul_rn(g.kappa, g.q), g.q) <= rhs);
}

// classify pair i: 1 = L+, 0 = L-, 2 = refine; counts for the scans
__global__ void k_classify(int64_t np, const int32_t* __restrict__ pt, const int32_t* __restrict__ ps, LvlGeo g,
                           const int64_t* __restrict__ tci, const int64_t* __restrict__ tcj,
                           const int64_t* __restrict__ tck, const int64_t* __restrict__ sci,
                           const int64_t* __restrict__ scj, const int64_t* __restrict__ sck,
                           const uint8_t* __restrict__ tleaf, const uint8_t* __restrict__ sleaf,
                           const int32_t* __restrict__ tch, const int32_t* __restrict__ sch, int64_t* __restrict__ nlp,
                           int64_t* __restrict__ nlm, int64_t* __restrict__ nnx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  const int32_t t = pt[i], s = ps[i];
  const bool a = adm_dev(g, tci[t], tcj[t], tck[t], sci[s], scj[s], sck[s]);
  int64_t lp = 0, lm = 0, nx = 0;
  if (tleaf[t] || sleaf[s]) {
    (a ? lp : lm) = 1;
  } else if (!a) {
    int ct = 0, cs = 0;
    for (int o = 0; o < 8; ++o) {
      ct += tch[(int64_t)t * 8 + o] >= 0;
      cs += sch[(int64_t)s * 8 + o] >= 0;
    }
    nx = (int64_t)ct * cs;
  } else {
    lp = 1;
  }
  nlp[i] = lp;
  nlm[i] = lm;
  nnx[i] = nx;
}

__global__ void k_emit(int64_t np, const int32_t* __restrict__ pt, const int32_t* __restrict__ ps,
                       const int64_t* __restrict__ olp, const int64_t* __restrict__ olm,
                       const int64_t* __restrict__ onx, int64_t tlp, int64_t tlm, int64_t tnx,
                       const int32_t* __restrict__ tch, const int32_t* __restrict__ sch, int32_t* __restrict__ lpt,
                       int32_t* __restrict__ lps, int32_t* __restrict__ lmt, int32_t* __restrict__ lms,
                       int32_t* __restrict__ nxt, int32_t* __restrict__ nxs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  const int32_t t = pt[i], s = ps[i];
  const int64_t a0 = olp[i], a1 = i + 1 < np ? olp[i + 1] : tlp;
  const int64_t b0 = olm[i], b1 = i + 1 < np ? olm[i + 1] : tlm;
  const int64_t c0 = onx[i], c1 = i + 1 < np ? onx[i + 1] : tnx;
  if (a1 > a0) {
    lpt[a0] = t;
    lps[a0] = s;
  }
  if (b1 > b0) {
    lmt[b0] = t;
    lms[b0] = s;
  }
  if (c1 > c0) {
    int64_t o = c0;
    for (int a = 0; a < 8; ++a) {
      const int32_t ta = tch[(int64_t)t * 8 + a];
      if (ta < 0) continue;
      for (int b = 0; b < 8; ++b) {
        const int32_t sb = sch[(int64_t)s * 8 + b];
        if (sb < 0) continue;
        nxt[o] = ta;
        nxs[o] = sb;
        ++o;
      }
    }
  }
}

// keys: lattice offsets of the L+ pairs, in a dense box [mn, mn + ext) per level
__device__ __forceinline__ void pair_offset(int64_t b, const int32_t* __restrict__ lpt, const int32_t* __restrict__ lps,
                                            const int64_t* __restrict__ tci, const int64_t* __restrict__ tcj,
                                            const int64_t* __restrict__ tck, const int64_t* __restrict__ sci,
                                            const int64_t* __restrict__ scj, const int64_t* __restrict__ sck,
                                            long long d[3]) {
  const int32_t t = lpt[b], s = lps[b];
  d[0] = tci[t] - sci[s];
  d[1] = tcj[t] - scj[s];
  d[2] = tck[t] - sck[s];
}
#define FDH_PAIR_ARGS                                                                                          \
  const int32_t *__restrict__ lpt, const int32_t *__restrict__ lps, const int64_t *__restrict__ tci,          \
      const int64_t *__restrict__ tcj, const int64_t *__restrict__ tck, const int64_t *__restrict__ sci,      \
      const int64_t *__restrict__ scj, const int64_t *__restrict__ sck
__global__ void k_minmax(int64_t nb, FDH_PAIR_ARGS, long long* __restrict__ mm) {
  __shared__ long long sh[6][256];
  long long v[6] = {LLONG_MAX, LLONG_MAX, LLONG_MAX, LLONG_MIN, LLONG_MIN, LLONG_MIN};
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    long long d[3];
    pair_offset(b, lpt, lps, tci, tcj, tck, sci, scj, sck, d);
    for (int a = 0; a < 3; ++a) {
      v[a] = min(v[a], d[a]);
      v[3 + a] = max(v[3 + a], d[a]);
    }
  }
  for (int k = 0; k < 6; ++k) sh[k][threadIdx.x] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < blockDim.x; ++t)
      for (int a = 0; a < 3; ++a) {
        v[a] = min(v[a], sh[a][t]);
        v[3 + a] = max(v[3 + a], sh[3 + a][t]);
      }
    for (int a = 0; a < 3; ++a) {
      atomicMin(mm + a, v[a]);
      atomicMax(mm + 3 + a, v[3 + a]);
    }
  }
}
__global__ void k_mark(int64_t nb, FDH_PAIR_ARGS, long long m0, long long m1, long long m2, long long e1,
                       long long e2, int64_t* __restrict__ tab) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  long long d[3];
  pair_offset(b, lpt, lps, tci, tcj, tck, sci, scj, sck, d);
  tab[((d[0] - m0) * e1 + (d[1] - m1)) * e2 + (d[2] - m2)] = 1;
}
__global__ void k_keyids(int64_t nb, FDH_PAIR_ARGS, long long m0, long long m1, long long m2, long long e1,
                         long long e2, const int64_t* __restrict__ tabscan, int32_t base, int32_t* __restrict__ key) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  long long d[3];
  pair_offset(b, lpt, lps, tci, tcj, tck, sci, scj, sck, d);
  key[b] = base + (int32_t)tabscan[((d[0] - m0) * e1 + (d[1] - m1)) * e2 + (d[2] - m2)];
}
__global__ void k_keylist(int64_t vol, const int64_t* __restrict__ flag, const int64_t* __restrict__ tabscan,
                          long long m0, long long m1, long long m2, long long e1, long long e2,
                          int64_t* __restrict__ kd) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= vol || !flag[v]) return;
  const int64_t id = tabscan[v];
  kd[3 * id] = v / (e1 * e2) + m0;
  kd[3 * id + 1] = (v / e2) % e1 + m1;
  kd[3 * id + 2] = v % e2 + m2;
}

// Def. 3 direction of a key: the device restatement of plan.cpp dir_map_vec
__global__ void k_keydir(int64_t nk, const int64_t* __restrict__ kd, int level, int lhf, double r0, double r1,
                         double r2, int32_t* __restrict__ dir) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nk) return;
  if (level > lhf) {
    dir[k] = 0;
    return;
  }
  const double v[3] = {__dmul_rn((double)kd[3 * k], r0), __dmul_rn((double)kd[3 * k + 1], r1),
                       __dmul_rn((double)kd[3 * k + 2], r2)};
  int a = 0;
  double M = fabs(v[0]);
  for (int i = 1; i < 3; ++i)
    if (fabs(v[i]) > M) {
      M = fabs(v[i]);
      a = i;
    }
  if (M == 0.0) {
    dir[k] = 0;
    return;
  }
  const int u = (a == 0) ? 1 : 0, w = (a == 2) ? 1 : 2;
  const double cu = __ddiv_rn(v[u], M), cw = __ddiv_rn(v[w], M);
  int j = 2 * a + (v[a] > 0.0 ? 1 : 0);
  double ulo = -1.0, uhi = 1.0, wlo = -1.0, whi = 1.0;
  for (int d = 0; d < lhf - level; ++d) {
    const double um = 0.5 * (ulo + uhi), wm = 0.5 * (wlo + whi);
    const int qu = cu > um ? 1 : 0, qw = cw > wm ? 1 : 0;
    if (qu) ulo = um; else uhi = um;
    if (qw) wlo = wm; else whi = wm;
    j = 4 * j + 2 * qu + qw;
  }
  dir[k] = j;
}

// D marks (Def. 4): kind[node * nD + dir(key)] = 1 (idempotent stores)
__global__ void k_mark_d(int64_t nb, const int32_t* __restrict__ node, const int32_t* __restrict__ key,
                         const int32_t* __restrict__ kdir, int nd, uint8_t* __restrict__ kind) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  kind[(int64_t)node[b] * nd + kdir[key[b]]] = 1;
}
// D^ from the parent's D u D^ (owner computes over the child)
__global__ void k_mark_dhat(int64_t nn, const int32_t* __restrict__ parent, const uint8_t* __restrict__ pkind,
                            int npd, int nd, int plevel, int lhf, uint8_t* __restrict__ kind) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  const int32_t p = parent[i];
  for (int c = 0; c < npd; ++c)
    if (pkind[(int64_t)p * npd + c]) {
      const int cc = (plevel + 1 > lhf) ? 0 : (c >> 2);
      kind[i * nd + cc] |= 2;
    }
}

// order-independent digest of the L+ rows (level, t coord, s coord, dir): sum of a
// splitmix64 row hash, the layout of plan.cpp structure_digest / oracle.cpp
__device__ __forceinline__ unsigned long long dmix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void k_lplus_digest(int64_t nb, FDH_PAIR_ARGS, const int32_t* __restrict__ key,
                               const int32_t* __restrict__ kdir, int level, unsigned long long* __restrict__ acc) {
  __shared__ unsigned long long sh[256];
  unsigned long long a = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = lpt[b], s = lps[b];
    const long long r[8] = {level, tci[t], tcj[t], tck[t], sci[s], scj[s], sck[s], kdir[key[b]]};
    unsigned long long h = 0x12345678ull;
#pragma unroll
    for (int i = 0; i < 8; ++i) h = dmix64(h ^ (unsigned long long)r[i]);
    a += h;
  }
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicAdd(acc, sh[0]);  // integer sum mod 2^64: exact in any order
}
// #L+ per target node (shard cost model); integer atomics, order-independent
__global__ void k_count_targets(int64_t nb, const int32_t* __restrict__ lpt, int32_t* __restrict__ cnt) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) atomicAdd(cnt + lpt[b], 1);
}
// keep the L+ blocks whose target is needed by this shard: flag, scan, stable emit
__global__ void k_needed_flags(int64_t nb, const int32_t* __restrict__ lpt, const uint8_t* __restrict__ need,
                               int64_t* __restrict__ f) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) f[b] = need[lpt[b]] ? 1 : 0;
}
__global__ void k_needed_emit(int64_t nb, const int32_t* __restrict__ lpt, const int32_t* __restrict__ lps,
                              const int32_t* __restrict__ key, const uint8_t* __restrict__ need,
                              const int64_t* __restrict__ pos, int32_t* __restrict__ ot, int32_t* __restrict__ os,
                              int32_t* __restrict__ ok) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb || !need[lpt[b]]) return;
  const int64_t o = pos[b];
  ot[o] = lpt[b];
  os[o] = lps[b];
  ok[o] = key[b];
}

}  // namespace

// ------------------------------------------------------------------ public
void gpu_build_structure(Plan& P, const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                         const double* sy, const double* sz, int64_t ns, const double lo[3], const double hi[3]) {
  Dev D;
  std::vector<DevLevel> dT, dS;
  tree_on_gpu(D, P.T, dT, tx, ty, tz, nt, lo, hi, P.prm.n_max, P.prm.depth_cap);
  tree_on_gpu(D, P.S, dS, sx, sy, sz, ns, lo, hi, P.prm.n_max, P.prm.depth_cap);
  // l_hf default and direction scale
  P.lhf = P.prm.l_hf;
  if (P.lhf == -2) {
    P.lhf = -1;
    for (int l = 0; l <= std::min(P.T.depth, P.S.depth); ++l)
      if (P.prm.kappa * std::max(P.T.diam[l], P.S.diam[l]) >= 3.0) P.lhf = l;
  }
  const double mn = std::min({P.T.side[0][0], P.T.side[0][1], P.T.side[0][2]});
  for (int a = 0; a < 3; ++a) P.rho[a] = P.T.side[0][a] / mn;

  // ---- block partition, level by level; candidate pairs in chunks of kPairChunk
  // (two passes: counts, then scan + emit at global offsets) so the scratch of a
  // 3e9-pair level (config 4) stays a few GB
  int64_t kPairChunk = (int64_t)1 << 27;
  if (const char* e = std::getenv("FDH_SETUP_PAIR_CHUNK")) kPairChunk = std::max(1024LL, std::atoll(e));  // testing
  const int maxl = std::min(P.T.depth, P.S.depth);
  P.blocks.assign(maxl + 1, {});
  int32_t* pt = D.up(std::vector<int32_t>{0});
  int32_t* ps = D.up(std::vector<int32_t>{0});
  int64_t np = 1;
  std::vector<int32_t*> lpt(maxl + 1, nullptr), lps(maxl + 1, nullptr), lpk(maxl + 1, nullptr);
  std::vector<int64_t> nlp(maxl + 1, 0);
  int32_t key_base = 0;
  for (int l = 0; np > 0; ++l) {
    if (l > maxl) throw PlanError{1, "internal: block recursion beyond tree depth"};
    LvlGeo g;
    g.q = std::max(P.T.diam[l], P.S.diam[l]);
    g.eta2 = P.prm.eta2;
    g.kappa = P.prm.kappa;
    for (int a = 0; a < 3; ++a) {
      g.tlo[a] = P.T.lo[a];
      g.slo[a] = P.S.lo[a];
      g.tside[a] = P.T.side[l][a];
      g.sside[a] = P.S.side[l][a];
    }
    const DevLevel& LT = dT[l];
    const DevLevel& LS = dS[l];
    const int64_t cap = std::min(np, kPairChunk);
    int64_t* olp = D.alloc<int64_t>(cap);
    int64_t* olm = D.alloc<int64_t>(cap);
    int64_t* onx = D.alloc<int64_t>(cap);
    // pass 1: totals per chunk
    std::vector<std::array<int64_t, 3>> ctot;
    for (int64_t c0 = 0; c0 < np; c0 += kPairChunk) {
      const int64_t nc = std::min(kPairChunk, np - c0);
      k_classify<<<nblocks(nc), 256>>>(nc, pt + c0, ps + c0, g, LT.ci, LT.cj, LT.ck, LS.ci, LS.cj, LS.ck, LT.leaf,
                                       LS.leaf, LT.child, LS.child, olp, olm, onx);
      SCK(cudaGetLastError());
      ctot.push_back({scan_excl(D, olp, nc), scan_excl(D, olm, nc), scan_excl(D, onx, nc)});
    }
    int64_t tlp = 0, tlm = 0, tnx = 0;
    for (auto& t : ctot) {
      tlp += t[0];
      tlm += t[1];
      tnx += t[2];
    }
    int32_t* a_t = D.alloc<int32_t>(tlp);
    int32_t* a_s = D.alloc<int32_t>(tlp);
    int32_t* m_t = D.alloc<int32_t>(tlm);
    int32_t* m_s = D.alloc<int32_t>(tlm);
    int32_t* n_t = D.alloc<int32_t>(tnx);
    int32_t* n_s = D.alloc<int32_t>(tnx);
    // pass 2: classify again, scan, emit at the chunk's global offsets
    int64_t blp = 0, blm = 0, bnx = 0;
    for (size_t ci = 0; ci * kPairChunk < (size_t)np; ++ci) {
      const int64_t c0 = (int64_t)ci * kPairChunk, nc = std::min(kPairChunk, np - c0);
      if (ctot.size() > 1) {
        k_classify<<<nblocks(nc), 256>>>(nc, pt + c0, ps + c0, g, LT.ci, LT.cj, LT.ck, LS.ci, LS.cj, LS.ck, LT.leaf,
                                         LS.leaf, LT.child, LS.child, olp, olm, onx);
        scan_excl(D, olp, nc);
        scan_excl(D, olm, nc);
        scan_excl(D, onx, nc);
      }
      k_emit<<<nblocks(nc), 256>>>(nc, pt + c0, ps + c0, olp, olm, onx, ctot[ci][0], ctot[ci][1], ctot[ci][2],
                                   LT.child, LS.child, a_t + blp, a_s + blp, m_t + blm, m_s + blm, n_t + bnx,
                                   n_s + bnx);
      SCK(cudaGetLastError());
      blp += ctot[ci][0];
      blm += ctot[ci][1];
      bnx += ctot[ci][2];
    }
    if (std::getenv("FDH_DEBUG_SETUP"))
      std::fprintf(stderr, "[setup] level %d: pairs %lld  L+ %lld  L- %lld  next %lld\n", l, (long long)np,
                   (long long)tlp, (long long)tlm, (long long)tnx);
    LevelBlocks& B = P.blocks[l];
    B.lm_t = down(m_t, tlm);
    B.lm_s = down(m_s, tlm);
    lpt[l] = a_t;
    lps[l] = a_s;
    nlp[l] = tlp;
    for (void* p : {(void*)olp, (void*)olm, (void*)onx, (void*)m_t, (void*)m_s, (void*)pt, (void*)ps}) D.release(p);
    // keys of this level: dense offset table, ids in (dx, dy, dz) order
    if (tlp > 0) {
      long long init[6] = {LLONG_MAX, LLONG_MAX, LLONG_MAX, LLONG_MIN, LLONG_MIN, LLONG_MIN};
      long long* mm = D.alloc<long long>(6);
      SCK(cudaMemcpy(mm, init, sizeof(init), cudaMemcpyHostToDevice));
      k_minmax<<<std::min<unsigned>(1024, nblocks(tlp)), 256>>>(tlp, a_t, a_s, LT.ci, LT.cj, LT.ck, LS.ci, LS.cj,
                                                                LS.ck, mm);
      std::vector<long long> m = down(mm, 6);
      const long long e0 = m[3] - m[0] + 1, e1 = m[4] - m[1] + 1, e2 = m[5] - m[2] + 1;
      const long long vol = e0 * e1 * e2;
      if (vol > (1ll << 28)) throw PlanError{4, "lattice offset range too large for the dense key table"};
      int64_t* tab = D.alloc<int64_t>(vol);
      SCK(cudaMemset(tab, 0, vol * 8));
      k_mark<<<nblocks(tlp), 256>>>(tlp, a_t, a_s, LT.ci, LT.cj, LT.ck, LS.ci, LS.cj, LS.ck, m[0], m[1], m[2], e1,
                                    e2, tab);
      int64_t* flag = D.alloc<int64_t>(vol);
      SCK(cudaMemcpy(flag, tab, vol * 8, cudaMemcpyDeviceToDevice));
      const int64_t nk = scan_excl(D, tab, vol);
      int32_t* key = D.alloc<int32_t>(tlp);
      k_keyids<<<nblocks(tlp), 256>>>(tlp, a_t, a_s, LT.ci, LT.cj, LT.ck, LS.ci, LS.cj, LS.ck, m[0], m[1], m[2], e1,
                                      e2, tab, key_base, key);
      int64_t* kd = D.alloc<int64_t>(3 * nk);
      k_keylist<<<nblocks(vol), 256>>>(vol, flag, tab, m[0], m[1], m[2], e1, e2, kd);
      int32_t* kdir = D.alloc<int32_t>(nk);
      k_keydir<<<nblocks(nk), 256>>>(nk, kd, l, P.lhf, P.rho[0], P.rho[1], P.rho[2], kdir);
      SCK(cudaGetLastError());
      const std::vector<int64_t> kdh = down(kd, 3 * nk);
      const std::vector<int32_t> kdirh = down(kdir, nk);
      for (int64_t k = 0; k < nk; ++k) {
        P.key_level.push_back(l);
        P.key_dx.push_back(kdh[3 * k]);
        P.key_dy.push_back(kdh[3 * k + 1]);
        P.key_dz.push_back(kdh[3 * k + 2]);
        P.key_dir.push_back(kdirh[k]);
      }
      lpk[l] = key;
      key_base += (int32_t)nk;
      for (void* p : {(void*)mm, (void*)tab, (void*)flag, (void*)kd, (void*)kdir}) D.release(p);
    }
    pt = n_t;
    ps = n_s;
    np = tnx;
  }
  P.n_sc = key_base;
  int32_t* kdir_all = D.up(P.key_dir);
  // ---- D / D^ and slots per tree (Def. 4)
  for (int w = 0; w < 2; ++w) {
    TreePlan& X = w == 0 ? P.T : P.S;
    const std::vector<DevLevel>& dl = w == 0 ? dT : dS;
    const int nl = X.depth + 1;
    X.ndir.resize(nl);
    X.kind.assign(nl, {});
    X.slot_of.assign(nl, {});
    std::vector<uint8_t*> kd(nl);
    for (int l = 0; l < nl; ++l) {
      X.ndir[l] = num_dirs(l, P.lhf);
      kd[l] = D.alloc<uint8_t>(dl[l].n * X.ndir[l]);
      SCK(cudaMemset(kd[l], 0, dl[l].n * X.ndir[l]));
      if (l < (int)P.blocks.size() && nlp[l] > 0)
        k_mark_d<<<nblocks(nlp[l]), 256>>>(nlp[l], w == 0 ? lpt[l] : lps[l], lpk[l], kdir_all, X.ndir[l], kd[l]);
      if (l > 0)
        k_mark_dhat<<<nblocks(dl[l].n), 256>>>(dl[l].n, dl[l].parent, kd[l - 1], X.ndir[l - 1], X.ndir[l], l - 1,
                                               P.lhf, kd[l]);
    }
    SCK(cudaGetLastError());
    int64_t s = 0;
    X.slot_level.clear();
    X.slot_node.clear();
    X.slot_dir.clear();
    for (int l = 0; l < nl; ++l) {
      X.kind[l] = down(kd[l], dl[l].n * X.ndir[l]);
      const int nd = X.ndir[l];
      X.slot_of[l].assign(X.kind[l].size(), -1);
      for (size_t i = 0; i < (size_t)dl[l].n; ++i)
        for (int c = 0; c < nd; ++c)
          if (X.kind[l][i * nd + c]) {
            X.slot_of[l][i * nd + c] = (int32_t)s++;
            X.slot_level.push_back(l);
            X.slot_node.push_back((int32_t)i);
            X.slot_dir.push_back(c);
          }
      D.release(kd[l]);
    }
    X.nslots = s;
  }
  // digest of the full L+ (the shard keeps only part of it on the host)
  {
    unsigned long long* acc = D.alloc<unsigned long long>(1);
    SCK(cudaMemset(acc, 0, sizeof(unsigned long long)));
    for (int l = 0; l <= maxl; ++l)
      if (nlp[l] > 0)
        k_lplus_digest<<<std::min<unsigned>(148 * 16, nblocks(nlp[l])), 256>>>(
            nlp[l], lpt[l], lps[l], dT[l].ci, dT[l].cj, dT[l].ck, dS[l].ci, dS[l].cj, dS[l].ck, lpk[l], kdir_all, l,
            acc);
    SCK(cudaGetLastError());
    P.lplus_digest = down(acc, 1)[0];
    P.lplus_digest_dev = true;
    D.release(acc);
  }
  P.n_c = 0;
  for (int l = 0; l <= maxl; ++l) P.n_c += nlp[l];
  // shards: the cost model from per-target L+ counts, ownership
  // and its ancestor closure on the host, then only the L+ blocks with a needed
  // target go to the host (config 4, rank r of 8: ~1/8 of the 3.47e9 blocks)
  const bool shard = P.prm.world > 1;
  if (shard) {
    P.lp_count.assign(maxl + 1, {});
    for (int l = 0; l <= maxl; ++l) {
      int32_t* cnt = D.alloc<int32_t>(dT[l].n);
      SCK(cudaMemset(cnt, 0, sizeof(int32_t) * dT[l].n));
      if (nlp[l] > 0) k_count_targets<<<nblocks(nlp[l]), 256>>>(nlp[l], lpt[l], cnt);
      SCK(cudaGetLastError());
      P.lp_count[l] = down(cnt, dT[l].n);
      D.release(cnt);
    }
    compute_ownership(P);
  }
  // L+ lists back to the host (the M2L tiles are assembled there)
  int64_t kChunk = (int64_t)1 << 27;
  if (const char* e = std::getenv("FDH_SETUP_PAIR_CHUNK")) kChunk = std::max(1024LL, std::atoll(e));  // testing
  for (int l = 0; l <= maxl; ++l) {
    LevelBlocks& B = P.blocks[l];
    if (!shard || nlp[l] == 0) {
      B.lp_t = down(lpt[l], nlp[l]);
      B.lp_s = down(lps[l], nlp[l]);
      B.lp_key = down(lpk[l], nlp[l]);
      continue;
    }
    std::vector<uint8_t> needh(P.t_needed[l].begin(), P.t_needed[l].end());
    uint8_t* need = D.up(needh);
    int64_t* f = D.alloc<int64_t>(std::min(nlp[l], kChunk));
    for (int64_t c0 = 0; c0 < nlp[l]; c0 += kChunk) {
      const int64_t nc = std::min(kChunk, nlp[l] - c0);
      k_needed_flags<<<nblocks(nc), 256>>>(nc, lpt[l] + c0, need, f);
      const int64_t k = scan_excl(D, f, nc);
      int32_t* ot = D.alloc<int32_t>(k);
      int32_t* os = D.alloc<int32_t>(k);
      int32_t* ok = D.alloc<int32_t>(k);
      k_needed_emit<<<nblocks(nc), 256>>>(nc, lpt[l] + c0, lps[l] + c0, lpk[l] + c0, need, f, ot, os, ok);
      SCK(cudaGetLastError());
      const auto ht = down(ot, k), hs = down(os, k), hk = down(ok, k);
      B.lp_t.insert(B.lp_t.end(), ht.begin(), ht.end());
      B.lp_s.insert(B.lp_s.end(), hs.begin(), hs.end());
      B.lp_key.insert(B.lp_key.end(), hk.begin(), hk.end());
      for (void* p : {(void*)ot, (void*)os, (void*)ok}) D.release(p);
    }
    D.release(f);
    D.release(need);
  }
  SCK(cudaDeviceSynchronize());
}

}  // namespace fdhelm
