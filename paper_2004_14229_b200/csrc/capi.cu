// capi.cu -- the C-ABI (include/fdhelm_c.h): operator setup, device residency
// and the Alg. 4 apply sequence on one CUDA stream.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is resolved at run time (dlopen), see nccl()
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges per setup stage and apply phase

#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fdhelm_c.h"
#include "kernels.hpp"
#include "plan.hpp"

using namespace fdhelm;

namespace {
thread_local std::string g_err;

struct CudaErr {
  std::string msg;
};
#define CK(x)                                                                                      \
  do {                                                                                             \
    cudaError_t e_ = (x);                                                                          \
    if (e_ != cudaSuccess) throw CudaErr{std::string(#x) + ": " + cudaGetErrorString(e_)};         \
  } while (0)

// NCCL, loaded on first multi-GPU use: the process's libnccl.so.2 if one is
// already loaded (e.g. by torch), else the system one -- no link-time dependency
struct NcclApi {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.CommInitAll = (decltype(api.CommInitAll))dlsym(h, "ncclCommInitAll");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
      api.Reduce = (decltype(api.Reduce))dlsym(h, "ncclReduce");
      api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
      api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    }
  }
  return api.CommInitAll && api.Reduce && api.Broadcast && api.GroupStart && api.GroupEnd ? &api : nullptr;
}
#define NK(x)                                                                                      \
  do {                                                                                             \
    ncclResult_t r_ = (x);                                                                         \
    if (r_ != ncclSuccess) throw CudaErr{std::string(#x) + ": " + nccl()->GetErrorString(r_)};     \
  } while (0)

struct LevelDev {
  int n = 0;
  int32_t *a = nullptr, *b = nullptr, *c = nullptr, *d = nullptr, *e = nullptr, *f = nullptr;
  int64_t* crd = nullptr;
};
}  // namespace

struct fdh_op {
  Plan P;
  int device = 0;
  cudaStream_t st = nullptr;
  std::vector<void*> allocs;
  int64_t bytes = 0;
  Consts* dC = nullptr;
  double* dirtab = nullptr;
  double kappa = 0.0;
  int64_t nt = 0, ns = 0;
  // trees (slot order)
  double *tx = nullptr, *ty = nullptr, *tz = nullptr, *sx = nullptr, *sy = nullptr, *sz = nullptr;
  uint32_t *perm_t = nullptr, *perm_s = nullptr;
  uint32_t* diag_slot = nullptr;  // zero diagonal: source slot of each target's original index
  int32_t* tslot_dir = nullptr;
  // S2M
  int n_s2m = 0;
  int32_t *s2m_slot = nullptr, *s2m_level = nullptr, *s2m_dir = nullptr;
  int64_t *s2m_ci = nullptr, *s2m_cj = nullptr, *s2m_ck = nullptr;
  uint32_t *s2m_beg = nullptr, *s2m_end = nullptr;
  std::vector<LevelDev> m2m, l2l;
  // L2T / P2P
  int n_leaf = 0;
  int32_t *l2t_level = nullptr, *l2t_slot0 = nullptr, *l2t_nslot = nullptr;
  int64_t *l2t_ci = nullptr, *l2t_cj = nullptr, *l2t_ck = nullptr;
  uint32_t *l2t_beg = nullptr, *l2t_end = nullptr;
  int64_t* p2p_ptr = nullptr;
  uint32_t *p2p_sbeg = nullptr, *p2p_send = nullptr;
  // M2L
  int n_item = 0, n_tile = 0;
  uint8_t *tile_cols = nullptr, *tile_cnt = nullptr, *tile_same = nullptr;
  int32_t *item_tile = nullptr, *item_seq = nullptr, *tile_keys = nullptr, *tile_src = nullptr,
          *tile_nitem = nullptr, *tile_tslot = nullptr;
  double* tile_acc = nullptr;
  int* ticket = nullptr;
  int* counter = nullptr;  // int8 M2L item-claim counters: passes x segments
  int64_t *item_k0 = nullptr, *item_k1 = nullptr;
  int32_t *key_level = nullptr, *key_dir = nullptr;
  int64_t* key_d = nullptr;
  double *W = nullptr, *mom = nullptr, *loc = nullptr;
  double* loc2 = nullptr;  // hybrid int8 M2L: the pair part's sums (added to loc after the M2L)
  // int8 tensor-core M2L (k_m2l_i8.cu): digits of W (setup) and of the moments (per apply)
  bool i8 = false;
  int nkq = 0;
  int8_t *Wq = nullptr, *Mq = nullptr;
  unsigned long long *lvmax_w = nullptr, *lvmax_v = nullptr;
  int32_t *tile_level_d = nullptr, *s_slot_level = nullptr;
  // on-the-fly coupling (W does not fit): segments of consecutive key chunks, 2-slot ring
  bool w_resident = true;
  struct Seg {
    int item0, item1;
    int64_t key0, key1;
    bool gen = true;   // generate the segment's W digits (on-the-fly mode; sub-segments share them)
    bool pair = false;  // items of the pair part (int8 pair / hybrid mode)
  };
  // int8 pair mode (P.m2l_pair): per-pair output buffer of one segment, the per-slot
  // pair lists and their cursors
  double* pair_out = nullptr;
  int64_t *red_ptr = nullptr, *red_idx = nullptr, *red_cur = nullptr;
  std::vector<Seg> segs;
  int64_t w_slot_keys = 0;
  double2* sctab = nullptr;  // (sin, cos)(i pi / 256), i < 512: near-field table sincos
  double2 *q = nullptr, *q4 = nullptr, *yslot = nullptr, *xin = nullptr, *yout = nullptr;
  int* flag = nullptr;
  bool timing = false;
  static constexpr int kRing = 64;
  cudaEvent_t ring[kRing][FDH_NPHASES + 6] = {};  // phase boundaries, M2L GEMM and P2P start/stop, L2T start
  cudaStream_t st2 = nullptr;                      // near field, concurrent with the far field
  cudaEvent_t ev_q = nullptr, ev_nf = nullptr;
  double2* ynear = nullptr;
  bool overlap_nf = false;
  int nsm = 148, nf_ctas = 1;  // persistent near-field grid when overlapped
  int ring_n = 0;                                 // applies recorded since the last reset
  int ring_done = 0;                              // ring entries already accumulated
  // timing inside the CUDA graph: the phase events are captured as external
  // event-record nodes (gev), read back after each replay
  cudaEvent_t gev[FDH_NPHASES + 6] = {};
  bool capturing_timed = false, gtimed = false, gpending = false;
  double tacc[FDH_NPHASES + 1] = {};              // accumulated phase / M2L-kernel ms
  int64_t tacc_n = 0;
  bool fresh = false;                              // ev_all holds an apply not yet collected
  double apply_ms_sum = 0.0;
  int64_t applies_collected = 0;
  cudaEvent_t ev[FDH_NPHASES + 1] = {};
  cudaEvent_t ev_all[2] = {};
  fdh_stats stats{};
  int64_t launches = 0;
  bool applied = false;
  int rank = 0, world = 1;
  int R = 1;  // right-hand sides per apply (rhs-major vectors)
  // the apply as one CUDA graph (captured on first use for a given (x, y, stream),
  // replayed after; the per-phase timing mode launches directly)
  bool graphs = true, graph_failed = false;
  cudaGraphExec_t gexec = nullptr;
  const void* gx = nullptr;
  const void* gy = nullptr;
  cudaStream_t gst = nullptr;
  int64_t graph_replays = 0;
  // ACA-compressed coupling (fdh_set_aca; opt-in, lossy): per-key rank (-1 dense),
  // factor offsets and the factors, resident in HBM
  double aca_eps = 0.0;
  int32_t* aca_rank = nullptr;
  int64_t *aca_uoff = nullptr, *aca_woff = nullptr;
  double2 *aca_U = nullptr, *aca_W = nullptr;
  std::vector<void*> aca_allocs;
  int64_t aca_bytes = 0;
  double aca_mean_rank = 0.0;
  // cached near-field kernel values (fdh_set_cache FDH_CACHE_NEARFIELD)
  int64_t *nf_koff = nullptr, *nf_poff = nullptr;
  uint32_t* nf_spos = nullptr;
  double2* nf_K = nullptr;
  std::vector<void*> nf_allocs;
  int64_t nf_bytes = 0;
  // multi-GPU operator (fdh_create with n_gpus > 1): one target-leaf shard per
  // device (rank g of n_gpus on device g), y reduced to device 0 over NCCL
  std::vector<fdh_op*> parts;
  std::vector<ncclComm_t> comms;

  ~fdh_op() {
    for (size_t g = 0; g < parts.size(); ++g) {
      cudaSetDevice(parts[g]->device);
      delete parts[g];
    }
    if (!parts.empty()) cudaSetDevice(0);  // the group's own buffers live on device 0
    for (ncclComm_t c : comms)
      if (c && nccl()) nccl()->CommDestroy(c);
    if (st) cudaStreamSynchronize(st);
    if (gexec) cudaGraphExecDestroy(gexec);
    for (void* p : allocs) cudaFree(p);
    for (void* p : aca_allocs) cudaFree(p);
    for (void* p : nf_allocs) cudaFree(p);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev_all)
      if (e) cudaEventDestroy(e);
    for (auto& r : ring)
      for (auto& e : r)
        if (e) cudaEventDestroy(e);
    for (auto& e : gev)
      if (e) cudaEventDestroy(e);
    if (st2) cudaStreamSynchronize(st2);
    if (ev_q) cudaEventDestroy(ev_q);
    if (ev_nf) cudaEventDestroy(ev_nf);
    if (st2) cudaStreamDestroy(st2);
    if (st) cudaStreamDestroy(st);
  }
  template <class T>
  T* alloc(size_t count) {
    if (count == 0) return nullptr;
    void* p = nullptr;
    const cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess)
      throw CudaErr{"cudaMalloc(" + std::to_string(count * sizeof(T)) + " B): " + cudaGetErrorString(e)};
    allocs.push_back(p);
    bytes += (int64_t)(count * sizeof(T));
    return static_cast<T*>(p);
  }
  template <class T>
  T* up(const std::vector<T>& v) {
    if (v.empty()) return nullptr;
    T* d = alloc<T>(v.size());
    CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  }
};

namespace {

int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}

void setup_device(fdh_op* o) {
  Plan& P = o->P;
  CK(cudaGetDevice(&o->device));
  CK(cudaStreamCreateWithFlags(&o->st, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&o->st2, cudaStreamNonBlocking));
  if (const char* e = std::getenv("FDH_OVERLAP_NEARFIELD")) o->overlap_nf = e[0] == '1';
  if (const char* e = std::getenv("FDH_CUDA_GRAPH")) o->graphs = e[0] != '0';
  CK(cudaDeviceGetAttribute(&o->nsm, cudaDevAttrMultiProcessorCount, o->device));
  if (const char* e = std::getenv("FDH_NF_CTAS")) o->nf_ctas = std::max(1, std::atoi(e));  // tuning knob
  CK(cudaEventCreateWithFlags(&o->ev_q, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&o->ev_nf, cudaEventDisableTiming));
  for (auto& e : o->ev) CK(cudaEventCreate(&e));
  for (auto& e : o->ev_all) CK(cudaEventCreate(&e));
  for (auto& r : o->ring)
    for (auto& e : r) CK(cudaEventCreate(&e));
  for (auto& e : o->gev) CK(cudaEventCreate(&e));
  // constants
  Consts C{};
  C.kappa = P.prm.kappa;
  C.m = P.prm.m;
  C.p = P.p;
  C.n = P.n;
  C.n_pad = P.n_pad;
  C.lhf = P.lhf;
  C.zero_diag = P.prm.zero_diagonal;
  for (int i = 0; i < P.p; ++i) C.cheb_cos[i] = P.cheb_cos[i];
  for (int h = 0; h < 2; ++h)
    for (int j = 0; j < P.p; ++j)
      for (int k = 0; k < P.p; ++k) C.half[(h * P.p + j) * P.p + k] = P.half[(h * P.p + j) * P.p + k];
  for (int a = 0; a < 3; ++a) {
    C.lo_t[a] = P.T.lo[a];
    C.lo_s[a] = P.S.lo[a];
  }
  if (P.T.depth >= kMaxLevels - 1 || P.S.depth >= kMaxLevels - 1) throw PlanError{4, "tree too deep"};
  for (int l = 0; l <= P.T.depth; ++l)
    for (int a = 0; a < 3; ++a) C.side_t[l][a] = P.T.side[l][a];
  for (int l = 0; l <= P.S.depth; ++l)
    for (int a = 0; a < 3; ++a) C.side_s[l][a] = P.S.side[l][a];
  std::vector<double> dt;
  for (int l = 0; l < (int)P.dirvec.size(); ++l) {
    C.dir_off[l] = (int)dt.size();
    dt.insert(dt.end(), P.dirvec[l].begin(), P.dirvec[l].end());
  }
  C.dir_off[P.dirvec.size()] = (int)dt.size();
  o->dC = o->alloc<Consts>(1);
  CK(cudaMemcpy(o->dC, &C, sizeof(C), cudaMemcpyHostToDevice));
  o->dirtab = o->up(dt);
  o->kappa = P.prm.kappa;
  // trees
  o->nt = (int64_t)P.T.perm.size();
  o->ns = (int64_t)P.S.perm.size();
  o->tx = o->up(P.T.x);
  o->ty = o->up(P.T.y);
  o->tz = o->up(P.T.z);
  o->sx = o->up(P.S.x);
  o->sy = o->up(P.S.y);
  o->sz = o->up(P.S.z);
  o->perm_t = o->up(P.T.perm);
  o->perm_s = o->up(P.S.perm);
  if (P.prm.zero_diagonal) {
    // zero diagonal: per target slot the source slot holding the same
    // original index (~0u if none), so the near field compares slot numbers
    std::vector<uint32_t> inv(P.S.perm.size()), dslot(P.T.perm.size(), ~0u);
    for (size_t k = 0; k < P.S.perm.size(); ++k) inv[P.S.perm[k]] = (uint32_t)k;
    for (size_t j = 0; j < P.T.perm.size(); ++j)
      if (P.T.perm[j] < P.S.perm.size()) dslot[j] = inv[P.T.perm[j]];
    o->diag_slot = o->up(dslot);
  }
  o->tslot_dir = o->up(P.T.slot_dir);
  // S2M
  o->n_s2m = (int)P.s2m_slot.size();
  o->s2m_slot = o->up(P.s2m_slot);
  o->s2m_level = o->up(P.s2m_level);
  o->s2m_dir = o->up(P.s2m_dir);
  o->s2m_ci = o->up(P.s2m_ci);
  o->s2m_cj = o->up(P.s2m_cj);
  o->s2m_ck = o->up(P.s2m_ck);
  o->s2m_beg = o->up(P.s2m_begin);
  o->s2m_end = o->up(P.s2m_end);
  // M2M / L2L per level
  o->m2m.assign(P.m2m_parent.size(), {});
  for (size_t l = 0; l < P.m2m_parent.size(); ++l) {
    LevelDev& D = o->m2m[l];
    D.n = (int)P.m2m_parent[l].size();
    D.a = o->up(P.m2m_parent[l]);
    D.b = o->up(P.m2m_dir[l]);
    D.c = o->up(P.m2m_cdir[l]);
    D.d = o->up(P.m2m_child[l]);
    D.crd = o->up(P.m2m_pc[l]);
  }
  o->l2l.assign(P.l2l_child.size(), {});
  for (size_t l = 0; l < P.l2l_child.size(); ++l) {
    LevelDev& D = o->l2l[l];
    D.n = (int)P.l2l_child[l].size();
    D.a = o->up(P.l2l_child[l]);
    D.b = o->up(P.l2l_cdir[l]);
    D.c = o->up(P.l2l_ptr[l]);
    D.d = o->up(P.l2l_pslot[l]);
    D.e = o->up(P.l2l_pdir[l]);
    D.f = o->up(P.l2l_oct[l]);
    D.crd = o->up(P.l2l_cc[l]);
  }
  // L2T / P2P
  o->n_leaf = (int)P.l2t_level.size();
  o->l2t_level = o->up(P.l2t_level);
  o->l2t_slot0 = o->up(P.l2t_slot0);
  o->l2t_nslot = o->up(P.l2t_nslot);
  o->l2t_ci = o->up(P.l2t_ci);
  o->l2t_cj = o->up(P.l2t_cj);
  o->l2t_ck = o->up(P.l2t_ck);
  o->l2t_beg = o->up(P.l2t_begin);
  o->l2t_end = o->up(P.l2t_end);
  o->p2p_ptr = o->up(P.p2p_ptr);
  o->p2p_sbeg = o->up(P.p2p_sbeg);
  o->p2p_send = o->up(P.p2p_send);
  // M2L
  o->n_item = (int)P.item_tile.size();
  o->n_tile = (int)P.tile_level.size();
  o->item_tile = o->up(P.item_tile);
  o->item_seq = o->up(P.item_seq);
  o->item_k0 = o->up(P.item_k0);
  o->item_k1 = o->up(P.item_k1);
  o->tile_keys = o->up(P.tile_keys);
  o->tile_src = o->up(P.tile_src);
  o->tile_cols = o->up(P.tile_cols);
  o->tile_cnt = o->up(P.tile_cnt);
  o->tile_same = o->up(P.tile_same);
  o->tile_nitem = o->up(P.tile_nitem);
  o->tile_tslot = o->up(P.tile_tslot);
  o->key_level = o->up(P.key_level);
  o->key_dir = o->up(P.key_dir);
  {
    std::vector<int64_t> kd(3 * P.key_level.size());
    for (size_t k = 0; k < P.key_level.size(); ++k) {
      kd[3 * k] = P.key_dx[k];
      kd[3 * k + 1] = P.key_dy[k];
      kd[3 * k + 2] = P.key_dz[k];
    }
    o->key_d = o->up(kd);
  }
  const int64_t np2 = 2 * (int64_t)P.n_pad;
  const int64_t nkeys = (int64_t)P.key_level.size();
  const int64_t wkey = P.n_pad * m2l_wplanes(P.n_pad) * (int64_t)P.n_k;  // doubles per coupling matrix
  const int64_t R = o->R = P.prm.nrhs;
  o->mom = o->alloc<double>((size_t)(R * P.S.nslots * np2));  // [rhs][slot][Re | Im]
  o->loc = o->alloc<double>((size_t)(R * P.T.nslots * np2));
  {  // chained tile accumulators of the target tiles (the pair part's tiles have one item: no chain)
    const int64_t nacc = P.m2l_pair ? P.m2l_pair_tile0 : (int64_t)o->n_tile;
    o->tile_acc = o->alloc<double>((size_t)std::max<int64_t>(1, nacc * P.n_pad * 2 * P.prm.tile));
  }
  o->ticket = o->alloc<int>((size_t)std::max(
      (P.prm.m2l_impl == 1 ? m2l_i8_passes(P.n, P.prm.tile) : 1) * o->n_tile, 1));  // one chain per M-block pass
  o->q = o->alloc<double2>((size_t)(R * o->ns));
  o->q4 = o->alloc<double2>((size_t)(R * o->ns));
  {
    std::vector<double2> tab(512);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int i = 0; i < 512; ++i) {
      const long double a = (long double)i * pi / 256.0L;
      tab[i] = make_double2((double)sinl(a), (double)cosl(a));
    }
    o->sctab = o->up(tab);
  }
  o->yslot = o->alloc<double2>((size_t)(R * o->nt));
  o->ynear = o->alloc<double2>((size_t)(R * o->nt));
  o->xin = o->alloc<double2>((size_t)(R * o->ns));
  o->yout = o->alloc<double2>((size_t)(R * o->nt));
  o->flag = o->alloc<int>(1);
  CK(cudaMemset(o->flag, 0, sizeof(int)));  // sticky between fdh_sync calls (device path)
  // coupling matrices: resident when they fit (70 % of the free
  // memory), else generated per apply in segments of key chunks (config 4: 240 GB)
  size_t fre = 0, tot = 0;
  CK(cudaMemGetInfo(&fre, &tot));
  const char* otf = std::getenv("FDH_W_ONTHEFLY");
  const bool force_otf = otf && otf[0] == '1';
  // segments of the chunk-major item list for a ring of 2 coupling slots of
  // slot_keys keys each (whole key chunks): cut where the chunk crosses a slot
  auto make_segments = [&](int64_t key_bytes) {
    double slot_bytes = std::min(8.0e9, 0.2 * (double)fre);
    if (const char* sm = std::getenv("FDH_W_SLOT_MB"))  // testing knob: small slots, many segments
      slot_bytes = std::max(1.0, std::atof(sm)) * 1048576.0;
    const int64_t slot_keys =
        std::max<int64_t>(P.m2l_chunk, (int64_t)(slot_bytes / (double)key_bytes) / P.m2l_chunk * P.m2l_chunk);
    o->w_slot_keys = slot_keys;
    const int64_t ni = (int64_t)P.item_tile.size();
    int64_t i = 0;
    while (i < ni) {
      const int64_t seg = P.tile_keys[P.item_k0[i]] / slot_keys;
      int64_t j = i;
      while (j < ni && P.tile_keys[P.item_k0[j]] / slot_keys == seg) ++j;
      o->segs.push_back({(int)i, (int)j, seg * slot_keys, std::min(nkeys, (seg + 1) * slot_keys)});
      i = j;
    }
    return slot_keys;
  };
  if (P.prm.m2l_impl == 1) {
    // int8 digits of the coupling matrices (k_m2l_i8.cu): per-level scales from a
    // first generation pass over every key (setup), digits from a second pass --
    // at setup for all keys when they fit (70 % of the free memory), else per
    // apply into a 2-slot ring in segments of key chunks (config 4: 229 GB)
    o->i8 = true;
    o->nkq = (P.n + 15) / 16 * 16;
    const int64_t wkq = m2l_i8_wbytes_per_key(P.n, o->nkq, P.prm.tile);
    const int64_t mq = m2l_i8_mbytes_per_slot(o->nkq) * P.S.nslots * R;
    o->w_resident = !force_otf && (double)(wkq * nkeys + mq) <= 0.7 * (double)fre;
    if (!o->w_resident && (double)mq > 0.3 * (double)fre) throw PlanError{-1, "int8 moment digits do not fit"};
    o->Mq = o->alloc<int8_t>((size_t)std::max<int64_t>(mq, 16));
    o->lvmax_w = o->alloc<unsigned long long>(kMaxLevels);
    o->lvmax_v = o->alloc<unsigned long long>(kMaxLevels * R);  // per (rhs, level)
    CK(cudaMemsetAsync(o->Mq, 0, (size_t)std::max<int64_t>(mq, 16), o->st));
    CK(cudaMemsetAsync(o->lvmax_w, 0, sizeof(unsigned long long) * kMaxLevels, o->st));
    o->tile_level_d = o->up(P.tile_level);
    o->s_slot_level = o->up(P.S.slot_level);
    const int64_t chunk = 4096;
    if (o->w_resident) {
      o->Wq = o->alloc<int8_t>((size_t)std::max<int64_t>(wkq * nkeys, 16));
      CK(cudaMemsetAsync(o->Wq, 0, (size_t)std::max<int64_t>(wkq * nkeys, 16), o->st));
      for (int pass = 0; pass < 2; ++pass)
        for (int64_t k0 = 0; k0 < nkeys; k0 += chunk)
          launch_coupling_i8(o->st, o->dC, o->dirtab, k0, std::min(chunk, nkeys - k0), o->key_level, o->key_d,
                             o->key_dir, pass, o->lvmax_w, o->Wq, P.n, o->nkq, m2l_i8_wgroup(P.n, P.prm.tile));
    } else {
      for (int64_t k0 = 0; k0 < nkeys; k0 += chunk)  // scales only
        launch_coupling_i8(o->st, o->dC, o->dirtab, k0, std::min(chunk, nkeys - k0), o->key_level, o->key_d,
                           o->key_dir, 0, o->lvmax_w, nullptr, P.n, o->nkq, m2l_i8_wgroup(P.n, P.prm.tile));
      const int64_t slot_keys = make_segments(wkq);
      o->Wq = o->alloc<int8_t>((size_t)(2 * slot_keys * wkq));
      CK(cudaMemsetAsync(o->Wq, 0, (size_t)(2 * slot_keys * wkq), o->st));  // padding rows / K stay zero
    }
    if (P.m2l_pair) {
      // pair part (pair / hybrid mode): segments cut at the first pair item and
      // into at most cap_items items (the pair output buffer), inside the W
      // segments when the digits are generated per apply
      CK(cudaMemGetInfo(&fre, &tot));
      double cap_bytes = std::min(8.0e9, 0.25 * (double)fre);
      if (const char* pb = std::getenv("FDH_PAIR_OUT_MB")) cap_bytes = std::max(1.0, std::atof(pb)) * 1048576.0;
      const int64_t TT = P.prm.tile;
      const int64_t cap_items = std::max<int64_t>(1, (int64_t)(cap_bytes / (16.0 * P.n_pad * TT)));
      const int ip0 = (int)P.m2l_pair_item0, ni = (int)P.item_tile.size();
      o->segs.clear();
      auto push_pairs = [&](int i0, int i1, int64_t k0, int64_t k1, bool gen) {
        for (int i = i0; i < i1; i += (int)cap_items) {
          o->segs.push_back({i, (int)std::min<int64_t>(i1, i + cap_items), k0, k1, gen, true});
          gen = false;
        }
      };
      if (o->w_resident) {
        if (ip0 > 0) o->segs.push_back({0, ip0, 0, nkeys, false, false});
        push_pairs(ip0, ni, 0, nkeys, false);
      } else {
        // per W slot (key range): its target-tile items, then its pair items, so the
        // slot's digits are generated once for both parts (both are key-ordered)
        const int64_t sk = o->w_slot_keys;
        auto slot_of = [&](int i) { return (int64_t)P.tile_keys[P.item_k0[i]] / sk; };
        int it = 0, ip = ip0;
        while (it < ip0 || ip < ni) {
          const int64_t sl = std::min(it < ip0 ? slot_of(it) : INT64_MAX, ip < ni ? slot_of(ip) : INT64_MAX);
          const int64_t k0 = sl * sk, k1 = std::min(nkeys, (sl + 1) * sk);
          bool gen = true;
          int j = it;
          while (j < ip0 && slot_of(j) == sl) ++j;
          if (j > it) {
            o->segs.push_back({it, j, k0, k1, true, false});
            gen = false;
          }
          it = j;
          j = ip;
          while (j < ni && slot_of(j) == sl) ++j;
          if (j > ip) push_pairs(ip, j, k0, k1, gen);
          ip = j;
        }
      }
      if (ip0 > 0) o->loc2 = o->alloc<double>((size_t)(P.T.nslots * 2 * P.n_pad));  // hybrid (one rhs)
      o->pair_out = o->alloc<double>((size_t)(cap_items * TT * 2 * P.n_pad));
      o->red_ptr = o->up(P.red_ptr);
      o->red_idx = o->up(P.red_idx);
      o->red_cur = o->alloc<int64_t>((size_t)std::max<int64_t>(1, P.T.nslots));
    }
    o->counter = o->alloc<int>((size_t)(m2l_i8_passes(P.n, P.prm.tile) * std::max<size_t>(1, o->segs.size())));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(o->st));
    return;
  }
  const double wbytes = 8.0 * (double)wkey * (double)nkeys;
  o->w_resident = !force_otf && wbytes <= 0.7 * (double)fre;
  if (o->w_resident) {
    o->W = o->alloc<double>((size_t)(nkeys * wkey));
    const int64_t chunk = 4096;
    for (int64_t k0 = 0; k0 < nkeys; k0 += chunk)
      launch_coupling(o->st, o->dC, o->dirtab, k0, std::min(chunk, nkeys - k0), o->key_level, o->key_d, o->key_dir,
                      o->W, P.n, P.n_pad, P.n_k, 0);
  } else {
    // ring of 2 slots, each ~min(8 GB, 20 % of free memory); segments = whole key chunks
    const int64_t slot_keys = make_segments(8 * wkey);
    o->W = o->alloc<double>((size_t)(2 * slot_keys * wkey));
  }
  o->counter = o->alloc<int>(std::max<size_t>(1, o->segs.size()));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(o->st));
  if (o->n_item > 0 && P.prm.m > 6)  // the FP64 DMMA kernels are compiled for m <= 6 (int8 path: any m)
    throw PlanError{4, "interpolation degree m=" + std::to_string(P.prm.m) + " has no compiled FP64 M2L kernel"};
}

// NVTX range per phase of the apply (host side: the launches / capture of the phase)
const char* const kPhaseName[FDH_NPHASES + 1] = {"fdh:h2d", "fdh:s2m", "fdh:m2m", "fdh:m2l", "fdh:l2l",
                                                 "fdh:l2t", "fdh:p2p", "fdh:d2h", "fdh:end"};
void rec(fdh_op* o, int ph, cudaStream_t st) {
  if (ph <= FDH_NPHASES) {
    if (ph > 0) nvtxRangePop();
    if (ph < FDH_NPHASES) nvtxRangePushA(kPhaseName[ph]);
  }
  if (!o->timing) return;
  if (o->capturing_timed)  // an event-record node of the graph being captured
    CK(cudaEventRecordWithFlags(o->gev[ph], st, cudaEventRecordExternal));
  else
    CK(cudaEventRecord(o->ring[o->ring_n % fdh_op::kRing][ph], st));
}

// Alg. 4 on the device: x_dev (original order) -> y_dev (original order); with
// R right-hand sides x and y hold R vectors each, rhs-major.  The M2L runs once
// for all of them (tile columns are (slot, rhs) pairs), the near field forms
// every kernel value once for up to 8 of them, the other passes run per rhs.
void apply_device(fdh_op* o, const double2* x, double2* y, cudaStream_t st, bool outer_events = true) {
  Plan& P = o->P;
  const int n = P.n, np = P.n_pad;
  const int R = o->R;
  const int64_t mstr = P.S.nslots * 2 * (int64_t)np, lstr = P.T.nslots * 2 * (int64_t)np;
  int64_t L = 0;
  if (outer_events) CK(cudaEventRecord(o->ev_all[0], st));  // (graph replays record them around the launch)
  rec(o, FDH_PHASE_H2D, st);
  for (int r = 0; r < R; ++r)
    launch_gather_charges(st, o->ns, o->perm_s, x + r * o->ns, o->q + r * o->ns, o->q4 + r * o->ns);
  L += R;
  rec(o, FDH_PHASE_S2M, st);
  for (int r = 0; r < R; ++r)
    launch_s2m(st, o->dC, o->dirtab, o->n_s2m, o->s2m_slot, o->s2m_level, o->s2m_dir, o->s2m_ci, o->s2m_cj,
               o->s2m_ck, o->s2m_beg, o->s2m_end, o->sx, o->sy, o->sz, o->q + r * o->ns, o->mom + r * mstr, n, np);
  L += R * (o->n_s2m > 0);
  rec(o, FDH_PHASE_M2M, st);
  for (int l = (int)o->m2m.size() - 1; l >= 0; --l) {
    const LevelDev& D = o->m2m[l];
    if (D.n == 0) continue;
    for (int r = 0; r < R; ++r) launch_m2m(st, o->dC, o->dirtab, l, D.n, D.a, D.b, D.c, D.d, D.crd, o->mom + r * mstr, n, np);
    L += R;
  }
  rec(o, FDH_PHASE_M2L, st);
  // near field (vi).  Sequential by default: on the main stream after the M2L.
  // FDH_OVERLAP_NEARFIELD=1 opts in to launching it on the second stream BEFORE
  // the M2L as a persistent grid of nf_ctas CTAs per SM (one near-field CTA beside
  // each M2L CTA, different pipes); measured no faster.
  auto near_field = [&](cudaStream_t snf, int grid) {
    rec(o, FDH_NPHASES + 3, snf);
    if (o->nf_K)
      launch_p2p_cached(snf, o->n_leaf, o->l2t_beg, o->l2t_end, o->nf_koff, o->nf_poff, o->nf_spos, o->nf_K, o->q,
                        o->ynear, R, o->ns, o->nt);
    else
      launch_p2p(snf, o->kappa, o->n_leaf, o->l2t_beg, o->l2t_end, o->p2p_ptr, o->p2p_sbeg, o->p2p_send, o->tx, o->ty,
                 o->tz, o->sx, o->sy, o->sz, o->q4, o->diag_slot, nullptr, P.prm.zero_diagonal, o->ynear, o->flag,
                 o->kappa * P.nf_max_dist, o->sctab, R, o->ns, o->nt, grid);
    L += (o->n_leaf > 0) * p2p_launches(R);
    rec(o, FDH_NPHASES + 4, snf);
  };
  if (o->overlap_nf) {
    CK(cudaEventRecord(o->ev_q, st));  // charges ready: the near field may start
    CK(cudaStreamWaitEvent(o->st2, o->ev_q, 0));
    near_field(o->st2, o->nsm * o->nf_ctas);
    CK(cudaEventRecord(o->ev_nf, o->st2));
  }
  CK(cudaMemsetAsync(o->loc, 0, sizeof(double) * (size_t)(R * lstr), st));
  const bool aca = o->n_item > 0 && o->aca_eps > 0.0;
  // ACA over a pair / hybrid plan: the low-rank M2L runs the target-tile items, the
  // pair part (partial (tile, key) rows) stays on the exact int8 path below
  const bool aca_pairs = aca && o->i8 && P.m2l_pair;
  if (aca && (!P.m2l_pair || P.m2l_pair_item0 > 0)) {
    // ACA-compressed coupling (fdh_set_aca): the low-rank M2L over the same plan
    CK(cudaMemsetAsync(o->ticket, 0, sizeof(int) * (size_t)o->n_tile, st));
    CK(cudaMemsetAsync(o->counter, 0, sizeof(int), st));
    M2LAcaArgs a;
    a.n_item = P.m2l_pair ? (int)P.m2l_pair_item0 : o->n_item;
    a.item_tile = o->item_tile;
    a.item_seq = o->item_seq;
    a.item_k0 = o->item_k0;
    a.item_k1 = o->item_k1;
    a.tile_nitem = o->tile_nitem;
    a.tile_tslot = o->tile_tslot;
    a.tile_keys = o->tile_keys;
    a.tile_src = o->tile_src;
    a.tile_cols = o->tile_cols;
    a.tile_cnt = o->tile_cnt;
    a.rank = o->aca_rank;
    a.uoff = o->aca_uoff;
    a.woff = o->aca_woff;
    a.U = o->aca_U;
    a.W = o->aca_W;
    a.mom = o->mom;
    a.tile_acc = o->tile_acc;
    a.ticket = o->ticket;
    a.loc = o->loc;
    a.counter = o->counter;
    rec(o, FDH_NPHASES + 1, st);
    if (launch_m2l_aca(st, n, np, P.prm.tile, a) != 0) throw PlanError{4, "ACA M2L: n > 384 not compiled"};
    if (!aca_pairs) rec(o, FDH_NPHASES + 2, st);
    L += 1;
  }
  if (aca && !aca_pairs) {
  } else if (o->n_item > 0 && o->i8) {
    const int npass = m2l_i8_passes(n, P.prm.tile);
    CK(cudaMemsetAsync(o->ticket, 0, sizeof(int) * (size_t)(npass * o->n_tile), st));
    CK(cudaMemsetAsync(o->counter, 0, sizeof(int) * (size_t)(npass * std::max<size_t>(1, o->segs.size())), st));
    launch_mom_quant(st, o->mom, o->s_slot_level, P.S.nslots, n, np, o->nkq, o->lvmax_v, o->Mq, R);
    M2LI8Args a;
    a.n_item = o->n_item;
    a.item_tile = o->item_tile;
    a.item_seq = o->item_seq;
    a.item_k0 = o->item_k0;
    a.item_k1 = o->item_k1;
    a.tile_nitem = o->tile_nitem;
    a.tile_tslot = o->tile_tslot;
    a.tile_level = o->tile_level_d;
    a.tile_keys = o->tile_keys;
    a.tile_src = o->tile_src;
    a.tile_cols = o->tile_cols;
    a.tile_cnt = o->tile_cnt;
    a.Wq = o->Wq;
    a.Mq = o->Mq;
    a.lvmax_w = o->lvmax_w;
    a.lvmax_v = o->lvmax_v;
    a.tile_acc = o->tile_acc;
    a.ticket = o->ticket;
    a.loc = o->loc;
    a.err = o->flag;
    a.nkq = o->nkq;
    a.n_pad = np;
    a.fkeys = P.prm.m2l_fkeys;
    a.n_tile = o->n_tile;
    a.nrhs = R;
    a.counter = o->counter;
    const int ng = npass;
    if (!aca_pairs) rec(o, FDH_NPHASES + 1, st);
    if (o->w_resident && o->segs.empty()) {
      if (launch_m2l_i8(st, n, P.prm.tile, a) != 0) throw PlanError{4, "no int8 M2L kernel for this n / tile"};
      L += 2 + ng;
    } else {
      // segments: W digits generated per apply into a 2-slot ring (when not
      // resident) and / or the pair part (pair / hybrid mode): per segment the
      // key-major M2L into the pair buffer, then the per-slot reduction into the
      // locals (a running sum in pair order = key order)
      if (P.m2l_pair)
        CK(cudaMemcpyAsync(o->red_cur, o->red_ptr, sizeof(int64_t) * (size_t)P.T.nslots, cudaMemcpyDeviceToDevice,
                           st));
      // hybrid: the pair part sums into its own buffer (running sum in pair order from 0)
      // and is added to the tiles' locals once at the end -- the same bits whatever the
      // order of tile and pair segments (the tiles' last items ASSIGN the locals)
      double* pair_sum = o->loc2 ? o->loc2 : o->loc;
      if (o->loc2) CK(cudaMemsetAsync(o->loc2, 0, sizeof(double) * (size_t)lstr, st));
      const int64_t wkq = m2l_i8_wbytes_per_key(n, o->nkq, P.prm.tile);
      const int64_t ip0 = P.m2l_pair_item0;
      int wslot = -1;
      int64_t wkey0 = -1;  // first key of the digits in the current W slot
      for (size_t sg = 0; sg < o->segs.size(); ++sg) {
        const auto& S = o->segs[sg];
        if (aca_pairs && !S.pair) continue;  // target-tile items done by the ACA kernel
        M2LI8Args b = a;
        b.item0 = S.item0;
        b.n_item = S.item1 - S.item0;
        b.counter = o->counter + sg * npass;
        if (!o->w_resident) {
          if (S.key0 != wkey0) {  // sub-segments of one key range share the slot's digits
            wkey0 = S.key0;
            wslot = (wslot + 1) & 1;
            launch_coupling_i8(st, o->dC, o->dirtab, S.key0, S.key1 - S.key0, o->key_level, o->key_d, o->key_dir, 1,
                               o->lvmax_w, o->Wq + (int64_t)wslot * o->w_slot_keys * wkq, n, o->nkq,
                               m2l_i8_wgroup(n, P.prm.tile), S.key0);
            L += 1;
          }
          b.Wq = o->Wq + (int64_t)wslot * o->w_slot_keys * wkq;
          b.key_base = S.key0;
        }
        if (S.pair) b.pair_out = o->pair_out;
        if (launch_m2l_i8(st, n, P.prm.tile, b) != 0) throw PlanError{4, "no int8 M2L kernel for this n / tile"};
        L += ng;
        if (S.pair) {
          launch_m2l_reduce(st, P.T.nslots, o->red_ptr, o->red_idx, o->red_cur, o->pair_out,
                            (S.item0 - ip0) * (int64_t)P.prm.tile, (S.item1 - ip0) * (int64_t)P.prm.tile, pair_sum, np);
          L += 1;
        }
      }
      if (o->loc2) {
        launch_m2l_add(st, o->loc, o->loc2, lstr);
        L += 2;
      }
      L += 3;
    }
    rec(o, FDH_NPHASES + 2, st);
  } else if (o->n_item > 0) {
    CK(cudaMemsetAsync(o->ticket, 0, sizeof(int) * (size_t)o->n_tile, st));
    CK(cudaMemsetAsync(o->counter, 0, sizeof(int) * std::max<size_t>(1, o->segs.size()), st));
    M2LArgs a;
    a.n_item = o->n_item;
    a.item_tile = o->item_tile;
    a.item_seq = o->item_seq;
    a.item_k0 = o->item_k0;
    a.item_k1 = o->item_k1;
    a.tile_nitem = o->tile_nitem;
    a.tile_tslot = o->tile_tslot;
    a.tile_keys = o->tile_keys;
    a.tile_src = o->tile_src;
    a.tile_cols = o->tile_cols;
    a.tile_cnt = o->tile_cnt;
    a.tile_same = o->tile_same;
    a.W = o->W;
    a.mom = o->mom;
    a.tile_acc = o->tile_acc;
    a.ticket = o->ticket;
    a.loc = o->loc;
    a.err = o->flag;
    a.counter = o->counter;
    rec(o, FDH_NPHASES + 1, st);
    if (o->w_resident) {
      if (launch_m2l_gemm(st, np, P.n_k, P.prm.tile, a) != 0)
        throw PlanError{4, "no M2L kernel for this n_pad / tile"};
    } else {
      for (size_t sg = 0; sg < o->segs.size(); ++sg) {
        const auto& S = o->segs[sg];
        double* slot = o->W + (int64_t)(sg & 1) * o->w_slot_keys * P.n_pad * m2l_wplanes(P.n_pad) * (int64_t)P.n_k;
        launch_coupling(st, o->dC, o->dirtab, S.key0, S.key1 - S.key0, o->key_level, o->key_d, o->key_dir, slot,
                        P.n, P.n_pad, P.n_k, S.key0);
        M2LArgs b = a;
        b.item0 = S.item0;
        b.n_item = S.item1 - S.item0;
        b.W = slot;
        b.key_base = S.key0;
        b.counter = o->counter + sg;
        if (launch_m2l_gemm(st, np, P.n_k, P.prm.tile, b) != 0)
          throw PlanError{4, "no M2L kernel for this n_pad / tile"};
        L += 2;
      }
    }
    rec(o, FDH_NPHASES + 2, st);
    L += 1;
  }
  if (!o->overlap_nf) near_field(st, 0);
  rec(o, FDH_PHASE_L2L, st);
  for (int l = 0; l < (int)o->l2l.size(); ++l) {
    const LevelDev& D = o->l2l[l];
    if (D.n == 0) continue;
    for (int r = 0; r < R; ++r)
      launch_l2l(st, o->dC, o->dirtab, l, D.n, D.a, D.b, D.crd, D.c, D.d, D.e, D.f, o->loc + r * lstr, n, np);
    L += R;
  }
  rec(o, FDH_PHASE_L2T, st);
  if (o->world > 1) CK(cudaMemsetAsync(o->yslot, 0, sizeof(double2) * (size_t)(R * o->nt), st));
  if (o->overlap_nf) CK(cudaStreamWaitEvent(st, o->ev_nf, 0));
  rec(o, FDH_NPHASES + 5, st);  // L2T proper starts once the near field is done
  for (int r = 0; r < R; ++r)
    launch_l2t(st, o->dC, o->dirtab, o->n_leaf, o->l2t_level, o->l2t_slot0, o->l2t_nslot, o->l2t_ci, o->l2t_cj,
               o->l2t_ck, o->l2t_beg, o->l2t_end, o->tx, o->ty, o->tz, o->tslot_dir, o->loc + r * lstr,
               o->ynear + r * o->nt, o->yslot + r * o->nt, n, np);
  L += R * (o->n_leaf > 0);
  rec(o, FDH_PHASE_P2P, st);  // (P2P itself ran concurrently on st2: see collect_times)
  rec(o, FDH_PHASE_D2H, st);
  for (int r = 0; r < R; ++r) launch_scatter_y(st, o->nt, o->perm_t, o->yslot + r * o->nt, y + r * o->nt);
  L += R;
  rec(o, FDH_NPHASES, st);
  if (outer_events) CK(cudaEventRecord(o->ev_all[1], st));
  CK(cudaGetLastError());
  o->launches = L;
  o->applied = true;
  if (outer_events) o->fresh = true;
  if (o->timing && !o->capturing_timed) ++o->ring_n;
}

// apply_device through a CUDA graph: ~10-20 kernel launches + memsets per apply
// become one graph launch (capture in relaxed mode: cudaFuncSetAttribute is
// called inside).  Any capture / instantiate failure disables graphs for the
// operator and the apply runs directly.
void collect_times(fdh_op* o);
void apply_graph(fdh_op* o, const double2* x, double2* y, cudaStream_t st) {
  if (!o->graphs || o->graph_failed) {
    apply_device(o, x, y, st);
    return;
  }
  if (o->gpending) {  // the previous replay's phase events must be read before they are re-recorded
    CK(cudaEventSynchronize(o->ev_all[1]));
    collect_times(o);
  }
  if (!(o->gexec && o->gx == x && o->gy == y && o->gst == st && o->gtimed == o->timing)) {
    if (o->gexec) {
      CK(cudaGraphExecDestroy(o->gexec));
      o->gexec = nullptr;
    }
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      o->capturing_timed = o->timing;
      try {
        apply_device(o, x, y, st, false);
      } catch (...) {
        ok = false;
      }
      o->capturing_timed = false;
      ok = (cudaStreamEndCapture(st, &g) == cudaSuccess) && ok && g != nullptr;
    }
    if (ok) ok = cudaGraphInstantiate(&o->gexec, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {
      (void)cudaGetLastError();
      o->gexec = nullptr;
      o->graph_failed = true;
      apply_device(o, x, y, st);
      return;
    }
    o->gx = x;
    o->gy = y;
    o->gst = st;
    o->gtimed = o->timing;
  }
  CK(cudaEventRecord(o->ev_all[0], st));
  CK(cudaGraphLaunch(o->gexec, st));
  CK(cudaEventRecord(o->ev_all[1], st));
  o->applied = true;
  o->fresh = true;
  if (o->gtimed) o->gpending = true;
  ++o->graph_replays;
}

// per-phase times of one apply from its event set (ring entry or graph events)
void phase_times(fdh_op* o, cudaEvent_t* E, double* acc) {
  float ms = 0;
  for (int ph = 0; ph < FDH_NPHASES; ++ph) {
    CK(cudaEventElapsedTime(&ms, E[ph], E[ph + 1]));
    acc[ph] += ms;
  }
  if (o->n_item > 0) {
    CK(cudaEventElapsedTime(&ms, E[FDH_NPHASES + 1], E[FDH_NPHASES + 2]));
    acc[FDH_NPHASES] += ms;
  }
  // L2T excludes the wait for the concurrent near field
  CK(cudaEventElapsedTime(&ms, E[FDH_PHASE_L2T], E[FDH_PHASE_L2T + 1]));
  acc[FDH_PHASE_L2T] -= ms;
  CK(cudaEventElapsedTime(&ms, E[FDH_NPHASES + 5], E[FDH_PHASE_L2T + 1]));
  acc[FDH_PHASE_L2T] += ms;
  CK(cudaEventElapsedTime(&ms, E[FDH_NPHASES + 3], E[FDH_NPHASES + 4]));
  acc[FDH_PHASE_P2P] += ms;  // replaces the (empty) P2P slot between L2T and D2H
  if (!o->overlap_nf) acc[FDH_PHASE_M2L] -= ms;  // sequential: it ran inside the M2L interval
  CK(cudaEventElapsedTime(&ms, E[FDH_PHASE_P2P], E[FDH_PHASE_P2P + 1]));
  acc[FDH_PHASE_P2P] -= ms;
}

void collect_times(fdh_op* o) {
  if (!o->applied) return;
  float ms = 0;
  if (o->fresh) {
    CK(cudaEventElapsedTime(&ms, o->ev_all[0], o->ev_all[1]));
    o->stats.apply_ms = ms;
    o->apply_ms_sum += ms;
    ++o->applies_collected;
    o->fresh = false;
  }
  // phase times accumulated since the last fdh_set_timing: graph replays (one
  // event set, read after each replay) and direct launches (ring of 64)
  if (o->gpending) {
    phase_times(o, o->gev, o->tacc);
    ++o->tacc_n;
    o->gpending = false;
  }
  if (o->ring_n - o->ring_done > fdh_op::kRing) o->ring_done = o->ring_n - fdh_op::kRing;
  for (; o->ring_done < o->ring_n; ++o->ring_done) {
    phase_times(o, o->ring[o->ring_done % fdh_op::kRing], o->tacc);
    ++o->tacc_n;
  }
  if (o->tacc_n > 0) {
    for (int ph = 0; ph < FDH_NPHASES; ++ph) o->stats.phase_ms[ph] = o->tacc[ph] / o->tacc_n;
    o->stats.m2l_gemm_ms = o->tacc[FDH_NPHASES] / o->tacc_n;
    o->stats.timed_applies = o->tacc_n;
  }
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return FDH_OK;
  } catch (const PlanError& e) {
    return fail(e.code, e.msg);
  } catch (const CudaErr& e) {
    return fail(FDH_ERR_CUDA, e.msg);
  } catch (const std::bad_alloc&) {
    return fail(FDH_ERR_MEMORY, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(FDH_ERR_ARG, e.what());
  }
}

int create_common(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                  const double* sy, const double* sz, int64_t ns, const double lo[3], const double hi[3],
                  double kappa, int n_max, int m, double eta2, int l_hf, int depth_cap, int zero_diagonal, int rank,
                  int world, fdh_op** out, bool device = true, int nrhs = 1) {
  if (!out) return fail(FDH_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (!tx || !ty || !tz || !sx || !sy || !sz || !lo || !hi) return fail(FDH_ERR_ARG, "NULL input pointer");
  if (world < 1 || rank < 0 || rank >= world) return fail(FDH_ERR_ARG, "invalid rank / world");
  if (nrhs < 1 || nrhs > 16 || (nrhs & (nrhs - 1)) != 0)
    return fail(FDH_ERR_ARG, "nrhs must be a power of two in 1..16");
  int ndev = 0;
  if (device && (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0))
    return fail(FDH_ERR_CUDA, "no CUDA device available");
  fdh_op* o = new fdh_op;
  const int rc = guard([&] {
    const auto t0 = std::chrono::steady_clock::now();
    PlanParams prm;
    prm.kappa = kappa;
    prm.n_max = n_max;
    prm.m = m;
    prm.eta2 = eta2;
    prm.l_hf = l_hf;
    prm.depth_cap = depth_cap;
    prm.zero_diagonal = zero_diagonal;
    prm.rank = rank;
    prm.world = world;
    prm.nrhs = nrhs;
    const char* hs = std::getenv("FDH_HOST_STRUCTURE");  // testing knob: host planner for the structure
    prm.gpu_structure = device && !(hs && hs[0] == '1');
    o->rank = rank;
    o->world = world;
    // M2L implementation: the int8 tcgen05 kernel where it is compiled (n <= 384
    // nodes per box, i.e. m <= 6), FP64 DMMA otherwise; FDH_M2L_IMPL=dmma overrides
    const int nbox = (m + 1) * (m + 1) * (m + 1);
    const char* mi = std::getenv("FDH_M2L_IMPL");
    const char* pi = std::getenv("FDH_PLAN_I8");  // analysis knob: plan-only operators with the int8 plan
    const bool want_i8 = (device || (pi && pi[0] == '1')) && m >= 1 && !(mi && std::string(mi) == "dmma");
    if (want_i8) {
      prm.m2l_impl = 1;
      // 16 target columns for two / three M-blocks (m = 5, 6); beyond, one 128-row
      // M-block per pass with 32 columns (any degree: m = 7 .. 10)
      // 32 target columns for one M-block (m <= 4) and beyond three (m >= 7); for
      // m = 5, 6 the planner chooses 16 or 32 from the sampled key-list overlap
      prm.tile = (nbox <= 128 || nbox > 384) ? 32 : -1;
      if (const char* tt = std::getenv("FDH_I8_TILE"))  // testing knob: force 16 or 32 for m = 5, 6
        prm.tile = prm.tile > 0 ? prm.tile : (std::atoi(tt) == 32 ? 32 : 16);
      prm.i8_digits = kI8Digits;
      prm.m2l_fkeys = m2l_i8_fkeys((nbox + 15) / 16 * 16);
      if (const char* fk = std::getenv("FDH_M2L_FKEYS"))  // testing knob: shorter items (more chaining)
        prm.m2l_fkeys = std::max(1, std::min(prm.m2l_fkeys, std::atoi(fk)));
    }
    nvtxRangePushA("fdh:setup:plan");
    build_plan(o->P, tx, ty, tz, nt, sx, sy, sz, ns, lo, hi, prm);
    nvtxRangePop();
    if (device) {
      try {
        nvtxRangePushA("fdh:setup:device");
        setup_device(o);
        nvtxRangePop();
      } catch (const PlanError& e) {
        if (e.code != -1) throw;
        // int8 moment digits do not fit: rebuild with the FP64 DMMA path
        delete o;
        o = new fdh_op;
        o->rank = rank;
        o->world = world;
        prm.m2l_impl = 0;
        prm.tile = 16;
        prm.m2l_fkeys = 0;
        build_plan(o->P, tx, ty, tz, nt, sx, sy, sz, ns, lo, hi, prm);
        setup_device(o);
      }
    }
    o->stats.setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  });
  if (rc != FDH_OK) {
    delete o;
    return rc;
  }
  *out = o;
  return FDH_OK;
}

// Multi-GPU apply: x on device 0 (xd) is broadcast to every shard over NCCL,
// every device applies its shard (its own stream, CUDA-graph replay), the shard
// outputs are summed into yd on device 0 by an NCCL reduce.  All on the shards'
// streams; the caller's stream on device 0 is joined by events.
void group_apply(fdh_op* G, const double2* xd, double2* yd, cudaStream_t st0) {
  const int N = (int)G->parts.size();
  fdh_op* p0 = G->parts[0];
  if (st0 && st0 != p0->st) {  // order after the caller's work on its stream
    CK(cudaSetDevice(p0->device));
    CK(cudaEventRecord(p0->ev_q, st0));
    CK(cudaStreamWaitEvent(p0->st, p0->ev_q, 0));
  }
  NK(nccl()->GroupStart());
  for (int g = 0; g < N; ++g) {
    fdh_op* p = G->parts[g];
    CK(cudaSetDevice(p->device));
    NK(nccl()->Broadcast(xd, g == 0 ? (void*)xd : (void*)p->xin, 2 * (size_t)p->ns, ncclDouble, 0, G->comms[g],
                         p->st));
  }
  NK(nccl()->GroupEnd());
  for (int g = 0; g < N; ++g) {
    fdh_op* p = G->parts[g];
    CK(cudaSetDevice(p->device));
    apply_graph(p, g == 0 ? xd : p->xin, p->yout, p->st);
  }
  NK(nccl()->GroupStart());
  for (int g = 0; g < N; ++g) {
    fdh_op* p = G->parts[g];
    CK(cudaSetDevice(p->device));
    NK(nccl()->Reduce(p->yout, yd, 2 * (size_t)p->nt, ncclDouble, ncclSum, 0, G->comms[g], p->st));
  }
  NK(nccl()->GroupEnd());
  if (st0 && st0 != p0->st) {
    CK(cudaSetDevice(p0->device));
    CK(cudaEventRecord(p0->ev_nf, p0->st));
    CK(cudaStreamWaitEvent(st0, p0->ev_nf, 0));
  }
  CK(cudaSetDevice(p0->device));
}

void group_sync(fdh_op* G, int* flag_or) {
  for (fdh_op* p : G->parts) {
    CK(cudaSetDevice(p->device));
    CK(cudaStreamSynchronize(p->st));
    int f = 0;
    CK(cudaMemcpy(&f, p->flag, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemset(p->flag, 0, sizeof(int)));
    collect_times(p);
    *flag_or |= f;
  }
  CK(cudaSetDevice(G->parts[0]->device));
}

}  // namespace

extern "C" {

const char* fdh_last_error(void) { return g_err.c_str(); }
const char* fdh_version(void) { return "fdhelm-b200 0.2 (sm_100a; M2L: tcgen05 int8 digit products, FP64 DMMA selectable)"; }

int fdh_create(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx, const double* sy,
               const double* sz, int64_t ns, const double root_lo[3], const double root_hi[3], double kappa, int n_max,
               int m, double eta2, int l_hf, int depth_cap, int zero_diagonal, int n_gpus, fdh_op** out) {
  if (!out) return fail(FDH_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n_gpus < 1) return fail(FDH_ERR_ARG, "n_gpus must be >= 1");
  const char* grp = std::getenv("FDH_GROUP");  // testing knob: the multi-GPU path with n_gpus = 1
  if (n_gpus == 1 && !(grp && grp[0] == '1'))
    return create_common(tx, ty, tz, nt, sx, sy, sz, ns, root_lo, root_hi, kappa, n_max, m, eta2, l_hf, depth_cap,
                         zero_diagonal, 0, 1, out);
  // one process, n_gpus devices (SURVEY.md 8(b) "internally multi-GPU"): rank g of
  // n_gpus (cost-balanced target-leaf shard, fdh_create_shard) on device g, the
  // shards set up concurrently by one host thread each; y is reduced over NCCL
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < n_gpus)
    return fail(FDH_ERR_UNSUPPORTED, "n_gpus = " + std::to_string(n_gpus) + " needs that many CUDA devices, found " +
                                         std::to_string(ndev));
  if (!nccl()) return fail(FDH_ERR_UNSUPPORTED, "n_gpus > 1 needs libnccl.so.2 (not found)");
  fdh_op* g = new fdh_op;
  g->parts.assign(n_gpus, nullptr);
  g->nt = nt;
  g->ns = ns;
  std::vector<int> rc(n_gpus, FDH_OK);
  std::vector<std::string> msg(n_gpus);
  const auto t0 = std::chrono::steady_clock::now();
  {
    std::vector<std::thread> th;
    for (int d = 0; d < n_gpus; ++d)
      th.emplace_back([&, d] {
        if (cudaSetDevice(d) != cudaSuccess) {
          rc[d] = FDH_ERR_CUDA;
          msg[d] = "cudaSetDevice failed";
          return;
        }
        rc[d] = create_common(tx, ty, tz, nt, sx, sy, sz, ns, root_lo, root_hi, kappa, n_max, m, eta2, l_hf,
                              depth_cap, zero_diagonal, d, n_gpus, &g->parts[d]);
        if (rc[d] != FDH_OK) msg[d] = g_err;
      });
    for (auto& t : th) t.join();
  }
  for (int d = 0; d < n_gpus; ++d)
    if (rc[d] != FDH_OK) {
      const int r = rc[d];
      const std::string m = "device " + std::to_string(d) + ": " + msg[d];
      delete g;
      return fail(r, m);
    }
  const int r = guard([&] {
    std::vector<int> devs(n_gpus);
    for (int d = 0; d < n_gpus; ++d) devs[d] = d;
    g->comms.assign(n_gpus, nullptr);
    NK(nccl()->CommInitAll(g->comms.data(), n_gpus, devs.data()));
    CK(cudaSetDevice(0));
    g->yout = g->alloc<double2>((size_t)nt);  // the reduced y on device 0
  });
  if (r != FDH_OK) {
    delete g;
    return r;
  }
  g->stats.setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  *out = g;
  return FDH_OK;
}

int fdh_create_shard(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                     const double* sy, const double* sz, int64_t ns, const double root_lo[3], const double root_hi[3],
                     double kappa, int n_max, int m, double eta2, int l_hf, int depth_cap, int zero_diagonal, int rank,
                     int world, fdh_op** out) {
  return create_common(tx, ty, tz, nt, sx, sy, sz, ns, root_lo, root_hi, kappa, n_max, m, eta2, l_hf, depth_cap,
                       zero_diagonal, rank, world, out);
}

int fdh_create_multi(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx,
                     const double* sy, const double* sz, int64_t ns, const double root_lo[3], const double root_hi[3],
                     double kappa, int n_max, int m, double eta2, int l_hf, int depth_cap, int zero_diagonal, int rank,
                     int world, int nrhs, fdh_op** out) {
  return create_common(tx, ty, tz, nt, sx, sy, sz, ns, root_lo, root_hi, kappa, n_max, m, eta2, l_hf, depth_cap,
                       zero_diagonal, rank, world, out, true, nrhs);
}

int fdh_plan_only(const double* tx, const double* ty, const double* tz, int64_t nt, const double* sx, const double* sy,
                  const double* sz, int64_t ns, const double root_lo[3], const double root_hi[3], double kappa,
                  int n_max, int m, double eta2, int l_hf, int depth_cap, int zero_diagonal, int rank, int world,
                  fdh_op** out) {
  return create_common(tx, ty, tz, nt, sx, sy, sz, ns, root_lo, root_hi, kappa, n_max, m, eta2, l_hf, depth_cap,
                       zero_diagonal, rank, world, out, false);
}

void fdh_destroy(fdh_op* op) { delete op; }

int fdh_apply_multi(fdh_op* o, const double* x, int64_t k, double* y) {
  if (!o || !x || !y) return fail(FDH_ERR_ARG, "NULL argument");
  if (k < 1) return fail(FDH_ERR_ARG, "need at least one right-hand side");
  if (!o->parts.empty()) {
    return guard([&] {
      fdh_op* p0 = o->parts[0];
      for (int64_t b = 0; b < k; ++b) {
        CK(cudaSetDevice(p0->device));
        CK(cudaMemcpyAsync(p0->xin, x + 2 * b * o->ns, sizeof(double2) * (size_t)o->ns, cudaMemcpyHostToDevice,
                           p0->st));
        group_apply(o, p0->xin, o->yout, nullptr);
        CK(cudaSetDevice(p0->device));
        CK(cudaMemcpyAsync(y + 2 * b * o->nt, o->yout, sizeof(double2) * (size_t)o->nt, cudaMemcpyDeviceToHost,
                           p0->st));
        int flag = 0;
        group_sync(o, &flag);
        if (flag & 1) throw PlanError{FDH_ERR_DOMAIN, "Helmholtz kernel is singular at x == y (near field)"};
      }
    });
  }
  if (!o->st) return fail(FDH_ERR_UNSUPPORTED, "operator was built with fdh_plan_only (no device state)");
  return guard([&] {
    CK(cudaSetDevice(o->device));
    const int64_t R = o->R;
    for (int64_t b = 0; b < k; b += R) {  // batches of R vectors; a short last batch runs with zero vectors
      const int64_t nb = std::min(R, k - b);
      if (nb < R)
        CK(cudaMemsetAsync(o->xin + nb * o->ns, 0, sizeof(double2) * (size_t)((R - nb) * o->ns), o->st));
      CK(cudaMemcpyAsync(o->xin, x + 2 * b * o->ns, sizeof(double2) * (size_t)(nb * o->ns), cudaMemcpyHostToDevice,
                         o->st));
      CK(cudaMemsetAsync(o->flag, 0, sizeof(int), o->st));
      apply_graph(o, o->xin, o->yout, o->st);
      CK(cudaMemcpyAsync(y + 2 * b * o->nt, o->yout, sizeof(double2) * (size_t)(nb * o->nt),
                         cudaMemcpyDeviceToHost, o->st));
      int flag = 0;
      CK(cudaMemcpyAsync(&flag, o->flag, sizeof(int), cudaMemcpyDeviceToHost, o->st));
      CK(cudaStreamSynchronize(o->st));
      collect_times(o);
      if (flag & 1) throw PlanError{FDH_ERR_DOMAIN, "Helmholtz kernel is singular at x == y (near field)"};
    }
  });
}

int fdh_apply(fdh_op* o, const double* x, double* y) { return fdh_apply_multi(o, x, 1, y); }

int fdh_apply_device(fdh_op* o, const double* x_dev, double* y_dev, void* stream) {
  if (!o || !x_dev || !y_dev) return fail(FDH_ERR_ARG, "NULL argument");
  if (!o->parts.empty())  // multi-GPU: x_dev / y_dev / stream on device 0
    return guard([&] {
      group_apply(o, reinterpret_cast<const double2*>(x_dev), reinterpret_cast<double2*>(y_dev),
                  static_cast<cudaStream_t>(stream));
    });
  if (!o->st) return fail(FDH_ERR_UNSUPPORTED, "operator was built with fdh_plan_only (no device state)");
  return guard([&] {
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : o->st;
    apply_graph(o, reinterpret_cast<const double2*>(x_dev), reinterpret_cast<double2*>(y_dev), st);
  });
}

int fdh_set_aca(fdh_op* o, double eps) {
  if (!o) return fail(FDH_ERR_ARG, "NULL op");
  if (!(eps >= 0.0 && eps < 1.0)) return fail(FDH_ERR_ARG, "ACA tolerance must be in [0, 1)");
  for (fdh_op* p : o->parts) {
    cudaSetDevice(p->device);
    if (const int rc = fdh_set_aca(p, eps)) return rc;
  }
  if (!o->parts.empty()) {
    cudaSetDevice(0);
    o->aca_eps = eps;
    return FDH_OK;
  }
  if (!o->st) return fail(FDH_ERR_UNSUPPORTED, "operator was built with fdh_plan_only (no device state)");
  if (o->R != 1) return fail(FDH_ERR_UNSUPPORTED, "ACA with several right-hand sides is not supported");
  return guard([&] {
    CK(cudaSetDevice(o->device));
    CK(cudaStreamSynchronize(o->st));
    for (void* p : o->aca_allocs) cudaFree(p);
    o->aca_allocs.clear();
    o->aca_eps = 0.0;
    o->aca_bytes = 0;
    o->gx = nullptr;  // re-capture the apply graph
    if (o->gexec) {
      CK(cudaGraphExecDestroy(o->gexec));
      o->gexec = nullptr;
    }
    if (eps == 0.0) return;
    Plan& P = o->P;
    const int n = P.n;
    if (n > 384) throw PlanError{FDH_ERR_UNSUPPORTED, "ACA M2L is compiled for n <= 384 (m <= 6)"};
    const int64_t nkeys = (int64_t)P.key_level.size();
    auto dalloc = [&](size_t bytes) {
      void* p = nullptr;
      const cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 16));
      if (e != cudaSuccess) throw PlanError{FDH_ERR_MEMORY, "ACA factors do not fit in device memory"};
      o->aca_allocs.push_back(p);
      return p;
    };
    o->aca_rank = static_cast<int32_t*>(dalloc(sizeof(int32_t) * (size_t)nkeys));
    // pass 0: ranks, in chunks of keys with a scratch of n (n + 1) complex per key
    const int64_t chunk = 1024;
    double2* scratch = static_cast<double2*>(dalloc(sizeof(double2) * (size_t)(chunk * n * (n + 1))));
    for (int64_t k0 = 0; k0 < nkeys; k0 += chunk)
      launch_aca_factor(o->st, o->dC, o->dirtab, k0, std::min(chunk, nkeys - k0), o->key_level, o->key_d, o->key_dir,
                        eps, n, 0, o->aca_rank, scratch, nullptr, nullptr, nullptr, nullptr);
    CK(cudaGetLastError());
    std::vector<int32_t> rk(nkeys);
    CK(cudaMemcpyAsync(rk.data(), o->aca_rank, sizeof(int32_t) * nkeys, cudaMemcpyDeviceToHost, o->st));
    CK(cudaStreamSynchronize(o->st));
    cudaFree(scratch);
    o->aca_allocs.pop_back();
    std::vector<int64_t> uo(nkeys, 0), wo(nkeys, 0);
    int64_t ut = 0, wt = 0, rsum = 0, nd = 0;
    for (int64_t k = 0; k < nkeys; ++k) {
      uo[k] = ut;
      wo[k] = wt;
      if (rk[k] < 0) {
        wt += (int64_t)n * n;
        ++nd;
      } else {
        ut += (int64_t)rk[k] * n;
        wt += (int64_t)rk[k] * n;
        rsum += rk[k];
      }
    }
    size_t fre = 0, tot = 0;
    CK(cudaMemGetInfo(&fre, &tot));
    const double need = 16.0 * (double)(ut + wt);
    if (need > 0.8 * (double)fre) throw PlanError{FDH_ERR_MEMORY, "ACA factors do not fit in device memory"};
    o->aca_U = static_cast<double2*>(dalloc(sizeof(double2) * (size_t)ut));
    o->aca_W = static_cast<double2*>(dalloc(sizeof(double2) * (size_t)wt));
    o->aca_uoff = static_cast<int64_t*>(dalloc(sizeof(int64_t) * (size_t)nkeys));
    o->aca_woff = static_cast<int64_t*>(dalloc(sizeof(int64_t) * (size_t)nkeys));
    CK(cudaMemcpy(o->aca_uoff, uo.data(), sizeof(int64_t) * nkeys, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(o->aca_woff, wo.data(), sizeof(int64_t) * nkeys, cudaMemcpyHostToDevice));
    // pass 1: the factors (same pivots) at their offsets; dense keys: W = A
    for (int64_t k0 = 0; k0 < nkeys; k0 += chunk)
      launch_aca_factor(o->st, o->dC, o->dirtab, k0, std::min(chunk, nkeys - k0), o->key_level, o->key_d, o->key_dir,
                        eps, n, 1, o->aca_rank, nullptr, o->aca_uoff, o->aca_woff, o->aca_U, o->aca_W);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(o->st));
    o->aca_bytes = (int64_t)need;
    o->aca_mean_rank = nkeys > nd ? (double)rsum / (double)(nkeys - nd) : 0.0;
    o->stats.aca_dense_keys = nd;
    o->aca_eps = eps;
  });
}

int fdh_set_cache(fdh_op* o, int flags) {
  if (!o) return fail(FDH_ERR_ARG, "NULL op");
  for (fdh_op* p : o->parts) {
    cudaSetDevice(p->device);
    if (const int rc = fdh_set_cache(p, flags)) return rc;
  }
  if (!o->parts.empty()) {
    cudaSetDevice(0);
    return FDH_OK;
  }
  if (!o->st) return fail(FDH_ERR_UNSUPPORTED, "operator was built with fdh_plan_only (no device state)");
  return guard([&] {
    CK(cudaSetDevice(o->device));
    CK(cudaStreamSynchronize(o->st));
    for (void* p : o->nf_allocs) cudaFree(p);
    o->nf_allocs.clear();
    o->nf_K = nullptr;
    o->nf_koff = nullptr;
    o->nf_bytes = 0;
    o->gx = nullptr;  // re-capture the apply graph
    if (o->gexec) {
      CK(cudaGraphExecDestroy(o->gexec));
      o->gexec = nullptr;
    }
    if (!(flags & FDH_CACHE_NEARFIELD)) return;
    const Plan& P = o->P;
    const int64_t ne = (int64_t)P.l2t_begin.size();
    std::vector<int64_t> koff(ne + 1, 0), poff(ne + 1, 0);
    for (int64_t e = 0; e < ne; ++e) {
      int64_t ns = 0;
      for (int64_t r = P.p2p_ptr[e]; r < P.p2p_ptr[e + 1]; ++r) ns += P.p2p_send[r] - P.p2p_sbeg[r];
      koff[e + 1] = koff[e] + ns * (int64_t)(P.l2t_end[e] - P.l2t_begin[e]);
      poff[e + 1] = poff[e] + ns;
    }
    size_t fre = 0, tot = 0;
    CK(cudaMemGetInfo(&fre, &tot));
    const double need = 16.0 * (double)koff[ne] + 4.0 * (double)poff[ne];
    if (need > 0.7 * (double)fre)
      throw PlanError{FDH_ERR_MEMORY, "near-field cache (" + std::to_string((long long)(need / 1e9)) +
                                          " GB) does not fit in device memory"};
    auto dalloc = [&](size_t bytes) {
      void* p = nullptr;
      if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess)
        throw PlanError{FDH_ERR_MEMORY, "near-field cache allocation failed"};
      o->nf_allocs.push_back(p);
      return p;
    };
    o->nf_koff = static_cast<int64_t*>(dalloc(sizeof(int64_t) * (ne + 1)));
    o->nf_poff = static_cast<int64_t*>(dalloc(sizeof(int64_t) * (ne + 1)));
    o->nf_K = static_cast<double2*>(dalloc(16 * (size_t)koff[ne]));
    o->nf_spos = static_cast<uint32_t*>(dalloc(4 * (size_t)poff[ne]));
    CK(cudaMemcpy(o->nf_koff, koff.data(), sizeof(int64_t) * (ne + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(o->nf_poff, poff.data(), sizeof(int64_t) * (ne + 1), cudaMemcpyHostToDevice));
    CK(cudaMemset(o->flag, 0, sizeof(int)));
    launch_p2p_cache_fill(o->st, o->kappa, (int)ne, o->l2t_beg, o->l2t_end, o->p2p_ptr, o->p2p_sbeg, o->p2p_send,
                          o->tx, o->ty, o->tz, o->sx, o->sy, o->sz, o->diag_slot, P.prm.zero_diagonal, o->nf_koff,
                          o->nf_poff, o->nf_K, o->nf_spos, o->flag);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(o->st));
    int f = 0;
    CK(cudaMemcpy(&f, o->flag, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemset(o->flag, 0, sizeof(int)));
    if (f & 1) {
      for (void* p : o->nf_allocs) cudaFree(p);
      o->nf_allocs.clear();
      o->nf_K = nullptr;
      throw PlanError{FDH_ERR_DOMAIN, "Helmholtz kernel is singular at x == y (near field)"};
    }
    o->nf_bytes = (int64_t)need;
  });
}

int fdh_sync(fdh_op* o) {
  if (!o) return fail(FDH_ERR_ARG, "NULL op");
  if (!o->parts.empty())
    return guard([&] {
      int flag = 0;
      group_sync(o, &flag);
      if (flag & 1) throw PlanError{FDH_ERR_DOMAIN, "Helmholtz kernel is singular at x == y (near field)"};
    });
  if (!o->st) return FDH_OK;
  return guard([&] {
    CK(cudaSetDevice(o->device));
    CK(cudaStreamSynchronize(o->st));
    if (o->gst && o->gst != o->st) CK(cudaStreamSynchronize(o->gst));
    int flag = 0;
    CK(cudaMemcpy(&flag, o->flag, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemset(o->flag, 0, sizeof(int)));
    if (flag & 1) throw PlanError{FDH_ERR_DOMAIN, "Helmholtz kernel is singular at x == y (near field)"};
  });
}

void* fdh_stream(fdh_op* o) {
  if (o && !o->parts.empty()) return static_cast<void*>(o->parts[0]->st);
  return o ? static_cast<void*>(o->st) : nullptr;
}

int fdh_set_timing(fdh_op* o, int enable) {
  if (!o) return fail(FDH_ERR_ARG, "NULL op");
  for (fdh_op* p : o->parts) {
    cudaSetDevice(p->device);
    if (const int rc = fdh_set_timing(p, enable)) return rc;
  }
  if (!o->parts.empty()) cudaSetDevice(0);
  return guard([&] {
    if (o->st) {
      CK(cudaStreamSynchronize(o->st));
      collect_times(o);  // flush what the previous mode recorded
    }
    o->timing = enable != 0;
    o->ring_n = o->ring_done = 0;
    o->tacc_n = 0;
    for (double& v : o->tacc) v = 0.0;
    o->apply_ms_sum = 0.0;
    o->applies_collected = 0;
  });
}

int fdh_get_stats(const fdh_op* o, fdh_stats* s) {
  if (!o || !s) return fail(FDH_ERR_ARG, "NULL argument");
  if (!o->parts.empty()) {
    // multi-GPU: structure counters of the (full) partition from device 0's shard,
    // times = max over the devices, bytes / launches summed
    fdh_stats t{};
    for (size_t g = 0; g < o->parts.size(); ++g) {
      cudaSetDevice(o->parts[g]->device);
      if (const int rc = fdh_get_stats(o->parts[g], g == 0 ? s : &t)) return rc;
      if (g == 0) continue;
      s->apply_ms = std::max(s->apply_ms, t.apply_ms);
      s->apply_ms_sum = std::max(s->apply_ms_sum, t.apply_ms_sum);
      for (int ph = 0; ph < FDH_NPHASES; ++ph) s->phase_ms[ph] = std::max(s->phase_ms[ph], t.phase_ms[ph]);
      s->m2l_gemm_ms = std::max(s->m2l_gemm_ms, t.m2l_gemm_ms);
      s->bytes_stored += t.bytes_stored;
      s->gpu_launches += t.gpu_launches;
      s->m2l_i8_ops += t.m2l_i8_ops;
      s->m2l_tiles += t.m2l_tiles;
      s->m2l_items += t.m2l_items;
    }
    cudaSetDevice(0);
    s->setup_ms = o->stats.setup_ms;
    s->shard_cost = s->total_cost;
    return FDH_OK;
  }
  fdh_op* m = const_cast<fdh_op*>(o);
  if (m->st) {
    cudaStreamSynchronize(m->st);
    try {
      collect_times(m);
    } catch (...) {
    }
  }
  const Plan& P = o->P;
  *s = o->stats;
  s->n_le = P.n_le;
  s->n_c = P.n_c;
  s->n_sc = P.n_sc;
  s->m_d = P.m_d;
  s->n_lminus = P.n_lminus;
  s->nf_percent = 100.0 * (double)P.m_d / ((double)o->nt * (double)o->ns);
  s->bytes_stored = o->bytes;
  s->depth_t = P.T.depth;
  s->depth_s = P.S.depth;
  s->l_hf = P.lhf;
  s->n_pad = P.n_pad;
  s->slots_t = P.T.nslots;
  s->slots_s = P.S.nslots;
  int64_t nn = 0;
  for (auto& L : P.T.lv) nn += (int64_t)L.size();
  s->nodes_t = nn;
  nn = 0;
  for (auto& L : P.S.lv) nn += (int64_t)L.size();
  s->nodes_s = nn;
  s->gpu_launches = o->launches;
  s->m2l_tiles = (int64_t)P.tile_level.size();
  s->m2l_items = (int64_t)P.item_tile.size();
  s->m2l_chunk = P.m2l_chunk;
  s->shard_cost = P.shard_cost;
  s->structure_ms = P.structure_ms;
  s->gpu_structure = P.prm.gpu_structure ? 1 : 0;
  s->w_resident = o->w_resident ? 1 : 0;
  s->w_segments = (int64_t)o->segs.size();
  s->nrhs = o->R;
  s->graph_replays = o->graph_replays;
  s->apply_ms_sum = o->apply_ms_sum;
  s->applies_collected = o->applies_collected;
  s->aca_eps = o->aca_eps;
  s->aca_mean_rank = o->aca_mean_rank;
  s->aca_bytes = o->aca_bytes;
  s->nf_cache_bytes = o->nf_bytes;
  s->m2l_pair_mode = P.m2l_pair ? 1 : 0;
  s->m2l_i8_digits = kI8Digits;
  s->m2l_i8_bits = kI8Bits;
  s->m2l_i8_products = i8_products();
  s->total_cost = P.total_cost;
  s->m2l_flops_executed = P.m2l_units_exec * 16 * (int64_t)P.n_pad * (int64_t)P.n_k;  // DMMA issued (M2LSplit units)
  s->m2l_impl = P.prm.m2l_impl;
  if (P.prm.m2l_impl == 1) {
    // int8 MACs issued by k_m2l_i8: per (tile, key) and K byte: 128 rows x sum_i (KS - i) 2 TT columns per m-block
    const int64_t cols = (int64_t)i8_products() * 2 * P.prm.tile;
    const int64_t nkq = (P.n + 15) / 16 * 16;
    s->m2l_flops_executed = 0;
    s->m2l_i8_ops = 2 * (int64_t)P.tile_keys.size() * ((P.n + 127) / 128) * 128 * (2 * nkq) * cols;
  }
  // algorithmic HBM bytes of the transfer passes per rhs: 16 n B per
  // moment / local vector read or written, 40 B per source point (S2M), 24 + 32 B per
  // target point (L2T: point read, y read-modify-write)
  const int64_t v16 = 16 * (int64_t)P.n;
  s->hbm_bytes[0] = 40 * (int64_t)P.S.perm.size() + v16 * (int64_t)P.s2m_slot.size();
  int64_t m2m = 0, l2l = 0, l2t = 0;
  for (size_t l = 0; l < P.m2m_parent.size(); ++l) {
    m2m += (int64_t)P.m2m_parent[l].size();
    for (int32_t c : P.m2m_child[l]) m2m += c >= 0;
  }
  for (size_t l = 0; l < P.l2l_child.size(); ++l) l2l += (int64_t)P.l2l_pslot[l].size() + 2 * (int64_t)P.l2l_child[l].size();
  for (size_t i = 0; i < P.l2t_nslot.size(); ++i) l2t += P.l2t_nslot[i];
  int64_t nt_own = 0;
  for (size_t i = 0; i < P.l2t_begin.size(); ++i) nt_own += (int64_t)P.l2t_end[i] - P.l2t_begin[i];
  s->hbm_bytes[1] = v16 * m2m;
  s->hbm_bytes[2] = v16 * l2l;
  s->hbm_bytes[3] = v16 * l2t + 56 * nt_own;
  return FDH_OK;
}

// introspection of a multi-GPU operator: device 0's shard (full trees, L-, D/D^;
// L+ and owned leaves of that shard)
static const fdh_op* prim(const fdh_op* o) { return (o && !o->parts.empty()) ? o->parts[0] : o; }

int64_t fdh_export_tree(const fdh_op* o, int which, int64_t* rows) {
  o = prim(o);
  return o ? export_tree(which == 0 ? o->P.T : o->P.S, rows) : -1;
}
int64_t fdh_export_perm(const fdh_op* o, int which, int64_t* perm) {
  o = prim(o);
  return o ? export_perm(which == 0 ? o->P.T : o->P.S, perm) : -1;
}
int64_t fdh_export_lplus(const fdh_op* o, int64_t* rows) { return (o = prim(o)) ? export_lplus(o->P, rows) : -1; }
int64_t fdh_export_lminus(const fdh_op* o, int64_t* rows) { return (o = prim(o)) ? export_lminus(o->P, rows) : -1; }
int64_t fdh_export_dirsets(const fdh_op* o, int which, int64_t* rows) {
  o = prim(o);
  return o ? export_dirsets(o->P, which, rows) : -1;
}

int64_t fdh_export_owned_leaves(const fdh_op* o, int64_t* rows) {
  if (o && !o->parts.empty()) {  // every device's leaves
    int64_t n = 0;
    for (const fdh_op* p : o->parts) n += export_owned_leaves(p->P, nullptr);
    if (!rows) return n;
    int64_t off = 0;
    for (const fdh_op* p : o->parts) off += export_owned_leaves(p->P, rows + 6 * off);
    return off;
  }
  return o ? export_owned_leaves(o->P, rows) : -1;
}

int fdh_structure_digest(const fdh_op* o, uint64_t* out6) {
  if (!o || !out6) return fail(FDH_ERR_ARG, "NULL argument");
  structure_digest(prim(o)->P, out6);
  return FDH_OK;
}

}  // extern "C"
