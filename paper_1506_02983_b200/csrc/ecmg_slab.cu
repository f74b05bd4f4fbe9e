// ecmg_slab.cu -- z-slab domain decomposition of the ECMG_jcg hot path.
//
// Levels whose z extent n satisfies n % (4P) == 0 and n / P >= 16 are sharded in z-slabs of node
// planes (slab_partition, host_common.h); smaller levels are replicated (solved identically by
// every rank, no communication). On a sharded level a rank holds:
//  * JCG work vectors x, r, p, p', b over its owned free planes plus one halo plane per side;
//  * full-layout per-level nodal vectors u_k, of which it fills its owned planes and one upper halo
//    plane (EXP_finite of the next level and EXP_true read at most that plane; the partition nests
//    across levels because slab boundaries are multiples of 4 fine planes).
// Per JCG iteration (Alg. 4 l.7-9, textbook PCG): K1 (local sums) -> allreduce(sigma) -> finalize ->
// K2 (local sums) -> allreduce(rho', rr) -> finalize -> halo exchange of r. K1 recomputes p on its
// halo planes from r and p_old there, so p never travels. Every rank sees the same allreduced
// scalars, so all ranks stop at the same iteration and issue the same communication sequence.
//
// Communication backends behind one interface:
//  * NCCL (real ranks, one GPU each): ncclAllReduce of the 3 scalars, grouped ncclSend / ncclRecv
//    of contiguous halo planes over NVLink. libnccl is the one PyTorch already loaded (dlopen).
//  * virtual slabs (all P slabs in one process on one GPU): the halo "messages" are device copies
//    and the allreduce is an in-order sum kernel. This is the test fixture that
//    runs the exact slab arithmetic on one GPU; no kernel ever waits on another.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "host_common.h"
#include "slab.h"

namespace ecmg {

// ---- NCCL through dlopen ----------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOLOAD | RTLD_LAZY);
  if (!h) h = dlopen("libnccl.so.2", RTLD_LAZY);
  if (!h) return api;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
  api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
  api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
  api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Send && api.Recv &&
           api.GroupStart && api.GroupEnd && api.AllGather;
  return api;
}

int nccl_unique_id(unsigned char id[128]) {
  NcclApi& n = nccl();
  if (!n.ok) return ECMG_ENCCL;
  ncclUniqueId u;
  if (n.GetUniqueId(&u) != ncclSuccess) return ECMG_ENCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return ECMG_OK;
}

// ---- one slab's device state ------------------------------------------------------------------
struct SlabCtx {
  int rank = 0;
  std::vector<LevelGeom> geom;
  std::vector<char> sharded;
  double* x = nullptr;
  double* r = nullptr;
  double* z = nullptr;   // element path: z = D^-1 r (K1 reads it on its halo planes)
  double* p[2] = {nullptr, nullptr};
  double* b = nullptr;
  double* beta = nullptr;
  double* b_fin = nullptr;      // the finest level's b / beta / 1D tables (its setup can run ahead)
  double* beta_fin = nullptr;
  double* s1d_fin = nullptr;
  double* partials = nullptr;
  double* scratch1d = nullptr;
  double* seeds = nullptr;
  JcgScalars* sc = nullptr;
  std::vector<double*> u;    // full-layout per level
  double* ut = nullptr;      // full-layout finest u~ scratch
  int maps_level = -1;
  bool maps_ok = false;
  CUtensorMap xh, xi, rh, ri, ph[2], bi;
  // fused halo exchange: base pointers of the lower [0] / upper [1] neighbour's r and z buffers (another
  // slab on this GPU, or a CUDA-IPC mapping of the neighbour rank's buffers), and per level the local
  // plane index of the neighbour's halo plane that receives this slab's boundary plane
  double* peer_r[2] = {nullptr, nullptr};
  double* peer_z[2] = {nullptr, nullptr};
  bool peer_ipc = false;                 // the peer pointers are IPC mappings (closed at destroy)
  std::vector<int> nb_lo_zend, nb_hi_zbeg;
};

struct SlabDriver {
  int P = 1, rank = 0;
  bool virt = false;
  std::vector<SlabCtx> s;    // local slabs: all P (virtual) or this rank's one (NCCL)
  ncclComm_t comm = nullptr;
  JcgScalars* sc_host = nullptr;
  JcgParams* param_host = nullptr;   // u_out stays null: slabs scatter separately
  cudaEvent_t ev[4];
  SlabCfg cfg{};
  int L = 0;
  double last_jcg_ms = 0.0;
  int last_jcg_iters = 0;
  long long last_free = 0;
  // the finest level's setup run ahead (hybrid cascade): its event, and whether it is pending
  cudaStream_t ahead_stream = nullptr;
  cudaEvent_t ahead_ev = nullptr, fork_ev = nullptr;
  bool fin_ahead = false;
  // device-driven loop of the sharded levels: one instantiated graph per level (built on first use, dropped
  // when the configuration changes); graph_failed: capture / instantiation failed once (e.g. a communication
  // backend that cannot be captured), the host loop is used from then on
  std::vector<cudaGraphExec_t> graphs;
  cudaStream_t cap_stream = nullptr;
  bool graph_failed = false;
  std::vector<std::pair<int, int>> graph_launches;   // per level: kernels of prologue + epilogue, of one body
  int cap_count[3] = {0, 0, 0};
};

namespace {

#define SL_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) {                            \
      if (std::getenv("ECMG_DEBUG"))                    \
        std::fprintf(stderr, "libecmg(slab): %s: %s\n", #call, cudaGetErrorString(e_)); \
      return e_ == cudaErrorMemoryAllocation ? ECMG_ENOMEM : ECMG_ECUDA; \
    }                                                   \
  } while (0)
#define SL_NCCL(call)                                   \
  do {                                                  \
    if ((call) != ncclSuccess) return ECMG_ENCCL;       \
  } while (0)

// the problem as level k's kernels see it (ECMG_PROB_ARRAYS: with that level's caller arrays)
Problem level_problem(const SlabCfg& cf, int k) {
  Problem p = cf.prob;
  if (p.id == PROB_ARRAYS && (int)cf.arrays.size() == 5 * cf.L)
    for (int j = 0; j < 5; ++j) p.arr[j] = cf.arrays[5 * k + j];
  return p;
}

// ---- communication ---------------------------------------------------------------------------
int comm_allreduce(SlabDriver* d, cudaStream_t st) {
  if (d->virt) {
    SlabScalars ss{};
    ss.n = (int)d->s.size();
    for (int i = 0; i < ss.n; ++i) ss.p[i] = d->s[i].sc;
    SL_CUDA(launch_vsum(ss, st));
    return ECMG_OK;
  }
  NcclApi& n = nccl();
  SlabCtx& c = d->s[0];
  SL_NCCL(n.AllReduce(c.sc->loc, c.sc->glob, 3, ncclDouble, ncclSum, d->comm, st));
  return ECMG_OK;
}

// halo planes of a work vector (which: 0 = x, 1 = r, 2 = z) on sharded level k
int comm_halo(SlabDriver* d, int k, int which, cudaStream_t st) {
  auto vec = [&](SlabCtx& c) { return which == 0 ? c.x : (which == 1 ? c.r : c.z); };
  if (d->virt) {
    for (size_t i = 0; i + 1 < d->s.size(); ++i) {
      SlabCtx& lo = d->s[i];
      SlabCtx& hi = d->s[i + 1];
      const LevelGeom& gl = lo.geom[k];
      const LevelGeom& gh = hi.geom[k];
      const size_t bytes = sizeof(double) * gl.S;
      SL_CUDA(cudaMemcpyAsync(vec(hi) + (long long)(gh.zbeg - 1) * gh.S, vec(lo) + (long long)(gl.zend - 1) * gl.S, bytes,
                              cudaMemcpyDeviceToDevice, st));
      SL_CUDA(cudaMemcpyAsync(vec(lo) + (long long)gl.zend * gl.S, vec(hi) + (long long)gh.zbeg * gh.S, bytes,
                              cudaMemcpyDeviceToDevice, st));
    }
    return ECMG_OK;
  }
  NcclApi& n = nccl();
  SlabCtx& c = d->s[0];
  const LevelGeom& g = c.geom[k];
  double* v = vec(c);
  const size_t cnt = (size_t)g.S;
  SL_NCCL(n.GroupStart());
  if (d->rank > 0) {
    SL_NCCL(n.Send(v + (long long)g.zbeg * g.S, cnt, ncclDouble, d->rank - 1, d->comm, st));
    SL_NCCL(n.Recv(v + (long long)(g.zbeg - 1) * g.S, cnt, ncclDouble, d->rank - 1, d->comm, st));
  }
  if (d->rank < d->P - 1) {
    SL_NCCL(n.Send(v + (long long)(g.zend - 1) * g.S, cnt, ncclDouble, d->rank + 1, d->comm, st));
    SL_NCCL(n.Recv(v + (long long)g.zend * g.S, cnt, ncclDouble, d->rank + 1, d->comm, st));
  }
  SL_NCCL(n.GroupEnd());
  return ECMG_OK;
}

// upper halo plane of the full-layout u_k: rank r's first owned plane goes to rank r-1
int comm_u_halo(SlabDriver* d, int k, cudaStream_t st) {
  if (d->virt) {
    for (size_t i = 0; i + 1 < d->s.size(); ++i) {
      const LevelGeom& gh = d->s[i + 1].geom[k];
      const long long pl = (long long)(gh.n[0] + 1) * (gh.n[1] + 1);
      SL_CUDA(cudaMemcpyAsync(d->s[i].u[k] + gh.zlo * pl, d->s[i + 1].u[k] + gh.zlo * pl, sizeof(double) * pl,
                              cudaMemcpyDeviceToDevice, st));
    }
    return ECMG_OK;
  }
  NcclApi& n = nccl();
  SlabCtx& c = d->s[0];
  const LevelGeom& g = c.geom[k];
  const long long pl = (long long)(g.n[0] + 1) * (g.n[1] + 1);
  SL_NCCL(n.GroupStart());
  if (d->rank > 0) SL_NCCL(n.Send(c.u[k] + g.zlo * pl, (size_t)pl, ncclDouble, d->rank - 1, d->comm, st));
  if (d->rank < d->P - 1) SL_NCCL(n.Recv(c.u[k] + g.zhi * pl, (size_t)pl, ncclDouble, d->rank + 1, d->comm, st));
  SL_NCCL(n.GroupEnd());
  return ECMG_OK;
}

// ---- per-slab kernels ------------------------------------------------------------------------
// right-hand side / element beta / 1D tables of level k: the finest level has its own (its setup can
// run ahead while the replicated levels are solved); the other sharded levels share one set
inline double* bvec(const SlabDriver* d, SlabCtx& c, int k) { return k == d->L - 1 ? c.b_fin : c.b; }
inline double* betavec(const SlabDriver* d, SlabCtx& c, int k) { return k == d->L - 1 ? c.beta_fin : c.beta; }
inline double* s1dvec(const SlabDriver* d, SlabCtx& c, int k) { return k == d->L - 1 ? c.s1d_fin : c.scratch1d; }

bool slab_maps(SlabDriver* d, SlabCtx& c, int k) {
  if (c.maps_level == k) return c.maps_ok;
  const LevelGeom& g = c.geom[k];
  const int hx = tma_halo_box_x(), hy = tma_halo_box_y(), ix = tma_int_box_x(), iy = tma_int_box_y();
  c.maps_ok = make_vec_tensor_map(&c.xh, c.x, g, hx, hy) == 0 && make_vec_tensor_map(&c.xi, c.x, g, ix, iy) == 0 &&
              make_vec_tensor_map(&c.rh, c.r, g, hx, hy) == 0 && make_vec_tensor_map(&c.ri, c.r, g, ix, iy) == 0 &&
              make_vec_tensor_map(&c.ph[0], c.p[0], g, hx, hy) == 0 &&
              make_vec_tensor_map(&c.ph[1], c.p[1], g, hx, hy) == 0 && make_vec_tensor_map(&c.bi, bvec(d, c, k), g, ix, iy) == 0;
  c.maps_level = k;
  return c.maps_ok;
}

cudaError_t slab_launch(SlabDriver* d, SlabCtx& c, int mode, int k, const KArgs& a, cudaStream_t st) {
  const SlabCfg& cf = d->cfg;
  const LevelGeom& g = c.geom[k];
  if (cf.elem_path) {
    const Problem pk = level_problem(cf, k);
    ElemStencil es = make_elem_stencil(g, pk, cf.precond);
    if (cf.beta_fly && a.beta) set_beta_fly(es, g, pk, a.beta);
    return launch_jcg_elem(mode, g, es, pk, a, st);
  }
  const ConstStencil cs = make_const_stencil(g, 1.0, cf.precond);
  if (cf.kernel_variant == 1 && slab_maps(d, c, k)) {
    auto halo = [&](const double* p) -> const CUtensorMap* {
      if (p == c.x) return &c.xh;
      if (p == c.r) return &c.rh;
      if (p == c.p[0]) return &c.ph[0];
      if (p == c.p[1]) return &c.ph[1];
      return nullptr;
    };
    auto inter = [&](const double* p) -> const CUtensorMap* {
      if (p == c.x) return &c.xi;
      if (p == c.r) return &c.ri;
      if (p == bvec(d, c, k)) return &c.bi;
      return nullptr;
    };
    const CUtensorMap* h0 = halo(a.h0);
    const CUtensorMap* h1 = a.h1 ? halo(a.h1) : h0;
    const CUtensorMap* i0 = a.i0 ? inter(a.i0) : h0;
    const CUtensorMap* i1 = a.i1 ? inter(a.i1) : h0;
    if (h0 && h1 && i0 && i1) {
      CUtensorMap m[4] = {*h0, *h1, *i0, *i1};
      return launch_jcg_const_tma(mode, g, cs, a, m, st);
    }
  }
  return launch_jcg_const(mode, g, cs, a, st);
}

KArgs base_args(SlabDriver* d, SlabCtx& c, int k, bool local_only) {
  KArgs a{};
  a.partials = c.partials;
  a.sc = c.sc;
  a.zc = auto_zc(d->cfg.zchunk, d->cfg.elem_path, c.geom[k]);
  a.beta = betavec(d, c, k);
  a.local_only = local_only ? 1 : 0;
  return a;
}

int setup_slab_level(SlabDriver* d, SlabCtx& c, int k, cudaStream_t st) {
  const SlabCfg& cf = d->cfg;
  const LevelGeom& g = c.geom[k];
  const Problem pk = level_problem(cf, k);
  const ElemStencil es = make_elem_stencil(g, pk, cf.precond);
  if (cf.elem_path) SL_CUDA(launch_beta(g, pk, betavec(d, c, k), st));
  SL_CUDA(launch_rhs(g, pk, es, 1.0, cf.elem_path ? betavec(d, c, k) : nullptr, bvec(d, c, k), s1dvec(d, c, k), st));
  return ECMG_OK;
}

int read_stats(SlabDriver* d, int k, double eps, ecmg_stats* st, cudaStream_t stream) {
  SL_CUDA(cudaMemcpyAsync(d->sc_host, d->s[0].sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, stream));
  SL_CUDA(cudaStreamSynchronize(stream));
  const JcgScalars s = *d->sc_host;
  d->last_jcg_iters = s.iter;
  long long nfree = 0;
  for (auto& c : d->s) nfree += free_count(c.geom[k]);
  d->last_free = nfree;
  const double nb = std::sqrt(s.bb), nbe = nb > 0.0 ? nb : 1.0;
  int status = s.status;
  const bool conv = (eps <= 0.0) || !(std::sqrt(s.rr) > eps * nbe);
  if (status == ECMG_OK && !conv) status = ECMG_ENOTCONV;
  if (st) {
    st->iterations = s.iter;
    st->rel_res_recur = std::sqrt(s.rr) / nbe;
    st->rel_res_true = std::sqrt(s.rr_true) / nbe;
    st->norm_b = nb;
    st->converged = conv && status == ECMG_OK;
    st->status = status;
  }
  return status;
}

// JCG on a level. Sharded: all local slabs, allreduce + halo exchange per pass. Replicated: slab 0
// (virtual) or this rank (NCCL) solves the whole level with no communication.
int slab_jcg(SlabDriver* d, int k, double eps, int max_iter, ecmg_stats* st, cudaStream_t stream) {
  if (max_iter <= 0 && eps > 0) max_iter = 10000;
  if (max_iter < 0) max_iter = 0;
  const bool sh = d->s[0].sharded[k];
  const int nloc = (sh || !d->virt) ? (int)d->s.size() : 1;
  d->param_host->eps = eps;
  d->param_host->max_iter = max_iter;
  d->param_host->u_out = nullptr;
  d->param_host->ut_out = nullptr;
  d->param_host->u2h = nullptr;
  for (int i = 0; i < nloc; ++i)
    SL_CUDA(cudaMemcpyAsync(&d->s[i].sc->in, d->param_host, sizeof(JcgParams), cudaMemcpyHostToDevice, stream));
  const cudaStream_t user_stream = stream;   // the work below goes to `stream`; graph capture points it elsewhere
  KArgs cond{};                              // the WHILE node's handle for the finalize kernels (graph build only)
  // one pass of `mode` over all local slabs (+ allreduce and finalize when sharded)
  auto pass = [&](int mode, auto fill) -> int {
    for (int i = 0; i < nloc; ++i) {
      KArgs a = base_args(d, d->s[i], k, sh);
      fill(d->s[i], a);
      SL_CUDA(slab_launch(d, d->s[i], mode, k, a, stream));
    }
    if (sh) {
      int r = comm_allreduce(d, stream);
      if (r) return r;
      for (int i = 0; i < nloc; ++i) {
        KArgs af = base_args(d, d->s[i], k, sh);
        af.use_cond = cond.use_cond; af.cond = cond.cond;
        SL_CUDA(launch_finalize(mode, af, stream));
      }
    }
    return ECMG_OK;
  };
  int rc;
  auto zero_boundary_halos = [&]() -> int {
    // halo planes at the global z boundary stand for Dirichlet / outside nodes: they must read as 0
    // (the buffers were used by earlier levels with other geometries)
    for (int i = 0; i < nloc; ++i) {
      SlabCtx& c = d->s[i];
      const LevelGeom& g = c.geom[k];
      const size_t plane = sizeof(double) * g.S;
      double* vecs[5] = {c.x, c.r, c.z, c.p[0], c.p[1]};
      for (double* v : vecs) {
        if (c.rank == 0) SL_CUDA(cudaMemsetAsync(v, 0, plane, stream));
        if (c.rank == d->P - 1) SL_CUDA(cudaMemsetAsync(v + (long long)g.zend * g.S, 0, plane, stream));
      }
    }
    return ECMG_OK;
  };
  // K1 reads r (constant stencil) or z = D^-1 r (element path) on its halo planes. Fused halo: the init
  // and K2 passes store their boundary planes of that vector straight into the neighbours' halo planes
  // (peer memory); the allreduce that follows every pass orders those stores before the next K1.
  const bool elem = d->cfg.elem_path != 0;
  const int k1_vec = elem ? 2 : 1;
  bool fused = sh && d->cfg.fused_halo != 0;
  for (int i = 0; i < nloc && fused; ++i) {
    const SlabCtx& c = d->s[i];
    if ((c.rank > 0 && !c.peer_r[0]) || (c.rank + 1 < d->P && !c.peer_r[1])) fused = false;
  }
  auto set_peers = [&](SlabCtx& c, KArgs& a) {
    if (!fused) return;
    const LevelGeom& g = c.geom[k];
    double* const* base = elem ? c.peer_z : c.peer_r;
    a.peer_lo = c.rank > 0 ? base[0] + (long long)c.nb_lo_zend[k] * g.S : nullptr;
    a.peer_hi = c.rank + 1 < d->P ? base[1] + (long long)(c.nb_hi_zbeg[k] - 1) * g.S : nullptr;
  };
  auto prologue = [&]() -> int {   // boundary halos, x halo, init pass (r = b - A x, rho, rr, ||b||)
    int q;
    if (sh && (q = zero_boundary_halos())) return q;
    if (sh && (q = comm_halo(d, k, 0, stream))) return q;
    if ((q = pass(MODE_INIT, [&](SlabCtx& c, KArgs& a) {
           a.h0 = c.x; a.i0 = bvec(d, c, k); a.o0 = c.r; a.o1 = c.z;
           set_peers(c, a);
         })))
      return q;
    if (sh && !fused && (q = comm_halo(d, k, k1_vec, stream))) return q;   // halo planes for the first K1
    return ECMG_OK;
  };
  long long it = 0;
  auto iteration = [&]() -> int {
    int q = pass(MODE_K1, [&](SlabCtx& c, KArgs& a) { a.h0 = elem ? c.z : c.r; a.h1 = c.p[it & 1]; a.o0 = c.p[(it + 1) & 1]; });
    if (q) return q;
    q = pass(MODE_K2, [&](SlabCtx& c, KArgs& a) {
      a.h0 = c.p[(it + 1) & 1]; a.i0 = c.x; a.i1 = elem ? c.z : c.r; a.o0 = c.x; a.o1 = c.r; a.o2 = c.z;
      set_peers(c, a);
    });
    if (q) return q;
    if (sh && !fused && (q = comm_halo(d, k, k1_vec, stream))) return q;
    ++it;
    return ECMG_OK;
  };
  auto epilogue = [&]() -> int {   // x halo, true residual ||b - A x||
    int q;
    if (sh && (q = comm_halo(d, k, 0, stream))) return q;
    return pass(MODE_TRUE, [&](SlabCtx& c, KArgs& a) { a.h0 = c.x; a.i0 = bvec(d, c, k); });
  };
  // Device-driven solve of a sharded level (Alg. 4 l.7-9 without host round trips): one CUDA graph =
  // prologue -> WHILE(cond){2 iterations: K1, allreduce, finalize, K2, allreduce, finalize (sets cond =
  // !done), halo} -> epilogue, captured once per level. Every rank's finalize sees the same allreduced
  // scalars, so all ranks run the same number of bodies (matching communication sequences); a
  // speculative second iteration after convergence is a no-op (the kernels and finalize check done).
  auto build_graph = [&](cudaGraphExec_t* out) -> int {
    if (!d->cap_stream) SL_CUDA(cudaStreamCreateWithFlags(&d->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    SL_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    cudaGraphNode_t cond_node = nullptr;
    std::vector<cudaGraphNode_t> leaves;
    int q = ECMG_OK;
    auto fail = [&](int code) { cudaStreamEndCapture(d->cap_stream, &graph); cudaGetLastError(); cudaGraphDestroy(graph); stream = user_stream; cond.use_cond = 0; return code; };
    if (cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault) != cudaSuccess) return fail(ECMG_ECUDA);
    cond.use_cond = 1; cond.cond = h;
    stream = d->cap_stream;
    if (cudaStreamBeginCaptureToGraph(stream, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return fail(ECMG_ECUDA);
    long long lc = ecmg_kernel_launches();
    if ((q = prologue())) return fail(q);
    if (cudaStreamEndCapture(stream, &graph) != cudaSuccess) return fail(ECMG_ECUDA);
    d->cap_count[0] = (int)(ecmg_kernel_launches() - lc);
    {   // the prologue's sinks (nodes without successors): the WHILE node follows them
      size_t nn = 0, ne = 0;
      if (cudaGraphGetNodes(graph, nullptr, &nn) != cudaSuccess || cudaGraphGetEdges(graph, nullptr, nullptr, &ne) != cudaSuccess)
        return fail(ECMG_ECUDA);
      std::vector<cudaGraphNode_t> nodes(nn), from(ne), to(ne);
      if (cudaGraphGetNodes(graph, nodes.data(), &nn) != cudaSuccess ||
          (ne && cudaGraphGetEdges(graph, from.data(), to.data(), &ne) != cudaSuccess))
        return fail(ECMG_ECUDA);
      for (cudaGraphNode_t nd : nodes)
        if (std::find(from.begin(), from.end(), nd) == from.end()) leaves.push_back(nd);
      if (leaves.empty()) return fail(ECMG_ECUDA);
    }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if (cudaGraphAddNode(&cond_node, graph, leaves.data(), leaves.size(), &cp) != cudaSuccess) return fail(ECMG_ECUDA);
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if (cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return fail(ECMG_ECUDA);
    it = 0;
    lc = ecmg_kernel_launches();
    if ((q = iteration()) || (q = iteration())) return fail(q);   // p ping-pong: two iterations per body
    if (cudaStreamEndCapture(stream, &body) != cudaSuccess) return fail(ECMG_ECUDA);
    d->cap_count[1] = (int)(ecmg_kernel_launches() - lc);
    cond.use_cond = 0;
    if (cudaStreamBeginCaptureToGraph(stream, graph, &cond_node, nullptr, 1, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return fail(ECMG_ECUDA);
    lc = ecmg_kernel_launches();
    if ((q = epilogue())) return fail(q);
    if (cudaStreamEndCapture(stream, &graph) != cudaSuccess) return fail(ECMG_ECUDA);
    d->cap_count[2] = (int)(ecmg_kernel_launches() - lc);
    stream = user_stream;
    const cudaError_t e = cudaGraphInstantiate(out, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) { cudaGetLastError(); *out = nullptr; return ECMG_ECUDA; }
    return ECMG_OK;
  };
  if (sh && eps > 0.0 && d->cfg.use_graph && !d->graph_failed) {
    if ((int)d->graphs.size() != d->L) d->graphs.assign(d->L, nullptr);
    if ((int)d->graph_launches.size() != d->L) d->graph_launches.assign(d->L, {0, 0});
    if (!d->graphs[k]) {
      // kernels are counted when they run, not when they are captured: the per-part counts are kept
      const long long l0 = ecmg_kernel_launches();
      const int q = build_graph(&d->graphs[k]);
      d->graph_launches[k] = {d->cap_count[0] + d->cap_count[2], d->cap_count[1]};
      count_launch((int)(l0 - ecmg_kernel_launches()));
      if (q != ECMG_OK) {
        d->graph_failed = true;   // host loop below
        if (std::getenv("ECMG_DEBUG")) std::fprintf(stderr, "libecmg(slab): graph capture failed at level %d; host loop\n", k);
      }
    }
    if (d->graphs[k]) {
      SL_CUDA(cudaEventRecord(d->ev[0], stream));
      SL_CUDA(cudaGraphLaunch(d->graphs[k], stream));
      SL_CUDA(cudaEventRecord(d->ev[1], stream));
      const int status = read_stats(d, k, eps, st, stream);
      count_launch(d->graph_launches[k].first + d->graph_launches[k].second * ((d->last_jcg_iters + 1) / 2));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, d->ev[0], d->ev[1]);
      d->last_jcg_ms = ms;   // prologue + loop + true residual (the host loop times the loop only)
      return status;
    }
  }
  if ((rc = prologue())) return rc;
  it = 0;
  SL_CUDA(cudaEventRecord(d->ev[0], stream));
  if (eps <= 0.0) {
    for (int i = 0; i < max_iter; ++i)
      if ((rc = iteration())) return rc;
  } else {
    // pipelined host loop: batch i+1 in flight while the host inspects batch i's scalars; every rank
    // sees the same scalars, so all ranks launch the same batches (matching NCCL sequences)
    int batch = 1;
    for (int i = 0; i < batch; ++i)
      if ((rc = iteration())) return rc;
    SL_CUDA(cudaMemcpyAsync(&d->sc_host[1], d->s[0].sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, stream));
    SL_CUDA(cudaEventRecord(d->ev[2], stream));
    int slot = 0;
    long long guard = 0;
    while (true) {
      batch = std::min(batch * 2, 8);
      for (int i = 0; i < batch; ++i)
        if ((rc = iteration())) return rc;
      SL_CUDA(cudaMemcpyAsync(&d->sc_host[2 - slot], d->s[0].sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, stream));
      SL_CUDA(cudaEventRecord(d->ev[3 - slot], stream));
      SL_CUDA(cudaEventSynchronize(d->ev[2 + slot]));
      if (d->sc_host[1 + slot].done) break;
      slot = 1 - slot;
      if (++guard > (long long)max_iter + 8) break;
    }
  }
  SL_CUDA(cudaEventRecord(d->ev[1], stream));
  if ((rc = epilogue())) return rc;
  const int status = read_stats(d, k, eps, st, stream);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, d->ev[0], d->ev[1]);
  d->last_jcg_ms = ms;
  return status;
}

}  // namespace

// CUDA-IPC mappings of the neighbour ranks' r and z buffers (NVLink peer memory): every rank exports
// the two handles, an ncclAllGather distributes them, ranks r-1 and r+1 open theirs. Any failure
// (no P2P path, IPC unsupported) leaves the pointers null and the NCCL halo path in use; the outcome
// is agreed on by all ranks (an allreduce of the success flags), so every rank takes the same path.
void exchange_ipc(SlabDriver* d) {
  NcclApi& n = nccl();
  SlabCtx& c = d->s[0];
  const int P = d->P, me = d->rank;
  constexpr size_t H = sizeof(cudaIpcMemHandle_t);
  std::vector<unsigned char> mine(2 * H, 0), all((size_t)P * 2 * H, 0);
  int ok = 1;
  cudaIpcMemHandle_t hr, hz;
  if (cudaIpcGetMemHandle(&hr, c.r) != cudaSuccess || cudaIpcGetMemHandle(&hz, c.z) != cudaSuccess) ok = 0;
  std::memcpy(mine.data(), &hr, H);
  std::memcpy(mine.data() + H, &hz, H);
  unsigned char* dbuf = nullptr;
  double* flag = nullptr;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&dbuf, (size_t)(P + 1) * 2 * H) != cudaSuccess || cudaMalloc(&flag, sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    ok = 0;
  }
  bool gathered = false;
  if (dbuf && flag && st) {
    cudaMemcpy(dbuf + (size_t)P * 2 * H, mine.data(), 2 * H, cudaMemcpyHostToDevice);
    gathered = n.AllGather(dbuf + (size_t)P * 2 * H, dbuf, 2 * H, ncclUint8, d->comm, st) == ncclSuccess &&
               cudaStreamSynchronize(st) == cudaSuccess &&
               cudaMemcpy(all.data(), dbuf, (size_t)P * 2 * H, cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  if (!gathered) ok = 0;
  for (int s = 0; s < 2 && ok; ++s) {
    const int nb = me + (s ? 1 : -1);
    if (nb < 0 || nb >= P) continue;
    cudaIpcMemHandle_t h[2];
    std::memcpy(&h[0], all.data() + (size_t)nb * 2 * H, H);
    std::memcpy(&h[1], all.data() + (size_t)nb * 2 * H + H, H);
    void* pr = nullptr;
    void* pz = nullptr;
    if (cudaIpcOpenMemHandle(&pr, h[0], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&pz, h[1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    c.peer_r[s] = static_cast<double*>(pr);
    c.peer_z[s] = static_cast<double*>(pz);
    c.peer_ipc = true;
  }
  // every rank must agree: min over ranks of ok (sum of failures == 0)
  double fail_local = ok ? 0.0 : 1.0, fail_sum = 1.0;
  if (flag && st) {
    cudaMemcpy(flag, &fail_local, sizeof(double), cudaMemcpyHostToDevice);
    if (n.AllReduce(flag, flag, 1, ncclDouble, ncclSum, d->comm, st) == ncclSuccess && cudaStreamSynchronize(st) == cudaSuccess)
      cudaMemcpy(&fail_sum, flag, sizeof(double), cudaMemcpyDeviceToHost);
  }
  if (fail_sum != 0.0) {   // someone failed: nobody uses peer stores
    for (int s = 0; s < 2; ++s) {
      if (c.peer_ipc && c.peer_r[s]) cudaIpcCloseMemHandle(c.peer_r[s]);
      if (c.peer_ipc && c.peer_z[s]) cudaIpcCloseMemHandle(c.peer_z[s]);
      c.peer_r[s] = c.peer_z[s] = nullptr;
    }
    c.peer_ipc = false;
  }
  if (dbuf) cudaFree(dbuf);
  if (flag) cudaFree(flag);
  if (st) cudaStreamDestroy(st);
  cudaGetLastError();
}

// ---- driver lifecycle ------------------------------------------------------------------------
SlabDriver* slab_driver_create(const SlabCfg& cfg, int P, int rank, bool virt, const unsigned char* nccl_id, int* status) {
  *status = ECMG_OK;
  SlabDriver* d = new SlabDriver;
  d->P = P;
  d->rank = rank;
  d->virt = virt;
  d->L = cfg.L;
  d->cfg = cfg;
  const int nloc = virt ? P : 1;
  d->s.resize(nloc);
  auto fail = [&](int st) { *status = st; slab_driver_destroy(d); return (SlabDriver*)nullptr; };
  if (!virt) {
    NcclApi& n = nccl();
    if (!n.ok) return fail(ECMG_ENCCL);
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, 128);
    if (n.CommInitRank(&d->comm, P, id, rank) != ncclSuccess) return fail(ECMG_ENCCL);
  }
  // worst-case sizes (all faces non-Dirichlet) over the levels, per slab
  int face_none[6] = {FACE_ROBIN, FACE_ROBIN, FACE_ROBIN, FACE_ROBIN, FACE_ROBIN, FACE_ROBIN};
  for (int i = 0; i < nloc; ++i) {
    SlabCtx& c = d->s[i];
    c.rank = virt ? i : rank;
    long long vec = 64;
    for (int k = 0; k < cfg.L; ++k) {
      bool sh;
      LevelGeom g = slab_geom(make_geom(cfg.dom, cfg.n0, k, face_none, 1), P, c.rank, &sh, cfg.shard_min);
      vec = std::max(vec, g.S * (long long)g.nza + 64);
    }
    const LevelGeom gf = make_geom(cfg.dom, cfg.n0, cfg.L - 1, face_none, 1);
    const long long beta_n = beta_doubles(gf);
    const long long part_n = 3LL * ((gf.nf[0] + 7) / 8) * ((gf.nf[1] + 7) / 8) * (gf.nf[2] + 3) / 4 * 4 + 3 * 65536;
    auto alloc = [&](double** p, long long n) -> bool {
      if (dmalloc(p, sizeof(double) * n) != cudaSuccess) { cudaGetLastError(); return false; }
      return cudaMemset(*p, 0, sizeof(double) * n) == cudaSuccess;
    };
    bool ok = alloc(&c.x, vec) && alloc(&c.r, vec) && alloc(&c.z, vec) && alloc(&c.p[0], vec) && alloc(&c.p[1], vec) && alloc(&c.b, vec) &&
              alloc(&c.beta, beta_n) && alloc(&c.partials, part_n) && alloc(&c.b_fin, vec) && alloc(&c.beta_fin, beta_n) &&
              alloc(&c.s1d_fin, 15LL * (std::max(gf.n[0], std::max(gf.n[1], gf.n[2])) + 1)) &&
              alloc(&c.scratch1d, 15LL * (std::max(gf.n[0], std::max(gf.n[1], gf.n[2])) + 1)) &&
              alloc(&c.seeds, (long long)(gf.n[0] / 2 + 1) * (gf.n[1] / 2 + 1) * (gf.n[2] / 2 + 1)) &&
              alloc(&c.ut, level_nodes(gf));
    if (ok) {
      if (dmalloc(&c.sc, sizeof(JcgScalars)) != cudaSuccess || cudaMemset(c.sc, 0, sizeof(JcgScalars)) != cudaSuccess) ok = false;
    }
    c.u.assign(cfg.L, nullptr);
    for (int k = 0; ok && k < cfg.L; ++k) ok = alloc(&c.u[k], level_nodes(make_geom(cfg.dom, cfg.n0, k, face_none, 1)));
    if (!ok) return fail(ECMG_ENOMEM);
  }
  if (cudaHostAlloc(&d->sc_host, 3 * sizeof(JcgScalars), cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(&d->param_host, sizeof(*d->param_host), cudaHostAllocDefault) != cudaSuccess)
    return fail(ECMG_ENOMEM);
  for (int i = 0; i < 4; ++i) cudaEventCreate(&d->ev[i]);
  if (virt) {
    for (int i = 0; i < nloc; ++i) {   // neighbours are slabs of this process
      SlabCtx& c = d->s[i];
      if (i > 0) { c.peer_r[0] = d->s[i - 1].r; c.peer_z[0] = d->s[i - 1].z; }
      if (i + 1 < nloc) { c.peer_r[1] = d->s[i + 1].r; c.peer_z[1] = d->s[i + 1].z; }
    }
  } else {
    exchange_ipc(d);   // best effort: without peer mappings the halo goes through ncclSend / ncclRecv
  }
  slab_driver_configure(d, cfg);
  return d;
}

void slab_driver_configure(SlabDriver* d, const SlabCfg& cfg) {
  for (cudaGraphExec_t& gx : d->graphs)   // captured for the previous configuration
    if (gx) { cudaGraphExecDestroy(gx); gx = nullptr; }
  d->cfg = cfg;
  d->fin_ahead = false;   // a pending ahead setup belongs to the previous configuration
  for (auto& c : d->s) {
    c.geom.clear();
    c.sharded.clear();
    c.nb_lo_zend.assign(cfg.L, 0);
    c.nb_hi_zbeg.assign(cfg.L, 0);
    for (int k = 0; k < cfg.L; ++k) {
      bool sh;
      const LevelGeom gk = make_geom(cfg.dom, cfg.n0, k, cfg.prob.face, cfg.elem_path);
      c.geom.push_back(slab_geom(gk, d->P, c.rank, &sh, cfg.shard_min));
      c.sharded.push_back(sh ? 1 : 0);
      bool s2;   // the neighbours' level geometries follow from the same partition
      if (c.rank > 0) c.nb_lo_zend[k] = slab_geom(gk, d->P, c.rank - 1, &s2, cfg.shard_min).zend;
      if (c.rank + 1 < d->P) c.nb_hi_zbeg[k] = slab_geom(gk, d->P, c.rank + 1, &s2, cfg.shard_min).zbeg;
    }
    c.maps_level = -1;
  }
}

void slab_driver_destroy(SlabDriver* d) {
  if (!d) return;
  cudaDeviceSynchronize();
  for (auto& c : d->s) {
    if (c.peer_ipc)
      for (int s = 0; s < 2; ++s) {
        if (c.peer_r[s]) cudaIpcCloseMemHandle(c.peer_r[s]);
        if (c.peer_z[s]) cudaIpcCloseMemHandle(c.peer_z[s]);
      }
    dfree(c.x); dfree(c.r); dfree(c.z); dfree(c.p[0]); dfree(c.p[1]); dfree(c.b); dfree(c.beta);
    dfree(c.b_fin); dfree(c.beta_fin); dfree(c.s1d_fin);
    dfree(c.partials); dfree(c.scratch1d); dfree(c.seeds); dfree(c.sc); dfree(c.ut);
    for (double* p : c.u) dfree(p);
  }
  if (d->comm) nccl().CommDestroy(d->comm);
  if (d->sc_host) cudaFreeHost(d->sc_host);
  if (d->param_host) cudaFreeHost(d->param_host);
  cudaGetLastError();
  if (d->ahead_stream) cudaStreamDestroy(d->ahead_stream);
  for (cudaGraphExec_t gx : d->graphs)
    if (gx) cudaGraphExecDestroy(gx);
  if (d->cap_stream) cudaStreamDestroy(d->cap_stream);
  if (d->ahead_ev) cudaEventDestroy(d->ahead_ev);
  if (d->fork_ev) cudaEventDestroy(d->fork_ev);
  delete d;
}

void slab_level_range(const SlabDriver* d, int k, int* zlo, int* zhi) {
  const LevelGeom& g = d->s[0].geom[k];
  if (d->virt) { *zlo = 0; *zhi = g.n[2] + 1; return; }
  *zlo = g.zlo;
  *zhi = g.zhi;
}

void slab_last_timing(const SlabDriver* d, double* ms, int* it, long long* nfree) {
  *ms = d->last_jcg_ms;
  *it = d->last_jcg_iters;
  *nfree = d->last_free;
}

// ---- Alg. 4 over slabs -------------------------------------------------------------------------
// u_out / ut_out: virtual slabs -> full-layout finest vectors (device or host); NCCL ranks -> this
// rank's owned planes [zlo, zhi) of the finest level.
// the finest level's setup (every local slab) on the driver's low-priority stream, forked from `stream`;
// slab_run's finest level waits for it instead of setting up in line
int slab_setup_ahead(SlabDriver* d, cudaStream_t stream) {
  const int k = d->L - 1;
  if (!d->ahead_stream) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    SL_CUDA(cudaStreamCreateWithPriority(&d->ahead_stream, cudaStreamNonBlocking, lo));
    SL_CUDA(cudaEventCreateWithFlags(&d->ahead_ev, cudaEventDisableTiming));
    SL_CUDA(cudaEventCreateWithFlags(&d->fork_ev, cudaEventDisableTiming));
  }
  SL_CUDA(cudaEventRecord(d->fork_ev, stream));
  SL_CUDA(cudaStreamWaitEvent(d->ahead_stream, d->fork_ev, 0));
  const bool sh = d->s[0].sharded[k];
  const int nloc = (sh || !d->virt) ? (int)d->s.size() : 1;
  for (int i = 0; i < nloc; ++i) { int r = setup_slab_level(d, d->s[i], k, d->ahead_stream); if (r) return r; }
  SL_CUDA(cudaEventRecord(d->ahead_ev, d->ahead_stream));
  d->fin_ahead = true;
  return ECMG_OK;
}

int slab_first_sharded(const SlabDriver* d) {
  const auto& sh = d->s[0].sharded;
  for (int k = 0; k < (int)sh.size(); ++k)
    if (sh[k]) return k;
  return (int)sh.size();
}

int slab_import_u(SlabDriver* d, int k, const double* u_full, cudaStream_t stream) {
  for (auto& c : d->s)
    SL_CUDA(cudaMemcpyAsync(c.u[k], u_full, sizeof(double) * level_nodes(c.geom[k]), cudaMemcpyDeviceToDevice, stream));
  return ECMG_OK;
}

int slab_run(SlabDriver* d, double eps, ecmg_stats* per_level, double* u_out, bool u_dev, double* ut_out, bool ut_dev,
             cudaStream_t stream, int k_begin) {
  const SlabCfg& cf = d->cfg;
  const int L = cf.L;
  int status = ECMG_OK;
  for (int k = k_begin; k < L; ++k) {
    ecmg_stats st{};
    const bool sh = d->s[0].sharded[k];
    const int nloc = (sh || !d->virt) ? (int)d->s.size() : 1;
    cudaEvent_t e0, e1, e2, e3;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
    SL_CUDA(cudaEventRecord(e0, stream));
    if (k == L - 1 && d->fin_ahead) {   // set up ahead (slab_setup_ahead) while the replicated levels ran
      SL_CUDA(cudaStreamWaitEvent(stream, d->ahead_ev, 0));
      d->fin_ahead = false;
    } else {
      for (int i = 0; i < nloc; ++i) { int r = setup_slab_level(d, d->s[i], k, stream); if (r) return r; }
    }
    SL_CUDA(cudaEventRecord(e1, stream));
    for (int i = 0; i < nloc; ++i) {
      SlabCtx& c = d->s[i];
      const LevelGeom& g = c.geom[k];
      if (k < 2) SL_CUDA(launch_zero_vec(g, c.x, stream));   // DSOLVE: zero free guess (reading A12)
      else SL_CUDA(launch_exp_finite(g, level_problem(cf, k), c.u[k - 1], c.u[k - 2], c.x, cf.exp_variant, c.seeds, 1, stream));
    }
    SL_CUDA(cudaEventRecord(e2, stream));
    int s = slab_jcg(d, k, k < 2 ? 1e-14 : eps, 10000, &st, stream);
    if (k < 2 && s == ECMG_ENOTCONV) s = ECMG_OK;
    if (s == ECMG_ECUDA || s == ECMG_ENOMEM || s == ECMG_ENCCL) return s;
    if (s != ECMG_OK && status == ECMG_OK) status = s;
    for (int i = 0; i < nloc; ++i) {
      SlabCtx& c = d->s[i];
      SL_CUDA(launch_scatter(c.geom[k], c.x, c.u[k], stream));
      SL_CUDA(launch_dirichlet_fill(c.geom[k], level_problem(cf, k), c.u[k], 0.0, 0, stream));
    }
    if (sh) {
      int r = comm_u_halo(d, k, stream);
      if (r) return r;
    } else if (d->virt) {   // replicated level solved once: every virtual slab gets the full vector
      for (size_t i = 1; i < d->s.size(); ++i)
        SL_CUDA(cudaMemcpyAsync(d->s[i].u[k], d->s[0].u[k], sizeof(double) * level_nodes(d->s[0].geom[k]),
                                cudaMemcpyDeviceToDevice, stream));
    }
    SL_CUDA(cudaEventRecord(e3, stream));
    if (k == L - 1 && k >= 2 && ut_out)
      for (int i = 0; i < nloc; ++i)
        SL_CUDA(launch_exp_true(d->s[i].geom[k], level_problem(cf, k), d->s[i].u[k], d->s[i].u[k - 1], d->s[i].ut, stream));
    SL_CUDA(cudaStreamSynchronize(stream));
    float a = 0.f, b = 0.f, c3 = 0.f;
    cudaEventElapsedTime(&a, e0, e1); cudaEventElapsedTime(&b, e1, e2); cudaEventElapsedTime(&c3, e2, e3);
    st.ms_setup = a; st.ms_exp = b; st.ms_solve = c3; st.ms_rich = 0.0;
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2); cudaEventDestroy(e3);
    if (per_level) per_level[k] = st;
  }
  // outputs
  const int kf = L - 1;
  const LevelGeom& gf0 = d->s[0].geom[kf];
  const long long pl = (long long)(gf0.n[0] + 1) * (gf0.n[1] + 1);
  const bool sh = d->s[0].sharded[kf];
  for (size_t i = 0; i < d->s.size(); ++i) {
    SlabCtx& c = d->s[i];
    const LevelGeom& g = c.geom[kf];
    const long long z0 = sh ? g.zlo : 0, z1 = sh ? g.zhi : g.n[2] + 1;
    if (d->virt && !sh && i > 0) break;   // replicated finest level: slab 0 has everything
    const long long dst0 = d->virt ? z0 * pl : 0;   // virtual: full layout; NCCL: local slab
    SL_CUDA(cudaMemcpyAsync(u_out + dst0, c.u[kf] + z0 * pl, sizeof(double) * (z1 - z0) * pl,
                            u_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, stream));
    if (ut_out)
      SL_CUDA(cudaMemcpyAsync(ut_out + dst0, c.ut + z0 * pl, sizeof(double) * (z1 - z0) * pl,
                              ut_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, stream));
  }
  SL_CUDA(cudaStreamSynchronize(stream));
  return status;
}

// JCG on one level through the slabs. u: full-layout (virtual) or this rank's planes [zlo, zhi)
// (NCCL) of the level; in = guess, out = iterate with g_D on Dirichlet nodes.
int slab_solve_level(SlabDriver* d, int k, double eps, int max_iter, double* u, ecmg_stats* st, cudaStream_t stream) {
  const SlabCfg& cf = d->cfg;
  const bool sh = d->s[0].sharded[k];
  const int nloc = (sh || !d->virt) ? (int)d->s.size() : 1;
  const LevelGeom& g0 = d->s[0].geom[k];
  const long long pl = (long long)(g0.n[0] + 1) * (g0.n[1] + 1);
  for (int i = 0; i < nloc; ++i) {
    SlabCtx& c = d->s[i];
    int r = setup_slab_level(d, c, k, stream);
    if (r) return r;
    // the caller's vector -> this slab's full-layout u_k (owned planes), then gather into x
    const long long z0 = c.geom[k].zlo, z1 = c.geom[k].zhi;
    const long long src0 = d->virt ? z0 * pl : 0;
    SL_CUDA(cudaMemcpyAsync(c.u[k] + z0 * pl, u + src0, sizeof(double) * (z1 - z0) * pl, cudaMemcpyDeviceToDevice, stream));
    SL_CUDA(launch_gather(c.geom[k], c.u[k], c.x, stream));
  }
  const int s = slab_jcg(d, k, eps, max_iter, st, stream);
  if (s == ECMG_ECUDA || s == ECMG_ENOMEM || s == ECMG_ENCCL) return s;
  for (int i = 0; i < nloc; ++i) {
    SlabCtx& c = d->s[i];
    SL_CUDA(launch_scatter(c.geom[k], c.x, c.u[k], stream));
    SL_CUDA(launch_dirichlet_fill(c.geom[k], level_problem(cf, k), c.u[k], 0.0, 0, stream));
    const long long z0 = c.geom[k].zlo, z1 = c.geom[k].zhi;
    const long long dst0 = d->virt ? z0 * pl : 0;
    SL_CUDA(cudaMemcpyAsync(u + dst0, c.u[k] + z0 * pl, sizeof(double) * (z1 - z0) * pl, cudaMemcpyDeviceToDevice, stream));
  }
  SL_CUDA(cudaStreamSynchronize(stream));
  return s;
}

}  // namespace ecmg
