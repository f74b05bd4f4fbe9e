// ecmg_api.cu -- host implementation of the C ABI in include/ecmg.h.
//
// Alg. 4 runs as a stream of kernel launches on the grid's CUDA stream. The JCG loop
// (Alg. 4 l.7-9) keeps every CG scalar on the device; the host only reads back a 64-byte scalar
// block once per launched batch, and launches the next batch before waiting on the previous
// one. Kernels launched after convergence see the device "done" flag and return immediately,
// so the iterate stops at exactly the iteration where ||r|| <= eps ||f|| (no check-every-k).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/ecmg.h"
#include "ecmg_internal.cuh"
#include "problems.cuh"
#include "host_common.h"
#include "slab.h"

using namespace ecmg;

#include <atomic>
static std::atomic<long long> g_launches{0};
namespace ecmg { void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); } }

#ifdef ECMG_TESTING
// test build: guard bands of kGuard bytes of the pattern 0xA5 before and after every device buffer; a write out of
// bounds by up to kGuard bytes on either side changes them. Checked on free and by ecmg_test_guard_check.
#include <mutex>
#include <unordered_map>
namespace {
constexpr size_t kGuard = 8192;
std::mutex g_guard_mu;
std::unordered_map<void*, size_t> g_guarded;   // user pointer -> size in bytes
long long g_guard_bad = 0;                      // corrupted guard bytes found on frees so far

long long guard_bad_bytes(const char* user, size_t bytes) {
  std::vector<unsigned char> h(2 * kGuard);
  const size_t tail = kGuard + (bytes + 255) / 256 * 256 - bytes;   // the pad to the next 256 B belongs to the band
  if (cudaMemcpy(h.data(), user - kGuard, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(h.data() + kGuard, user + bytes, std::min(tail, kGuard), cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  long long bad = 0;
  for (size_t i = 0; i < kGuard + std::min(tail, kGuard); ++i) bad += h[i] != 0xA5;
  return bad;
}
}  // namespace
namespace ecmg {
cudaError_t dev_malloc(void** p, size_t bytes) {
  char* base = nullptr;
  const size_t padded = (bytes + 255) / 256 * 256;
  cudaError_t e = cudaMalloc(&base, padded + 2 * kGuard);
  if (e != cudaSuccess) { *p = nullptr; return e; }
  cudaMemset(base, 0xA5, kGuard);
  cudaMemset(base + kGuard + bytes, 0xA5, padded - bytes + kGuard);
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(g_guard_mu);
  g_guarded[base + kGuard] = bytes;
  *p = base + kGuard;
  return cudaSuccess;
}
void dev_free(void* p) {
  if (!p) return;
  size_t bytes = 0;
  {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    auto it = g_guarded.find(p);
    if (it == g_guarded.end()) { cudaFree(p); return; }
    bytes = it->second;
    g_guarded.erase(it);
  }
  cudaDeviceSynchronize();
  const long long bad = guard_bad_bytes(static_cast<const char*>(p), bytes);
  if (bad) {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    g_guard_bad += bad > 0 ? bad : 1;
  }
  cudaFree(static_cast<char*>(p) - kGuard);
}
}  // namespace ecmg
// corrupted guard bytes over every live device buffer plus those found on frees since the last call (then reset)
extern "C" long long ecmg_test_guard_check(void) {
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(g_guard_mu);
  long long bad = g_guard_bad;
  g_guard_bad = 0;
  for (const auto& kv : g_guarded) {
    const long long b = guard_bad_bytes(static_cast<const char*>(kv.first), kv.second);
    bad += b > 0 ? b : (b < 0 ? 1 : 0);
  }
  return bad;
}
extern "C" long long ecmg_test_guarded_buffers(void) {
  std::lock_guard<std::mutex> lk(g_guard_mu);
  return (long long)g_guarded.size();
}
#else
namespace ecmg {
cudaError_t dev_malloc(void** p, size_t bytes) { return cudaMalloc(p, bytes); }
void dev_free(void* p) { cudaFree(p); }
}  // namespace ecmg
#endif

using ParamHost = JcgParams;

struct ecmg_grid {
  int device = 0;
  cudaStream_t stream = nullptr;
  ecmg_box dom{};
  int n0[3] = {0, 0, 0};
  int L = 0;
  bool has_problem = false;
  Problem prob{};
  int elem_path = 0;
  int exp_variant = 0, precond = 1, zchunk = 0;
  std::vector<LevelGeom> geom;
  // device workspace
  double* x = nullptr;
  double* r = nullptr;
  double* p[2] = {nullptr, nullptr};
  double* b = nullptr;             // finest level's right-hand side (bl[L-1])
  std::vector<double*> bl;         // per-level right-hand sides (setup of every level can run ahead)
  std::vector<double*> betal;      // per-level element beta (element path)
  std::vector<double*> s1d;        // per-level 1D Gauss load tables (separable right-hand sides)
  std::vector<char> setup_ok;      // level k's b / beta hold the current problem's data
  std::vector<const double*> arrays;   // ECMG_PROB_ARRAYS: the caller's device arrays, 5 per level (alpha_q may be null)
  int setup_ahead = 1;             // ECMG_OPT_SETUP_AHEAD
  int beta_fly = 0;                // ECMG_OPT_BETA_FLY: element kernels form analytic beta from axis tables (measured:
                                   // 16 B/unknown less traffic but no faster -- the element kernels are latency bound)
  int exp_fused = 1;               // ECMG_OPT_EXP_KERNEL: 1 fused one-pass EXP_finite, 0 seeds + interpolation passes
  int rhs_sym_min = 248;           // ECMG_OPT_RHS_SYM: smallest free-box extent for the permutation-symmetric C4 load
  int setup_ctas = 0;              // ECMG_OPT_SETUP_CTAS: CTAs per SM of the ALU-bound RHS kernel when run ahead
  cudaStream_t hi_stream = nullptr, lo_stream = nullptr;   // ecmg_run: solves (high) / level setup (low priority)
  cudaStream_t lo2_stream = nullptr;                        // the finest level's setup (starts at once, beside lo_stream)
  int setup_ahead_prio = 1;   // the coarse levels' setups at the solves' priority (they are short and needed soon)
  std::vector<cudaEvent_t> setup_ev;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  double* zv = nullptr;            // element path: z = D^-1 r (K2 / INIT write it, K1 reads it)
  double* partials = nullptr;
  JcgScalars* sc = nullptr;
  JcgScalars* sc_host = nullptr;   // pinned, 2 slots
  std::vector<double*> u;          // per-level full nodal vectors (ecmg_run)
  double* ut_tmp = nullptr;
  double* seeds = nullptr;         // EXP_finite: extrapolated values on the 2h grid of the finest level
  long long vec_doubles = 0, beta_doubles = 0, partial_doubles = 0;
  cudaEvent_t ev[16];
  bool ev_init = false;
  int kernel_variant = 1;   // ECMG_OPT_KERNEL
  int use_graph = 1;        // ECMG_OPT_GRAPH: device-driven JCG loop (CUDA graph, conditional WHILE node)
  int unfused = 0;          // ECMG_OPT_UNFUSED: fixed-count constant-stencil solves by the textbook sequence
  int p0_init = 1;          // ECMG_OPT_P0_INIT: the init pass stores p_0 = D^-1 r_0 instead of r_0 (KArgs::p0)
  int rich_fused = 1;       // ECMG_OPT_RICH_FUSED: the finest level's true-residual pass also forms EXP_true
  double* rich_ut = nullptr;          // set by run_cascade around the finest level's solve (else null)
  const double* rich_u2h = nullptr;
  int xdefer = 1;           // ECMG_OPT_XDEFER: TMA K2 updates x every second iteration (bitwise the same iterates)
  int shard_min = kShardMinDefault;   // ECMG_OPT_SHARD_MIN: z-slabs split only levels with >= this many z cells
  int hybrid = 1;           // ECMG_OPT_SLAB_HYBRID: z-slabs, replicated levels through the single-GPU path
  int fused_halo = 1;       // ECMG_OPT_FUSED_HALO: z-slab halo planes stored by K2 / init into the neighbours
  int pdl = 0;              // ECMG_OPT_PDL: programmatic dependent launch between the JCG kernels (measured: no gain
                            // inside the CUDA graphs, tools/tune_pdl.py; off by default)
  long long cta_max = 1000;           // ECMG_OPT_CTA_SOLVE: one-CTA solve up to this many free unknowns (0: off)
  long long pers_tma_max = 20000000;  // ECMG_OPT_PERS_TMA: constant stencil, one cooperative TMA solve up to this size (256^3: 2.68 -> 2.29 ms per solve, tools/tts_ab.py)
  long long persistent_max = 40000;   // ECMG_OPT_PERSISTENT: register-resident cooperative solve up to this size (tools/tune_persistent.py:
                                      // 64^3 is faster as the cooperative TMA solve, 0.67 vs 0.82 ms on C4)
  double* aux[2] = {nullptr, nullptr};   // persistent element-path solve: w = A p and D^-1 (level-sized)
  long long aux_doubles = 0;
  cudaStream_t cap_stream = nullptr;          // private stream used only for graph capture
  ParamHost* param_host = nullptr;   // pinned
  std::vector<cudaGraphExec_t> graphs;        // per level, lazily built
  struct Maps { int level = -1; CUtensorMap xh, xi, rh, ri, ph[2], pi[2], bi; bool ok = false; } maps;
  double last_jcg_ms = 0.0;
  int last_jcg_iters = 0;
  long long last_free = 0;
  // z-slabs: NCCL ranks (dist) or virtual slabs on this GPU (ECMG_OPT_VIRTUAL_SLABS)
  int nranks = 1, rank = 0;
  int size_level = 0;   // the single-GPU workspace covers levels <= size_level (z-slabs: the replicated ones)
  unsigned char nccl_id[128] = {0};
  int virt_slabs = 0;
  SlabDriver* slab = nullptr;
  // asynchronous ecmg_run: per-level parameters / scalars (pinned) and events
  ParamHost* lvl_param = nullptr;
  JcgScalars* lvl_sc = nullptr;
  std::vector<cudaEvent_t> lvl_ev;
  std::vector<char> lvl_graph;     // the level's last async solve ran its CUDA graph (launch count from iterations)
};

namespace {

void clear_graphs(ecmg_grid* G) {
  for (auto& e : G->graphs)
    if (e) cudaGraphExecDestroy(e);
  G->graphs.assign(G->L, nullptr);
}

inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? ECMG_OK : (e == cudaErrorMemoryAllocation ? ECMG_ENOMEM : ECMG_ECUDA); }

// ECMG_DEBUG=1 in the environment prints the failing call and the CUDA error string
inline int report_cuda(cudaError_t e, const char* what, int line) {
  static const bool dbg = std::getenv("ECMG_DEBUG") != nullptr;
  if (dbg) std::fprintf(stderr, "libecmg: %s failed at ecmg_api.cu:%d: %s\n", what, line, cudaGetErrorString(e));
  return cuda_status(e);
}

#define ECMG_CUDA(call)                                              \
  do {                                                               \
    cudaError_t e_ = (call);                                         \
    if (e_ != cudaSuccess) return report_cuda(e_, #call, __LINE__);  \
  } while (0)

SlabCfg slab_cfg(const ecmg_grid* G) {
  SlabCfg c{};
  c.dom = G->dom;
  for (int d = 0; d < 3; ++d) c.n0[d] = G->n0[d];
  c.L = G->L;
  c.prob = G->prob;
  c.elem_path = G->elem_path;
  c.exp_variant = G->exp_variant;
  c.precond = G->precond;
  c.kernel_variant = G->kernel_variant;
  c.zchunk = G->zchunk;
  c.fused_halo = G->fused_halo;
  c.beta_fly = G->beta_fly;
  c.shard_min = G->shard_min;
  c.use_graph = G->use_graph;
  c.arrays = G->arrays;
  return c;
}

// TMA descriptors of the free-box work vectors for one level (cached; rebuilt when the level changes)
bool ensure_maps(ecmg_grid* G, const LevelGeom& g, int level) {
  auto& M = G->maps;
  if (M.level == level) return M.ok;
  const int hx = tma_halo_box_x(), hy = tma_halo_box_y(), ix = tma_int_box_x(), iy = tma_int_box_y();
  M.ok = make_vec_tensor_map(&M.xh, G->x, g, hx, hy) == 0 && make_vec_tensor_map(&M.xi, G->x, g, ix, iy) == 0 &&
         make_vec_tensor_map(&M.rh, G->r, g, hx, hy) == 0 && make_vec_tensor_map(&M.ri, G->r, g, ix, iy) == 0 &&
         make_vec_tensor_map(&M.ph[0], G->p[0], g, hx, hy) == 0 && make_vec_tensor_map(&M.ph[1], G->p[1], g, hx, hy) == 0 &&
         make_vec_tensor_map(&M.pi[0], G->p[0], g, ix, iy) == 0 && make_vec_tensor_map(&M.pi[1], G->p[1], g, ix, iy) == 0 &&
         make_vec_tensor_map(&M.bi, G->bl[level], g, ix, iy) == 0;
  M.level = level;
  return M.ok;
}

const CUtensorMap* halo_map(ecmg_grid* G, const double* p) {
  auto& M = G->maps;
  if (p == G->x) return &M.xh;
  if (p == G->r) return &M.rh;
  if (p == G->p[0]) return &M.ph[0];
  if (p == G->p[1]) return &M.ph[1];
  return nullptr;
}
const CUtensorMap* int_map(ecmg_grid* G, const double* p) {
  auto& M = G->maps;
  if (p == G->x) return &M.xi;
  if (p == G->r) return &M.ri;
  if (p == G->p[0]) return &M.pi[0];
  if (p == G->p[1]) return &M.pi[1];
  if (M.level >= 0 && p == G->bl[M.level]) return &M.bi;
  return nullptr;
}

int level_of(const ecmg_grid* G, const LevelGeom& g) {
  for (int k = 0; k < G->L; ++k) if (&G->geom[k] == &g) return k;
  return -1;
}

Problem level_prob(const ecmg_grid* G, int k);

cudaError_t launch_mode(ecmg_grid* G, int mode, const LevelGeom& g, const KArgs& a) {
  if (G->elem_path) {
    ElemStencil es = make_elem_stencil(g, level_prob(G, level_of(G, g)), G->precond);
    if (G->beta_fly && a.beta) set_beta_fly(es, g, G->prob, a.beta);
    return launch_jcg_elem(mode, g, es, G->prob, a, G->stream);
  }
  const ConstStencil cs = make_const_stencil(g, 1.0, G->precond);
  if (G->kernel_variant == 1 && ensure_maps(G, g, level_of(G, g))) {
    const CUtensorMap* h0 = halo_map(G, a.h0);
    const CUtensorMap* h1 = a.h1 ? halo_map(G, a.h1) : h0;
    // (KArgs::p0: the first K1 reads p_0 from its own output vector -- that halo map rides in the I0 slot)
    const CUtensorMap* i0 = (mode == MODE_K1 && a.p0) ? halo_map(G, a.o0) : (a.i0 ? int_map(G, a.i0) : h0);
    const CUtensorMap* i1 = a.i1 ? int_map(G, a.i1) : h0;
    const CUtensorMap* i2 = a.i2 ? int_map(G, a.i2) : h0;
    if (h0 && h1 && i0 && i1 && i2) {
      CUtensorMap m[5] = {*h0, *h1, *i0, *i1, *i2};
      return launch_jcg_const_tma(mode, g, cs, a, m, G->stream);
    }
  }
  return launch_jcg_const(mode, g, cs, a, G->stream);
}

// Level setup (row a1): element beta, lifted right-hand side b_k. Independent of every solution, so
// ecmg_run enqueues it for all levels up front on a low-priority stream (ECMG_OPT_SETUP_AHEAD).
// the problem as level k's kernels see it (ECMG_PROB_ARRAYS: with that level's caller arrays)
Problem level_prob(const ecmg_grid* G, int k) {
  Problem p = G->prob;
  if (p.id == PROB_ARRAYS && (int)G->arrays.size() == 5 * G->L)
    for (int j = 0; j < 5; ++j) p.arr[j] = G->arrays[5 * k + j];
  return p;
}

int setup_level_on(ecmg_grid* G, int k, cudaStream_t st, int ctas_per_sm = 0) {
  const LevelGeom& g = G->geom[k];
  const Problem pk = level_prob(G, k);
  const ElemStencil es = make_elem_stencil(g, pk, G->precond);
  if (G->elem_path) ECMG_CUDA(launch_beta(g, pk, G->betal[k], st));
  ECMG_CUDA(launch_rhs(g, pk, es, 1.0, G->elem_path ? G->betal[k] : nullptr, G->bl[k], G->s1d[k], st, ctas_per_sm, G->rhs_sym_min));
  G->setup_ok[k] = 1;
  return ECMG_OK;
}
int setup_level(ecmg_grid* G, int k) { return setup_level_on(G, k, G->stream); }
void invalidate_setup(ecmg_grid* G) { std::fill(G->setup_ok.begin(), G->setup_ok.end(), 0); }


int stats_from(const JcgScalars& s, double eps, ecmg_stats* st) {
  const double nb = std::sqrt(s.bb);
  const double nbe = nb > 0.0 ? nb : 1.0;
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

int fill_stats(ecmg_grid* G, const LevelGeom& g, double eps, ecmg_stats* st) {
  const JcgScalars s = G->sc_host[0];
  G->last_jcg_iters = s.iter;
  G->last_free = free_count(g);
  const double nb = std::sqrt(s.bb);
  const double nbe = nb > 0.0 ? nb : 1.0;
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

// Device-driven JCG (Alg. 4 l.7-9): one CUDA graph per level = init -> WHILE(cond){K1,K2,K1,K2} -> true
// residual. The init pass and every K2 (and K1 on breakdown) set cond = !done from their last CTA,
// so the loop stops after exactly the iteration that meets ||r|| <= eps ||f|| (the second K1/K2 of a
// body run after convergence sees done and returns). No host round trip per iteration.
// deferred x update (KArgs::xdefer): the launched TMA K1 / K2 kernels -- the constant
// stencil, and the element operator with beta from the array and per-face alpha (the conditions under which
// launch_jcg_elem has the deferred-x K2 variants; they must agree, the host owes the update k_xfix applies)
bool use_xdefer(ecmg_grid* G, const LevelGeom& g) {
  if (!G->xdefer) return false;
  if (G->elem_path) {
    const int k = level_of(G, g);
    // (value 2 only: measured slower there -- the element kernels are issue bound, not HBM bound)
    return G->xdefer == 2 && k >= 0 && !G->beta_fly && !(G->prob.id == PROB_ARRAYS && level_prob(G, k).arr[4]);
  }
  return G->kernel_variant == 1 && ensure_maps(G, g, level_of(G, g));
}

bool rich_level_ok(ecmg_grid* G, int k);

// p_0 from the init pass (KArgs::p0): the launched constant-stencil TMA kernels
// of this grid's own (single-GPU) solves
bool use_p0(ecmg_grid* G, const LevelGeom& g) {
  return G->p0_init && !G->elem_path && G->kernel_variant == 1 && ensure_maps(G, g, level_of(G, g));
}

cudaError_t build_level_graph(ecmg_grid* G, int k, cudaGraphExec_t* out) {
  const LevelGeom& g = G->geom[k];
  const bool defer = use_xdefer(G, g);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaGraphCreate(&graph, 0);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle h;
  e = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault);
  KArgs a{};
  a.partials = G->partials; a.sc = G->sc; a.pdl = G->pdl; a.zc = auto_zc(G->zchunk, G->elem_path, g); a.beta = G->betal[k];
  a.cond = h; a.use_cond = 1;
  const long long launches_before = ecmg_kernel_launches();
  cudaStream_t user = G->stream;
  G->stream = G->cap_stream;   // launchers enqueue on G->stream: point it at the capture stream
  cudaGraphNode_t init_node = nullptr, cond_node = nullptr;
  auto done = [&](cudaError_t err) { G->stream = user; return err; };
  if (e != cudaSuccess) return done(e);
  // init pass
  e = cudaStreamBeginCaptureToGraph(G->cap_stream, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return done(e);
  const bool p0 = use_p0(G, g);
  a.p0 = p0 ? 1 : 0;   // (the init pass then writes p_0 into p[1], the first K1's output vector)
  { KArgs ai = a; ai.h0 = G->x; ai.i0 = G->bl[k]; ai.o0 = p0 ? G->p[1] : G->r; ai.o1 = G->zv; e = launch_mode(G, MODE_INIT, g, ai); }
  cudaError_t e2 = cudaStreamEndCapture(G->cap_stream, &graph);
  if (e != cudaSuccess || e2 != cudaSuccess) return done(e != cudaSuccess ? e : e2);
  size_t nn = 1;
  e = cudaGraphGetNodes(graph, &init_node, &nn);
  if (e != cudaSuccess || nn != 1) return done(e != cudaSuccess ? e : cudaErrorUnknown);
  // WHILE node and its body (two JCG iterations: p ping-pong)
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  e = cudaGraphAddNode(&cond_node, graph, &init_node, 1, &cp);
  if (e != cudaSuccess) return done(e);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(G->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return done(e);
  for (int half = 0; half < 2 && e == cudaSuccess; ++half) {
    KArgs a1 = a;
    a1.h0 = G->elem_path ? G->zv : G->r; a1.h1 = G->p[half]; a1.o0 = G->p[1 - half];
    e = launch_mode(G, MODE_K1, g, a1);
    if (e != cudaSuccess) break;
    KArgs a2 = a;
    a2.h0 = G->p[1 - half]; a2.i0 = G->x; a2.i1 = G->elem_path ? G->zv : G->r; a2.o0 = G->x; a2.o1 = G->r; a2.o2 = G->zv;
    if (defer) { a2.xdefer = 1 + half; a2.i2 = G->p[half]; }   // even k: skip x; odd k: both updates
    e = launch_mode(G, MODE_K2, g, a2);
  }
  e2 = cudaStreamEndCapture(G->cap_stream, &body);
  if (e != cudaSuccess || e2 != cudaSuccess) return done(e != cudaSuccess ? e : e2);
  // true residual after the loop
  e = cudaStreamBeginCaptureToGraph(G->cap_stream, graph, &cond_node, nullptr, 1, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return done(e);
  if (defer) e = launch_xfix(g, G->x, G->p[1], G->sc, G->stream);   // a skipped update still owed
  if (e == cudaSuccess) {
    KArgs at = a; at.use_cond = 0; at.h0 = G->x; at.i0 = G->bl[k];
    at.rich = rich_level_ok(G, k) ? 1 : 0;   // (forms u~_h only in a run that sets JcgParams::ut_out)
    e = launch_mode(G, MODE_TRUE, g, at);
  }
  e2 = cudaStreamEndCapture(G->cap_stream, &graph);
  if (e != cudaSuccess || e2 != cudaSuccess) return done(e != cudaSuccess ? e : e2);
  e = cudaGraphInstantiate(out, graph, 0);
  cudaGraphDestroy(graph);
  count_launch((int)(launches_before - ecmg_kernel_launches()));   // captured, not launched
  return done(e);
}

int run_jcg_graph(ecmg_grid* G, int k, double eps, ecmg_stats* st) {
  const LevelGeom& g = G->geom[k];
  if ((int)G->graphs.size() != G->L) G->graphs.assign(G->L, nullptr);
  if (!G->graphs[k]) ECMG_CUDA(build_level_graph(G, k, &G->graphs[k]));
  ECMG_CUDA(cudaEventRecord(G->ev[0], G->stream));
  ECMG_CUDA(cudaGraphLaunch(G->graphs[k], G->stream));
  ECMG_CUDA(cudaEventRecord(G->ev[1], G->stream));
  ECMG_CUDA(cudaMemcpyAsync(&G->sc_host[0], G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
  ECMG_CUDA(cudaStreamSynchronize(G->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, G->ev[0], G->ev[1]);
  G->last_jcg_ms = ms;
  const int it = G->sc_host[0].iter;
  count_launch(2 + 4 * ((it + 1) / 2));   // init + true residual + executed loop bodies
  return fill_stats(G, g, eps, st);
}

// (these selectors act on this grid's own single-GPU buffers; on z-slab grids only the replicated levels
// of the hybrid cascade reach them)
// the smallest levels: the whole solve in one CTA with every vector in shared memory
bool use_cta(const ecmg_grid* G, const LevelGeom& g) {
  return G->cta_max > 0 && cta_solve_fits(g, G->elem_path, G->cta_max);
}

bool use_persistent(const ecmg_grid* G, const LevelGeom& g) {
  if (use_cta(G, g)) return true;
  if (G->persistent_max <= 0 || free_count(g) > G->persistent_max) return false;
  const long long nbricks = (long long)((g.nf[0] + 7) / 8) * ((g.nf[1] + 7) / 8) * ((g.nf[2] + 3) / 4);
  return nbricks <= persistent_max_bricks(G->elem_path);   // every brick's nodes stay in registers
}

// mid-size levels, constant stencil: the whole solve in one cooperative launch of TMA z-marching passes
constexpr long long kElemPersTmaMax = 3000000;

bool use_pers_tma(ecmg_grid* G, const LevelGeom& g) {
  if (G->pers_tma_max <= 0 || free_count(g) > G->pers_tma_max) return false;
  // the cooperative launch needs every (x, y) tile resident at once: wide, flat levels (or a GPU with
  // fewer SMs) take the graph path instead
  // the element operator's cooperative solve is capped at 128^3: at C3's 256^3 it measured slower than the
  // graph loop of K1 / K2 (32.5 -> 37.4 ms for the level, tools/tts_ab.py)
  if (G->elem_path) return free_count(g) <= kElemPersTmaMax && elem_pers_fits(g);
  return const_pers_fits(g) && G->kernel_variant == 1 && ensure_maps(G, g, level_of(G, g));
}

// EXP_true inside the true-residual pass (ECMG_OPT_RICH_FUSED): the launched constant-stencil TMA TRUE kernel of
// the finest level has the variant that also forms u~_h (KArgs::rich; it acts only when JcgParams::ut_out is set)
bool rich_level_ok(ecmg_grid* G, int k) {
  return G->rich_fused && !G->elem_path && G->kernel_variant == 1 && G->nranks == 1 && !G->slab && k == G->L - 1 && k >= 2 &&
         ensure_maps(G, G->geom[k], k);
}
// ... and the level's solve ends in that launched kernel (graph loop or host loop), not in a one-launch solve
bool rich_fused_solve(ecmg_grid* G, int k, double eps) {
  const LevelGeom& g = G->geom[k];
  return rich_level_ok(G, k) && !use_persistent(G, g) && !(eps > 0.0 && G->use_graph && use_pers_tma(G, g));
}

cudaError_t launch_pers_tma(ecmg_grid* G, const LevelGeom& g) {
  const int k = level_of(G, g);
  const ConstStencil cs = make_const_stencil(g, 1.0, G->precond);
  if (G->elem_path) {
    ElemStencil es = make_elem_stencil(g, level_prob(G, k), G->precond);
    if (G->beta_fly) set_beta_fly(es, g, G->prob, G->betal[k]);
    return launch_jcg_elem_pers(g, es, G->x, G->r, G->zv, G->p[0], G->p[1], G->bl[k], G->betal[k], G->partials, G->sc,
                                G->stream);
  }
  const auto& M = G->maps;
  CUtensorMap maps[7] = {M.xh, M.rh, M.ph[0], M.ph[1], M.xi, M.ri, M.bi};
  return launch_jcg_const_pers(g, cs, G->x, G->r, G->p[0], G->p[1], G->partials, G->sc, maps, G->stream, G->p0_init ? 1 : 0);
}

// the whole solve of a small level in one cooperative launch (kernels_jcg_persistent.cu)
cudaError_t launch_persistent(ecmg_grid* G, const LevelGeom& g) {
  const int k = level_of(G, g);
  const ConstStencil cs = make_const_stencil(g, 1.0, G->precond);
  if (use_cta(G, g)) {
    if (!G->elem_path) return launch_jcg_cta(g, cs, nullptr, G->x, G->r, nullptr, G->bl[k], G->sc, G->stream);
    const ElemStencil es = make_elem_stencil(g, level_prob(G, k), G->precond);
    return launch_jcg_cta(g, cs, &es, G->x, G->r, G->betal[k], G->bl[k], G->sc, G->stream);
  }
  // w = A p (and on the element path D^-1) in scratch vectors sized for the level (grown on demand)
  const long long need = g.S * g.nza + 64;
  if (G->aux_doubles < need) {
    dfree(G->aux[0]);
    dfree(G->aux[1]);
    G->aux[0] = G->aux[1] = nullptr;
    G->aux_doubles = 0;
    cudaError_t e = dmalloc(&G->aux[0], sizeof(double) * need);
    if (e == cudaSuccess) e = dmalloc(&G->aux[1], sizeof(double) * need);
    if (e != cudaSuccess) return e;
    G->aux_doubles = need;
  }
  if (!G->elem_path)
    return launch_jcg_persistent(g, cs, nullptr, G->x, G->r, nullptr, G->p[0], G->p[1], G->aux[0], nullptr, nullptr, G->bl[k],
                                 G->partials, G->sc, G->stream);
  const ElemStencil es = make_elem_stencil(g, level_prob(G, k), G->precond);
  return launch_jcg_persistent(g, cs, &es, G->x, G->r, G->zv, G->p[0], G->p[1], G->aux[0], G->aux[1], G->betal[k], G->bl[k],
                               G->partials, G->sc, G->stream);
}

// small levels: the whole solve in one cooperative launch (latency bound)
int run_jcg_persistent(ecmg_grid* G, int k, double eps, ecmg_stats* st) {
  const LevelGeom& g = G->geom[k];
  ECMG_CUDA(cudaEventRecord(G->ev[0], G->stream));
  ECMG_CUDA(launch_persistent(G, g));
  ECMG_CUDA(cudaEventRecord(G->ev[1], G->stream));
  ECMG_CUDA(cudaMemcpyAsync(&G->sc_host[0], G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
  ECMG_CUDA(cudaStreamSynchronize(G->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, G->ev[0], G->ev[1]);
  G->last_jcg_ms = ms;
  return fill_stats(G, g, eps, st);
}

// Enqueue a device-driven JCG solve (graph or persistent path) without any host synchronisation;
// the final scalars land in *slot (pinned) when the stream reaches them. Returns ECMG_EINVAL if
// the level needs the host loop (ablation path).
int enqueue_jcg(ecmg_grid* G, int k, double eps, int max_iter, double* u_out, ParamHost* param, JcgScalars* slot) {
  const LevelGeom& g = G->geom[k];
  const bool persistent = use_persistent(G, g);
  if (!(eps > 0.0) || (!persistent && !G->use_graph)) return ECMG_EINVAL;
  param->eps = eps;
  param->max_iter = max_iter;
  param->u_out = u_out;
  param->ut_out = G->rich_ut;
  param->u2h = G->rich_u2h;
  ECMG_CUDA(cudaMemcpyAsync(&G->sc->in, param, sizeof(JcgParams), cudaMemcpyHostToDevice, G->stream));
  if (free_count(g) == 0) {   // nothing to solve
    ECMG_CUDA(launch_empty_solve(G->sc, G->stream));
    if ((int)G->lvl_graph.size() != G->L) G->lvl_graph.assign(G->L, 0);
    G->lvl_graph[k] = 0;
    ECMG_CUDA(cudaMemcpyAsync(slot, G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
    return ECMG_OK;
  }
  if (persistent) {
    ECMG_CUDA(launch_persistent(G, g));
  } else if (use_pers_tma(G, g)) {
    ECMG_CUDA(launch_pers_tma(G, g));
  } else {
    if ((int)G->graphs.size() != G->L) G->graphs.assign(G->L, nullptr);
    if (!G->graphs[k]) ECMG_CUDA(build_level_graph(G, k, &G->graphs[k]));
    ECMG_CUDA(cudaGraphLaunch(G->graphs[k], G->stream));
  }
  if ((int)G->lvl_graph.size() != G->L) G->lvl_graph.assign(G->L, 0);
  G->lvl_graph[k] = (!persistent && !use_pers_tma(G, g)) ? 1 : 0;
  ECMG_CUDA(cudaMemcpyAsync(slot, G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
  return ECMG_OK;
}

// JCG on level k (right-hand side in G->bl[k]), starting from G->x. Fills stats (except timings). The true
// residual pass writes the solution into the free nodes of the full-layout vector u_out (if not null).
int run_jcg(ecmg_grid* G, int k, double eps, int max_iter, double* u_out, ecmg_stats* st) {
  const LevelGeom& g = G->geom[k];
  if (max_iter <= 0 && eps > 0) max_iter = 10000;
  if (max_iter < 0) max_iter = 0;
  KArgs a{};
  a.partials = G->partials;
  a.sc = G->sc;
  a.pdl = G->pdl;
  a.zc = auto_zc(G->zchunk, G->elem_path, g);
  a.beta = G->betal[k];
  // eps and max_iter reach the init pass through the device scalars
  G->param_host->eps = eps;
  G->param_host->max_iter = max_iter;
  G->param_host->u_out = u_out;
  G->param_host->ut_out = G->rich_ut;
  G->param_host->u2h = G->rich_u2h;
  ECMG_CUDA(cudaMemcpyAsync(&G->sc->in, G->param_host, sizeof(JcgParams), cudaMemcpyHostToDevice, G->stream));
  if (free_count(g) == 0) {   // nothing to solve
    ECMG_CUDA(cudaEventRecord(G->ev[0], G->stream));
    ECMG_CUDA(launch_empty_solve(G->sc, G->stream));
    ECMG_CUDA(cudaEventRecord(G->ev[1], G->stream));
    ECMG_CUDA(cudaMemcpyAsync(&G->sc_host[0], G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
    ECMG_CUDA(cudaStreamSynchronize(G->stream));
    G->last_jcg_ms = 0.0;
    return fill_stats(G, g, eps, st);
  }
  if (use_persistent(G, g)) return run_jcg_persistent(G, k, eps, st);
  if (eps > 0.0 && G->use_graph && use_pers_tma(G, g)) {
    ECMG_CUDA(cudaEventRecord(G->ev[0], G->stream));
    ECMG_CUDA(launch_pers_tma(G, g));
    ECMG_CUDA(cudaEventRecord(G->ev[1], G->stream));
    ECMG_CUDA(cudaMemcpyAsync(&G->sc_host[0], G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
    ECMG_CUDA(cudaStreamSynchronize(G->stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, G->ev[0], G->ev[1]);
    G->last_jcg_ms = ms;
    return fill_stats(G, g, eps, st);
  }
  if (eps > 0.0 && G->use_graph) return run_jcg_graph(G, k, eps, st);
  const bool defer = use_xdefer(G, g) && !(eps <= 0.0 && G->unfused);
  const bool p0 = use_p0(G, g) && !(eps <= 0.0 && G->unfused);
  a.p0 = p0 ? 1 : 0;
  // r = b - A x, rho = r.z, rr = r.r, stop test
  {
    KArgs ai = a;
    ai.h0 = G->x; ai.i0 = G->bl[k]; ai.o0 = p0 ? G->p[1] : G->r; ai.o1 = G->zv;
    ECMG_CUDA(launch_mode(G, MODE_INIT, g, ai));
  }
  long long it = 0;
  auto launch_iter = [&]() -> cudaError_t {
    KArgs a1 = a;
    a1.h0 = G->elem_path ? G->zv : G->r; a1.h1 = G->p[it & 1]; a1.o0 = G->p[(it + 1) & 1];
    cudaError_t e = launch_mode(G, MODE_K1, g, a1);
    if (e != cudaSuccess) return e;
    KArgs a2 = a;
    a2.h0 = G->p[(it + 1) & 1]; a2.i0 = G->x; a2.i1 = G->elem_path ? G->zv : G->r; a2.o0 = G->x; a2.o1 = G->r; a2.o2 = G->zv;
    if (defer) { a2.xdefer = 1 + (int)(it & 1); a2.i2 = G->p[it & 1]; }
    e = launch_mode(G, MODE_K2, g, a2);
    ++it;
    return e;
  };
  if (eps <= 0.0 && G->unfused && !G->elem_path) {
    // the ablation's scratch z is allocated before the timed window opens
    const long long need = g.S * g.nza + 64;
    if (G->aux_doubles < need) {
      dfree(G->aux[0]); dfree(G->aux[1]);
      G->aux[0] = G->aux[1] = nullptr;
      G->aux_doubles = 0;
      ECMG_CUDA(dmalloc(&G->aux[0], sizeof(double) * need));
      ECMG_CUDA(dmalloc(&G->aux[1], sizeof(double) * need));
      G->aux_doubles = need;
    }
  }
  ECMG_CUDA(cudaEventRecord(G->ev[0], G->stream));
  if (eps <= 0.0 && G->unfused && !G->elem_path) {
    // ablation: the unfused textbook sequence (kernels_textbook.cu), nine passes per iteration
    double* z = G->aux[0];
    double* p = G->p[0];
    double* w = G->p[1];
    const double dinv = make_const_stencil(g, 1.0, G->precond).dinv;
    ECMG_CUDA(launch_textbook(3, g, z, G->r, nullptr, G->sc, dinv, G->stream));   // z0 = D^-1 r0
    ECMG_CUDA(launch_textbook(4, g, p, z, nullptr, G->sc, 1.0, G->stream));       // p0 = z0
    for (int i = 0; i < max_iter; ++i) {
      if (i > 0) ECMG_CUDA(launch_textbook(4, g, p, z, nullptr, G->sc, 0.0, G->stream));   // p = z + beta p
      KArgs aa = a;
      aa.h0 = p; aa.o0 = w;
      ECMG_CUDA(launch_mode(G, MODE_APPLY, g, aa));                                           // w = A p
      ECMG_CUDA(launch_textbook(0, g, p, w, G->partials, G->sc, 0.0, G->stream));             // p.w
      ECMG_CUDA(launch_textbook(1, g, nullptr, nullptr, G->partials, G->sc, 0.0, G->stream)); // alpha
      ECMG_CUDA(launch_textbook(2, g, G->x, p, nullptr, G->sc, 1.0, G->stream));              // x += alpha p
      ECMG_CUDA(launch_textbook(2, g, G->r, w, nullptr, G->sc, -1.0, G->stream));             // r -= alpha w
      ECMG_CUDA(launch_textbook(3, g, z, G->r, nullptr, G->sc, dinv, G->stream));             // z = D^-1 r
      ECMG_CUDA(launch_textbook(0, g, G->r, z, G->partials, G->sc, 0.0, G->stream));          // r.z
      ECMG_CUDA(launch_textbook(1, g, nullptr, nullptr, G->partials, G->sc, 1.0, G->stream)); // beta, rho
      ECMG_CUDA(launch_textbook(0, g, G->r, G->r, G->partials, G->sc, 0.0, G->stream));       // r.r
      ECMG_CUDA(launch_textbook(1, g, nullptr, nullptr, G->partials, G->sc, 2.0, G->stream)); // rr, iter
    }
  } else if (eps <= 0.0) {
    for (int i = 0; i < max_iter; ++i) ECMG_CUDA(launch_iter());
  } else {
    const long long nfree = free_count(g);
    const bool small = nfree < (1LL << 20);
    int batch = 1;
    auto next_batch = [&]() { if (small) batch = std::min(batch * 2, 16); };
    // pipelined: batch i+1 is in flight while the host inspects batch i's scalars
    for (int i = 0; i < batch; ++i) ECMG_CUDA(launch_iter());
    ECMG_CUDA(cudaMemcpyAsync(&G->sc_host[0], G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
    ECMG_CUDA(cudaEventRecord(G->ev[2], G->stream));
    int slot = 0;
    long long guard = 0;
    while (true) {
      next_batch();
      for (int i = 0; i < batch; ++i) ECMG_CUDA(launch_iter());
      ECMG_CUDA(cudaMemcpyAsync(&G->sc_host[1 - slot], G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
      ECMG_CUDA(cudaEventRecord(G->ev[3 - slot], G->stream));
      ECMG_CUDA(cudaEventSynchronize(G->ev[2 + slot]));
      if (G->sc_host[slot].done) break;
      slot = 1 - slot;
      if (++guard > (long long)max_iter + 8) break;   // cannot happen: done is set at max_iter
    }
  }
  if (defer) ECMG_CUDA(launch_xfix(g, G->x, G->p[1], G->sc, G->stream));   // inside the timed window
  ECMG_CUDA(cudaEventRecord(G->ev[1], G->stream));
  // true residual RRe = ||b - A x|| / ||b||
  {
    KArgs at = a;
    at.h0 = G->x; at.i0 = G->bl[k];
    at.rich = rich_level_ok(G, k) ? 1 : 0;
    ECMG_CUDA(launch_mode(G, MODE_TRUE, g, at));
  }
  ECMG_CUDA(cudaMemcpyAsync(&G->sc_host[0], G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
  ECMG_CUDA(cudaStreamSynchronize(G->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, G->ev[0], G->ev[1]);
  G->last_jcg_ms = ms;
  return fill_stats(G, g, eps, st);
}

// DSOLVE (Alg. 4 l.1-2) runs JCG from zero to 1e-14 (reading A12), a target rounding may keep the recurrence
// residual just above on an ill-conditioned coarse grid. The direct-solve contract is the TRUE residual:
// rel_res_true <= 1e-12 is a solved level (status OK), anything above is reported as ENOTCONV (it would signal
// an assembly bug: SPEC coarse_solve).
constexpr double kDsolveTrueTol = 1e-12;
int dsolve_status(int s, ecmg_stats& st) {
  if (s != ECMG_ENOTCONV) return s;
  if (st.rel_res_true <= kDsolveTrueTol) { st.converged = 1; st.status = ECMG_OK; return ECMG_OK; }
  return ECMG_ENOTCONV;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}


float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) { cudaGetLastError(); return 0.f; }
  return ms;
}

}  // namespace

extern "C" {

long long ecmg_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int ecmg_slab_partition(int n_cells_z, int nranks, int rank, int* z_lo, int* z_hi) {
  if (n_cells_z < 1 || nranks < 1 || rank < 0 || rank >= nranks || !z_lo || !z_hi) return ECMG_EINVAL;
  return slab_partition(n_cells_z, nranks, rank, z_lo, z_hi) ? 1 : 0;
}

int ecmg_nccl_unique_id(unsigned char id[128]) {
  if (!id) return ECMG_EINVAL;
  return nccl_unique_id(id);
}

const char* ecmg_strerror(int s) {
  switch (s) {
    case ECMG_OK: return "ok";
    case ECMG_EINVAL: return "invalid argument";
    case ECMG_ENOMEM: return "out of device memory";
    case ECMG_ENOTCONV: return "JCG did not reach the relative-residual tolerance within max_iter";
    case ECMG_EBREAKDOWN: return "JCG breakdown: p.Ap <= 0 (operator not SPD)";
    case ECMG_EDIAG: return "non-positive diagonal entry";
    case ECMG_EMISMATCH: return "level / grid embedding mismatch";
    case ECMG_ECUDA: return "CUDA error or no CUDA device";
    case ECMG_ENCCL: return "NCCL error";
    default: return "unknown status";
  }
}

int ecmg_create_grid(const ecmg_box* dom, const int coarsest_cells[3], int num_levels, const ecmg_dist* dist,
                     void* cuda_stream, ecmg_grid** out) {
  if (!out) return ECMG_EINVAL;
  *out = nullptr;
  if (!dom || !coarsest_cells || num_levels < 3 || num_levels > 12) return ECMG_EINVAL;
  if (dist && (dist->nranks < 1 || dist->nranks > 16 || dist->rank < 0 || dist->rank >= dist->nranks)) return ECMG_EINVAL;
  for (int d = 0; d < 3; ++d) {
    if (!(dom->hi[d] > dom->lo[d]) || coarsest_cells[d] < 1) return ECMG_EINVAL;
    if ((long long)coarsest_cells[d] << (num_levels - 1) > 8192) return ECMG_EINVAL;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { cudaGetLastError(); return ECMG_ECUDA; }
  ecmg_grid* G = new (std::nothrow) ecmg_grid;
  if (!G) return ECMG_ENOMEM;
  cudaGetDevice(&G->device);
  G->stream = (cudaStream_t)cuda_stream;
  G->dom = *dom;
  for (int d = 0; d < 3; ++d) G->n0[d] = coarsest_cells[d];
  G->L = num_levels;
  // size workspace for the finest level with the largest possible free box (no Dirichlet faces)
  int face_none[6] = {FACE_ROBIN, FACE_ROBIN, FACE_ROBIN, FACE_ROBIN, FACE_ROBIN, FACE_ROBIN};
  // NCCL ranks keep the sharded levels' work vectors in the slab driver; the levels below the first
  // sharded one are solved replicated by this grid's single-GPU kernels (ecmg_run), so size for those
  int size_level = num_levels - 1;
  if (dist && dist->nranks > 1) {
    size_level = 0;
    for (int k = 0; k < num_levels; ++k) {
      int zlo, zhi;
      if (slab_partition((coarsest_cells[2]) << k, dist->nranks, 0, &zlo, &zhi, kShardMinDefault)) break;
      size_level = k;
    }
  }
  G->size_level = size_level;
  LevelGeom gmax = make_geom(*dom, coarsest_cells, size_level, face_none, 1);
  G->vec_doubles = gmax.S * gmax.nf[2] + 64;
  G->beta_doubles = beta_doubles(gmax);
  const long long rhs_blocks = (long long)((gmax.nf[0] + 7) / 8) * ((gmax.nf[1] + 7) / 8) * ((gmax.nf[2] + 3) / 4);
  const long long jcg_blocks = (long long)((gmax.nf[0] + 31) / 32) * ((gmax.nf[1] + 7) / 8) * gmax.nf[2];
  G->partial_doubles = 3 * std::max(rhs_blocks, jcg_blocks) + 64;   // grown below for the cooperative solves
  int st = ECMG_OK;
  auto alloc = [&](double** p, long long n) {
    if (st != ECMG_OK) return;
    if (dmalloc(p, sizeof(double) * n) != cudaSuccess) { cudaGetLastError(); st = ECMG_ENOMEM; return; }
    if (cudaMemsetAsync(*p, 0, sizeof(double) * n, G->stream) != cudaSuccess) st = ECMG_ECUDA;
  };
  alloc(&G->x, G->vec_doubles);
  alloc(&G->r, G->vec_doubles);
  alloc(&G->p[0], G->vec_doubles);
  alloc(&G->p[1], G->vec_doubles);
  // per-level right-hand sides and 1D load tables (the finest level's b is the full-size G->b)
  G->bl.assign(num_levels, nullptr);
  G->betal.assign(num_levels, nullptr);
  G->s1d.assign(num_levels, nullptr);
  G->setup_ok.assign(num_levels, 0);
  for (int k = 0; k < num_levels; ++k) {
    const LevelGeom gk = make_geom(*dom, coarsest_cells, std::min(k, size_level), face_none, 1);
    alloc(&G->bl[k], k == num_levels - 1 ? G->vec_doubles : gk.S * gk.nf[2] + 64);
    alloc(&G->s1d[k], 15LL * (   // 1D Gauss loads: up to 5 separable terms x 3 axes
        std::max(gk.n[0], std::max(gk.n[1], gk.n[2])) + 1));
  }
  G->b = G->bl[num_levels - 1];
  alloc(&G->seeds, (long long)(gmax.n[0] / 2 + 1) * (gmax.n[1] / 2 + 1) * (gmax.n[2] / 2 + 1));
  if (st == ECMG_OK && dmalloc(&G->sc, sizeof(JcgScalars)) != cudaSuccess) st = ECMG_ENOMEM;
  if (st == ECMG_OK && cudaMemsetAsync(G->sc, 0, sizeof(JcgScalars), G->stream) != cudaSuccess) st = ECMG_ECUDA;
  if (st == ECMG_OK && cudaHostAlloc(&G->sc_host, 2 * sizeof(JcgScalars), cudaHostAllocDefault) != cudaSuccess) st = ECMG_ENOMEM;
  if (st == ECMG_OK && cudaHostAlloc(&G->param_host, sizeof(*G->param_host), cudaHostAllocDefault) != cudaSuccess) st = ECMG_ENOMEM;
  if (st == ECMG_OK && cudaStreamCreateWithFlags(&G->cap_stream, cudaStreamNonBlocking) != cudaSuccess) st = ECMG_ECUDA;
  if (st == ECMG_OK) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);   // lo = least priority, hi = greatest
    if (cudaStreamCreateWithPriority(&G->hi_stream, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&G->lo_stream, cudaStreamNonBlocking, G->setup_ahead_prio ? hi : lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&G->lo2_stream, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&G->fork_ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&G->join_ev, cudaEventDisableTiming) != cudaSuccess)
      st = ECMG_ECUDA;
    G->setup_ev.assign(num_levels, nullptr);
    for (auto& e : G->setup_ev)
      if (st == ECMG_OK && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) st = ECMG_ECUDA;
  }
  G->graphs.assign(num_levels, nullptr);
  if (st == ECMG_OK && cudaHostAlloc(&G->lvl_param, sizeof(ParamHost) * num_levels, cudaHostAllocDefault) != cudaSuccess) st = ECMG_ENOMEM;
  if (st == ECMG_OK && cudaHostAlloc(&G->lvl_sc, sizeof(JcgScalars) * num_levels, cudaHostAllocDefault) != cudaSuccess) st = ECMG_ENOMEM;
  if (st == ECMG_OK) {
    G->lvl_ev.assign(5 * num_levels, nullptr);
    for (auto& e : G->lvl_ev) cudaEventCreate(&e);
  }
  if (st == ECMG_OK && (init_tma_kernel_attributes() != cudaSuccess || init_elem_kernel_attributes() != cudaSuccess ||
                        init_setup_kernel_attributes() != cudaSuccess || init_cta_kernel_attributes() != cudaSuccess ||
                        init_pers_kernel_attributes() != cudaSuccess || init_elem_pers_attributes() != cudaSuccess))
    st = ECMG_ECUDA;
  // the partial sums: per-CTA triples of the z-marching passes, or the two ping-pong buffers of the
  // cooperative solves (6 doubles per co-resident CTA), whichever is larger
  if (st == ECMG_OK) G->partial_doubles = std::max(G->partial_doubles, coop_partials_doubles());
  alloc(&G->partials, G->partial_doubles);
  if (st == ECMG_OK) {
    for (int i = 0; i < 16; ++i) cudaEventCreate(&G->ev[i]);
    G->ev_init = true;
  }
  if (st == ECMG_OK && cudaStreamSynchronize(G->stream) != cudaSuccess) st = ECMG_ECUDA;
#ifdef ECMG_TESTING
  // test build only (libecmg_test.so): ECMG_TEST_NCCL_SINGLE=1 with nranks == 1 runs the NCCL slab path on one rank
  const bool nccl_single = dist && dist->nranks == 1 && std::getenv("ECMG_TEST_NCCL_SINGLE") != nullptr;
#else
  const bool nccl_single = false;
#endif
  if (nccl_single) slab_force_single() = true;
  if (st == ECMG_OK && dist && (dist->nranks > 1 || nccl_single)) {
    // NCCL ranks: the communicator is created here (collective over all ranks)
    G->nranks = dist->nranks;
    G->rank = dist->rank;
    std::memcpy(G->nccl_id, dist->nccl_id, 128);
    int face_d[6] = {0, 0, 0, 0, 0, 0};
    for (int f = 0; f < 6; ++f) G->prob.face[f] = face_d[f];
    G->prob.id = 1;
    G->geom.clear();
    for (int k = 0; k < G->L; ++k) G->geom.push_back(make_geom(G->dom, G->n0, k, face_d, 0));
    int s2 = ECMG_OK;
    G->slab = slab_driver_create(slab_cfg(G), G->nranks, G->rank, false, G->nccl_id, &s2);
    if (!G->slab) st = s2;
  }
  if (st != ECMG_OK) { cudaGetLastError(); ecmg_destroy_grid(G); return st; }
  *out = G;
  return ECMG_OK;
}

int ecmg_destroy_grid(ecmg_grid* G) {
  if (!G) return ECMG_EINVAL;
  if (G->stream) cudaStreamSynchronize(G->stream); else cudaDeviceSynchronize();
  if (G->slab) slab_driver_destroy(G->slab);
  dfree(G->x); dfree(G->r); dfree(G->p[0]); dfree(G->p[1]);
  for (double* p : G->bl) dfree(p);
  for (double* p : G->betal) dfree(p);
  for (double* p : G->s1d) dfree(p);
  dfree(G->zv); dfree(G->aux[0]); dfree(G->aux[1]); dfree(G->partials); dfree(G->sc);
  for (double* p : G->u) dfree(p);
  dfree(G->ut_tmp);
  for (auto& e : G->setup_ev) if (e) cudaEventDestroy(e);
  if (G->fork_ev) cudaEventDestroy(G->fork_ev);
  if (G->join_ev) cudaEventDestroy(G->join_ev);
  if (G->hi_stream) cudaStreamDestroy(G->hi_stream);
  if (G->lo_stream) cudaStreamDestroy(G->lo_stream);
  if (G->lo2_stream) cudaStreamDestroy(G->lo2_stream);
  dfree(G->seeds);
  if (G->sc_host) cudaFreeHost(G->sc_host);
  if (G->param_host) cudaFreeHost(G->param_host);
  if (G->lvl_param) cudaFreeHost(G->lvl_param);
  if (G->lvl_sc) cudaFreeHost(G->lvl_sc);
  for (auto& e : G->lvl_ev) if (e) cudaEventDestroy(e);
  clear_graphs(G);
  if (G->cap_stream) cudaStreamDestroy(G->cap_stream);
  if (G->ev_init) for (int i = 0; i < 16; ++i) cudaEventDestroy(G->ev[i]);
  cudaGetLastError();
  delete G;
  return ECMG_OK;
}

int ecmg_set_coeffs(ecmg_grid* G, const ecmg_problem* pr) {
  if (!G || !pr) return ECMG_EINVAL;
  Problem pb{};
  int need = 0;
  bool arrays_beta = false;
  if (pr->problem_id == ECMG_PROB_ARRAYS) {
    // caller data per level, alpha per face in params[0..5] (or at the face Gauss points); on
    // z-slabs every rank holds the global-domain arrays and reads its planes by global index
    if (!pr->level_arrays || (pr->n_level_arrays != 4 * G->L && pr->n_level_arrays != 5 * G->L) || pr->n_params != 6 ||
        !pr->params)
      return ECMG_EINVAL;
    for (int f = 0; f < 6; ++f) {
      if (pr->face[f] != ECMG_DIRICHLET && pr->face[f] != ECMG_ROBIN) return ECMG_EINVAL;
      pb.face[f] = pr->face[f];
      pb.alpha[f] = pr->face[f] == ECMG_ROBIN ? pr->params[f] : 0.0;
      if (!(pr->params[f] >= 0.0)) return ECMG_EINVAL;   // alpha >= 0
    }
    arrays_beta = pr->level_arrays[0] != nullptr;
    for (int k = 0; k < G->L; ++k)
      if ((pr->level_arrays[4 * k] != nullptr) != arrays_beta) return ECMG_EINVAL;   // beta on every level or none
  } else if (!problem_faces(pr->problem_id, pb.face, pb.alpha, &need)) return ECMG_EINVAL;
  for (int f = 0; f < 6; ++f)
    if ((int)pr->face[f] != pb.face[f]) return ECMG_EINVAL;
  if (pr->n_params < need || pr->n_params > kMaxParams || (need > 0 && !pr->params)) return ECMG_EINVAL;
  pb.id = pr->problem_id;
  pb.n_params = pr->n_params;
  for (int i = 0; i < pr->n_params; ++i) pb.params[i] = pr->params[i];
  if (need >= 15) {
    for (int l = 0; l < 8; ++l) if (!(pb.params[7 + l] > 0.0)) return ECMG_EINVAL;   // beta > 0
  }
  if (need >= 48) {
    for (int k = 0; k < 4; ++k) if (!(pb.params[15 + 7 * k + 6] > 0.0)) return ECMG_EINVAL;
    if (!(pb.params[46] > 0.0)) return ECMG_EINVAL;
  }
  for (int f = 0; f < 6; ++f) if (pb.alpha[f] < 0.0) return ECMG_EINVAL;   // alpha >= 0
  bool all_dir = true;
  for (int f = 0; f < 6; ++f) all_dir = all_dir && pb.face[f] == FACE_DIRICHLET;
  const int elem_path = pb.id == PROB_ARRAYS ? (arrays_beta || !all_dir) : !(prob_beta_is_one(pb.id) && all_dir);
  if (elem_path && !G->betal.back()) {
    const int size_level = G->size_level;
    int face_none[6] = {FACE_ROBIN, FACE_ROBIN, FACE_ROBIN, FACE_ROBIN, FACE_ROBIN, FACE_ROBIN};
    for (int k = 0; k < G->L; ++k) {
      const LevelGeom gk = make_geom(G->dom, G->n0, std::min(k, size_level), face_none, 1);
      if (dmalloc(&G->betal[k], sizeof(double) * beta_doubles(gk)) != cudaSuccess) { cudaGetLastError(); return ECMG_ENOMEM; }
    }
  }
  if (elem_path && !G->zv) {
    if (dmalloc(&G->zv, sizeof(double) * G->vec_doubles) != cudaSuccess) { cudaGetLastError(); return ECMG_ENOMEM; }
    if (cudaMemsetAsync(G->zv, 0, sizeof(double) * G->vec_doubles, G->stream) != cudaSuccess) return ECMG_ECUDA;
  }
  G->prob = pb;
  G->elem_path = elem_path;
  if (pb.id == PROB_ARRAYS) {   // 5 per level: beta_e, f_q, g_D, g_R, alpha_q (alpha_q null: alpha per face)
    G->arrays.assign(5 * G->L, nullptr);
    for (int k = 0; k < G->L; ++k) {
      for (int j = 0; j < 4; ++j) G->arrays[5 * k + j] = pr->level_arrays[4 * k + j];
      if (pr->n_level_arrays == 5 * G->L) G->arrays[5 * k + 4] = pr->level_arrays[4 * G->L + k];
    }
  } else {
    G->arrays.clear();
  }
  G->geom.clear();
  for (int k = 0; k < G->L; ++k) G->geom.push_back(make_geom(G->dom, G->n0, k, pb.face, elem_path));
  G->has_problem = true;
  invalidate_setup(G);
  G->maps.level = -1;
  clear_graphs(G);
  if (G->slab) slab_driver_configure(G->slab, slab_cfg(G));
  return ECMG_OK;
}

int ecmg_set_option(ecmg_grid* G, int option, int value) {
  if (!G) return ECMG_EINVAL;
  switch (option) {
    case ECMG_OPT_EXP_VARIANT: if (value != 0 && value != 1) return ECMG_EINVAL; G->exp_variant = value; break;
    case ECMG_OPT_PRECOND: if (value != 0 && value != 1) return ECMG_EINVAL; G->precond = value; invalidate_setup(G); clear_graphs(G); break;
    case ECMG_OPT_SETUP_AHEAD: if (value != 0 && value != 1) return ECMG_EINVAL; G->setup_ahead = value; break;
    case ECMG_OPT_BETA_FLY: if (value != 0 && value != 1) return ECMG_EINVAL; G->beta_fly = value; clear_graphs(G); break;
    case ECMG_OPT_EXP_KERNEL: if (value != 0 && value != 1) return ECMG_EINVAL; G->exp_fused = value; break;
    case ECMG_OPT_RHS_SYM: if (value < 0) return ECMG_EINVAL; G->rhs_sym_min = value; invalidate_setup(G); break;
    case ECMG_OPT_SETUP_CTAS: if (value < 0) return ECMG_EINVAL; G->setup_ctas = value; break;
    case ECMG_OPT_ZCHUNK: if (value < 0) return ECMG_EINVAL; G->zchunk = value; clear_graphs(G); break;
    case ECMG_OPT_KERNEL: if (value != 0 && value != 1) return ECMG_EINVAL; G->kernel_variant = value; clear_graphs(G); break;
    case ECMG_OPT_GRAPH: if (value != 0 && value != 1) return ECMG_EINVAL; G->use_graph = value; break;
    case ECMG_OPT_PERSISTENT: if (value < 0) return ECMG_EINVAL; G->persistent_max = value; break;
    case ECMG_OPT_PERS_TMA: if (value < 0) return ECMG_EINVAL; G->pers_tma_max = value; break;
    case ECMG_OPT_UNFUSED: if (value != 0 && value != 1) return ECMG_EINVAL; G->unfused = value; break;
    case ECMG_OPT_P0_INIT: if (value != 0 && value != 1) return ECMG_EINVAL; G->p0_init = value; clear_graphs(G); break;
    case ECMG_OPT_RICH_FUSED: if (value != 0 && value != 1) return ECMG_EINVAL; G->rich_fused = value; clear_graphs(G); break;
    case ECMG_OPT_XDEFER: if (value < 0 || value > 2) return ECMG_EINVAL; G->xdefer = value; clear_graphs(G); break;
    case ECMG_OPT_SHARD_MIN: if (value < 0) return ECMG_EINVAL; G->shard_min = value; break;
    case ECMG_OPT_SLAB_HYBRID: if (value != 0 && value != 1) return ECMG_EINVAL; G->hybrid = value; break;
    case ECMG_OPT_CTA_SOLVE: if (value < 0) return ECMG_EINVAL; G->cta_max = value; break;
    case ECMG_OPT_PDL: if (value != 0 && value != 1) return ECMG_EINVAL; G->pdl = value; clear_graphs(G); break;
    case ECMG_OPT_FUSED_HALO: if (value != 0 && value != 1) return ECMG_EINVAL; G->fused_halo = value; break;
    case ECMG_OPT_VIRTUAL_SLABS: {
      if (value < 0 || value > 16 || G->nranks > 1) return ECMG_EINVAL;
      if (G->slab) { slab_driver_destroy(G->slab); G->slab = nullptr; }
      G->virt_slabs = value > 1 ? value : 0;
      if (G->virt_slabs) {
        int s2 = ECMG_OK;
        G->slab = slab_driver_create(slab_cfg(G), G->virt_slabs, 0, true, nullptr, &s2);
        if (!G->slab) { G->virt_slabs = 0; return s2; }
      }
      return ECMG_OK;
    }
    default: return ECMG_EINVAL;
  }
  if (G->slab) slab_driver_configure(G->slab, slab_cfg(G));
  return ECMG_OK;
}

int ecmg_level_shape(const ecmg_grid* G, int level, int n_cells3[3], long long* nodes, int* z_lo, int* z_hi) {
  if (!G || level < 0 || level >= G->L) return ECMG_EINVAL;
  int n[3];
  for (int d = 0; d < 3; ++d) n[d] = G->n0[d] << level;
  int zlo = 0, zhi = n[2] + 1;
  if (G->slab && G->has_problem) slab_level_range(G->slab, level, &zlo, &zhi);
  if (n_cells3) for (int d = 0; d < 3; ++d) n_cells3[d] = n[d];
  if (nodes) *nodes = (long long)(n[0] + 1) * (n[1] + 1) * (zhi - zlo);
  if (z_lo) *z_lo = zlo;
  if (z_hi) *z_hi = zhi;
  return ECMG_OK;
}

int ecmg_solve_level(ecmg_grid* G, int level, double eps, int max_iter, double* u, ecmg_stats* stats) {
  if (!G || !u || !G->has_problem || level < 0 || level >= G->L) return ECMG_EINVAL;
  if (G->slab) {
    ecmg_stats tmp{};
    const int s = slab_solve_level(G->slab, level, eps, max_iter, u, stats ? stats : &tmp, G->stream);
    slab_last_timing(G->slab, &G->last_jcg_ms, &G->last_jcg_iters, &G->last_free);
    return s;
  }
  const LevelGeom& g = G->geom[level];
  ECMG_CUDA(cudaEventRecord(G->ev[4], G->stream));
  if (!G->setup_ok[level]) { int s = setup_level(G, level); if (s) return s; }
  ECMG_CUDA(cudaEventRecord(G->ev[5], G->stream));
  ECMG_CUDA(launch_gather(g, u, G->x, G->stream));
  const int st = run_jcg(G, level, eps, max_iter, u, stats);   // the true-residual pass fills u's free nodes
  if (st == ECMG_ECUDA || st == ECMG_ENOMEM) return st;
  ECMG_CUDA(launch_dirichlet_fill(g, level_prob(G, level), u, 0.0, 0, G->stream));
  ECMG_CUDA(cudaEventRecord(G->ev[6], G->stream));
  ECMG_CUDA(cudaStreamSynchronize(G->stream));
  if (stats) {
    stats->ms_setup = elapsed(G->ev[4], G->ev[5]);
    stats->ms_solve = elapsed(G->ev[5], G->ev[6]);
    stats->ms_exp = stats->ms_rich = 0.0;
  }
  return st;
}

int ecmg_prolongate_extrapolate(ecmg_grid* G, int level, const double* u2h, const double* u4h, double* w) {
  if (!G || !u2h || !u4h || !w || !G->has_problem || level < 2 || level >= G->L || G->nranks > 1) return ECMG_EINVAL;
  const LevelGeom& g = G->geom[level];
  for (int d = 0; d < 3; ++d) if (g.n[d] % 4) return ECMG_EMISMATCH;
  ECMG_CUDA(launch_exp_finite(g, level_prob(G, level), u2h, u4h, w, G->exp_variant, G->seeds, 0, G->stream, G->exp_fused));
  ECMG_CUDA(cudaStreamSynchronize(G->stream));
  return ECMG_OK;
}

int ecmg_richardson(ecmg_grid* G, int level, const double* uh, const double* u2h, double* ut) {
  if (!G || !uh || !u2h || !ut || !G->has_problem || level < 1 || level >= G->L || G->nranks > 1) return ECMG_EINVAL;
  const LevelGeom& g = G->geom[level];
  for (int d = 0; d < 3; ++d) if (g.n[d] % 2) return ECMG_EMISMATCH;
  ECMG_CUDA(launch_exp_true(g, level_prob(G, level), uh, u2h, ut, G->stream));
  ECMG_CUDA(cudaStreamSynchronize(G->stream));
  return ECMG_OK;
}

int ecmg_apply_operator(ecmg_grid* G, int level, const double* p, double* q) {
  if (!G || !p || !q || !G->has_problem || level < 0 || level >= G->L || G->nranks > 1) return ECMG_EINVAL;
  const LevelGeom& g = G->geom[level];
  if (G->elem_path && !G->setup_ok[level]) { int s = setup_level(G, level); if (s) return s; }
  ECMG_CUDA(launch_gather(g, p, G->p[0], G->stream));
  KArgs a{};
  a.partials = G->partials; a.sc = G->sc; a.pdl = G->pdl; a.zc = auto_zc(G->zchunk, G->elem_path, g); a.beta = G->betal[level];
  a.h0 = G->p[0]; a.o0 = G->r;
  ECMG_CUDA(launch_mode(G, MODE_APPLY, g, a));
  ECMG_CUDA(cudaMemsetAsync(q, 0, sizeof(double) * level_nodes(g), G->stream));
  ECMG_CUDA(launch_scatter(g, G->r, q, G->stream));
  ECMG_CUDA(cudaStreamSynchronize(G->stream));
  return ECMG_OK;
}

int ecmg_level_rhs(ecmg_grid* G, int level, double* bout, double* norm_b) {
  if (!G || !bout || !G->has_problem || level < 0 || level >= G->L || G->nranks > 1) return ECMG_EINVAL;
  const LevelGeom& g = G->geom[level];
  if (!G->setup_ok[level]) { int s = setup_level(G, level); if (s) return s; }
  ECMG_CUDA(cudaMemsetAsync(bout, 0, sizeof(double) * level_nodes(g), G->stream));
  ECMG_CUDA(launch_scatter(g, G->bl[level], bout, G->stream));
  // ||b||^2 is accumulated by the JCG init pass; run it at x = 0
  ECMG_CUDA(launch_zero_vec(g, G->x, G->stream));
  {
    KArgs a{};
    a.partials = G->partials; a.sc = G->sc; a.pdl = G->pdl; a.zc = auto_zc(G->zchunk, G->elem_path, g); a.beta = G->betal[level];
    a.h0 = G->x; a.i0 = G->bl[level]; a.o0 = G->r; a.o1 = G->zv;
    ECMG_CUDA(launch_mode(G, MODE_INIT, g, a));
  }
  ECMG_CUDA(cudaMemcpyAsync(&G->sc_host[0], G->sc, sizeof(JcgScalars), cudaMemcpyDeviceToHost, G->stream));
  ECMG_CUDA(cudaStreamSynchronize(G->stream));
  if (norm_b) *norm_b = std::sqrt(G->sc_host[0].bb);
  return ECMG_OK;
}

int ecmg_last_jcg_timing(const ecmg_grid* G, double* ms, int* iterations, long long* free_unknowns) {
  if (!G) return ECMG_EINVAL;
  if (ms) *ms = G->last_jcg_ms;
  if (iterations) *iterations = G->last_jcg_iters;
  if (free_unknowns) *free_unknowns = G->last_free;
  return ECMG_OK;
}

}  // extern "C"

// Alg. 4 / Alg. 3 cascade with per-level (eps, max_iter) for the ECMG levels k >= 2 (eps <= 0:
// exactly max_iter iterations). Levels 0, 1: DSOLVE.
// k_end < L: only levels [0, k_end) (z-slabs: the replicated levels before the first sharded one); u_k
// of every level stays in G->u and u_fine / ut_fine are not written.
static int run_cascade(ecmg_grid* G, const std::vector<double>& eps_lv, const std::vector<int>& maxit_lv,
                       ecmg_stats* per_level, double* u_fine, double* ut_fine, int k_end = -1) {
  const double eps = eps_lv.back();
  // ECMG_HOSTPROF=1: host-side time of the phases of this call on stderr (enqueue, wait for the GPU, statistics)
  static const bool hostprof = std::getenv("ECMG_HOSTPROF") != nullptr;
  const auto hp0 = std::chrono::steady_clock::now();
  auto hp_us = [&](std::chrono::steady_clock::time_point t) { return std::chrono::duration<double, std::micro>(t - hp0).count(); };
  if (k_end < 0) k_end = G ? G->L : 0;
  const bool partial = G && k_end < G->L;
  if (!G || !G->has_problem || (!u_fine && !partial)) return ECMG_EINVAL;
  if (partial) { u_fine = nullptr; ut_fine = nullptr; }
  for (int k = 2; k < G->L; ++k)
    for (int d = 0; d < 3; ++d) if (G->geom[k].n[d] % 4) return ECMG_EMISMATCH;
  if ((int)G->u.size() != G->L) {
    for (double* p : G->u) dfree(p);
    G->u.assign(G->L, nullptr);
  }
  for (int k = 0; k < k_end; ++k)   // per-level solutions, allocated on first use
    if (!G->u[k] && dmalloc(&G->u[k], sizeof(double) * level_nodes(G->geom[k])) != cudaSuccess) {
      cudaGetLastError();
      return ECMG_ENOMEM;
    }
  const bool ut_dev = ut_fine && is_device_ptr(ut_fine);
  const bool u_dev = u_fine && is_device_ptr(u_fine);
  const long long Nf = level_nodes(G->geom[G->L - 1]);
  if (ut_fine && !ut_dev && !G->ut_tmp) {
    if (dmalloc(&G->ut_tmp, sizeof(double) * Nf) != cudaSuccess) { cudaGetLastError(); return ECMG_ENOMEM; }
  }
  int status = ECMG_OK;
  std::vector<ecmg_stats> stv(G->L);
  std::vector<char> async(G->L, 0);
  for (auto& st : stv) std::memset(&st, 0, sizeof(st));
  auto level_u = [&](int k) { return (k == G->L - 1 && u_dev) ? u_fine : G->u[k]; };
  const int L_run = k_end;
  // Setup ahead (ECMG_OPT_SETUP_AHEAD): the level setups (row a1: beta, lifted b, g_D on the Dirichlet
  // nodes of u_k) depend on no solution, so they are all enqueued up front on a low-priority stream and
  // run under the latency-bound coarse solves, which go to a high-priority stream; level k's solve
  // waits for its setup event only. The caller's stream forks into both and joins at the end.
  const bool ahead = G->setup_ahead != 0;
  cudaStream_t user = G->stream;
  // On every exit (the error returns included) the caller's stream is joined after all the work forked
  // from it -- kernels still writing b_k / beta_k / u_k must not outlive the call on the caller's
  // ordering -- and G->stream is restored.
  struct Join {
    ecmg_grid* G; cudaStream_t user; bool forked = false;
    ~Join() {
      if (forked)
        for (cudaStream_t s : {G->hi_stream, G->lo_stream, G->lo2_stream})
          if (cudaEventRecord(G->join_ev, s) == cudaSuccess) cudaStreamWaitEvent(user, G->join_ev, 0);
      G->stream = user;
    }
  } join{G, user};
  if (ahead) {
    ECMG_CUDA(cudaEventRecord(G->fork_ev, user));
    join.forked = true;
    ECMG_CUDA(cudaStreamWaitEvent(G->hi_stream, G->fork_ev, 0));
    ECMG_CUDA(cudaStreamWaitEvent(G->lo_stream, G->fork_ev, 0));
    ECMG_CUDA(cudaStreamWaitEvent(G->lo2_stream, G->fork_ev, 0));
    // the finest level's setup (most of the work) on its own stream, so that it starts at once; the
    // coarser levels' setups in level order beside it
    G->stream = G->hi_stream;
  }
  // host enqueue order: the finest level's setup first (it starts at once on its own stream), then the
  // coarse setups two levels ahead of the solves, so that the first solve is enqueued after a handful of
  // launches instead of every level's setup
  int next_setup = 0;
  auto enqueue_setup = [&](int k) -> int {
    cudaStream_t s_k = k == L_run - 1 ? G->lo2_stream : G->lo_stream;
    { int s = setup_level_on(G, k, s_k, G->setup_ctas); if (s) return s; }
    ECMG_CUDA(launch_dirichlet_fill(G->geom[k], level_prob(G, k), level_u(k), 0.0, 0, s_k));
    ECMG_CUDA(cudaEventRecord(G->setup_ev[k], s_k));
    return ECMG_OK;
  };
  auto setups_until = [&](int k_last) -> int {   // enqueue the coarse setups up to level k_last
    for (; next_setup <= std::min(k_last, L_run - 2); ++next_setup) {
      const int s = enqueue_setup(next_setup);
      if (s) return s;
    }
    return ECMG_OK;
  };
  if (ahead) {
    { int s = enqueue_setup(L_run - 1); if (s) return s; }
    { int s = setups_until(1); if (s) return s; }
  }
  // the whole cascade is enqueued without host synchronisation when every solve is device driven
  for (int k = 0; k < L_run; ++k) {
    const LevelGeom& g = G->geom[k];
    ecmg_stats& st = stv[k];
    cudaEvent_t* e = &G->lvl_ev[5 * k];
    ECMG_CUDA(cudaEventRecord(e[0], G->stream));
    if (ahead) ECMG_CUDA(cudaStreamWaitEvent(G->stream, G->setup_ev[k], 0));
    else { int s = setup_level(G, k); if (s) return s; }
    ECMG_CUDA(cudaEventRecord(e[1], G->stream));
    if (k < 2) {
      // DSOLVE (Alg. 4 l.1-2): JCG from a zero free guess to 1e-14 (reading §8c A12)
      ECMG_CUDA(launch_zero_vec(g, G->x, G->stream));
    } else {
      // W_h = EXP_finite(u_2h, u_4h) (Alg. 4 l.6), written straight into the free-box work vector
      ECMG_CUDA(launch_exp_finite(g, level_prob(G, k), G->u[k - 1], G->u[k - 2], G->x, G->exp_variant, G->seeds, 1, G->stream, G->exp_fused));
    }
    ECMG_CUDA(cudaEventRecord(e[2], G->stream));
    const double eps_k = k < 2 ? 1e-14 : eps_lv[k];   // JCG from W_h (l.7-9)
    const int maxit_k = k < 2 ? 10000 : maxit_lv[k];
    // u_k: the finest level goes straight into the caller's device buffer (no copy at the end); the
    // true-residual pass of the solve writes its free nodes (fused scatter)
    double* uk = level_u(k);
    // the finest level's true-residual pass also forms u~_h = EXP_true(u_h, u_2h) (l.10) when it is the launched
    // constant-stencil TMA kernel: x is read once for the residual, the scatter of u_h and u~_h
    const bool fuse_rich = k >= 2 && k == G->L - 1 && ut_fine && rich_fused_solve(G, k, eps_k);
    if (fuse_rich) { G->rich_ut = ut_dev ? ut_fine : G->ut_tmp; G->rich_u2h = G->u[k - 1]; }
    struct RichOff { ecmg_grid* G; ~RichOff() { G->rich_ut = nullptr; G->rich_u2h = nullptr; } } rich_off{G};
    int s = enqueue_jcg(G, k, eps_k, maxit_k, uk, &G->lvl_param[k], &G->lvl_sc[k]);
    if (s == ECMG_OK) {
      async[k] = 1;
    } else if (s == ECMG_EINVAL) {
      s = run_jcg(G, k, eps_k, maxit_k, uk, &st);   // host loop (ablation path / fixed counts)
      if (k < 2) s = dsolve_status(s, st);
      if (s != ECMG_OK && status == ECMG_OK) status = s;
    }
    if (s == ECMG_ECUDA || s == ECMG_ENOMEM) return s;
    if (!ahead) ECMG_CUDA(launch_dirichlet_fill(g, level_prob(G, k), uk, 0.0, 0, G->stream));
    ECMG_CUDA(cudaEventRecord(e[3], G->stream));
    if (k >= 2 && k == G->L - 1 && ut_fine) {
      // u~_h = EXP_true(u_h, u_2h) (Alg. 4 l.10) on the finest level
      if (fuse_rich)   // the free nodes are written by the solve's last pass; u~ = g_D on the Dirichlet nodes (A15)
        ECMG_CUDA(launch_dirichlet_fill(g, level_prob(G, k), ut_dev ? ut_fine : G->ut_tmp, 0.0, 0, G->stream));
      else
        ECMG_CUDA(launch_exp_true(g, level_prob(G, k), uk, G->u[k - 1], ut_dev ? ut_fine : G->ut_tmp, G->stream));
    }
    ECMG_CUDA(cudaEventRecord(e[4], G->stream));
    if (ahead) { int s = setups_until(k + 2); if (s) return s; }
  }
  if (u_fine && !u_dev)
    ECMG_CUDA(cudaMemcpyAsync(u_fine, G->u[G->L - 1], sizeof(double) * Nf, cudaMemcpyDeviceToHost, G->stream));
  if (ut_fine && !ut_dev)
    ECMG_CUDA(cudaMemcpyAsync(ut_fine, G->ut_tmp, sizeof(double) * Nf, cudaMemcpyDeviceToHost, G->stream));
  const auto hp1 = std::chrono::steady_clock::now();
  ECMG_CUDA(cudaStreamSynchronize(G->stream));   // (the caller's stream is joined by `join` on return)
  const auto hp2 = std::chrono::steady_clock::now();
  for (int k = 0; k < L_run; ++k) {
    ecmg_stats& st = stv[k];
    if (async[k]) {
      // kernels the level's graph ran: init + true residual + the executed two-iteration loop bodies
      if ((int)G->lvl_graph.size() == G->L && G->lvl_graph[k]) count_launch(2 + 4 * ((G->lvl_sc[k].iter + 1) / 2));
      int s = stats_from(G->lvl_sc[k], k < 2 ? 1e-14 : eps_lv[k], &st);
      if (k < 2) s = dsolve_status(s, st);
      if (s != ECMG_OK && status == ECMG_OK) status = s;
    }
    cudaEvent_t* e = &G->lvl_ev[5 * k];
    st.ms_setup = elapsed(e[0], e[1]);
    st.ms_exp = elapsed(e[1], e[2]);
    st.ms_solve = elapsed(e[2], e[3]);
    st.ms_rich = elapsed(e[3], e[4]);
  }
  if (async[L_run - 1]) {
    G->last_jcg_iters = G->lvl_sc[L_run - 1].iter;
    G->last_free = free_count(G->geom[L_run - 1]);
    G->last_jcg_ms = elapsed(G->lvl_ev[5 * (L_run - 1) + 2], G->lvl_ev[5 * (L_run - 1) + 3]);
  }
  if (per_level) for (int k = 0; k < L_run; ++k) per_level[k] = stv[k];
  if (hostprof)
    std::fprintf(stderr, "ecmg host: enqueued at %.0f us, GPU done at %.0f us, statistics done at %.0f us\n", hp_us(hp1),
                 hp_us(hp2), hp_us(std::chrono::steady_clock::now()));
  (void)eps;
  return status;
}

extern "C" {

int ecmg_run(ecmg_grid* G, double eps, ecmg_stats* per_level, double* u_fine, double* ut_fine) {
  if (!G || !G->has_problem || !u_fine || !(eps > 0.0)) return ECMG_EINVAL;
  if (G->slab) {
    for (int k = 2; k < G->L; ++k)
      for (int d = 0; d < 3; ++d) if (G->geom[k].n[d] % 4) return ECMG_EMISMATCH;
    std::vector<ecmg_stats> stv(G->L);
    // Hybrid cascade: the levels before the first sharded one are replicated (every rank solves them
    // whole, with no communication), so they run through this grid's single-GPU path (one-CTA /
    // persistent / graph solves, setup ahead); their last two solutions seed the first sharded level's
    // EXP_finite in every local slab, and the slab driver takes over from there.
    int kc = slab_first_sharded(G->slab);
    if (G->hybrid && kc >= G->L && G->size_level >= G->L - 1) {   // nothing split: the single-GPU run
      return run_cascade(G, std::vector<double>(G->L, eps), std::vector<int>(G->L, 10000), per_level, u_fine, ut_fine);
    }
    if (G->hybrid && kc >= 2 && kc < G->L && kc <= G->size_level + 1) {
      // the finest (split) level's setup runs ahead on the slab driver's stream meanwhile
      if (G->setup_ahead) { const int r = slab_setup_ahead(G->slab, G->stream); if (r) return r; }
      int s0 = run_cascade(G, std::vector<double>(G->L, eps), std::vector<int>(G->L, 10000), stv.data(), nullptr,
                           nullptr, kc);
      if (s0 == ECMG_ECUDA || s0 == ECMG_ENOMEM) return s0;
      for (int k = kc - 2; k < kc; ++k) {
        const int r = slab_import_u(G->slab, k, G->u[k], G->stream);
        if (r) return r;
      }
      const int s = slab_run(G->slab, eps, stv.data(), u_fine, is_device_ptr(u_fine), ut_fine,
                             ut_fine ? is_device_ptr(ut_fine) : false, G->stream, kc);
      slab_last_timing(G->slab, &G->last_jcg_ms, &G->last_jcg_iters, &G->last_free);
      if (per_level) for (int k = 0; k < G->L; ++k) per_level[k] = stv[k];
      return s != ECMG_OK ? s : s0;
    }
    const int s = slab_run(G->slab, eps, stv.data(), u_fine, is_device_ptr(u_fine), ut_fine,
                           ut_fine ? is_device_ptr(ut_fine) : false, G->stream, 0);
    slab_last_timing(G->slab, &G->last_jcg_ms, &G->last_jcg_iters, &G->last_free);
    if (per_level) for (int k = 0; k < G->L; ++k) per_level[k] = stv[k];
    return s;
  }
  return run_cascade(G, std::vector<double>(G->L, eps), std::vector<int>(G->L, 10000), per_level, u_fine, ut_fine);
}

int ecmg_run_fixed(ecmg_grid* G, int m_L, double ratio, ecmg_stats* per_level, double* u_fine, double* ut_fine) {
  if (!G || !G->has_problem || !u_fine || m_L < 0 || !(ratio > 0.0) || G->slab) return ECMG_EINVAL;
  const int Lc = G->L - 2;
  std::vector<double> e(G->L, 0.0);
  std::vector<int> m(G->L, 0);
  for (int k = 2; k < G->L; ++k)   // Eq. (ee): m_j = ceil(m_L ratio^(L-j)), j = k - 1
    m[k] = (int)std::ceil(m_L * std::pow(ratio, (double)(Lc - (k - 1))) - 1e-12);
  return run_cascade(G, e, m, per_level, u_fine, ut_fine);
}

}  // extern "C"
