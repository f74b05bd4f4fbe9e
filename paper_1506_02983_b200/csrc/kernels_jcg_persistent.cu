// kernels_jcg_persistent.cu -- the whole JCG solve of a small level (Alg. 4 l.7-9, textbook PCG,
// SURVEY.md §8c O7) in ONE cooperative launch, for the constant stencil and the element-beta operator.
//
// The coarse levels of the cascade are latency bound: a few microseconds of L2-resident traffic per
// iteration, while a launched K1/K2 pair costs ~20 us of launch, pipeline fill and tail. Here every CTA
// stays resident and an iteration is two phases separated by grid-wide reductions (measured grid.sync
// cost on B200: 1.2 us, independent of the grid size; tools/gridsync_probe.cu):
//   phase 1: p_new = z + beta_cg p_old at the node and its neighbours (p ping-pongs between two buffers,
//            so neighbours never race), w = A p_new, sigma = p_new . w   | grid sum -> alpha
//   phase 2: x += alpha p_new, r -= alpha w, z = D^-1 r, rho' = r.z, rr  | grid sum -> beta_cg, stop test
// z = D^-1 r is not stored on the constant path (D constant). The element path computes D^-1 once in the
// init phase (kappa_0 sum_e beta_e + Robin diagonal) into a scratch vector.
// Reductions are deterministic and identical in every CTA: each CTA writes its partial, and after the
// barrier every CTA reduces all partials with the same fixed tree (ping-pong partial buffers).
#include <cooperative_groups.h>
#include "ecmg_internal.cuh"
#include "jcg_common.cuh"

namespace cg = cooperative_groups;

namespace ecmg {
namespace {

constexpr int PNTH = 256;

struct PArgs {
  double* x;
  double* r;
  double* z;          // element path: D^-1 r
  double* p[2];       // ping-pong search directions
  double* w;          // A p
  const double* b;
  double* dinv;       // element path: D^-1 per node (init phase)
  const double* beta; // element path: beta_e with zero ring
  double* partials;   // 2 x gridDim.x x 3
  JcgScalars* sc;
};

// fixed-tree block sum of 3 values, result in every thread
__device__ void block_sum3_all(double v[3]) {
  __shared__ double red[3 * (PNTH / 32)];
  __shared__ double res[3];
  const int tid = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  if ((tid & 31) == 0)
    for (int k = 0; k < 3; ++k) red[3 * (tid >> 5) + k] = v[k];
  __syncthreads();
  if (tid < 3) {
    double s = 0.0;
    for (int w = 0; w < PNTH / 32; ++w) s += red[3 * w + tid];
    res[tid] = s;
  }
  __syncthreads();
  v[0] = res[0]; v[1] = res[1]; v[2] = res[2];
  __syncthreads();
}

// grid-wide sum of 3 values: per-CTA partials, barrier, then every CTA reduces all partials in CTA
// order with the same tree (bitwise identical in every CTA)
__device__ void grid_sum3(double v[3], double* partials, int& buf, cg::grid_group& grid) {
  block_sum3_all(v);
  double* pb = partials + (size_t)buf * gridDim.x * 3;
  if (threadIdx.x == 0)
    for (int k = 0; k < 3; ++k) pb[3 * blockIdx.x + k] = v[k];
  grid.sync();
  double s[3] = {0.0, 0.0, 0.0};
  for (unsigned c = threadIdx.x; c < gridDim.x; c += PNTH)
    for (int k = 0; k < 3; ++k) s[k] += __ldcg(pb + 3 * c + k);
  block_sum3_all(s);
  v[0] = s[0]; v[1] = s[1]; v[2] = s[2];
  buf ^= 1;
}

struct Node {
  int fx, fy, fz, off;
};
__device__ __forceinline__ Node node_of(const LevelGeom& g, int i) {
  const int nx = g.nf[0], nxy = g.nf[0] * g.nf[1];
  Node n;
  n.fz = i / nxy;
  const int rem = i - n.fz * nxy;
  n.fy = rem / nx;
  n.fx = rem - n.fy * nx;
  n.off = n.fz * (int)g.S + n.fy * (int)g.P + n.fx;
  return n;
}

// the 27 values of v (or of p_new = zsrc + bcg p_old when FORM) around a node; 0 outside the free box
template <bool FORM>
__device__ __forceinline__ void gather27(const LevelGeom& g, const Node& n, const double* v, const double* pold,
                                         double scale, double bcg, double p27[3][3][3]) {
#pragma unroll
  for (int dz = 0; dz < 3; ++dz)
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int x = n.fx + dx - 1, y = n.fy + dy - 1, z = n.fz + dz - 1;
        double val = 0.0;
        if (x >= 0 && x < g.nf[0] && y >= 0 && y < g.nf[1] && z >= 0 && z < g.nf[2]) {
          const int o = n.off + (dz - 1) * (int)g.S + (dy - 1) * (int)g.P + (dx - 1);
          const double zv = FORM ? scale * __ldcg(v + o) : __ldcg(v + o);
          val = (FORM && bcg != 0.0) ? __fma_rn(bcg, __ldcg(pold + o), zv) : zv;
        }
        p27[dz][dy][dx] = val;
      }
}

__device__ __forceinline__ double apply_const(const ConstStencil& cs, const double p27[3][3][3]) {
  double acc = 0.0;
#pragma unroll
  for (int dz = 0; dz < 3; ++dz) {
    const int az = dz != 1;
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const double c = (dx == 1) ? (dy == 1 ? cs.c0[az] : cs.cy[az]) : (dy == 1 ? cs.cx[az] : cs.cd[az]);
        acc = __fma_rn(c, p27[dz][dy][dx], acc);
      }
  }
  return acc;
}

// which Robin faces (alpha != 0) the node lies on: bit F
__device__ __forceinline__ int robin_mask(const LevelGeom& g, const ElemStencil& es, const Node& n) {
  const int gx = g.flo[0] + n.fx, gy = g.flo[1] + n.fy, gz = g.flo[2] + g.zoff + n.fz;
  int m = 0;
  if (gx == 0 && es.robin[0] != 0.0) m |= 1;
  if (gx == g.n[0] && es.robin[1] != 0.0) m |= 2;
  if (gy == 0 && es.robin[2] != 0.0) m |= 4;
  if (gy == g.n[1] && es.robin[3] != 0.0) m |= 8;
  if (gz == 0 && es.robin[4] != 0.0) m |= 16;
  if (gz == g.n[2] && es.robin[5] != 0.0) m |= 32;
  return m;
}

// betas of the 8 elements around the node (zero ring outside the domain)
__device__ __forceinline__ void gather_beta(const LevelGeom& g, const Node& n, const double* beta, double b8[2][2][2]) {
  const int gx = g.flo[0] + n.fx, gy = g.flo[1] + n.fy, gz = g.flo[2] + g.zoff + n.fz;
#pragma unroll
  for (int ez = 0; ez < 2; ++ez)
#pragma unroll
    for (int ey = 0; ey < 2; ++ey)
#pragma unroll
      for (int ex = 0; ex < 2; ++ex)   // element g - 1 + e at index g + 1 + e (ring of 2)
        b8[ez][ey][ex] = __ldg(beta + (long long)(gz + 1 + ez) * g.BS + (long long)(gy + 1 + ey) * g.BP + (gx + 1 + ex));
}

// (A p)_i = sum_{e ni i} beta_e sum_{j in e} kappa[pat(i,j)] p_j + Robin face mass
__device__ double apply_elem(const ElemStencil& es, int rm, const double b8[2][2][2], const double p27[3][3][3]) {
  double ap = 0.0;
#pragma unroll
  for (int ez = 0; ez < 2; ++ez)
#pragma unroll
    for (int ey = 0; ey < 2; ++ey)
#pragma unroll
      for (int ex = 0; ex < 2; ++ex) {
        double t = 0.0;
#pragma unroll
        for (int bz = 0; bz < 2; ++bz)
#pragma unroll
          for (int by = 0; by < 2; ++by)
#pragma unroll
            for (int bx = 0; bx < 2; ++bx) {
              const int pat = ((ex + bx) != 1 ? 1 : 0) | ((ey + by) != 1 ? 2 : 0) | ((ez + bz) != 1 ? 4 : 0);
              t = __fma_rn(es.kappa[pat], p27[ez + bz][ey + by][ex + bx], t);
            }
        ap = __fma_rn(b8[ez][ey][ex], t, ap);
      }
  if (rm) {   // Robin face mass alpha h1 h2 (m (x) m) of the face elements around the node
    for (int F = 0; F < 6; ++F) {
      if (!(rm & (1 << F))) continue;
      const int d = F >> 1;
      for (int ez = 0; ez < 2; ++ez)
        for (int ey = 0; ey < 2; ++ey)
          for (int ex = 0; ex < 2; ++ex) {
            if (b8[ez][ey][ex] == 0.0) continue;   // element outside the domain
            const int e3[3] = {ex, ey, ez};
            for (int bb = 0; bb < 8; ++bb) {
              const int b3[3] = {bb & 1, (bb >> 1) & 1, (bb >> 2) & 1};
              if (b3[d] != 1 - e3[d]) continue;   // node of the element face on F
              int nd = 0;
              for (int t = 0; t < 3; ++t)
                if (t != d && b3[t] != 1 - e3[t]) ++nd;
              const double m2 = nd == 0 ? (1.0 / 9.0) : (nd == 1 ? (1.0 / 18.0) : (1.0 / 36.0));
              ap += es.robin[F] * m2 * p27[ez + b3[2]][ey + b3[1]][ex + b3[0]];
            }
          }
    }
  }
  return ap;
}

__device__ double diag_elem(const ElemStencil& es, int rm, const double b8[2][2][2]) {
  double sb = 0.0, rob = 0.0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const double be = b8[e >> 2][(e >> 1) & 1][e & 1];
    sb += be;
    if (rm && be != 0.0)
      for (int F = 0; F < 6; ++F)
        if (rm & (1 << F)) rob += es.robin[F] * (1.0 / 9.0);
  }
  return es.kappa[0] * sb + rob;
}

template <bool ELEM>
__global__ void __launch_bounds__(PNTH) k_jcg_persistent(const LevelGeom g, const ConstStencil cs, const ElemStencil es,
                                                         const PArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int n = g.nf[0] * g.nf[1] * g.nf[2];   // small levels only: 32-bit index math
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  const double cdinv = cs.dinv;
  JcgScalars* sc = a.sc;
  const double eps = sc->eps_in;
  const int max_iter = sc->max_iter_in;
  int buf = 0;
  // init: D^-1 (element path), r = b - A x, z = D^-1 r, rho = r.z, rr, ||b||^2
  double v[3] = {0.0, 0.0, 0.0};
  for (int i = t0; i < n; i += stride) {
    const Node nd = node_of(g, i);
    double p27[3][3][3];
    gather27<false>(g, nd, a.x, nullptr, 1.0, 0.0, p27);
    double ax, di;
    if (ELEM) {
      double b8[2][2][2];
      gather_beta(g, nd, a.beta, b8);
      const int rm = robin_mask(g, es, nd);
      ax = apply_elem(es, rm, b8, p27);
      const double d = diag_elem(es, rm, b8);
      di = es.precond ? (d > 0.0 ? 1.0 / d : 0.0) : 1.0;
      a.dinv[nd.off] = di;
    } else {
      ax = apply_const(cs, p27);
      di = cdinv;
    }
    const double bi = a.b[nd.off];
    const double rn = bi - ax;
    const double zz = di * rn;
    a.r[nd.off] = rn;
    if (ELEM) a.z[nd.off] = zz;
    v[0] = __fma_rn(rn, zz, v[0]);
    v[1] = __fma_rn(rn, rn, v[1]);
    v[2] = __fma_rn(bi, bi, v[2]);
  }
  grid_sum3(v, a.partials, buf, grid);
  double rho = v[0], rr = v[1];
  const double bb = v[2];
  const double nb = sqrt(bb), nbe = nb > 0.0 ? nb : 1.0;
  const double thresh = eps > 0.0 ? eps * nbe : -1.0;
  int status = ST_OK, iter = 0;
  double beta = 0.0;
  bool done = (max_iter <= 0) || (thresh > 0.0 && !(sqrt(rr) > thresh));
  if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  int cur = 0;   // a.p[cur] holds p_old
  while (!done) {
    // phase 1: p_new = z + beta p_old around every node, w = A p_new, sigma = p_new . w
    const double* zsrc = ELEM ? a.z : a.r;
    const double zscale = ELEM ? 1.0 : cdinv;
    const double bcg = iter == 0 ? 0.0 : beta;
    double* pnew = a.p[cur ^ 1];
    const double* pold = a.p[cur];
    v[0] = v[1] = v[2] = 0.0;
    for (int i = t0; i < n; i += stride) {
      const Node nd = node_of(g, i);
      double p27[3][3][3];
      gather27<true>(g, nd, zsrc, pold, zscale, bcg, p27);
      double wi;
      if (ELEM) {
        double b8[2][2][2];
        gather_beta(g, nd, a.beta, b8);
        wi = apply_elem(es, robin_mask(g, es, nd), b8, p27);
      } else {
        wi = apply_const(cs, p27);
      }
      const double pc = p27[1][1][1];
      pnew[nd.off] = pc;
      a.w[nd.off] = wi;
      v[0] = __fma_rn(pc, wi, v[0]);
    }
    grid_sum3(v, a.partials, buf, grid);
    const double sigma = v[0];
    if (!(sigma > 0.0)) { status = ST_EBREAKDOWN; break; }
    const double alpha = rho / sigma;
    // phase 2: x += alpha p, r -= alpha w, z = D^-1 r, rho' = r.z, rr = r.r
    v[0] = v[1] = v[2] = 0.0;
    for (int i = t0; i < n; i += stride) {
      const Node nd = node_of(g, i);
      const int o = nd.off;
      a.x[o] = __fma_rn(alpha, pnew[o], a.x[o]);
      const double rn = __fma_rn(-alpha, a.w[o], a.r[o]);
      a.r[o] = rn;
      const double zz = (ELEM ? a.dinv[o] : cdinv) * rn;
      if (ELEM) a.z[o] = zz;
      v[0] = __fma_rn(rn, zz, v[0]);
      v[1] = __fma_rn(rn, rn, v[1]);
    }
    grid_sum3(v, a.partials, buf, grid);
    beta = v[0] / rho;
    rho = v[0];
    rr = v[1];
    cur ^= 1;
    ++iter;
    done = (iter >= max_iter) || (thresh > 0.0 && !(sqrt(rr) > thresh));
    if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  }
  // true residual ||b - A x||
  v[0] = v[1] = v[2] = 0.0;
  for (int i = t0; i < n; i += stride) {
    const Node nd = node_of(g, i);
    double p27[3][3][3];
    gather27<false>(g, nd, a.x, nullptr, 1.0, 0.0, p27);
    double ax;
    if (ELEM) {
      double b8[2][2][2];
      gather_beta(g, nd, a.beta, b8);
      ax = apply_elem(es, robin_mask(g, es, nd), b8, p27);
    } else {
      ax = apply_const(cs, p27);
    }
    const double rn = a.b[nd.off] - ax;
    v[1] = __fma_rn(rn, rn, v[1]);
  }
  grid_sum3(v, a.partials, buf, grid);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->rho = rho; sc->rr = rr; sc->bb = bb; sc->rr_true = v[1]; sc->beta = beta;
    sc->iter = iter; sc->max_iter = max_iter; sc->thresh = thresh; sc->status = status; sc->done = 1;
  }
}

template <bool ELEM>
int persistent_grid(int want) {
  static int slots = 0;
  if (!slots) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jcg_persistent<ELEM>, PNTH, 0);
    slots = sms * std::max(1, per_sm);
  }
  return std::max(1, std::min(want, slots));
}

}  // namespace

// One cooperative launch: the whole solve. Element path (es != nullptr): z, dinv and w are scratch
// vectors of the level's size; beta as in KArgs. Constant path: z, dinv, beta unused.
cudaError_t launch_jcg_persistent(const LevelGeom& g, const ConstStencil& cs, const ElemStencil* es, double* x, double* r,
                                  double* z, double* p0, double* p1, double* w, double* dinv, const double* beta,
                                  const double* b, double* partials, JcgScalars* sc, cudaStream_t st) {
  const long long n = (long long)g.nf[0] * g.nf[1] * g.nf[2];
  const int want = (int)std::min<long long>((n + PNTH - 1) / PNTH, 1 << 20);
  PArgs a{x, r, z, {p0, p1}, w, b, dinv, beta, partials, sc};
  const ElemStencil e = es ? *es : ElemStencil{};
  void* args[] = {(void*)&g, (void*)&cs, (void*)&e, (void*)&a};
  count_launch();
  if (es)
    return cudaLaunchCooperativeKernel((const void*)k_jcg_persistent<true>, dim3(persistent_grid<true>(want)), dim3(PNTH),
                                       args, 0, st);
  return cudaLaunchCooperativeKernel((const void*)k_jcg_persistent<false>, dim3(persistent_grid<false>(want)),
                                     dim3(PNTH), args, 0, st);
}

}  // namespace ecmg
