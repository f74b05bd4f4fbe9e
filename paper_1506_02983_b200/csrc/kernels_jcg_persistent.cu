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
#include <algorithm>
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
__device__ __forceinline__ void block_sum3_all(double v[3]) {
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
__device__ __forceinline__ void grid_sum3(double v[3], double* partials, int& buf, cg::grid_group& grid) {
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

// value of p27 at offset (o1, o2) along the two tangential axes of a face normal to axis D
template <int D>
__device__ __forceinline__ double face_at(const double p27[3][3][3], int o1, int o2) {
  if (D == 0) return p27[1 + o2][1 + o1][1];   // tangential axes y, z
  if (D == 1) return p27[1 + o2][1][1 + o1];   // x, z
  return p27[1][1 + o2][1 + o1];               // x, y
}

// Robin face mass alpha h1 h2 (m (x) m) on the face normal to axis D through the node: the face
// elements around it in the two tangential axes, present where the index range of the box domain has
// them (cm / cp: element on the minus / plus side exists). Adds to (A p) and to the diagonal.
template <int D>
__device__ __forceinline__ void robin_face(double rf, const double p27[3][3][3], const double cm[3], const double cp[3],
                                           double& ap, double& dg) {
  constexpr int t1 = D == 0 ? 1 : 0, t2 = D == 2 ? 1 : 2;
  double acc = 0.0, cnt = 0.0;
#pragma unroll
  for (int s2 = -1; s2 <= 1; s2 += 2)
#pragma unroll
    for (int s1 = -1; s1 <= 1; s1 += 2) {
      const double chi = (s1 < 0 ? cm[t1] : cp[t1]) * (s2 < 0 ? cm[t2] : cp[t2]);
      acc += chi * ((1.0 / 9.0) * face_at<D>(p27, 0, 0) + (1.0 / 18.0) * face_at<D>(p27, s1, 0) +
                    (1.0 / 18.0) * face_at<D>(p27, 0, s2) + (1.0 / 36.0) * face_at<D>(p27, s1, s2));
      cnt += chi;
    }
  ap += rf * acc;
  dg += rf * cnt * (1.0 / 9.0);
}

// (A p)_i = sum_{e ni i} beta_e sum_{j in e} kappa[pat(i,j)] p_j + Robin face mass; the
// Jacobi diagonal kappa_0 sum_e beta_e + Robin diagonal in *diag if asked
__device__ __forceinline__ double apply_elem(const LevelGeom& g, const ElemStencil& es, const Node& nd,
                                             const double b8[2][2][2], const double p27[3][3][3], double* diag) {
  double ap = 0.0, sb = 0.0;
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
        sb += b8[ez][ey][ex];
      }
  double dg = es.kappa[0] * sb;
  const int gx = g.flo[0] + nd.fx, gy = g.flo[1] + nd.fy, gz = g.flo[2] + g.zoff + nd.fz;
  const double rfx = (gx == 0 ? es.robin[0] : 0.0) + (gx == g.n[0] ? es.robin[1] : 0.0);
  const double rfy = (gy == 0 ? es.robin[2] : 0.0) + (gy == g.n[1] ? es.robin[3] : 0.0);
  const double rfz = (gz == 0 ? es.robin[4] : 0.0) + (gz == g.n[2] ? es.robin[5] : 0.0);
  if ((rfx != 0.0 || rfy != 0.0 || rfz != 0.0) && es.aq) {
    // alpha at the face Gauss points (ARRAYS alpha_q): every face element of every Robin face through the node
    const int gc[3] = {gx, gy, gz};
#pragma unroll
    for (int F = 0; F < 6; ++F) {
      const int D = F >> 1;
      if (es.robin[F] == 0.0 || gc[D] != ((F & 1) ? g.n[D] : 0)) continue;
      const int t1 = D == 0 ? 1 : 0, t2 = D == 2 ? 1 : 2;
      for (int s2 = 0; s2 < 2; ++s2)
        for (int s1 = 0; s1 < 2; ++s1) {
          const int e1 = gc[t1] - 1 + s1, e2 = gc[t2] - 1 + s2;
          if (e1 < 0 || e1 >= g.n[t1] || e2 < 0 || e2 >= g.n[t2]) continue;
          const double* a4 = robin_aq(es.aq, g.n, F, e1, e2);
          double v[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {   // element corner (e1 + (c & 1), e2 + (c >> 1)) at offsets from the node
            const int o1 = s1 - 1 + (c & 1), o2 = s2 - 1 + (c >> 1);
            v[c] = D == 0 ? p27[1 + o2][1 + o1][1] : (D == 1 ? p27[1 + o2][1][1 + o1] : p27[1][1 + o2][1 + o1]);
          }
          robin_elem_row(a4, 1 - s1, 1 - s2, v[0], v[1], v[2], v[3], es.robin[F], ap, dg);
        }
    }
  } else if (rfx != 0.0 || rfy != 0.0 || rfz != 0.0) {
    const double cm[3] = {gx >= 1 ? 1.0 : 0.0, gy >= 1 ? 1.0 : 0.0, gz >= 1 ? 1.0 : 0.0};
    const double cp[3] = {gx < g.n[0] ? 1.0 : 0.0, gy < g.n[1] ? 1.0 : 0.0, gz < g.n[2] ? 1.0 : 0.0};
    if (rfx != 0.0) robin_face<0>(rfx, p27, cm, cp, ap, dg);
    if (rfy != 0.0) robin_face<1>(rfy, p27, cm, cp, ap, dg);
    if (rfz != 0.0) robin_face<2>(rfz, p27, cm, cp, ap, dg);
  }
  if (diag) *diag = dg;
  return ap;
}

// Bricks of 8 x 8 x 4 nodes, one node per thread; the brick and its one-node halo (10 x 10 x 6) are staged
// in shared memory with coalesced L2 loads whenever neighbours' values are needed (L1 is not coherent
// across SMs, so data written by other CTAs in the previous phase is read with ld.cg). A node is always
// handled by the same thread, so its own x, r, z, D^-1, p_new, w need no such care.
constexpr int BX = 8, BY = 8, BZ = 4;
constexpr int SX = BX + 2, SY = BY + 2, SZ = BZ + 2, SN = SX * SY * SZ;

struct Brick {
  int X0, Y0, Z0;
};
__device__ __forceinline__ Brick brick_of(const LevelGeom& g, int k) {
  const int nbx = (g.nf[0] + BX - 1) / BX, nby = (g.nf[1] + BY - 1) / BY;
  Brick br;
  br.X0 = (k % nbx) * BX;
  br.Y0 = ((k / nbx) % nby) * BY;
  br.Z0 = (k / (nbx * nby)) * BZ;
  return br;
}

// s[...] = FORM ? zscale * zsrc + bcg * pold : zsrc over the brick and its halo (0 outside the free box)
template <bool FORM>
__device__ __forceinline__ void stage(const LevelGeom& g, const Brick& br, const double* zsrc, const double* pold,
                                      double zscale, double bcg, double* s) {
  for (int t = threadIdx.x; t < SN; t += PNTH) {
    const int hx = t % SX, hy = (t / SX) % SY, hz = t / (SX * SY);
    const int x = br.X0 - 1 + hx, y = br.Y0 - 1 + hy, z = br.Z0 - 1 + hz;
    double v = 0.0;
    if (x >= 0 && x < g.nf[0] && y >= 0 && y < g.nf[1] && z >= 0 && z < g.nf[2]) {
      const int o = z * (int)g.S + y * (int)g.P + x;
      v = __ldcg(zsrc + o);
      if (FORM) {
        v *= zscale;
        if (bcg != 0.0) v = __fma_rn(bcg, __ldcg(pold + o), v);
      }
    }
    s[t] = v;
  }
}

// The halo windows of all nb bricks of a CTA (origins in sb[3 i ..]), in batches of 8 loads per thread that
// are all in flight together (one L2 latency per batch instead of one per value); values as in stage().
template <bool FORM, int NBMAX>
__device__ __forceinline__ void stage_all(const LevelGeom& g, const int* sb, int nb, const double* zsrc, const double* pold,
                                          double zscale, double bcg, double* s) {
  const int tot = nb * SN;
  for (int base = 0; base < tot; base += 8 * PNTH) {
    double v[8], w[8];
    int o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int t = base + q * PNTH + threadIdx.x;
      o[q] = -1;
      if (t < tot) {
        const int i = t / SN, h = t - i * SN;
        const int hx = h % SX, hy = (h / SX) % SY, hz = h / (SX * SY);
        const int x = sb[3 * i] - 1 + hx, y = sb[3 * i + 1] - 1 + hy, z = sb[3 * i + 2] - 1 + hz;
        if (x >= 0 && x < g.nf[0] && y >= 0 && y < g.nf[1] && z >= 0 && z < g.nf[2]) o[q] = z * (int)g.S + y * (int)g.P + x;
      }
      v[q] = o[q] >= 0 ? __ldcg(zsrc + o[q]) : 0.0;
      w[q] = (FORM && bcg != 0.0 && o[q] >= 0) ? __ldcg(pold + o[q]) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int t = base + q * PNTH + threadIdx.x;
      if (t >= tot) break;
      double val = v[q];
      if (FORM) {
        val *= zscale;
        if (bcg != 0.0) val = __fma_rn(bcg, w[q], val);
      }
      s[t] = val;
    }
  }
}

__device__ __forceinline__ void window27(const double* s, int lx, int ly, int lz, double p27[3][3][3]) {
#pragma unroll
  for (int dz = 0; dz < 3; ++dz)
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) p27[dz][dy][dx] = s[((lz + dz) * SY + (ly + dy)) * SX + lx + dx];
}

template <bool ELEM>
__device__ __forceinline__ double apply_node(const LevelGeom& g, const ConstStencil& cs, const ElemStencil& es,
                                             const double* beta, const Node& nd, const double p27[3][3][3], double* diag) {
  if (ELEM) {
    double b8[2][2][2];
    gather_beta(g, nd, beta, b8);
    return apply_elem(g, es, nd, b8, p27, diag);
  }
  return apply_const(cs, p27);
}

// Each CTA owns at most MB bricks (k = blockIdx.x + i gridDim.x) for the whole solve, and each thread
// keeps its nodes' x, r, D^-1, p_new and A p_new in registers: phase 2 needs no global loads, A p is never
// stored, x is stored once at the end. Only the halo exchange goes through L2: z (element path) or r
// (constant path, z = D^-1 r with D constant) and p_new. The halo windows of all of a CTA's bricks are
// staged in one round of loads (one L2 latency per phase, not one per brick).
// Two launch forms:
//  * cooperative (CL = false): up to MAXB = 4 bricks per CTA, grid reductions through L2 partials and
//    grid.sync (measured 1.2 us per barrier);
//  * one thread-block cluster (CL = true, <= 16 CTAs of one brick each): the levels of at most 16 bricks
//    (16^3 cells). The reductions go through distributed shared memory -- every CTA publishes its block sum
//    in its own shared memory, one cluster barrier (release / acquire: it also orders the global halo
//    stores), then every CTA reads the C sums in rank order, so every CTA holds the bitwise same total --
//    and the solve occupies at most 16 SMs, leaving the rest of the GPU to the setups that run ahead beside
//    the coarse solves. Measured on C4 (tools/tts_ab.py): 16^3 0.225 -> 0.179 ms; at 32^3 (128 bricks: 8
//    per CTA of a 16-CTA cluster) 0.364 -> 0.549 ms, so 32^3 stays on the cooperative form.
constexpr int MAXB = 4, MAXBC = 1, MAXC = 16;

// cluster-wide sum of 3 values through distributed shared memory, result in every thread of every CTA
__device__ __forceinline__ void cluster_sum3(double v[3], double (*csum)[3], int& buf) {
  block_sum3_all(v);
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0)
    for (int k = 0; k < 3; ++k) csum[buf][k] = v[k];
  cl.sync();
  __shared__ double res[3];
  const unsigned C = cl.num_blocks();
  if (threadIdx.x < 3) {
    double part[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c)   // independent remote loads first, then the fixed-order sum
      part[c] = c < (int)C ? *cl.map_shared_rank(&csum[buf][threadIdx.x], (unsigned)c) : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < (int)C) sum += part[c];
    res[threadIdx.x] = sum;
  }
  __syncthreads();
  v[0] = res[0]; v[1] = res[1]; v[2] = res[2];
  __syncthreads();
  buf ^= 1;   // the other buffer next time: a slow CTA may still be reading this one
}

template <bool ELEM, bool CL>
__global__ void __launch_bounds__(PNTH, CL ? 1 : 2) k_jcg_persistent(const LevelGeom g, const ConstStencil cs,
                                                                    const ElemStencil es, const PArgs a) {
  constexpr int MB = CL ? MAXBC : MAXB;
  extern __shared__ double sp_all[];       // MB halo windows of SN values
  __shared__ double csum[2][3];            // cluster form: this CTA's block sums (ping-pong)
  const int nbricks = ((g.nf[0] + BX - 1) / BX) * ((g.nf[1] + BY - 1) / BY) * ((g.nf[2] + BZ - 1) / BZ);
  const int lx = threadIdx.x % BX, ly = (threadIdx.x / BX) % BY, lz = threadIdx.x / (BX * BY);
  const double cdinv = cs.dinv;
  JcgScalars* sc = a.sc;
  const double eps = sc->in.eps;
  const int max_iter = sc->in.max_iter;
  double* const u_out = sc->in.u_out;
  double* const zsrc = ELEM ? a.z : a.r;   // what neighbours stage: p_new = zscale * zsrc + beta p_old
  const double zscale = ELEM ? 1.0 : cdinv;
  int buf = 0;
  auto allsum = [&](double v[3]) {
    if constexpr (CL) {
      cluster_sum3(v, csum, buf);
    } else {
      cg::grid_group grid = cg::this_grid();
      grid_sum3(v, a.partials, buf, grid);
    }
  };
  auto allsync = [&]() {
    if constexpr (CL) cg::this_cluster().sync();
    else cg::this_grid().sync();
  };

  bool act[MB], own[MB];
  Brick br[MB];
  Node nd[MB];
  __shared__ int sb[3 * MB];   // brick origins for the batched staging
  int nact = 0;                // active bricks of this CTA: 0 .. nact-1
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int k = blockIdx.x + i * gridDim.x;
    act[i] = k < nbricks;   // uniform over the CTA
    nact += act[i] ? 1 : 0;
    br[i] = brick_of(g, act[i] ? k : 0);
    if (threadIdx.x == 0) { sb[3 * i] = br[i].X0; sb[3 * i + 1] = br[i].Y0; sb[3 * i + 2] = br[i].Z0; }
    nd[i].fx = br[i].X0 + lx; nd[i].fy = br[i].Y0 + ly; nd[i].fz = br[i].Z0 + lz;
    nd[i].off = nd[i].fz * (int)g.S + nd[i].fy * (int)g.P + nd[i].fx;
    own[i] = act[i] && nd[i].fx < g.nf[0] && nd[i].fy < g.nf[1] && nd[i].fz < g.nf[2];
  }
  double xr[MB], rr_[MB], di[MB], pc[MB], wv[MB];
  // init: D^-1 (element path), r = b - A x, z = D^-1 r, rho = r.z, rr, ||b||^2
  double v[3] = {0.0, 0.0, 0.0};
  __syncthreads();   // sb
  stage_all<false, MB>(g, sb, nact, a.x, nullptr, 1.0, 0.0, sp_all);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    xr[i] = rr_[i] = pc[i] = wv[i] = 0.0;
    di[i] = cdinv;
    if (!own[i]) continue;
    double p27[3][3][3];
    window27(sp_all + i * SN, lx, ly, lz, p27);
    double d = 0.0;
    const double ax = apply_node<ELEM>(g, cs, es, a.beta, nd[i], p27, &d);
    if (ELEM) di[i] = es.precond ? (d > 0.0 ? 1.0 / d : 0.0) : 1.0;
    xr[i] = p27[1][1][1];
    const double bi = a.b[nd[i].off];
    const double rn = bi - ax;
    const double zz = di[i] * rn;
    rr_[i] = rn;
    zsrc[nd[i].off] = ELEM ? zz : rn;
    v[0] = __fma_rn(rn, zz, v[0]);
    v[1] = __fma_rn(rn, rn, v[1]);
    v[2] = __fma_rn(bi, bi, v[2]);
  }
  allsum(v);
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
    // phase 1: p_new = z + beta p_old on the bricks and their halos, w = A p_new, sigma = p_new . w
    const double bcg = iter == 0 ? 0.0 : beta;
    double* pnew = a.p[cur ^ 1];
    const double* pold = a.p[cur];
    v[0] = v[1] = v[2] = 0.0;
    __syncthreads();   // the previous phase's windows consumed
    stage_all<true, MB>(g, sb, nact, zsrc, pold, zscale, bcg, sp_all);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      if (!own[i]) continue;
      double p27[3][3][3];
      window27(sp_all + i * SN, lx, ly, lz, p27);
      wv[i] = apply_node<ELEM>(g, cs, es, a.beta, nd[i], p27, nullptr);
      pc[i] = p27[1][1][1];
      pnew[nd[i].off] = pc[i];
      v[0] = __fma_rn(pc[i], wv[i], v[0]);
    }
    allsum(v);
    const double sigma = v[0];
    if (!(sigma > 0.0)) { status = ST_EBREAKDOWN; break; }
    const double alpha = rho / sigma;
    // phase 2 (own nodes, registers): x += alpha p, r -= alpha w, z = D^-1 r, rho' = r.z, rr = r.r
    v[0] = v[1] = v[2] = 0.0;
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      if (!own[i]) continue;
      xr[i] = __fma_rn(alpha, pc[i], xr[i]);
      const double rn = __fma_rn(-alpha, wv[i], rr_[i]);
      rr_[i] = rn;
      const double zz = di[i] * rn;
      zsrc[nd[i].off] = ELEM ? zz : rn;
      v[0] = __fma_rn(rn, zz, v[0]);
      v[1] = __fma_rn(rn, rn, v[1]);
    }
    allsum(v);
    beta = v[0] / rho;
    rho = v[0];
    rr = v[1];
    cur ^= 1;
    ++iter;
    done = (iter >= max_iter) || (thresh > 0.0 && !(sqrt(rr) > thresh));
    if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  }
  // x (and r, for the caller's inspection) back to memory, then the true residual ||b - A x||
#pragma unroll
  for (int i = 0; i < MB; ++i)
    if (own[i]) { a.x[nd[i].off] = xr[i]; a.r[nd[i].off] = rr_[i]; }
  allsync();
  v[0] = v[1] = v[2] = 0.0;
  stage_all<false, MB>(g, sb, nact, a.x, nullptr, 1.0, 0.0, sp_all);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    if (!own[i]) continue;
    double p27[3][3][3];
    window27(sp_all + i * SN, lx, ly, lz, p27);
    const double rn = a.b[nd[i].off] - apply_node<ELEM>(g, cs, es, a.beta, nd[i], p27, nullptr);
    v[1] = __fma_rn(rn, rn, v[1]);
    if (u_out) u_out[full_index(g, nd[i].fx, nd[i].fy, nd[i].fz)] = xr[i];   // fused scatter of u_h
  }
  allsum(v);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->rho = rho; sc->rr = rr; sc->bb = bb; sc->rr_true = v[1]; sc->beta = beta;
    sc->iter = iter; sc->max_iter = max_iter; sc->thresh = thresh; sc->status = status; sc->done = 1;
  }
  if constexpr (CL) cg::this_cluster().sync();   // no CTA exits while another may still read its csum
}

// ---- the smallest levels: the whole solve in ONE CTA, every vector in shared memory -------------------
// Levels of at most CNODES free unknowns (4^3 .. 16^3) do not need a grid: one CTA of CNTH threads keeps
// p (with a zero halo ring), x, r, w = A p and (element path) D^-1 in shared memory, so an iteration is
// two block reductions and a few barriers with no L2 round trip and no grid barrier. Each thread owns
// the nodes t, t + CNTH, ... (x fastest) for the whole solve; the arithmetic per node is the persistent
// kernel's (apply_const / apply_elem on a 27-value window).
constexpr int CNTH = 512, CMAXN = 8, CNODES = CNTH * CMAXN;

__device__ __forceinline__ void cta_sum3(double v[3], double* red) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  if ((tid & 31) == 0)
    for (int k = 0; k < 3; ++k) red[3 * (tid >> 5) + k] = v[k];
  __syncthreads();
  if (tid < 3) {
    double sum = 0.0;
    for (int w = 0; w < CNTH / 32; ++w) sum += red[3 * w + tid];
    red[3 * (CNTH / 32) + tid] = sum;
  }
  __syncthreads();
  v[0] = red[3 * (CNTH / 32)]; v[1] = red[3 * (CNTH / 32) + 1]; v[2] = red[3 * (CNTH / 32) + 2];
  __syncthreads();   // red reusable
}

template <bool ELEM>
__global__ void __launch_bounds__(CNTH, 1) k_jcg_cta(const LevelGeom g, const ConstStencil cs, const ElemStencil es,
                                                   const PArgs a) {
  extern __shared__ double csm[];
  const int nfx = g.nf[0], nfy = g.nf[1], nfz = g.nf[2];
  const int n = nfx * nfy * nfz;
  const int hx = nfx + 2, hxy = hx * (nfy + 2);
  const int nh = hxy * (nfz + 2);
  double* P = csm;              // p with a zero halo ring, index ((z+1) hxy + (y+1) hx + x+1)
  double* X = P + nh;
  double* R = X + n;
  double* W = R + n;
  double* DI = W + n;           // element path only
  double* red = DI + (ELEM ? n : 0);
  const int tid = threadIdx.x;
  JcgScalars* sc = a.sc;
  const double eps = sc->in.eps;
  const int max_iter = sc->in.max_iter;
  double* const u_out = sc->in.u_out;
  const double cdinv = cs.dinv;
  Node nd[CMAXN];
  int hp[CMAXN];
  bool own[CMAXN];
#pragma unroll
  for (int q = 0; q < CMAXN; ++q) {
    const int i = tid + q * CNTH;
    own[q] = i < n;
    const int ii = own[q] ? i : 0;
    nd[q].fx = ii % nfx; nd[q].fy = (ii / nfx) % nfy; nd[q].fz = ii / (nfx * nfy);
    nd[q].off = nd[q].fz * (int)g.S + nd[q].fy * (int)g.P + nd[q].fx;
    hp[q] = (nd[q].fz + 1) * hxy + (nd[q].fy + 1) * hx + nd[q].fx + 1;
  }
  auto win = [&](int h, double p27[3][3][3]) {
#pragma unroll
    for (int dz = 0; dz < 3; ++dz)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) p27[dz][dy][dx] = P[h + (dz - 1) * hxy + (dy - 1) * hx + (dx - 1)];
  };
  auto applyq = [&](int q, double* diag) {
    double p27[3][3][3];
    win(hp[q], p27);
    return apply_node<ELEM>(g, cs, es, a.beta, nd[q], p27, diag);
  };
  // init: P = x (zero halo), r = b - A x, D^-1, z = D^-1 r, rho = r.z, rr, ||b||^2
  for (int t = tid; t < nh; t += CNTH) P[t] = 0.0;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < CMAXN; ++q)
    if (own[q]) P[hp[q]] = a.x[nd[q].off];
  __syncthreads();
  double v[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int q = 0; q < CMAXN; ++q) {
    if (!own[q]) continue;
    const int i = tid + q * CNTH;
    double d = 0.0;
    const double ax = applyq(q, &d);
    const double di = ELEM ? (es.precond ? (d > 0.0 ? 1.0 / d : 0.0) : 1.0) : cdinv;
    if (ELEM) DI[i] = di;
    const double bi = a.b[nd[q].off];
    const double rn = bi - ax;
    X[i] = P[hp[q]];
    R[i] = rn;
    const double zz = di * rn;
    v[0] = __fma_rn(rn, zz, v[0]);
    v[1] = __fma_rn(rn, rn, v[1]);
    v[2] = __fma_rn(bi, bi, v[2]);
  }
  cta_sum3(v, red);
  double rho = v[0], rr = v[1];
  const double bb = v[2];
  const double nb = sqrt(bb), nbe = nb > 0.0 ? nb : 1.0;
  const double thresh = eps > 0.0 ? eps * nbe : -1.0;
  int status = ST_OK, iter = 0;
  double beta = 0.0;
  bool done = (max_iter <= 0) || (thresh > 0.0 && !(sqrt(rr) > thresh));
  if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  while (!done) {
    // p_new = z + beta p_old (pointwise, in place), then w = A p_new, sigma = p.w
#pragma unroll
    for (int q = 0; q < CMAXN; ++q) {
      if (!own[q]) continue;
      const int i = tid + q * CNTH;
      const double zz = (ELEM ? DI[i] : cdinv) * R[i];
      P[hp[q]] = iter == 0 ? zz : __fma_rn(beta, P[hp[q]], zz);
    }
    __syncthreads();
    v[0] = v[1] = v[2] = 0.0;
#pragma unroll
    for (int q = 0; q < CMAXN; ++q) {
      if (!own[q]) continue;
      const int i = tid + q * CNTH;
      const double w = applyq(q, nullptr);
      W[i] = w;
      v[0] = __fma_rn(P[hp[q]], w, v[0]);
    }
    cta_sum3(v, red);
    const double sigma = v[0];
    if (!(sigma > 0.0)) { status = ST_EBREAKDOWN; break; }
    const double alpha = rho / sigma;
    v[0] = v[1] = v[2] = 0.0;
#pragma unroll
    for (int q = 0; q < CMAXN; ++q) {
      if (!own[q]) continue;
      const int i = tid + q * CNTH;
      X[i] = __fma_rn(alpha, P[hp[q]], X[i]);
      const double rn = __fma_rn(-alpha, W[i], R[i]);
      R[i] = rn;
      const double zz = (ELEM ? DI[i] : cdinv) * rn;
      v[0] = __fma_rn(rn, zz, v[0]);
      v[1] = __fma_rn(rn, rn, v[1]);
    }
    cta_sum3(v, red);
    beta = v[0] / rho;
    rho = v[0];
    rr = v[1];
    ++iter;
    done = (iter >= max_iter) || (thresh > 0.0 && !(sqrt(rr) > thresh));
    if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  }
  // x, r back to memory; true residual ||b - A x|| with x staged in P; fused scatter of u_h
  __syncthreads();
#pragma unroll
  for (int q = 0; q < CMAXN; ++q) {
    if (!own[q]) continue;
    const int i = tid + q * CNTH;
    a.x[nd[q].off] = X[i];
    a.r[nd[q].off] = R[i];
    P[hp[q]] = X[i];
  }
  __syncthreads();
  v[0] = v[1] = v[2] = 0.0;
#pragma unroll
  for (int q = 0; q < CMAXN; ++q) {
    if (!own[q]) continue;
    const double rn = a.b[nd[q].off] - applyq(q, nullptr);
    v[1] = __fma_rn(rn, rn, v[1]);
    if (u_out) u_out[full_index(g, nd[q].fx, nd[q].fy, nd[q].fz)] = P[hp[q]];
  }
  cta_sum3(v, red);
  if (tid == 0) {
    sc->rho = rho; sc->rr = rr; sc->bb = bb; sc->rr_true = v[1]; sc->beta = beta;
    sc->iter = iter; sc->max_iter = max_iter; sc->thresh = thresh; sc->status = status; sc->done = 1;
  }
}

size_t cta_smem_bytes(const LevelGeom& g, bool elem) {
  const long long n = (long long)g.nf[0] * g.nf[1] * g.nf[2];
  const long long nh = (long long)(g.nf[0] + 2) * (g.nf[1] + 2) * (g.nf[2] + 2);
  return sizeof(double) * (size_t)(nh + (elem ? 4 : 3) * n + 3 * (CNTH / 32) + 3);
}

template <bool ELEM>
int persistent_grid(int want) {
  static int slots = 0;
  if (!slots) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jcg_persistent<ELEM, false>, PNTH, sizeof(double) * MAXB * SN);
    slots = sms * std::max(1, per_sm);
  }
  return std::max(1, std::min(want, slots));
}

#ifndef ECMG_PERS_CLUSTER
#define ECMG_PERS_CLUSTER 1
#endif
// the cluster form of the persistent solve: can a cluster of C CTAs run on this GPU? (checked once per C)
template <bool ELEM>
bool cluster_fits(int C) {
  static int ok[MAXC + 1] = {0};   // 0 unknown, 1 yes, -1 no
  if (C < 1 || C > MAXC) return false;
  if (!ok[C]) {
    const void* fn = (const void*)k_jcg_persistent<ELEM, true>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(C); cfg.blockDim = dim3(PNTH); cfg.dynamicSmemBytes = sizeof(double) * MAXBC * SN;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, fn, &cfg);
    if (e != cudaSuccess) cudaGetLastError();
    ok[C] = (e == cudaSuccess && n >= 1) ? 1 : -1;
  }
  return ok[C] > 0;
}

}  // namespace

// the single-CTA solve takes the level if its free box fits (nodes and shared memory; not z-slabs)
bool cta_solve_fits(const LevelGeom& g, int elem_path, long long max_nodes) {
  const long long n = (long long)g.nf[0] * g.nf[1] * g.nf[2];
  if (n > std::min<long long>(max_nodes, CNODES) || g.nza != g.nf[2] || g.zoff != 0) return false;
  return cta_smem_bytes(g, elem_path != 0) <= 200 * 1024;
}

cudaError_t init_cta_kernel_attributes() {
  cudaError_t e = cudaFuncSetAttribute(k_jcg_cta<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_cta<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  return e;
}

// One launch of one CTA: the whole solve of a small level (cta_solve_fits). Arguments as
// launch_jcg_persistent (z and w unused).
cudaError_t launch_jcg_cta(const LevelGeom& g, const ConstStencil& cs, const ElemStencil* es, double* x, double* r,
                           const double* beta, const double* b, JcgScalars* sc, cudaStream_t st) {
  PArgs a{x, r, nullptr, {nullptr, nullptr}, nullptr, b, nullptr, beta, nullptr, sc};
  const ElemStencil e = es ? *es : ElemStencil{};
  const size_t smem = cta_smem_bytes(g, es != nullptr);
  count_launch();
  if (es) k_jcg_cta<true><<<1, CNTH, smem, st>>>(g, cs, e, a);
  else k_jcg_cta<false><<<1, CNTH, smem, st>>>(g, cs, e, a);
  return cudaGetLastError();
}

// partial-sum doubles the cooperative solves need: grid_sum3 / pers_grid_sum3 / elem_grid_sum3 ping-pong two
// buffers of 3 doubles per CTA, and their grids are at most the co-resident CTAs of each kernel
long long coop_partials_doubles() {
  const long long g = std::max<long long>(std::max(persistent_grid<true>(1 << 30), persistent_grid<false>(1 << 30)),
                                          std::max(const_pers_slots(), elem_pers_slots_count()));
  return 6 * g + 64;
}

// largest level (in bricks of 8 x 8 x 4 nodes) the persistent kernel takes: MAXB bricks per resident CTA
long long persistent_max_bricks(int elem_path) {
  return (long long)MAXB * (elem_path ? persistent_grid<true>(1 << 30) : persistent_grid<false>(1 << 30));
}

// One cooperative launch: the whole solve. Element path (es != nullptr): z, dinv and w are scratch
// vectors of the level's size; beta as in KArgs. Constant path: z, dinv, beta unused.
cudaError_t launch_jcg_persistent(const LevelGeom& g, const ConstStencil& cs, const ElemStencil* es, double* x, double* r,
                                  double* z, double* p0, double* p1, double* w, double* dinv, const double* beta,
                                  const double* b, double* partials, JcgScalars* sc, cudaStream_t st) {
  const long long nbricks = (long long)((g.nf[0] + BX - 1) / BX) * ((g.nf[1] + BY - 1) / BY) * ((g.nf[2] + BZ - 1) / BZ);
  PArgs a{x, r, z, {p0, p1}, w, b, dinv, beta, partials, sc};
  const ElemStencil e = es ? *es : ElemStencil{};
  void* args[] = {(void*)&g, (void*)&cs, (void*)&e, (void*)&a};
  // levels of at most MAXC bricks: one thread-block cluster, one brick per CTA
  const int C = (int)std::min<long long>(nbricks, MAXC);
  if (ECMG_PERS_CLUSTER && nbricks <= (long long)MAXC * MAXBC && (es ? cluster_fits<true>(C) : cluster_fits<false>(C))) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(C); cfg.blockDim = dim3(PNTH); cfg.dynamicSmemBytes = sizeof(double) * MAXBC * SN;
    cfg.stream = st; cfg.attrs = at; cfg.numAttrs = 1;
    count_launch();
    return cudaLaunchKernelExC(&cfg, es ? (const void*)k_jcg_persistent<true, true> : (const void*)k_jcg_persistent<false, true>,
                               args);
  }
  // one brick per CTA while the CTAs fit (parallelism), up to MAXB per CTA beyond that
  const int slots = es ? persistent_grid<true>(1 << 30) : persistent_grid<false>(1 << 30);
  if (nbricks > (long long)MAXB * slots) return cudaErrorInvalidValue;
  const int want = (int)std::min<long long>(nbricks, slots);
  count_launch();
  if (es)
    return cudaLaunchCooperativeKernel((const void*)k_jcg_persistent<true, false>, dim3(persistent_grid<true>(want)),
                                       dim3(PNTH), args, sizeof(double) * MAXB * SN, st);
  return cudaLaunchCooperativeKernel((const void*)k_jcg_persistent<false, false>, dim3(persistent_grid<false>(want)),
                                     dim3(PNTH), args, sizeof(double) * MAXB * SN, st);
}

}  // namespace ecmg
