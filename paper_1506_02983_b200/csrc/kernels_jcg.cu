// kernels_jcg.cu -- fused JCG kernels for the Q1 system A_h u_h = f_h, the hot loop of
// Alg. 4 l.7-9: textbook PCG with M = diag(A_h).
//
// One iteration = two kernels (SURVEY.md §8a "a5"):
//   K1: p_new = D^-1 r + beta_cg p_old (recomputed on the tile halo), w = A p_new, sigma = p_new.w,
//       alpha = rho / sigma (last CTA)                       -- reads r, p_old; writes p_new
//   K2: w = A p_new recomputed, x += alpha p, r -= alpha w, z = D^-1 r, rho' = r.z, rr = r.r,
//       beta_cg = rho'/rho, stop test (last CTA)             -- reads x, r, p; writes x, r
// = 8 fp64 accesses = 64 B per free unknown and iteration (+8 B per kernel for beta_e on the
// element path). Dot products are deterministic: a fixed shuffle tree per CTA, per-CTA partials,
// and the last CTA to finish sums the partials in CTA order. All CG scalars stay on the device.
//
// Both kernels march along z: a CTA owns a 32 x TY tile of (x, y) columns and a chunk of z
// planes; each plane of the input is read once from HBM (plus a 1-node halo ring, L2 hits from
// neighbouring CTAs) and staged in shared memory; the 27-point stencil is split into per-plane
// partial sums kept in registers, so every value is loaded from shared memory a few times only.
#include <algorithm>
#include "ecmg_internal.cuh"
#include "problems.cuh"
#include "jcg_common.cuh"

namespace ecmg {
namespace {

// ============================================================================================
// Constant-coefficient path (beta constant, all faces Dirichlet): C1, C2, C4 and the patch test.
// Tile 32 x 32 columns (each warp owns 4 rows), 34 x 34 halo plane in shared memory.
// ============================================================================================
constexpr int CRY = 4;
constexpr int CTY = WARPS * CRY;   // 32
constexpr int CHX = TX + 2;        // 34
constexpr int CHY = CTY + 2;       // 34

template <int MODE>
__global__ void __launch_bounds__(NTH, 2) k_jcg_const(const LevelGeom g, const ConstStencil cs, const KArgs a) {
  __shared__ double Pl[2][CHY][CHX];
  JcgScalars* sc = a.sc;
  if (MODE == MODE_K1 || MODE == MODE_K2) {
    if (*(volatile int*)&sc->done) return;   // converged / failed: speculative launches are no-ops
  }
  const int lane = threadIdx.x, w = threadIdx.y, tid = lane + TX * w;
  const int nfx = g.nf[0], nfy = g.nf[1], nfz = g.nza;   // local planes
  const long long P = g.P, S = g.S;
  const int X0 = blockIdx.x * TX, Y0 = blockIdx.y * CTY;
  const int z0 = g.zbeg + blockIdx.z * a.zc;
  const int z1 = min(z0 + a.zc, g.zend);
  const int x = X0 + lane;
  const int yb = Y0 + CRY * w;

  // halo ring slot of this thread (132 slots: 2 rows of 34, 2 columns of 32)
  int rhx = -1, rhy = -1;
  if (tid < 2 * CHX) { rhx = tid % CHX; rhy = (tid < CHX) ? 0 : CHY - 1; }
  else if (tid < 2 * CHX + 2 * CTY) { const int t = tid - 2 * CHX; rhx = (t < CTY) ? 0 : CHX - 1; rhy = 1 + (t % CTY); }
  const int rgx = X0 - 1 + rhx, rgy = Y0 - 1 + rhy;
  const bool ring_ok = rhx >= 0 && rgx >= 0 && rgx < nfx && rgy >= 0 && rgy < nfy;
  const long long ring_off = ring_ok ? (long long)rgy * P + rgx : 0;
  bool own_ok[CRY];
  long long own_off[CRY];
#pragma unroll
  for (int j = 0; j < CRY; ++j) {
    own_ok[j] = (x < nfx) && (yb + j < nfy);
    own_off[j] = own_ok[j] ? (long long)(yb + j) * P + x : 0;
  }

  double bcg = 0.0, alpha = 0.0;
  bool first = false;
  if (MODE == MODE_K1) { bcg = sc->beta; first = (sc->iter == 0); }
  if (MODE == MODE_K2) alpha = sc->alpha;
  double* const u_out = (MODE == MODE_TRUE) ? sc->in.u_out : nullptr;
  const double dinv = cs.dinv;
  constexpr bool kTwoHalo = (MODE == MODE_K1);
  constexpr bool kInt0 = (MODE == MODE_K2 || MODE == MODE_INIT || MODE == MODE_TRUE);
  constexpr bool kInt1 = (MODE == MODE_K2);

  double nh0[CRY], nh1[CRY], nr0 = 0.0, nr1 = 0.0;   // prefetched halo-array values, plane zl+1
  double ni0[CRY], ni1[CRY];                          // prefetched interior values, plane zl
#pragma unroll
  for (int j = 0; j < CRY; ++j) { nh0[j] = nh1[j] = ni0[j] = ni1[j] = 0.0; }

  auto load_halo = [&](int z) {
    const bool zok = (z >= 0) && (z < nfz);
    const long long zo = zok ? (long long)z * S : 0;
#pragma unroll
    for (int j = 0; j < CRY; ++j) nh0[j] = (zok && own_ok[j]) ? __ldg(a.h0 + zo + own_off[j]) : 0.0;
    nr0 = (zok && ring_ok) ? __ldg(a.h0 + zo + ring_off) : 0.0;
    if (kTwoHalo && !first) {
#pragma unroll
      for (int j = 0; j < CRY; ++j) nh1[j] = (zok && own_ok[j]) ? __ldg(a.h1 + zo + own_off[j]) : 0.0;
      nr1 = (zok && ring_ok) ? __ldg(a.h1 + zo + ring_off) : 0.0;
    }
  };
  auto load_int = [&](int z) {
    const long long zo = (long long)z * S;
#pragma unroll
    for (int j = 0; j < CRY; ++j) {
      if (kInt0) ni0[j] = own_ok[j] ? __ldg(a.i0 + zo + own_off[j]) : 0.0;
      if (kInt1) ni1[j] = own_ok[j] ? __ldg(a.i1 + zo + own_off[j]) : 0.0;
    }
  };
  auto transform = [&](double v0, double v1) -> double {
    if (MODE == MODE_K1) return pcg_direction(dinv, v0, bcg, v1, first);
    return v0;
  };

  double part[CRY], q1p[CRY], pp[CRY];
#pragma unroll
  for (int j = 0; j < CRY; ++j) { part[j] = q1p[j] = pp[j] = 0.0; }
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;

  load_halo(z0 - 1);
  const int nsteps = z1 - z0 + 2;
  for (int s = 0; s < nsteps; ++s) {
    const int zl = z0 - 1 + s;
    double c0[CRY], c1[CRY], ii0[CRY], ii1[CRY];
#pragma unroll
    for (int j = 0; j < CRY; ++j) { c0[j] = nh0[j]; c1[j] = nh1[j]; ii0[j] = ni0[j]; ii1[j] = ni1[j]; }
    const double cr0 = nr0, cr1 = nr1;
    if (s + 1 < nsteps) load_halo(zl + 1);
    if ((kInt0 || kInt1) && zl >= z0 && zl < z1) load_int(zl);

    double (*Pb)[CHX] = Pl[s & 1];
    const bool halo_store = (MODE == MODE_K1) && (zl == g.zbeg - 1 || zl == g.zend) && zl >= 0 && zl < nfz;
#pragma unroll
    for (int j = 0; j < CRY; ++j) {
      const double v = transform(c0[j], c1[j]);
      Pb[1 + CRY * w + j][1 + lane] = v;
      if (halo_store && own_ok[j]) a.o0[(long long)zl * S + own_off[j]] = v;   // slab halo plane of p
    }
    if (rhx >= 0) Pb[rhy][rhx] = transform(cr0, cr1);
    __syncthreads();

    double col[CRY + 2][3];
#pragma unroll
    for (int r = 0; r < CRY + 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) col[r][c] = Pb[CRY * w + r][lane + c];

    const int z = zl - 1;   // plane completed in this step (valid for s >= 2)
#pragma unroll
    for (int j = 0; j < CRY; ++j) {
      const double cc = col[j + 1][1];
      const double ax = col[j + 1][0] + col[j + 1][2];
      const double ay = col[j][1] + col[j + 2][1];
      const double dd = (col[j][0] + col[j][2]) + (col[j + 2][0] + col[j + 2][2]);
      double q0, q1;
      stencil_q(cs, cc, ax, ay, dd, q0, q1);
      if (s >= 2 && own_ok[j]) {
        const double ap = part[j] + q1;   // (A p) at plane z
        const long long off = (long long)z * S + own_off[j];
        if (MODE == MODE_K1) {
          acc0 = __fma_rn(pp[j], ap, acc0);
          a.o0[off] = pp[j];
        } else if (MODE == MODE_K2) {
          const double xn = __fma_rn(alpha, pp[j], ii0[j]);
          const double rn = __fma_rn(-alpha, ap, ii1[j]);
          const double zz = dinv * rn;
          acc0 = __fma_rn(rn, zz, acc0);
          acc1 = __fma_rn(rn, rn, acc1);
          a.o0[off] = xn;
          a.o1[off] = rn;
          if (z == g.zbeg && a.peer_lo) a.peer_lo[own_off[j]] = rn;      // fused halo exchange
          if (z == g.zend - 1 && a.peer_hi) a.peer_hi[own_off[j]] = rn;
        } else if (MODE == MODE_INIT) {
          acc2 = __fma_rn(ii0[j], ii0[j], acc2);
          const double rn = ii0[j] - ap;
          const double zz = dinv * rn;
          acc0 = __fma_rn(rn, zz, acc0);
          acc1 = __fma_rn(rn, rn, acc1);
          a.o0[off] = rn;
          if (z == g.zbeg && a.peer_lo) a.peer_lo[own_off[j]] = rn;      // fused halo exchange
          if (z == g.zend - 1 && a.peer_hi) a.peer_hi[own_off[j]] = rn;
        } else if (MODE == MODE_TRUE) {
          const double rn = ii0[j] - ap;
          acc1 = __fma_rn(rn, rn, acc1);
          if (u_out) u_out[full_index(g, x, yb + j, z)] = pp[j];   // fused scatter of u_h
        } else {
          a.o0[off] = ap;
        }
      }
      part[j] = q1p[j] + q0;
      q1p[j] = q1;
      pp[j] = cc;
    }
  }
  if ((MODE == MODE_K2 || MODE == MODE_INIT) && (a.peer_lo || a.peer_hi)) __threadfence_system();   // peer stores
  if (MODE != MODE_APPLY) reduce_finalize(MODE, a, acc0, acc1, acc2);
}

}  // namespace

namespace {
template <int MODE>
__global__ void k_finalize(const KArgs a) {
  if (MODE == MODE_K1 || MODE == MODE_K2) {
    if (*(volatile int*)&a.sc->done) return;   // converged: the speculative pass is a no-op
  }
  finalize(MODE, a, a.sc->glob[0], a.sc->glob[1], a.sc->glob[2]);
}
__global__ void k_vsum(const SlabScalars s) {
  for (int k = 0; k < 3; ++k) {
    double t = 0.0;
    for (int i = 0; i < s.n; ++i) t += s.p[i]->loc[k];   // slab order: deterministic
    for (int i = 0; i < s.n; ++i) s.p[i]->glob[k] = t;
  }
}
}  // namespace

cudaError_t launch_finalize(int mode, const KArgs& a, cudaStream_t st) {
  count_launch();
  switch (mode) {
    case MODE_K1: k_finalize<MODE_K1><<<1, 1, 0, st>>>(a); break;
    case MODE_K2: k_finalize<MODE_K2><<<1, 1, 0, st>>>(a); break;
    case MODE_INIT: k_finalize<MODE_INIT><<<1, 1, 0, st>>>(a); break;
    case MODE_TRUE: k_finalize<MODE_TRUE><<<1, 1, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// a level without free unknowns (one cell along an all-Dirichlet axis): the solve is empty -- 0 iterations,
// ||b|| = 0, the residuals 0 -- and its scalars are written as a finished solve would leave them
__global__ void k_empty_solve(JcgScalars* sc) {
  sc->rho = 0.0; sc->rr = 0.0; sc->bb = 0.0; sc->rr_true = 0.0; sc->beta = 0.0; sc->alpha = 0.0; sc->sigma = 0.0;
  sc->iter = 0; sc->max_iter = sc->in.max_iter; sc->thresh = -1.0; sc->status = ST_OK; sc->done = 1; sc->counter = 0;
}
cudaError_t launch_empty_solve(JcgScalars* sc, cudaStream_t st) {
  count_launch();
  k_empty_solve<<<1, 1, 0, st>>>(sc);
  return cudaGetLastError();
}

// deferred x update (KArgs::xdefer): a solve that stopped after a skipping K2 (iteration count odd) still owes
// x += alpha_{k} p_{k} with p_k in p; otherwise a no-op. Same rounding as the K2 update it stands in for.
__global__ void k_xfix(const LevelGeom g, double* __restrict__ x, const double* __restrict__ p, const JcgScalars* sc) {
  if (!(sc->iter & 1)) return;
  const double alpha = sc->alpha;
  const long long nrow = (long long)g.nf[1] * (g.zend - g.zbeg);
  for (long long row = blockIdx.x * (long long)blockDim.y + threadIdx.y; row < nrow; row += (long long)gridDim.x * blockDim.y) {
    const long long off = (long long)(g.zbeg + row / g.nf[1]) * g.S + (row % g.nf[1]) * g.P;
    for (int i = threadIdx.x; i < g.nf[0]; i += blockDim.x) x[off + i] = __fma_rn(alpha, p[off + i], x[off + i]);
  }
}
cudaError_t launch_xfix(const LevelGeom& g, double* x, const double* p, const JcgScalars* sc, cudaStream_t st) {
  count_launch();
  const long long nrow = (long long)g.nf[1] * (g.zend - g.zbeg);
  const int blocks = (int)std::max(1LL, std::min(nrow / 8 + 1, 148LL * 16));
  k_xfix<<<blocks, dim3(32, 8), 0, st>>>(g, x, p, sc);
  return cudaGetLastError();
}

cudaError_t launch_vsum(const SlabScalars& s, cudaStream_t st) {
  count_launch();
  k_vsum<<<1, 1, 0, st>>>(s);
  return cudaGetLastError();
}

int jcg_num_blocks(const LevelGeom& g, int elem_path, int zc) {
  const int ty = elem_path ? 16 : CTY;
  const int bx = (g.nf[0] + TX - 1) / TX, by = (g.nf[1] + ty - 1) / ty, bz = (g.zend - g.zbeg + zc - 1) / zc;
  return bx * by * bz;
}

cudaError_t launch_jcg_const(int mode, const LevelGeom& g, const ConstStencil& cs, const KArgs& a, cudaStream_t st) {
  dim3 block(TX, WARPS);
  dim3 grid((g.nf[0] + TX - 1) / TX, (g.nf[1] + CTY - 1) / CTY, (g.zend - g.zbeg + a.zc - 1) / a.zc);
  switch (mode) {
    case MODE_K1: count_launch(); k_jcg_const<MODE_K1><<<grid, block, 0, st>>>(g, cs, a); break;
    case MODE_K2: count_launch(); k_jcg_const<MODE_K2><<<grid, block, 0, st>>>(g, cs, a); break;
    case MODE_INIT: count_launch(); k_jcg_const<MODE_INIT><<<grid, block, 0, st>>>(g, cs, a); break;
    case MODE_TRUE: count_launch(); k_jcg_const<MODE_TRUE><<<grid, block, 0, st>>>(g, cs, a); break;
    case MODE_APPLY: count_launch(); k_jcg_const<MODE_APPLY><<<grid, block, 0, st>>>(g, cs, a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace ecmg
