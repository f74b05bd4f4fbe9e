// kernels_jcg_elem.cu -- TMA-fed z-marching JCG kernels for the element-beta operator: beta_e per
// element and / or Robin / Neumann faces (C3, C5, P1-P3, the layered and Robin patch problems;
// SURVEY.md §8a a4/a5). Same device-side CG recurrences as the constant-stencil kernels
// (Alg. 4 l.7-9; textbook PCG, §8c O7).
//
// Operator (§8c A3): (A p)_i = sum_{e ni i} beta_e sum_{j in e} kappa[pat(i,j)] p_j
//   + sum_{Robin faces F ni i} alpha_F h1 h2 sum_{face elements f ni i} sum_{j in f} m2[pat] p_j,
// pat = bit d set if i, j differ along axis d (ElemStencil), m2 = {1/9, 1/18, 1/18, 1/36}.
//
// Element-layer split. The element layer between node planes d and u = d + 1 contributes to the
// nodes of both planes. For a node column c and the four layer elements around it (betas
// b_LB, b_RB, b_LA, b_RA: left / right in x, below / above in y), the beta-weighted in-plane sums
// of a node plane v are
//   G0(v) = B4 v_c,   G1(v) = W_x- v_x- + W_x+ v_x+,   G2(v) = W_y- v_y- + W_y+ v_y+,
//   G3(v) = b_LB v_(x-,y-) + b_RB v_(x+,y-) + b_LA v_(x-,y+) + b_RA v_(x+,y+),
// with B4 the sum of the four betas and W the sum of the two betas of the elements holding the edge.
// The layer adds  sum_j kappa[j] G_j(p_d) + kappa[j+4] G_j(p_u)  to node (c, d) and
//                 sum_j kappa[j] G_j(p_u) + kappa[j+4] G_j(p_d)  to node (c, u)
// (pattern bit 4: the partner is in the other plane). A node completes once the layer above it is
// added; the layer-below half rides in registers from the previous step. About 40 fp64 operations
// per node instead of the 64 + 8 of the element-by-element form, and every beta is read once.
//
// CG data flow of this path: the residual is carried as z = D^-1 r only (D = Jacobi diagonal
// kappa_0 sum_{e ni i} beta_e + Robin diagonal, formed from the beta sums the kernel holds anyway): INIT
// writes z_0, K2 forms r_k = D z_k at its own nodes, updates r_{k+1} = r_k - alpha A p and writes z_{k+1};
// K1 needs only z and p_old on its halo (p = z + beta_cg p_old): no diagonal on halo nodes, no r vector.
// HBM per unknown and iteration: K1 reads z, p_old, beta, writes p (32 B); K2 reads p, beta, x, z and
// writes x, z (48 B): 80 B, the algorithmic figure of SURVEY.md §8d D.3 (reading R8).
//
// Data movement as in kernels_jcg_tma.cu: one cp.async.bulk.tensor.3d per CTA and vector per plane
// into an NS-deep ring (mbarrier expect_tx), out-of-bounds boxes zero-filled (= p on Dirichlet /
// outside nodes, beta outside the domain). Tile 32 x 16 nodes, 2 rows per warp.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <mutex>
#include <type_traits>
#include <cooperative_groups.h>
#include "ecmg_internal.cuh"
#include "jcg_common.cuh"

namespace ecmg {
namespace {

#ifndef ELEM_RY
#define ELEM_RY 2
#endif
constexpr int RY = ELEM_RY;           // node rows per warp (two fp64 plane windows stay in registers)
constexpr int TY = WARPS * RY;        // 16
constexpr int HX = TX + 4;            // 36: node halo box x = X0-2 .. X0+33 (16-B aligned start)
constexpr int XO = 2;                 // smem column of x = X0
constexpr int HY = TY + 2;            // 18
constexpr int HBYTES = HX * HY * 8;
constexpr int HSTRIDE = (HBYTES + 127) / 128 * 128;
constexpr int EBX = TX + 4;           // 36 element columns: beta-array index X0 .. X0+35
constexpr int EBY = TY + 1;           // 17 element rows
constexpr int EBYTES = EBX * EBY * 8;
constexpr int ESTRIDE = (EBYTES + 127) / 128 * 128;
constexpr int IBYTES = TX * TY * 8;
#ifndef ELEM_MINB
#define ELEM_MINB 2
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// XD: deferred x update of K2 (KArgs::xdefer): interior boxes x, z (0) | z (1: x skipped) | x, z, p_{k-1} (2)
template <int MODE, int XD = 0>
struct ElemCfg {
  static constexpr bool kH1 = (MODE == MODE_K1);
  static constexpr int kNI = (MODE == MODE_K2) ? (XD == 1 ? 1 : (XD == 2 ? 3 : 2)) : ((MODE == MODE_INIT || MODE == MODE_TRUE) ? 1 : 0);
  static constexpr int OFF_E = HSTRIDE * (kH1 ? 2 : 1);
  static constexpr int OFF_I = OFF_E + ESTRIDE;
  static constexpr int SBYTES = OFF_I + IBYTES * kNI;
};

// loads of step t: node plane zh = z0-1+t (halo boxes), element layer (zh-1, zh), interior plane zh-1
template <int MODE, int SB, int BF, int XD = 0>
__device__ __forceinline__ void issue_elem_stage(unsigned char* smem, uint64_t* full, int st, int t, int z0, int X0,
                                                 int Y0, int ey0, int ez_base, uint32_t tx_bytes, bool first,
                                                 const CUtensorMap* pH0, const CUtensorMap* pH1, const CUtensorMap* pE,
                                                 const CUtensorMap* pI0, const CUtensorMap* pI1,
                                                 const CUtensorMap* pI2 = nullptr) {
  using C = ElemCfg<MODE, XD>;
  unsigned char* base = smem + st * SB;
  mbar_expect_tx(&full[st], tx_bytes);
  const int zh = z0 - 1 + t;
  tma_load_3d(base, pH0, X0 - XO, Y0 - 1, zh, &full[st]);
  if (C::kH1) tma_load_3d(base + HSTRIDE, pH1, X0 - XO, Y0 - 1, zh, &full[st]);
  if (BF == 0) tma_load_3d(base + C::OFF_E, pE, X0, ey0, ez_base + zh, &full[st]);   // else: beta on the fly
  if (C::kNI >= 1) tma_load_3d(base + C::OFF_I, pI0, X0, Y0, zh - 1, &full[st]);
  if (C::kNI >= 2) tma_load_3d(base + C::OFF_I + IBYTES, pI1, X0, Y0, zh - 1, &full[st]);
  if (C::kNI >= 3) tma_load_3d(base + C::OFF_I + 2 * IBYTES, pI2, X0, Y0, zh - 1, &full[st]);
}

// One z-march of the CTA over its (tile, z chunk) in mode MODE (the body of k_jcg_elem_tma): the stage
// ring continues at the running step count G (stage (G + s) % NS, parity ((G + s) / NS) & 1), so that a
// persistent CTA can run several passes over the same mbarriers. Adds the thread's partial sums to
// acc0..acc2. The caller has initialised the mbarriers and synchronised the CTA since its previous pass.
// BFA: 0 = beta from the array (TMA box per layer); 1 = on the fly, product kind (C3); 2 = on the fly,
// bit-mask kinds (beta = 1, layers, C5 boxes) -- see beta_combine; 3 = beta from the array and the Robin alpha
// at the face Gauss points (ARRAYS alpha_q, es.aq): the only instantiations that carry that branch
// XD: deferred x update of K2 (KArgs::xdefer): 1 = x untouched (the one interior box, pI0, is z); 2 = both pending
// updates, x <- fma(alpha, p_k, fma(alpha0, p_{k-1}, x)) with p_{k-1} in the third interior box pI2
template <int MODE, int NS, bool CUBE, int SB, int BFA, int XD = 0>
__device__ __forceinline__ void elem_pass(const LevelGeom& g, const ElemStencil& es, const KArgs& a, int X0, int Y0, int z0,
                                          int z1, double bcg_eff, bool first, double alpha, double* u_out,
                                          const CUtensorMap* pH0, const CUtensorMap* pH1, const CUtensorMap* pE,
                                          const CUtensorMap* pI0, const CUtensorMap* pI1, unsigned char* smem, uint64_t* full,
                                          const uint32_t G, double& acc0, double& acc1, double& acc2,
                                          const CUtensorMap* pI2 = nullptr, double alpha0 = 0.0) {
  using C = ElemCfg<MODE, XD>;
  constexpr int BF = BFA == 3 ? 0 : BFA;   // how beta arrives
  constexpr bool AQ = BFA == 3;            // alpha at the face Gauss points
  const int lane = threadIdx.x, w = threadIdx.y, tid = lane + TX * w;
  const int nfx = g.nf[0], nfy = g.nf[1];
  const long long S = g.S;
  const int P = (int)g.P;
  const uint32_t tx_bytes = HBYTES * (C::kH1 ? 2 : 1) + (BF ? 0 : EBYTES) + IBYTES * C::kNI;
  const int ez_base = g.flo[2] + g.zoff + 1;       // beta-array plane of the layer below node plane 0, + 1
  const int eo = g.flo[0] + 1;                     // smem column of the left element of lane 0
  const bool zrobin = es.robin[4] != 0.0 || es.robin[5] != 0.0;
#define k0 es.kappa[0]
#define k1 es.kappa[1]
#define k2 es.kappa[2]
#define k3 es.kappa[3]
#define k4 es.kappa[4]
#define k5 es.kappa[5]
#define k6 es.kappa[6]
#define k7 es.kappa[7]
  constexpr double c9 = 1.0 / 9.0, c18 = 1.0 / 18.0, c36 = 1.0 / 36.0;
  if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int x = X0 + lane, yb = Y0 + RY * w;
  const int nsteps = z1 - z0 + 2;
  const int ey0 = g.flo[1] + Y0 + 1;               // beta-array row of the element below node row Y0
  if (tid == 0) {
    for (int t = 0; t < NS - 1 && t < nsteps; ++t)
      issue_elem_stage<MODE, SB, BF, XD>(smem, full, (G + t) % NS, t, z0, X0, Y0, ey0, ez_base, tx_bytes, first, pH0, pH1, pE, pI0,
                             pI1, pI2);
  }

  bool own_ok[RY];
  int own_off[RY];
#pragma unroll
  for (int j = 0; j < RY; ++j) {
    own_ok[j] = (x < nfx) && (yb + j < nfy);
    own_off[j] = own_ok[j] ? (yb + j) * P + x : 0;
  }
  // Robin faces (rare path): does a node of this thread lie on a Robin x- or y-face
  const int gx = g.flo[0] + x, gy0 = g.flo[1] + yb;
  const bool edge = (gx == 0 && es.robin[0] != 0.0) || (gx == g.n[0] && es.robin[1] != 0.0) ||
                    (gy0 <= 0 && gy0 + RY - 1 >= 0 && es.robin[2] != 0.0) ||
                    (gy0 <= g.n[1] && gy0 + RY - 1 >= g.n[1] && es.robin[3] != 0.0);

  double part[RY], dpart[RY];
#pragma unroll
  for (int j = 0; j < RY; ++j) { part[j] = 0.0; dpart[j] = 0.0; }
  // beta on the fly: the thread's 2 element columns x 3 element rows are fixed for the pass; per layer
  // one (uniform) table entry. pk: 5 bits (exists, boxes) per (row, column); bt: products Ax Ay (C3)
  const int BW = es.bw;
  const double* tA = es.baxes;
  const int* tM = reinterpret_cast<const int*>(es.baxes + 3LL * BW);
  const double* boxb = es.baxes + 3LL * BW + (3LL * BW + 1) / 2;
  int pk = 0;
  double bt[RY + 1][2];
  if (BF) {
    double axc[2], ayr[RY + 1];
    int mxc[2], myr[RY + 1];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int ex = X0 + g.flo[0] - 1 + lane + c;
      const bool in = ex >= -2 && ex < g.n[0] + 2;
      axc[c] = (BF == 1 && in) ? tA[ex + 2] : 0.0;
      mxc[c] = in ? tM[ex + 2] : 0;
    }
#pragma unroll
    for (int r = 0; r < RY + 1; ++r) {
      const int ey = g.flo[1] + Y0 - 1 + RY * w + r;
      const bool in = ey >= -2 && ey < g.n[1] + 2;
      ayr[r] = (BF == 1 && in) ? tA[BW + ey + 2] : 0.0;
      myr[r] = in ? tM[BW + ey + 2] : 0;
    }
#pragma unroll
    for (int r = 0; r < RY + 1; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        pk |= ((mxc[c] & myr[r]) & 31) << (5 * (2 * r + c));
        bt[r][c] = BF == 1 ? axc[c] * ayr[r] : 0.0;
      }
  }

  // one z step: node plane zl = z0-1+s arrives in wu; wd holds plane zl-1 (previous step)
  auto step = [&](int s, double (&wd)[RY + 2][3], double (&wu)[RY + 2][3]) {
    const int zl = z0 - 1 + s;
    const uint32_t gs = G + s;
    const int st = gs % NS;
    if (s > 0) __syncthreads();   // every thread is done with step s-1: its stage may be refilled
    if (tid == 0 && s + NS - 1 < nsteps) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int t = s + NS - 1;
      issue_elem_stage<MODE, SB, BF, XD>(smem, full, (G + t) % NS, t, z0, X0, Y0, ey0, ez_base, tx_bytes, first, pH0, pH1, pE,
                             pI0, pI1, pI2);
    }
    mbar_wait(&full[st], (gs / NS) & 1u);
    unsigned char* stage = smem + st * SB;
    const double* H = reinterpret_cast<const double*>(stage);
    if (MODE == MODE_K1) {   // p = z + beta_cg p_old, formed per thread for its whole window
      const double* H1 = reinterpret_cast<const double*>(stage + HSTRIDE);
#pragma unroll
      for (int r = 0; r < RY + 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int o = (RY * w + r) * HX + XO - 1 + lane + c;
          wu[r][c] = __fma_rn(bcg_eff, H1[o], H[o]);
        }
      if ((zl == g.zbeg - 1 || zl == g.zend) && zl >= 0 && zl < g.nza) {
#pragma unroll
        for (int j = 0; j < RY; ++j)
          if (own_ok[j]) a.o0[(long long)zl * S + own_off[j]] = wu[j + 1][1];   // slab halo plane of p
      }
    } else {
#pragma unroll
      for (int r = 0; r < RY + 2; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) wu[r][c] = H[(RY * w + r) * HX + XO - 1 + lane + c];
    }
    if (s == 0) return;
    double bl[RY + 1][2];
    if (BF) {   // beta_combine on the layer's table entry (same function and inputs as the array, k_beta)
      const int ez = g.flo[2] + g.zoff - 1 + zl;
      const bool in = ez >= -2 && ez < g.n[2] + 2;
      const double az = in ? tA[2 * BW + ez + 2] : 0.0;
      const int mz = in ? tM[2 * BW + ez + 2] : 0;
#pragma unroll
      for (int r = 0; r < RY + 1; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int m = (pk >> (5 * (2 * r + c))) & mz;
          if (BF == 1) bl[r][c] = (m & 16) ? __fma_rn(bt[r][c], az, 1.0) : 0.0;
          else bl[r][c] = beta_combine(es.bkind, 0.0, 0.0, az, m, 31, 31, boxb);
        }
    } else {
      const double* E = reinterpret_cast<const double*>(stage + C::OFF_E);
#pragma unroll
      for (int r = 0; r < RY + 1; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) bl[r][c] = E[(RY * w + r) * EBX + eo + lane + c];
    }
    const double* I0 = reinterpret_cast<const double*>(stage + C::OFF_I);
    const double* I1 = I0 + TX * TY;
    const int d = zl - 1;   // node plane completed in this step
    const int gzd = g.flo[2] + g.zoff + d;
    const bool layer_ok = gzd >= 0 && gzd < g.n[2];
    const double rz = zrobin ? ((gzd == 0 ? es.robin[4] : 0.0) + (gzd == g.n[2] ? es.robin[5] : 0.0)) : 0.0;
    const bool rare = edge || rz != 0.0;
#pragma unroll
    for (int j = 0; j < RY; ++j) {
      const double bLB = bl[j][0], bRB = bl[j][1], bLA = bl[j + 1][0], bRA = bl[j + 1][1];
      const double Wxm = bLB + bLA, Wxp = bRB + bRA, Wym = bLB + bRB, Wyp = bLA + bRA;
      const double B4 = Wxm + Wxp;
      double upd, dnu;
      if (CUBE) {
        // cubic cells: kappa = {4c, 0, 0, -c, 0, -c, -c, -c} by pattern (K_e = c{4,0,-1,-1}), so
        //   to d: kappa_0 G0(p_d) + kappa_7 (G3(p_d) + Sg(p_u)),  to u: kappa_0 G0(p_u) + kappa_7 (G3(p_u) + Sg(p_d))
        // with Sg = G1 + G2 + G3 (the axis-weight zeros are dropped: |kappa_1| <= 1e-16 kappa_0 in fp64)
        const double gd3 = __fma_rn(bRA, wd[j + 2][2], __fma_rn(bLA, wd[j + 2][0], __fma_rn(bRB, wd[j][2], bLB * wd[j][0])));
        const double gu3 = __fma_rn(bRA, wu[j + 2][2], __fma_rn(bLA, wu[j + 2][0], __fma_rn(bRB, wu[j][2], bLB * wu[j][0])));
        const double sd = __fma_rn(Wyp, wd[j + 2][1], __fma_rn(Wym, wd[j][1], __fma_rn(Wxp, wd[j + 1][2], __fma_rn(Wxm, wd[j + 1][0], gd3))));
        const double su = __fma_rn(Wyp, wu[j + 2][1], __fma_rn(Wym, wu[j][1], __fma_rn(Wxp, wu[j + 1][2], __fma_rn(Wxm, wu[j + 1][0], gu3))));
        upd = __fma_rn(k0, B4 * wd[j + 1][1], k7 * (gd3 + su));
        dnu = __fma_rn(k0, B4 * wu[j + 1][1], k7 * (gu3 + sd));
      } else {
      const double gd0 = B4 * wd[j + 1][1], gu0 = B4 * wu[j + 1][1];
      const double gd1 = __fma_rn(Wxp, wd[j + 1][2], Wxm * wd[j + 1][0]);
      const double gu1 = __fma_rn(Wxp, wu[j + 1][2], Wxm * wu[j + 1][0]);
      const double gd2 = __fma_rn(Wyp, wd[j + 2][1], Wym * wd[j][1]);
      const double gu2 = __fma_rn(Wyp, wu[j + 2][1], Wym * wu[j][1]);
      const double gd3 = __fma_rn(bRA, wd[j + 2][2], __fma_rn(bLA, wd[j + 2][0], __fma_rn(bRB, wd[j][2], bLB * wd[j][0])));
      const double gu3 = __fma_rn(bRA, wu[j + 2][2], __fma_rn(bLA, wu[j + 2][0], __fma_rn(bRB, wu[j][2], bLB * wu[j][0])));
      upd = __fma_rn(k0, gd0, __fma_rn(k1, gd1, __fma_rn(k2, gd2, __fma_rn(k3, gd3,
            __fma_rn(k4, gu0, __fma_rn(k5, gu1, __fma_rn(k6, gu2, k7 * gu3)))))));
      dnu = __fma_rn(k0, gu0, __fma_rn(k1, gu1, __fma_rn(k2, gu2, __fma_rn(k3, gu3,
            __fma_rn(k4, gd0, __fma_rn(k5, gd1, __fma_rn(k6, gd2, k7 * gd3)))))));
      }
      double diag_d = k0 * B4, diag_u = k0 * B4;
      if (AQ && rare) {
        // Robin face mass with alpha at the face Gauss points (ARRAYS alpha_q): per face element, its 4 alphas
        // read from the caller's array (boundary nodes only). Windows: rows j..j+2 = y-1..y+1, columns 0..2 =
        // x-1..x+1 of planes d (wd) and u (wu)
        double ad = 0.0, au = 0.0, gdd = 0.0, gdu = 0.0;
        const int gy = gy0 + j;
        if (layer_ok)
          for (int F = 0; F < 2; ++F) {   // x faces through this layer: face elements (y-1 | y) x (layer)
            if (es.robin[F] == 0.0 || gx != (F ? g.n[0] : 0)) continue;
            const double hh = es.robin[F];
            if (gy >= 1) {
              const double* a4 = robin_aq(es.aq, g.n, F, gy - 1, gzd);
              robin_elem_row(a4, 1, 0, wd[j][1], wd[j + 1][1], wu[j][1], wu[j + 1][1], hh, ad, gdd);
              robin_elem_row(a4, 1, 1, wd[j][1], wd[j + 1][1], wu[j][1], wu[j + 1][1], hh, au, gdu);
            }
            if (gy < g.n[1]) {
              const double* a4 = robin_aq(es.aq, g.n, F, gy, gzd);
              robin_elem_row(a4, 0, 0, wd[j + 1][1], wd[j + 2][1], wu[j + 1][1], wu[j + 2][1], hh, ad, gdd);
              robin_elem_row(a4, 0, 1, wd[j + 1][1], wd[j + 2][1], wu[j + 1][1], wu[j + 2][1], hh, au, gdu);
            }
          }
        if (layer_ok)
          for (int F = 2; F < 4; ++F) {   // y faces through this layer: face elements (x-1 | x) x (layer)
            if (es.robin[F] == 0.0 || gy != (F == 3 ? g.n[1] : 0)) continue;
            const double hh = es.robin[F];
            if (gx >= 1) {
              const double* a4 = robin_aq(es.aq, g.n, F, gx - 1, gzd);
              robin_elem_row(a4, 1, 0, wd[j + 1][0], wd[j + 1][1], wu[j + 1][0], wu[j + 1][1], hh, ad, gdd);
              robin_elem_row(a4, 1, 1, wd[j + 1][0], wd[j + 1][1], wu[j + 1][0], wu[j + 1][1], hh, au, gdu);
            }
            if (gx < g.n[0]) {
              const double* a4 = robin_aq(es.aq, g.n, F, gx, gzd);
              robin_elem_row(a4, 0, 0, wd[j + 1][1], wd[j + 1][2], wu[j + 1][1], wu[j + 1][2], hh, ad, gdd);
              robin_elem_row(a4, 0, 1, wd[j + 1][1], wd[j + 1][2], wu[j + 1][1], wu[j + 1][2], hh, au, gdu);
            }
          }
        for (int F = 4; F < 6; ++F) {     // z face through plane d: the in-plane face elements (x-1 | x) x (y-1 | y)
          if (es.robin[F] == 0.0 || gzd != (F == 5 ? g.n[2] : 0)) continue;
          const double hh = es.robin[F];
          for (int sy = 0; sy < 2; ++sy)
            for (int sx = 0; sx < 2; ++sx) {
              const int ex = gx - 1 + sx, ey = gy - 1 + sy;
              if (ex < 0 || ex >= g.n[0] || ey < 0 || ey >= g.n[1]) continue;
              const double* a4 = robin_aq(es.aq, g.n, F, ex, ey);
              // element corners (ex, ey) .. (ex+1, ey+1) at window rows j+sy, j+sy+1 and columns sx, sx+1
              robin_elem_row(a4, 1 - sx, 1 - sy, wd[j + sy][sx], wd[j + sy][sx + 1], wd[j + sy + 1][sx],
                             wd[j + sy + 1][sx + 1], hh, ad, gdd);
            }
        }
        upd += ad;
        dnu += au;
        diag_d += gdd;
        diag_u += gdu;
      } else if (rare) {
        // Robin face mass: x- / y-faces through this layer, z-face of plane d (in-plane)
        double ad = 0.0, au = 0.0, gdg = 0.0;
        const int gy = gy0 + j;
        const double rx = (gx == 0 ? es.robin[0] : 0.0) + (gx == g.n[0] ? es.robin[1] : 0.0);
        const double ryj = (gy == 0 ? es.robin[2] : 0.0) + (gy == g.n[1] ? es.robin[3] : 0.0);
        const double cxm = gx >= 1 ? 1.0 : 0.0, cxp = gx < g.n[0] ? 1.0 : 0.0;
        const double cym = gy >= 1 ? 1.0 : 0.0, cyp = gy < g.n[1] ? 1.0 : 0.0;
        if (layer_ok && rx != 0.0) {   // face elements (y-1/2 | y+1/2) x (layer)
          const double cm = cym, cp = cyp, c2 = cm + cp;
          ad += rx * (c2 * (c9 * wd[j + 1][1] + c18 * wu[j + 1][1]) + cm * (c18 * wd[j][1] + c36 * wu[j][1]) +
                      cp * (c18 * wd[j + 2][1] + c36 * wu[j + 2][1]));
          au += rx * (c2 * (c9 * wu[j + 1][1] + c18 * wd[j + 1][1]) + cm * (c18 * wu[j][1] + c36 * wd[j][1]) +
                      cp * (c18 * wu[j + 2][1] + c36 * wd[j + 2][1]));
          gdg += rx * c2 * c9;
        }
        if (layer_ok && ryj != 0.0) {   // face elements (x-1/2 | x+1/2) x (layer)
          const double cm = cxm, cp = cxp, c2 = cm + cp;
          ad += ryj * (c2 * (c9 * wd[j + 1][1] + c18 * wu[j + 1][1]) + cm * (c18 * wd[j + 1][0] + c36 * wu[j + 1][0]) +
                         cp * (c18 * wd[j + 1][2] + c36 * wu[j + 1][2]));
          au += ryj * (c2 * (c9 * wu[j + 1][1] + c18 * wd[j + 1][1]) + cm * (c18 * wu[j + 1][0] + c36 * wd[j + 1][0]) +
                         cp * (c18 * wu[j + 1][2] + c36 * wd[j + 1][2]));
          gdg += ryj * c2 * c9;
        }
        diag_u += gdg;
        diag_d += gdg;
        if (rz != 0.0) {   // z-face through plane d: the in-plane elements (x+-1/2, y+-1/2)
          const double sx = cxm + cxp, sy = cym + cyp;
          ad += rz * (c9 * sx * sy * wd[j + 1][1] + c18 * (sy * (cxm * wd[j + 1][0] + cxp * wd[j + 1][2]) +
                                                            sx * (cym * wd[j][1] + cyp * wd[j + 2][1])) +
                      c36 * (cxm * cym * wd[j][0] + cxp * cym * wd[j][2] + cxm * cyp * wd[j + 2][0] +
                             cxp * cyp * wd[j + 2][2]));
          diag_d += rz * c9 * sx * sy;
        }
        upd += ad;
        dnu += au;
      }
      if (s >= 2 && own_ok[j]) {
        const double ap = part[j] + upd;
        const double diag = dpart[j] + diag_d;
        const double pc = wd[j + 1][1];
        const long long off = (long long)d * S + own_off[j];
        const int io = (RY * w + j) * TX + lane;
        if (MODE == MODE_K1) {
          acc0 = __fma_rn(pc, ap, acc0);
          a.o0[off] = pc;
        } else if (MODE == MODE_K2) {
          const double dinv = es.precond ? (diag > 0.0 ? __drcp_rn(diag) : 0.0) : 1.0;
          const double zk = XD == 1 ? I0[io] : I1[io];
          // r_k = D z_k: the residual is not stored on this path, only z = D^-1 r (reading R8)
          const double rk = es.precond ? diag * zk : zk;
          const double rn = __fma_rn(-alpha, ap, rk);
          const double zz = dinv * rn;
          acc0 = __fma_rn(rn, zz, acc0);
          acc1 = __fma_rn(rn, rn, acc1);
          if (XD == 0) a.o0[off] = __fma_rn(alpha, pc, I0[io]);
          if (XD == 2) a.o0[off] = __fma_rn(alpha, pc, __fma_rn(alpha0, I1[TX * TY + io], I0[io]));
          a.o2[off] = zz;
          if (d == g.zbeg && a.peer_lo) a.peer_lo[own_off[j]] = zz;      // fused halo exchange (z)
          if (d == g.zend - 1 && a.peer_hi) a.peer_hi[own_off[j]] = zz;
        } else if (MODE == MODE_INIT) {
          const double dinv = es.precond ? (diag > 0.0 ? __drcp_rn(diag) : 0.0) : 1.0;
          const double bv = I0[io];
          acc2 = __fma_rn(bv, bv, acc2);
          const double rn = bv - ap;
          const double zz = dinv * rn;
          acc0 = __fma_rn(rn, zz, acc0);
          acc1 = __fma_rn(rn, rn, acc1);
          a.o1[off] = zz;   // r itself is not stored (K2 forms r_k = D z_k)
          if (d == g.zbeg && a.peer_lo) a.peer_lo[own_off[j]] = zz;      // fused halo exchange (z)
          if (d == g.zend - 1 && a.peer_hi) a.peer_hi[own_off[j]] = zz;
        } else if (MODE == MODE_TRUE) {
          const double rn = I0[io] - ap;
          acc1 = __fma_rn(rn, rn, acc1);
          if (u_out) u_out[full_index(g, x, yb + j, d)] = pc;   // fused scatter of u_h
        } else {
          a.o0[off] = ap;
        }
      }
      part[j] = dnu;
      dpart[j] = diag_u;
    }
  };

  double wA[RY + 2][3], wB[RY + 2][3];
  for (int s = 0; s < nsteps; s += 2) {   // unrolled by two: the two plane windows swap roles
    step(s, wB, wA);
    if (s + 1 < nsteps) step(s + 1, wA, wB);
  }
#undef k0
#undef k1
#undef k2
#undef k3
#undef k4
#undef k5
#undef k6
#undef k7
}

// XD != 0 (K2 only): the slot of mH1 (K1's second halo vector, unused by K2) carries the interior map of p_{k-1}
template <int MODE, int NS, bool CUBE, int BF, int XD = 0>
__global__ void __launch_bounds__(NTH, ELEM_MINB)
    k_jcg_elem_tma(const LevelGeom g, const ElemStencil es, const KArgs a, const __grid_constant__ CUtensorMap mH0,
                   const __grid_constant__ CUtensorMap mH1, const __grid_constant__ CUtensorMap mE,
                   const __grid_constant__ CUtensorMap mI0, const __grid_constant__ CUtensorMap mI1) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[NS];
  // (offset from smem_raw, not a uintptr_t round trip: the pointer must stay in the shared window so
  // the reads compile to LDS, not generic LD)
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  JcgScalars* sc = a.sc;
  pdl_trigger();
  pdl_wait();
  if (MODE == MODE_K1 || MODE == MODE_K2) {
    if (*(volatile int*)&sc->done) return;
  }
  const int tid = threadIdx.x + TX * threadIdx.y;
  double bcg = 0.0, alpha = 0.0, alpha0 = 0.0;
  bool first = false;
  if (MODE == MODE_K1) { bcg = sc->beta; first = (sc->iter == 0); }
  if (MODE == MODE_K2) { alpha = sc->alpha; alpha0 = XD == 2 ? sc->alpha_prev : 0.0; }
  double* const u_out = (MODE == MODE_TRUE) ? sc->in.u_out : nullptr;
  // iteration 0 of K1 (p = z): the p_old slot is filled from z and beta_cg = 0 (exact for finite z), so
  // the window update is one FMA with no per-element select
  const double bcg_eff = first ? 0.0 : bcg;
  const CUtensorMap* pH1 = (MODE == MODE_K1 && first) ? &mH0 : &mH1;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // Work distribution: grid (x tiles, y tiles, z chunks of a.zc planes). All tiles of a z chunk march
  // side by side, so the halo rows / columns that neighbouring CTAs both read (boxes are 1.2-1.27x the
  // tile) are L2 hits. (Measured: giving each of 2 x 148 persistent CTAs an equal contiguous range of
  // the tile-major (tile, plane) space removes the partial last wave but de-phases neighbouring
  // tiles, and costs 40 % at 256^3: 0.444 vs 0.315 ms per iteration.)
  const int X0 = blockIdx.x * TX, Y0 = blockIdx.y * TY;
  const int z0 = g.zbeg + blockIdx.z * a.zc;
  const int z1 = min(z0 + a.zc, g.zend);
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  elem_pass<MODE, NS, CUBE, ElemCfg<MODE, XD>::SBYTES, BF, XD>(g, es, a, X0, Y0, z0, z1, bcg_eff, first, alpha, u_out, &mH0, pH1, &mE, &mI0, &mI1, smem, full,
                            0u, acc0, acc1, acc2, &mH1, alpha0);
  if ((MODE == MODE_K2 || MODE == MODE_INIT) && (a.peer_lo || a.peer_hi)) __threadfence_system();   // peer stores
  if (MODE != MODE_APPLY) reduce_finalize(MODE, a, acc0, acc1, acc2);
}

// ---- the whole JCG solve of a level in ONE cooperative launch (element path), as k_jcg_const_pers in
// kernels_jcg_tma.cu: each CTA owns a fixed list of (tile, z chunk) items and runs init -> { K1 pass,
// grid sum, K2 pass, grid sum } -> true residual with deterministic grid sums (every CTA reduces all
// partials in CTA order and holds the same CG scalars).
constexpr int EP_NS = 5;
constexpr int EP_SB = ElemCfg<MODE_K2>::SBYTES > ElemCfg<MODE_K1>::SBYTES ? ElemCfg<MODE_K2>::SBYTES : ElemCfg<MODE_K1>::SBYTES;
constexpr int EP_SMEM = EP_SB * EP_NS + 128;

struct ElemPersMaps { CUtensorMap xh, zh, ph0, ph1, be, xi, zi, bi; };

__device__ __forceinline__ void elem_grid_sum3(double v[3], double* partials, int& buf, double* red,
                                               cooperative_groups::grid_group& grid) {
  block_sum3(v[0], v[1], v[2], red);   // thread 0 holds the CTA sums
  const int tid = threadIdx.x + TX * threadIdx.y;
  double* pb = partials + (size_t)buf * gridDim.x * 3;
  if (tid == 0)
    for (int k = 0; k < 3; ++k) pb[3 * blockIdx.x + k] = v[k];
  grid.sync();
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (unsigned c = tid; c < gridDim.x; c += NTH) {
    s0 += __ldcg(pb + 3 * c);
    s1 += __ldcg(pb + 3 * c + 1);
    s2 += __ldcg(pb + 3 * c + 2);
  }
  block_sum3(s0, s1, s2, red);
  __shared__ double bc[3];
  if (tid == 0) { bc[0] = s0; bc[1] = s1; bc[2] = s2; }
  __syncthreads();
  v[0] = bc[0]; v[1] = bc[1]; v[2] = bc[2];
  __syncthreads();
  buf ^= 1;
}

#ifndef ELEM_PERS_MINB   // 2 CTAs / SM spill ~200 B per thread; 1 (no spills, half the CTAs) measured on C3:
#define ELEM_PERS_MINB ELEM_MINB   // 64^3 1.24 -> 1.15 ms but 128^3 4.72 -> 5.2 ms, TTS 40.4 -> 40.8 ms
#endif
template <bool CUBE, int BF>
__global__ void __launch_bounds__(NTH, ELEM_PERS_MINB)
    k_jcg_elem_pers(const LevelGeom g, const ElemStencil es, double* x, double* r, double* z, double* p0, double* p1,
                    double* partials, JcgScalars* sc, int zc, int ntx, int nty, int items,
                    const __grid_constant__ ElemPersMaps M) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[EP_NS];
  __shared__ double red[3 * (NTH / 32)];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int tid = threadIdx.x + TX * threadIdx.y;
  if (tid == 0) {
    for (int i = 0; i < EP_NS; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double eps = sc->in.eps;
  const int max_iter = sc->in.max_iter;
  double* const u_out = sc->in.u_out;
  uint32_t gstep = 0;
  int buf = 0;
  KArgs a{};
  auto pass = [&](auto mode_tag, const CUtensorMap* h0, const CUtensorMap* h1, const CUtensorMap* i0, const CUtensorMap* i1,
                  double bcg, bool first, double alpha, double v[3]) {
    constexpr int MODE = decltype(mode_tag)::value;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      const int X0 = (it % ntx) * TX, Y0 = ((it / ntx) % nty) * TY;
      const int z0 = (it / (ntx * nty)) * zc, z1 = min(z0 + zc, g.zend);
      elem_pass<MODE, EP_NS, CUBE, EP_SB, BF>(g, es, a, X0, Y0, z0, z1, bcg, first, alpha, u_out, h0, h1, &M.be, i0, i1, smem,
                                          full, gstep, acc0, acc1, acc2);
      gstep += (uint32_t)(z1 - z0 + 2);
      __syncthreads();   // every stage consumed before the next pass's prefill
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");   // stores read by other CTAs' TMA next pass
    v[0] = acc0; v[1] = acc1; v[2] = acc2;
    elem_grid_sum3(v, partials, buf, red, grid);
    if (tid == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
  };
  double v[3];
  a.o1 = z;   // init: r = b - A x, z = D^-1 r (stored), rho = r.z, rr, ||b||^2
  pass(std::integral_constant<int, MODE_INIT>{}, &M.xh, &M.xh, &M.bi, &M.bi, 0.0, false, 0.0, v);
  double rho = v[0], rr = v[1];
  const double bb = v[2];
  const double nb = sqrt(bb), nbe = nb > 0.0 ? nb : 1.0;
  const double thresh = eps > 0.0 ? eps * nbe : -1.0;
  int status = ST_OK, iter = 0;
  double beta = 0.0;
  bool done = (max_iter <= 0) || (thresh > 0.0 && !(sqrt(rr) > thresh));
  if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  int cur = 0;   // p_cur holds p_old
  while (!done) {
    a.o0 = cur ? p0 : p1;
    // iteration 0: p = z (the p_old slot is filled from z and beta_cg = 0, as in k_jcg_elem_tma)
    pass(std::integral_constant<int, MODE_K1>{}, &M.zh, iter == 0 ? &M.zh : (cur ? &M.ph1 : &M.ph0), &M.zh, &M.zh,
         iter == 0 ? 0.0 : beta, iter == 0, 0.0, v);
    const double sigma = v[0];
    if (!(sigma > 0.0)) { status = ST_EBREAKDOWN; break; }
    const double alpha = rho / sigma;
    a.o0 = x; a.o2 = z;
    pass(std::integral_constant<int, MODE_K2>{}, cur ? &M.ph0 : &M.ph1, &M.zh, &M.xi, &M.zi, 0.0, false, alpha, v);
    beta = v[0] / rho;
    rho = v[0];
    rr = v[1];
    cur ^= 1;
    ++iter;
    done = (iter >= max_iter) || (thresh > 0.0 && !(sqrt(rr) > thresh));
    if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  }
  pass(std::integral_constant<int, MODE_TRUE>{}, &M.xh, &M.xh, &M.bi, &M.bi, 0.0, false, 0.0, v);
  if (blockIdx.x == 0 && tid == 0) {
    sc->rho = rho; sc->rr = rr; sc->bb = bb; sc->rr_true = v[1]; sc->beta = beta;
    sc->iter = iter; sc->max_iter = max_iter; sc->thresh = thresh; sc->status = status; sc->done = 1;
    sc->counter = 0;
  }
}

template <int MODE, int NS, int XD = 0>
constexpr int elem_smem() { return ElemCfg<MODE, XD>::SBYTES * NS + 128; }

template <int MODE, int NS>
cudaError_t set_elem_tma_attr() {
  const int sm = elem_smem<MODE, NS>();
  cudaError_t e = cudaFuncSetAttribute(k_jcg_elem_tma<MODE, NS, false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_tma<MODE, NS, true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_tma<MODE, NS, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_tma<MODE, NS, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_tma<MODE, NS, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_tma<MODE, NS, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  return e;
}
// the deferred-x K2 variants exist for beta from the array only (BF = 0)
template <int NS, int XD>
cudaError_t set_elem_xd_attr() {
  const int sm = elem_smem<MODE_K2, NS, XD>();
  cudaError_t e = cudaFuncSetAttribute(k_jcg_elem_tma<MODE_K2, NS, false, 0, XD>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_tma<MODE_K2, NS, true, 0, XD>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  return e;
}
template <int NS, int XD>
cudaError_t launch_elem_k2_xd(const LevelGeom& g, const ElemStencil& es, const KArgs& a, const CUtensorMap* m, cudaStream_t st) {
  dim3 grid((g.nf[0] + TX - 1) / TX, (g.nf[1] + TY - 1) / TY, (g.zend - g.zbeg + a.zc - 1) / a.zc);
  count_launch();
  const int sm = elem_smem<MODE_K2, NS, XD>();
  const dim3 blk(TX, WARPS);
  if (es.cube) return launch_maybe_pdl(k_jcg_elem_tma<MODE_K2, NS, true, 0, XD>, grid, blk, sm, st, a.pdl, g, es, a, m[0], m[1], m[2], m[3], m[4]);
  return launch_maybe_pdl(k_jcg_elem_tma<MODE_K2, NS, false, 0, XD>, grid, blk, sm, st, a.pdl, g, es, a, m[0], m[1], m[2], m[3], m[4]);
}

// beta on the fly for cubic cells with the level's tables (ElemStencil::bkind >= 0): 1 = product kind
inline int beta_fly_variant(const ElemStencil& es) {
  if (!es.cube || es.bkind < 0 || !es.baxes) return 0;
  return es.bkind == BETA_KIND_C3 ? 1 : 2;
}

template <int MODE, int NS>
cudaError_t launch_elem_tma_mode(const LevelGeom& g, const ElemStencil& es, const KArgs& a, const CUtensorMap* m,
                                 cudaStream_t st) {
  dim3 grid((g.nf[0] + TX - 1) / TX, (g.nf[1] + TY - 1) / TY, (g.zend - g.zbeg + a.zc - 1) / a.zc);
  count_launch();
  const int sm = elem_smem<MODE, NS>();
  const dim3 blk(TX, WARPS);
  if (es.aq) {   // Robin alpha at the face Gauss points (ARRAYS)
    if (es.cube) return launch_maybe_pdl(k_jcg_elem_tma<MODE, NS, true, 3>, grid, blk, sm, st, a.pdl, g, es, a, m[0], m[1], m[2], m[3], m[4]);
    return launch_maybe_pdl(k_jcg_elem_tma<MODE, NS, false, 3>, grid, blk, sm, st, a.pdl, g, es, a, m[0], m[1], m[2], m[3], m[4]);
  }
  switch (es.cube ? 1 + beta_fly_variant(es) : 0) {
    case 1: return launch_maybe_pdl(k_jcg_elem_tma<MODE, NS, true, 0>, grid, blk, sm, st, a.pdl, g, es, a, m[0], m[1], m[2], m[3], m[4]);
    case 2: return launch_maybe_pdl(k_jcg_elem_tma<MODE, NS, true, 1>, grid, blk, sm, st, a.pdl, g, es, a, m[0], m[1], m[2], m[3], m[4]);
    case 3: return launch_maybe_pdl(k_jcg_elem_tma<MODE, NS, true, 2>, grid, blk, sm, st, a.pdl, g, es, a, m[0], m[1], m[2], m[3], m[4]);
    default: return launch_maybe_pdl(k_jcg_elem_tma<MODE, NS, false, 0>, grid, blk, sm, st, a.pdl, g, es, a, m[0], m[1], m[2], m[3], m[4]);
  }
}

// ---- tensor-map cache: (base, geometry, box) -> CUtensorMap; an entry is a pure function of its key
struct MapKey {
  const void* base;
  long long d0, d1, d2, s1, s2;
  int bx, by;
  bool operator==(const MapKey& o) const {
    return base == o.base && d0 == o.d0 && d1 == o.d1 && d2 == o.d2 && s1 == o.s1 && s2 == o.s2 && bx == o.bx &&
           by == o.by;
  }
};
struct MapEntry { MapKey k; CUtensorMap m; };
constexpr int kMapCache = 64;

bool encode_map(CUtensorMap* out, const MapKey& k) {
  static std::mutex mu;
  static MapEntry cache[kMapCache];
  static int used = 0, next = 0;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < used; ++i)
    if (cache[i].k == k) { *out = cache[i].m; return true; }
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return false;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[3] = {(cuuint64_t)k.d0, (cuuint64_t)k.d1, (cuuint64_t)k.d2};
  cuuint64_t strides[2] = {(cuuint64_t)k.s1 * 8, (cuuint64_t)k.s2 * 8};
  cuuint32_t box[3] = {(cuuint32_t)k.bx, (cuuint32_t)k.by, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap m;
  if (encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(k.base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, ECMG_TMA_PROMO,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  const int slot = used < kMapCache ? used++ : (next++ % kMapCache);
  cache[slot].k = k;
  cache[slot].m = m;
  *out = m;
  return true;
}

bool vec_map(CUtensorMap* m, const double* base, const LevelGeom& g, int bx, int by) {
  const MapKey k{base, g.nf[0], g.nf[1], g.nza, g.P, g.S, bx, by};
  return encode_map(m, k);
}
bool beta_map(CUtensorMap* m, const double* beta, const LevelGeom& g) {
  const MapKey k{beta, g.n[0] + 4, g.n[1] + 4, g.n[2] + 4, g.BP, g.BS, EBX, EBY};
  return encode_map(m, k);
}

}  // namespace

// ring depth per mode: two CTAs per SM (register bound) leave ~110 KB of shared memory each
#ifndef ELEM_NS_K1
#define ELEM_NS_K1 6
#endif
#ifndef ELEM_NS_K2
#define ELEM_NS_K2 5
#endif
#ifndef ELEM_NS_K2_SKIP
#define ELEM_NS_K2_SKIP 6
#endif
#ifndef ELEM_NS_K2_BOTH
#define ELEM_NS_K2_BOTH 4
#endif
constexpr int NS_K1 = ELEM_NS_K1, NS_K2 = ELEM_NS_K2, NS_OTHER = 4, NS_K2_SKIP = ELEM_NS_K2_SKIP, NS_K2_BOTH = ELEM_NS_K2_BOTH;

cudaError_t init_elem_kernel_attributes() {
  cudaError_t e = set_elem_tma_attr<MODE_K1, NS_K1>();
  if (e == cudaSuccess) e = set_elem_tma_attr<MODE_K2, NS_K2>();
  if (e == cudaSuccess) e = set_elem_tma_attr<MODE_INIT, NS_OTHER>();
  if (e == cudaSuccess) e = set_elem_tma_attr<MODE_TRUE, NS_OTHER>();
  if (e == cudaSuccess) e = set_elem_tma_attr<MODE_APPLY, NS_OTHER>();
  if (e == cudaSuccess) e = set_elem_xd_attr<NS_K2_SKIP, 1>();
  if (e == cudaSuccess) e = set_elem_xd_attr<NS_K2_BOTH, 2>();
  return e;
}

int elem_tile_rows() { return TY; }

static int elem_pers_slots() {
  static int slots = 0;
  if (!slots) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jcg_elem_pers<true, 0>, NTH, EP_SMEM);
    slots = sms * std::max(1, per_sm);
  }
  return slots;
}

int elem_pers_slots_count() { return elem_pers_slots(); }

bool elem_pers_fits(const LevelGeom& g) {
  const long long tiles = (long long)((g.nf[0] + TX - 1) / TX) * ((g.nf[1] + TY - 1) / TY);
  return g.BP % 2 == 0 && g.zbeg == 0 && tiles <= elem_pers_slots();
}

cudaError_t init_elem_pers_attributes() {
  cudaError_t e = cudaFuncSetAttribute(k_jcg_elem_pers<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, EP_SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_pers<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, EP_SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_pers<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, EP_SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_pers<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, EP_SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_pers<true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, EP_SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem_pers<false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, EP_SMEM);
  return e;
}

// the whole tolerance-stopped solve of an element-path level in one cooperative launch (single GPU)
cudaError_t launch_jcg_elem_pers(const LevelGeom& g, const ElemStencil& es, double* x, double* r, double* z, double* p0,
                                 double* p1, const double* b, const double* beta, double* partials, JcgScalars* sc,
                                 cudaStream_t st) {
  if (g.BP % 2 != 0 || g.zbeg != 0) return cudaErrorInvalidValue;
  const int ntx = (g.nf[0] + TX - 1) / TX, nty = (g.nf[1] + TY - 1) / TY;
  const int nz = g.zend - g.zbeg;
  const int slots = elem_pers_slots();
  const long long tiles = (long long)ntx * nty;
  if (tiles > slots) return cudaErrorInvalidValue;
  const int nch = (int)std::max(1LL, slots / tiles);
  const int zc = (nz + nch - 1) / nch;
  const int items = (int)(tiles * ((nz + zc - 1) / zc));
  ElemPersMaps M;
  const bool ok = vec_map(&M.xh, x, g, HX, HY) && vec_map(&M.zh, z, g, HX, HY) && vec_map(&M.ph0, p0, g, HX, HY) &&
                  vec_map(&M.ph1, p1, g, HX, HY) && beta_map(&M.be, beta, g) && vec_map(&M.xi, x, g, TX, TY) &&
                  vec_map(&M.zi, z, g, TX, TY) && vec_map(&M.bi, b, g, TX, TY);
  if (!ok) return cudaErrorInvalidValue;
  const int grid = std::min(items, slots);
  void* args[] = {(void*)&g, (void*)&es, (void*)&x, (void*)&r, (void*)&z, (void*)&p0, (void*)&p1, (void*)&partials,
                  (void*)&sc, (void*)&zc, (void*)&ntx, (void*)&nty, (void*)&items, (void*)&M};
  count_launch();
  const void* fn = (const void*)k_jcg_elem_pers<false, 0>;
  if (es.aq) fn = es.cube ? (const void*)k_jcg_elem_pers<true, 3> : (const void*)k_jcg_elem_pers<false, 3>;
  else switch (es.cube ? 1 + beta_fly_variant(es) : 0) {
    case 1: fn = (const void*)k_jcg_elem_pers<true, 0>; break;
    case 2: fn = (const void*)k_jcg_elem_pers<true, 1>; break;
    case 3: fn = (const void*)k_jcg_elem_pers<true, 2>; break;
    default: break;
  }
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(TX, WARPS), args, EP_SMEM, st);
}

// K1: h0 = z, h1 = p_old, o0 = p. K2: h0 = p, i0 = x, i1 = z, o0 = x, o2 = z.
// INIT: h0 = x, i0 = b, o1 = z. TRUE: h0 = x, i0 = b. APPLY: h0 = p, o0 = A p.
cudaError_t launch_jcg_elem(int mode, const LevelGeom& g, const ElemStencil& es, const Problem&, const KArgs& a,
                            cudaStream_t st) {
  if (g.BP % 2 != 0 || !a.h0 || !a.beta) return cudaErrorInvalidValue;
  CUtensorMap m[5];
  bool ok = vec_map(&m[0], a.h0, g, HX, HY) && beta_map(&m[2], a.beta, g);
  m[1] = m[0];
  m[3] = m[0];
  m[4] = m[0];
  if (ok && mode == MODE_K1) ok = a.h1 && vec_map(&m[1], a.h1, g, HX, HY);
  if (ok && (mode == MODE_K2 || mode == MODE_INIT || mode == MODE_TRUE)) ok = a.i0 && vec_map(&m[3], a.i0, g, TX, TY);
  if (ok && mode == MODE_K2) ok = a.i1 && vec_map(&m[4], a.i1, g, TX, TY);
  // deferred x update (KArgs::xdefer; beta from the array, no alpha_q): 1 = the one interior box is z;
  // 2 = x, z and p_{k-1} (its interior map rides in the slot of K1's second halo vector)
  const bool xd = mode == MODE_K2 && a.xdefer && !es.aq && !(es.cube && beta_fly_variant(es));
  if (ok && xd && a.xdefer == 1) m[3] = m[4];
  if (ok && xd && a.xdefer == 2) ok = a.i2 && vec_map(&m[1], a.i2, g, TX, TY);
  if (!ok) return cudaErrorInvalidValue;
  if (xd) return a.xdefer == 1 ? launch_elem_k2_xd<NS_K2_SKIP, 1>(g, es, a, m, st) : launch_elem_k2_xd<NS_K2_BOTH, 2>(g, es, a, m, st);
  switch (mode) {
    case MODE_K1: return launch_elem_tma_mode<MODE_K1, NS_K1>(g, es, a, m, st);
    case MODE_K2: return launch_elem_tma_mode<MODE_K2, NS_K2>(g, es, a, m, st);
    case MODE_INIT: return launch_elem_tma_mode<MODE_INIT, NS_OTHER>(g, es, a, m, st);
    case MODE_TRUE: return launch_elem_tma_mode<MODE_TRUE, NS_OTHER>(g, es, a, m, st);
    case MODE_APPLY: return launch_elem_tma_mode<MODE_APPLY, NS_OTHER>(g, es, a, m, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ecmg
