// kernels_exp.cu -- the level-to-level extrapolation operators of Alg. 4.
//
// EXP_finite (l.6; §4.3), two passes:
//  (1) k_exp_seeds, one thread per 2h node: the extrapolated value of the 2h node in its 4h block --
//      corners (5U^1-U^0)/4 (Eq. jiedian), edge midpoints
//      U^1_m + (U^1_a-U^0_a+U^1_b-U^0_b)/8 along the edge (Eq. zhongdian), face and cell
//      centres the mean of Eq. (zhongdian) over the face / space diagonals (Remark 2, P:513-516;
//      used by the Lagrange variant only). Every value depends only on its own edge / face / cell,
//      so it is the same for all 4h blocks sharing it.
//  (2) k_exp_interp, one thread per (4h block bx, fine row y, fine plane z), 4 fine nodes along x
//      (5 in the last block): with eta, zeta fixed per thread, the interpolant is collapsed to a
//      few per-row coefficients and each node costs ~5 FMAs.
//      variant 0 (default): 20-node tri-quadratic Serendipity in its blending form
//        W = P_x + P_y + P_z - 2T (P_d: quadratic along the 4 d-edges blended bilinearly across
//        them, T: trilinear in the corners). It lies in the 20-dim Serendipity space and
//        interpolates the 20 seeds, hence equals sum_i N_i W_i of Eq. (inter).
//      variant 1 (Remark 2): tri-quadratic Lagrange through the 27 values.
// Owner block of fine node i: b = min(i/4, n_4h - 1) per axis (reading §8c A14). Dirichlet nodes
// take g_D (§8c A15). Output either the full nodal vector or, inside ecmg_run, straight into the
// free-box work vector of the next JCG solve.
//
// EXP_true (l.10): u~ = u_h + (1/3) I_trilinear(u_h|_2h - u_2h), which equals
// Eq. (t1) at 2h nodes, Eq. (chenlin) at 2h edge centres and the mean of Eq. (chenlin) over the
// 2 face diagonals / 4 space diagonals at face / cell centres (reading §8c A13; derived identity,
// DESIGN.md). A z-march over 64 x 8 fine tiles (coalesced rows) with the corner differences of two 2h
// planes in shared memory. Dirichlet nodes take g_D (A15) from the face kernel launched after the full-layout
// outputs (launch_dirichlet_fill), so that no g_D evaluation sits in the marching loops.
#include <algorithm>
#include "ecmg_internal.cuh"
#include "problems.cuh"

namespace ecmg {
namespace {

// (1) extrapolated values at all 2h nodes of the fine level gf (2h grid: n/2 cells per axis)
__global__ void k_exp_seeds(const LevelGeom gf, const double* __restrict__ u2h, const double* __restrict__ u4h,
                            double* __restrict__ S, int variant, int K0) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y, K = K0 + blockIdx.z;
  const int n2x = gf.n[0] / 2, n2y = gf.n[1] / 2;
  if (I > n2x) return;
  const long long nn2x = n2x + 1, nn2y = n2y + 1;
  const long long nn4x = gf.n[0] / 4 + 1, nn4y = gf.n[1] / 4 + 1;
  auto U1 = [&](int i, int j, int k) { return __ldg(u2h + i + nn2x * (j + nn2y * (long long)k)); };
  auto U0 = [&](int i, int j, int k) { return __ldg(u4h + (i >> 1) + nn4x * ((j >> 1) + nn4y * (long long)(k >> 1))); };
  auto D = [&](int i, int j, int k) { return U1(i, j, k) - U0(i, j, k); };   // at 4h-coincident 2h nodes
  const int odd[3] = {I & 1, J & 1, K & 1};
  const int nodd = odd[0] + odd[1] + odd[2];
  double v = 0.0;
  if (nodd == 0) {
    v = (5.0 * U1(I, J, K) - U0(I, J, K)) / 4.0;                           // Eq. (jiedian)
  } else if (nodd == 1) {
    const int dx = odd[0], dy = odd[1], dz = odd[2];
    v = U1(I, J, K) + (D(I - dx, J - dy, K - dz) + D(I + dx, J + dy, K + dz)) / 8.0;   // Eq. (zhongdian)
  } else if (variant == 1) {
    // face / cell centre: mean of Eq. (zhongdian) over the diagonals through the node (Remark 2)
    double sum = 0.0;
    // explicit enumeration of the 2 (face) or 4 (cell) diagonals
    int ax[3], na = 0;
    for (int d = 0; d < 3; ++d) if (odd[d]) ax[na++] = d;
    const int nseg = 1 << (na - 1);
    for (int sgn = 0; sgn < nseg; ++sgn) {
      int oa[3] = {0, 0, 0};
      oa[ax[0]] = -1;
      for (int t = 1; t < na; ++t) oa[ax[t]] = ((sgn >> (t - 1)) & 1) ? -1 : 1;
      sum += U1(I, J, K) + (D(I + oa[0], J + oa[1], K + oa[2]) + D(I - oa[0], J - oa[1], K - oa[2])) / 8.0;
    }
    v = sum / nseg;
  }
  S[I + nn2x * (J + nn2y * (long long)K)] = v;
}

// 1D quadratic (nodes t = -1, 0, 1) and linear weights at the five natural coordinates xi = (l-2)/2
__device__ __forceinline__ void quad_w(int l, double q[3]) {
  const double t = (l - 2) * 0.5;
  q[0] = t * (t - 1.0) * 0.5; q[1] = 1.0 - t * t; q[2] = t * (t + 1.0) * 0.5;
}
__device__ __forceinline__ void lin_w(int l, double w[2]) {
  const double t = (l - 2) * 0.5;
  w[0] = (1.0 - t) * 0.5; w[1] = (1.0 + t) * 0.5;
}

// (2) interpolation. FREEBOX: write the free nodes into the pitched free-box vector x, else the
// full nodal vector w (with g_D on Dirichlet nodes).
template <bool FREEBOX>
__global__ void __launch_bounds__(64) k_exp_interp(const LevelGeom gf, const Problem pb, const double* __restrict__ S,
                                                   double* __restrict__ out, int variant, int F0) {
  // one thread per (4h block bx, 4h block row by, fine plane fz): the 27 seeds are loaded once and
  // reused for the 4 (5 in the last block row) fine rows of the block and 4 (5) nodes per row
  const int n4x = gf.n[0] / 4, n4y = gf.n[1] / 4, n4z = gf.n[2] / 4;
  const int bx = blockIdx.x * blockDim.x + threadIdx.x, by = blockIdx.y, fz = F0 + blockIdx.z;
  if (bx >= n4x) return;
  const int bz = min(fz / 4, n4z - 1);
  const int lz = fz - 4 * bz;
  const long long nn2x = gf.n[0] / 2 + 1, nn2y = gf.n[1] / 2 + 1;
  double s[3][3][3];   // [k][j][i] seeds of block (bx, by, bz)
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int i = 0; i < 3; ++i)
        s[k][j][i] = __ldg(S + (2 * bx + i) + nn2x * ((2 * by + j) + nn2y * (long long)(2 * bz + k)));
  double qz[3], lz2[2];
  quad_w(lz, qz); lin_w(lz, lz2);
  const int nl = (bx == n4x - 1) ? 5 : 4;
  const int nrow = (by == n4y - 1) ? 5 : 4;
  const long long nx = gf.n[0] + 1, ny = gf.n[1] + 1;
  const bool plane_free = fz >= gf.flo[2] && fz < gf.flo[2] + gf.nf[2];
  for (int ly = 0; ly < nrow; ++ly) {
    const int fy = 4 * by + ly;
    double qy[3], ly2[2];
    quad_w(ly, qy); lin_w(ly, ly2);
    // per-row coefficients: W(xi) = sum_i qx_i(xi) C[i] + sum_a lx_a(xi) E[a]
    double C[3], E[2];
    if (variant == 1) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) t += qz[k] * (qy[0] * s[k][0][i] + qy[1] * s[k][1][i] + qy[2] * s[k][2][i]);
        C[i] = t;
      }
      E[0] = E[1] = 0.0;
    } else {
#pragma unroll
      for (int i = 0; i < 3; ++i)   // P_x: x-edges at (y, z) in {0,2}^2 blended bilinearly
        C[i] = ly2[0] * (lz2[0] * s[0][0][i] + lz2[1] * s[2][0][i]) + ly2[1] * (lz2[0] * s[0][2][i] + lz2[1] * s[2][2][i]);
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int A = 2 * a;
        const double Py = lz2[0] * (qy[0] * s[0][0][A] + qy[1] * s[0][1][A] + qy[2] * s[0][2][A]) +
                          lz2[1] * (qy[0] * s[2][0][A] + qy[1] * s[2][1][A] + qy[2] * s[2][2][A]);
        const double Pz = ly2[0] * (qz[0] * s[0][0][A] + qz[1] * s[1][0][A] + qz[2] * s[2][0][A]) +
                          ly2[1] * (qz[0] * s[0][2][A] + qz[1] * s[1][2][A] + qz[2] * s[2][2][A]);
        const double T = ly2[0] * (lz2[0] * s[0][0][A] + lz2[1] * s[2][0][A]) + ly2[1] * (lz2[0] * s[0][2][A] + lz2[1] * s[2][2][A]);
        E[a] = Py + Pz - 2.0 * T;
      }
    }
    const bool row_free = plane_free && fy >= gf.flo[1] && fy < gf.flo[1] + gf.nf[1];
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      if (l >= nl) break;
      const int fx = 4 * bx + l;
      double qx[3], lx[2];
      quad_w(l, qx); lin_w(l, lx);
      double W = qx[0] * C[0] + qx[1] * C[1] + qx[2] * C[2] + lx[0] * E[0] + lx[1] * E[1];
      const bool fr = row_free && fx >= gf.flo[0] && fx < gf.flo[0] + gf.nf[0];
      if (FREEBOX) {
        if (fr) out[(long long)(fz - gf.flo[2] - gf.zoff) * gf.S + (long long)(fy - gf.flo[1]) * gf.P + (fx - gf.flo[0])] = W;
      } else {
        out[(long long)fx + nx * ((long long)fy + ny * fz)] = W;   // Dirichlet nodes: launch_exp_finite's face fill
      }
    }
  }
}

// (1+2) fused: EXP_finite as one z-march over 4h block layers, evaluated SEPARABLY. A CTA owns XB x YB 4h
// blocks in (x, y) (64 x 8 fine nodes, plus the domain's last node row / column) and a chunk of 4h layers.
// Per layer it stages the three 2h planes of u_2h and the two 4h planes of u_4h it touches in shared memory
// and forms there the values at all 27 2h nodes of every block:
//   * corners and edge midpoints: Eq. (jiedian) / Eq. (zhongdian), k_exp_seeds' expressions;
//   * face and cell centres: variant 0 (Serendipity) the value of the 20-node interpolant W there -- face
//     centre = 1/2 (its 4 edge midpoints) - 1/4 (its 4 corners), cell centre = 1/4 (12 midpoints) - 1/4 (8
//     corners) (pinned for the oracle in tests/test_oracle_exp.py); variant 1 (Remark 2,
//     P:513-516) the mean of Eq. (zhongdian) over the diagonals.
// The 20-node Serendipity space lies inside the tri-quadratic space Q2, so W equals the Q2
// Lagrange interpolant of its own 27 values; with the centres filled that way both variants are the
// tensor-product quadratic interpolation of the 27 values, applied axis by axis: along x into XS (fine x,
// 2h y, 2h z), then, per thread (fine column x, fine plane z), along z to the five 2h rows and along y to
// the eight fine rows, stored with coalesced row stores. Every per-node index map (which 2h node a thread
// forms, from which staged values) is fixed per thread and computed once before the z-march. HBM traffic:
// the fine level written once (8 B / node) plus ~1/8 + 1/64 of it read. Results equal the two-pass blending
// evaluation (k_exp_seeds + k_exp_interp) to rounding (tests/test_gpu_parity.py).
#ifndef EXP_YB
#define EXP_YB 2
#endif
constexpr int XB = 16, YB = EXP_YB;                            // 4h blocks per tile
constexpr int FXT = 4 * XB + 1, FYT = 4 * YB + 1;              // fine nodes per tile incl. the last node
constexpr int S2X = 2 * XB + 1, S2Y = 2 * YB + 1;              // 2h nodes per tile plane
constexpr int FNTH = 256;
constexpr int N1 = 3 * S2Y * S2X, N0 = 2 * (YB + 1) * (XB + 1);   // staged u_2h / u_4h values per layer
constexpr int NQ = (N1 + FNTH - 1) / FNTH;                        // u_2h values (and 2h nodes) per thread
constexpr int NCK1 = S2Y * S2X - (YB + 1) * (XB + 1), NCK0 = YB * XB;   // face / cell centres (k = 1; k = 0, 2)
constexpr int NCQ = (NCK1 + 2 * NCK0 + FNTH - 1) / FNTH;
static_assert(FNTH == 4 * 64 && FXT == 65, "thread map: (fine column, fine plane) = (tid & 63, tid >> 6)");
static_assert(N0 <= FNTH && N1 < 1024, "per-thread maps");

// 1D quadratic through the 2h nodes (t = -1, 0, 1) of a 4h block at fine offset l = 0..4 (t = (l - 2) / 2)
__device__ __forceinline__ void q2w(int l, double& w0, double& w1, double& w2) {
  w0 = (l == 0) ? 1.0 : (l == 1) ? 0.375 : (l == 3) ? -0.125 : 0.0;
  w1 = (l == 2) ? 1.0 : (l == 1 || l == 3) ? 0.75 : 0.0;
  w2 = (l == 4) ? 1.0 : (l == 1) ? -0.125 : (l == 3) ? 0.375 : 0.0;
}

// flat index of tile-local 2h node (i, j, k) in U1s / Ss, and of tile-local 4h node (i, j, k) in U0s
__device__ __forceinline__ int f2(int i, int j, int k) { return i + S2X * (j + S2Y * k); }
__device__ __forceinline__ int f4(int i, int j, int k) { return i + (XB + 1) * (j + (YB + 1) * k); }

template <bool FREEBOX, int VARIANT>
#ifndef EXP_FUSED_MINB
#define EXP_FUSED_MINB 4   // 64 registers, 4 CTAs / SM: 512^3 in-run 0.387 -> 0.369 ms (3 CTAs: 0.387; 5: spills, 0.434)
#endif
__global__ void __launch_bounds__(FNTH, EXP_FUSED_MINB) k_exp_fused(const LevelGeom gf, const double* __restrict__ u2h,
                                                                    const double* __restrict__ u4h, double* __restrict__ out,
                                                                    int F0, int F1, int bzA, int lchunk) {
  __shared__ double U1s[N1];                   // u_2h on 2h planes 2bz .. 2bz+2 (f2 layout)
  __shared__ double U0s[N0];                   // u_4h on 4h planes bz, bz+1 (f4 layout)
  __shared__ double Ss[N1];                    // the 27 values of every block of the layer (f2 layout)
  __shared__ double XS[3][S2Y][FXT];           // ... interpolated along x: (fine x, 2h y, 2h z)
  const int tid = threadIdx.x;
  const int n4x = gf.n[0] / 4, n4y = gf.n[1] / 4, n4z = gf.n[2] / 4;
  const int n2x = gf.n[0] / 2, n2y = gf.n[1] / 2;
  const int nn2x = n2x + 1, nn2y = n2y + 1, nn4x = n4x + 1, nn4y = n4y + 1;
  const int bx0 = blockIdx.x * XB, by0 = blockIdx.y * YB;
  const int nbx = min(XB, n4x - bx0), nby = min(YB, n4y - by0);   // blocks in this tile
  const int X0 = 4 * bx0, Y0 = 4 * by0;
  const int nfx = 4 * nbx + (bx0 + nbx == n4x ? 1 : 0);          // fine nodes of the tile along x
  const int nfy = 4 * nby + (by0 + nby == n4y ? 1 : 0);
  const long long nx = gf.n[0] + 1, ny = gf.n[1] + 1;
  const int bzs = bzA + blockIdx.z * lchunk, bze = min(bzs + lchunk, n4z);
  const long long pl2 = (long long)nn2x * nn2y, pl4 = (long long)nn4x * nn4y;
  const double* u2t = u2h + 2 * bx0 + (long long)nn2x * 2 * by0;   // the tile's corner on 2h plane 0
  const double* u4t = u4h + bx0 + (long long)nn4x * by0;
  // ---- per-thread maps, fixed for the whole z-march ------------------------------------------------------
  // staging: u_2h values t = tid + 256 q (f2 order) at offset i + nn2x (j + nn2y k) from the layer's corner
  // (-1: outside the domain / tile); the u_4h value tid likewise
  int so1[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int t = tid + q * FNTH;
    const int i = t % S2X, j = (t / S2X) % S2Y, k = t / (S2X * S2Y);
    so1[q] = (t < N1 && 2 * bx0 + i <= n2x && 2 * by0 + j <= n2y) ? i + nn2x * (j + nn2y * k) : -1;
  }
  int so0;
  {
    const int i = tid % (XB + 1), j = (tid / (XB + 1)) % (YB + 1), k = tid / ((XB + 1) * (YB + 1));
    so0 = (tid < N0 && bx0 + i <= n4x && by0 + j <= n4y) ? i + nn4x * (j + nn4y * k) : -1;
  }
  // 2h-node values of nodes t = tid + 256 q, packed: kind (bits 0-1: 0 corner, 1 edge midpoint, 2 centre),
  // stride of the midpoint's odd axis (bits 2-11), its two 4h-coincident ends in U0s (bits 12-20, 21-29; a
  // corner: its own 4h node in bits 12-20)
  int sm[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int t = min(tid + q * FNTH, N1 - 1);
    const int i = t % S2X, j = (t / S2X) % S2Y, k = t / (S2X * S2Y);
    const int oi = i & 1, oj = j & 1, ok = k & 1, nodd = oi + oj + ok;
    const int kind = nodd == 0 ? 0 : nodd == 1 ? 1 : 2;
    const int a = nodd == 0 ? f4(i >> 1, j >> 1, k >> 1) : f4((i - oi) >> 1, (j - oj) >> 1, (k - ok) >> 1);
    const int b = f4((i + oi) >> 1, (j + oj) >> 1, (k + ok) >> 1);
    sm[q] = kind | (f2(oi, oj, ok) << 2) | (a << 12) | (b << 21);
  }
  // Serendipity face / cell centres (VARIANT 0): nodes c = tid + 256 q of the tile's 2h nodes with >= 2 odd
  // indices (k = 1: i or j odd; k = 0, 2: i and j odd), packed: node (bits 0-9), strides e, f of its two odd
  // axes (bits 10-19, 20-29; a face centre), bit 30 = cell centre; -1 = none
  int cm[NCQ];
#pragma unroll
  for (int q = 0; q < NCQ; ++q) {
    cm[q] = -1;
    int c = tid + q * FNTH;
    if (VARIANT != 0) continue;
    if (c < NCK1) {
      int i = 0, j = 0, m = c;
      for (j = 0; j < S2Y; ++j) {
        const int cnt = (j & 1) ? S2X : XB;   // odd row: every node; even row: odd i only
        if (m < cnt) { i = (j & 1) ? m : 2 * m + 1; break; }
        m -= cnt;
      }
      const int cell = (i & 1) && (j & 1);
      const int e = (i & 1) ? f2(1, 0, 0) : f2(0, 1, 0);
      const int f = cell ? 0 : f2(0, 0, 1);
      cm[q] = f2(i, j, 1) | (e << 10) | (f << 20) | (cell << 30);
    } else if (c < NCK1 + 2 * NCK0) {
      c -= NCK1;
      const int k = 2 * (c / NCK0), m = c % NCK0;
      cm[q] = f2(2 * (m % XB) + 1, 2 * (m / XB) + 1, k) | (f2(1, 0, 0) << 10) | (f2(0, 1, 0) << 20);
    }
  }
  // x pass: lane lx of a line reads 2h nodes xb .. xb+2 with weights (wx0, wx1, wx2) -- a unit weight on an
  // even (2h-coincident) column, so those are copied exactly, and xb kept inside the line
  const int lx = tid & 63, lzt = tid >> 6;
  int xb;
  double wx0, wx1, wx2;
  {
    const int m = lx >> 1;
    if (lx & 1) { xb = (lx & 2) ? m - 1 : m; q2w(lx & 3, wx0, wx1, wx2); }
    else { xb = min(m, S2X - 3); wx0 = (m == xb) ? 1.0 : 0.0; wx1 = (m == xb + 1) ? 1.0 : 0.0; wx2 = 0.0; }
  }
  double wz0, wz1, wz2;
  q2w(lzt, wz0, wz1, wz2);
  // rows of the tile inside the free box (FREEBOX output)
  const int rlo = FREEBOX ? max(0, gf.flo[1] - Y0) : 0;
  const int rhi = FREEBOX ? min(nfy, gf.flo[1] + gf.nf[1] - Y0) : nfy;
  const long long rstride = FREEBOX ? gf.P : nx;
  // one fine column (x = X0 + cx) of fine plane fz0 + cz: along z to the five 2h rows, along y to the rows
  auto column = [&](int cx, int cz, double a0, double a1, double a2, int fz0) {
    double Z[S2Y];
#pragma unroll
    for (int j = 0; j < S2Y; ++j) Z[j] = a0 * XS[0][j][cx] + a1 * XS[1][j][cx] + a2 * XS[2][j][cx];
    const int fx = X0 + cx, fz = fz0 + cz;
    if (FREEBOX && !(fz >= gf.flo[2] && fz < gf.flo[2] + gf.nf[2] && fx >= gf.flo[0] && fx < gf.flo[0] + gf.nf[0])) return;
    double* o = FREEBOX ? out + (long long)(fz - gf.flo[2] - gf.zoff) * gf.S + (long long)(Y0 - gf.flo[1]) * gf.P + (fx - gf.flo[0])
                        : out + fx + nx * ((long long)Y0 + ny * fz);
#pragma unroll
    for (int r = 0; r < FYT; ++r) {
      const int b = 2 * (r >> 2), l = r & 3;   // row 8 (the domain's last): 2h row 4
      double W;
      if (l == 0) W = Z[b];
      else if (l == 2) W = Z[b + 1];
      else if (l == 1) W = 0.375 * Z[b] + 0.75 * Z[b + 1] - 0.125 * Z[b + 2];
      else W = -0.125 * Z[b] + 0.75 * Z[b + 1] + 0.375 * Z[b + 2];
      if (r >= rlo && r < rhi) o[r * rstride] = W;   // full output: Dirichlet nodes by launch_exp_finite's face fill
    }
  };
  double r1[NQ], r0 = 0.0;
  // the next layer's first u_2h / u_4h planes, advanced by one 4h layer per fetch (loop-carried: the per-thread
  // offsets above are 32-bit, the layer bases uniform)
  const double* b2 = u2t + 2LL * bzs * pl2;
  const double* b4 = u4t + (long long)bzs * pl4;
  auto fetch = [&]() {
#pragma unroll
    for (int q = 0; q < NQ; ++q) r1[q] = so1[q] >= 0 ? __ldg(b2 + so1[q]) : 0.0;
    r0 = so0 >= 0 ? __ldg(b4 + so0) : 0.0;
    b2 += 2 * pl2;
    b4 += pl4;
  };
  if (bzs < bze) fetch();
  for (int bz = bzs; bz < bze; ++bz) {
    const int fz0 = 4 * bz, nfz = (bz == n4z - 1) ? 5 : 4;
    const int pz0 = max(fz0, F0), pz1 = min(fz0 + nfz, F1);   // fine planes of this layer to write
    __syncthreads();   // previous layer's tiles consumed
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (tid + q * FNTH < N1) U1s[tid + q * FNTH] = r1[q];
    if (tid < N0) U0s[tid] = r0;
    if (bz + 1 < bze) fetch();   // next layer's loads in flight during this layer's work
    __syncthreads();
    if (pz0 >= pz1) continue;
    // the 2h-node values
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int t = tid + q * FNTH;
      if (t >= N1) break;
      const int kind = sm[q] & 3, se = (sm[q] >> 2) & 1023, ua = (sm[q] >> 12) & 511, ub = (sm[q] >> 21) & 511;
      double v = 0.0;
      if (kind == 0) {
        v = (5.0 * U1s[t] - U0s[ua]) / 4.0;                                               // Eq. (jiedian)
      } else if (kind == 1) {
        v = U1s[t] + ((U1s[t - se] - U0s[ua]) + (U1s[t + se] - U0s[ub])) / 8.0;           // Eq. (zhongdian)
      } else if (VARIANT == 1) {   // Remark 2: mean of Eq. (zhongdian) over the diagonals through the node
        const int i = t % S2X, j = (t / S2X) % S2Y, k = t / (S2X * S2Y);
        const int odd[3] = {i & 1, j & 1, k & 1};
        auto D = [&](int a, int b, int c) { return U1s[f2(a, b, c)] - U0s[f4(a >> 1, b >> 1, c >> 1)]; };
        double sum = 0.0;
        int ax[3], na = 0;
        for (int d = 0; d < 3; ++d) if (odd[d]) ax[na++] = d;
        const int nseg = 1 << (na - 1);
        for (int sgn = 0; sgn < nseg; ++sgn) {
          int oa[3] = {0, 0, 0};
          oa[ax[0]] = -1;
          for (int qq = 1; qq < na; ++qq) oa[ax[qq]] = ((sgn >> (qq - 1)) & 1) ? -1 : 1;
          sum += U1s[t] + (D(i + oa[0], j + oa[1], k + oa[2]) + D(i - oa[0], j - oa[1], k - oa[2])) / 8.0;
        }
        v = sum / nseg;
      }
      Ss[t] = v;   // outside the tile's blocks: finite, never used with a nonzero weight
    }
    __syncthreads();
    if (VARIANT == 0) {   // Serendipity: the face and cell centres from the block's corners and midpoints
#pragma unroll
      for (int q = 0; q < NCQ; ++q) {
        if (cm[q] < 0) continue;
        const int ct = cm[q] & 1023;
        double v;
        if (!(cm[q] >> 30)) {   // face centre: midpoints at +-e, +-f, corners at +-e+-f
          const int ce = (cm[q] >> 10) & 1023, cf = (cm[q] >> 20) & 1023;
          const double mids = Ss[ct + ce] + Ss[ct - ce] + Ss[ct + cf] + Ss[ct - cf];
          const double corn = Ss[ct + ce + cf] + Ss[ct + ce - cf] + Ss[ct - ce + cf] + Ss[ct - ce - cf];
          v = 0.5 * mids - 0.25 * corn;
        } else {                // cell centre
          constexpr int X = 1, Y = S2X, Zs = S2X * S2Y;
          const double mids = Ss[ct + Y + Zs] + Ss[ct - Y + Zs] + Ss[ct + Y - Zs] + Ss[ct - Y - Zs] +
                              Ss[ct + X + Zs] + Ss[ct - X + Zs] + Ss[ct + X - Zs] + Ss[ct - X - Zs] +
                              Ss[ct + X + Y] + Ss[ct - X + Y] + Ss[ct + X - Y] + Ss[ct - X - Y];
          const double corn = Ss[ct + X + Y + Zs] + Ss[ct - X + Y + Zs] + Ss[ct + X - Y + Zs] + Ss[ct - X - Y + Zs] +
                              Ss[ct + X + Y - Zs] + Ss[ct - X + Y - Zs] + Ss[ct + X - Y - Zs] + Ss[ct - X - Y - Zs];
          v = 0.25 * mids - 0.25 * corn;
        }
        Ss[ct] = v;   // reads only nodes with at most one odd index: no race with the writes
      }
      __syncthreads();
    }
    // along x: XS[k][j][x] for the 3 x S2Y lines, lanes = fine columns 0..63, column 64 by a few threads
#pragma unroll
    for (int q = 0; q < (3 * S2Y + 3) / 4; ++q) {
      const int line = lzt + 4 * q;
      if (line < 3 * S2Y) {
        const double* sl = Ss + line * S2X;
        (&XS[0][0][0])[line * FXT + lx] = wx0 * sl[xb] + wx1 * sl[xb + 1] + wx2 * sl[xb + 2];
      }
    }
    if (tid < 3 * S2Y) (&XS[0][0][0])[tid * FXT + 64] = Ss[tid * S2X + 2 * XB];
    __syncthreads();
    const int lzs = pz0 - fz0, lze = pz1 - fz0;   // planes of the layer to produce
    if (lx < nfx && lzt >= lzs && lzt < lze) column(lx, lzt, wz0, wz1, wz2, fz0);
    // extras: column 64 (the domain's last node column) for planes 0..3, plane 4 (the domain's last plane)
    const int nA = (nfx > 64) ? 4 : 0, nC = (lze > 4) ? nfx : 0;
    for (int t = tid; t < nA + nC; t += FNTH) {
      const int cx = t < nA ? 64 : t - nA, cz = t < nA ? t : 4;
      if (cz < lzs || cz >= lze) continue;
      double a0, a1, a2;
      q2w(cz, a0, a1, a2);
      column(cx, cz, a0, a1, a2, fz0);
    }
  }
}

// EXP_true as a z-march over a 64 x 8 fine tile (threads 32 x 8; thread (lane, w) owns the nodes
// X0 + lane and X0 + 32 + lane of fine row Y0 + w, so every load / store instruction of a warp covers
// 256 contiguous bytes). u~ = u_h + (1/3) I_trilinear(d), d = u_h|_2h - u_2h (reading A13), with the
// trilinear interpolant applied axis by axis: per 2h plane K the tile's 33 x 5 corner differences are
// interpolated along x into a 64 x 5 shared array (one pass for the whole CTA), then each thread
// interpolates its two nodes along y in registers; fine plane 2K takes plane K's values, the odd plane
// 2K-1 the mean of planes K-1 and K (registers carried from the previous step). The weights are (1, 0)
// on a 2h node and (1/2, 1/2) between two, so every stage equals the mean of its two inputs bit for bit.
// Dirichlet nodes: overwritten with g_D (A15) by the face kernel launched after this one.
constexpr int ETX = 64, ETY = 8, EDX = ETX / 2 + 1, EDY = ETY / 2 + 1;   // 33 x 5 corner values per plane

// no min-blocks hint: ptxas picks 72 registers (3 CTAs / SM); measured at 512^3: hint 1 -> 102 registers,
// 0.71 ms; hint 3 -> 80, 0.60 ms; hint 4 -> 64, 0.67 ms; none 0.60 ms
__global__ void __launch_bounds__(256) k_exp_true(const LevelGeom gf, const Problem pb, const double* __restrict__ uh,
                                                  const double* __restrict__ u2h, double* __restrict__ ut, int c0,
                                                  int cchunk, double third) {
  __shared__ double D[2][EDY][EDX];     // corner differences of 2h plane K (slot K & 1)
  __shared__ double XI[2][EDY][ETX];    // ... interpolated along x to the tile's 64 fine columns
  __shared__ double UB[3][2][ETY][ETX];   // u_h of fine planes 2K-1, 2K: cp.async ring, two steps ahead
  const int lane = threadIdx.x, w = threadIdx.y, tid = lane + 32 * w;
  const int n2x = gf.n[0] / 2, n2y = gf.n[1] / 2, n2z = gf.n[2] / 2;
  const int X0 = blockIdx.x * ETX, Y0 = blockIdx.y * ETY;
  const int I0 = X0 / 2, J0 = Y0 / 2;
  const int Ca = c0 + blockIdx.z * cchunk, Cb = min(Ca + cchunk, min(gf.zhi / 2, n2z));   // 2h cells [Ca, Cb)
  if (Ca >= Cb) return;
  const long long nx = gf.n[0] + 1, ny = gf.n[1] + 1, pl = nx * ny;
  const long long nx2 = n2x + 1, pl2 = nx2 * (n2y + 1);
  const int fy = Y0 + w;
  const bool row_ok = fy <= gf.n[1];
  const int fxa = X0 + lane, fxb = X0 + 32 + lane;
  // corner differences: thread tid < 165 loads 2h node (di, dj) of each plane, one step ahead
  const bool dthr = tid < EDX * EDY;
  const int di = tid % EDX, dj = tid / EDX;
  const bool d_ok = dthr && I0 + di <= n2x && J0 + dj <= n2y;
  const long long doff_h = (long long)(2 * (J0 + dj)) * nx + 2 * (I0 + di), doff_2 = (long long)(J0 + dj) * nx2 + (I0 + di);
  auto load_d = [&](int K, double& a, double& b) {   // u_h at the 2h node and u_2h, plane K
    a = b = 0.0;
    if (d_ok) {
      a = __ldg(uh + (long long)(2 * K) * pl + doff_h);
      b = __ldg(u2h + (long long)K * pl2 + doff_2);
    }
  };
  // x pass: thread t < 320 (and t + 256 < 320) produces XI[r][c] = w0 D[r][c/2] + w1 D[r][c/2 + 1]
  auto xpass = [&](int sl) {
    for (int t = tid; t < EDY * ETX; t += 256) {
      const int r = t / ETX, c = t % ETX, i = c >> 1;
      const double w1 = (c & 1) ? 0.5 : 0.0, w0 = 1.0 - w1;
      XI[sl][r][c] = w0 * D[sl][r][i] + w1 * D[sl][r][i + 1];
    }
  };
  // y pass of this thread's two nodes (row w between 2h rows w/2 and w/2 + 1)
  const int jr = w >> 1;
  const double wy1 = (w & 1) ? 0.5 : 0.0, wy0 = 1.0 - wy1;
  auto ypass = [&](int sl, double& va, double& vb) {
    va = wy0 * XI[sl][jr][lane] + wy1 * XI[sl][jr + 1][lane];
    vb = wy0 * XI[sl][jr][lane + 32] + wy1 * XI[sl][jr + 1][lane + 32];
  };
  const bool okA = row_ok && fxa <= gf.n[0], okB = row_ok && fxb <= gf.n[0];
  const long long rowoff = (long long)fy * nx;
  // u_h rows of the thread's two nodes go to shared memory with cp.async (8-byte, cached), two steps
  // ahead, one commit group per step: the loads are in flight without holding registers
  auto cp8 = [&](double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
  };
  auto issue_u = [&](int K) {   // fine planes 2K-1 (if K > Ca) and 2K (if even_of(K)) into slot (K - Ca) % 3
    double* u0 = &UB[(K - Ca) % 3][0][w][0];
    double* u1 = &UB[(K - Ca) % 3][1][w][0];
    if (K > Ca) {
      const double* row = uh + (long long)(2 * K - 1) * pl + rowoff;
      if (okA) cp8(u0 + lane, row + fxa);
      if (okB) cp8(u0 + 32 + lane, row + fxb);
    }
    if (K < Cb || K == n2z) {
      const double* row = uh + (long long)(2 * K) * pl + rowoff;
      if (okA) cp8(u1 + lane, row + fxa);
      if (okB) cp8(u1 + 32 + lane, row + fxb);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // u~ on plane fz at this thread's nodes, every node by the formula: the Dirichlet nodes are overwritten with
  // g_D by the face kernel launched after this one (launch_exp_true), which keeps the rare g_D evaluation
  // (an out-of-line call with its stack frame) out of this loop
  auto put = [&](int fz, double ua, double ub, double ia_, double ib_) {
    const long long row = (long long)fz * pl + rowoff;
    if (okA) ut[row + fxa] = __fma_rn(ia_, third, ua);
    if (okB) ut[row + fxb] = __fma_rn(ib_, third, ub);
  };
  double dh, d2, pa = 0.0, pb_ = 0.0;   // pa, pb_: plane K-1's interpolated d at the thread's nodes
  load_d(Ca, dh, d2);
  issue_u(Ca);
  if (Ca + 1 <= Cb) issue_u(Ca + 1); else asm volatile("cp.async.commit_group;" ::: "memory");
  // D and XI are double buffered by plane parity: two barriers per step (D written -> x pass -> y pass);
  // slot K & 1 was last read in step K - 2, which every thread finished before step K - 1's barriers
  for (int K = Ca; K <= Cb; ++K) {
    const int pk = K & 1;
    if (dthr) D[pk][dj][di] = dh - d2;   // corner differences of 2h plane K
    if (K < Cb) load_d(K + 1, dh, d2);
    if (K + 2 <= Cb) issue_u(K + 2); else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 2;" ::: "memory");   // this step's group (own slots only: no barrier)
    const int sl = (K - Ca) % 3;
    const double uoa = UB[sl][0][w][lane], uob = UB[sl][0][w][lane + 32];
    const double uea = UB[sl][1][w][lane], ueb = UB[sl][1][w][lane + 32];
    const bool odd = K > Ca, even = K < Cb || K == n2z;
    __syncthreads();
    xpass(pk);
    __syncthreads();
    double ca, cb;
    ypass(pk, ca, cb);
    if (odd) put(2 * K - 1, uoa, uob, 0.5 * (pa + ca), 0.5 * (pb_ + cb));   // odd fine plane between K-1 and K
    if (even) put(2 * K, uea, ueb, ca, cb);                                // even fine plane 2K
    pa = ca;
    pb_ = cb;
  }
}


}  // namespace

cudaError_t launch_exp_finite(const LevelGeom& gf, const Problem& pb, const double* u2h, const double* u4h, double* w,
                              int variant, double* seeds, int freebox, cudaStream_t st, int fused) {
  // fine planes produced: the rank's free planes (free-box output) or its owned node planes (full output)
  const int F0 = freebox ? gf.flo[2] + gf.zoff + gf.zbeg : gf.zlo;
  const int F1 = freebox ? gf.flo[2] + gf.zoff + gf.zend : gf.zhi;
  if (F1 <= F0) return cudaSuccess;
  const int n4z = gf.n[2] / 4;
  const int bz0 = std::min(F0 / 4, n4z - 1), bz1 = std::min((F1 - 1) / 4, n4z - 1);
  if (fused) {
    const int nl = bz1 - bz0 + 1;
    const int tiles = ((gf.n[0] / 4 + XB - 1) / XB) * ((gf.n[1] / 4 + YB - 1) / YB);
    // >= ~2000 CTAs where the level allows (16 or 32 layers per CTA at 512^3: measured no faster)
    const int lchunk = std::max(1, std::min(8, tiles * nl / 2000));
    dim3 g((gf.n[0] / 4 + XB - 1) / XB, (gf.n[1] / 4 + YB - 1) / YB, (nl + lchunk - 1) / lchunk);
    count_launch();
    if (freebox && variant == 0) k_exp_fused<true, 0><<<g, FNTH, 0, st>>>(gf, u2h, u4h, w, F0, F1, bz0, lchunk);
    else if (freebox) k_exp_fused<true, 1><<<g, FNTH, 0, st>>>(gf, u2h, u4h, w, F0, F1, bz0, lchunk);
    else if (variant == 0) k_exp_fused<false, 0><<<g, FNTH, 0, st>>>(gf, u2h, u4h, w, F0, F1, bz0, lchunk);
    else k_exp_fused<false, 1><<<g, FNTH, 0, st>>>(gf, u2h, u4h, w, F0, F1, bz0, lchunk);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || freebox) return e;
    return launch_dirichlet_fill(gf, pb, w, 0.0, 0, st);   // full output: g_D on the Dirichlet nodes (§8c A15)
  }
  const int K0 = 2 * bz0, K1 = 2 * bz1 + 2;   // 2h planes of the touched 4h blocks
  dim3 g1((gf.n[0] / 2 + 1 + 127) / 128, gf.n[1] / 2 + 1, K1 - K0 + 1);
  count_launch();
  k_exp_seeds<<<g1, 128, 0, st>>>(gf, u2h, u4h, seeds, variant, K0);
  dim3 g2((gf.n[0] / 4 + 63) / 64, gf.n[1] / 4, F1 - F0);
  count_launch();
  if (freebox) k_exp_interp<true><<<g2, 64, 0, st>>>(gf, pb, seeds, w, variant, F0);
  else k_exp_interp<false><<<g2, 64, 0, st>>>(gf, pb, seeds, w, variant, F0);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || freebox) return e;
  return launch_dirichlet_fill(gf, pb, w, 0.0, 0, st);
}

cudaError_t launch_exp_true(const LevelGeom& gf, const Problem& pb, const double* uh, const double* u2h, double* ut,
                            cudaStream_t st) {
  const int c0 = gf.zlo / 2, c1 = std::min(gf.zhi / 2, gf.n[2] / 2);   // 2h cells owning this rank's planes
  if (c1 <= c0) return cudaSuccess;
  const int cchunk = 32;   // 2h cells (64 fine planes) per CTA
  dim3 grid((gf.n[0] + 1 + ETX - 1) / ETX, (gf.n[1] + 1 + ETY - 1) / ETY, (c1 - c0 + cchunk - 1) / cchunk);
  count_launch();
  k_exp_true<<<grid, dim3(32, 8), 0, st>>>(gf, pb, uh, u2h, ut, c0, cchunk, 1.0 / 3.0);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_dirichlet_fill(gf, pb, ut, 0.0, 0, st);   // Dirichlet overwrite (§8c A15): u~ = g_D there
}

}  // namespace ecmg
