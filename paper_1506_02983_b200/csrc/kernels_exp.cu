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
// DESIGN.md). One thread per 2h cell computes its (up to 27) owned fine nodes from the 8 corner
// differences. Dirichlet nodes take g_D.
#include <algorithm>
#include "ecmg_internal.cuh"
#include "problems.cuh"

namespace ecmg {
namespace {

__device__ __forceinline__ bool is_free(const LevelGeom& g, int gx, int gy, int gz) {
  return gx >= g.flo[0] && gx < g.flo[0] + g.nf[0] && gy >= g.flo[1] && gy < g.flo[1] + g.nf[1] &&
         gz >= g.flo[2] && gz < g.flo[2] + g.nf[2];
}

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
        if (!fr) W = prob_gD(pb, gf.lo[0] + fx * gf.h[0], gf.lo[1] + fy * gf.h[1], gf.lo[2] + fz * gf.h[2]);
        out[(long long)fx + nx * ((long long)fy + ny * fz)] = W;
      }
    }
  }
}

// EXP_true, one thread per 2h cell (cx, cy, cz); owned fine nodes 2c + {0,1} per axis (+2 in the
// last cell along an axis). Cells whose owned nodes are all free take the fast path (no Dirichlet
// tests, pointer increments only).
__global__ void __launch_bounds__(128, 6) k_exp_true(const LevelGeom gf, const Problem pb, const double* __restrict__ uh,
                                                  const double* __restrict__ u2h, double* __restrict__ ut) {
  const int n2x = gf.n[0] / 2, n2y = gf.n[1] / 2, n2z = gf.n[2] / 2;
  const int cx = blockIdx.x * blockDim.x + threadIdx.x, cy = blockIdx.y, cz = gf.zlo / 2 + blockIdx.z;
  if (cx >= n2x) return;
  const long long nx = gf.n[0] + 1, ny = gf.n[1] + 1, pl = nx * ny;
  const long long nx2 = n2x + 1, pl2 = nx2 * (n2y + 1);
  const long long c0 = 2LL * cx + nx * 2LL * cy + pl * 2LL * cz;     // fine index of the cell's first node
  const long long k0 = (long long)cx + nx2 * cy + pl2 * cz;          // 2h index of the cell's first corner
  double d[2][2][2];
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a)
        d[c][b][a] = __ldg(uh + c0 + 2 * (a + nx * b + pl * c)) - __ldg(u2h + k0 + a + nx2 * b + pl2 * c);
  const bool last = (cx == n2x - 1) || (cy == n2y - 1) || (cz == n2z - 1);
  const bool inner = !last && 2 * cx >= gf.flo[0] && 2 * cy >= gf.flo[1] && 2 * cz >= gf.flo[2] &&
                     2 * cx + 1 < gf.flo[0] + gf.nf[0] && 2 * cy + 1 < gf.flo[1] + gf.nf[1] && 2 * cz + 1 < gf.flo[2] + gf.nf[2];
  if (inner) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const double wz1 = 0.5 * c, wz0 = 1.0 - wz1, wy1 = 0.5 * b, wy0 = 1.0 - wy1;
        const double r0 = wz0 * (wy0 * d[0][0][0] + wy1 * d[0][1][0]) + wz1 * (wy0 * d[1][0][0] + wy1 * d[1][1][0]);
        const double r1 = wz0 * (wy0 * d[0][0][1] + wy1 * d[0][1][1]) + wz1 * (wy0 * d[1][0][1] + wy1 * d[1][1][1]);
        const long long i = c0 + nx * b + pl * c;
        ut[i] = __ldg(uh + i) + r0 / 3.0;
        ut[i + 1] = __ldg(uh + i + 1) + (0.5 * r0 + 0.5 * r1) / 3.0;
      }
    return;
  }
  const int ea = (cx == n2x - 1) ? 3 : 2, eb = (cy == n2y - 1) ? 3 : 2, ec = (cz == n2z - 1) ? 3 : 2;
  for (int c = 0; c < ec; ++c) {
    const double wz[2] = {1.0 - 0.5 * c, 0.5 * c};
    const int fz = 2 * cz + c;
    for (int b = 0; b < eb; ++b) {
      const double wy[2] = {1.0 - 0.5 * b, 0.5 * b};
      const int fy = 2 * cy + b;
      const double r0 = wz[0] * (wy[0] * d[0][0][0] + wy[1] * d[0][1][0]) + wz[1] * (wy[0] * d[1][0][0] + wy[1] * d[1][1][0]);
      const double r1 = wz[0] * (wy[0] * d[0][0][1] + wy[1] * d[0][1][1]) + wz[1] * (wy[0] * d[1][0][1] + wy[1] * d[1][1][1]);
      for (int a = 0; a < ea; ++a) {
        const int fx = 2 * cx + a;
        const long long i = (long long)fx + nx * ((long long)fy + ny * fz);
        double v;
        if (!is_free(gf, fx, fy, fz)) {
          v = prob_gD(pb, gf.lo[0] + fx * gf.h[0], gf.lo[1] + fy * gf.h[1], gf.lo[2] + fz * gf.h[2]);
        } else {
          const double I = (1.0 - 0.5 * a) * r0 + 0.5 * a * r1;
          v = __ldg(uh + i) + I / 3.0;
        }
        ut[i] = v;
      }
    }
  }
}

}  // namespace

cudaError_t launch_exp_finite(const LevelGeom& gf, const Problem& pb, const double* u2h, const double* u4h, double* w,
                              int variant, double* seeds, int freebox, cudaStream_t st) {
  // fine planes produced: the rank's free planes (free-box output) or its owned node planes (full output)
  const int F0 = freebox ? gf.flo[2] + gf.zoff + gf.zbeg : gf.zlo;
  const int F1 = freebox ? gf.flo[2] + gf.zoff + gf.zend : gf.zhi;
  if (F1 <= F0) return cudaSuccess;
  const int n4z = gf.n[2] / 4;
  const int bz0 = std::min(F0 / 4, n4z - 1), bz1 = std::min((F1 - 1) / 4, n4z - 1);
  const int K0 = 2 * bz0, K1 = 2 * bz1 + 2;   // 2h planes of the touched 4h blocks
  dim3 g1((gf.n[0] / 2 + 1 + 127) / 128, gf.n[1] / 2 + 1, K1 - K0 + 1);
  count_launch();
  k_exp_seeds<<<g1, 128, 0, st>>>(gf, u2h, u4h, seeds, variant, K0);
  dim3 g2((gf.n[0] / 4 + 63) / 64, gf.n[1] / 4, F1 - F0);
  count_launch();
  if (freebox) k_exp_interp<true><<<g2, 64, 0, st>>>(gf, pb, seeds, w, variant, F0);
  else k_exp_interp<false><<<g2, 64, 0, st>>>(gf, pb, seeds, w, variant, F0);
  return cudaGetLastError();
}

cudaError_t launch_exp_true(const LevelGeom& gf, const Problem& pb, const double* uh, const double* u2h, double* ut,
                            cudaStream_t st) {
  const int c0 = gf.zlo / 2, c1 = std::min(gf.zhi / 2, gf.n[2] / 2);   // 2h cells owning this rank's planes
  if (c1 <= c0) return cudaSuccess;
  dim3 grid((gf.n[0] / 2 + 127) / 128, gf.n[1] / 2, c1 - c0);
  count_launch();
  k_exp_true<<<grid, 128, 0, st>>>(gf, pb, uh, u2h, ut);
  return cudaGetLastError();
}

}  // namespace ecmg
