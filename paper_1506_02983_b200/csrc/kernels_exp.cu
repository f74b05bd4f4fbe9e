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
// planes in shared memory. Dirichlet nodes take g_D.
#include <algorithm>
#include "ecmg_internal.cuh"
#include "problems.cuh"

namespace ecmg {
namespace {

// g_D at fine node (fx, fy, fz): kept out of line (boundary faces only) so the marching loops stay lean
__device__ __noinline__ double gD_at(const LevelGeom& gf, const Problem& pb, int fx, int fy, int fz) {
  return prob_gD(pb, gf.lo[0] + fx * gf.h[0], gf.lo[1] + fy * gf.h[1], gf.lo[2] + fz * gf.h[2]);
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
        if (!fr) W = gD_at(gf, pb, fx, fy, fz);
        out[(long long)fx + nx * ((long long)fy + ny * fz)] = W;
      }
    }
  }
}

// EXP_true as a z-march over a 64 x 8 fine tile (threads 32 x 8; thread (lane, w) owns the nodes
// X0 + lane and X0 + 32 + lane of fine row Y0 + w, so every load / store instruction of a warp covers
// 256 contiguous bytes). Per 2h plane K: (a) the tile's 33 x 5 corner differences
// d = u_h|_2h - u_2h of plane K go to a two-plane shared ring; (b) fine plane 2K-1 is written from
// d planes K-1, K and (c) fine plane 2K from d plane K: u~ = u_h + (1/3) I_trilinear(d), where the
// trilinear interpolant at a fine node is d at the 2h node it sits on, or the mean of the two / four /
// eight 2h nodes around it (reading A13). Dirichlet nodes take g_D (A15).
constexpr int ETX = 64, ETY = 8, EDX = ETX / 2 + 1, EDY = ETY / 2 + 1;   // 33 x 5 corner values per plane

__global__ void __launch_bounds__(256) k_exp_true(const LevelGeom gf, const Problem pb, const double* __restrict__ uh,
                                                  const double* __restrict__ u2h, double* __restrict__ ut, int c0,
                                                  int cchunk) {
  __shared__ double D[2][EDY][EDX];
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
  // interpolation stencil of the thread's nodes: 2h column(s) and row(s) below / above
  const int ia = lane >> 1, iaw = lane & 1;                 // node fxa: d column ia (+1 if odd)
  const int ib = 16 + (lane >> 1);                          // node fxb: d column ib (+1 if odd)
  const int jr = w >> 1, jw = w & 1;                        // row: d row jr (+1 if odd)
  // (y, x)-interpolated d of plane slot s at the two nodes of this thread
  auto dxy = [&](int s, double& va, double& vb) {
    double a = D[s][jr][ia], b = D[s][jr][ib];
    if (iaw) { a = 0.5 * (a + D[s][jr][ia + 1]); b = 0.5 * (b + D[s][jr][ib + 1]); }
    if (jw) {
      double a2 = D[s][jr + 1][ia], b2 = D[s][jr + 1][ib];
      if (iaw) { a2 = 0.5 * (a2 + D[s][jr + 1][ia + 1]); b2 = 0.5 * (b2 + D[s][jr + 1][ib + 1]); }
      a = 0.5 * (a + a2);
      b = 0.5 * (b + b2);
    }
    va = a;
    vb = b;
  };
  // loads are issued one step ahead (registers), so the global latency overlaps the barrier and the
  // shared-memory interpolation of the current step
  const bool dthr = tid < EDX * EDY;
  const int di = tid % EDX, dj = tid / EDX;
  const bool d_ok = dthr && I0 + di <= n2x && J0 + dj <= n2y;
  auto load_d = [&](int K, double& a, double& b) {   // u_h at the 2h node and u_2h, plane K
    a = b = 0.0;
    if (d_ok) {
      a = __ldg(uh + (long long)(2 * K) * pl + (long long)(2 * (J0 + dj)) * nx + 2 * (I0 + di));
      b = __ldg(u2h + (long long)K * pl2 + (J0 + dj) * nx2 + (I0 + di));
    }
  };
  const bool okA = row_ok && fxa <= gf.n[0], okB = row_ok && fxb <= gf.n[0];
  auto load_u = [&](int fz, double& a, double& b) {
    const long long row = (long long)fz * pl + (long long)fy * nx;
    a = okA ? __ldg(uh + row + fxa) : 0.0;
    b = okB ? __ldg(uh + row + fxb) : 0.0;
  };
  auto put = [&](int fz, double ua, double ub, double ia_, double ib_) {   // u~ on plane fz, this thread's nodes
    const long long row = (long long)fz * pl + (long long)fy * nx;
    const bool zf = fz >= gf.flo[2] && fz < gf.flo[2] + gf.nf[2], yf = fy >= gf.flo[1] && fy < gf.flo[1] + gf.nf[1];
    if (okA) {
      const bool fr = zf && yf && fxa >= gf.flo[0] && fxa < gf.flo[0] + gf.nf[0];
      ut[row + fxa] = fr ? ua + ia_ / 3.0 : gD_at(gf, pb, fxa, fy, fz);
    }
    if (okB) {
      const bool fr = zf && yf && fxb >= gf.flo[0] && fxb < gf.flo[0] + gf.nf[0];
      ut[row + fxb] = fr ? ub + ib_ / 3.0 : gD_at(gf, pb, fxb, fy, fz);
    }
  };
  double dh, d2;
  load_d(Ca, dh, d2);
  for (int K = Ca; K <= Cb; ++K) {
    __syncthreads();   // the slot of plane K (plane K-2's) is free
    if (dthr) D[K & 1][dj][di] = dh - d2;   // (a) corner differences of 2h plane K
    if (K < Cb) load_d(K + 1, dh, d2);
    double uoa = 0.0, uob = 0.0, uea = 0.0, ueb = 0.0;
    const bool odd = K > Ca, even = K < Cb || K == n2z;
    if (odd) load_u(2 * K - 1, uoa, uob);
    if (even) load_u(2 * K, uea, ueb);
    __syncthreads();
    if (odd) {   // (b) odd fine plane 2K-1 between d planes K-1 and K
      double a0, b0, a1, b1;
      dxy((K - 1) & 1, a0, b0);
      dxy(K & 1, a1, b1);
      put(2 * K - 1, uoa, uob, 0.5 * (a0 + a1), 0.5 * (b0 + b1));
    }
    if (even) {   // (c) even fine plane 2K (the last 2h plane also ends the level)
      double a0, b0;
      dxy(K & 1, a0, b0);
      put(2 * K, uea, ueb, a0, b0);
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
  const int cchunk = 32;   // 2h cells (64 fine planes) per CTA
  dim3 grid((gf.n[0] + 1 + ETX - 1) / ETX, (gf.n[1] + 1 + ETY - 1) / ETY, (c1 - c0 + cchunk - 1) / cchunk);
  count_launch();
  k_exp_true<<<grid, dim3(32, 8), 0, st>>>(gf, pb, uh, u2h, ut, c0, cchunk);
  return cudaGetLastError();
}

}  // namespace ecmg
