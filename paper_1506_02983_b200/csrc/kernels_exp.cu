// kernels_exp.cu -- the level-to-level extrapolation operators of Alg. 4.
//
// EXP_finite (l.6; §4.3). CTA = 8 coarse (4h) blocks along x, one block row in y
// and z (fine tile 32 x 4 x 4 nodes). Phase 1: the extrapolated values at the 27 2h nodes of each
// block go to shared memory -- corners (5U^1-U^0)/4 (Eq. jiedian), edge midpoints
// U^1_m + (U^1_a-U^0_a+U^1_b-U^0_b)/8 (Eq. zhongdian), and, for Remark 2's variant
// only, face / cell centres as the mean of Eq. (zhongdian) over the face / space diagonals
// (P:513-516). Phase 2: every fine node interpolates from its block's values:
//   variant 0 (default): the 20-node tri-quadratic Serendipity interpolant, evaluated
//     in its blending form W = P_x + P_y + P_z - 2T (P_d = quadratic along the 4 d-edges blended
//     bilinearly across them, T = trilinear in the corners). It lies in the 20-dim Serendipity
//     space and interpolates the 20 seeds, hence equals sum_i N_i W_i of Eq. (inter).
//   variant 1 (Remark 2): tri-quadratic Lagrange through all 27 values.
// Owner block of fine node i: b = min(i/4, n_4h - 1) per axis (reading §8c A14). Dirichlet nodes
// then take g_D (§8c A15).
//
// EXP_true (l.10): u~ = u_h + (1/3) I_trilinear(u_h|_2h - u_2h), which equals
// Eq. (t1) at 2h nodes, Eq. (chenlin) at 2h edge centres and the mean of Eq. (chenlin) over the
// 2 face diagonals / 4 space diagonals at face / cell centres (reading §8c A13; derived identity,
// DESIGN.md). Dirichlet nodes take g_D.
#include "ecmg_internal.cuh"
#include "problems.cuh"

namespace ecmg {
namespace {

constexpr int EBX = 8;              // 4h blocks per CTA along x
constexpr int EFX = 4 * EBX;        // 32 fine nodes along x
constexpr int ENTH = EFX * 4 * 4;   // 512 threads: 32 x 4 x 4 fine nodes

__device__ __forceinline__ bool is_free(const LevelGeom& g, int gx, int gy, int gz) {
  return gx >= g.flo[0] && gx < g.flo[0] + g.nf[0] && gy >= g.flo[1] && gy < g.flo[1] + g.nf[1] &&
         gz >= g.flo[2] && gz < g.flo[2] + g.nf[2];
}

__global__ void __launch_bounds__(ENTH) k_exp_finite(const LevelGeom gf, const Problem pb, const double* __restrict__ u2h,
                                                      const double* __restrict__ u4h, double* __restrict__ w, int variant) {
  __shared__ double seed[EBX][3][3][3];   // [block][k][j][i] extrapolated values at the block's 2h nodes
  const int n4[3] = {gf.n[0] / 4, gf.n[1] / 4, gf.n[2] / 4};
  const long long nn2x = gf.n[0] / 2 + 1, nn2y = gf.n[1] / 2 + 1;
  const long long nn4x = n4[0] + 1, nn4y = n4[1] + 1;
  const int tid = threadIdx.x;
  // fine tile: x in [32 bx, 32 bx + 32), y in [4 by, 4 by + 4), z in [4 bz, 4 bz + 4)
  const int fx0 = blockIdx.x * EFX, fy0 = blockIdx.y * 4, fz0 = blockIdx.z * 4;
  const int bxmin = min(fx0 / 4, n4[0] - 1);
  const int by = min(fy0 / 4, n4[1] - 1), bz = min(fz0 / 4, n4[2] - 1);

  auto U1 = [&](long long i, long long j, long long k) { return __ldg(u2h + i + nn2x * (j + nn2y * k)); };
  auto U0 = [&](long long i, long long j, long long k) { return __ldg(u4h + i + nn4x * (j + nn4y * k)); };

  for (int t = tid; t < EBX * 27; t += ENTH) {
    const int lb = t / 27, c = t % 27;
    const int ci = c % 3, cj = (c / 3) % 3, ck = c / 9;
    const int bx = bxmin + lb;
    double v = 0.0;
    if (bx < n4[0]) {
      const int cc[3] = {ci, cj, ck};
      const int nmid = (ci == 1) + (cj == 1) + (ck == 1);
      const long long g2[3] = {2LL * bx + ci, 2LL * by + cj, 2LL * bz + ck};
      if (nmid == 0) {
        v = (5.0 * U1(g2[0], g2[1], g2[2]) - U0(bx + ci / 2, by + cj / 2, bz + ck / 2)) / 4.0;
      } else if (nmid == 1 || variant == 1) {
        // mean of Eq. (zhongdian) over the segments through this 2h node whose ends are corners
        int ax[3], na = 0;
        for (int d = 0; d < 3; ++d) if (cc[d] == 1) ax[na++] = d;
        const int nseg = 1 << (na - 1);
        double sum = 0.0;
        for (int s = 0; s < nseg; ++s) {
          int ca[3] = {ci, cj, ck}, cb[3] = {ci, cj, ck};
          ca[ax[0]] = 0; cb[ax[0]] = 2;
          for (int q = 1; q < na; ++q) {
            const bool plus = (s >> (q - 1)) & 1;
            ca[ax[q]] = plus ? 0 : 2; cb[ax[q]] = plus ? 2 : 0;
          }
          const double a1 = U1(2LL * bx + ca[0], 2LL * by + ca[1], 2LL * bz + ca[2]);
          const double a0 = U0(bx + ca[0] / 2, by + ca[1] / 2, bz + ca[2] / 2);
          const double b1 = U1(2LL * bx + cb[0], 2LL * by + cb[1], 2LL * bz + cb[2]);
          const double b0 = U0(bx + cb[0] / 2, by + cb[1] / 2, bz + cb[2] / 2);
          sum += U1(g2[0], g2[1], g2[2]) + (a1 - a0 + b1 - b0) / 8.0;
        }
        v = sum / nseg;
      }
    }
    seed[lb][ck][cj][ci] = v;
  }
  __syncthreads();

  const int lx = tid % EFX, ly = (tid / EFX) % 4, lz = tid / (EFX * 4);
  const int fx = fx0 + lx, fy = fy0 + ly, fz = fz0 + lz;
  if (fx > gf.n[0] || fy > gf.n[1] || fz > gf.n[2]) return;
  const int bx = min(fx / 4, n4[0] - 1);
  const int lb = bx - bxmin;
  const double xi = (fx - 4 * bx - 2) * 0.5, eta = (fy - 4 * by - 2) * 0.5, zeta = (fz - 4 * bz - 2) * 0.5;
  const double (*s)[3][3] = seed[lb];
  double W;
  if (variant == 1) {
    const double qx[3] = {xi * (xi - 1.0) * 0.5, 1.0 - xi * xi, xi * (xi + 1.0) * 0.5};
    const double qy[3] = {eta * (eta - 1.0) * 0.5, 1.0 - eta * eta, eta * (eta + 1.0) * 0.5};
    const double qz[3] = {zeta * (zeta - 1.0) * 0.5, 1.0 - zeta * zeta, zeta * (zeta + 1.0) * 0.5};
    W = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j)
        t += qy[j] * (qx[0] * s[k][j][0] + qx[1] * s[k][j][1] + qx[2] * s[k][j][2]);
      W += qz[k] * t;
    }
  } else {
    const double qx[3] = {xi * (xi - 1.0) * 0.5, 1.0 - xi * xi, xi * (xi + 1.0) * 0.5};
    const double qy[3] = {eta * (eta - 1.0) * 0.5, 1.0 - eta * eta, eta * (eta + 1.0) * 0.5};
    const double qz[3] = {zeta * (zeta - 1.0) * 0.5, 1.0 - zeta * zeta, zeta * (zeta + 1.0) * 0.5};
    const double lx2[2] = {(1.0 - xi) * 0.5, (1.0 + xi) * 0.5};
    const double ly2[2] = {(1.0 - eta) * 0.5, (1.0 + eta) * 0.5};
    const double lz2[2] = {(1.0 - zeta) * 0.5, (1.0 + zeta) * 0.5};
    double Px = 0.0, Py = 0.0, Pz = 0.0, T = 0.0;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int A = 2 * a, B = 2 * b;
        // x-edge at (y,z) = (A, B): quadratic in xi, weight ly2[a] lz2[b]
        Px += ly2[a] * lz2[b] * (qx[0] * s[B][A][0] + qx[1] * s[B][A][1] + qx[2] * s[B][A][2]);
        // y-edge at (x,z) = (A, B)
        Py += lx2[a] * lz2[b] * (qy[0] * s[B][0][A] + qy[1] * s[B][1][A] + qy[2] * s[B][2][A]);
        // z-edge at (x,y) = (A, B)
        Pz += lx2[a] * ly2[b] * (qz[0] * s[0][B][A] + qz[1] * s[1][B][A] + qz[2] * s[2][B][A]);
      }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int a = 0; a < 2; ++a) T += lx2[a] * ly2[b] * lz2[c] * s[2 * c][2 * b][2 * a];
    W = Px + Py + Pz - 2.0 * T;
  }
  if (!is_free(gf, fx, fy, fz))
    W = prob_gD(pb, gf.lo[0] + fx * gf.h[0], gf.lo[1] + fy * gf.h[1], gf.lo[2] + fz * gf.h[2]);
  const long long nx = gf.n[0] + 1, ny = gf.n[1] + 1;
  w[(long long)fx + nx * ((long long)fy + ny * fz)] = W;
}

__global__ void k_exp_true(const LevelGeom gf, const Problem pb, const double* __restrict__ uh, const double* __restrict__ u2h,
                           double* __restrict__ ut) {
  const int fx = blockIdx.x * blockDim.x + threadIdx.x, fy = blockIdx.y, fz = blockIdx.z;
  if (fx > gf.n[0]) return;
  const long long nx = gf.n[0] + 1, ny = gf.n[1] + 1;
  const long long nx2 = gf.n[0] / 2 + 1, ny2 = gf.n[1] / 2 + 1;
  const long long i = (long long)fx + nx * ((long long)fy + ny * fz);
  double v;
  if (!is_free(gf, fx, fy, fz)) {
    v = prob_gD(pb, gf.lo[0] + fx * gf.h[0], gf.lo[1] + fy * gf.h[1], gf.lo[2] + fz * gf.h[2]);
  } else {
    // 2h cell containing the node and trilinear weights of d = u_h|_2h - u_2h at its corners
    const int cx = min(fx / 2, gf.n[0] / 2 - 1), cy = min(fy / 2, gf.n[1] / 2 - 1), cz = min(fz / 2, gf.n[2] / 2 - 1);
    const double tx = (fx - 2 * cx) * 0.5, ty = (fy - 2 * cy) * 0.5, tz = (fz - 2 * cz) * 0.5;
    double I = 0.0;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double wz = c ? tz : 1.0 - tz;
      if (wz == 0.0) continue;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const double wy = b ? ty : 1.0 - ty;
        if (wy == 0.0) continue;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const double wx = a ? tx : 1.0 - tx;
          if (wx == 0.0) continue;
          const long long X = cx + a, Y = cy + b, Z = cz + c;
          const double d = __ldg(uh + 2 * X + nx * (2 * Y + ny * 2 * Z)) - __ldg(u2h + X + nx2 * (Y + ny2 * Z));
          I += wx * wy * wz * d;
        }
      }
    }
    v = __ldg(uh + i) + I / 3.0;
  }
  ut[i] = v;
}

}  // namespace

cudaError_t launch_exp_finite(const LevelGeom& gf, const Problem& pb, const double* u2h, const double* u4h, double* w,
                              int variant, cudaStream_t st) {
  dim3 grid((gf.n[0] + 1 + EFX - 1) / EFX, (gf.n[1] + 1 + 3) / 4, (gf.n[2] + 1 + 3) / 4);
  count_launch();
  k_exp_finite<<<grid, ENTH, 0, st>>>(gf, pb, u2h, u4h, w, variant);
  return cudaGetLastError();
}

cudaError_t launch_exp_true(const LevelGeom& gf, const Problem& pb, const double* uh, const double* u2h, double* ut,
                            cudaStream_t st) {
  dim3 grid((gf.n[0] + 1 + 127) / 128, gf.n[1] + 1, gf.n[2] + 1);
  count_launch();
  k_exp_true<<<grid, 128, 0, st>>>(gf, pb, uh, u2h, ut);
  return cudaGetLastError();
}

}  // namespace ecmg
