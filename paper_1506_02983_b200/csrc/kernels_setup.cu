// kernels_setup.cu -- per-level setup of the Q1 system: element coefficients,
// load vector by 2x2x2 Gauss quadrature (reading §8c A2), Robin face load by 2x2 Gauss (§8c A4),
// symmetric Dirichlet elimination (lifting, §8c A5), ||f_h||_2, and the gather / scatter between
// caller-visible nodal vectors and the free-box work vectors.
#include <algorithm>
#include "ecmg_internal.cuh"
#include "host_common.h"
#include "problems.cuh"

namespace ecmg {
namespace {

constexpr double kGauss = 0.57735026918962576451;  // 1/sqrt(3)

// ---- element coefficients beta_e = beta(centroid) (§8c A3), zero outside the domain ----------
// Per-axis tables of beta_combine (ecmg_internal.cuh) at the element centroids lo + (e + 1/2) h, e in
// [-2, n_d + 1]: the factor / layer value A and the bits M (element exists; inside box k along the axis).
__global__ void k_beta_axes(const LevelGeom g, const Problem pb, double* __restrict__ tab, int W, int kind) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  double* A = tab;
  int* M = reinterpret_cast<int*>(tab + 3LL * W);
  double* boxb = tab + 3LL * W + (3LL * W + 1) / 2;
  if (t < 4) boxb[t] = (kind == BETA_KIND_C5) ? pb.params[15 + 7 * t + 6] : 0.0;
  if (t >= 3 * W) return;
  const int d = t / W, e = t % W - 2;
  double a = 0.0;
  int m = 0;
  if (e >= -2 && e < g.n[d] + 2) {
    const double c = g.lo[d] + (e + 0.5) * g.h[d];
    if (e >= 0 && e < g.n[d]) m |= 16;
    const double tp = 2.0 * kPi() * c;
    if (kind == BETA_KIND_C3) a = d == 0 ? 0.5 * sin(tp) : (d == 1 ? cos(tp) : sin(tp));
    if ((kind == BETA_KIND_LAYERS || kind == BETA_KIND_C5) && d == 2) a = layer_beta(pb, c);
    if (kind == BETA_KIND_C5)
      for (int k = 0; k < 4; ++k) {
        const double* q = &pb.params[15 + 7 * k];
        if (fabs(c - q[d]) < q[3 + d]) m |= 1 << k;
      }
  }
  A[t] = a;
  M[t] = m;
}

__global__ void k_beta(const LevelGeom g, double* __restrict__ beta, const double* __restrict__ tab, int W, int kind) {
  // element planes this rank's work vectors touch: [flo+zoff-2, flo+zoff+nza] (all planes on one GPU)
  const int e0 = max(-2, g.flo[2] + g.zoff - 2), e1 = min(g.n[2] + 1, g.flo[2] + g.zoff + g.nza);
  const long long ne0 = g.n[0] + 4, ne1 = g.n[1] + 4, ne2 = e1 - e0 + 1;
  const long long total = ne0 * ne1 * ne2;
  const double* A = tab;
  const int* M = reinterpret_cast<const int*>(tab + 3LL * W);
  const double* boxb = tab + 3LL * W + (3LL * W + 1) / 2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int ex = (int)(t % ne0) - 2, ey = (int)((t / ne0) % ne1) - 2, ez = (int)(t / (ne0 * ne1)) + e0;
    const double v = beta_combine(kind, A[ex + 2], A[W + ey + 2], A[2 * W + ez + 2], M[ex + 2], M[W + ey + 2],
                                  M[2 * W + ez + 2], boxb);
    beta[(long long)(ez + 2) * g.BS + (long long)(ey + 2) * g.BP + (ex + 2)] = v;
  }
}

// PROB_ARRAYS: beta_e from the caller's element array (x fastest), 1 if absent, 0 on the ring
__global__ void k_beta_arr(const LevelGeom g, double* __restrict__ beta, const double* __restrict__ be) {
  const int e0 = max(-2, g.flo[2] + g.zoff - 2), e1 = min(g.n[2] + 1, g.flo[2] + g.zoff + g.nza);
  const long long ne0 = g.n[0] + 4, ne1 = g.n[1] + 4, ne2 = e1 - e0 + 1;
  const long long total = ne0 * ne1 * ne2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int ex = (int)(t % ne0) - 2, ey = (int)((t / ne0) % ne1) - 2, ez = (int)(t / (ne0 * ne1)) + e0;
    const bool in = ex >= 0 && ex < g.n[0] && ey >= 0 && ey < g.n[1] && ez >= 0 && ez < g.n[2];
    const double v = !in ? 0.0 : (be ? be[(long long)ex + g.n[0] * ((long long)ey + (long long)g.n[1] * ez)] : 1.0);
    beta[(long long)(ez + 2) * g.BS + (long long)(ey + 2) * g.BP + (ex + 2)] = v;
  }
}

// ---- right-hand side ---------------------------------------------------------------------------
// b_f = F_f + G_f - A_fD g_D (§8c A2/A4/A5) in up to three passes:
//  (1) volume load F by 2x2x2 Gauss. Separable f = sum_k A_k g_k^x(x) g_k^y(y) g_k^z(z) (rank 1: C1, C2,
//      C5, P1, P2, the patch tests; rank 5: C3): F_i = sum_k A_k L_kx(i_x) L_ky(i_y) L_kz(i_z), with the
//      1D Gauss loads L_kd(i) = sum_{e in {i-1,i}} (h_d/2) sum_{q=+-} g_kd(x_q) N(xi_q) (the 3D rule
//      factorises exactly). Otherwise (C4, P3): z-marching CTAs evaluate f once per Gauss point of
//      each element plane (shared memory), form the element load vectors, and every node gathers its
//      8 entries.
//  (2) boundary shell of the free box: Robin face load G (2x2 Gauss) and the lifting -A_fD g_D.
// ||b||^2 is accumulated by the JCG init pass, which reads b anyway.
// node tile 31 x 7 -> element tile 32 x 8 = 256 = one element (and 8 Gauss points) per thread
constexpr int VX = 31, VY = 7, VNTH = 256;
constexpr int VEX = VX + 1, VEY = VY + 1, VNE = VEX * VEY;     // 32 x 8 elements per plane
constexpr int VSMEM = (VNE * 8 + 2 * VNE * 8) * (int)sizeof(double);

// f as a sum of R products of 1D functions, f = sum_k A_k g_k^x(x) g_k^y(y) g_k^z(z); R = 0: not
// separable (volume kernel). C3's f = -beta Lap u - grad beta . grad u with beta = 1 + 1/2 sin(2 pi x)
// cos(2 pi y) sin(2 pi z), u = cos(pi x) cos(pi y) e^z expands into 5 such terms:
//   -(1 - 2 pi^2) [cx][cy][e^z]            -(1 - 2 pi^2)/2 [s2x cx][c2y cy][s2z e^z]   (-beta Lap u)
//   +pi^2 [c2x sx][c2y cy][s2z e^z]        -pi^2 [s2x cx][s2y sy][s2z e^z]             (-beta_x u_x, -beta_y u_y)
//   -pi [s2x cx][c2y cy][c2z e^z]                                                        (-beta_z u_z)
// (sx = sin(pi x), s2x = sin(2 pi x), ...). The 2x2x2 Gauss rule factorises exactly per term.
constexpr int kMaxSepRank = 5;
__host__ __device__ inline int prob_sep_rank(int id) {
  switch (id) {
    case 1: case 2: case 5: case 11: case 12: case 21: case 22: case 23: case 24: case 25: return 1;
    case 3: return 5;
    default: return 0;
  }
}
__host__ __device__ inline bool prob_separable(int id) { return prob_sep_rank(id) > 0; }
__device__ inline double sep_amp(const Problem& P, int k) {
  const double pi = kPi();
  switch (P.id) {
    case 1: return 3.0 * pi * pi;
    case 2: return -3.0;
    case 3: {
      const double A[5] = {-(1.0 - 2.0 * pi * pi), -0.5 * (1.0 - 2.0 * pi * pi), pi * pi, -pi * pi, -pi};
      return A[k];
    }
    case 5: return P.params[47];
    case 11: return 0.75 * pi * pi;
    case 12: return -(1.0 - 2.5 * pi * pi);
    case 24: return 1.0;
    default: return 0.0;   // patch tests: f = 0
  }
}
__device__ inline double sep_g(const Problem& P, int k, int d, double t) {
  const double pi = kPi();
  switch (P.id) {
    case 1: return sin(pi * t);
    case 2: return exp(t);
    case 3: {
      double s1, c1, s2, c2;
      sincospi(t, &s1, &c1);
      sincospi(2.0 * t, &s2, &c2);
      if (d == 0) { const double gx[5] = {c1, s2 * c1, c2 * s1, s2 * c1, s2 * c1}; return gx[k]; }
      if (d == 1) { const double gy[5] = {c1, c2 * c1, c2 * c1, s2 * s1, c2 * c1}; return gy[k]; }
      const double e = exp(t);
      const double gz[5] = {e, s2 * e, s2 * e, s2 * e, c2 * e};
      return gz[k];
    }
    case 5: { const double c = P.params[43 + d], s = P.params[46]; return exp(-(t - c) * (t - c) / (2.0 * s * s)); }
    case 11: return sin(0.5 * pi * t);
    case 12: return d == 0 ? sin(1.5 * pi * t) : (d == 1 ? sin(0.5 * pi * t) : exp(t));
    default: return 1.0;
  }
}

// L_{k,d}(i), i = 0..n_d, for term k and axis d stored at L[(3 k + d) * (nmax + 1) + i]
__global__ void k_load1d(const LevelGeom g, const Problem pb, double* __restrict__ L, int stride) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, d = blockIdx.y % 3, k = blockIdx.y / 3;
  if (i > g.n[d] || k >= kMaxSepRank) return;
  double v = 0.0;
  for (int e = i - 1; e <= i; ++e) {
    if (e < 0 || e >= g.n[d]) continue;
    const double side = (e == i - 1) ? 1.0 : -1.0;   // node is local 1 (xi = +1) of e = i-1, local 0 of e = i
    for (int q = 0; q < 2; ++q) {
      const double xi = q ? kGauss : -kGauss;
      v += sep_g(pb, k, d, g.lo[d] + (e + (1.0 + xi) / 2.0) * g.h[d]) * ((1.0 + side * xi) / 2.0) * (g.h[d] / 2.0);
    }
  }
  L[(long long)blockIdx.y * stride + i] = v;
}

__global__ void k_rhs_sep(const LevelGeom g, const Problem pb, const double* __restrict__ L, int stride,
                          double* __restrict__ b) {
  const int fx = blockIdx.x * blockDim.x + threadIdx.x, fy = blockIdx.y, lz = g.zbeg + blockIdx.z;
  if (fx >= g.nf[0]) return;
  const int R = prob_sep_rank(pb.id);
  double v = 0.0;
  for (int k = 0; k < R; ++k) {
    const double* Lk = L + 3LL * k * stride;
    v += sep_amp(pb, k) * __ldg(Lk + g.flo[0] + fx) * __ldg(Lk + stride + g.flo[1] + fy) *
         __ldg(Lk + 2 * stride + g.flo[2] + g.zoff + lz);
  }
  b[(long long)lz * g.S + (long long)fy * g.P + fx] = v;
}

// f specialised per problem at compile time (PID = 0: generic registry switch)
template <int PID>
__device__ __forceinline__ double f_at(const Problem& pb, double x, double y, double z) {
  return prob_f(pb, x, y, z);
}

template <int PID>
__global__ void __launch_bounds__(VNTH, 3) k_rhs_vol(const LevelGeom g, const Problem pb, double* __restrict__ b, int zc) {
  extern __shared__ double vs[];
  // structure-of-arrays layouts (consecutive threads -> consecutive doubles: no bank conflicts)
  double* fq = vs;              // fq[q * VNE + e]: f at Gauss point q of element e of the plane
  double* Fe = vs + VNE * 8;    // Fe[slot][a * VNE + e]: element load vectors, ring of two planes
  const int lane = threadIdx.x, w = threadIdx.y, tid = lane + 32 * w;
  const int X0 = blockIdx.x * VX, Y0 = blockIdx.y * VY;
  const int z0 = g.zbeg + blockIdx.z * zc, z1 = min(z0 + zc, g.zend);   // local planes
  const double detJ = g.h[0] * g.h[1] * g.h[2] / 8.0;
  const double wA = (1.0 + kGauss) / 2.0, wB = (1.0 - kGauss) / 2.0;   // N at the near / far Gauss point
  for (int fez = z0 - 1; fez < z1; ++fez) {
    // (a) f at the 8 Gauss points of every element of the plane (33 x 9 x 8 evaluations)
    const int gez = g.flo[2] + g.zoff + fez;
    for (int t = tid; t < VNE * 8; t += VNTH) {
      const int q = t / VNE, e = t - q * VNE;
      const int gex = g.flo[0] + X0 - 1 + e % VEX, gey = g.flo[1] + Y0 - 1 + e / VEX;
      double v = 0.0;
      if (PID == PROB_ARRAYS) {   // the caller's f at Gauss point q of the element
        if (gex >= 0 && gex < g.n[0] && gey >= 0 && gey < g.n[1] && gez >= 0 && gez < g.n[2] && pb.arr[1])
          v = pb.arr[1][8 * ((long long)gex + g.n[0] * ((long long)gey + (long long)g.n[1] * gez)) + q];
      } else if (gex >= 0 && gex < g.n[0] && gey >= 0 && gey < g.n[1] && gez >= 0 && gez < g.n[2]) {
        const double xi = (q & 1) ? kGauss : -kGauss, eta = (q & 2) ? kGauss : -kGauss, ze = (q & 4) ? kGauss : -kGauss;
        v = f_at<PID>(pb, g.lo[0] + (gex + (1.0 + xi) / 2.0) * g.h[0], g.lo[1] + (gey + (1.0 + eta) / 2.0) * g.h[1],
                      g.lo[2] + (gez + (1.0 + ze) / 2.0) * g.h[2]);
      }
      fq[t] = v;
    }
    __syncthreads();
    // (b) element load vectors F_e[a] = detJ sum_q f_q N_a(q): a 2x2x2 tensor transform
    double* Fp = Fe + (fez & 1) * VNE * 8;
    for (int e = tid; e < VNE; e += VNTH) {
      double f[8], t1[8], t2[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) f[q] = fq[q * VNE + e];
#pragma unroll
      for (int i = 0; i < 8; ++i) {   // along x: node bit 0 vs Gauss bit 0
        const int qb = i & ~1;
        t1[i] = (i & 1) ? (wB * f[qb] + wA * f[qb | 1]) : (wA * f[qb] + wB * f[qb | 1]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {   // along y
        const int qb = i & ~2;
        t2[i] = (i & 2) ? (wB * t1[qb] + wA * t1[qb | 2]) : (wA * t1[qb] + wB * t1[qb | 2]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {   // along z
        const int qb = i & ~4;
        Fp[i * VNE + e] = detJ * ((i & 4) ? (wB * t2[qb] + wA * t2[qb | 4]) : (wA * t2[qb] + wB * t2[qb | 4]));
      }
    }
    __syncthreads();
    // (c) node plane fz = fez gathers from element planes fez-1 and fez
    const int fz = fez, fx = X0 + lane, fy = Y0 + w;
    if (fz >= z0 && lane < VX && w < VY && fx < g.nf[0] && fy < g.nf[1]) {
      double v = 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int ex = e & 1, ey = (e >> 1) & 1, ez = (e >> 2) & 1;   // element = node - 1 + e_d
        const int a = (1 - ex) | ((1 - ey) << 1) | ((1 - ez) << 2);
        v += Fe[((fz - 1 + ez) & 1) * VNE * 8 + a * VNE + (lane + ex) + VEX * (w + ey)];
      }
      b[(long long)fz * g.S + (long long)fy * g.P + fx] = v;
    }
  }
}

// fp64 constants of k_rhs_c4 as kernel parameters (constant bank operands instead of per-use
// immediate materialisation)
struct RhsC4Consts {
  double wA, wB;   // N at the near / far Gauss point
  double dA, dB;   // detJ * (-15/4) * wA, wB: the z pass of the contraction
  double one, c3;   // 1, 1/4: y (1 + e/4)
};

// (r^2)^{-1/4} to fp64 accuracy. fp32 seed: r^2 rounded to fp32 (F2F), rsqrt.approx and sqrt.approx (MUFU,
// relative error ~3e-7) and one fp32 Newton step of y <- y (5 - x y^4) / 4 (to ~1e-7, the fp32 rounding
// level); y widened to fp64 exactly by bit operations (no second F2F: the XU pipe that executes MUFU and
// F2F is this kernel's limit, 3 instead of 4 XU instructions per Gauss point); then one fp64 step in the
// form y (1 + e/4), e = 1 - r^2 y^4 (error 5e^2/32: ~3e-14). r^2 > 0 at every Gauss point (interior to
// the elements) and stays in the normal fp32 range on every level.
__device__ __forceinline__ double rpow_m14(double r2, const RhsC4Consts& k) {
  const float xf = (float)r2;   // (an F2F-free narrowing by integer operations measured no faster: 1.762 ms either way)
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(xf));
  asm("sqrt.approx.ftz.f32 %0, %0;" : "+f"(y));
  const float y2f = y * y;
  y = (y * 0.25f) * fmaf(-xf, y2f * y2f, 5.0f);
  const unsigned yb = __float_as_uint(y);
  const double yd = __hiloint2double((int)((yb >> 3) + ((1023u - 127u) << 20)), (int)(yb << 29));
  const double y2 = yd * yd;
  const double e = __fma_rn(-r2, y2 * y2, k.one);
  return __fma_rn(yd * k.c3, e, yd);
}

// C4 volume load (f = -(15/4) r^{-1/2}, the corner singularity of u = r^{3/2}). 512 threads = 32 x 16
// elements per plane (node tile 31 x 15), one element per thread, z-marching over element layers. r^2 at a
// Gauss point is (x^2 + y^2) + z^2 with the four in-plane sums fixed per thread and z^2 per layer, so a
// Gauss point costs one add and the (r^2)^{-1/4} evaluation. The 2x2x2 Gauss load of node i,
// F_i = detJ sum_{q} f_q N_i(q) over the 64 Gauss points of its 8 elements, factorises per axis (the 1D
// weight of a Gauss point is wA at the point nearer the node, wB at the farther one) and is contracted
// axis by axis: x within the thread, then the right node column takes its left neighbour element's
// share by a warp shuffle; y the same across warps through shared memory; z with the lower layer's share
// carried in a register. ~75 fp64 operations per element instead of ~113 for the 8 x 8 element-vector
// transform. Work items (tile, z chunk) are linear, taken by a grid-stride loop.
constexpr int C4X = 31, C4Y = 15, C4NTH = 512;
#ifndef RHS_C4_MINB
#define RHS_C4_MINB 2
#endif
__global__ void __launch_bounds__(C4NTH, RHS_C4_MINB) k_rhs_c4(const LevelGeom g, double* __restrict__ b, int zc,
                                                    const RhsC4Consts k, int tx, int ty, int items) {
  __shared__ double lo_s[2][2][16][32];   // [layer parity][qz][element row][lane]: y share of the row below
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double ga = (1.0 - kGauss) / 2.0, gb = (1.0 + kGauss) / 2.0;   // Gauss points at xi = -+1/sqrt(3)
  const double wA = k.wA, wB = k.wB, dA = k.dA, dB = k.dB;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int X0 = (item % tx) * C4X, Y0 = ((item / tx) % ty) * C4Y;
    const int z0 = g.zbeg + (item / (tx * ty)) * zc, z1 = min(z0 + zc, g.zend);   // local planes
    const int gex = g.flo[0] + X0 - 1 + lane, gey = g.flo[1] + Y0 - 1 + w;
    const bool xy_in = gex >= 0 && gex < g.n[0] && gey >= 0 && gey < g.n[1];
    const double xa = g.lo[0] + (gex + ga) * g.h[0], xb = g.lo[0] + (gex + gb) * g.h[0];
    const double ya = g.lo[1] + (gey + ga) * g.h[1], yb = g.lo[1] + (gey + gb) * g.h[1];
    const double sxy[2][2] = {{xa * xa + ya * ya, xb * xb + ya * ya}, {xa * xa + yb * yb, xb * xb + yb * yb}};   // [qy][qx]
    const int fx = X0 + lane, fy = Y0 + w;
    const bool node_ok = lane < C4X && w < C4Y && fx < g.nf[0] && fy < g.nf[1];
    double carry = 0.0;
    int par = 0;
    for (int fez = z0 - 1; fez < z1; ++fez, par ^= 1) {
      const int gez = g.flo[2] + g.zoff + fez;
      double X[2][2];   // [qy][qz]: x-contracted load of node column fx (this element's right node)
      {
        double h0[2][2], h1[2][2];
        if (xy_in && gez >= 0 && gez < g.n[2]) {
          const double za = g.lo[2] + (gez + ga) * g.h[2], zb = g.lo[2] + (gez + gb) * g.h[2];
          const double z2[2] = {za * za, zb * zb};
#pragma unroll
          for (int qy = 0; qy < 2; ++qy)
#pragma unroll
            for (int qz = 0; qz < 2; ++qz) {
              const double fa = rpow_m14(sxy[qy][0] + z2[qz], k);
              const double fb = rpow_m14(sxy[qy][1] + z2[qz], k);
              h0[qy][qz] = __fma_rn(wA, fa, wB * fb);   // to the element's left node
              h1[qy][qz] = __fma_rn(wB, fa, wA * fb);   // to its right node
            }
        } else {
#pragma unroll
          for (int qy = 0; qy < 2; ++qy)
#pragma unroll
            for (int qz = 0; qz < 2; ++qz) h0[qy][qz] = h1[qy][qz] = 0.0;
        }
#pragma unroll
        for (int qy = 0; qy < 2; ++qy)
#pragma unroll
          for (int qz = 0; qz < 2; ++qz) X[qy][qz] = h1[qy][qz] + __shfl_down_sync(0xffffffffu, h0[qy][qz], 1);
      }
      // y: node row fy = element row + 1 takes hi of this row and lo of the row above
      double hi[2];
#pragma unroll
      for (int qz = 0; qz < 2; ++qz) {
        lo_s[par][qz][w][lane] = __fma_rn(wA, X[0][qz], wB * X[1][qz]);
        hi[qz] = __fma_rn(wB, X[0][qz], wA * X[1][qz]);
      }
      __syncthreads();
      if (node_ok) {
        const double Ya = hi[0] + lo_s[par][0][w + 1][lane];
        const double Yb = hi[1] + lo_s[par][1][w + 1][lane];
        if (fez >= z0) b[(long long)fez * g.S + (long long)fy * g.P + fx] = carry + __fma_rn(dA, Ya, dB * Yb);
        carry = __fma_rn(dB, Ya, dA * Yb);
      }
    }
    __syncthreads();   // lo_s of this item's last layers consumed before the next item
  }
}

// C4 volume load on a cubic level (same n, h, lo and free box along the three axes): f depends on r only, so the
// load is invariant under every permutation of the node indices, F(i, j, k) = F(j, i, k) = F(i, k, j) = ...
// The free box is cut into cubic tiles of 31^3 nodes, tile index (a, b, c) along (x, y, z), and only about a third
// of them is evaluated; the others are written as permuted copies by the CTA that evaluates their image:
//   * a >= b >= c: the tile itself; its x<->y transpose at (b, a, c) if a != b; its y<->z swap at (a, c, b) if
//     b != c; the image (i, j, k) -> (j, k, i) at (b, c, a) if a != b;
//   * a < c <= b (x strictly lowest): the tile itself and its y<->z swap at (a, c, b) if b != c.
// Every tile of the box is written exactly once (the cases are disjoint and cover all index triples), every store
// is a row segment along x (the transposes go through shared memory), and a value is the same function of its
// three Gauss abscissa sets whichever image carries it, so the result differs from k_rhs_c4's by rounding order only.
// 1024 threads = 32 x 32 elements per plane (node tile 31 x 31), the same per-element arithmetic as k_rhs_c4.
constexpr int C4S = 31, C4SNTH = 1024;
#ifndef C4S_ZCH
#define C4S_ZCH 2   // z chunks per tile (a chunk re-evaluates one element layer; shorter CTAs give way sooner to the
                    // high-priority coarse solves: measured 1 / 2 / 4, profiles/r02/tuning/ab_rhs_sym_variants.log)
#endif
constexpr int C4SZ = (C4S + C4S_ZCH - 1) / C4S_ZCH;
__global__ void __launch_bounds__(C4SNTH, 1) k_rhs_c4_sym(const LevelGeom g, double* __restrict__ b, const RhsC4Consts k) {
  const int ta = blockIdx.x, tb = blockIdx.y, tc = blockIdx.z / C4S_ZCH, ch = blockIdx.z % C4S_ZCH;
  const bool canon = ta >= tb && tb >= tc, lowx = ta < tc && tc <= tb;
  if (!canon && !lowx) return;
  const bool f_xy = canon && ta != tb;    // (i, j, k) -> (j, i, k) at tile (b, a, c)
  const bool f_yz = tb != tc;             // (i, j, k) -> (i, k, j) at tile (a, c, b)
  const bool f_rot = canon && ta != tb;   // (i, j, k) -> (j, k, i) at tile (b, c, a)
  __shared__ double lo_s[2][2][32][32];   // [layer parity][qz][element row][lane]: y share of the row below
  __shared__ double tr[32][33];           // in-plane transpose of the node plane
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double ga = (1.0 - kGauss) / 2.0, gb = (1.0 + kGauss) / 2.0;   // Gauss points at xi = -+1/sqrt(3)
  const double wA = k.wA, wB = k.wB, dA = k.dA, dB = k.dB;
  const int X0 = ta * C4S, Y0 = tb * C4S, z0 = tc * C4S + ch * C4SZ, z1 = min(min(z0 + C4SZ, (tc + 1) * C4S), g.nf[2]);
  if (z0 >= z1) return;
  const int gex = g.flo[0] + X0 - 1 + lane, gey = g.flo[1] + Y0 - 1 + w;
  const bool xy_in = gex >= 0 && gex < g.n[0] && gey >= 0 && gey < g.n[1];
  const double xa = g.lo[0] + (gex + ga) * g.h[0], xb = g.lo[0] + (gex + gb) * g.h[0];
  const double ya = g.lo[1] + (gey + ga) * g.h[1], yb = g.lo[1] + (gey + gb) * g.h[1];
  const double sxy[2][2] = {{xa * xa + ya * ya, xb * xb + ya * ya}, {xa * xa + yb * yb, xb * xb + yb * yb}};   // [qy][qx]
  const int fx = X0 + lane, fy = Y0 + w;
  const bool node_ok = lane < C4S && w < C4S && fx < g.nf[0] && fy < g.nf[1];
  // the transposed node of this thread: (i, j) = (w, lane) of the tile
  const int tx = Y0 + lane, ty = X0 + w;
  const bool tnode_ok = lane < C4S && w < C4S && tx < g.nf[1] && ty < g.nf[0];
  double carry = 0.0;
  int par = 0;
  for (int fez = z0 - 1; fez < z1; ++fez, par ^= 1) {
    const int gez = g.flo[2] + fez;
    double X[2][2];   // [qy][qz]: x-contracted load of node column fx (this element's right node)
    {
      double h0[2][2], h1[2][2];
      if (xy_in && gez >= 0 && gez < g.n[2]) {
        const double za = g.lo[2] + (gez + ga) * g.h[2], zb = g.lo[2] + (gez + gb) * g.h[2];
        const double z2[2] = {za * za, zb * zb};
#pragma unroll
        for (int qy = 0; qy < 2; ++qy)
#pragma unroll
          for (int qz = 0; qz < 2; ++qz) {
            const double fa = rpow_m14(sxy[qy][0] + z2[qz], k);
            const double fb = rpow_m14(sxy[qy][1] + z2[qz], k);
            h0[qy][qz] = __fma_rn(wA, fa, wB * fb);   // to the element's left node
            h1[qy][qz] = __fma_rn(wB, fa, wA * fb);   // to its right node
          }
      } else {
#pragma unroll
        for (int qy = 0; qy < 2; ++qy)
#pragma unroll
          for (int qz = 0; qz < 2; ++qz) h0[qy][qz] = h1[qy][qz] = 0.0;
      }
#pragma unroll
      for (int qy = 0; qy < 2; ++qy)
#pragma unroll
        for (int qz = 0; qz < 2; ++qz) X[qy][qz] = h1[qy][qz] + __shfl_down_sync(0xffffffffu, h0[qy][qz], 1);
    }
    double hi[2];
#pragma unroll
    for (int qz = 0; qz < 2; ++qz) {
      lo_s[par][qz][w][lane] = __fma_rn(wA, X[0][qz], wB * X[1][qz]);
      hi[qz] = __fma_rn(wB, X[0][qz], wA * X[1][qz]);
    }
    __syncthreads();   // (also: every thread has read tr of the previous plane)
    double v = 0.0;
    if (node_ok) {
      const double Ya = hi[0] + lo_s[par][0][w + 1][lane];
      const double Yb = hi[1] + lo_s[par][1][w + 1][lane];
      v = carry + __fma_rn(dA, Ya, dB * Yb);
      carry = __fma_rn(dB, Ya, dA * Yb);
    }
    if (fez < z0) continue;   // (CTA-uniform) the layer below the tile only feeds carry
    if (node_ok) {
      b[(long long)fez * g.S + (long long)fy * g.P + fx] = v;
      if (f_yz) b[(long long)fy * g.S + (long long)fez * g.P + fx] = v;
    }
    if (f_xy) {   // (CTA-uniform)
      tr[w][lane] = v;
      __syncthreads();
      if (tnode_ok) {
        const double vt = tr[lane][w];
        b[(long long)fez * g.S + (long long)ty * g.P + tx] = vt;
        if (f_rot) b[(long long)ty * g.S + (long long)fez * g.P + tx] = vt;
      }
    }
  }
}

// the symmetric C4 load applies when the level is a cube in every respect the load depends on
static bool rhs_c4_sym_ok(const LevelGeom& g, int sym_min) {
  if (sym_min <= 0) return false;
  for (int d = 1; d < 3; ++d)
    if (g.n[d] != g.n[0] || g.nf[d] != g.nf[0] || g.flo[d] != g.flo[0] || g.h[d] != g.h[0] || g.lo[d] != g.lo[0]) return false;
  return g.zoff == 0 && g.zbeg == 0 && g.zend == g.nf[2] && g.nf[0] >= sym_min;
}

__device__ __forceinline__ int sel3(int d, int a, int b, int c) { return d == 0 ? a : (d == 1 ? b : c); }

// Boundary shell of the free box: Robin load G and lifting -A_fD g_D, added to b.
// blockIdx.z = face of the free box (axis d = face/2, side = face&1); a node is handled by the
// lowest-numbered free-box face it lies on.
__global__ void k_rhs_shell(const LevelGeom g, const Problem pb, const ElemStencil es, double beta_const,
                            const double* __restrict__ beta, double* __restrict__ b) {
  const int face = blockIdx.z, d = face >> 1, side = face & 1;
  const int d1 = (d == 0) ? 1 : 0, d2 = (d == 2) ? 1 : 2;
  // extents of the face in global free coordinates; z is restricted to this rank's planes
  const int zb = g.zoff + g.zbeg, ze = g.zoff + g.zend;
  const int ext1 = (d1 == 2) ? ze - zb : g.nf[d1], off1 = (d1 == 2) ? zb : 0;
  const int ext2 = (d2 == 2) ? ze - zb : g.nf[d2], off2 = (d2 == 2) ? zb : 0;
  const int i1 = blockIdx.x * blockDim.x + threadIdx.x, i2 = blockIdx.y;
  if (i1 >= ext1 || i2 >= ext2) return;
  // free-box coordinates of the node (scalars: no dynamically indexed local arrays)
  const int fx = d == 0 ? (side ? g.nf[0] - 1 : 0) : off1 + i1;
  const int fy = d == 1 ? (side ? g.nf[1] - 1 : 0) : (d == 0 ? off1 + i1 : off2 + i2);
  const int fz = d == 2 ? (side ? g.nf[2] - 1 : 0) : off2 + i2;
  if (d == 2 && (fz < zb || fz >= ze)) return;   // z face not in this slab
#pragma unroll
  for (int fc = 0; fc < 5; ++fc) {   // owned by a lower face?
    if (fc >= face) break;
    const int dd = fc >> 1;
    if (sel3(dd, fx, fy, fz) == ((fc & 1) ? g.nf[dd] - 1 : 0)) return;
  }
  const int gx = g.flo[0] + fx, gy = g.flo[1] + fy, gz = g.flo[2] + fz;
  double v = 0.0;
  // Robin face load G = sum_q g_R(x_q) N_c h1 h2 / 4 on every Robin face through the node
#pragma unroll
  for (int F = 0; F < 6; ++F) {
    if (pb.face[F] != FACE_ROBIN) continue;
    const int dF = F >> 1;
    if (sel3(dF, gx, gy, gz) != ((F & 1) ? g.n[dF] : 0)) continue;
    const int e1d = (dF == 0) ? 1 : 0, e2d = (dF == 2) ? 1 : 2;
    const double hh = g.h[e1d] * g.h[e2d] / 4.0;
    long long gR_block = 0;   // PROB_ARRAYS: this face's block of g_R values (faces in order, 4 n_d1 n_d2 each)
    for (int F2 = 0; F2 < F; ++F2) {
      const int a = F2 >> 1;
      gR_block += 4LL * g.n[(a == 0) ? 1 : 0] * g.n[(a == 2) ? 1 : 2];
    }
    for (int e2 = -1; e2 <= 0; ++e2)
      for (int e1 = -1; e1 <= 0; ++e1) {
        const int f1 = sel3(e1d, gx, gy, gz) + e1, f2 = sel3(e2d, gx, gy, gz) + e2;
        if (f1 < 0 || f1 >= g.n[e1d] || f2 < 0 || f2 >= g.n[e2d]) continue;
        for (int q = 0; q < 4; ++q) {
          const double xi1 = (q & 1) ? kGauss : -kGauss, xi2 = (q & 2) ? kGauss : -kGauss;
          double xq[3];
          xq[dF] = g.lo[dF] + sel3(dF, gx, gy, gz) * g.h[dF];
          xq[e1d] = g.lo[e1d] + (f1 + (1.0 + xi1) / 2.0) * g.h[e1d];
          xq[e2d] = g.lo[e2d] + (f2 + (1.0 + xi2) / 2.0) * g.h[e2d];
          const double N = ((1.0 + (e1 ? xi1 : -xi1)) / 2.0) * ((1.0 + (e2 ? xi2 : -xi2)) / 2.0);
          const double gR = pb.id == PROB_ARRAYS
                                ? (pb.arr[3] ? pb.arr[3][gR_block + 4LL * (f1 + (long long)g.n[e1d] * f2) + q] : 0.0)
                                : prob_gR(pb, F, xq[0], xq[1], xq[2]);
          v += gR * N * hh;
        }
      }
  }
  // lifting: couplings to Dirichlet neighbours (domain nodes outside the free box)
  double sub = 0.0;
  bool any_robin = false;
#pragma unroll
  for (int F = 0; F < 6; ++F) any_robin = any_robin || es.robin[F] != 0.0;
  for (int e = 0; e < 8; ++e) {
    const int ex = e & 1, ey = (e >> 1) & 1, ez = (e >> 2) & 1;
    const int ge[3] = {gx - 1 + ex, gy - 1 + ey, gz - 1 + ez};
    if (ge[0] < 0 || ge[0] >= g.n[0] || ge[1] < 0 || ge[1] >= g.n[1] || ge[2] < 0 || ge[2] >= g.n[2]) continue;
    const double be = beta ? beta[(long long)(ge[2] + 2) * g.BS + (long long)(ge[1] + 2) * g.BP + (ge[0] + 2)] : beta_const;
    for (int bn = 0; bn < 8; ++bn) {
      const int bx = bn & 1, by = (bn >> 1) & 1, bz = (bn >> 2) & 1;
      const int jx = ge[0] + bx, jy = ge[1] + by, jz = ge[2] + bz;
      const bool jfree = jx >= g.flo[0] && jx < g.flo[0] + g.nf[0] && jy >= g.flo[1] && jy < g.flo[1] + g.nf[1] &&
                         jz >= g.flo[2] && jz < g.flo[2] + g.nf[2];
      if (jfree) continue;
      const double gD = prob_gD_node(pb, g, jx, jy, jz);
      const int pat = ((ex + bx) != 1 ? 1 : 0) | ((ey + by) != 1 ? 2 : 0) | ((ez + bz) != 1 ? 4 : 0);
      sub += be * es.kappa[pat] * gD;
      if (!any_robin) continue;   // (all-Dirichlet problems: most of the pairs; the face loop below is 6 tests each)
      // Robin face mass between this node and the Dirichlet node j on a common Robin face
#pragma unroll
      for (int F = 0; F < 6; ++F) {
        if (es.robin[F] == 0.0) continue;
        const int dF = F >> 1;
        const int plane = (F & 1) ? g.n[dF] : 0;
        if (sel3(dF, gx, gy, gz) != plane || sel3(dF, jx, jy, jz) != plane) continue;
        if (es.aq) {   // alpha at the face Gauss points: the entry of this volume element's face element
          const int t1 = dF == 0 ? 1 : 0, t2 = dF == 2 ? 1 : 2;
          const int e1 = ge[t1], e2 = ge[t2];
          const double* a4 = robin_aq(es.aq, g.n, F, e1, e2);
          sub += robin_elem_entry(a4, sel3(t1, gx, gy, gz) - e1, sel3(t2, gx, gy, gz) - e2, sel3(t1, jx, jy, jz) - e1,
                                  sel3(t2, jx, jy, jz) - e2, es.robin[F]) * gD;
          continue;
        }
        const int nd = (dF != 0 && jx != gx) + (dF != 1 && jy != gy) + (dF != 2 && jz != gz);
        sub += es.robin[F] * (nd == 0 ? (1.0 / 9.0) : (nd == 1 ? (1.0 / 18.0) : (1.0 / 36.0))) * gD;
      }
    }
  }
  if (v != 0.0 || sub != 0.0) b[(long long)(fz - g.zoff) * g.S + (long long)fy * g.P + fx] += v - sub;
}

// ---- gather / scatter between full nodal vectors and the free box ------------------------------
__global__ void k_gather(const LevelGeom g, const double* __restrict__ u, double* __restrict__ x) {
  const int fx = blockIdx.x * blockDim.x + threadIdx.x;
  const int fy = blockIdx.y, lz = g.zbeg + blockIdx.z;
  if (fx >= g.nf[0]) return;
  const long long nx = g.n[0] + 1, ny = g.n[1] + 1;
  const long long gi = (long long)(g.flo[0] + fx) + nx * ((long long)(g.flo[1] + fy) + ny * (g.flo[2] + g.zoff + lz));
  x[(long long)lz * g.S + (long long)fy * g.P + fx] = u[gi];
}

__global__ void k_scatter(const LevelGeom g, const double* __restrict__ x, double* __restrict__ u) {
  const int fx = blockIdx.x * blockDim.x + threadIdx.x;
  const int fy = blockIdx.y, lz = g.zbeg + blockIdx.z;
  if (fx >= g.nf[0]) return;
  const long long nx = g.n[0] + 1, ny = g.n[1] + 1;
  const long long gi = (long long)(g.flo[0] + fx) + nx * ((long long)(g.flo[1] + fy) + ny * (g.flo[2] + g.zoff + lz));
  u[gi] = x[(long long)lz * g.S + (long long)fy * g.P + fx];
}

// Dirichlet nodes (outside the free box) of a full nodal vector := g_D (or 0). One launch for all
// faces: blockIdx.z = face (non-Dirichlet faces return); nodes on shared edges are written twice with
// the same value.
__global__ void k_dirichlet_face(const LevelGeom g, const Problem pb, double* __restrict__ u, int zero) {
  const int F = blockIdx.z;
  if (pb.face[F] != FACE_DIRICHLET) return;
  const int d = F >> 1, side = F & 1;
  const int d1 = (d == 0) ? 1 : 0, d2 = (d == 2) ? 1 : 2;
  const int i1 = blockIdx.x * blockDim.x + threadIdx.x, i2 = blockIdx.y;
  if (i1 > g.n[d1] || i2 > g.n[d2]) return;
  int gi[3];
  gi[d] = side ? g.n[d] : 0;
  gi[d1] = i1;
  gi[d2] = i2;
  if (gi[2] < g.zlo || gi[2] >= g.zhi) return;   // only this rank's planes
  const long long nx = g.n[0] + 1, ny = g.n[1] + 1;
  const double v = zero ? 0.0 : prob_gD_node(pb, g, gi[0], gi[1], gi[2]);
  u[(long long)gi[0] + nx * ((long long)gi[1] + ny * gi[2])] = v;
}

__global__ void k_zero_free(const LevelGeom g, double* __restrict__ v) {
  const int fx = blockIdx.x * blockDim.x + threadIdx.x;
  if (fx >= g.nf[0]) return;
  v[(long long)blockIdx.z * g.S + (long long)blockIdx.y * g.P + fx] = 0.0;   // all allocated planes
}

}  // namespace

// beta array of the level and, behind it, the per-axis tables it is formed from (beta_combine)
cudaError_t launch_beta(const LevelGeom& g, const Problem& pb, double* beta, cudaStream_t st) {
  if (pb.id == PROB_ARRAYS) {
    const long long total = (long long)(g.n[0] + 4) * (g.n[1] + 4) * (g.n[2] + 4);
    count_launch();
    k_beta_arr<<<(int)std::min<long long>((total + 255) / 256, 148LL * 32), 256, 0, st>>>(g, beta, pb.arr[0]);
    return cudaGetLastError();
  }
  const int W = beta_axes_w(g), kind = beta_kind(pb.id);
  double* tab = beta + g.BS * (g.n[2] + 4);
  count_launch();
  k_beta_axes<<<(3 * W + 127) / 128, 128, 0, st>>>(g, pb, tab, W, kind);
  const long long total = (long long)(g.n[0] + 4) * (g.n[1] + 4) * (g.n[2] + 4);
  const int nb = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  count_launch();
  k_beta<<<nb, 256, 0, st>>>(g, beta, tab, W, kind);
  return cudaGetLastError();
}

cudaError_t init_setup_kernel_attributes() {
  cudaError_t e = cudaFuncSetAttribute(k_rhs_vol<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, VSMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_rhs_vol<PROB_ARRAYS>, cudaFuncAttributeMaxDynamicSharedMemorySize, VSMEM);
  return e;
}

cudaError_t launch_rhs(const LevelGeom& g, const Problem& pb, const ElemStencil& es, double beta_const, const double* beta,
                       double* b, double* scratch, cudaStream_t st, int ctas_per_sm, int sym_min) {
  // an empty free box (a level of 1 cell along an all-Dirichlet axis): there is no right-hand side to form
  if (g.nf[0] <= 0 || g.nf[1] <= 0 || g.zend <= g.zbeg) return cudaSuccess;
  if (prob_separable(pb.id)) {
    const int nmax = std::max(g.n[0], std::max(g.n[1], g.n[2]));
    const int stride = nmax + 1;
    dim3 g1((stride + 127) / 128, 3 * prob_sep_rank(pb.id));
    count_launch();
    k_load1d<<<g1, 128, 0, st>>>(g, pb, scratch, stride);
    dim3 g2((g.nf[0] + 127) / 128, g.nf[1], g.zend - g.zbeg);
    count_launch();
    k_rhs_sep<<<g2, 128, 0, st>>>(g, pb, scratch, stride, b);
  } else {
    // element planes per CTA: 32 on large levels (a chunk re-evaluates one element plane), shorter on
    // small ones so that the grid has ~1000 CTAs instead of a few long serial chains
    const bool c4 = pb.id == 4;
    const int TX = c4 ? C4X : VX, TY = c4 ? C4Y : VY;
    const long long tiles = (long long)((g.nf[0] + TX - 1) / TX) * ((g.nf[1] + TY - 1) / TY);
    const int nz = g.zend - g.zbeg;
#ifndef RHS_ZC_MAX
#define RHS_ZC_MAX 32
#endif
    const int zc = (int)std::max(4LL, std::min((long long)RHS_ZC_MAX, tiles * nz / (c4 ? 500 : 1000)));
    dim3 grid((g.nf[0] + TX - 1) / TX, (g.nf[1] + TY - 1) / TY, (nz + zc - 1) / zc);
    count_launch();
    if (c4) {
      RhsC4Consts k;
      k.wA = (1.0 + kGauss) / 2.0;
      k.wB = (1.0 - kGauss) / 2.0;
      const double detJ = -3.75 * (g.h[0] * g.h[1] * g.h[2] / 8.0);   // f = -15/4 (r^2)^{-1/4}
      k.dA = detJ * k.wA;
      k.dB = detJ * k.wB;
      k.one = 1.0; k.c3 = 0.25;
      if (rhs_c4_sym_ok(g, sym_min)) {
        const int nt = (g.nf[0] + C4S - 1) / C4S;
        k_rhs_c4_sym<<<dim3(nt, nt, nt * C4S_ZCH), C4SNTH, 0, st>>>(g, b, k);
      } else {
        const int items = (int)(grid.x * grid.y * grid.z);
        int nblk = items;
        if (ctas_per_sm > 0) {
          int dev = 0, sms = 148;
          cudaGetDevice(&dev);
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
          nblk = std::min(items, sms * ctas_per_sm);
        }
        k_rhs_c4<<<nblk, C4NTH, 0, st>>>(g, b, zc, k, (int)grid.x, (int)grid.y, items);
      }
    }
    else if (pb.id == PROB_ARRAYS) k_rhs_vol<PROB_ARRAYS><<<grid, dim3(32, 8), VSMEM, st>>>(g, pb, b, zc);
    else k_rhs_vol<0><<<grid, dim3(32, 8), VSMEM, st>>>(g, pb, b, zc);
  }
  const int m = std::max(g.nf[0], std::max(g.nf[1], g.nf[2]));
  dim3 gs((m + 127) / 128, m, 6);
  count_launch();
  k_rhs_shell<<<gs, 128, 0, st>>>(g, pb, es, beta_const, beta, b);
  return cudaGetLastError();
}

cudaError_t launch_gather(const LevelGeom& g, const double* u, double* x, cudaStream_t st) {
  dim3 grid((g.nf[0] + 127) / 128, g.nf[1], g.zend - g.zbeg);
  count_launch();
  k_gather<<<grid, 128, 0, st>>>(g, u, x);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const LevelGeom& g, const double* x, double* u, cudaStream_t st) {
  dim3 grid((g.nf[0] + 127) / 128, g.nf[1], g.zend - g.zbeg);
  count_launch();
  k_scatter<<<grid, 128, 0, st>>>(g, x, u);
  return cudaGetLastError();
}

cudaError_t launch_dirichlet_fill(const LevelGeom& g, const Problem& pb, double* u, double, int zero_instead,
                                  cudaStream_t st) {
  bool any = false;
  for (int F = 0; F < 6; ++F) any = any || pb.face[F] == FACE_DIRICHLET;
  if (!any) return cudaSuccess;
  const int m = std::max(g.n[0], std::max(g.n[1], g.n[2])) + 1;
  dim3 grid((m + 127) / 128, m, 6);
  count_launch();
  k_dirichlet_face<<<grid, 128, 0, st>>>(g, pb, u, zero_instead);
  return cudaGetLastError();
}

cudaError_t launch_zero_vec(const LevelGeom& g, double* v, cudaStream_t st) {
  if (g.nf[0] <= 0 || g.nf[1] <= 0 || g.nza <= 0) return cudaSuccess;   // an empty free box
  dim3 grid((g.nf[0] + 127) / 128, g.nf[1], g.nza);
  count_launch();
  k_zero_free<<<grid, 128, 0, st>>>(g, v);
  return cudaGetLastError();
}

}  // namespace ecmg
