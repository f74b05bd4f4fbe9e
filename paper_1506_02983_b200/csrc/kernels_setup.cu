// kernels_setup.cu -- per-level setup of the Q1 system: element coefficients,
// load vector by 2x2x2 Gauss quadrature (reading §8c A2), Robin face load by 2x2 Gauss (§8c A4),
// symmetric Dirichlet elimination (lifting, §8c A5), ||f_h||_2, and the gather / scatter between
// caller-visible nodal vectors and the free-box work vectors.
#include "ecmg_internal.cuh"
#include "problems.cuh"

namespace ecmg {
namespace {

constexpr double kGauss = 0.57735026918962576451;  // 1/sqrt(3)

// ---- element coefficients beta_e = beta(centroid) (§8c A3), zero outside the domain ----------
__global__ void k_beta(const LevelGeom g, const Problem pb, double* __restrict__ beta) {
  const long long ne0 = g.n[0] + 4, ne1 = g.n[1] + 4, ne2 = g.n[2] + 4;
  const long long total = ne0 * ne1 * ne2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int ex = (int)(t % ne0) - 2, ey = (int)((t / ne0) % ne1) - 2, ez = (int)(t / (ne0 * ne1)) - 2;
    double v = 0.0;
    if (ex >= 0 && ex < g.n[0] && ey >= 0 && ey < g.n[1] && ez >= 0 && ez < g.n[2]) {
      v = prob_beta(pb, g.lo[0] + (ex + 0.5) * g.h[0], g.lo[1] + (ey + 0.5) * g.h[1], g.lo[2] + (ez + 0.5) * g.h[2]);
    }
    beta[(long long)(ez + 2) * g.BS + (long long)(ey + 2) * g.BP + (ex + 2)] = v;
  }
}

// ---- right-hand side ---------------------------------------------------------------------------
// CTA = 8 x 8 x 4 free nodes. Phase 1: the element load vectors F_e[a] = sum_q f(x_q) N_a(xi_q) V/8
// of the 9 x 9 x 5 elements touching the tile go to shared memory (each f evaluation done once
// per tile). Phase 2: each node gathers its 8 element entries, adds the Robin face load
// G = sum_q g_R(x_q) N_c h1 h2 / 4 and subtracts A_fD g_D (element-wise couplings beta_e kappa
// plus Robin face mass to Dirichlet neighbours), giving b_f = F_f + G_f - A_fD g_D.
constexpr int RX = 8, RY = 8, RZ = 4, RNTH = RX * RY * RZ;
constexpr int REX = RX + 1, REY = RY + 1, REZ = RZ + 1, RNE = REX * REY * REZ;

__device__ __forceinline__ double beta_at(const LevelGeom& g, const double* beta, double beta_const, int gex, int gey,
                                          int gez) {
  if (gex < 0 || gex >= g.n[0] || gey < 0 || gey >= g.n[1] || gez < 0 || gez >= g.n[2]) return 0.0;
  if (!beta) return beta_const;
  return beta[(long long)(gez + 2) * g.BS + (long long)(gey + 2) * g.BP + (gex + 2)];
}

__global__ void __launch_bounds__(RNTH) k_rhs(const LevelGeom g, const Problem pb, const ElemStencil es, double beta_const,
                                              const double* __restrict__ beta, double* __restrict__ b, double* partials,
                                              JcgScalars* sc) {
  __shared__ double Fe[RNE][8];
  __shared__ double red[2 * (RNTH / 32)];
  __shared__ int is_last;
  const int tid = threadIdx.x;
  const int X0 = blockIdx.x * RX, Y0 = blockIdx.y * RY, Z0 = blockIdx.z * RZ;
  const double detJ = g.h[0] * g.h[1] * g.h[2] / 8.0;

  // phase 1: element loads
  for (int e = tid; e < RNE; e += RNTH) {
    const int lx = e % REX, ly = (e / REX) % REY, lz = e / (REX * REY);
    const int gex = g.flo[0] + X0 - 1 + lx, gey = g.flo[1] + Y0 - 1 + ly, gez = g.flo[2] + Z0 - 1 + lz;
    double F[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) F[a] = 0.0;
    if (gex >= 0 && gex < g.n[0] && gey >= 0 && gey < g.n[1] && gez >= 0 && gez < g.n[2]) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double xi[3] = {(q & 1) ? kGauss : -kGauss, (q & 2) ? kGauss : -kGauss, (q & 4) ? kGauss : -kGauss};
        const double fq = prob_f(pb, g.lo[0] + (gex + (1.0 + xi[0]) / 2.0) * g.h[0],
                                 g.lo[1] + (gey + (1.0 + xi[1]) / 2.0) * g.h[1],
                                 g.lo[2] + (gez + (1.0 + xi[2]) / 2.0) * g.h[2]);
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const double N = ((1.0 + ((a & 1) ? xi[0] : -xi[0])) / 2.0) * ((1.0 + ((a & 2) ? xi[1] : -xi[1])) / 2.0) *
                           ((1.0 + ((a & 4) ? xi[2] : -xi[2])) / 2.0);
          F[a] += fq * N * detJ;
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) Fe[e][a] = F[a];
  }
  __syncthreads();

  // phase 2: nodes
  const int lx = tid % RX, ly = (tid / RX) % RY, lz = tid / (RX * RY);
  const int fx = X0 + lx, fy = Y0 + ly, fz = Z0 + lz;
  double bsq = 0.0;
  if (fx < g.nf[0] && fy < g.nf[1] && fz < g.nf[2]) {
    const int gx = g.flo[0] + fx, gy = g.flo[1] + fy, gz = g.flo[2] + fz;
    const int gi[3] = {gx, gy, gz};
    double v = 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ex = e & 1, ey = (e >> 1) & 1, ez = (e >> 2) & 1;   // element = node - 1 + e_d
      const int a = (1 - ex) | ((1 - ey) << 1) | ((1 - ez) << 2);    // node's local index in it
      v += Fe[(lx + ex) + REX * ((ly + ey) + REY * (lz + ez))][a];
    }
    // Robin faces: load G and face-mass coupling
    for (int F = 0; F < 6; ++F) {
      if (pb.face[F] != FACE_ROBIN) continue;
      const int d = F >> 1, side = F & 1;
      if (gi[d] != (side ? g.n[d] : 0)) continue;
      const int d1 = (d == 0) ? 1 : 0, d2 = (d == 2) ? 1 : 2;
      const double hh = g.h[d1] * g.h[d2] / 4.0;
      for (int e2 = -1; e2 <= 0; ++e2)
        for (int e1 = -1; e1 <= 0; ++e1) {
          const int f1 = gi[d1] + e1, f2 = gi[d2] + e2;   // face element lower corner
          if (f1 < 0 || f1 >= g.n[d1] || f2 < 0 || f2 >= g.n[d2]) continue;
          const int c1 = -e1, c2 = -e2;                  // node's local face index
          for (int q = 0; q < 4; ++q) {
            const double xi1 = (q & 1) ? kGauss : -kGauss, xi2 = (q & 2) ? kGauss : -kGauss;
            double xq[3];
            xq[d] = g.lo[d] + gi[d] * g.h[d];
            xq[d1] = g.lo[d1] + (f1 + (1.0 + xi1) / 2.0) * g.h[d1];
            xq[d2] = g.lo[d2] + (f2 + (1.0 + xi2) / 2.0) * g.h[d2];
            const double N = ((1.0 + (c1 ? xi1 : -xi1)) / 2.0) * ((1.0 + (c2 ? xi2 : -xi2)) / 2.0);
            v += prob_gR(pb, F, xq[0], xq[1], xq[2]) * N * hh;
          }
        }
    }
    // lifting: subtract couplings to Dirichlet neighbours (nodes outside the free box)
    const bool near = (fx == 0 && g.flo[0] == 1) || (fx == g.nf[0] - 1 && g.flo[0] + g.nf[0] == g.n[0]) ||
                      (fy == 0 && g.flo[1] == 1) || (fy == g.nf[1] - 1 && g.flo[1] + g.nf[1] == g.n[1]) ||
                      (fz == 0 && g.flo[2] == 1) || (fz == g.nf[2] - 1 && g.flo[2] + g.nf[2] == g.n[2]);
    if (near) {
      double sub = 0.0;
      for (int e = 0; e < 8; ++e) {
        const int ex = e & 1, ey = (e >> 1) & 1, ez = (e >> 2) & 1;
        const double be = beta_at(g, beta, beta_const, gx - 1 + ex, gy - 1 + ey, gz - 1 + ez);
        if (be == 0.0) continue;
        for (int bn = 0; bn < 8; ++bn) {
          const int bx = bn & 1, by = (bn >> 1) & 1, bz = (bn >> 2) & 1;
          const int jx = gx - 1 + ex + bx, jy = gy - 1 + ey + by, jz = gz - 1 + ez + bz;
          const bool jfree = jx >= g.flo[0] && jx < g.flo[0] + g.nf[0] && jy >= g.flo[1] && jy < g.flo[1] + g.nf[1] &&
                             jz >= g.flo[2] && jz < g.flo[2] + g.nf[2];
          if (jfree) continue;
          const int pat = ((ex + bx) != 1 ? 1 : 0) | ((ey + by) != 1 ? 2 : 0) | ((ez + bz) != 1 ? 4 : 0);
          const double gD = prob_gD(pb, g.lo[0] + jx * g.h[0], g.lo[1] + jy * g.h[1], g.lo[2] + jz * g.h[2]);
          sub += be * es.kappa[pat] * gD;
        }
        // Robin face mass coupling with Dirichlet nodes on the same face
        for (int F = 0; F < 6; ++F) {
          if (es.robin[F] == 0.0) continue;
          const int d = F >> 1, side = F & 1;
          if (gi[d] != (side ? g.n[d] : 0)) continue;
          const int e3[3] = {ex, ey, ez};
          for (int bn = 0; bn < 8; ++bn) {
            const int b3[3] = {bn & 1, (bn >> 1) & 1, (bn >> 2) & 1};
            if (b3[d] != 1 - e3[d]) continue;
            const int jx = gx - 1 + ex + b3[0], jy = gy - 1 + ey + b3[1], jz = gz - 1 + ez + b3[2];
            const bool jfree = jx >= g.flo[0] && jx < g.flo[0] + g.nf[0] && jy >= g.flo[1] && jy < g.flo[1] + g.nf[1] &&
                               jz >= g.flo[2] && jz < g.flo[2] + g.nf[2];
            if (jfree) continue;
            int nd = 0;
            for (int t = 0; t < 3; ++t) if (t != d && b3[t] != 1 - e3[t]) ++nd;
            const double m2 = nd == 0 ? (1.0 / 9.0) : (nd == 1 ? (1.0 / 18.0) : (1.0 / 36.0));
            const double gD = prob_gD(pb, g.lo[0] + jx * g.h[0], g.lo[1] + jy * g.h[1], g.lo[2] + jz * g.h[2]);
            sub += es.robin[F] * m2 * gD;
          }
        }
      }
      v -= sub;
    }
    b[(long long)fz * g.S + (long long)fy * g.P + fx] = v;
    bsq = v * v;
  }

  // ||b||^2: deterministic block reduction + last-CTA sum in CTA order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bsq += __shfl_down_sync(0xffffffffu, bsq, o);
  if ((tid & 31) == 0) red[tid >> 5] = bsq;
  __syncthreads();
  const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < RNTH / 32; ++w) s += red[w];
    partials[bid] = s;
    __threadfence();
    is_last = (atomicAdd(&sc->counter, 1u) == nb - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double s = 0.0;
  for (unsigned k = tid; k < nb; k += RNTH) s += __ldcg(partials + k);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < RNTH / 32; ++w) t += red[w];
    sc->bb = t;
    sc->counter = 0;
  }
}

// ---- gather / scatter between full nodal vectors and the free box ------------------------------
__global__ void k_gather(const LevelGeom g, const double* __restrict__ u, double* __restrict__ x) {
  const int fx = blockIdx.x * blockDim.x + threadIdx.x;
  const int fy = blockIdx.y, fz = blockIdx.z;
  if (fx >= g.nf[0]) return;
  const long long nx = g.n[0] + 1, ny = g.n[1] + 1;
  const long long gi = (long long)(g.flo[0] + fx) + nx * ((long long)(g.flo[1] + fy) + ny * (g.flo[2] + fz));
  x[(long long)fz * g.S + (long long)fy * g.P + fx] = u[gi];
}

__global__ void k_scatter(const LevelGeom g, const double* __restrict__ x, double* __restrict__ u) {
  const int fx = blockIdx.x * blockDim.x + threadIdx.x;
  const int fy = blockIdx.y, fz = blockIdx.z;
  if (fx >= g.nf[0]) return;
  const long long nx = g.n[0] + 1, ny = g.n[1] + 1;
  const long long gi = (long long)(g.flo[0] + fx) + nx * ((long long)(g.flo[1] + fy) + ny * (g.flo[2] + fz));
  u[gi] = x[(long long)fz * g.S + (long long)fy * g.P + fx];
}

// Dirichlet nodes (outside the free box) of a full nodal vector := g_D (or 0). One launch per
// boundary face; nodes on shared edges are written twice with the same value.
__global__ void k_dirichlet_face(const LevelGeom g, const Problem pb, double* __restrict__ u, int F, int zero) {
  const int d = F >> 1, side = F & 1;
  const int d1 = (d == 0) ? 1 : 0, d2 = (d == 2) ? 1 : 2;
  const int i1 = blockIdx.x * blockDim.x + threadIdx.x, i2 = blockIdx.y;
  if (i1 > g.n[d1] || i2 > g.n[d2]) return;
  int gi[3];
  gi[d] = side ? g.n[d] : 0;
  gi[d1] = i1;
  gi[d2] = i2;
  const long long nx = g.n[0] + 1, ny = g.n[1] + 1;
  const double v = zero ? 0.0 : prob_gD(pb, g.lo[0] + gi[0] * g.h[0], g.lo[1] + gi[1] * g.h[1], g.lo[2] + gi[2] * g.h[2]);
  u[(long long)gi[0] + nx * ((long long)gi[1] + ny * gi[2])] = v;
}

__global__ void k_zero_free(const LevelGeom g, double* __restrict__ v) {
  const int fx = blockIdx.x * blockDim.x + threadIdx.x;
  if (fx >= g.nf[0]) return;
  v[(long long)blockIdx.z * g.S + (long long)blockIdx.y * g.P + fx] = 0.0;
}

}  // namespace

cudaError_t launch_beta(const LevelGeom& g, const Problem& pb, double* beta, cudaStream_t st) {
  const long long total = (long long)(g.n[0] + 4) * (g.n[1] + 4) * (g.n[2] + 4);
  const int nb = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  count_launch();
  k_beta<<<nb, 256, 0, st>>>(g, pb, beta);
  return cudaGetLastError();
}

cudaError_t launch_rhs(const LevelGeom& g, const Problem& pb, const ElemStencil& es, double beta_const, const double* beta,
                       double* b, double* partials, JcgScalars* sc, cudaStream_t st) {
  dim3 grid((g.nf[0] + RX - 1) / RX, (g.nf[1] + RY - 1) / RY, (g.nf[2] + RZ - 1) / RZ);
  count_launch();
  k_rhs<<<grid, RNTH, 0, st>>>(g, pb, es, beta_const, beta, b, partials, sc);
  return cudaGetLastError();
}

cudaError_t launch_gather(const LevelGeom& g, const double* u, double* x, cudaStream_t st) {
  dim3 grid((g.nf[0] + 127) / 128, g.nf[1], g.nf[2]);
  count_launch();
  k_gather<<<grid, 128, 0, st>>>(g, u, x);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const LevelGeom& g, const double* x, double* u, cudaStream_t st) {
  dim3 grid((g.nf[0] + 127) / 128, g.nf[1], g.nf[2]);
  count_launch();
  k_scatter<<<grid, 128, 0, st>>>(g, x, u);
  return cudaGetLastError();
}

cudaError_t launch_dirichlet_fill(const LevelGeom& g, const Problem& pb, double* u, double, int zero_instead,
                                  cudaStream_t st) {
  for (int F = 0; F < 6; ++F) {
    if (pb.face[F] != FACE_DIRICHLET) continue;
    const int d = F >> 1;
    const int d1 = (d == 0) ? 1 : 0, d2 = (d == 2) ? 1 : 2;
    dim3 grid((g.n[d1] + 1 + 127) / 128, g.n[d2] + 1);
    count_launch();
    k_dirichlet_face<<<grid, 128, 0, st>>>(g, pb, u, F, zero_instead);
  }
  return cudaGetLastError();
}

cudaError_t launch_zero_vec(const LevelGeom& g, double* v, cudaStream_t st) {
  dim3 grid((g.nf[0] + 127) / 128, g.nf[1], g.nf[2]);
  count_launch();
  k_zero_free<<<grid, 128, 0, st>>>(g, v);
  return cudaGetLastError();
}

}  // namespace ecmg
