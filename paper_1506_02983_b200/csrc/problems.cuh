// problems.cuh -- device-side problem registry: beta, f, g_D, alpha, g_R of Eq. (bvp)
// for the built-in problems (ids in include/ecmg.h). f = -div(beta grad u) from the exact u.
#pragma once
#include "ecmg_internal.cuh"

namespace ecmg {

__host__ __device__ inline double kPi() { return 3.14159265358979323846; }

// C5 / layered geometry, params layout as documented in synth/__init__.py:
// [0:7] interface heights, [7:15] layer beta, [15:43] 4 boxes (c, s, beta), [43:46] x0, [46] sigma, [47] amp
__host__ __device__ inline double layer_beta(const Problem& P, double z) {
  int l = 0;
  while (l < 7 && !(z < P.params[l])) ++l;
  return P.params[7 + l];
}

__host__ __device__ inline double prob_beta(const Problem& P, double x, double y, double z) {
  const double pi = kPi();
  switch (P.id) {
    case 3: return 1.0 + 0.5 * sin(2.0 * pi * x) * cos(2.0 * pi * y) * sin(2.0 * pi * z);
    case 5: {
      double b = layer_beta(P, z);
      for (int k = 0; k < 4; ++k) {
        const double* q = &P.params[15 + 7 * k];
        if (fabs(x - q[0]) < q[3] && fabs(y - q[1]) < q[4] && fabs(z - q[2]) < q[5]) b = q[6];
      }
      return b;
    }
    case 22: return layer_beta(P, z);
    default: return 1.0;
  }
}

__host__ __device__ inline double prob_exact(const Problem& P, double x, double y, double z) {
  const double pi = kPi();
  switch (P.id) {
    case 1: return sin(pi * x) * sin(pi * y) * sin(pi * z);
    case 2: return exp(x + y + z);
    case 3: return cos(pi * x) * cos(pi * y) * exp(z);
    case 4: { double r2 = x * x + y * y + z * z; return sqrt(r2) * sqrt(sqrt(r2)); }  // r^{3/2}
    case 11: return sin(0.5 * pi * x) * sin(0.5 * pi * y) * sin(0.5 * pi * z);
    case 12: return exp(z) * sin(1.5 * pi * x) * sin(0.5 * pi * y);
    case 13: { double r2 = x * x + y * y + z * z; if (r2 == 0.0) return 0.0; return x * y * z / (sqrt(r2) * sqrt(sqrt(r2))); }
    case 21: return 1.0 + x + 2.0 * y - z + x * y + 3.0 * x * y * z;
    case 22: return 0.5 + 1.5 * x - 0.75 * y;
    case 23: case 25: return 0.3 + 0.7 * x - 0.4 * y + 0.9 * z;
    default: return 0.0;
  }
}

__host__ __device__ inline double prob_f(const Problem& P, double x, double y, double z) {
  const double pi = kPi();
  switch (P.id) {
    case 1: return 3.0 * pi * pi * prob_exact(P, x, y, z);
    case 2: return -3.0 * exp(x + y + z);
    case 3: {
      // f = -beta Lap u - grad beta . grad u, Lap u = (1 - 2 pi^2) u   (sincospi: sin(pi t), cos(pi t))
      double sx, cx, sy, cy, s2x, c2x, s2y, c2y, s2z, c2z;
      sincospi(x, &sx, &cx); sincospi(y, &sy, &cy);
      sincospi(2.0 * x, &s2x, &c2x); sincospi(2.0 * y, &s2y, &c2y); sincospi(2.0 * z, &s2z, &c2z);
      const double ez = exp(z);
      const double u = cx * cy * ez;
      const double b = 1.0 + 0.5 * s2x * c2y * s2z;
      const double bx = pi * c2x * c2y * s2z, by = -pi * s2x * s2y * s2z, bz = pi * s2x * c2y * c2z;
      const double ux = -pi * sx * cy * ez, uy = -pi * cx * sy * ez;
      return -b * (1.0 - 2.0 * pi * pi) * u - (bx * ux + by * uy + bz * u);
    }
    case 4: {  // -Lap r^{3/2} = -(15/4) r^{-1/2}; f(0) := 0 (never evaluated at a node)
      double r2 = x * x + y * y + z * z;
      if (r2 == 0.0) return 0.0;
      return -3.75 * rsqrt(sqrt(r2));   // r^{-1/2}
    }
    case 5: {
      const double* x0 = &P.params[43];
      double s = P.params[46], amp = P.params[47];
      double dx = x - x0[0], dy = y - x0[1], dz = z - x0[2];
      return amp * exp(-(dx * dx + dy * dy + dz * dz) / (2.0 * s * s));
    }
    case 11: return 0.75 * pi * pi * prob_exact(P, x, y, z);
    case 12: return -(1.0 - 2.5 * pi * pi) * prob_exact(P, x, y, z);
    case 13: {
      double r2 = x * x + y * y + z * z;
      if (r2 == 0.0) return 0.0;
      double r4 = sqrt(sqrt(r2));            // r^{1/2}
      double r35 = r2 * sqrt(r2) * r4;        // r^{7/2}
      return 33.0 * x * y * z / (4.0 * r35);
    }
    case 24: return 1.0;
    default: return 0.0;
  }
}

__host__ __device__ inline double prob_gD(const Problem& P, double x, double y, double z) {
  return prob_exact(P, x, y, z);
}

// g_D at global node (ix, iy, iz) of level g: the caller's nodal array (PROB_ARRAYS) or the registry's g_D
__device__ inline double prob_gD_node(const Problem& P, const LevelGeom& g, int ix, int iy, int iz) {
  if (P.id == PROB_ARRAYS)
    return P.arr[2] ? P.arr[2][(long long)ix + (g.n[0] + 1LL) * ((long long)iy + (g.n[1] + 1LL) * iz)] : 0.0;
  return prob_gD(P, g.lo[0] + ix * g.h[0], g.lo[1] + iy * g.h[1], g.lo[2] + iz * g.h[2]);
}

// Robin data g_R = alpha u + beta du/dn on face `face`
__host__ __device__ inline double prob_gR(const Problem& P, int face, double x, double y, double z) {
  switch (P.id) {
    case 3: return (P.alpha[face] + prob_beta(P, x, y, z)) * prob_exact(P, x, y, z);  // du/dz = u on z = 1
    case 23: return P.alpha[face] * prob_exact(P, x, y, z) + 0.9;
    case 25: {   // Robin on the four side faces: alpha_F u + du/dn_F, grad u = (0.7, -0.4, 0.9)
      const double dudn[6] = {-0.7, 0.7, 0.4, -0.4, -0.9, 0.9};
      return P.alpha[face] * prob_exact(P, x, y, z) + dudn[face];
    }
    default: return 0.0;  // P1, P2: homogeneous Neumann
  }
}

// true if beta is analytically constant (= 1) for the problem
__host__ inline bool prob_beta_is_one(int id) {
  return !(id == 3 || id == 5 || id == 22);
}

}  // namespace ecmg
