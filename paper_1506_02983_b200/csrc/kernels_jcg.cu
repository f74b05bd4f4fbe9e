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
        } else if (MODE == MODE_INIT) {
          acc2 = __fma_rn(ii0[j], ii0[j], acc2);
          const double rn = ii0[j] - ap;
          const double zz = dinv * rn;
          acc0 = __fma_rn(rn, zz, acc0);
          acc1 = __fma_rn(rn, rn, acc1);
          a.o0[off] = rn;
        } else if (MODE == MODE_TRUE) {
          const double rn = ii0[j] - ap;
          acc1 = __fma_rn(rn, rn, acc1);
        } else {
          a.o0[off] = ap;
        }
      }
      part[j] = q1p[j] + q0;
      q1p[j] = q1;
      pp[j] = cc;
    }
  }
  if (MODE != MODE_APPLY) reduce_finalize(MODE, a, acc0, acc1, acc2);
}

// ============================================================================================
// Element-beta path: beta_e per element (C3, C5, layered patch), Robin / Neumann faces (C3, P1,
// P2, Robin patch). (A p)_i = sum_{e ni i} beta_e sum_{j in e} kappa[pattern(i,j)] p_j
// + Robin face mass; diag_i = kappa[0] sum_e beta_e + Robin diagonal, recomputed from beta.
// Tile 32 x 8 columns, 4-slot rings of node planes (34 x 10) and element planes (35 x 11).
// ============================================================================================
constexpr int ETY = WARPS;        // 8 rows, one per warp
constexpr int EHX = TX + 2;       // 34
constexpr int EHY = ETY + 2;      // 10
constexpr int EEX = TX + 3;       // 35 elements: X0-2 .. X0+32
constexpr int EEY = ETY + 3;      // 11
constexpr int NRING = 4;
constexpr int ELEM_SMEM = NRING * (EHX * EHY + EEX * EEY) * (int)sizeof(double);
// cubic cells: + a ring of element layers of T_e = beta_e * S_e (S_e = sum of p over the element)
constexpr int ELEM_SMEM_CUBE = ELEM_SMEM + NRING * EEY * EEX * (int)sizeof(double);

// Robin face mass alpha h1 h2 (m (x) m) of the face elements around a node on Robin faces:
// rarely executed (one boundary plane), kept out of line so the main path keeps few registers.
__device__ __noinline__ void robin_terms(const ElemStencil& es, int rm, const double (*Pr)[EHY][EHX],
                                         const double (*Br)[EEY][EEX], int z, int w, int lane, double* ap, double* diag) {
  double a = 0.0, dg = 0.0;
  for (int F = 0; F < 6; ++F) {
    if (!(rm & (1 << F))) continue;
    const int d = F >> 1;
    for (int ez = 0; ez < 2; ++ez)
      for (int ey = 0; ey < 2; ++ey)
        for (int ex = 0; ex < 2; ++ex) {
          const double be = Br[(z - 1 + ez + 8) & 3][w + 1 + ey][lane + 1 + ex];
          if (be == 0.0) continue;
          dg += es.robin[F] * (1.0 / 9.0);
          const int e3[3] = {ex, ey, ez};
          for (int b = 0; b < 8; ++b) {
            const int b3[3] = {b & 1, (b >> 1) & 1, (b >> 2) & 1};
            if (b3[d] != 1 - e3[d]) continue;   // node of the element face on F
            int nd = 0;
            for (int t = 0; t < 3; ++t) if (t != d && b3[t] != 1 - e3[t]) ++nd;
            const double m2 = nd == 0 ? (1.0 / 9.0) : (nd == 1 ? (1.0 / 18.0) : (1.0 / 36.0));
            a += es.robin[F] * m2 * Pr[(z - 1 + ez + b3[2] + 8) & 3][w + ey + b3[1]][lane + ex + b3[0]];
          }
        }
  }
  *ap += a;
  *diag += dg;
}
constexpr int EBSLOTS = (EEX * EEY + NTH - 1) / NTH;   // beta loads per thread per plane (2)

__device__ __forceinline__ int ring(int p) { return (p + 2 * NRING) & (NRING - 1); }

template <int MODE, bool CUBE>
__global__ void __launch_bounds__(NTH, 2) k_jcg_elem(const LevelGeom g, const ElemStencil es, const Problem pb,
                                                     const KArgs a) {
  extern __shared__ double smem[];
  double (*Pr)[EHY][EHX] = reinterpret_cast<double (*)[EHY][EHX]>(smem);
  double (*Br)[EEY][EEX] = reinterpret_cast<double (*)[EEY][EEX]>(smem + NRING * EHY * EHX);
  double (*Tr)[EEY][EEX] = reinterpret_cast<double (*)[EEY][EEX]>(smem + NRING * (EHY * EHX + EEY * EEX));
  JcgScalars* sc = a.sc;
  if (MODE == MODE_K1 || MODE == MODE_K2) {
    if (*(volatile int*)&sc->done) return;
  }
  const int lane = threadIdx.x, w = threadIdx.y, tid = lane + TX * w;
  const int nfx = g.nf[0], nfy = g.nf[1], nfz = g.nza;   // local planes
  const long long P = g.P, S = g.S;
  const int X0 = blockIdx.x * TX, Y0 = blockIdx.y * ETY;
  const int z0 = g.zbeg + blockIdx.z * a.zc;
  const int z1 = min(z0 + a.zc, g.zend);
  const int x = X0 + lane, y = Y0 + w;
  const bool own_ok = x < nfx && y < nfy;
  const long long own_off = own_ok ? (long long)y * P + x : 0;

  // node ring slot (84 slots: 2 rows of 34, 2 columns of 8)
  int rhx = -1, rhy = -1;
  if (tid < 2 * EHX) { rhx = tid % EHX; rhy = (tid < EHX) ? 0 : EHY - 1; }
  else if (tid < 2 * EHX + 2 * ETY) { const int t = tid - 2 * EHX; rhx = (t < ETY) ? 0 : EHX - 1; rhy = 1 + (t % ETY); }
  const int rgx = X0 - 1 + rhx, rgy = Y0 - 1 + rhy;
  const bool ring_ok = rhx >= 0 && rgx >= 0 && rgx < nfx && rgy >= 0 && rgy < nfy;
  const long long ring_off = ring_ok ? (long long)rgy * P + rgx : 0;

  // element slots: element tile coords (ex, ey) -> free element coords (X0-2+ex, Y0-2+ey) -> global +flo
  int eslot_x[EBSLOTS], eslot_y[EBSLOTS];
  bool eslot_xy_ok[EBSLOTS];
  long long eslot_off[EBSLOTS];
#pragma unroll
  for (int k = 0; k < EBSLOTS; ++k) {
    const int t = tid + k * NTH;
    const bool in = t < EEX * EEY;
    eslot_x[k] = in ? t % EEX : 0;
    eslot_y[k] = in ? t / EEX : 0;
    const int gex = g.flo[0] + X0 - 2 + eslot_x[k], gey = g.flo[1] + Y0 - 2 + eslot_y[k];
    eslot_xy_ok[k] = in && gex >= -2 && gex <= g.n[0] + 1 && gey >= -2 && gey <= g.n[1] + 1;
    eslot_off[k] = eslot_xy_ok[k] ? (long long)(gey + 2) * g.BP + (gex + 2) : 0;
    if (!in) eslot_x[k] = -1;
  }

  double bcg = 0.0, alpha = 0.0;
  bool first = false;
  if (MODE == MODE_K1) { bcg = sc->beta; first = (sc->iter == 0); }
  if (MODE == MODE_K2) alpha = sc->alpha;
  constexpr bool kTwoHalo = (MODE == MODE_K1);
  constexpr bool kInt0 = (MODE == MODE_K2 || MODE == MODE_INIT || MODE == MODE_TRUE);
  constexpr bool kInt1 = (MODE == MODE_K2);
  const bool robin_any = (es.robin[0] != 0.0) || (es.robin[1] != 0.0) || (es.robin[2] != 0.0) ||
                         (es.robin[3] != 0.0) || (es.robin[4] != 0.0) || (es.robin[5] != 0.0);

  double nh0 = 0.0, nh1 = 0.0, nr0 = 0.0, nr1 = 0.0, ni0 = 0.0, ni1 = 0.0;
  double nb[EBSLOTS];
#pragma unroll
  for (int k = 0; k < EBSLOTS; ++k) nb[k] = 0.0;

  auto load_halo = [&](int z) {
    const bool zok = (z >= 0) && (z < nfz);
    const long long zo = zok ? (long long)z * S : 0;
    nh0 = (zok && own_ok) ? __ldg(a.h0 + zo + own_off) : 0.0;
    nr0 = (zok && ring_ok) ? __ldg(a.h0 + zo + ring_off) : 0.0;
    if (kTwoHalo && !first) {
      nh1 = (zok && own_ok) ? __ldg(a.h1 + zo + own_off) : 0.0;
      nr1 = (zok && ring_ok) ? __ldg(a.h1 + zo + ring_off) : 0.0;
    }
  };
  auto load_beta = [&](int fez) {   // element plane (local free element coords)
    const int gez = g.flo[2] + g.zoff + fez;
    const bool zok = gez >= -2 && gez <= g.n[2] + 1;
    const long long zo = zok ? (long long)(gez + 2) * g.BS : 0;
#pragma unroll
    for (int k = 0; k < EBSLOTS; ++k) nb[k] = (zok && eslot_xy_ok[k]) ? __ldg(a.beta + zo + eslot_off[k]) : 0.0;
  };
  auto load_int = [&](int z) {
    const long long zo = (long long)z * S;
    if (kInt0) ni0 = own_ok ? __ldg(a.i0 + zo + own_off) : 0.0;
    if (kInt1) ni1 = own_ok ? __ldg(a.i1 + zo + own_off) : 0.0;
  };

  // which Robin faces (alpha != 0) a free node (fx, fy, fz) lies on: bit F
  auto robin_mask = [&](int fx, int fy, int fz) -> int {
    if (!robin_any) return 0;
    const int gx = g.flo[0] + fx, gy = g.flo[1] + fy, gz = g.flo[2] + g.zoff + fz;
    int m = 0;
    if (gx == 0 && es.robin[0] != 0.0) m |= 1;
    if (gx == g.n[0] && es.robin[1] != 0.0) m |= 2;
    if (gy == 0 && es.robin[2] != 0.0) m |= 4;
    if (gy == g.n[1] && es.robin[3] != 0.0) m |= 8;
    if (gz == 0 && es.robin[4] != 0.0) m |= 16;
    if (gz == g.n[2] && es.robin[5] != 0.0) m |= 32;
    return m;
  };
  // diagonal at node-tile position (hx, hy) of node plane zn (elements from the beta ring)
  auto diag_at = [&](int hx, int hy, int zn, int fx, int fy) -> double {
    double sb = 0.0, rob = 0.0;
    const int rm = robin_mask(fx, fy, zn);
#pragma unroll
    for (int ez = 0; ez < 2; ++ez) {
      const int sl = ring(zn - 1 + ez);
#pragma unroll
      for (int ey = 0; ey < 2; ++ey)
#pragma unroll
        for (int ex = 0; ex < 2; ++ex) {
          const double be = Br[sl][hy + ey][hx + ex];
          sb += be;
          if (rm && be != 0.0) {
#pragma unroll
            for (int F = 0; F < 6; ++F)
              if (rm & (1 << F)) rob += es.robin[F] * (1.0 / 9.0);
          }
        }
    }
    return es.kappa[0] * sb + rob;
  };

  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  load_halo(z0 - 1);
  load_beta(z0 - 2);
  // prologue: element plane z0-2 into its ring slot
#pragma unroll
  for (int k = 0; k < EBSLOTS; ++k)
    if (eslot_x[k] >= 0) Br[ring(z0 - 2)][eslot_y[k]][eslot_x[k]] = nb[k];
  load_beta(z0 - 1);

  const int nsteps = z1 - z0 + 2;
  for (int s = 0; s < nsteps; ++s) {
    const int zl = z0 - 1 + s;
    const double c0 = nh0, c1 = nh1, cr0 = nr0, cr1 = nr1, ii0 = ni0, ii1 = ni1;
    double cb[EBSLOTS];
#pragma unroll
    for (int k = 0; k < EBSLOTS; ++k) cb[k] = nb[k];
    if (s + 1 < nsteps) { load_halo(zl + 1); load_beta(zl + 1); }
    if ((kInt0 || kInt1) && zl >= z0 && zl < z1) load_int(zl);

    // element plane zl -> ring
#pragma unroll
    for (int k = 0; k < EBSLOTS; ++k)
      if (eslot_x[k] >= 0) Br[ring(zl)][eslot_y[k]][eslot_x[k]] = cb[k];
    __syncthreads();

    // node plane zl: transform into the ring
    {
      double v = c0;
      if (MODE == MODE_K1) {
        double di = 1.0;
        if (own_ok && zl >= 0 && zl < nfz && es.precond) {
          const double d = diag_at(lane + 1, w + 1, zl, x, y);
          di = d > 0.0 ? 1.0 / d : 0.0;
        }
        v = first ? di * c0 : di * c0 + bcg * c1;
      }
      Pr[ring(zl)][w + 1][lane + 1] = v;
      if (MODE == MODE_K1 && own_ok && (zl == g.zbeg - 1 || zl == g.zend) && zl >= 0 && zl < nfz)
        a.o0[(long long)zl * S + own_off] = v;   // slab halo plane of p
      if (rhx >= 0) {
        double vr = cr0;
        if (MODE == MODE_K1) {
          double di = 1.0;
          if (ring_ok && zl >= 0 && zl < nfz && es.precond) {
            const double d = diag_at(rhx, rhy, zl, rgx, rgy);
            di = d > 0.0 ? 1.0 / d : 0.0;
          }
          vr = first ? di * cr0 : di * cr0 + bcg * cr1;
        }
        Pr[ring(zl)][rhy][rhx] = vr;
      }
    }
    __syncthreads();

    if (CUBE && s >= 1) {
      // element layer el = zl - 1 (node planes zl-1, zl): T_e = beta_e * S_e for the 33 x 9 elements of
      // the own nodes (element tile coords 1..33 x 1..9; its nodes are node-tile coords e-1, e)
      const int el = zl - 1;
      for (int t = tid; t < 33 * 9; t += NTH) {
        const int ex = 1 + t % 33, ey = 1 + t / 33;
        const double be = Br[ring(el)][ey][ex];
        double sum = 0.0;
        if (be != 0.0) {
#pragma unroll
          for (int dz = 0; dz < 2; ++dz)
            sum += (Pr[ring(el + dz)][ey - 1][ex - 1] + Pr[ring(el + dz)][ey - 1][ex]) +
                   (Pr[ring(el + dz)][ey][ex - 1] + Pr[ring(el + dz)][ey][ex]);
        }
        Tr[ring(el)][ey][ex] = be * sum;
      }
      __syncthreads();
    }
    if (CUBE && s >= 2 && own_ok) {
      // cubic cells: (A p)_i = c [5 p_i B_i + sum_{6 axis j} W_ij p_j - sum_{e ni i} beta_e S_e], c = h/12
      // (K_e = c{4, 0, -1, -1}: K_e p = c (5 p_a + sum_axis - S_e)); B_i, W_ij: beta sums over the
      // 8 / 4 elements containing i / i and j
      const int z = zl - 1;
      const int rd = ring(z - 1), ru = ring(z), rz = ring(z), rzm = ring(z - 1), rzp = ring(z + 1);
      double b[2][2][2];
#pragma unroll
      for (int ez = 0; ez < 2; ++ez)
#pragma unroll
        for (int ey = 0; ey < 2; ++ey)
#pragma unroll
          for (int ex = 0; ex < 2; ++ex) b[ez][ey][ex] = Br[ez ? ru : rd][w + 1 + ey][lane + 1 + ex];
      const double Wxm = (b[0][0][0] + b[0][1][0]) + (b[1][0][0] + b[1][1][0]);
      const double Wxp = (b[0][0][1] + b[0][1][1]) + (b[1][0][1] + b[1][1][1]);
      const double Wym = (b[0][0][0] + b[0][0][1]) + (b[1][0][0] + b[1][0][1]);
      const double Wyp = (b[0][1][0] + b[0][1][1]) + (b[1][1][0] + b[1][1][1]);
      const double Wzm = (b[0][0][0] + b[0][0][1]) + (b[0][1][0] + b[0][1][1]);
      const double Wzp = (b[1][0][0] + b[1][0][1]) + (b[1][1][0] + b[1][1][1]);
      const double B = Wzm + Wzp;
      double T = 0.0;
#pragma unroll
      for (int ez = 0; ez < 2; ++ez)
        T += (Tr[ez ? ru : rd][w + 1][lane + 1] + Tr[ez ? ru : rd][w + 1][lane + 2]) +
             (Tr[ez ? ru : rd][w + 2][lane + 1] + Tr[ez ? ru : rd][w + 2][lane + 2]);
      const double pc = Pr[rz][w + 1][lane + 1];
      const double c = 0.25 * es.kappa[0];
      double ap = 5.0 * pc * B - T;
      ap = __fma_rn(Pr[rz][w + 1][lane], Wxm, ap);
      ap = __fma_rn(Pr[rz][w + 1][lane + 2], Wxp, ap);
      ap = __fma_rn(Pr[rz][w][lane + 1], Wym, ap);
      ap = __fma_rn(Pr[rz][w + 2][lane + 1], Wyp, ap);
      ap = __fma_rn(Pr[rzm][w + 1][lane + 1], Wzm, ap);
      ap = __fma_rn(Pr[rzp][w + 1][lane + 1], Wzp, ap);
      ap *= c;
      double diag = es.kappa[0] * B;
      const int rm = robin_mask(x, y, z);
      if (rm) robin_terms(es, rm, Pr, Br, z, w, lane, &ap, &diag);
      const double dinv = es.precond ? (diag > 0.0 ? 1.0 / diag : 0.0) : 1.0;
      const long long off = (long long)z * S + own_off;
      if (MODE == MODE_K1) {
        acc0 += pc * ap;
        a.o0[off] = pc;
      } else if (MODE == MODE_K2) {
        const double xn = ii0 + alpha * pc;
        const double rn = ii1 - alpha * ap;
        const double zz = dinv * rn;
        acc0 = __fma_rn(rn, zz, acc0);
        acc1 = __fma_rn(rn, rn, acc1);
        a.o0[off] = xn;
        a.o1[off] = rn;
      } else if (MODE == MODE_INIT) {
        acc2 += ii0 * ii0;
        const double rn = ii0 - ap;
        const double zz = dinv * rn;
        acc0 = __fma_rn(rn, zz, acc0);
        acc1 = __fma_rn(rn, rn, acc1);
        a.o0[off] = rn;
      } else if (MODE == MODE_TRUE) {
        const double rn = ii0 - ap;
        acc1 = __fma_rn(rn, rn, acc1);
      } else {
        a.o0[off] = ap;
      }
    }
    if (!CUBE && s >= 2 && own_ok) {
      const int z = zl - 1;
      double p27[3][3][3];
#pragma unroll
      for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) p27[dz][dy][dx] = Pr[ring(z - 1 + dz)][w + dy][lane + dx];
      double ap = 0.0, sb = 0.0;
#pragma unroll
      for (int ez = 0; ez < 2; ++ez)
#pragma unroll
        for (int ey = 0; ey < 2; ++ey)
#pragma unroll
          for (int ex = 0; ex < 2; ++ex) {
            const double be = Br[ring(z - 1 + ez)][w + 1 + ey][lane + 1 + ex];
            sb += be;
            double t = 0.0;
#pragma unroll
            for (int bz = 0; bz < 2; ++bz)
#pragma unroll
              for (int by = 0; by < 2; ++by)
#pragma unroll
                for (int bx = 0; bx < 2; ++bx) {
                  const int pat = ((ex + bx) != 1 ? 1 : 0) | ((ey + by) != 1 ? 2 : 0) | ((ez + bz) != 1 ? 4 : 0);
                  t += es.kappa[pat] * p27[ez + bz][ey + by][ex + bx];
                }
            ap += be * t;
          }
      double diag = es.kappa[0] * sb;
      const int rm = robin_mask(x, y, z);
      if (rm) {
        // Robin face mass alpha h1 h2 (m (x) m) on each face element around the node
#pragma unroll
        for (int F = 0; F < 6; ++F) {
          if (!(rm & (1 << F))) continue;
          const int d = F >> 1;
          for (int ez = 0; ez < 2; ++ez)
            for (int ey = 0; ey < 2; ++ey)
              for (int ex = 0; ex < 2; ++ex) {
                const double be = Br[ring(z - 1 + ez)][w + 1 + ey][lane + 1 + ex];
                if (be == 0.0) continue;
                diag += es.robin[F] * (1.0 / 9.0);
                const int e3[3] = {ex, ey, ez};
                for (int b = 0; b < 8; ++b) {
                  const int b3[3] = {b & 1, (b >> 1) & 1, (b >> 2) & 1};
                  if (b3[d] != 1 - e3[d]) continue;   // node of the element face on F
                  int nd = 0;
                  for (int t = 0; t < 3; ++t) if (t != d && b3[t] != 1 - e3[t]) ++nd;
                  const double m2 = nd == 0 ? (1.0 / 9.0) : (nd == 1 ? (1.0 / 18.0) : (1.0 / 36.0));
                  ap += es.robin[F] * m2 * p27[ez + b3[2]][ey + b3[1]][ex + b3[0]];
                }
              }
        }
      }
      const double dinv = es.precond ? (diag > 0.0 ? 1.0 / diag : 0.0) : 1.0;
      const double pc = p27[1][1][1];
      const long long off = (long long)z * S + own_off;
      if (MODE == MODE_K1) {
        acc0 += pc * ap;
        a.o0[off] = pc;
      } else if (MODE == MODE_K2) {
        const double xn = ii0 + alpha * pc;
        const double rn = ii1 - alpha * ap;
        const double zz = dinv * rn;
        acc0 = __fma_rn(rn, zz, acc0);
        acc1 = __fma_rn(rn, rn, acc1);
        a.o0[off] = xn;
        a.o1[off] = rn;
      } else if (MODE == MODE_INIT) {
        acc2 += ii0 * ii0;
        const double rn = ii0 - ap;
        const double zz = dinv * rn;
        acc0 = __fma_rn(rn, zz, acc0);
        acc1 = __fma_rn(rn, rn, acc1);
        a.o0[off] = rn;
      } else if (MODE == MODE_TRUE) {
        const double rn = ii0 - ap;
        acc1 = __fma_rn(rn, rn, acc1);
      } else {
        a.o0[off] = ap;
      }
    }
  }
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

cudaError_t launch_vsum(const SlabScalars& s, cudaStream_t st) {
  count_launch();
  k_vsum<<<1, 1, 0, st>>>(s);
  return cudaGetLastError();
}

int jcg_num_blocks(const LevelGeom& g, int elem_path, int zc) {
  const int ty = elem_path ? ETY : CTY;
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

template <bool CUBE>
static cudaError_t set_elem_attr() {
  const int sm = CUBE ? ELEM_SMEM_CUBE : ELEM_SMEM;
  cudaError_t e = cudaFuncSetAttribute(k_jcg_elem<MODE_K1, CUBE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem<MODE_K2, CUBE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem<MODE_INIT, CUBE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem<MODE_TRUE, CUBE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_jcg_elem<MODE_APPLY, CUBE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  return e;
}

cudaError_t init_elem_kernel_attributes() {
  cudaError_t e = set_elem_attr<false>();
  if (e == cudaSuccess) e = set_elem_attr<true>();
  return e;
}

template <int MODE>
static cudaError_t launch_elem_mode(dim3 grid, dim3 block, const LevelGeom& g, const ElemStencil& es,
                                    const Problem& pb, const KArgs& a, cudaStream_t st) {
  // cubic cells: the beta-sum form of the element stencil. Measured slower than the general form on
  // C3 (1.08 vs 0.90 ms per iteration: the T_e layer pass adds a barrier and ~70 instructions per node
  // at the same 25% occupancy), so it is kept for reference but not selected.
  constexpr bool kUseCube = false;
  const bool cube = kUseCube && fabs(g.h[0] - g.h[1]) <= 1e-12 * g.h[0] && fabs(g.h[0] - g.h[2]) <= 1e-12 * g.h[0];
  if (cube) {
    count_launch();
    k_jcg_elem<MODE, true><<<grid, block, ELEM_SMEM_CUBE, st>>>(g, es, pb, a);
    return cudaGetLastError();
  }
  count_launch();
  k_jcg_elem<MODE, false><<<grid, block, ELEM_SMEM, st>>>(g, es, pb, a);
  return cudaGetLastError();
}

cudaError_t launch_jcg_elem(int mode, const LevelGeom& g, const ElemStencil& es, const Problem& pb, const KArgs& a,
                            cudaStream_t st) {
  dim3 block(TX, WARPS);
  dim3 grid((g.nf[0] + TX - 1) / TX, (g.nf[1] + ETY - 1) / ETY, (g.zend - g.zbeg + a.zc - 1) / a.zc);
  switch (mode) {
    case MODE_K1: return launch_elem_mode<MODE_K1>(grid, block, g, es, pb, a, st);
    case MODE_K2: return launch_elem_mode<MODE_K2>(grid, block, g, es, pb, a, st);
    case MODE_INIT: return launch_elem_mode<MODE_INIT>(grid, block, g, es, pb, a, st);
    case MODE_TRUE: return launch_elem_mode<MODE_TRUE>(grid, block, g, es, pb, a, st);
    case MODE_APPLY: return launch_elem_mode<MODE_APPLY>(grid, block, g, es, pb, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ecmg
