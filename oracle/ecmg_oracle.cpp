// ecmg_oracle.cpp -- plain, slow, obviously-correct CPU oracle for ECMG_jcg (arXiv:1506.02983).
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library. The product path (paper_1506_02983_b200/) never
// links, imports or executes anything under oracle/, and this file shares no code, header,
// table or constant generator with it.
//
// Citations: "P:n" = /root/reference/PAPER.md line n (with the section / equation label),
// "S:n" = SPEC.md line n, "§8c Ax" = the reading recorded in SURVEY.md §8c and DESIGN.md.
//
// What it computes, step by step, in the paper's order and notation:
//   * the Q1 FE system A_h u_h = f_h of Eq. (fe_equation) for the BVP of Eq. (bvp)
//     (P:39-51): element stiffness K_e[a][b] = sum_q w_q beta_e grad N_a . grad N_b detJ by
//     2x2x2 Gauss (§8c A2, A3), element load by 2x2x2 Gauss, Robin face mass / load by 2x2 Gauss
//     (§8c A4), explicit global assembly into a 27-band matrix (every (row, neighbour-offset)
//     entry stored; no column indices), symmetric Dirichlet elimination (lifting, §8c A5);
//   * JCG = textbook PCG with M = diag(A_ff) (Alg. 4 l.7-9), stopped by the
//     relative residual rule ||r||_2 > eps ||f||_2 checked before every iteration (§8c A7-A10);
//   * DSOLVE = band Cholesky of A_ff (exact direct solve, Alg. 4 l.1-2; §8c A12);
//   * EXP_finite literally: corner seeds by Eq. (jiedian), edge-midpoint seeds by
//     Eq. (zhongdian), the remaining 105 nodes by the printed Serendipity shape
//     functions N_i of Eq. (inter), owner block b = min(i/4, n_4h-1) (§8c A14),
//     Dirichlet overwrite (§8c A15);
//   * EXP_true literally node class by node class: Eq. (t1) at 2h nodes, Eq. (chenlin)
//     at 2h edge centres, mean of chenlin over face / space diagonals at face and cell
//     centres (Remark 2 P:514-516; §8c A13), Dirichlet overwrite;
//   * Alg. 4 level by level, with the diagnostics of Tables 4-10 (errors, r_h,
//     P:725-729; norms per §8c A21).
//
// Built with -O2 -ffp-contract=off (§8c A23). Single threaded by default. orc_set_threads(T > 1) runs the
// node-row loops (assembly scatter, lifting, A_ff p, the vector updates, EXP_finite, EXP_true) over T
// OpenMP threads so that the full-size configs (C3 256^3, C4 512^3, C5 to 512^3) finish in minutes. Every
// result is BITWISE the single-threaded one: each row / node is still computed by the same expression from
// the same operands in the same order (the element contributions to a row keep the lexicographic element
// order, see build_level), and every reduction -- dot products, ||b||^2, norms -- stays one serial loop in
// node order (pinned: tests/test_oracle_threads.py).

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <chrono>
#include <vector>

#include <omp.h>

namespace {

int g_threads = 1;   // orc_set_threads; 1 = the plain serial program

// ----------------------------------------------------------------------------------------------
// Status codes (same numeric meaning as the product ABI, declared independently here).
// ----------------------------------------------------------------------------------------------
enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_ENOMEM = -2, ORC_ENOTCONV = -3, ORC_EBREAKDOWN = -4,
       ORC_EDIAG = -5, ORC_EMISMATCH = -6 };

enum { FACE_DIRICHLET = 0, FACE_ROBIN = 1 };

// Problem ids (interface numbers; the CUDA registry defines the same ids independently).
enum {
  PROB_C1 = 1, PROB_C2 = 2, PROB_C3 = 3, PROB_C4 = 4, PROB_C5 = 5,
  PROB_P1 = 11, PROB_P2 = 12, PROB_P3 = 13,
  PROB_PATCH_TRILINEAR = 21, PROB_PATCH_LAYERED = 22, PROB_PATCH_ROBIN = 23, PROB_CONST_F = 24,
  PROB_PATCH_ROBIN_XY = 25,
  PROB_ARRAYS = 100,   // caller data per level (SURVEY.md §8b ECMG_PROB_ARRAYS; reading R6)
};

const double PI = 3.14159265358979323846;

// ----------------------------------------------------------------------------------------------
// Problem registry: beta, f, g_D, alpha, g_R and (if known) the exact u of Eq. (bvp).
// ----------------------------------------------------------------------------------------------
struct Problem {
  int id = 0;
  int face[6] = {0, 0, 0, 0, 0, 0};  // x-, x+, y-, y+, z-, z+
  std::vector<double> params;
  bool has_exact = false;
  // PROB_ARRAYS: the data of Eq. (bvp) given on one level at the quadrature / nodal points the
  // discretisation reads: beta_e per element (element e = ex + n_x (ey + n_y ez)), f at the 8
  // Gauss points of each element (index 8 e + q, q = q_x + 2 q_y + 4 q_z, bit set = +1/sqrt(3)), g_D per
  // node, g_R at the 4 Gauss points of each Robin face element (per face F in order x-..z+ a block of
  // n_d1 n_d2 4 values, index 4 (e1 + n_d1 e2) + q, q = q_1 + 2 q_2, d1 < d2 the in-face axes); alpha
  // at the same face Gauss points in the same layout (Eq. bvp: alpha piecewise smooth), or, if that
  // array is null, one alpha per face = params[F]. A null array means beta = 1, f = 0, g_D = 0, g_R = 0.
  const double *a_beta = nullptr, *a_f = nullptr, *a_gD = nullptr, *a_gR = nullptr, *a_alpha = nullptr;

  // C5 / layered geometry (params layout documented in synth/__init__.py)
  double layer_beta_at(double z) const {
    int l = 0;
    while (l < 7 && !(z < params[l])) ++l;  // layer = first l with z < z_l (strict), else 7
    return params[7 + l];
  }
  double c5_beta(double x, double y, double z) const {
    double b = layer_beta_at(z);
    for (int k = 0; k < 4; ++k) {  // a later box overrides an earlier one
      const double* q = &params[15 + 7 * k];
      if (std::fabs(x - q[0]) < q[3] && std::fabs(y - q[1]) < q[4] && std::fabs(z - q[2]) < q[5]) b = q[6];
    }
    return b;
  }

  double beta(double x, double y, double z) const {
    switch (id) {
      case PROB_C3: return 1.0 + 0.5 * std::sin(2 * PI * x) * std::cos(2 * PI * y) * std::sin(2 * PI * z);
      case PROB_C5: return c5_beta(x, y, z);
      case PROB_PATCH_LAYERED: return layer_beta_at(z);
      default: return 1.0;
    }
  }

  double exact(double x, double y, double z) const {
    switch (id) {
      case PROB_C1: return std::sin(PI * x) * std::sin(PI * y) * std::sin(PI * z);
      case PROB_C2: return std::exp(x + y + z);
      case PROB_C3: return std::cos(PI * x) * std::cos(PI * y) * std::exp(z);
      case PROB_C4: { double r2 = x * x + y * y + z * z; return std::pow(r2, 0.75); }
      case PROB_P1: return std::sin(0.5 * PI * x) * std::sin(0.5 * PI * y) * std::sin(0.5 * PI * z);
      case PROB_P2: return std::exp(z) * std::sin(1.5 * PI * x) * std::sin(0.5 * PI * y);
      case PROB_P3: { double r2 = x * x + y * y + z * z; if (r2 == 0.0) return 0.0; return x * y * z / std::pow(r2, 0.75); }
      case PROB_PATCH_TRILINEAR: return 1.0 + x + 2.0 * y - z + x * y + 3.0 * x * y * z;
      case PROB_PATCH_LAYERED: return 0.5 + 1.5 * x - 0.75 * y;
      case PROB_PATCH_ROBIN: case PROB_PATCH_ROBIN_XY: return 0.3 + 0.7 * x - 0.4 * y + 0.9 * z;
      default: return 0.0;
    }
  }

  // f = -div(beta grad u)
  double f(double x, double y, double z) const {
    switch (id) {
      case PROB_C1: return 3.0 * PI * PI * exact(x, y, z);
      case PROB_C2: return -3.0 * exact(x, y, z);
      case PROB_C3: {
        double u = exact(x, y, z);
        double b = beta(x, y, z);
        double bx = PI * std::cos(2 * PI * x) * std::cos(2 * PI * y) * std::sin(2 * PI * z);
        double by = -PI * std::sin(2 * PI * x) * std::sin(2 * PI * y) * std::sin(2 * PI * z);
        double bz = PI * std::sin(2 * PI * x) * std::cos(2 * PI * y) * std::cos(2 * PI * z);
        double ux = -PI * std::sin(PI * x) * std::cos(PI * y) * std::exp(z);
        double uy = -PI * std::cos(PI * x) * std::sin(PI * y) * std::exp(z);
        double uz = u;
        return -b * (1.0 - 2.0 * PI * PI) * u - (bx * ux + by * uy + bz * uz);
      }
      case PROB_C4: {  // -Laplace r^{3/2} = -(15/4) r^{-1/2}; f(0) := 0 (§8c A20)
        double r2 = x * x + y * y + z * z;
        if (r2 == 0.0) return 0.0;
        return -3.75 / std::pow(r2, 0.25);
      }
      case PROB_C5: {
        const double* x0 = &params[43];
        double s = params[46], amp = params[47];
        double d2 = (x - x0[0]) * (x - x0[0]) + (y - x0[1]) * (y - x0[1]) + (z - x0[2]) * (z - x0[2]);
        return amp * std::exp(-d2 / (2.0 * s * s));
      }
      case PROB_P1: return 0.75 * PI * PI * exact(x, y, z);                 // Eq. (prob1)
      case PROB_P2: return -(1.0 - 2.5 * PI * PI) * exact(x, y, z);         // Eq. (prob2)
      case PROB_P3: {                                                       // Eq. (prob3)
        double r2 = x * x + y * y + z * z;
        if (r2 == 0.0) return 0.0;
        return 33.0 * x * y * z / (4.0 * std::pow(r2, 1.75));
      }
      case PROB_CONST_F: return 1.0;
      default: return 0.0;  // patch tests: f = 0
    }
  }

  double gD(double x, double y, double z) const { return exact(x, y, z); }

  double alpha(int face_id) const {
    switch (id) {
      case PROB_ARRAYS: return params[face_id];
      case PROB_C3: case PROB_PATCH_ROBIN: return 1.0;
      case PROB_PATCH_ROBIN_XY: {   // Robin on x-, x+, y-, y+ with a different alpha each
        const double a[6] = {2.0, 0.5, 1.5, 3.0, 0.0, 0.0};
        return a[face_id];
      }
      default: return 0.0;  // P1, P2: Neumann = Robin with alpha = 0
    }
  }

  // g_R = alpha u + beta du/dn on the Robin faces
  double gR(int face_id, double x, double y, double z) const {
    switch (id) {
      case PROB_C3: return (alpha(face_id) + beta(x, y, z)) * exact(x, y, z);  // du/dz = u, n = +z
      case PROB_PATCH_ROBIN: return alpha(face_id) * exact(x, y, z) + 1.0 * 0.9;
      case PROB_PATCH_ROBIN_XY: {   // beta du/dn with grad u = (0.7, -0.4, 0.9) and the outward normal
        const double dudn[6] = {-0.7, 0.7, 0.4, -0.4, -0.9, 0.9};
        return alpha(face_id) * exact(x, y, z) + dudn[face_id];
      }
      default: return 0.0;  // P1, P2: homogeneous Neumann
    }
  }
};

bool make_problem(int id, const double* params, int nparams, const int* face_in, Problem* P) {
  P->id = id;
  P->params.assign(params ? params : nullptr, params ? params + nparams : nullptr);
  for (int f = 0; f < 6; ++f) P->face[f] = FACE_DIRICHLET;
  switch (id) {
    case PROB_C1: case PROB_C2: case PROB_C4: case PROB_P3: case PROB_PATCH_TRILINEAR:
      P->has_exact = true; break;
    case PROB_C3: case PROB_PATCH_ROBIN:
      P->has_exact = true; P->face[5] = FACE_ROBIN; break;
    case PROB_PATCH_ROBIN_XY:
      P->has_exact = true; P->face[0] = P->face[1] = P->face[2] = P->face[3] = FACE_ROBIN; break;
    case PROB_P1:
      P->has_exact = true; P->face[1] = P->face[3] = P->face[5] = FACE_ROBIN; break;
    case PROB_P2:
      P->has_exact = true; P->face[1] = P->face[3] = FACE_ROBIN; break;
    case PROB_C5:
      if (nparams < 48) return false;
      P->has_exact = false; break;
    case PROB_PATCH_LAYERED:
      if (nparams < 15) return false;
      P->has_exact = true; break;
    case PROB_CONST_F:
      P->has_exact = false; break;
    case PROB_ARRAYS:
      if (nparams < 6) return false;
      for (int f = 0; f < 6; ++f) if (!(params[f] >= 0.0)) return false;
      P->has_exact = false; break;
    default: return false;
  }
  if (face_in) for (int f = 0; f < 6; ++f) P->face[f] = face_in[f];
  return true;
}

// ----------------------------------------------------------------------------------------------
// Element integrals (§2; quadrature per §8c A2/A4).
// Local node a = ax + 2 ay + 4 az, sign s_ad = (bit d of a) ? +1 : -1, N_a = prod_d (1 + s_ad xi_d)/2.
// ----------------------------------------------------------------------------------------------
const double GAUSS = 0.57735026918962576451;  // 1/sqrt(3)

inline int sgn(int a, int d) { return ((a >> d) & 1) ? 1 : -1; }

void element_stiffness(const double h[3], double beta, double K[8][8]) {
  for (int a = 0; a < 8; ++a) for (int b = 0; b < 8; ++b) K[a][b] = 0.0;
  const double detJ = h[0] * h[1] * h[2] / 8.0;
  for (int q = 0; q < 8; ++q) {
    double xi[3] = {sgn(q, 0) * GAUSS, sgn(q, 1) * GAUSS, sgn(q, 2) * GAUSS};
    double grad[8][3];
    for (int a = 0; a < 8; ++a) {
      for (int d = 0; d < 3; ++d) {
        double g = sgn(a, d) / h[d];  // dN/dxi_d * dxi_d/dx_d = (s/2) * (2/h_d)
        for (int e = 0; e < 3; ++e)
          if (e != d) g *= (1.0 + sgn(a, e) * xi[e]) / 2.0;
        grad[a][d] = g;
      }
    }
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b) {
        double dot = grad[a][0] * grad[b][0] + grad[a][1] * grad[b][1] + grad[a][2] * grad[b][2];
        K[a][b] += beta * dot * detJ;  // weight 1
      }
  }
}

// F_e[a] = sum_q f(x_q) N_a(xi_q) detJ, element with lower corner node index (ex,ey,ez)
void element_load(const Problem& P, const double lo[3], const double h[3], const int e[3], double F[8],
                  const double* f_arr = nullptr /* PROB_ARRAYS: f at this element's 8 Gauss points */) {
  for (int a = 0; a < 8; ++a) F[a] = 0.0;
  const double detJ = h[0] * h[1] * h[2] / 8.0;
  for (int q = 0; q < 8; ++q) {
    double xi[3] = {sgn(q, 0) * GAUSS, sgn(q, 1) * GAUSS, sgn(q, 2) * GAUSS};
    double x[3];
    for (int d = 0; d < 3; ++d) x[d] = lo[d] + (e[d] + (1.0 + xi[d]) / 2.0) * h[d];
    double fq = P.id == PROB_ARRAYS ? (f_arr ? f_arr[q] : 0.0) : P.f(x[0], x[1], x[2]);
    for (int a = 0; a < 8; ++a) {
      double N = 1.0;
      for (int d = 0; d < 3; ++d) N *= (1.0 + sgn(a, d) * xi[d]) / 2.0;
      F[a] += fq * N * detJ;
    }
  }
}

// Face integrals on a rectangle with sides h1, h2 (local face node c = c1 + 2 c2):
// M[c][d] = sum_q alpha_q N_c N_d detJf, G[c] = sum_q g_q N_c detJf, with alpha_q, g_q at the
// 2x2 Gauss points q = q1 + 2 q2 (xi = -g for bit 0, +g for bit 1).
void face_integrals(double h1, double h2, const double alpha_q[4], const double g_q[4], double M[4][4], double G[4]) {
  for (int c = 0; c < 4; ++c) { G[c] = 0.0; for (int d = 0; d < 4; ++d) M[c][d] = 0.0; }
  const double detJf = h1 * h2 / 4.0;
  for (int q = 0; q < 4; ++q) {
    double xi[2] = {sgn(q, 0) * GAUSS, sgn(q, 1) * GAUSS};
    double N[4];
    for (int c = 0; c < 4; ++c) N[c] = (1.0 + sgn(c, 0) * xi[0]) / 2.0 * ((1.0 + sgn(c, 1) * xi[1]) / 2.0);
    for (int c = 0; c < 4; ++c) {
      G[c] += g_q[q] * N[c] * detJf;
      for (int d = 0; d < 4; ++d) M[c][d] += alpha_q[q] * (N[c] * N[d]) * detJf;
    }
  }
}

// ----------------------------------------------------------------------------------------------
// One grid level: explicit assembled 27-band matrix, load, lifted RHS.
// Node index i = ix + (nx+1)(iy + (ny+1) iz); band slot k = (dx+1) + 3(dy+1) + 9(dz+1).
// ----------------------------------------------------------------------------------------------
struct Level {
  int n[3];
  double lo[3], hi[3], h[3];
  long nn[3];
  long N;
  Problem P;
  std::vector<double> A;          // N * 27, full assembled matrix (before elimination)
  std::vector<double> F;          // F + G (volume + Robin load)
  std::vector<unsigned char> dir; // 1 = Dirichlet node
  std::vector<double> gDv;        // g_D on Dirichlet nodes, 0 elsewhere
  std::vector<double> b;          // lifted RHS on free rows, 0 on Dirichlet rows
  double normb = 0.0;

  long idx(long ix, long iy, long iz) const { return ix + nn[0] * (iy + nn[1] * iz); }
  double coord(int d, long i) const { return lo[d] + i * h[d]; }
};

inline int slot(int dx, int dy, int dz) { return (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1); }

bool build_level(Level* L, const double lo[3], const double hi[3], const int n[3], const Problem& P) {
  for (int d = 0; d < 3; ++d) {
    if (n[d] < 1 || !(hi[d] > lo[d])) return false;
    L->n[d] = n[d]; L->lo[d] = lo[d]; L->hi[d] = hi[d];
    L->h[d] = (hi[d] - lo[d]) / n[d];
    L->nn[d] = n[d] + 1;
  }
  L->P = P;
  L->N = L->nn[0] * L->nn[1] * L->nn[2];
  const long N = L->N;
  L->A.assign(N * 27, 0.0);
  L->F.assign(N, 0.0);
  L->dir.assign(N, 0);
  L->gDv.assign(N, 0.0);
  L->b.assign(N, 0.0);

  // node classes: Dirichlet dominates on shared edges (§8c A6)
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (long iz = 0; iz < L->nn[2]; ++iz)
    for (long iy = 0; iy < L->nn[1]; ++iy)
      for (long ix = 0; ix < L->nn[0]; ++ix) {
        long id[3] = {ix, iy, iz};
        bool D = false;
        for (int d = 0; d < 3; ++d) {
          if (id[d] == 0 && P.face[2 * d] == FACE_DIRICHLET) D = true;
          if (id[d] == L->n[d] && P.face[2 * d + 1] == FACE_DIRICHLET) D = true;
        }
        long i = L->idx(ix, iy, iz);
        L->dir[i] = D ? 1 : 0;
        if (D) L->gDv[i] = P.id == PROB_ARRAYS ? (P.a_gD ? P.a_gD[i] : 0.0)
                                               : P.gD(L->coord(0, ix), L->coord(1, iy), L->coord(2, iz));
      }

  // volume terms, elements in lexicographic order
  const double Kh[3] = {L->h[0], L->h[1], L->h[2]};
  auto element_terms = [&](int ex, int ey, int ez, double K[8][8], double Fe[8]) {
    // beta_e = beta at the element centroid (§8c A3)
    double cx = L->lo[0] + (ex + 0.5) * L->h[0];
    double cy = L->lo[1] + (ey + 0.5) * L->h[1];
    double cz = L->lo[2] + (ez + 0.5) * L->h[2];
    const long el = ex + (long)n[0] * (ey + (long)n[1] * ez);
    const double be = P.id == PROB_ARRAYS ? (P.a_beta ? P.a_beta[el] : 1.0) : P.beta(cx, cy, cz);
    element_stiffness(Kh, be, K);
    int e[3] = {ex, ey, ez};
    element_load(P, L->lo, L->h, e, Fe, P.a_f ? P.a_f + 8 * el : nullptr);
  };
  // add element (ex, ey, ez)'s row a to the global row of its local node a
  auto scatter_row = [&](int ex, int ey, int ez, int a, const double K[8][8], const double Fe[8]) {
    long ia = L->idx(ex + (a & 1), ey + ((a >> 1) & 1), ez + ((a >> 2) & 1));
    L->F[ia] += Fe[a];
    for (int bb = 0; bb < 8; ++bb) {
      int dx = (bb & 1) - (a & 1), dy = ((bb >> 1) & 1) - ((a >> 1) & 1), dz = ((bb >> 2) & 1) - ((a >> 2) & 1);
      L->A[ia * 27 + slot(dx, dy, dz)] += K[a][bb];
    }
  };
  if (g_threads <= 1) {
    double K[8][8], Fe[8];
    for (int ez = 0; ez < n[2]; ++ez)
      for (int ey = 0; ey < n[1]; ++ey)
        for (int ex = 0; ex < n[0]; ++ex) {
          element_terms(ex, ey, ez, K, Fe);
          for (int a = 0; a < 8; ++a) scatter_row(ex, ey, ez, a, K, Fe);
        }
  } else {
    // Threaded: one element plane at a time. The plane's element matrices are formed in parallel, then
    // every node row of the two node planes it touches adds its (up to 4) elements of this plane in
    // lexicographic (ey, ex) order. Planes go in ez order, so each row receives the same terms in the
    // same order as in the serial loop above: bitwise the same sums.
    const long npl = (long)n[0] * n[1];
    std::vector<double> Kp((size_t)npl * 64), Fp((size_t)npl * 8);
    for (int ez = 0; ez < n[2]; ++ez) {
#pragma omp parallel for schedule(static) num_threads(g_threads)
      for (long t = 0; t < npl; ++t)
        element_terms((int)(t % n[0]), (int)(t / n[0]), ez, reinterpret_cast<double(*)[8]>(&Kp[(size_t)t * 64]),
                      &Fp[(size_t)t * 8]);
      const long rows_pl = L->nn[0] * L->nn[1];
#pragma omp parallel for schedule(static) num_threads(g_threads)
      for (long t = 0; t < 2 * rows_pl; ++t) {
        const int az = (int)(t / rows_pl);
        const long ix = (t % rows_pl) % L->nn[0], iy = (t % rows_pl) / L->nn[0];
        for (long ey = iy - 1; ey <= iy; ++ey)
          for (long ex = ix - 1; ex <= ix; ++ex) {
            if (ex < 0 || ey < 0 || ex >= n[0] || ey >= n[1]) continue;
            const long e = ex + (long)n[0] * ey;
            const int a = (int)(ix - ex) + 2 * (int)(iy - ey) + 4 * az;
            scatter_row((int)ex, (int)ey, ez, a, reinterpret_cast<const double(*)[8]>(&Kp[(size_t)e * 64]),
                        &Fp[(size_t)e * 8]);
          }
      }
    }
  }

  // Robin faces (a(u,v) gets int alpha u v, f(v) gets int g_R v)
  long gR_block = 0;   // PROB_ARRAYS: offset of this face's block of g_R values
  for (int face = 0; face < 6; ++face) {
    const int d = face / 2, side = face % 2;
    const int d1 = (d == 0) ? 1 : 0, d2 = (d == 2) ? 1 : 2;
    const long block = gR_block;
    gR_block += 4L * n[d1] * n[d2];
    if (P.face[face] != FACE_ROBIN) continue;
    const long fixed = side ? L->n[d] : 0;
    for (int e2 = 0; e2 < n[d2]; ++e2)
      for (int e1 = 0; e1 < n[d1]; ++e1) {
        double aq[4], gq[4];
        for (int q = 0; q < 4; ++q) {
          double xi1 = sgn(q, 0) * GAUSS, xi2 = sgn(q, 1) * GAUSS;
          double x[3];
          x[d] = L->coord(d, fixed);
          x[d1] = L->lo[d1] + (e1 + (1.0 + xi1) / 2.0) * L->h[d1];
          x[d2] = L->lo[d2] + (e2 + (1.0 + xi2) / 2.0) * L->h[d2];
          aq[q] = (P.id == PROB_ARRAYS && P.a_alpha) ? P.a_alpha[block + 4L * (e1 + (long)n[d1] * e2) + q]
                                                     : P.alpha(face);
          gq[q] = P.id == PROB_ARRAYS ? (P.a_gR ? P.a_gR[block + 4L * (e1 + (long)n[d1] * e2) + q] : 0.0)
                                      : P.gR(face, x[0], x[1], x[2]);
        }
        double M[4][4], G[4];
        face_integrals(L->h[d1], L->h[d2], aq, gq, M, G);
        for (int c = 0; c < 4; ++c) {
          long ic[3]; ic[d] = fixed; ic[d1] = e1 + (c & 1); ic[d2] = e2 + ((c >> 1) & 1);
          long i = L->idx(ic[0], ic[1], ic[2]);
          L->F[i] += G[c];
          for (int c2 = 0; c2 < 4; ++c2) {
            int off[3] = {0, 0, 0};
            off[d1] = (c2 & 1) - (c & 1);
            off[d2] = ((c2 >> 1) & 1) - ((c >> 1) & 1);
            L->A[i * 27 + slot(off[0], off[1], off[2])] += M[c][c2];
          }
        }
      }
  }

  // symmetric Dirichlet elimination (lifting): b_f = F_f - A_fD g_D (§8c A5)
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (long iz = 0; iz < L->nn[2]; ++iz)
    for (long iy = 0; iy < L->nn[1]; ++iy)
      for (long ix = 0; ix < L->nn[0]; ++ix) {
        long i = L->idx(ix, iy, iz);
        if (L->dir[i]) { L->b[i] = 0.0; continue; }
        double s = L->F[i];
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              long jx = ix + dx, jy = iy + dy, jz = iz + dz;
              if (jx < 0 || jy < 0 || jz < 0 || jx >= L->nn[0] || jy >= L->nn[1] || jz >= L->nn[2]) continue;
              long j = L->idx(jx, jy, jz);
              if (L->dir[j]) s -= L->A[i * 27 + slot(dx, dy, dz)] * L->gDv[j];
            }
        L->b[i] = s;
      }
  double bb = 0.0;   // ||b||^2, serial in node order
  for (long i = 0; i < N; ++i)
    if (!L->dir[i]) bb += L->b[i] * L->b[i];
  L->normb = std::sqrt(bb);
  return true;
}

// q_f = A_ff p_f on free rows (only free columns), q = 0 on Dirichlet rows
void apply_ff(const Level& L, const double* p, double* q) {
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (long iz = 0; iz < L.nn[2]; ++iz)
    for (long iy = 0; iy < L.nn[1]; ++iy)
      for (long ix = 0; ix < L.nn[0]; ++ix) {
        long i = L.idx(ix, iy, iz);
        if (L.dir[i]) { q[i] = 0.0; continue; }
        double s = 0.0;
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              long jx = ix + dx, jy = iy + dy, jz = iz + dz;
              if (jx < 0 || jy < 0 || jz < 0 || jx >= L.nn[0] || jy >= L.nn[1] || jz >= L.nn[2]) continue;
              long j = L.idx(jx, jy, jz);
              if (L.dir[j]) continue;
              s += L.A[i * 27 + slot(dx, dy, dz)] * p[j];
            }
        q[i] = s;
      }
}

double dot_free(const Level& L, const double* a, const double* b) {
  double s = 0.0;
  for (long i = 0; i < L.N; ++i)
    if (!L.dir[i]) s += a[i] * b[i];
  return s;
}

// the same sum in reverse node order: used only to measure the oracle's own rounding-order spread
// of CG iterates (reading §8c A22), never for a reported result
double dot_free_reversed(const Level& L, const double* a, const double* b) {
  double s = 0.0;
  for (long i = L.N - 1; i >= 0; --i)
    if (!L.dir[i]) s += a[i] * b[i];
  return s;
}

struct SolveStats {
  int iterations = 0;
  double rel_recur = 0.0, rel_true = 0.0, normb = 0.0;
  int status = ORC_OK;
};

// Textbook JCG (precond = 1) or CG (precond = 0), SURVEY.md §8c O7. x is a full nodal vector:
// on entry its free part is the initial guess, on exit the iterate; Dirichlet entries := g_D.
// eps <= 0 means "run exactly max_iter iterations" (fixed-iteration parity and benchmark mode).
SolveStats jcg(const Level& L, double* x, double eps, int max_iter, int precond, int dot_reverse = 0) {
  SolveStats st;
  auto dot_free = [&](const Level& LL, const double* a, const double* b) {
    return dot_reverse ? dot_free_reversed(LL, a, b) : ::dot_free(LL, a, b);
  };
  const long N = L.N;
  std::vector<double> r(N, 0.0), z(N, 0.0), p(N, 0.0), w(N, 0.0), dinv(N, 0.0);
  for (long i = 0; i < N; ++i) {
    if (L.dir[i]) { x[i] = L.gDv[i]; continue; }
    double d = L.A[i * 27 + 13];
    if (!(d > 0.0)) { st.status = ORC_EDIAG; return st; }
    dinv[i] = precond ? 1.0 / d : 1.0;
  }
  apply_ff(L, x, w.data());  // A_ff x_f (Dirichlet columns are skipped by apply_ff)
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (long i = 0; i < N; ++i) if (!L.dir[i]) r[i] = L.b[i] - w[i];
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (long i = 0; i < N; ++i) if (!L.dir[i]) { z[i] = dinv[i] * r[i]; p[i] = z[i]; }
  double rho = dot_free(L, r.data(), z.data());
  double rr = dot_free(L, r.data(), r.data());
  const double nb = (L.normb > 0.0) ? L.normb : 1.0;  // ||b|| = 0: absolute residual (§8c A11)
  st.normb = L.normb;
  int k = 0;
  while (k < max_iter && (eps <= 0.0 || std::sqrt(rr) > eps * nb)) {
    apply_ff(L, p.data(), w.data());
    double sigma = dot_free(L, p.data(), w.data());
    if (!(sigma > 0.0)) { st.status = ORC_EBREAKDOWN; break; }
    double alpha = rho / sigma;
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
    for (long i = 0; i < N; ++i)
      if (!L.dir[i]) { x[i] = x[i] + alpha * p[i]; r[i] = r[i] - alpha * w[i]; }
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
    for (long i = 0; i < N; ++i) if (!L.dir[i]) z[i] = dinv[i] * r[i];
    double rho_new = dot_free(L, r.data(), z.data());
    double beta = rho_new / rho;
    rho = rho_new;
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
    for (long i = 0; i < N; ++i) if (!L.dir[i]) p[i] = z[i] + beta * p[i];
    rr = dot_free(L, r.data(), r.data());
    ++k;
  }
  st.iterations = k;
  st.rel_recur = std::sqrt(rr) / nb;
  apply_ff(L, x, w.data());
  double tr = 0.0;   // serial in node order
  for (long i = 0; i < N; ++i) if (!L.dir[i]) { double t = L.b[i] - w[i]; tr += t * t; }
  st.rel_true = std::sqrt(tr) / nb;
  if (st.status == ORC_OK && eps > 0.0 && std::sqrt(rr) > eps * nb) st.status = ORC_ENOTCONV;
  return st;
}

// DSOLVE: band Cholesky of A_ff (free nodes numbered lexicographically; they form a box because
// Dirichlet is imposed per face). Exact up to rounding (Alg. 4 l.1-2; §8c A12).
int dsolve(const Level& L, double* x) {
  std::vector<long> fidx;  // free node -> node index
  fidx.reserve(L.N);
  std::vector<long> inv(L.N, -1);
  for (long i = 0; i < L.N; ++i) if (!L.dir[i]) { inv[i] = (long)fidx.size(); fidx.push_back(i); }
  const long M = (long)fidx.size();
  for (long i = 0; i < L.N; ++i) if (L.dir[i]) x[i] = L.gDv[i];
  if (M == 0) return ORC_OK;
  // bandwidth: max |inv[j] - inv[i]| over couplings
  long bw = 0;
  for (long f = 0; f < M; ++f) {
    long i = fidx[f];
    long ix = i % L.nn[0], iy = (i / L.nn[0]) % L.nn[1], iz = i / (L.nn[0] * L.nn[1]);
    for (int dz = -1; dz <= 1; ++dz) for (int dy = -1; dy <= 1; ++dy) for (int dx = -1; dx <= 1; ++dx) {
      long jx = ix + dx, jy = iy + dy, jz = iz + dz;
      if (jx < 0 || jy < 0 || jz < 0 || jx >= L.nn[0] || jy >= L.nn[1] || jz >= L.nn[2]) continue;
      long j = L.idx(jx, jy, jz);
      if (inv[j] >= 0) { long d = inv[j] - f; if (d < 0) d = -d; if (d > bw) bw = d; }
    }
  }
  auto Aff = [&](long fi, long fj) -> double {
    long i = fidx[fi], j = fidx[fj];
    long ix = i % L.nn[0], iy = (i / L.nn[0]) % L.nn[1], iz = i / (L.nn[0] * L.nn[1]);
    long jx = j % L.nn[0], jy = (j / L.nn[0]) % L.nn[1], jz = j / (L.nn[0] * L.nn[1]);
    long dx = jx - ix, dy = jy - iy, dz = jz - iz;
    if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) return 0.0;
    return L.A[i * 27 + slot((int)dx, (int)dy, (int)dz)];
  };
  // Lb[f*(bw+1) + (f - j)] = L(f, j) for f - bw <= j <= f
  std::vector<double> Lb((size_t)M * (bw + 1), 0.0);
  auto Lr = [&](long i, long j) -> double& { return Lb[(size_t)i * (bw + 1) + (i - j)]; };
  for (long j = 0; j < M; ++j) {
    double s = Aff(j, j);
    for (long k = std::max(0L, j - bw); k < j; ++k) s -= Lr(j, k) * Lr(j, k);
    if (!(s > 0.0)) return ORC_EBREAKDOWN;
    double djj = std::sqrt(s);
    Lr(j, j) = djj;
    for (long i = j + 1; i <= std::min(M - 1, j + bw); ++i) {
      double t = Aff(i, j);
      for (long k = std::max(0L, i - bw); k < j; ++k) t -= Lr(i, k) * Lr(j, k);
      Lr(i, j) = t / djj;
    }
  }
  std::vector<double> y(M);
  for (long i = 0; i < M; ++i) {
    double s = L.b[fidx[i]];
    for (long k = std::max(0L, i - bw); k < i; ++k) s -= Lr(i, k) * y[k];
    y[i] = s / Lr(i, i);
  }
  for (long i = M - 1; i >= 0; --i) {
    double s = y[i];
    for (long k = i + 1; k <= std::min(M - 1, i + bw); ++k) s -= Lr(k, i) * y[k];
    y[i] = s / Lr(i, i);
  }
  for (long f = 0; f < M; ++f) x[fidx[f]] = y[f];
  return ORC_OK;
}

// ----------------------------------------------------------------------------------------------
// Serendipity shape functions of Eq. (inter), literally, in label order.
// Label = 1 + lx + 5 ly + 25 lz on the 5x5x5 block (Fig. 3).
// ----------------------------------------------------------------------------------------------
const int SEED_LABEL[20] = {1, 3, 5, 11, 15, 21, 23, 25, 51, 55, 71, 75, 101, 103, 105, 111, 115, 121, 123, 125};

inline void label_local(int label, int l[3]) {
  int t = label - 1;
  l[0] = t % 5; l[1] = (t / 5) % 5; l[2] = t / 25;
}

// N_i(xi, eta, zeta) for seed label i
double serendipity_N(int label, double xi, double eta, double zeta) {
  int l[3]; label_local(label, l);
  double xi_i = (l[0] - 2) / 2.0, eta_i = (l[1] - 2) / 2.0, zeta_i = (l[2] - 2) / 2.0;
  switch (label) {
    case 1: case 5: case 21: case 25: case 101: case 105: case 121: case 125:
      return 0.125 * (1 + xi_i * xi) * (1 + eta_i * eta) * (1 + zeta_i * zeta) * (xi_i * xi + eta_i * eta + zeta_i * zeta - 2);
    case 3: case 23: case 103: case 123:
      return 0.25 * (1 - xi * xi) * (1 + eta_i * eta) * (1 + zeta_i * zeta);
    case 11: case 15: case 111: case 115:
      return 0.25 * (1 - eta * eta) * (1 + xi_i * xi) * (1 + zeta_i * zeta);
    case 51: case 55: case 71: case 75:
      return 0.25 * (1 - zeta * zeta) * (1 + xi_i * xi) * (1 + eta_i * eta);
  }
  return 0.0;
}

// EXP_finite (Alg. 4 l.6 "w_h = EXP_finite(u_2h, u_4h)"; §4.3) at fine node
// (ix, iy, iz) of a level with n cells per axis (before the Dirichlet overwrite): the owner 4h block's
// 20 seeds by Eqs. (jiedian) / (zhongdian), then W = sum_i N_i W_i (Eq. inter) in label order.
double exp_finite_node(const int n[3], const double* u2h, const double* u4h, long ix, long iy, long iz) {
  const long n4[3] = {n[0] / 4, n[1] / 4, n[2] / 4};
  const long nn2[3] = {n[0] / 2 + 1, n[1] / 2 + 1, n[2] / 2 + 1};
  const long nn4[3] = {n4[0] + 1, n4[1] + 1, n4[2] + 1};
  auto U1 = [&](long i, long j, long k) { return u2h[i + nn2[0] * (j + nn2[1] * k)]; };
  auto U0 = [&](long i, long j, long k) { return u4h[i + nn4[0] * (j + nn4[1] * k)]; };
  long id[3] = {ix, iy, iz}, b[3], l[3];
  for (int d = 0; d < 3; ++d) { b[d] = std::min(id[d] / 4, n4[d] - 1); l[d] = id[d] - 4 * b[d]; }
  // the 20 seeds of block b, in label order
  double seed[20];
  for (int s = 0; s < 20; ++s) {
    int ls[3]; label_local(SEED_LABEL[s], ls);
    int nmid = (ls[0] == 2) + (ls[1] == 2) + (ls[2] == 2);
    if (nmid == 0) {
      // corner: W = (5 U^1 - U^0)/4, Eq. (jiedian)
      double u1 = U1(2 * b[0] + ls[0] / 2, 2 * b[1] + ls[1] / 2, 2 * b[2] + ls[2] / 2);
      double u0 = U0(b[0] + ls[0] / 4, b[1] + ls[1] / 4, b[2] + ls[2] / 4);
      seed[s] = (5.0 * u1 - u0) / 4.0;
    } else {
      // edge midpoint: W = U^1_mid + (1/8)(U^1_a - U^0_a + U^1_b - U^0_b), Eq. (zhongdian)
      int dm = (ls[0] == 2) ? 0 : (ls[1] == 2 ? 1 : 2);
      long la[3] = {ls[0], ls[1], ls[2]}, lb[3] = {ls[0], ls[1], ls[2]};
      la[dm] = 0; lb[dm] = 4;
      double um = U1(2 * b[0] + ls[0] / 2, 2 * b[1] + ls[1] / 2, 2 * b[2] + ls[2] / 2);
      double u1a = U1(2 * b[0] + la[0] / 2, 2 * b[1] + la[1] / 2, 2 * b[2] + la[2] / 2);
      double u0a = U0(b[0] + la[0] / 4, b[1] + la[1] / 4, b[2] + la[2] / 4);
      double u1b = U1(2 * b[0] + lb[0] / 2, 2 * b[1] + lb[1] / 2, 2 * b[2] + lb[2] / 2);
      double u0b = U0(b[0] + lb[0] / 4, b[1] + lb[1] / 4, b[2] + lb[2] / 4);
      seed[s] = um + (1.0 / 8.0) * (u1a - u0a + u1b - u0b);
    }
  }
  double xi = (l[0] - 2) / 2.0, eta = (l[1] - 2) / 2.0, zeta = (l[2] - 2) / 2.0;
  double W = 0.0;
  for (int s = 0; s < 20; ++s) W += serendipity_N(SEED_LABEL[s], xi, eta, zeta) * seed[s];
  return W;
}

void exp_finite(const Level& Lf, const double* u2h, const double* u4h, double* w) {
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (long iz = 0; iz < Lf.nn[2]; ++iz)
    for (long iy = 0; iy < Lf.nn[1]; ++iy)
      for (long ix = 0; ix < Lf.nn[0]; ++ix) {
        long i = Lf.idx(ix, iy, iz);
        w[i] = Lf.dir[i] ? Lf.gDv[i] : exp_finite_node(Lf.n, u2h, u4h, ix, iy, iz);  // Dirichlet overwrite (§8c A15)
      }
}

// EXP_finite, Remark 2 variant: the 27 2h nodes of each 4h block get extrapolated
// values -- corners by Eq. (jiedian), edge midpoints by Eq. (zhongdian), face centres by the mean
// of Eq. (zhongdian) along the 2 face diagonals, the cell centre by the mean along the 4 space
// diagonals -- and the remaining 98 nodes by tri-quadratic Lagrange interpolation of those 27.
double lagrange_quadratic(int node, double t) {  // node in {0,1,2} at t = -1, 0, 1
  if (node == 0) return t * (t - 1.0) / 2.0;
  if (node == 1) return 1.0 - t * t;
  return t * (t + 1.0) / 2.0;
}

double exp_finite_lagrange_node(const int n[3], const double* u2h, const double* u4h, long ix, long iy, long iz) {
  const long n4[3] = {n[0] / 4, n[1] / 4, n[2] / 4};
  const long nn2[3] = {n[0] / 2 + 1, n[1] / 2 + 1, n[2] / 2 + 1};
  const long nn4[3] = {n4[0] + 1, n4[1] + 1, n4[2] + 1};
  auto U1 = [&](long i, long j, long k) { return u2h[i + nn2[0] * (j + nn2[1] * k)]; };
  auto U0 = [&](long i, long j, long k) { return u4h[i + nn4[0] * (j + nn4[1] * k)]; };
  long id[3] = {ix, iy, iz}, b[3], l[3];
  for (int d = 0; d < 3; ++d) { b[d] = std::min(id[d] / 4, n4[d] - 1); l[d] = id[d] - 4 * b[d]; }
  double seed[3][3][3];  // [k][j][i] local 2h offsets 0..2 in the block
  for (int k = 0; k < 3; ++k)
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) {
        int c[3] = {i, j, k};
        int ax[3], na = 0;
        for (int d = 0; d < 3; ++d) if (c[d] == 1) ax[na++] = d;
        long g[3] = {2 * b[0] + i, 2 * b[1] + j, 2 * b[2] + k};  // 2h index
        if (na == 0) {
          seed[k][j][i] = (5.0 * U1(g[0], g[1], g[2]) - U0(b[0] + i / 2, b[1] + j / 2, b[2] + k / 2)) / 4.0;
          continue;
        }
        int nseg = 1 << (na - 1);
        double sum = 0.0;
        for (int s = 0; s < nseg; ++s) {
          int ca[3] = {i, j, k}, cb[3] = {i, j, k};
          ca[ax[0]] = 0; cb[ax[0]] = 2;
          for (int t = 1; t < na; ++t) {
            bool plus = (s >> (t - 1)) & 1;
            ca[ax[t]] = plus ? 0 : 2; cb[ax[t]] = plus ? 2 : 0;
          }
          double ua1 = U1(2 * b[0] + ca[0], 2 * b[1] + ca[1], 2 * b[2] + ca[2]);
          double ua0 = U0(b[0] + ca[0] / 2, b[1] + ca[1] / 2, b[2] + ca[2] / 2);
          double ub1 = U1(2 * b[0] + cb[0], 2 * b[1] + cb[1], 2 * b[2] + cb[2]);
          double ub0 = U0(b[0] + cb[0] / 2, b[1] + cb[1] / 2, b[2] + cb[2] / 2);
          sum += U1(g[0], g[1], g[2]) + (1.0 / 8.0) * (ua1 - ua0 + ub1 - ub0);  // Eq. (zhongdian)
        }
        seed[k][j][i] = sum / nseg;
      }
  double xi = (l[0] - 2) / 2.0, eta = (l[1] - 2) / 2.0, zeta = (l[2] - 2) / 2.0;
  double W = 0.0;
  for (int k = 0; k < 3; ++k)
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i)
        W += lagrange_quadratic(i, xi) * lagrange_quadratic(j, eta) * lagrange_quadratic(k, zeta) * seed[k][j][i];
  return W;
}

void exp_finite_lagrange(const Level& Lf, const double* u2h, const double* u4h, double* w) {
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (long iz = 0; iz < Lf.nn[2]; ++iz)
    for (long iy = 0; iy < Lf.nn[1]; ++iy)
      for (long ix = 0; ix < Lf.nn[0]; ++ix) {
        long ii = Lf.idx(ix, iy, iz);
        w[ii] = Lf.dir[ii] ? Lf.gDv[ii] : exp_finite_lagrange_node(Lf.n, u2h, u4h, ix, iy, iz);
      }
}

// EXP_true (Alg. 4 l.10 "u~_h = EXP_true(u_h, u_2h)") at fine node (ix, iy, iz)
// of a level with n cells per axis, before the Dirichlet overwrite
double exp_true_node(const int n[3], const double* uh, const double* u2h, long ix, long iy, long iz) {
  const long nn[3] = {n[0] + 1L, n[1] + 1L, n[2] + 1L};
  const long nn2[3] = {n[0] / 2 + 1, n[1] / 2 + 1, n[2] / 2 + 1};
  auto U1 = [&](long i, long j, long k) { return uh[i + nn[0] * (j + nn[1] * k)]; };
  auto U0 = [&](long i, long j, long k) { return u2h[(i / 2) + nn2[0] * ((j / 2) + nn2[1] * (k / 2))]; };
  // Chen-Lin value at midpoint m of the segment a..b (a, b coarse-coincident), Eq. (chenlin)
  auto chenlin = [&](const long m[3], const long a[3], const long b[3]) {
    return U1(m[0], m[1], m[2]) + (1.0 / 6.0) * (U1(a[0], a[1], a[2]) - U0(a[0], a[1], a[2]) +
                                                   U1(b[0], b[1], b[2]) - U0(b[0], b[1], b[2]));
  };
  long m[3] = {ix, iy, iz};
  int odd[3] = {(int)(ix & 1), (int)(iy & 1), (int)(iz & 1)};
  int nodd = odd[0] + odd[1] + odd[2];
  if (nodd == 0) return (4.0 * U1(ix, iy, iz) - U0(ix, iy, iz)) / 3.0;  // Eq. (t1)
  // enumerate the diagonals through m: sign patterns over the odd axes with the first odd
  // axis fixed to -1 (a) / +1 (b): 1 segment (edge), 2 (face), 4 (cell)
  int ax[3], na = 0;
  for (int d = 0; d < 3; ++d) if (odd[d]) ax[na++] = d;
  int nseg = 1 << (na - 1);
  double sum = 0.0;
  for (int s = 0; s < nseg; ++s) {
    long a[3] = {ix, iy, iz}, b[3] = {ix, iy, iz};
    a[ax[0]] -= 1; b[ax[0]] += 1;
    for (int t = 1; t < na; ++t) {
      int sg = ((s >> (t - 1)) & 1) ? 1 : -1;
      a[ax[t]] -= sg; b[ax[t]] += sg;
    }
    sum += chenlin(m, a, b);
  }
  return sum / nseg;  // arithmetic mean over the diagonals (§8c A13)
}

void exp_true(const Level& Lf, const double* uh, const double* u2h, double* ut) {
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (long iz = 0; iz < Lf.nn[2]; ++iz)
    for (long iy = 0; iy < Lf.nn[1]; ++iy)
      for (long ix = 0; ix < Lf.nn[0]; ++ix) {
        long i = Lf.idx(ix, iy, iz);
        ut[i] = Lf.dir[i] ? Lf.gDv[i] : exp_true_node(Lf.n, uh, u2h, ix, iy, iz);
      }
}

// ---- one row at a time (parity at full size on sampled nodes: no global matrix) -------------
// Row i = (ix, iy, iz) of the assembled matrix (27 entries by neighbour offset, before elimination)
// and its load F_i, accumulated exactly as build_level does: the (up to 8) elements around the node
// in the same lexicographic element order, then the Robin faces in face and face-element order. Every
// entry is therefore the same sum in the same order as build_level's.
bool node_is_dirichlet(const Problem& P, const int n[3], long ix, long iy, long iz) {
  long id[3] = {ix, iy, iz};
  for (int d = 0; d < 3; ++d) {
    if (id[d] == 0 && P.face[2 * d] == FACE_DIRICHLET) return true;
    if (id[d] == n[d] && P.face[2 * d + 1] == FACE_DIRICHLET) return true;
  }
  return false;
}

void assemble_row(const Problem& P, const double lo[3], const double h[3], const int n[3], long ix, long iy, long iz,
                  double A27[27], double* F) {
  for (int t = 0; t < 27; ++t) A27[t] = 0.0;
  *F = 0.0;
  double K[8][8], Fe[8];
  const long id[3] = {ix, iy, iz};
  for (long ez = iz - 1; ez <= iz; ++ez)
    for (long ey = iy - 1; ey <= iy; ++ey)
      for (long ex = ix - 1; ex <= ix; ++ex) {
        if (ex < 0 || ey < 0 || ez < 0 || ex >= n[0] || ey >= n[1] || ez >= n[2]) continue;
        double cx = lo[0] + (ex + 0.5) * h[0];
        double cy = lo[1] + (ey + 0.5) * h[1];
        double cz = lo[2] + (ez + 0.5) * h[2];
        element_stiffness(h, P.beta(cx, cy, cz), K);
        int e[3] = {(int)ex, (int)ey, (int)ez};
        element_load(P, lo, h, e, Fe);
        const int a = (int)(ix - ex) + 2 * (int)(iy - ey) + 4 * (int)(iz - ez);
        *F += Fe[a];
        for (int bb = 0; bb < 8; ++bb) {
          int dx = (bb & 1) - (a & 1), dy = ((bb >> 1) & 1) - ((a >> 1) & 1), dz = ((bb >> 2) & 1) - ((a >> 2) & 1);
          A27[slot(dx, dy, dz)] += K[a][bb];
        }
      }
  for (int face = 0; face < 6; ++face) {
    if (P.face[face] != FACE_ROBIN) continue;
    const int d = face / 2, side = face % 2;
    const int d1 = (d == 0) ? 1 : 0, d2 = (d == 2) ? 1 : 2;
    const long fixed = side ? n[d] : 0;
    if (id[d] != fixed) continue;
    for (long e2 = id[d2] - 1; e2 <= id[d2]; ++e2)
      for (long e1 = id[d1] - 1; e1 <= id[d1]; ++e1) {
        if (e1 < 0 || e2 < 0 || e1 >= n[d1] || e2 >= n[d2]) continue;
        double aq[4], gq[4];
        for (int q = 0; q < 4; ++q) {
          double xi1 = sgn(q, 0) * GAUSS, xi2 = sgn(q, 1) * GAUSS;
          double x[3];
          x[d] = lo[d] + fixed * h[d];
          x[d1] = lo[d1] + (e1 + (1.0 + xi1) / 2.0) * h[d1];
          x[d2] = lo[d2] + (e2 + (1.0 + xi2) / 2.0) * h[d2];
          aq[q] = P.alpha(face);
          gq[q] = P.gR(face, x[0], x[1], x[2]);
        }
        double M[4][4], G[4];
        face_integrals(h[d1], h[d2], aq, gq, M, G);
        const int c = (int)(id[d1] - e1) + 2 * (int)(id[d2] - e2);
        *F += G[c];
        for (int c2 = 0; c2 < 4; ++c2) {
          int off[3] = {0, 0, 0};
          off[d1] = (c2 & 1) - (c & 1);
          off[d2] = ((c2 >> 1) & 1) - ((c >> 1) & 1);
          A27[slot(off[0], off[1], off[2])] += M[c][c2];
        }
      }
  }
}

void norms(const Level& L, const double* e, double* l2, double* linf) {
  double s = 0.0, m = 0.0;
  for (long i = 0; i < L.N; ++i) { s += e[i] * e[i]; double a = std::fabs(e[i]); if (a > m) m = a; }
  // Discrete L2 = RMS over all nodes, sqrt(sum e_i^2 / N_nodes). Reading of §8c A21 fixed by the
  // paper itself: with this normalisation the oracle reproduces the L2 columns of Tables 4, 6, 8
  // and 10 (e.g. ||U-u||_2 = 1.42e-4 at 32^3; 2.97e-4 at 40x16x20), while
  // sqrt(h^3 sum e^2) is larger by exactly sqrt((n+1)^3/n^3).
  *l2 = std::sqrt(s / (double)L.N);
  *linf = m;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// ==============================================================================================
// C interface (ctypes, oracle/__init__.py)
// ==============================================================================================
extern "C" {

struct orc_level { Level L; };

orc_level* orc_build_level(const double* lo, const double* hi, const int* n, int problem_id,
                           const double* params, int nparams, const int* face) {
  Problem P;
  if (problem_id == PROB_ARRAYS || !make_problem(problem_id, params, nparams, face, &P)) return nullptr;
  orc_level* h = new orc_level;
  if (!build_level(&h->L, lo, hi, n, P)) { delete h; return nullptr; }
  return h;
}

// PROB_ARRAYS level: alpha[6] per face (used where alpha_q is NULL), arrays as documented at Problem::a_beta
// (each may be NULL)
orc_level* orc_build_level_arrays(const double* lo, const double* hi, const int* n, const int* face,
                                  const double* alpha, const double* beta_e, const double* f_q, const double* gD_n,
                                  const double* gR_q, const double* alpha_q) {
  Problem P;
  if (!make_problem(PROB_ARRAYS, alpha, 6, face, &P)) return nullptr;
  P.a_beta = beta_e; P.a_f = f_q; P.a_gD = gD_n; P.a_gR = gR_q; P.a_alpha = alpha_q;
  orc_level* h = new orc_level;
  if (!build_level(&h->L, lo, hi, n, P)) { delete h; return nullptr; }
  return h;
}

void orc_free_level(orc_level* h) { delete h; }

// Threads of the row loops (1 = serial, the default); results are bitwise independent of it.
int orc_set_threads(int t) {
  if (t < 1) return ORC_EINVAL;
  g_threads = t;
  return ORC_OK;
}
int orc_get_threads(void) { return g_threads; }
int orc_max_threads(void) { return omp_get_num_procs(); }
long orc_num_nodes(const orc_level* h) { return h->L.N; }
void orc_get_matrix(const orc_level* h, double* band) { std::memcpy(band, h->L.A.data(), sizeof(double) * h->L.N * 27); }
void orc_get_load(const orc_level* h, double* F) { std::memcpy(F, h->L.F.data(), sizeof(double) * h->L.N); }
double orc_get_rhs(const orc_level* h, double* b) { std::memcpy(b, h->L.b.data(), sizeof(double) * h->L.N); return h->L.normb; }
void orc_get_dirichlet(const orc_level* h, unsigned char* mask, double* gD) {
  std::memcpy(mask, h->L.dir.data(), h->L.N);
  std::memcpy(gD, h->L.gDv.data(), sizeof(double) * h->L.N);
}
void orc_apply(const orc_level* h, const double* p, double* q) { apply_ff(h->L, p, q); }

int orc_jcg(const orc_level* h, double* x, double eps, int max_iter, int precond, int dot_reverse, int* iters,
            double* rel_recur, double* rel_true, double* normb) {
  SolveStats st = jcg(h->L, x, eps, max_iter, precond, dot_reverse);
  *iters = st.iterations; *rel_recur = st.rel_recur; *rel_true = st.rel_true; *normb = st.normb;
  return st.status;
}

int orc_dsolve(const orc_level* h, double* x) { return dsolve(h->L, x); }

void orc_exact(const orc_level* h, double* u) {
  const Level& L = h->L;
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
  for (long iz = 0; iz < L.nn[2]; ++iz)
    for (long iy = 0; iy < L.nn[1]; ++iy)
      for (long ix = 0; ix < L.nn[0]; ++ix)
        u[L.idx(ix, iy, iz)] = L.P.exact(L.coord(0, ix), L.coord(1, iy), L.coord(2, iz));
}

int orc_exp_finite(const orc_level* fine, const double* u2h, const double* u4h, double* w, int variant) {
  for (int d = 0; d < 3; ++d) if (fine->L.n[d] % 4) return ORC_EMISMATCH;
  if (variant == 1) exp_finite_lagrange(fine->L, u2h, u4h, w);
  else exp_finite(fine->L, u2h, u4h, w);
  return ORC_OK;
}

int orc_exp_true(const orc_level* fine, const double* uh, const double* u2h, double* ut) {
  for (int d = 0; d < 3; ++d) if (fine->L.n[d] % 2) return ORC_EMISMATCH;
  exp_true(fine->L, uh, u2h, ut);
  return ORC_OK;
}

void orc_norms(const orc_level* h, const double* e, double* l2, double* linf) { norms(h->L, e, l2, linf); }

// Sampled rows of a level without assembling it: for node k of `nodes` (ix, iy, iz triples),
// q[k] = (A_ff p)_i (0 on Dirichlet rows; p a full nodal vector, free entries used) and b[k] = the lifted
// right-hand side b_f,i = F_i - sum_{j Dirichlet} A_ij g_D(x_j) (0 on Dirichlet rows), with the
// neighbour loops in apply_ff's / build_level's order; dg[k] = A_ii. p, q, b, dg may be NULL.
int orc_rows(const double* lo, const double* hi, const int* n, int problem_id, const double* params, int nparams,
             const int* face, const long long* nodes, long count, const double* p, double* q, double* b, double* dg) {
  if (problem_id == PROB_ARRAYS) return ORC_EINVAL;   // per-level arrays: orc_build_level_arrays
  Problem P;
  if (!make_problem(problem_id, params, nparams, face, &P)) return ORC_EINVAL;
  double h[3];
  long nn[3];
  for (int d = 0; d < 3; ++d) {
    if (n[d] < 1 || !(hi[d] > lo[d])) return ORC_EINVAL;
    h[d] = (hi[d] - lo[d]) / n[d];
    nn[d] = n[d] + 1;
  }
  auto idx = [&](long x, long y, long z) { return x + nn[0] * (y + nn[1] * z); };
  auto coord = [&](int d, long i) { return lo[d] + i * h[d]; };
  for (long k = 0; k < count; ++k) {
    const long ix = nodes[3 * k], iy = nodes[3 * k + 1], iz = nodes[3 * k + 2];
    if (ix < 0 || iy < 0 || iz < 0 || ix > n[0] || iy > n[1] || iz > n[2]) return ORC_EINVAL;
    if (node_is_dirichlet(P, n, ix, iy, iz)) {
      if (q) q[k] = 0.0;
      if (b) b[k] = 0.0;
      if (dg) dg[k] = 0.0;
      continue;
    }
    double A27[27], F;
    assemble_row(P, lo, h, n, ix, iy, iz, A27, &F);
    if (dg) dg[k] = A27[slot(0, 0, 0)];   // the Jacobi diagonal A_ii
    double sq = 0.0, sb = F;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          long jx = ix + dx, jy = iy + dy, jz = iz + dz;
          if (jx < 0 || jy < 0 || jz < 0 || jx >= nn[0] || jy >= nn[1] || jz >= nn[2]) continue;
          if (node_is_dirichlet(P, n, jx, jy, jz)) {
            sb -= A27[slot(dx, dy, dz)] * P.gD(coord(0, jx), coord(1, jy), coord(2, jz));
          } else if (p) {
            sq += A27[slot(dx, dy, dz)] * p[idx(jx, jy, jz)];
          }
        }
    if (q) q[k] = sq;
    if (b) b[k] = sb;
  }
  return ORC_OK;
}

// EXP_finite / EXP_true at sampled fine nodes (with the Dirichlet overwrite by g_D), per-node bodies
// of exp_finite / exp_finite_lagrange / exp_true
int orc_exp_nodes(const double* lo, const double* hi, const int* n, int problem_id, const double* params, int nparams,
                  const int* face, int which /* 0 Serendipity, 1 Lagrange, 2 EXP_true */, const double* a,
                  const double* c, const long long* nodes, long count, double* out) {
  if (problem_id == PROB_ARRAYS) return ORC_EINVAL;   // per-level arrays: orc_build_level_arrays
  Problem P;
  if (!make_problem(problem_id, params, nparams, face, &P)) return ORC_EINVAL;
  for (int d = 0; d < 3; ++d) if (n[d] % (which == 2 ? 2 : 4)) return ORC_EMISMATCH;
  for (long k = 0; k < count; ++k) {
    const long ix = nodes[3 * k], iy = nodes[3 * k + 1], iz = nodes[3 * k + 2];
    if (ix < 0 || iy < 0 || iz < 0 || ix > n[0] || iy > n[1] || iz > n[2]) return ORC_EINVAL;
    if (node_is_dirichlet(P, n, ix, iy, iz)) {
      const double h0 = (hi[0] - lo[0]) / n[0], h1 = (hi[1] - lo[1]) / n[1], h2 = (hi[2] - lo[2]) / n[2];
      out[k] = P.gD(lo[0] + ix * h0, lo[1] + iy * h1, lo[2] + iz * h2);
      continue;
    }
    out[k] = which == 2 ? exp_true_node(n, a, c, ix, iy, iz)
                        : (which == 1 ? exp_finite_lagrange_node(n, a, c, ix, iy, iz) : exp_finite_node(n, a, c, ix, iy, iz));
  }
  return ORC_OK;
}

void orc_element_stiffness(const double* h, double beta, double* K) {
  double Kl[8][8];
  element_stiffness(h, beta, Kl);
  std::memcpy(K, Kl, sizeof(Kl));
}

void orc_face_integrals(double h1, double h2, const double* alpha_q, const double* g_q, double* M, double* G) {
  double Ml[4][4];
  face_integrals(h1, h2, alpha_q, g_q, Ml, G);
  std::memcpy(M, Ml, sizeof(Ml));
}

void orc_serendipity_weights(double xi, double eta, double zeta, double* w20) {
  for (int s = 0; s < 20; ++s) w20[s] = serendipity_N(SEED_LABEL[s], xi, eta, zeta);
}

// Per-level stats row layout (ORC_NSTAT doubles per level):
//  0 iterations (-1 for DSOLVE levels), 1 rel_recur, 2 rel_true, 3 normb,
//  4 ||U-u||_2, 5 ||U-u||_inf, 6 ||u~-u||_2, 7 ||u~-u||_inf, 8 ||W-U||_2, 9 ||W-U||_inf, 10 r_h,
//  11 t_setup, 12 t_exp, 13 t_solve, 14 t_rich, 15 status, 16 free unknowns
#define ORC_NSTAT 17

// Alg. 4. exp_variant 0 = 20-node Serendipity, 1 = Remark 2's 27-node
// Lagrange. precond 1 = ECMG_jcg, 0 = ECMG_cg. Levels 0..num_levels-1, level k has coarsest*2^k cells per axis.
// u_fine / ut_fine (may be NULL) receive u_h and u~_h of the finest level; w_fine (may be NULL)
// receives W_h of the finest level. Errors are NaN when the problem has no exact solution.
// Shared body of Alg. 4 and Alg. 3: level k >= 2 solves with (eps_k[k], maxit_k[k]); eps_k <= 0
// means exactly maxit_k[k] CG / JCG iterations (Alg. 3's fixed counts).
static int ecmg_impl(const double* lo, const double* hi, const int* coarsest, int num_levels, int problem_id,
                     const double* params, int nparams, const int* face, const double* eps_k, const int* maxit_k,
                     int precond, int exp_variant, double* stats, double* u_fine, double* ut_fine, double* w_fine,
                     const double* const* level_arrays = nullptr /* PROB_ARRAYS: 4 per level */,
                     int n_level_arrays = 0 /* 4 L, or 5 L: [4 L + k] = alpha at the face Gauss points of level k */) {
  Problem P;
  if (!make_problem(problem_id, params, nparams, face, &P)) return ORC_EINVAL;
  if (num_levels < 3) return ORC_EINVAL;
  std::vector<double> u_prev2, u_prev1;  // u_{4h}, u_{2h}
  int status = ORC_OK;
  double rh_prev = 0.0; (void)rh_prev;
  for (int k = 0; k < num_levels; ++k) {
    double* row = stats + (size_t)k * ORC_NSTAT;
    for (int t = 0; t < ORC_NSTAT; ++t) row[t] = NAN;
    int n[3] = {coarsest[0] << k, coarsest[1] << k, coarsest[2] << k};
    double t0 = now_s();
    Level* L = new Level;
    if (problem_id == PROB_ARRAYS) {
      if (!level_arrays) { delete L; return ORC_EINVAL; }
      P.a_beta = level_arrays[4 * k]; P.a_f = level_arrays[4 * k + 1];
      P.a_gD = level_arrays[4 * k + 2]; P.a_gR = level_arrays[4 * k + 3];
      P.a_alpha = n_level_arrays >= 5 * num_levels ? level_arrays[4 * num_levels + k] : nullptr;
    }
    if (!build_level(L, lo, hi, n, P)) { delete L; return ORC_EINVAL; }
    double t1 = now_s();
    row[11] = t1 - t0;
    row[3] = L->normb;
    long nfree = 0; for (long i = 0; i < L->N; ++i) nfree += !L->dir[i];
    row[16] = (double)nfree;
    std::vector<double> u(L->N, 0.0), w, ut;
    if (k < 2) {
      // DSOLVE (Alg. 4 l.1-2)
      int s = dsolve(*L, u.data());
      double t2 = now_s();
      row[13] = t2 - t1;
      row[0] = -1; row[15] = s;
      if (s != ORC_OK) { delete L; return s; }
      // report the true residual of the direct solve
      std::vector<double> q(L->N);
      apply_ff(*L, u.data(), q.data());
      double tr = 0.0; for (long i = 0; i < L->N; ++i) if (!L->dir[i]) { double t = L->b[i] - q[i]; tr += t * t; }
      double nb = L->normb > 0 ? L->normb : 1.0;
      row[1] = row[2] = std::sqrt(tr) / nb;
    } else {
      // W_h = EXP_finite(u_2h, u_4h)  (Alg. 4 l.6)
      w.assign(L->N, 0.0);
      if (exp_variant == 1) exp_finite_lagrange(*L, u_prev1.data(), u_prev2.data(), w.data());
      else exp_finite(*L, u_prev1.data(), u_prev2.data(), w.data());
      double t2 = now_s();
      row[12] = t2 - t1;
      u = w;
      // while ||A u - f|| > eps ||f||: u <= JCG(A, u, f)  (Alg. 4 l.7-9)
      SolveStats st = jcg(*L, u.data(), eps_k[k], maxit_k[k], precond);
      double t3 = now_s();
      row[13] = t3 - t2;
      row[0] = st.iterations; row[1] = st.rel_recur; row[2] = st.rel_true; row[15] = st.status;
      if (st.status != ORC_OK && status == ORC_OK) status = st.status;
      // u~_h = EXP_true(u_h, u_2h)  (Alg. 4 l.10)
      ut.assign(L->N, 0.0);
      exp_true(*L, u.data(), u_prev1.data(), ut.data());
      row[14] = now_s() - t3;
    }
    if (P.has_exact) {
      std::vector<double> ex(L->N), e(L->N);
#pragma omp parallel for schedule(static) num_threads(g_threads) if (g_threads > 1)
      for (long iz = 0; iz < L->nn[2]; ++iz)
        for (long iy = 0; iy < L->nn[1]; ++iy)
          for (long ix = 0; ix < L->nn[0]; ++ix)
            ex[L->idx(ix, iy, iz)] = P.exact(L->coord(0, ix), L->coord(1, iy), L->coord(2, iz));
      for (long i = 0; i < L->N; ++i) e[i] = u[i] - ex[i];
      norms(*L, e.data(), &row[4], &row[5]);
      if (k >= 2) {
        for (long i = 0; i < L->N; ++i) e[i] = ut[i] - ex[i];
        norms(*L, e.data(), &row[6], &row[7]);
      }
    }
    if (k >= 2) {
      std::vector<double> e(L->N);
      for (long i = 0; i < L->N; ++i) e[i] = w[i] - u[i];
      norms(*L, e.data(), &row[8], &row[9]);
      if (P.has_exact) row[10] = row[8] / row[4];  // r_h = ||W-U||_2 / ||U-u||_2
    }
    if (k == num_levels - 1) {
      if (u_fine) std::memcpy(u_fine, u.data(), sizeof(double) * L->N);
      if (ut_fine && k >= 2) std::memcpy(ut_fine, ut.data(), sizeof(double) * L->N);
      if (w_fine && k >= 2) std::memcpy(w_fine, w.data(), sizeof(double) * L->N);
    }
    u_prev2.swap(u_prev1);
    u_prev1.swap(u);
    delete L;
  }
  return status;
}

int orc_ecmg(const double* lo, const double* hi, const int* coarsest, int num_levels, int problem_id,
             const double* params, int nparams, const int* face, double eps, int max_iter, int precond,
             int exp_variant, double* stats, double* u_fine, double* ut_fine, double* w_fine) {
  if (num_levels < 3 || num_levels > 16) return ORC_EINVAL;
  std::vector<double> e(num_levels, eps);
  std::vector<int> m(num_levels, max_iter);
  return ecmg_impl(lo, hi, coarsest, num_levels, problem_id, params, nparams, face, e.data(), m.data(), precond,
                   exp_variant, stats, u_fine, ut_fine, w_fine);
}

// Alg. 3: the original ECMG with a fixed number of iterations per level, Eq. (ee)
// (P:290-295): m_j = ceil(m_L * ratio^(L-j)) on the j-th ECMG level (j = 1..L, L = num_levels - 2;
// reading R4 in DESIGN.md), plain CG by default (precond = 0). Levels 0, 1: DSOLVE.
// Alg. 4 on PROB_ARRAYS data: level_arrays[4 k + {0, 1, 2, 3}] = beta_e, f_q, gD_n, gR_q of level k, and with
// n_level_arrays = 5 L also [4 L + k] = alpha at the face Gauss points of level k
int orc_ecmg_arrays(const double* lo, const double* hi, const int* coarsest, int num_levels, const double* alpha,
                    const int* face, const double* const* level_arrays, int n_level_arrays, double eps, int max_iter,
                    int precond, int exp_variant, double* stats, double* u_fine, double* ut_fine, double* w_fine) {
  if (num_levels < 3 || num_levels > 16 || !level_arrays) return ORC_EINVAL;
  if (n_level_arrays != 4 * num_levels && n_level_arrays != 5 * num_levels) return ORC_EINVAL;
  std::vector<double> e(num_levels, eps);
  std::vector<int> m(num_levels, max_iter);
  return ecmg_impl(lo, hi, coarsest, num_levels, PROB_ARRAYS, alpha, 6, face, e.data(), m.data(), precond,
                   exp_variant, stats, u_fine, ut_fine, w_fine, level_arrays, n_level_arrays);
}

static int ecmg_fixed_impl(const double* lo, const double* hi, const int* coarsest, int num_levels, int problem_id,
                           const double* params, int nparams, const int* face, int m_L, double ratio, int precond,
                           int exp_variant, double* stats, double* u_fine, double* ut_fine, double* w_fine,
                           const double* const* level_arrays, int n_level_arrays) {
  if (num_levels < 3 || num_levels > 16 || m_L < 0 || !(ratio > 0.0)) return ORC_EINVAL;
  const int Lc = num_levels - 2;
  std::vector<double> e(num_levels, 0.0);
  std::vector<int> m(num_levels, 0);
  for (int k = 2; k < num_levels; ++k) {
    const int j = k - 1;   // j-th ECMG level, j = 1..Lc
    m[k] = (int)std::ceil(m_L * std::pow(ratio, (double)(Lc - j)) - 1e-12);
  }
  return ecmg_impl(lo, hi, coarsest, num_levels, problem_id, params, nparams, face, e.data(), m.data(), precond,
                   exp_variant, stats, u_fine, ut_fine, w_fine, level_arrays, n_level_arrays);
}

int orc_ecmg_fixed(const double* lo, const double* hi, const int* coarsest, int num_levels, int problem_id,
                   const double* params, int nparams, const int* face, int m_L, double ratio, int precond,
                   int exp_variant, double* stats, double* u_fine, double* ut_fine, double* w_fine) {
  return ecmg_fixed_impl(lo, hi, coarsest, num_levels, problem_id, params, nparams, face, m_L, ratio, precond,
                         exp_variant, stats, u_fine, ut_fine, w_fine, nullptr, 0);
}

// Alg. 3 on PROB_ARRAYS data (level_arrays, n_level_arrays as in orc_ecmg_arrays)
int orc_ecmg_fixed_arrays(const double* lo, const double* hi, const int* coarsest, int num_levels,
                          const double* alpha, const int* face, const double* const* level_arrays, int n_level_arrays,
                          int m_L, double ratio, int precond, int exp_variant, double* stats, double* u_fine,
                          double* ut_fine, double* w_fine) {
  if (!level_arrays) return ORC_EINVAL;
  if (n_level_arrays != 4 * num_levels && n_level_arrays != 5 * num_levels) return ORC_EINVAL;
  return ecmg_fixed_impl(lo, hi, coarsest, num_levels, PROB_ARRAYS, alpha, 6, face, m_L, ratio, precond,
                         exp_variant, stats, u_fine, ut_fine, w_fine, level_arrays, n_level_arrays);
}

}  // extern "C"
