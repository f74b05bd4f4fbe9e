// ecmg_internal.cuh -- internal types of libecmg (B200 / sm_100a). Not part of the ABI.
//
// Data layout in HBM:
//  * Caller-visible nodal vectors: contiguous (nx+1)(ny+1)(nz+1) fp64, x fastest.
//  * JCG work vectors x, r, p, b live on the FREE BOX only. Dirichlet is imposed per face, so the
//    free nodes of a level are the box [flo, flo+nf) per axis (flo = 1 if the face is Dirichlet,
//    nf = n+1 minus the Dirichlet faces). Row pitch P = nf_x rounded up to 32 doubles (256 B
//    rows), plane stride S = P * nf_y. Nodes outside the box are never stored: loads outside it
//    return 0, which is exactly "p = 0 on Dirichlet nodes" of the eliminated system (§8c A5).
//  * Element coefficients beta_e (element-beta path) on the global element grid with a zero
//    ring of width 2: element (ex,ey,ez), -2 <= e <= n+1, at beta[(ez+2)*BS + (ey+2)*BP + ex+2].
//    beta_e = 0 outside the domain, which truncates the stencil at Robin / Neumann faces.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

namespace ecmg {

constexpr int kMaxParams = 48;

enum Face { XM = 0, XP = 1, YM = 2, YP = 3, ZM = 4, ZP = 5 };
enum { FACE_DIRICHLET = 0, FACE_ROBIN = 1 };

// Problem registry entry passed by value to kernels (device-side evaluation of Eq. (bvp) data).
struct Problem {
  int id;
  int face[6];
  double alpha[6];        // Robin alpha per face (0 = Neumann)
  double params[kMaxParams];
  int n_params;
  // PROB_ARRAYS: the caller's device arrays of ONE level (beta_e, f at the Gauss points, g_D per node, g_R and
  // alpha at the face Gauss points; layouts in include/ecmg.h), set per launch by the host (level_prob);
  // null = 0 / 1 (alpha: null = alpha[F] per face)
  const double* arr[5];
};
constexpr int PROB_ARRAYS = 100;

struct LevelGeom {
  int n[3];          // cells per axis
  double lo[3], h[3];
  int flo[3];        // free box origin (global node index)
  int nf[3];         // free box extent (nodes)
  long long P, S;    // free-box vector row pitch / plane stride (doubles)
  long long BP, BS;  // element-beta row pitch / plane stride (doubles), zero ring of 2
  int elem_path;     // 1: element-beta stencil (variable beta or Robin faces); 0: constant stencil
  // z-slab decomposition (one GPU: zoff = 0, zbeg = 0, zend = nza = nf[2], zlo = 0, zhi = n[2] + 1)
  int zoff;          // global free-z index of local work-vector plane 0
  int zbeg, zend;    // local work-vector planes this rank computes, [zbeg, zend)
  int nza;           // allocated local work-vector planes (owned + halo planes)
  int zlo, zhi;      // global node planes [zlo, zhi) this rank owns in full-layout nodal vectors
};

// Constant-coefficient 27-point stencil (beta constant, all faces Dirichlet):
// (A p)_i = sum_{oz} [c0[|oz|] p + cx[|oz|] (p_{x-1}+p_{x+1}) + cy[|oz|] (p_{y-1}+p_{y+1})
//                    + cd[|oz|] (4 in-plane diagonals)] over the planes z+oz, oz in {-1,0,1}.
// Derived from A = beta (K_x (x) M_y (x) M_z + M_x (x) K_y (x) M_z + M_x (x) M_y (x) K_z) with the
// 1D stiffness K_d = [-1,2,-1]/h_d and mass M_d = h_d [1/6,2/3,1/6] (exact Q1 integrals).
struct ConstStencil {
  double c0[2], cx[2], cy[2], cd[2];
  double dinv;   // 1 / diag (Jacobi), or 1 for plain CG
  double diag;   // diag (Jacobi), or 1: r_0 = diag p_0 where only p_0 = D^-1 r_0 is stored (KArgs::p0)
};

// Element stencil: K_ref[a][b] = kappa[pattern(a,b)], pattern = bit d set if a, b differ along d.
// kappa[pat] = V sum_d (1/h_d^2) k(pat_d) prod_{e != d} m(pat_e), k(same)=1, k(diff)=-1,
// m(same)=1/3, m(diff)=1/6. Robin face mass on face F: alpha h1 h2 m2[pat2], m2 = {1/9,1/18,1/18,1/36}.
struct ElemStencil {
  double kappa[8];
  double robin[6];     // alpha_F * h1 * h2 for Robin faces with alpha != 0, else 0
  int precond;         // 1 = Jacobi, 0 = plain CG (dinv = 1)
  int cube;            // h_x = h_y = h_z: kappa = c{4,0,0,-1,0,-1,-1,-1} (the element kernel's short form)
  // beta on the fly (analytic beta, BETA_KIND_*): the element kernels form beta_e from per-axis tables in
  // registers instead of reading the beta array (8 B per unknown less in each of K1 and K2). bkind < 0:
  // read the array. baxes: the tables of the level (beta_axes_* below), written by launch_beta.
  int bkind;
  int bw;              // table row width W = max_d n_d + 4
  const double* baxes;
  // PROB_ARRAYS with alpha at the face Gauss points: the level's alpha_q array (include/ecmg.h layout); then
  // robin[F] = h1 h2 marks the Robin faces and the face mass is formed per face element (robin_elem_row)
  const double* aq;
};

// ---- Robin face mass with alpha at the 2x2 face Gauss points (Eq. bvp's piecewise smooth alpha) -------
// first value of face F's block of alpha_q (blocks x-, x+, y-, y+, z-, z+ of 4 n_d1 n_d2 values, d1 < d2 the in-face
// axes) and of its face element (e1, e2)
__host__ __device__ inline const double* robin_aq(const double* aq, const int n[3], int F, int e1, int e2) {
  long long off = 0;
  for (int f = 0; f < F; ++f) {
    const int d = f >> 1, a1 = d == 0 ? 1 : 0, a2 = d == 2 ? 1 : 2;
    off += 4LL * n[a1] * n[a2];
  }
  const int d = F >> 1, a1 = d == 0 ? 1 : 0;
  return aq + off + 4LL * (e1 + (long long)n[a1] * e2);
}
// 1D linear shape value of local node c (0 / 1) at Gauss point q (0: xi = -1/sqrt3, 1: +1/sqrt3)
__host__ __device__ inline double robin_n(int c, int q) {
  const double ga = 0.21132486540518711775, gb = 0.78867513459481288225;   // (1 -+ 1/sqrt3) / 2
  return c == q ? gb : ga;
}
// face element of area hh with alpha a4[q] (q = q1 + 2 q2) at its Gauss points: the mass row of local corner
// (c1, c2) against nodal values v0..v3 (index c1' + 2 c2') added to acc, its diagonal entry to dg:
// M[c][d] = hh / 4 sum_q a_q N_c(q) N_d(q), evaluated as hh / 4 sum_q a_q N_c(q) v(q)
__host__ __device__ inline void robin_elem_row(const double* a4, int c1, int c2, double v0, double v1, double v2, double v3,
                                                double hh, double& acc, double& dg) {
  double s = 0.0, d = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int q1 = q & 1, q2 = q >> 1;
    const double n10 = robin_n(0, q1), n11 = robin_n(1, q1), n20 = robin_n(0, q2), n21 = robin_n(1, q2);
    const double vq = n20 * (n10 * v0 + n11 * v1) + n21 * (n10 * v2 + n11 * v3);
    const double nc = robin_n(c1, q1) * robin_n(c2, q2);
    const double a = a4[q];
    s += a * nc * vq;
    d += a * nc * nc;
  }
  acc += 0.25 * hh * s;
  dg += 0.25 * hh * d;
}
// one entry M[c][j] of that face element (the lifting against a Dirichlet node j of the same face element)
__host__ __device__ inline double robin_elem_entry(const double* a4, int c1, int c2, int j1, int j2, double hh) {
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int q1 = q & 1, q2 = q >> 1;
    s += a4[q] * (robin_n(c1, q1) * robin_n(c2, q2)) * (robin_n(j1, q1) * robin_n(j2, q2));
  }
  return 0.25 * hh * s;
}

// Analytic beta at element centroids (Eq. bvp, reading A3) from per-axis tables, so that the beta array
// (k_beta) and the element kernels' on-the-fly values are the same function of the same table entries:
//   kind 0 (beta = 1): valid ? 1 : 0
//   kind 1 (C3: 1 + 1/2 sin 2pi x cos 2pi y sin 2pi z): valid ? fma(Ax Ay, Az, 1) : 0, Ax = sin(2pi x)/2, Ay = cos, Az = sin
//   kind 2 (layers in z): valid ? Az : 0, Az = layer beta at the centroid's z
//   kind 3 (C5: layers + 4 boxes, a later box overriding an earlier one): the highest box whose x, y and z
//          ranges all contain the centroid, else the layer value
// Tables at baxes: A[3][W] doubles, then M[3][W] ints (bit 4: the element exists, bits 0-3: inside box k
// along that axis), then the 4 box betas; entry (d, e) for element index e in [-2, n_d + 1] at e + 2.
enum { BETA_KIND_ONE = 0, BETA_KIND_C3 = 1, BETA_KIND_LAYERS = 2, BETA_KIND_C5 = 3 };
__host__ __device__ inline long long beta_axes_doubles(int W) { return 3LL * W + (3LL * W + 1) / 2 + 4 + 1; }
__device__ __forceinline__ double beta_combine(int kind, double ax, double ay, double az, int mx, int my, int mz,
                                               const double* boxb) {
  const int m = mx & my & mz;
  if (!(m & 16)) return 0.0;
  switch (kind) {
    case BETA_KIND_C3: return __fma_rn(ax * ay, az, 1.0);
    case BETA_KIND_LAYERS: return az;
    case BETA_KIND_C5: {
      const int bits = m & 15;
      return bits ? boxb[31 - __clz(bits)] : az;
    }
    default: return 1.0;
  }
}

// Per-solve inputs, written by one host-to-device copy before the init pass (pinned host copy).
struct JcgParams {
  double eps;        // requested eps (<= 0: exactly max_iter iterations)
  double* u_out;     // single GPU: full-layout nodal vector whose free nodes the true-residual pass
                     // fills with the solution (fused scatter); nullptr: no write
  int max_iter;      // requested max_iter
  int pad_;
  // the finest level's true-residual pass in its EXP_true form (KArgs::rich): u~_h = EXP_true(u_h, u_2h) is written
  // to the free nodes of ut_out (full layout) from u2h = the 2h level's solution (full layout); nullptr: not formed
  double* ut_out;
  const double* u2h;
};

// Device-resident CG scalars (no host round trip inside the iteration).
struct JcgScalars {
  double rho;        // r.z
  double rr;         // r.r
  double alpha, beta, sigma;
  double bb;         // ||b||^2 (set by the RHS kernel)
  double rr_true;    // ||b - A x||^2 (set by the true-residual pass)
  double thresh;     // eps * ||b|| (or eps if ||b|| = 0); <= 0: fixed-iteration mode
  JcgParams in;      // eps, max_iter, u_out of the current solve (written by the host before the init pass)
  int iter, max_iter, done, status;
  unsigned int counter;   // last-block-done counter (reset by the last block)
  int pad_;
  double loc[3];     // z-slabs: this slab's partial dot products (before the allreduce)
  double glob[3];    // z-slabs: allreduced dot products (input of the finalize pass)
  double alpha_prev; // alpha of the previous iteration (deferred x update, KArgs::xdefer)
};

enum KMode { MODE_K1 = 1, MODE_K2 = 2, MODE_INIT = 3, MODE_TRUE = 4, MODE_APPLY = 5 };

// index of free node (fx, fy, local plane fz) in the caller-visible full-layout vector (single GPU)
__host__ __device__ inline long long full_index(const LevelGeom& g, int fx, int fy, int fz) {
  const long long nx = g.n[0] + 1, ny = g.n[1] + 1;
  return (long long)(g.flo[2] + g.zoff + fz) * nx * ny + (long long)(g.flo[1] + fy) * nx + (g.flo[0] + fx);
}

struct KArgs {
  const double* h0;   // halo-read vector (K1: r (element path: z), K2: p, INIT/TRUE: x, APPLY: p)
  const double* h1;   // K1: p_old
  const double* i0;   // interior-read vector (K2: x, INIT/TRUE: b)
  const double* i1;   // K2: r
  double* o0;         // K1: p_new, K2: x, INIT: r, APPLY: q
  double* o1;         // K2: r; element path INIT: z = D^-1 r
  double* o2;         // element path K2: z = D^-1 r
  const double* beta; // element path: beta_e with zero ring
  double* partials;   // per-block partial dot products (2 per block)
  JcgScalars* sc;
  int zc;             // planes per CTA
  cudaGraphConditionalHandle cond;   // CUDA-graph WHILE condition (device-driven JCG loop)
  int use_cond;                      // 1: the init / K2 passes set `cond` = !done
  int local_only;                    // z-slabs: write this slab's sums to sc->loc, finalize later
  int pdl;                           // launch with programmatic stream serialization (ECMG_OPT_PDL)
  // z-slabs, fused halo exchange (K2 and init passes): the neighbours' halo planes of the vector the
  // next K1 reads (r, or z on the element path): peer_lo receives this slab's first owned plane (it is
  // the lower neighbour's upper halo plane), peer_hi its last. Same (P, S) layout on every slab; a
  // device pointer of another slab on this GPU (virtual slabs) or a CUDA-IPC mapping of the
  // neighbour rank's buffer over NVLink. nullptr: no fused store (halo by copy / NCCL).
  double* peer_lo;
  double* peer_hi;
  // deferred solution update (K2 of the TMA kernels): 0 = x += alpha_k p_k every
  // iteration; 1 = skip (even k: x is neither read nor written); 2 = combine (odd k: x += alpha_{k-1} p_{k-1}
  // + alpha_k p_k with p_{k-1} = i2, the same two roundings as two single updates, so the iterates are
  // bitwise those of xdefer = 0)
  int xdefer;
  // p0 (constant-stencil TMA kernels, one GPU): the init pass stores p_0 = D^-1 r_0 (into the first K1's output
  // vector) instead of r_0; the first K1 reads it (no transform, no store) and the first K2 forms r_0 = D p_0
  // instead of reading r: 16 B per unknown less in iteration 0
  int p0;
  int rich;           // TRUE (constant-stencil TMA kernel): the variant that also forms EXP_true (JcgParams::ut_out)
  const double* i2;   // K2, xdefer = 2: p_{k-1} (interior box)
};

// launch kernel<<<grid, block, smem, st>>>(args...), with programmatic dependent launch if pdl
template <typename... KArgsT, typename... Act>
inline cudaError_t launch_maybe_pdl(void (*kernel)(KArgsT...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int pdl,
                                    Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

// status codes (mirror of ecmg_status)
enum { ST_OK = 0, ST_EINVAL = -1, ST_ENOMEM = -2, ST_ENOTCONV = -3, ST_EBREAKDOWN = -4, ST_EDIAG = -5,
       ST_EMISMATCH = -6, ST_ECUDA = -7, ST_ENCCL = -8 };

// ---- launchers (kernels_*.cu) -------------------------------------------------------------
// Every launcher bumps this process-wide counter once per kernel launch (ecmg_kernel_launches).
void count_launch(int n = 1);
cudaError_t launch_jcg_const(int mode, const LevelGeom& g, const ConstStencil& cs, const KArgs& a,
                             cudaStream_t st);
cudaError_t launch_jcg_elem(int mode, const LevelGeom& g, const ElemStencil& es, const Problem& pb,
                            const KArgs& a, cudaStream_t st);
int jcg_num_blocks(const LevelGeom& g, int elem_path, int zc);
}  // namespace ecmg
#include <cuda.h>
// L2 promotion of the TMA loads (tuning macro): none measured 0.7 % faster than 256 B on the C4 JCG
// iteration (1.460 vs 1.471 ms at 512^3, tools/build_full_variants.sh + tools/tune_elem.py), equal on C3
#ifndef ECMG_TMA_PROMO
#define ECMG_TMA_PROMO CU_TENSOR_MAP_L2_PROMOTION_NONE
#endif
namespace ecmg {
cudaError_t launch_jcg_const_tma(int mode, const LevelGeom& g, const ConstStencil& cs, const KArgs& a,
                                 const CUtensorMap* maps, cudaStream_t st);
int make_vec_tensor_map(CUtensorMap* map, const double* base, const LevelGeom& g, int bx, int by);
cudaError_t init_pers_kernel_attributes();
// the unfused textbook PCG sequence (ablation, kernels_textbook.cu): step 0 dot(y, x) -> partials,
// 1 finish(arg = op), 2 y += arg * alpha x, 3 y = arg * x, 4 y(p) = x(z) + beta p (arg = first)
long long textbook_partials(const LevelGeom& g);
cudaError_t launch_textbook(int step, const LevelGeom& g, double* y, const double* x, double* partials, JcgScalars* sc,
                            double arg, cudaStream_t st);
cudaError_t init_elem_pers_attributes();
cudaError_t launch_jcg_elem_pers(const LevelGeom& g, const ElemStencil& es, double* x, double* r, double* z, double* p0,
                                 double* p1, const double* b, const double* beta, double* partials, JcgScalars* sc,
                                 cudaStream_t st);
cudaError_t launch_jcg_const_pers(const LevelGeom& g, const ConstStencil& cs, double* x, double* r, double* p0, double* p1,
                                  double* partials, JcgScalars* sc, const CUtensorMap* maps, cudaStream_t st, int p0_init);
// z-slabs: finalize pass after the allreduce, and the in-order sum of P slabs' partial dots
// (virtual slabs on one GPU; NCCL's allreduce on real ranks)
cudaError_t launch_finalize(int mode, const KArgs& a, cudaStream_t st);
cudaError_t launch_empty_solve(JcgScalars* sc, cudaStream_t st);
cudaError_t launch_xfix(const LevelGeom& g, double* x, const double* p, const JcgScalars* sc, cudaStream_t st);
struct SlabScalars { JcgScalars* p[16]; int n; };
cudaError_t launch_vsum(const SlabScalars& s, cudaStream_t st);
cudaError_t launch_jcg_persistent(const LevelGeom& g, const ConstStencil& cs, const ElemStencil* es, double* x, double* r,
                                  double* z, double* p0, double* p1, double* w, double* dinv, const double* beta,
                                  const double* b, double* partials, JcgScalars* sc, cudaStream_t st);
long long persistent_max_bricks(int elem_path);
// co-resident CTAs of the cooperative TMA solves, and the partial-sum doubles every cooperative solve needs
// (6 per CTA of the largest grid + 64); call after the init_*_attributes
int const_pers_slots();
int elem_pers_slots_count();
long long coop_partials_doubles();
bool const_pers_fits(const LevelGeom& g);   // the cooperative TMA solves take this level's shape
bool elem_pers_fits(const LevelGeom& g);
bool cta_solve_fits(const LevelGeom& g, int elem_path, long long max_nodes);
cudaError_t init_cta_kernel_attributes();
cudaError_t launch_jcg_cta(const LevelGeom& g, const ConstStencil& cs, const ElemStencil* es, double* x, double* r,
                           const double* beta, const double* b, JcgScalars* sc, cudaStream_t st);
cudaError_t init_tma_kernel_attributes();
cudaError_t init_elem_kernel_attributes();
int elem_tile_rows();
cudaError_t init_setup_kernel_attributes();
int tma_halo_box_x();
int tma_halo_box_y();
int tma_int_box_x();
int tma_int_box_y();

cudaError_t launch_beta(const LevelGeom& g, const Problem& pb, double* beta, cudaStream_t st);
cudaError_t launch_rhs(const LevelGeom& g, const Problem& pb, const ElemStencil& es, double beta_const,
                       const double* beta, double* b, double* scratch, cudaStream_t st, int ctas_per_sm = 0,
                       int sym_min = 248);
cudaError_t launch_gather(const LevelGeom& g, const double* u, double* x, cudaStream_t st);
cudaError_t launch_scatter(const LevelGeom& g, const double* x, double* u, cudaStream_t st);
cudaError_t launch_dirichlet_fill(const LevelGeom& g, const Problem& pb, double* u, double value_if_none,
                                  int zero_instead, cudaStream_t st);
cudaError_t launch_exp_finite(const LevelGeom& gf, const Problem& pb, const double* u2h, const double* u4h,
                              double* w, int variant, double* seeds, int freebox, cudaStream_t st, int fused = 1);
cudaError_t launch_exp_true(const LevelGeom& gf, const Problem& pb, const double* uh, const double* u2h,
                            double* ut, cudaStream_t st);
cudaError_t launch_zero_vec(const LevelGeom& g, double* v, cudaStream_t st);

// Device workspace allocation. The product build is cudaMalloc / cudaFree; the test build (libecmg_test.so,
// -DECMG_TESTING, defined in ecmg_api.cu) surrounds every buffer with guard bands of a fixed byte pattern and
// checks them on free and on request (ecmg_test_guard_check), the out-of-bounds-write check that stands in for
// compute-sanitizer memcheck (closed on this GPU pool).
cudaError_t dev_malloc(void** p, size_t bytes);
void dev_free(void* p);
template <class T>
cudaError_t dmalloc(T** p, size_t bytes) { return dev_malloc(reinterpret_cast<void**>(p), bytes); }
inline void dfree(void* p) { dev_free(p); }

}  // namespace ecmg
