// kernels_jcg_tma.cu -- TMA-fed z-marching JCG kernels for the constant-coefficient stencil
// (beta constant, all faces Dirichlet: C1, C2, C4). Same arithmetic and the
// same device-side CG scalar recurrences as kernels_jcg.cu (Alg. 4 l.7-9).
//
// Data movement (B200-native): every z-plane of every input vector reaches shared memory through
// ONE cp.async.bulk.tensor.3d per CTA (box 34 x 34 for halo-read vectors, 32 x 32 for interior
// vectors), issued by one thread into an NS-deep ring of stages and completed on an mbarrier
// (expect_tx). Out-of-bounds boxes are zero-filled by the TMA unit, which is exactly "p = 0 on
// Dirichlet nodes" of the eliminated system, so the kernel has no boundary predication on loads.
// Stage k holds halo plane zl and interior plane zl-1 (the plane whose A.p completes in that step).
// The refill of a stage is issued one step after it was consumed, right after the per-plane
// __syncthreads, so no separate "empty" barrier is needed.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cooperative_groups.h>
#include <type_traits>
#include <algorithm>
#include "ecmg_internal.cuh"
#include "jcg_common.cuh"

namespace ecmg {
namespace {

constexpr int RY = 4;             // rows per warp
constexpr int TY = WARPS * RY;    // 32
// The innermost TMA box start must be 16-byte aligned (x = -1 traps with an illegal instruction
// on sm_100a, measured: tools/tma_probe3.cu), so the halo box starts at x = X0 - 2 and is 36 wide;
// columns 0 and 35 are loaded but unused.
constexpr int HX = TX + 4;        // 36 (x = X0-2 .. X0+33)
constexpr int XO = 2;             // smem column of x = X0
constexpr int HY = TY + 2;        // 34
constexpr int HBYTES = HX * HY * 8;            // 9792
constexpr int HSTRIDE = (HBYTES + 127) / 128 * 128;   // 9856
constexpr int IBYTES = TX * TY * 8;            // 8192

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// interior boxes per stage: K2 x, r (xdefer 0) | r (1) | x, r, p_{k-1} (2); INIT / TRUE b
template <int MODE, int XD>
__host__ __device__ constexpr int num_interior() {
  return MODE == MODE_K2 ? (XD == 1 ? 1 : (XD == 2 ? 3 : 2)) : ((MODE == MODE_INIT || MODE == MODE_TRUE) ? 1 : 0);
}

// loads of step t (halo plane z0-1+t, interior plane z0-2+t) into stage st
template <bool kH1, int kNI, int SBYTES>
__device__ __forceinline__ void issue_stage(unsigned char* smem, uint64_t* full, int st, int t, int z0, int X0, int Y0,
                                            uint32_t tx_bytes, bool first, const CUtensorMap* pH0, const CUtensorMap* pH1,
                                            const CUtensorMap* pI0, const CUtensorMap* pI1, const CUtensorMap* pI2,
                                            int skip_int = -1) {   // interior box not loaded (K2 of iteration 0, KArgs::p0)
  unsigned char* base = smem + st * SBYTES;
  mbar_expect_tx(&full[st], tx_bytes);
  const int zh = z0 - 1 + t;
  tma_load_3d(base, pH0, X0 - XO, Y0 - 1, zh, &full[st]);
  if (kH1 && !first) tma_load_3d(base + HSTRIDE, pH1, X0 - XO, Y0 - 1, zh, &full[st]);
  if (kNI >= 1 && skip_int != 0) tma_load_3d(base + HSTRIDE * (kH1 ? 2 : 1), pI0, X0, Y0, zh - 1, &full[st]);
  if (kNI >= 2 && skip_int != 1) tma_load_3d(base + HSTRIDE * (kH1 ? 2 : 1) + IBYTES, pI1, X0, Y0, zh - 1, &full[st]);
  if (kNI >= 3) tma_load_3d(base + HSTRIDE * (kH1 ? 2 : 1) + 2 * IBYTES, pI2, X0, Y0, zh - 1, &full[st]);
}

// One z-march of the CTA over its (tile, z chunk) in mode MODE: the per-plane TMA pipeline of the kernels
// below, with the stage ring continuing at the running step count gstep (stage (gstep + s) % NS, parity
// ((gstep + s) / NS) & 1), so that a persistent CTA can run several passes over the same mbarriers.
// Returns the thread's partial sums in acc0..acc2. The caller has initialised the mbarriers and
// synchronised the CTA since its previous pass.
// XD: deferred x update of K2 (KArgs::xdefer); alpha0 = alpha_{k-1} for XD = 2
template <int MODE, int NS, int SBYTES, int XD = 0>
__device__ __forceinline__ void tma_pass(const LevelGeom& g, const ConstStencil& cs, const KArgs& a, int X0, int Y0, int z0,
                                         int z1, double bcg, bool first, double alpha, double* u_out,
                                         const CUtensorMap* pH0, const CUtensorMap* pH1, const CUtensorMap* pI0,
                                         const CUtensorMap* pI1, unsigned char* smem, uint64_t* full, uint32_t gstep,
                                         double& acc0, double& acc1, double& acc2, const CUtensorMap* pI2 = nullptr,
                                         double alpha0 = 0.0, const double* rich_u2h = nullptr, double* rich_ut = nullptr) {
  constexpr bool kH1 = (MODE == MODE_K1);
  // MODE_TRUE with XD = 3: the true-residual pass also forms u~_h = EXP_true(u_h, u_2h) (Alg. 4 l.10) at its own
  // nodes, from the x planes it holds anyway (see the step loop); rich_ut == nullptr: plain true-residual pass
  constexpr bool kRich = (MODE == MODE_TRUE && XD == 3);
  const bool rich = kRich && rich_ut != nullptr;
  constexpr int kNI = num_interior<MODE, XD>();
  const int lane = threadIdx.x, w = threadIdx.y, tid = lane + TX * w;
  const int nfx = g.nf[0], nfy = g.nf[1];
  const long long P = g.P, S = g.S;
  const int x = X0 + lane, yb = Y0 + RY * w;
  const int nsteps = z1 - z0 + 2;
  const double dinv = cs.dinv;
  // KArgs::p0, iteration 0 (`first`): K1 reads p_0 as stored by the init pass (pH0 is its map: no transform, no
  // store); K2 forms r_0 = diag p_0 and does not load r (interior box XD == 1 ? 0 : 1)
  const bool p0k1 = MODE == MODE_K1 && first && a.p0, p0k2 = MODE == MODE_K2 && first && a.p0;
  const int skip_int = p0k2 ? (XD == 1 ? 0 : 1) : -1;
  const uint32_t tx_bytes = HBYTES + ((kH1 && !first) ? HBYTES : 0) + IBYTES * kNI - (p0k2 ? IBYTES : 0);
  auto stage_ptr = [&](int st) { return smem + st * SBYTES; };
  if (tid == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic accesses before async-proxy writes
    for (int t = 0; t < NS - 1 && t < nsteps; ++t)
      issue_stage<kH1, kNI, SBYTES>(smem, full, (gstep + t) % NS, t, z0, X0, Y0, tx_bytes, first, pH0, pH1, pI0, pI1, pI2, skip_int);
  }

  // halo ring slot of this thread (transform in place, K1 only): rows y = Y0-1, Y0+32 (x = X0-1 ..
  // X0+32, smem columns 1..34) and columns x = X0-1, X0+32 (smem columns 1, 34) of rows Y0..Y0+31
  constexpr int RW = TX + 2;   // 34
  int rhx = -1, rhy = -1;
  if (tid < 2 * RW) { rhx = 1 + tid % RW; rhy = (tid < RW) ? 0 : HY - 1; }
  else if (tid < 2 * RW + 2 * TY) { const int t = tid - 2 * RW; rhx = (t < TY) ? 1 : RW; rhy = 1 + (t % TY); }

  bool own_ok[RY];
  long long own_off[RY];
#pragma unroll
  for (int j = 0; j < RY; ++j) {
    own_ok[j] = (x < nfx) && (yb + j < nfy);
    own_off[j] = own_ok[j] ? (long long)(yb + j) * P + x : 0;
  }
  double part[RY], q1p[RY], pp[RY];
#pragma unroll
  for (int j = 0; j < RY; ++j) { part[j] = q1p[j] = pp[j] = 0.0; }
  // EXP_true inside the true-residual pass (kRich). u~ = u_h + (1/3) I(d), d = u_h - u_2h at the 2h nodes and I the
  // trilinear interpolation (A13; k_exp_true evaluates the same expression, means along x, then y, then
  // z, so the two agree bit for bit). ea / eb: I_xy(d) at the thread's nodes on the last two even (2h) node planes.
  // Nodes outside the free box are Dirichlet nodes, where u_h = u_2h = g_D and d = 0.
  double ea[RY], eb[RY];
#pragma unroll
  for (int j = 0; j < RY; ++j) { ea[j] = eb[j] = 0.0; }
  const int gx = g.flo[0] + x, gy0 = g.flo[1] + yb;   // global node indices of the thread's column / first row
  const int xodd = gx & 1;
  const long long nx2 = g.n[0] / 2 + 1, pl2 = nx2 * (g.n[1] / 2 + 1);
  const bool fxl = x - xodd >= 0 && x - xodd < nfx, fxr = x + xodd >= 0 && x + xodd < nfx;   // 2h columns in the free box
  // u_2h at the 2h nodes the thread needs on the NEXT 2h plane, fetched one 2h plane (two steps) ahead so that no
  // step waits for these loads: rows rp, rp + 2, rp + 4 of the window (rp = parity of its first row: CTA-uniform),
  // left / right 2h column; 0 outside the free box, where the x planes hold 0 as well (TMA zero fill), so d = 0
  double u2n[3][2];
  const int rp = (gy0 - 1) & 1;
  auto fetch_u2 = [&](int zn) {   // for the arriving plane zn (local free index)
    const bool zf = kRich && rich && g.zoff + zn >= 0 && g.zoff + zn < g.nf[2] && zn <= z1;
    const double* u2p = zf ? rich_u2h + (long long)((g.flo[2] + g.zoff + zn) >> 1) * pl2 : nullptr;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int r = rp + 2 * i, fy = yb - 1 + r;
      const bool rf = zf && r < RY + 2 && fy >= 0 && fy < nfy;
      const double* u2r = rf ? u2p + (long long)((gy0 - 1 + r) >> 1) * nx2 : nullptr;
      u2n[i][0] = (rf && fxl) ? __ldg(u2r + ((gx - xodd) >> 1)) : 0.0;
      u2n[i][1] = (rf && fxr) ? __ldg(u2r + ((gx + xodd) >> 1)) : 0.0;
    }
  };
  if (kRich && rich) fetch_u2(z0 - 1 + ((g.flo[2] + g.zoff + z0 - 1) & 1));   // the first 2h plane of the march

  for (int s = 0; s < nsteps; ++s) {
    const int zl = z0 - 1 + s;
    const int st = (gstep + s) % NS;
    if (s > 0) __syncthreads();   // every thread is done with step s-1: its stage may be refilled
    if (tid == 0 && s + NS - 1 < nsteps) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes before async-proxy writes
      const int t = s + NS - 1;                                      // into stage (s-1) % NS
      issue_stage<kH1, kNI, SBYTES>(smem, full, (gstep + t) % NS, t, z0, X0, Y0, tx_bytes, first, pH0, pH1, pI0, pI1, pI2, skip_int);
    }
    mbar_wait(&full[st], (uint32_t)(((gstep + s) / NS) & 1));
    double* H = reinterpret_cast<double*>(stage_ptr(st));
    if (MODE == MODE_K1) {
      const double* H1 = reinterpret_cast<const double*>(stage_ptr(st) + HSTRIDE);
      const bool halo_store = (zl == g.zbeg - 1 || zl == g.zend) && zl >= 0 && zl < g.nza;
      if (!p0k1) {   // (uniform)
#pragma unroll
        for (int j = 0; j < RY; ++j) {
          const int o = (1 + RY * w + j) * HX + XO + lane;
          H[o] = pcg_direction(dinv, H[o], bcg, H1[o], first);
          if (halo_store && own_ok[j]) a.o0[(long long)zl * S + own_off[j]] = H[o];   // slab halo plane of p
        }
        if (rhx >= 0) {
          const int o = rhy * HX + rhx;
          H[o] = pcg_direction(dinv, H[o], bcg, H1[o], first);
        }
        __syncthreads();
      }
    }
    double col[RY + 2][3];
#pragma unroll
    for (int r = 0; r < RY + 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) col[r][c] = H[(RY * w + r) * HX + XO - 1 + lane + c];
    const double* I0 = reinterpret_cast<const double*>(stage_ptr(st) + HSTRIDE * (kH1 ? 2 : 1));
    const double* I1 = I0 + TX * TY;
    const int z = zl - 1;
    if (kRich && rich && !((g.flo[2] + g.zoff + zl) & 1)) {   // (CTA-uniform) a 2h node plane arrives
      auto plane = [&](auto rp_tag) {
        constexpr int RP = decltype(rp_tag)::value;
        double xi[3];   // I_x(d) on the window's 2h rows RP, RP + 2, RP + 4
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int r = RP + 2 * i;
          if (r >= RY + 2) { xi[i] = 0.0; continue; }
          const double dl = (xodd ? col[r][0] : col[r][1]) - u2n[i][0];
          const double dr = (xodd ? col[r][2] : col[r][1]) - u2n[i][1];
          xi[i] = 0.5 * dl + 0.5 * dr;
        }
#pragma unroll
        for (int j = 0; j < RY; ++j) {   // node row j = window row j + 1: a 2h row iff (j + 1 - RP) is even
          ea[j] = eb[j];
          eb[j] = ((j + 1 - RP) & 1) ? 0.5 * xi[(j - RP) / 2] + 0.5 * xi[(j - RP) / 2 + 1] : xi[(j + 1 - RP) / 2];
        }
      };
      if (rp) plane(std::integral_constant<int, 1>{}); else plane(std::integral_constant<int, 0>{});
      fetch_u2(zl + 2);
    }
#pragma unroll
    for (int j = 0; j < RY; ++j) {
      const double cc = col[j + 1][1];
      const double ax = col[j + 1][0] + col[j + 1][2];
      const double ay = col[j][1] + col[j + 2][1];
      const double dd = (col[j][0] + col[j][2]) + (col[j + 2][0] + col[j + 2][2]);
      double q0, q1;
      stencil_q(cs, cc, ax, ay, dd, q0, q1);
      if (s >= 2 && own_ok[j]) {
        const double ap = part[j] + q1;
        const long long off = (long long)z * S + own_off[j];
        const int io = (RY * w + j) * TX + lane;
        if (MODE == MODE_K1) {
          acc0 = __fma_rn(pp[j], ap, acc0);
          if (!p0k1) a.o0[off] = pp[j];
        } else if (MODE == MODE_K2) {
          // interior boxes: XD 0 (x, r), 1 (r), 2 (x, r, p_{k-1})
          const double rn = __fma_rn(-alpha, ap, p0k2 ? cs.diag * pp[j] : (XD == 1 ? I0[io] : I1[io]));
          const double zz = dinv * rn;
          acc0 = __fma_rn(rn, zz, acc0);
          acc1 = __fma_rn(rn, rn, acc1);
          if (XD == 0) a.o0[off] = __fma_rn(alpha, pp[j], I0[io]);
          if (XD == 2) a.o0[off] = __fma_rn(alpha, pp[j], __fma_rn(alpha0, I1[TX * TY + io], I0[io]));
          a.o1[off] = rn;
          if (z == g.zbeg && a.peer_lo) a.peer_lo[own_off[j]] = rn;      // fused halo exchange
          if (z == g.zend - 1 && a.peer_hi) a.peer_hi[own_off[j]] = rn;
        } else if (MODE == MODE_INIT) {
          acc2 = __fma_rn(I0[io], I0[io], acc2);
          const double rn = I0[io] - ap;
          const double zz = dinv * rn;
          acc0 = __fma_rn(rn, zz, acc0);
          acc1 = __fma_rn(rn, rn, acc1);
          a.o0[off] = a.p0 ? zz : rn;   // (p0: o0 is the first K1's output vector and receives p_0 = D^-1 r_0)
          if (z == g.zbeg && a.peer_lo) a.peer_lo[own_off[j]] = rn;      // fused halo exchange
          if (z == g.zend - 1 && a.peer_hi) a.peer_hi[own_off[j]] = rn;
        } else if (MODE == MODE_TRUE) {
          const double rn = I0[io] - ap;
          acc1 = __fma_rn(rn, rn, acc1);
          if (u_out) u_out[full_index(g, x, yb + j, z)] = pp[j];   // fused scatter of u_h
          if (kRich && rich) {   // plane z between two 2h planes: the mean of their I_xy(d); on a 2h plane: its own
            const double e = ((g.flo[2] + g.zoff + z) & 1) ? 0.5 * (ea[j] + eb[j]) : eb[j];
            rich_ut[full_index(g, x, yb + j, z)] = __fma_rn(e, 1.0 / 3.0, pp[j]);
          }
        } else {
          a.o0[off] = ap;
        }
      }
      part[j] = q1p[j] + q0;
      q1p[j] = q1;
      pp[j] = cc;
    }
  }
}

template <int MODE, int NS, int XD>
__global__ void __launch_bounds__(NTH, 2)
    k_jcg_const_tma(const LevelGeom g, const ConstStencil cs, const KArgs a, const __grid_constant__ CUtensorMap mH0,
                    const __grid_constant__ CUtensorMap mH1, const __grid_constant__ CUtensorMap mI0,
                    const __grid_constant__ CUtensorMap mI1, const __grid_constant__ CUtensorMap mI2) {
  constexpr bool kH1 = (MODE == MODE_K1);
  constexpr int kNI = num_interior<MODE, XD>();
  constexpr int SBYTES = HSTRIDE * (kH1 ? 2 : 1) + IBYTES * kNI;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[NS];
  // TMA destinations must be 128-byte aligned in the shared window: align the stage base explicitly
  // (offset from smem_raw, not a uintptr_t round trip: the pointer must stay in the shared window so
  // the reads compile to LDS, not generic LD)
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  JcgScalars* sc = a.sc;
  pdl_trigger();
  pdl_wait();
  if (MODE == MODE_K1 || MODE == MODE_K2) {
    if (*(volatile int*)&sc->done) return;
  }
  const int tid = threadIdx.x + TX * threadIdx.y;
  const int X0 = blockIdx.x * TX, Y0 = blockIdx.y * TY;
  const int z0 = g.zbeg + blockIdx.z * a.zc;
  const int z1 = min(z0 + a.zc, g.zend);
  double bcg = 0.0, alpha = 0.0, alpha0 = 0.0;
  bool first = false;
  if (MODE == MODE_K1) { bcg = sc->beta; first = (sc->iter == 0); }
  if (MODE == MODE_K2) { alpha = sc->alpha; alpha0 = XD == 2 ? sc->alpha_prev : 0.0; first = a.p0 && sc->iter == 0; }
  double* const u_out = (MODE == MODE_TRUE) ? sc->in.u_out : nullptr;
  double* const rich_ut = (MODE == MODE_TRUE && XD == 3) ? sc->in.ut_out : nullptr;
  const double* const rich_u2h = (MODE == MODE_TRUE && XD == 3) ? sc->in.u2h : nullptr;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  // XD = 1 (K2 without x): the one interior box is r (I1)
  // (p0, the first K1: the halo map of its own output vector, which holds p_0, rides in the I0 slot)
  tma_pass<MODE, NS, SBYTES, XD>(g, cs, a, X0, Y0, z0, z1, bcg, first, alpha, u_out,
                                 (MODE == MODE_K1 && first && a.p0) ? &mI0 : &mH0, &mH1, XD == 1 ? &mI1 : &mI0, &mI1,
                                 smem, full, 0u, acc0, acc1, acc2, &mI2, alpha0, rich_u2h, rich_ut);
  if ((MODE == MODE_K2 || MODE == MODE_INIT) && (a.peer_lo || a.peer_hi)) __threadfence_system();   // peer stores
  if (MODE != MODE_APPLY) reduce_finalize(MODE, a, acc0, acc1, acc2);
}

// ---- the whole JCG solve of a level in ONE cooperative launch, TMA z-marching passes -------------
// (mid-size levels, e.g. 128^3: a launched K1/K2 pair costs ~36 us there, mostly launch, pipeline fill
// and tail, against ~20 us of traffic). Each CTA owns a fixed list of (tile, z chunk) items and runs
// init -> { K1 pass, grid sum, K2 pass, grid sum } -> true residual; the grid sums are deterministic
// (per-CTA partials, grid barrier, every CTA reduces all partials in CTA order), so every CTA holds the
// same CG scalars and takes the same stop decision. Same per-node arithmetic as the kernels above.
constexpr int PS_NS = 3;
constexpr int PS_SBYTES = HSTRIDE + 2 * IBYTES;   // the largest stage (K2: p halo + x, r interior)
static_assert(PS_SBYTES >= 2 * HSTRIDE, "K1 stage (r and p_old halo boxes) must fit");

struct PersMaps { CUtensorMap xh, rh, ph0, ph1, xi, ri, bi; };

__device__ __forceinline__ void pers_grid_sum3(double v[3], double* partials, int& buf, double* red,
                                               cooperative_groups::grid_group& grid) {
  block_sum3(v[0], v[1], v[2], red);   // thread 0 holds the CTA sums
  const int tid = threadIdx.x + TX * threadIdx.y;
  double* pb = partials + (size_t)buf * gridDim.x * 3;
  if (tid == 0)
    for (int k = 0; k < 3; ++k) pb[3 * blockIdx.x + k] = v[k];
  grid.sync();
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (unsigned c = tid; c < gridDim.x; c += NTH) {
    s0 += __ldcg(pb + 3 * c);
    s1 += __ldcg(pb + 3 * c + 1);
    s2 += __ldcg(pb + 3 * c + 2);
  }
  block_sum3(s0, s1, s2, red);
  __shared__ double bc[3];
  if (tid == 0) { bc[0] = s0; bc[1] = s1; bc[2] = s2; }
  __syncthreads();
  v[0] = bc[0]; v[1] = bc[1]; v[2] = bc[2];
  __syncthreads();
  buf ^= 1;
}

__global__ void __launch_bounds__(NTH, 2)
    k_jcg_const_pers(const LevelGeom g, const ConstStencil cs, double* x, double* r, double* p0, double* p1, double* partials,
                     JcgScalars* sc, int zc, int ntx, int nty, int items, int p0_init, const __grid_constant__ PersMaps M) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[PS_NS];
  __shared__ double red[3 * (NTH / 32)];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int tid = threadIdx.x + TX * threadIdx.y;
  if (tid == 0) {
    for (int i = 0; i < PS_NS; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double eps = sc->in.eps;
  const int max_iter = sc->in.max_iter;
  double* const u_out = sc->in.u_out;
  uint32_t gstep = 0;
  int buf = 0;
  KArgs a{};
  a.p0 = p0_init;   // p_0 from the init pass (KArgs::p0), as on the launched kernels
  // one pass of MODE over this CTA's items
  auto pass = [&](auto mode_tag, const CUtensorMap* h0, const CUtensorMap* h1, const CUtensorMap* i0, const CUtensorMap* i1,
                  double bcg, bool first, double alpha, double v[3]) {
    constexpr int MODE = decltype(mode_tag)::value;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      const int X0 = (it % ntx) * TX, Y0 = ((it / ntx) % nty) * TY;
      const int z0 = (it / (ntx * nty)) * zc, z1 = min(z0 + zc, g.zend);
      tma_pass<MODE, PS_NS, PS_SBYTES>(g, cs, a, X0, Y0, z0, z1, bcg, first, alpha, u_out, h0, h1, i0, i1, smem, full,
                                       gstep, acc0, acc1, acc2);
      gstep += (uint32_t)(z1 - z0 + 2);
      __syncthreads();   // every stage consumed before the next pass's prefill
    }
    // this pass's global stores are read by other CTAs' TMA (async proxy) in the next pass
    asm volatile("fence.proxy.async.global;" ::: "memory");
    v[0] = acc0; v[1] = acc1; v[2] = acc2;
    pers_grid_sum3(v, partials, buf, red, grid);
    if (tid == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
  };
  // init: r = b - A x, rho = r.z, rr, ||b||^2
  double v[3];
  a.o0 = a.p0 ? p1 : r;   // (p0: p_0 = D^-1 r_0 goes to the first K1's output vector)
  pass(std::integral_constant<int, MODE_INIT>{}, &M.xh, &M.xh, &M.bi, &M.bi, 0.0, false, 0.0, v);
  double rho = v[0], rr = v[1];
  const double bb = v[2];
  const double nb = sqrt(bb), nbe = nb > 0.0 ? nb : 1.0;
  const double thresh = eps > 0.0 ? eps * nbe : -1.0;
  int status = ST_OK, iter = 0;
  double beta = 0.0;
  bool done = (max_iter <= 0) || (thresh > 0.0 && !(sqrt(rr) > thresh));
  if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  int cur = 0;   // p_cur holds p_old
  while (!done) {
    double* pnew = cur ? p0 : p1;
    a.o0 = pnew;
    // (p0, iteration 0: the halo vector is p_0 itself, in the output vector p1)
    pass(std::integral_constant<int, MODE_K1>{}, (a.p0 && iter == 0) ? &M.ph1 : &M.rh, cur ? &M.ph1 : &M.ph0, &M.rh, &M.rh,
         beta, iter == 0, 0.0, v);
    const double sigma = v[0];
    if (!(sigma > 0.0)) { status = ST_EBREAKDOWN; break; }
    const double alpha = rho / sigma;
    a.o0 = x; a.o1 = r;
    pass(std::integral_constant<int, MODE_K2>{}, cur ? &M.ph0 : &M.ph1, &M.rh, &M.xi, &M.ri, 0.0, iter == 0, alpha, v);
    beta = v[0] / rho;
    rho = v[0];
    rr = v[1];
    cur ^= 1;
    ++iter;
    done = (iter >= max_iter) || (thresh > 0.0 && !(sqrt(rr) > thresh));
    if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  }
  // true residual ||b - A x|| and the fused scatter of u_h
  pass(std::integral_constant<int, MODE_TRUE>{}, &M.xh, &M.xh, &M.bi, &M.bi, 0.0, false, 0.0, v);
  if (blockIdx.x == 0 && tid == 0) {
    sc->rho = rho; sc->rr = rr; sc->bb = bb; sc->rr_true = v[1]; sc->beta = beta;
    sc->iter = iter; sc->max_iter = max_iter; sc->thresh = thresh; sc->status = status; sc->done = 1;
    sc->counter = 0;
  }
}

template <int MODE, int NS, int XD = 0>
cudaError_t launch_tma_mode(dim3 grid, dim3 block, const LevelGeom& g, const ConstStencil& cs, const KArgs& a,
                            const CUtensorMap* maps, cudaStream_t st) {
  constexpr bool kH1 = (MODE == MODE_K1);
  constexpr int SBYTES = HSTRIDE * (kH1 ? 2 : 1) + IBYTES * num_interior<MODE, XD>();
  constexpr int SMEM = SBYTES * NS + 128;
  count_launch();
  return launch_maybe_pdl(k_jcg_const_tma<MODE, NS, XD>, grid, block, SMEM, st, a.pdl, g, cs, a, maps[0], maps[1], maps[2],
                          maps[3], maps[4]);
}

template <int MODE, int NS, int XD = 0>
cudaError_t set_tma_attr() {
  constexpr bool kH1 = (MODE == MODE_K1);
  constexpr int SMEM = (HSTRIDE * (kH1 ? 2 : 1) + IBYTES * num_interior<MODE, XD>()) * NS + 128;
  return cudaFuncSetAttribute(k_jcg_const_tma<MODE, NS, XD>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
}

}  // namespace

#ifndef NS_K2_SKIP   // ring depth of the x-less K2 (p halo + r interior per stage, the K1 stage size)
#define NS_K2_SKIP 4
#endif

// set every dynamic-smem attribute up front (never inside a stream capture)
cudaError_t init_tma_kernel_attributes() {
  cudaError_t e = set_tma_attr<MODE_K1, 4>();
  if (e == cudaSuccess) e = set_tma_attr<MODE_K2, 3>();
  if (e == cudaSuccess) e = set_tma_attr<MODE_K2, NS_K2_SKIP, 1>();
  if (e == cudaSuccess) e = set_tma_attr<MODE_K2, 3, 2>();
  if (e == cudaSuccess) e = set_tma_attr<MODE_INIT, 4>();
  if (e == cudaSuccess) e = set_tma_attr<MODE_TRUE, 4>();
  if (e == cudaSuccess) e = set_tma_attr<MODE_TRUE, 4, 3>();
  if (e == cudaSuccess) e = set_tma_attr<MODE_APPLY, 4>();
  return e;
}

// maps[0..4] = H0, H1, I0, I1, I2 tensor maps (unused entries may be any valid map)
cudaError_t launch_jcg_const_tma(int mode, const LevelGeom& g, const ConstStencil& cs, const KArgs& a,
                                 const CUtensorMap* maps, cudaStream_t st) {
  dim3 block(TX, WARPS);
  dim3 grid((g.nf[0] + TX - 1) / TX, (g.nf[1] + TY - 1) / TY, (g.zend - g.zbeg + a.zc - 1) / a.zc);
  switch (mode) {
    case MODE_K1: return launch_tma_mode<MODE_K1, 4>(grid, block, g, cs, a, maps, st);
    case MODE_K2:
      if (a.xdefer == 1) return launch_tma_mode<MODE_K2, NS_K2_SKIP, 1>(grid, block, g, cs, a, maps, st);
      if (a.xdefer == 2) return launch_tma_mode<MODE_K2, 3, 2>(grid, block, g, cs, a, maps, st);
      return launch_tma_mode<MODE_K2, 3>(grid, block, g, cs, a, maps, st);
    case MODE_INIT: return launch_tma_mode<MODE_INIT, 4>(grid, block, g, cs, a, maps, st);
    case MODE_TRUE:
      if (a.rich) return launch_tma_mode<MODE_TRUE, 4, 3>(grid, block, g, cs, a, maps, st);   // + EXP_true (JcgParams::ut_out)
      return launch_tma_mode<MODE_TRUE, 4>(grid, block, g, cs, a, maps, st);
    case MODE_APPLY: return launch_tma_mode<MODE_APPLY, 4>(grid, block, g, cs, a, maps, st);
    default: return cudaErrorInvalidValue;
  }
}

// Tensor map of a free-box work vector: dims (nf_x, nf_y, nf_z), strides (P, S) doubles,
// box (bx, by, 1), zero fill out of bounds.
int make_vec_tensor_map(CUtensorMap* map, const double* base, const LevelGeom& g, int bx, int by) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return -1;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[3] = {(cuuint64_t)g.nf[0], (cuuint64_t)g.nf[1], (cuuint64_t)g.nza};
  cuuint64_t strides[2] = {(cuuint64_t)g.P * 8, (cuuint64_t)g.S * 8};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, ECMG_TMA_PROMO,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

// grid of the persistent TMA solve: at most the co-resident CTAs (2 per SM); z chunks sized so that the
// (tile, chunk) items come to about one per CTA
static int pers_slots() {
  static int slots = 0;
  if (!slots) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jcg_const_pers, NTH, PS_SBYTES * PS_NS + 128);
    slots = sms * std::max(1, per_sm);
  }
  return slots;
}

int const_pers_slots() { return pers_slots(); }

bool const_pers_fits(const LevelGeom& g) {
  const long long tiles = (long long)((g.nf[0] + TX - 1) / TX) * ((g.nf[1] + TY - 1) / TY);
  return g.zbeg == 0 && tiles <= pers_slots();
}

cudaError_t init_pers_kernel_attributes() {
  return cudaFuncSetAttribute(k_jcg_const_pers, cudaFuncAttributeMaxDynamicSharedMemorySize, PS_SBYTES * PS_NS + 128);
}

// maps: x halo, r halo, p0 halo, p1 halo, x interior, r interior, b interior (make_vec_tensor_map)
cudaError_t launch_jcg_const_pers(const LevelGeom& g, const ConstStencil& cs, double* x, double* r, double* p0, double* p1,
                                  double* partials, JcgScalars* sc, const CUtensorMap* maps, cudaStream_t st, int p0_init) {
  const int ntx = (g.nf[0] + TX - 1) / TX, nty = (g.nf[1] + TY - 1) / TY;
  const int nz = g.zend - g.zbeg;
  const int slots = pers_slots();
  const long long tiles = (long long)ntx * nty;
  if (tiles > slots || g.zbeg != 0) return cudaErrorInvalidValue;
  const int nch = (int)std::max(1LL, slots / tiles);          // z chunks per tile
#ifndef PERS_MIN_ZC
// planes per (tile, chunk) item, at least. Round 2 first ran 4 (the 64^3 level on 64 CTAs instead of 252, 0.66 ->
// 0.89 ms) to leave SMs to the finest level's ALU-bound right-hand side running ahead beside the coarse solves;
// with the permutation-symmetric C4 load (k_rhs_c4_sym, 0.69 instead of 1.55 ms) the finest level no longer waits
// for its setup and 1 measures faster again (tools/tts_ab.py, 2 x 15 runs: TTS 14.63 -> 14.39 ms with 2 z chunks
// per load tile; profiles/r02/tuning/ab_rhs_sym_variants.log)
#define PERS_MIN_ZC 1
#endif
  const int zc = std::max(PERS_MIN_ZC, (nz + nch - 1) / nch);
  const int items = (int)(tiles * ((nz + zc - 1) / zc));
  PersMaps M{maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6]};
  int grid = std::min(items, slots);
  void* args[] = {(void*)&g, (void*)&cs, (void*)&x, (void*)&r, (void*)&p0, (void*)&p1, (void*)&partials, (void*)&sc,
                  (void*)&zc, (void*)&ntx, (void*)&nty, (void*)&items, (void*)&p0_init, (void*)&M};
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)k_jcg_const_pers, dim3(grid), dim3(TX, WARPS), args,
                                     PS_SBYTES * PS_NS + 128, st);
}

int tma_halo_box_x() { return HX; }
int tma_halo_box_y() { return HY; }
int tma_int_box_x() { return TX; }
int tma_int_box_y() { return TY; }

}  // namespace ecmg
