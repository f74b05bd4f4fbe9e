// jcg_common.cuh -- device helpers shared by the JCG kernels: deterministic block / grid
// reductions and the device-side CG scalar updates (textbook PCG recurrences).
#pragma once
#include "ecmg_internal.cuh"

namespace ecmg {
namespace {

constexpr int TX = 32;
constexpr int WARPS = 8;
constexpr int NTH = TX * WARPS;

// ---- programmatic dependent launch (sm_90+): a JCG kernel lets the next one in the stream start
// launching as soon as all its CTAs run, and waits for its predecessor's completion (and memory) before
// it reads the CG scalars or any vector. Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- deterministic reductions and the device-side CG scalar updates -----------------------

// ---- the per-node arithmetic of the constant-stencil kernels, with explicit rounding ------------
// (shared by the TMA-fed and the register-prefetch kernels so both produce bitwise-equal iterates)
// p_new = D^-1 r + beta_cg p_old (textbook PCG search direction, O7)
__device__ __forceinline__ double pcg_direction(double dinv, double r, double bcg, double pold, bool first) {
  return first ? dinv * r : __fma_rn(bcg, pold, dinv * r);
}
// per-plane partial sums of the constant 27-point stencil: q0 (plane is the centre plane) and
// q1 (plane is a neighbour plane) from the centre value and the in-plane sums
__device__ __forceinline__ void stencil_q(const ConstStencil& cs, double cc, double ax, double ay, double dd, double& q0,
                                          double& q1) {
  q0 = __fma_rn(cs.cd[0], dd, __fma_rn(cs.cy[0], ay, __fma_rn(cs.cx[0], ax, cs.c0[0] * cc)));
  q1 = __fma_rn(cs.cd[1], dd, __fma_rn(cs.cy[1], ay, __fma_rn(cs.cx[1], ax, cs.c0[1] * cc)));
}

__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* red) {
  const int tid = threadIdx.x + TX * threadIdx.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
  }
  if ((tid & 31) == 0) { red[3 * (tid >> 5)] = a; red[3 * (tid >> 5) + 1] = b; red[3 * (tid >> 5) + 2] = c; }
  __syncthreads();
  if (tid == 0) {
    double sa = 0.0, sb = 0.0, sc = 0.0;
    for (int w = 0; w < NTH / 32; ++w) { sa += red[3 * w]; sb += red[3 * w + 1]; sc += red[3 * w + 2]; }
    a = sa; b = sb; c = sc;
  }
}

__device__ void finalize(int mode, const KArgs& a, double s0, double s1, double s2) {
  JcgScalars* sc = a.sc;
  switch (mode) {
    case MODE_INIT: {
      sc->bb = s2;   // ||b||^2 of the lifted right-hand side (read by this pass anyway)
      sc->rho = s0; sc->rr = s1; sc->alpha = 0.0; sc->beta = 0.0; sc->sigma = 0.0;
      const double eps = sc->in.eps;
      const int max_iter = sc->in.max_iter;
      sc->iter = 0; sc->status = ST_OK; sc->max_iter = max_iter;
      const double nb = sqrt(sc->bb);
      const double nbe = nb > 0.0 ? nb : 1.0;             // ||f|| = 0: absolute residual (§8c A11)
      sc->thresh = eps > 0.0 ? eps * nbe : -1.0;          // eps <= 0: fixed iteration count
      int done = (max_iter <= 0) || (sc->thresh > 0.0 && !(sqrt(s1) > sc->thresh));
      if (!isfinite(s1)) { sc->status = ST_EBREAKDOWN; done = 1; }
      sc->done = done;
      if (a.use_cond) cudaGraphSetConditional(a.cond, done ? 0u : 1u);
      break;
    }
    case MODE_K1: {
      sc->sigma = s0;
      if (!(s0 > 0.0)) {   // p.Ap <= 0
        sc->status = ST_EBREAKDOWN;
        sc->done = 1;
        if (a.use_cond) cudaGraphSetConditional(a.cond, 0u);
      }
      else { sc->alpha_prev = sc->alpha; sc->alpha = sc->rho / s0; }
      break;
    }
    case MODE_K2: {
      const double rho_new = s0;
      sc->beta = rho_new / sc->rho;
      sc->rho = rho_new;
      sc->rr = s1;
      sc->iter += 1;
      int done = (sc->iter >= sc->max_iter) || (sc->thresh > 0.0 && !(sqrt(s1) > sc->thresh));
      if (!isfinite(s1)) { sc->status = ST_EBREAKDOWN; done = 1; }
      sc->done = done;
      if (a.use_cond) cudaGraphSetConditional(a.cond, done ? 0u : 1u);
      break;
    }
    case MODE_TRUE: sc->rr_true = s1; break;
    default: break;
  }
}

__device__ void reduce_finalize(int mode, const KArgs& a, double v0, double v1, double v2 = 0.0) {
  __shared__ double red[3 * (NTH / 32)];
  __shared__ int is_last;
  block_sum3(v0, v1, v2, red);
  const int tid = threadIdx.x + TX * threadIdx.y;
  const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (tid == 0) {
    a.partials[3 * bid] = v0;
    a.partials[3 * bid + 1] = v1;
    a.partials[3 * bid + 2] = v2;
    __threadfence();
    const unsigned prev = atomicAdd(&a.sc->counter, 1u);
    is_last = (prev == nb - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (unsigned b = tid; b < nb; b += NTH) {
    s0 += __ldcg(a.partials + 3 * b);
    s1 += __ldcg(a.partials + 3 * b + 1);
    s2 += __ldcg(a.partials + 3 * b + 2);
  }
  block_sum3(s0, s1, s2, red);
  if (tid == 0) {
    if (a.local_only) {   // z-slab: partial sums of this slab; the allreduce + finalize pass follow
      a.sc->loc[0] = s0; a.sc->loc[1] = s1; a.sc->loc[2] = s2;
    } else {
      finalize(mode, a, s0, s1, s2);
    }
    a.sc->counter = 0;
  }
}

}  // namespace
}  // namespace ecmg
