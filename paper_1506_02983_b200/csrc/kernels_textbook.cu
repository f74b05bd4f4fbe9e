// kernels_textbook.cu -- the unfused textbook PCG sequence (Alg. 4 l.7-9) as the
// ablation of the fused K1 / K2 kernels ("store the ncu profile of the unfused textbook
// sequence; it is the ablation showing the fusion gain"). One iteration is nine passes over the free box:
//   w = A p (the TMA stencil kernel in MODE_APPLY) | sigma = p.w | x += alpha p | r -= alpha w |
//   z = D^-1 r | rho' = r.z | rr = r.r | p = z + beta p
// each its own launch reading and writing HBM: 144 B per unknown and iteration against the fused 64 B.
// The scalars stay on the device (alpha, beta, rho in JcgScalars); dot products reduce deterministically
// (per-block partials in block order, then one block). Constant-stencil levels, fixed iteration counts.
#include "ecmg_internal.cuh"

namespace ecmg {
namespace {

constexpr int TB = 256;

// one thread per free node of a (row, plane): grid (ceil(nf_x / TB), nf_y, planes)
__device__ __forceinline__ bool tb_node(const LevelGeom& g, long long* off) {
  const int fx = blockIdx.x * TB + threadIdx.x;
  if (fx >= g.nf[0]) return false;
  *off = (long long)(g.zbeg + blockIdx.z) * g.S + (long long)blockIdx.y * g.P + fx;
  return true;
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[TB / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < TB / 32; ++w) s += red[w];
  return s;   // thread 0
}

__global__ void k_tb_dot(const LevelGeom g, const double* __restrict__ a, const double* __restrict__ b,
                         double* __restrict__ partials) {
  long long o;
  double v = 0.0;
  if (tb_node(g, &o)) v = a[o] * b[o];
  const double s = block_sum(v);
  if (threadIdx.x == 0) partials[blockIdx.x + gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z)] = s;
}

// op 0: sigma = sum -> alpha = rho / sigma; 1: rho' = sum -> beta = rho' / rho, rho = rho'; 2: rr = sum, iter++
__global__ void k_tb_finish(const double* __restrict__ partials, long long n, JcgScalars* sc, int op) {
  double v = 0.0;
  for (long long i = threadIdx.x; i < n; i += TB) v += partials[i];
  const double s = block_sum(v);
  if (threadIdx.x != 0) return;
  if (op == 0) { sc->sigma = s; sc->alpha = sc->rho / s; }
  else if (op == 1) { sc->beta = s / sc->rho; sc->rho = s; }
  else { sc->rr = s; sc->iter += 1; }
}

// y += sign * alpha * x
__global__ void k_tb_axpy(const LevelGeom g, double* __restrict__ y, const double* __restrict__ x, const JcgScalars* sc,
                          double sign) {
  long long o;
  if (!tb_node(g, &o)) return;
  y[o] = __fma_rn(sign * sc->alpha, x[o], y[o]);
}

__global__ void k_tb_scale(const LevelGeom g, double* __restrict__ z, const double* __restrict__ r, double dinv) {
  long long o;
  if (!tb_node(g, &o)) return;
  z[o] = dinv * r[o];
}

// p = z + beta p (first: p = z)
__global__ void k_tb_pupdate(const LevelGeom g, double* __restrict__ p, const double* __restrict__ z, const JcgScalars* sc,
                             int first) {
  long long o;
  if (!tb_node(g, &o)) return;
  p[o] = first ? z[o] : __fma_rn(sc->beta, p[o], z[o]);
}

}  // namespace

long long textbook_partials(const LevelGeom& g) {
  return (long long)((g.nf[0] + TB - 1) / TB) * g.nf[1] * (g.zend - g.zbeg);
}

cudaError_t launch_textbook(int step, const LevelGeom& g, double* y, const double* x, double* partials, JcgScalars* sc,
                            double arg, cudaStream_t st) {
  const dim3 grid((g.nf[0] + TB - 1) / TB, g.nf[1], g.zend - g.zbeg);
  count_launch();
  switch (step) {
    case 0: k_tb_dot<<<grid, TB, 0, st>>>(g, y, x, partials); break;
    case 1: k_tb_finish<<<1, TB, 0, st>>>(partials, textbook_partials(g), sc, (int)arg); break;
    case 2: k_tb_axpy<<<grid, TB, 0, st>>>(g, y, x, sc, arg); break;
    case 3: k_tb_scale<<<grid, TB, 0, st>>>(g, y, x, arg); break;
    case 4: k_tb_pupdate<<<grid, TB, 0, st>>>(g, y, x, sc, (int)arg); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace ecmg
