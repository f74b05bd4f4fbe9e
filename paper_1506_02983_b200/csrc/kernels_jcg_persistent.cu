// kernels_jcg_persistent.cu -- the whole JCG solve of a small constant-stencil level (Alg. 4
// l.7-9) in ONE cooperative launch. The coarse levels of the cascade are latency bound (a few
// microseconds of memory traffic per iteration, dominated by launch and pipeline-fill latency), so
// here every CTA stays resident and the phases of an iteration are separated by grid-wide
// barriers instead of kernel boundaries:
//   p = D^-1 r + beta p (pointwise) | sync | w = A p, sigma partials | sync | alpha |
//   x += alpha p, r -= alpha w, rho', rr partials | sync | beta, stop test
// Reductions are deterministic: every CTA writes its partial sum, and after the barrier every CTA
// sums all partials in CTA order (ping-pong buffers keep a barrier between reuse). The textbook
// PCG recurrences and the stopping rule are those of jcg_common.cuh.
#include <cooperative_groups.h>
#include "ecmg_internal.cuh"
#include "jcg_common.cuh"

namespace cg = cooperative_groups;

namespace ecmg {
namespace {

constexpr int PNTH = 256;

struct PArgs {
  double* x;
  double* r;
  double* p;
  double* w;
  const double* b;
  double* partials;   // 2 x gridDim.x x 3
  JcgScalars* sc;
};

__device__ __forceinline__ double stencil_at(const LevelGeom& g, const ConstStencil& cs, const double* v, int fx, int fy,
                                             int fz) {
  double acc = 0.0;
#pragma unroll
  for (int dz = -1; dz <= 1; ++dz) {
    const int z = fz + dz;
    if (z < 0 || z >= g.nf[2]) continue;
    const int az = dz != 0;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int y = fy + dy;
      if (y < 0 || y >= g.nf[1]) continue;
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int x = fx + dx;
        if (x < 0 || x >= g.nf[0]) continue;
        const double c = (dx == 0) ? (dy == 0 ? cs.c0[az] : cs.cy[az]) : (dy == 0 ? cs.cx[az] : cs.cd[az]);
        acc = __fma_rn(c, v[z * (int)g.S + y * (int)g.P + x], acc);
      }
    }
  }
  return acc;
}

// block reduction of 3 values; the grid-wide sum of all blocks' partials, identical in every CTA
__device__ void grid_sum3(double v[3], double* partials, int buf, double out[3], cg::grid_group& grid) {
  __shared__ double red[3 * (PNTH / 32)];
  __shared__ double res[3];
  const int tid = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  if ((tid & 31) == 0)
    for (int k = 0; k < 3; ++k) red[3 * (tid >> 5) + k] = v[k];
  __syncthreads();
  double* pb = partials + (size_t)buf * gridDim.x * 3;
  if (tid == 0) {
    for (int k = 0; k < 3; ++k) {
      double s = 0.0;
      for (int w = 0; w < PNTH / 32; ++w) s += red[3 * w + k];
      pb[3 * blockIdx.x + k] = s;
    }
  }
  grid.sync();
  if (tid < 3) {
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += __ldcg(pb + 3 * b + tid);   // CTA order
    res[tid] = s;
  }
  __syncthreads();
  out[0] = res[0]; out[1] = res[1]; out[2] = res[2];
  __syncthreads();
}

__global__ void __launch_bounds__(PNTH) k_jcg_persistent(const LevelGeom g, const ConstStencil cs, const PArgs a) {
  cg::grid_group grid = cg::this_grid();
  // small levels only (n < 2^31): 32-bit index math
  const int nx = g.nf[0], nxy = g.nf[0] * g.nf[1];
  const int n = nxy * g.nf[2];
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  const int P = (int)g.P, S = (int)g.S;
  const double dinv = cs.dinv;
  JcgScalars* sc = a.sc;
  const double eps = sc->eps_in;
  const int max_iter = sc->max_iter_in;
  auto off = [&](int i, int& fx, int& fy, int& fz) {
    fz = i / nxy;
    const int rem = i - fz * nxy;
    fy = rem / nx;
    fx = rem - fy * nx;
    return fz * S + fy * P + fx;
  };
  int buf = 0;
  // init: r = b - A x, rho = r.D^-1 r, rr, ||b||^2
  double v[3] = {0.0, 0.0, 0.0}, s3[3];
  for (int i = t0; i < n; i += stride) {
    int fx, fy, fz;
    const int o = off(i, fx, fy, fz);
    const double bi = a.b[o];
    const double rn = bi - stencil_at(g, cs, a.x, fx, fy, fz);
    a.r[o] = rn;
    a.p[o] = 0.0;
    v[0] = __fma_rn(rn, dinv * rn, v[0]);
    v[1] = __fma_rn(rn, rn, v[1]);
    v[2] = __fma_rn(bi, bi, v[2]);
  }
  grid_sum3(v, a.partials, buf, s3, grid);
  buf ^= 1;
  double rho = s3[0], rr = s3[1];
  const double bb = s3[2];
  const double nb = sqrt(bb), nbe = nb > 0.0 ? nb : 1.0;
  const double thresh = eps > 0.0 ? eps * nbe : -1.0;
  int status = ST_OK, iter = 0;
  double beta = 0.0;
  bool done = (max_iter <= 0) || (thresh > 0.0 && !(sqrt(rr) > thresh));
  if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  while (!done) {
    // p = D^-1 r + beta p
    for (int i = t0; i < n; i += stride) {
      int fx, fy, fz;
      const int o = off(i, fx, fy, fz);
      a.p[o] = pcg_direction(dinv, a.r[o], beta, a.p[o], iter == 0);
    }
    grid.sync();
    // w = A p, sigma = p.w
    v[0] = v[1] = v[2] = 0.0;
    for (int i = t0; i < n; i += stride) {
      int fx, fy, fz;
      const int o = off(i, fx, fy, fz);
      const double wi = stencil_at(g, cs, a.p, fx, fy, fz);
      a.w[o] = wi;
      v[0] = __fma_rn(a.p[o], wi, v[0]);
    }
    grid_sum3(v, a.partials, buf, s3, grid);
    buf ^= 1;
    const double sigma = s3[0];
    if (!(sigma > 0.0)) { status = ST_EBREAKDOWN; break; }
    const double alpha = rho / sigma;
    // x += alpha p, r -= alpha w, rho' = r.D^-1 r, rr = r.r
    v[0] = v[1] = v[2] = 0.0;
    for (int i = t0; i < n; i += stride) {
      int fx, fy, fz;
      const int o = off(i, fx, fy, fz);
      a.x[o] = __fma_rn(alpha, a.p[o], a.x[o]);
      const double rn = __fma_rn(-alpha, a.w[o], a.r[o]);
      a.r[o] = rn;
      v[0] = __fma_rn(rn, dinv * rn, v[0]);
      v[1] = __fma_rn(rn, rn, v[1]);
    }
    grid_sum3(v, a.partials, buf, s3, grid);
    buf ^= 1;
    beta = s3[0] / rho;
    rho = s3[0];
    rr = s3[1];
    ++iter;
    done = (iter >= max_iter) || (thresh > 0.0 && !(sqrt(rr) > thresh));
    if (!isfinite(rr)) { status = ST_EBREAKDOWN; done = true; }
  }
  // true residual
  v[0] = v[1] = v[2] = 0.0;
  for (int i = t0; i < n; i += stride) {
    int fx, fy, fz;
    const int o = off(i, fx, fy, fz);
    const double rn = a.b[o] - stencil_at(g, cs, a.x, fx, fy, fz);
    v[1] = __fma_rn(rn, rn, v[1]);
  }
  grid_sum3(v, a.partials, buf, s3, grid);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->rho = rho; sc->rr = rr; sc->bb = bb; sc->rr_true = s3[1]; sc->beta = beta;
    sc->iter = iter; sc->max_iter = max_iter; sc->thresh = thresh; sc->status = status; sc->done = 1;
  }
}

}  // namespace

// grid size for the cooperative launch (all CTAs co-resident), at most `want`
int persistent_grid(int want) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jcg_persistent, PNTH, 0);
  return std::max(1, std::min(want, sms * std::max(1, per_sm)));
}

cudaError_t launch_jcg_persistent(const LevelGeom& g, const ConstStencil& cs, double* x, double* r, double* p, double* w,
                                  const double* b, double* partials, JcgScalars* sc, cudaStream_t st) {
  const long long n = (long long)g.nf[0] * g.nf[1] * g.nf[2];
  const int want = (int)std::min<long long>((n + PNTH - 1) / PNTH, 1 << 20);
  const int grid = persistent_grid(want);
  PArgs a{x, r, p, w, b, partials, sc};
  void* args[] = {(void*)&g, (void*)&cs, (void*)&a};
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)k_jcg_persistent, dim3(grid), dim3(PNTH), args, 0, st);
}

}  // namespace ecmg
