// gridsync_probe.cu -- cost of a grid-wide barrier on this GPU: cooperative_groups grid.sync() vs a
// sense-reversing atomic barrier (one arrive per CTA, spin with ld.acquire), for G CTAs of 256 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync_probe tools/gridsync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int n, double* out) {
  cg::grid_group grid = cg::this_grid();
  double v = threadIdx.x;
  for (int i = 0; i < n; ++i) { v = v * 1.0000001 + 1.0; grid.sync(); }
  if (v == -1.0) out[0] = v;
}

__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;
__device__ __forceinline__ void bar(unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int want = gen + 1;
    if (atomicAdd(&g_count, 1u) == nblocks - 1) {
      g_count = 0;
      __threadfence();
      atomicExch((unsigned int*)&g_gen, want);
    } else {
      unsigned int cur;
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(&g_gen)); } while (cur != want);
    }
  }
  gen += 1;
  __syncthreads();
}
__global__ void k_atomic(int n, double* out) {
  unsigned int gen = g_gen;
  double v = threadIdx.x;
  for (int i = 0; i < n; ++i) { v = v * 1.0000001 + 1.0; bar(gridDim.x, gen); }
  if (v == -1.0) out[0] = v;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int G : {1, 8, 16, 32, 64, 148, 296}) {
    int n = 2000;
    void* args[] = {&n, &out};
    float t1 = 0, t2 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, G, 256, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t1, a, b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_atomic, G, 256, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t2, a, b);
    }
    printf("G=%4d  cg grid.sync %.3f us   atomic barrier %.3f us   (%s)\n", G, t1 * 1e3 / n, t2 * 1e3 / n,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
