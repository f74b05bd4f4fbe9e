// tma_probe.cu -- standalone probe of the TMA / mbarrier sequence used by kernels_jcg_tma.cu.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_probe tools/tma_probe.cu
// ./tma_probe <variant>: 0 = box 34x34x1 on a 15x15x15 tensor (like the 16^3 level)
//                       1 = box 34x34x1 on a 63x63x63 tensor
//                       2 = variant 0 without fence.mbarrier_init
//                       3 = box 32x32x1 on 63^3, interior box, 4 loads in flight
#include <cuda.h>
#include <cuda/barrier>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, double* out, int bx, int by, int x0, int y0, int z0,
                      int use_fence) {
  extern __shared__ __align__(128) unsigned char raw[];
  __shared__ __align__(8) uint64_t bar;
  unsigned char* sm = (unsigned char*)(((uintptr_t)raw + 127) & ~uintptr_t(127));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
    if (use_fence) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t bytes = bx * by * 8;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            su32(sm)),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(x0), "r"(y0), "r"(z0), "r"(su32(&bar))
        : "memory");
  }
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(su32(&bar)), "r"(0)
                 : "memory");
  } while (!done);
  const double* d = reinterpret_cast<const double*>(sm);
  for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = d[i];
}

using lbarrier = cuda::barrier<cuda::thread_scope_block>;
namespace cde = cuda::device::experimental;

// the CUDA programming guide's TMA pattern via libcu++
__global__ void probe_lib(const __grid_constant__ CUtensorMap map, double* out, int bx, int by) {
  __shared__ alignas(128) double sm[34 * 34];
#pragma nv_diag_suppress static_var_with_dynamic_init
  __shared__ lbarrier bar;
  if (threadIdx.x == 0) {
    init(&bar, blockDim.x);
    cde::fence_proxy_async_shared_cta();
  }
  __syncthreads();
  lbarrier::arrival_token token;
  if (threadIdx.x == 0) {
    cde::cp_async_bulk_tensor_3d_global_to_shared(sm, &map, -1, -1, 2, bar);
    token = cuda::device::barrier_arrive_tx(bar, 1, sizeof(double) * bx * by);
  } else {
    token = bar.arrive();
  }
  bar.wait(std::move(token));
  for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  int n = (variant == 0 || variant == 2) ? 15 : 63;
  int bx = variant == 3 ? 32 : 34, by = bx;
  long long P = (n + 31) / 32 * 32, S = P * n;
  std::vector<double> h(S * n);
  for (long long k = 0; k < n; ++k)
    for (long long j = 0; j < n; ++j)
      for (long long i = 0; i < n; ++i) h[k * S + j * P + i] = 1000000.0 * k + 1000.0 * j + i;
  double *d, *out;
  cudaMalloc(&d, sizeof(double) * h.size());
  cudaMalloc(&out, sizeof(double) * bx * by);
  cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)P * 8, (cuuint64_t)S * 8};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUtensorMapDataType dt = (variant == 5) ? CU_TENSOR_MAP_DATA_TYPE_INT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  CUresult r = encode(&map, dt, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("variant %d encode=%d\n", variant, (int)r);
  int smem = bx * by * 8 + 128;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (variant == 4) probe_lib<<<1, 128>>>(map, out, bx, by);
  else probe<<<1, 128, smem>>>(map, out, bx, by, -1, -1, 2, variant == 2 ? 0 : 1);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d kernel: %s\n", variant, cudaGetErrorString(e));
  if (e == cudaSuccess) {
    std::vector<double> o(bx * by);
    cudaMemcpy(o.data(), out, sizeof(double) * o.size(), cudaMemcpyDeviceToHost);
    printf("out[0]=%g out[1]=%g out[%d]=%g out[%d]=%g\n", o[0], o[1], bx + 1, o[bx + 1], bx + 2, o[bx + 2]);
  }
  return 0;
}
