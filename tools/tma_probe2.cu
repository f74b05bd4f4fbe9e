// tma_probe2.cu -- canonical 2D float32 TMA load, descriptor encoded (a) via the runtime entry point,
// (b) via libcuda's cuTensorMapEncodeTiled linked directly.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k2d(const __grid_constant__ CUtensorMap map, float* out) {
  __shared__ alignas(128) float sm[32 * 32];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(sm)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(0), "r"(su32(&bar)) : "memory");
  }
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(&bar)), "r"(0) : "memory");
  } while (!done);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
  int how = argc > 1 ? atoi(argv[1]) : 0;
  std::vector<float> h(64 * 64);
  for (int i = 0; i < 64 * 64; ++i) h[i] = (float)i;
  float *d, *out;
  cudaMalloc(&d, 4 * h.size()); cudaMalloc(&out, 4 * 1024);
  cudaMemcpy(d, h.data(), 4 * h.size(), cudaMemcpyHostToDevice);
  CUtensorMap map;
  cuuint64_t dims[2] = {64, 64};
  cuuint64_t strides[1] = {64 * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r;
  if (how == 0) {
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
    r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  printf("how %d encode=%d\n", how, (int)r);
  k2d<<<1, 128>>>(map, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("how %d kernel: %s\n", how, cudaGetErrorString(e));
  if (e == cudaSuccess) { std::vector<float> o(1024); cudaMemcpy(o.data(), out, 4096, cudaMemcpyDeviceToHost); printf("o[0]=%g o[33]=%g o[1023]=%g\n", o[0], o[33], o[1023]); }
  return 0;
}
