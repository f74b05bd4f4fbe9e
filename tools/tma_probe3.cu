// tma_probe3.cu -- sweep: ./tma_probe3 rank dtype(4|8) bx by cx cy promo
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void kload(const __grid_constant__ CUtensorMap map, int rank, int cx, int cy, uint32_t bytes, double* out) {
  __shared__ alignas(128) unsigned char sm[40 * 40 * 8];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
    if (rank == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sm)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(cx), "r"(cy), "r"(su32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(su32(sm)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(cx), "r"(cy), "r"(2), "r"(su32(&bar)) : "memory");
  }
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(&bar)), "r"(0) : "memory");
  } while (!done);
  if (threadIdx.x == 0) out[0] = *(double*)sm;
}
int main(int argc, char** argv) {
  int rank = atoi(argv[1]), es = atoi(argv[2]), bx = atoi(argv[3]), by = atoi(argv[4]), cx = atoi(argv[5]), cy = atoi(argv[6]), promo = atoi(argv[7]);
  int n = 64;
  void* d; double* out;
  cudaMalloc(&d, (size_t)8 * n * n * n); cudaMalloc(&out, 8);
  cudaMemset(d, 0, (size_t)8 * n * n * n);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)n * es, (cuuint64_t)n * n * es};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
  cuuint32_t est[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims,
      strides, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
      promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  kload<<<1, 32>>>(map, rank, cx, cy, (uint32_t)(bx * by * es), out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("rank=%d es=%d box=%dx%d c=(%d,%d) promo=%d encode=%d -> %s\n", rank, es, bx, by, cx, cy, promo, (int)r, cudaGetErrorString(e));
  return 0;
}
