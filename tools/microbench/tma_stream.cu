// Microbenchmark: raw TMA streaming of a [rows][128] bf16 array through
// shared memory (no compute), the memory side of the tree-attention kernel.
// Each CTA streams contiguous 128-row blocks of K and V (2 x 32 KB per stage)
// with `stages` stages; the consumer releases a stage as soon as it lands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu -lcuda
//   ./tma_stream [stages] [ctas_per_sm]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
               : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int x, int y, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su32(dst)), "l"((uint64_t)m), "r"(x), "r"(y), "r"(su32(b)) : "memory");
}

__global__ void stream_kernel(const __grid_constant__ CUtensorMap km, const __grid_constant__ CUtensorMap vm,
                              int blocks_per_cta, int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * 65536);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int y0 = blockIdx.x * blocks_per_cta * 128;
  unsigned long long acc = 0;
  for (int j = 0; j < blocks_per_cta + stages; ++j) {
    if (j >= stages) {  // consume block j - stages
      const int jc = j - stages, st = jc % stages;
      while (!try_wait(&full[st], (jc / stages) & 1)) {
      }
      acc += sm[st * 65536];
    }
    if (j < blocks_per_cta) {
      const int st = j % stages;
      uint8_t* d = sm + st * 65536;
      expect_tx(&full[st], 65536);
      tma2d(d, &km, 0, y0 + j * 128, &full[st]);
      tma2d(d + 16384, &km, 64, y0 + j * 128, &full[st]);
      tma2d(d + 32768, &vm, 0, y0 + j * 128, &full[st]);
      tma2d(d + 49152, &vm, 64, y0 + j * 128, &full[st]);
    }
  }
  if (acc == 12345) *sink = acc;
}

int main(int argc, char** argv) {
  const int stages = argc > 1 ? atoi(argv[1]) : 3;
  const int per_sm = argc > 2 ? atoi(argv[2]) : 1;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int ctas = nsm * per_sm, bpc = 57 / per_sm;
  const size_t rows = (size_t)ctas * bpc * 128;
  void *k, *v;
  cudaMalloc(&k, rows * 256);
  cudaMalloc(&v, rows * 256);
  cudaMemset(k, 1, rows * 256);
  cudaMemset(v, 1, rows * 256);
  void* flush;
  cudaMalloc(&flush, 256 << 20);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap km, vm;
  cuuint64_t dims[2] = {128, rows};
  cuuint64_t str[1] = {256};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&km, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&vm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, v, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = stages * 65536 + 1024;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int it = 0; it < 10; ++it) {
    cudaMemsetAsync(flush, it, 256 << 20);
    cudaEventRecord(a);
    stream_kernel<<<ctas, 32, smem>>>(km, vm, bpc, stages, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it >= 2 && ms < best) best = ms;
  }
  const double bytes = 2.0 * rows * 256;
  printf("stages %d ctas/SM %d: %.1f MB in %.4f ms = %.0f GB/s (%s)\n", stages, per_sm, bytes / 1e6, best,
         bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
