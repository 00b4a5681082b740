// Cost model of tcgen05.mma kind::i8 (M=128, K=32, SWIZZLE_NONE K-major) issue streams.
//   knobs: dalt = alternate the TMEM accumulator per step; avary = A descriptor differs per MMA;
//          bvary = B descriptor differs per MMA; N
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8_cost umma_i8_cost.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) | ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__global__ void k(int N, int dalt, int avary, int bvary, int steps, long long *clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t A0 = smem_u32(sm), B0 = A0 + 7 * 4096;
    const long long t0 = clock64();
    for (int s = 0; s < steps; s++) {
#pragma unroll
      for (int a = 0; a < 7; a++) {
        const uint64_t ad = sdesc(A0 + (avary ? a * 4096 : 0), 2048, 128);
        const uint64_t bd = sdesc(B0 + (bvary ? (6 - a) * 128 : 0), 256 * 16, 128);
        mma_i8(tm + (dalt ? (s & 1) * 256 : 0), ad, bd, id, (s | a) ? 1u : 0u);
      }
    }
    commit(&bar);
    mbar_wait(&bar, 0);
    clk[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  long long *dclk; cudaMalloc(&dclk, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int steps = 3000;
  for (int N : {32, 48, 112, 208})
    for (int dalt = 0; dalt < 2; dalt++)
      for (int av = 0; av < 2; av++)
        for (int bv = 0; bv < 2; bv++) {
          k<<<148, 128, 160 * 1024>>>(N, dalt, av, bv, steps, dclk);
          cudaError_t e = cudaDeviceSynchronize();
          long long c; cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
          printf("N=%3d dalt=%d avary=%d bvary=%d: %.1f clk per MMA %s\n", N, dalt, av, bv, c / (7.0 * steps), e ? cudaGetErrorString(e) : "");
        }
  return 0;
}
