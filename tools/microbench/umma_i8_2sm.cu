// tcgen05.mma kind::i8 throughput: one CTA (cta_group::1, M = 128) vs a CTA pair (cta_group::2,
// M = 256: each CTA holds 128 rows of A and N/2 rows of B in its own shared memory, each CTA's TMEM
// receives its 128 rows x N).  7 MMAs per step as in the MAC (same B, A plane a, accumulator window
// shifted by a*16 columns).  Prints clk per MMA (of the issuing CTA) for N = 112 and N = 208.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8_2sm umma_i8_2sm.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) | ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int PAIR>
__global__ void __cluster_dims__(2, 1, 1) k(int N, int steps, long long *clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t nb = PAIR ? N / 2 : N;                // B rows held by this CTA
  if (threadIdx.x == 0 && (!PAIR || rank == 0)) {
    const uint32_t id = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24);
    const uint32_t A0 = smem_u32(sm), B0 = A0 + 7 * 4096;
    const long long t0 = clock64();
    for (int s = 0; s < steps; s++) {
#pragma unroll
      for (int a = 0; a < 7; a++) {
        const uint64_t ad = sdesc(A0 + a * 4096, 2048, 128);
        const uint64_t bd = sdesc(B0, nb * 16, 128);
        const uint32_t d = tm + (s & 1) * 256 + a * 16, acc = (s | a) ? 1u : 0u;
        if (PAIR)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc));
      }
    }
    if (PAIR)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    mbar_wait(&bar, 0);
    clk[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 0 && PAIR) {
    mbar_wait(&bar, 0);                                 // the peer's accumulators are written too
    clk[blockIdx.x] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}
int main() {
  long long *dclk; cudaMalloc(&dclk, 148 * 8);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int steps = 3000;
  for (int N : {112, 208, 256}) {
    for (int pair = 0; pair < 2; pair++) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (pair) k<1><<<148, 128, 64 * 1024>>>(N, steps, dclk); else k<0><<<148, 128, 64 * 1024>>>(N, steps, dclk);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
      long long c; cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
      const double rows = pair ? 256.0 : 128.0, ctas_mma = pair ? 74 : 148;
      printf("N=%3d %s: %.1f clk per MMA (issuer), %.3f ms; rows x N per SM per clk = %.1f %s\n", N, pair ? "cta_group::2 M=256" : "cta_group::1 M=128",
             c / (7.0 * steps), ms, rows * N / (c / (7.0 * steps)) * ctas_mma / 148, e ? cudaGetErrorString(e) : "");
    }
  }
  return 0;
}
