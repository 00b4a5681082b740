// tcgen05.mma kind::i8 M=128 K=32 rate vs the shared-memory layout of A and B (K-major):
// SWIZZLE_NONE (core matrices 8 rows x 16 B, rows 16 B apart), SWIZZLE_32B / 64B / 128B
// (rows 32 / 64 / 128 B apart, 8-row atoms), rotating over 8 stage buffers like the MAC ring.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8_swz umma_i8_swz.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) | ((uint64_t)((sbo >> 4) & 0x3fff) << 32) |
         (1ull << 46) | ((uint64_t)layout << 61);
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
// layout: 0 none, 6 = 32B, 4 = 64B, 2 = 128B.  pitch = row pitch in bytes (16 for none)
__global__ void k(int layout, int pitch, int N, int nst, int steps, long long *clk, int var) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const int abytes = 128 * 32 * 2, bbytes = 256 * 32 * 2, sb = abytes + bbytes;   // generous
  for (int i = threadIdx.x; i < nst * sb / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const long long t0 = clock64();
    for (int s = 0; s < steps; s++) {
      const int st = s % nst;
      const uint32_t a0 = smem_u32(sm + st * sb), b0 = a0 + abytes;
      // none: lbo = K-half distance (rows*16), sbo = 128;  swizzled: lbo unused (16), sbo = 8 rows * pitch
      uint32_t alb = layout ? 16 : 128 * 16, blb = layout ? 16 : N * 16;
      uint32_t asb = layout ? 8 * pitch : 128, bsb = layout ? 8 * pitch : 128;
      if (!layout && var == 1) { alb += 128; blb += 128; }          // pad the K-half distance by 128 B
      if (!layout && var == 2) { alb += 64; blb += 64; }
      if (!layout && var == 3) { alb = 128; blb = 128; asb = 256; bsb = 256; }   // K halves adjacent per 8-row group
      // for swizzled layouts with pitch > 32 B, 7 MMAs walk the K extent of a row (32 B per K-step)
      const int kper = layout ? pitch / 32 : 1;
#pragma unroll
      for (int a = 0; a < 7; a++) {
        const uint32_t koff = layout ? (a % kper) * 32 : 0;
        mma_i8(tm + (s & 1) * 256, sdesc(a0 + koff, alb, asb, layout), sdesc(b0 + koff, blb, bsb, layout), id, (s | a) ? 1u : 0u);
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
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int steps = 3000, nst = 8;
  const int sb = 128 * 32 * 2 + 256 * 32 * 2;
  struct { int layout, pitch; const char *name; } L[] = {{0, 16, "none"}, {6, 32, "sw32"}, {4, 64, "sw64"}, {2, 128, "sw128"}};
  for (int N : {48, 112, 208})
    for (int var = 0; var < 4; var++)
      for (int ns : {8, 1}) {
        k<<<148, 128, nst * sb>>>(0, 16, N, ns, steps, dclk, var);
        cudaError_t e = cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
        printf("N=%3d none var%d nst=%d %.1f clk per MMA %s\n", N, var, ns, c / (7.0 * steps), e ? cudaGetErrorString(e) : "");
      }
  for (int N : {48, 112})
    for (int li = 1; li < 3; li++)
      for (int ns : {8, 1}) {
        k<<<148, 128, nst * sb>>>(L[li].layout, L[li].pitch, N, ns, steps, dclk, 0);
        cudaError_t e = cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
        printf("N=%3d %-6s nst=%d %.1f clk per MMA %s\n", N, L[li].name, ns, c / (7.0 * steps), e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
