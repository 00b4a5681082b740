// Which factors slow tcgen05.mma kind::i8 (M=128, N=112, K=32) inside the MAC kernel?
//   mode 0: 7 MMAs per step on one fixed stage (baseline)
//   mode 1: + tcgen05.commit to an mbarrier after every step
//   mode 2: rotate over NST stage buffers (A rows = RT layout, LBO = 16*RT)
//   mode 3: mode 1 + mode 2
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8_pipe umma_i8_pipe.cu
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
constexpr int N = 112, CW = 8, ZR = N + 6 * CW;
__global__ void k(int mode, int rt, int nst, int sb, int steps, long long *clk) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bars[16];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < nst * sb / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
  if (threadIdx.x == 0) { for (int i = 0; i < 16; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i]))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const long long t0 = clock64();
    const bool rot = mode & 2, com = mode & 1;
    for (int s = 0; s < steps; s++) {
      const int st = rot ? s % nst : 0;
      const uint32_t z0 = smem_u32(sm + st * sb), a0 = z0 + 2 * ZR * 16 + 32 * CW * 8;
#pragma unroll
      for (int a = 0; a < 7; a++) mma_i8(tm + (s & 1) * N, sdesc(a0 + a * 32 * rt, rt * 16, 128), sdesc(z0 + (6 - a) * CW * 16, ZR * 16, 128), id, (s | a) ? 1u : 0u);
      if (com) commit(&bars[st]);
    }
    commit(&bars[15]);
    mbar_wait(&bars[15], 0);
    clk[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}
int main() {
  long long *dclk; cudaMalloc(&dclk, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int steps = 3000;
  for (int rt : {128, 48, 72}) {
    const int sb = ((2 * ZR * 16 + 32 * CW * 8 + 208 * rt + 2048) + 127) / 128 * 128;
    const int nst = (200 * 1024) / sb > 12 ? 12 : (200 * 1024) / sb;
    for (int mode = 0; mode < 4; mode++) {
      k<<<148, 128, nst * sb>>>(mode, rt, nst, sb, steps, dclk);
      cudaError_t e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
      printf("rt=%3d nst=%2d mode %d: %.1f clk per MMA %s\n", rt, nst, mode, c / (7.0 * steps), e ? cudaGetErrorString(e) : "");
    }
  }
  return 0;
}
