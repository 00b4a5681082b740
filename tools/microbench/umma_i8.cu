// tcgen05.mma kind::i8 on sm_100a: correctness of the descriptor conventions used by the
// tensor-core MAC engine (K-major, no swizzle, shifted B descriptors = Toeplitz limb products),
// and the u8 x u8 -> s32 MMA rate per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8 umma_i8.cu && ./umma_i8
//
// Test: A = 7 byte planes w_a [128 rows][32 K], Z = B image [2 K-halves][ZR rows][16 B] with
// the limb rows x_b at rows (b+6)*CW + c; MMA a uses B descriptor start + (6-a)*CW rows.
// D[i][d*CW + c] must equal sum_a sum_k w_a[i][k] x_{d-a}[c][k].
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

template <int CW> struct G {
  static constexpr int N = ((13 * CW + 15) / 16) * 16;      // MMA N
  static constexpr int ZR = N + 6 * CW;                     // B image rows
  static constexpr int A_BYTES = 7 * 2 * 128 * 16;
  static constexpr int Z_BYTES = 2 * ZR * 16;
  static constexpr int TCOLS = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
               ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

template <int CW, int M = 128>
__global__ void k_test(const uint8_t *A, const uint8_t *Z, int32_t *D, int reps, long long *clk) {
  using g = G<CW>;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *sA = sm, *sZ = sm + g::A_BYTES;
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < g::A_BYTES / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sA)[i] = reinterpret_cast<const uint4 *>(A)[i];
  for (int i = threadIdx.x; i < g::Z_BYTES / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sZ)[i] = reinterpret_cast<const uint4 *>(Z)[i];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(g::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_i8(M, g::N);
    t0 = clock64();
    for (int r = 0; r < reps; r++) {
#pragma unroll
      for (int a = 0; a < 7; a++) {
        const uint64_t ad = sdesc(smem_u32(sA + a * 2 * 128 * 16), 128 * 16, 128);
        const uint64_t bd = sdesc(smem_u32(sZ + (6 - a) * CW * 16), g::ZR * 16, 128);
        mma_i8(tm, ad, bd, id, (r | a) ? 1u : 0u);
      }
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) { t1 = clock64(); clk[blockIdx.x] = t1 - t0; }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w reads lanes 32w..32w+31, 8 columns per load
  const int lane_row = 32 * warp + (threadIdx.x & 31);
  for (int c0 = 0; c0 < g::N; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tm + ((uint32_t)(32 * warp) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (blockIdx.x == 0)
      for (int j = 0; j < 8; j++) D[lane_row * g::N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(g::TCOLS));
}

template <int CW, int M = 128>
int run(int reps, int nblk) {
  using g = G<CW>;
  std::vector<uint8_t> A(g::A_BYTES), Z(g::Z_BYTES, 0);
  // w[a][i][k], x[b][c][k]
  uint8_t w[7][128][32], x[7][16][32];
  srand(1234 + CW);
  for (int a = 0; a < 7; a++) for (int i = 0; i < 128; i++) for (int k = 0; k < 32; k++) w[a][i][k] = rand() & 255;
  for (int b = 0; b < 7; b++) for (int c = 0; c < CW; c++) for (int k = 0; k < 32; k++) x[b][c][k] = rand() & 255;
  for (int a = 0; a < 7; a++) for (int i = 0; i < 128; i++) for (int k = 0; k < 32; k++)
    A[((a * 2 + k / 16) * 128 + i) * 16 + k % 16] = w[a][i][k];
  for (int b = 0; b < 7; b++) for (int c = 0; c < CW; c++) for (int k = 0; k < 32; k++)
    Z[((k / 16) * g::ZR + (b + 6) * CW + c) * 16 + k % 16] = x[b][c][k];
  uint8_t *dA, *dZ; int32_t *dD; long long *dclk;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dZ, Z.size()));
  CK(cudaMalloc(&dD, 128 * g::N * 4)); CK(cudaMalloc(&dclk, nblk * 8));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dZ, Z.data(), Z.size(), cudaMemcpyHostToDevice));
  const int smem = g::A_BYTES + g::Z_BYTES;
  CK(cudaFuncSetAttribute(k_test<CW, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_test<CW, M><<<1, 128, smem>>>(dA, dZ, dD, 1, dclk);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<int32_t> D(128 * g::N);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  if (M == 64) {   // locate where row i landed: print lane of first match for a few rows
    for (int i = 0; i < 64; i += 1) {
      long long e0 = 0;
      for (int k = 0; k < 32; k++) e0 += (long long)w[0][i][k] * x[0][0][k];   // d=0,c=0 column
      int found = -1, nf = 0;
      for (int ln = 0; ln < 128; ln++) if (D[ln * g::N + 0] == e0) { if (found < 0) found = ln; nf++; }
      if (i < 20 || i % 16 == 15) printf("M=64 row %d -> lane %d (%d matches)\n", i, found, nf);
    }
  }
  for (int i = 0; i < (M == 64 ? 0 : 128); i++)
    for (int d = 0; d < 13; d++)
      for (int c = 0; c < CW; c++) {
        long long e = 0;
        for (int a = 0; a < 7; a++) {
          const int b = d - a;
          if (b < 0 || b > 6) continue;
          for (int k = 0; k < 32; k++) e += (long long)w[a][i][k] * x[b][c][k];
        }
        const long long got = D[i * g::N + d * CW + c];
        if (got != e && bad++ < 5) printf("CW=%d mismatch i=%d d=%d c=%d got %lld exp %lld\n", CW, i, d, c, got, e);
      }
  printf("M=%d CW=%d N=%d correctness: %s (%d bad)\n", M, CW, g::N, bad ? "FAIL" : "ok", bad);
  // throughput: every SM, reps x 7 MMAs
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_test<CW, M><<<nblk, 128, smem>>>(dA, dZ, dD, reps, dclk);
  cudaEventRecord(e0);
  k_test<CW, M><<<nblk, 128, smem>>>(dA, dZ, dD, reps, dclk);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> clk(nblk);
  CK(cudaMemcpy(clk.data(), dclk, nblk * 8, cudaMemcpyDeviceToHost));
  double macs = (double)nblk * reps * 7 * (double)M * g::N * 32;
  printf("CW=%d N=%d: %d CTAs x %d x 7 MMAs: %.3f ms, %.1f T MAC/s, %.0f MAC/clk/SM (clk64 %lld)\n", CW, g::N, nblk,
         reps, ms, macs / ms / 1e9, macs / nblk / (double)clk[0], clk[0]);
  cudaFree(dA); cudaFree(dZ); cudaFree(dD); cudaFree(dclk);
  return bad;
}

int main() {
  int bad = 0;
  bad += run<2>(2000, 148);
  bad += run<4>(2000, 148);
  bad += run<8>(2000, 148);
  bad += run<16>(2000, 148);
  bad += run<8, 64>(2000, 148);
  bad += run<16, 64>(2000, 148);
  printf(bad ? "FAILED\n" : "ALL OK\n");
  return bad != 0;
}
