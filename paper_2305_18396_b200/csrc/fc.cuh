// fc.cuh -- SURVEY.md §8(f) row f1: the server side of the FC-layer protocol.
// Included by kernels.cu after mac_tc.cuh (uses its UMMA / mbarrier helpers).
//
// With the layer input shared as x = <x>_0 + <x>_1 (client, server), the client's share of
// y = W x + b is its decrypted share of Pi_MatMul(W, <x>_0) and the server's is
//     <y>_1 = <W<x>_0>_1 + W<x>_1 + b                     (mod 2^l)
// i.e. in the layout of X.W (reading C1): share_server[Nb][Ma] += X1.W + b (mod 2^t).
// X1.W mod 2^t (t = 2^37) is a plain dense product -- on the int8 tensor cores: values split into
// 5 unsigned byte limbs, X1 = sum_a x_a 2^(8a), W = sum_b w_b 2^(8b); mod 2^37 only the limb pairs
// with a + b <= 4 survive (2^(8(a+b)) = 0 mod 2^40 otherwise), so 15 MMAs per 32-K step
// accumulate S_d = sum_{a+b=d} x_a . w_b (d = 0..4, exact s32 for R <= 6400) in 5 TMEM
// accumulators; the epilogue forms sum_d S_d 2^(8d) + b + share mod 2^t.
//
// Layouts (UMMA canonical K-major, no swizzle):
//   W planes (hl_fc_encode_weights, offline) [N tile of 48 cols][32-K step][plane b][K half][48][16 B]
//   X1 planes (per call, k_fc_x_planes)      [M tile of 128 rows][32-K step][plane a][K half][128][16 B]
// Kernel: one CTA per (M tile, N tile), 256 threads: warp 0 TMA producer (one bulk copy per
// operand per K step), warp 1 TMEM allocator + MMA issuer, warps 4-7 epilogue.
#pragma once

constexpr int kFcNT = 48;                          // N tile (output columns)
constexpr int kFcMT = 128;                         // M tile (rows)
constexpr int kFcLimbs = 5;                        // 5 bytes cover t <= 40 bits
constexpr int kFcAStage = kFcLimbs * 2 * kFcMT * 16;   // 20480 B
constexpr int kFcBStage = kFcLimbs * 2 * kFcNT * 16;   // 7680 B
constexpr int kFcStage = kFcAStage + kFcBStage;
constexpr int kFcNst = 4;
constexpr int kFcSmem = kFcNst * kFcStage + 256;

struct FcGeom {
  int64_t Nb, R, Ma;
  int nMt, nNt, nKc;                               // tiles of 128 rows, 48 columns, 32 K
  int kps;                                         // 32-K steps per split (grid z = split-K)
  uint64_t tmask;
};

// W [R][Ma] (< 2^t) -> byte planes, zero padded (columns >= Ma, K >= R).  Flags W >= 2^t.
__global__ void k_fc_w_planes(const uint64_t *__restrict__ W, uint8_t *__restrict__ wp, FcGeom g, uint32_t *flags) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;      // one element (k, j) of the padded grid
  const int64_t ncol = (int64_t)g.nNt * kFcNT, nk = (int64_t)g.nKc * 32;
  if (e >= ncol * nk) return;
  const int64_t k = e / ncol, j = e % ncol;
  uint64_t w = 0;
  if (k < g.R && j < g.Ma) {
    w = W[k * g.Ma + j];
    if (w & ~g.tmask) atomicOr(&flags[0], 1u);
  }
  const int nt = (int)(j / kFcNT), jr = (int)(j % kFcNT), kc = (int)(k >> 5), h = (int)((k >> 4) & 1), kk = (int)(k & 15);
  uint8_t *dst = wp + ((size_t)nt * g.nKc + kc) * kFcBStage + h * kFcNT * 16 + jr * 16 + kk;
#pragma unroll
  for (int b = 0; b < kFcLimbs; b++) dst[b * 2 * kFcNT * 16] = (uint8_t)(w >> (8 * b));
}

// X1 [Nb][R] -> byte planes (taken mod 2^t), zero padded (rows >= Nb, K >= R); a thread packs 4
// consecutive k of one row: one 4-byte store per plane
__global__ void k_fc_x_planes(const uint64_t *__restrict__ X1, uint8_t *__restrict__ xp, FcGeom g) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nrow = (int64_t)g.nMt * kFcMT, nk4 = (int64_t)g.nKc * 8;
  if (e >= nrow * nk4) return;
  const int64_t i = e / nk4, k0 = (e % nk4) * 4;
  uint32_t w[kFcLimbs] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int64_t k = k0 + j;
    const uint64_t x = (i < g.Nb && k < g.R) ? (X1[i * g.R + k] & g.tmask) : 0;
#pragma unroll
    for (int a = 0; a < kFcLimbs; a++) w[a] |= (uint32_t)((x >> (8 * a)) & 0xff) << (8 * j);
  }
  const int mt = (int)(i / kFcMT), ir = (int)(i % kFcMT), kc = (int)(k0 >> 5), h = (int)((k0 >> 4) & 1), kk = (int)(k0 & 15);
  uint8_t *dst = xp + ((size_t)mt * g.nKc + kc) * kFcAStage + h * kFcMT * 16 + ir * 16 + kk;
#pragma unroll
  for (int a = 0; a < kFcLimbs; a++) *reinterpret_cast<uint32_t *>(dst + a * 2 * kFcMT * 16) = w[a];
}

// share &= 2^t - 1 after the split-K partial sums were added (wrapping u64 = exact mod 2^t)
__global__ void k_fc_mask(uint64_t *__restrict__ share, int64_t n, uint64_t tmask) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) share[i] &= tmask;
}

__global__ void __launch_bounds__(256, 1)
k_fc_gemm(const uint8_t *__restrict__ xp, const uint8_t *__restrict__ wp, const uint64_t *__restrict__ bias,
          uint64_t *__restrict__ share, FcGeom g) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kFcNst * kFcStage);
  uint64_t *empty = full + kFcNst, *tfull = empty + kFcNst;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = blockIdx.x, mt = blockIdx.y;
  const int kc0 = blockIdx.z * g.kps, kc1 = min(g.nKc, kc0 + g.kps);   // this CTA's split of K
  if (threadIdx.x == 0) {
    for (int i = 0; i < kFcNst; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint8_t *xa = xp + (size_t)mt * g.nKc * kFcAStage, *wb = wp + (size_t)nt * g.nKc * kFcBStage;
      for (int kc = kc0; kc < kc1; kc++) {
        const int st = (kc - kc0) % kFcNst;
        mbar_wait(&empty[st], (((kc - kc0) / kFcNst) & 1) ^ 1);
        unsigned char *dst = smem + st * kFcStage;
        mbar_expect_tx(&full[st], kFcStage);
        bulk_g2s(dst, xa + (size_t)kc * kFcAStage, kFcAStage, &full[st]);
        bulk_g2s(dst + kFcAStage, wb + (size_t)kc * kFcBStage, kFcBStage, &full[st]);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = umma_idesc_u8(kFcMT, kFcNT);
    for (int kc = kc0; kc < kc1; kc++) {
      const int st = (kc - kc0) % kFcNst;
      mbar_wait(&full[st], ((kc - kc0) / kFcNst) & 1);
      tc_fence_after();
      const uint32_t a0 = smem_u32(smem + st * kFcStage), b0 = a0 + kFcAStage;
      if (elect_one()) {
#pragma unroll
        for (int a = 0; a < kFcLimbs; a++)
#pragma unroll
          for (int b = 0; a + b < kFcLimbs; b++)
            umma_i8(tmem + (a + b) * kFcNT, umma_sdesc(a0 + a * 2 * kFcMT * 16, kFcMT * 16, 128),
                    umma_sdesc(b0 + b * 2 * kFcNT * 16, kFcNT * 16, 128), idesc, (kc > kc0 || a > 0) ? 1u : 0u);   // a == 0 writes accumulator d first
        umma_commit(&empty[st]);
        if (kc == kc1 - 1) umma_commit(tfull);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // accumulator d of row (lane quadrant) in TMEM columns d*48 .. d*48+47
    const int q = warp & 3;
    const int64_t row = (int64_t)mt * kFcMT + 32 * q + lane;
    mbar_wait(tfull, 0);
    tc_fence_after();
    const uint32_t base = tmem + ((uint32_t)(32 * q) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < kFcNT; c0 += 8) {
      uint32_t v[kFcLimbs][8];
#pragma unroll
      for (int d = 0; d < kFcLimbs; d++) tmem_ld_cw<8>(base + d * kFcNT + c0, v[d]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < g.Nb) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int64_t col = (int64_t)nt * kFcNT + c0 + j;
          if (col >= g.Ma) break;
          uint64_t acc = 0;
#pragma unroll
          for (int d = 0; d < kFcLimbs; d++) acc += (uint64_t)v[d][j] << (8 * d);   // wraps mod 2^64
          if (blockIdx.z == 0 && bias) acc += bias[col];
          atomicAdd(reinterpret_cast<unsigned long long *>(share + row * g.Ma + col), (unsigned long long)acc);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}
