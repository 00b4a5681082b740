// IMAD.WIDE.U32 / IMAD / IMAD.HI / DFMA peak on sm_100a with operands that cannot be hoisted:
// the multiplier of chain c is the low word of chain c+1 (no extra ALU instructions).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 2048
#define CH 8
__global__ void k_wide(uint64_t *out, uint32_t seed) {
  uint64_t acc[CH];
  const uint32_t y = seed ^ threadIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = seed + c * 77 + threadIdx.x;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++)
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[c]) : "r"((uint32_t)acc[(c + 1) % CH]), "r"(y));
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}
__global__ void k_wide_mixed(uint64_t *out, uint32_t seed) {   // 2 IMAD.WIDE : 1 IMAD
  uint64_t acc[CH]; uint32_t a32[CH];
  const uint32_t y = seed ^ threadIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) { acc[c] = seed + c * 77 + threadIdx.x; a32[c] = c; }
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[c]) : "r"((uint32_t)acc[(c + 1) % CH]), "r"(y));
      if (c & 1) asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a32[c]) : "r"((uint32_t)acc[c]), "r"(y));
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c] + a32[c];
  if (s == 0x12345) out[0] = s;
}
__global__ void k_wide_dfma(uint64_t *out, uint32_t seed) {   // 1 IMAD.WIDE : 1 DFMA (pipe overlap?)
  uint64_t acc[CH]; double d[CH];
  const uint32_t y = seed ^ threadIdx.x;
  const double yd = 1.0 + 1e-9 * y;
#pragma unroll
  for (int c = 0; c < CH; c++) { acc[c] = seed + c * 77 + threadIdx.x; d[c] = c; }
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[c]) : "r"((uint32_t)acc[(c + 1) % CH]), "r"(y));
      asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(d[c]) : "d"(d[(c + 1) % CH]), "d"(yd));
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c] + (uint64_t)d[c];
  if (s == 0x12345) out[0] = s;
}
__global__ void k_lo(uint64_t *out, uint32_t seed) {
  uint32_t acc[CH];
  const uint32_t y = seed ^ threadIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = seed + c * 77 + threadIdx.x;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++)
      asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[c]) : "r"(acc[(c + 1) % CH]), "r"(y));
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}
__global__ void k_dfma(uint64_t *out, uint32_t seed) {
  double acc[CH];
  const double y = 1.0 + 1e-9 * (seed ^ threadIdx.x);
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = c + 1e-7 * threadIdx.x;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++)
      asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc[c]) : "d"(acc[(c + 1) % CH]), "d"(y));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += acc[c];
  if (s == 0.5) out[0] = 1;
}
typedef void (*kern_t)(uint64_t *, uint32_t);
void run(const char *name, kern_t k, double ops, int bps) {
  uint64_t *d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * bps, threads = 256;
  for (int w = 0; w < 2; w++) k<<<blocks, threads>>>(d, 12345u);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) k<<<blocks, threads>>>(d, 12345u);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double r = 5.0 * blocks * threads * ITERS * ops / (ms * 1e-3);
  printf("%-11s warps/SM %3d  %8.1f G/s  %6.2f /clk/SM @max clock\n", name, bps * 8, r / 1e9, r / ((double)sms * clk * 1e3));
}
int main() {
  for (int bps : {2, 4, 8}) {
    run("imad.wide", k_wide, CH, bps);
    run("wide(2:1lo)", k_wide_mixed, CH, bps);
    run("wide+dfma", k_wide_dfma, CH, bps);
    run("imad.lo", k_lo, CH, bps);
    run("dfma", k_dfma, CH, bps);
  }
}
