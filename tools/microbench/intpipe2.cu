// Integer-pipe throughput on sm_100a, with per-iteration-varying operands so that ptxas
// cannot hoist or strength-reduce the multiplies (tools/microbench/intpipe.cu could).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
#define CH 8

// IMAD.WIDE.U32: acc_c += x_c * y   (x_c advanced by an ALU add each iteration)
__global__ void k_wide(uint64_t *out, uint32_t seed) {
  uint64_t acc[CH]; uint32_t x[CH];
  const uint32_t y = seed ^ threadIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) { acc[c] = c; x[c] = seed + c * 77 + threadIdx.x; }
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[c]) : "r"(x[c]), "r"(y));
      asm volatile("add.u32 %0, %0, 0x9e3779b9;" : "+r"(x[c]));
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

// IMAD (32-bit lo): acc_c = x_c * y + acc_c
__global__ void k_lo(uint64_t *out, uint32_t seed) {
  uint32_t acc[CH]; uint32_t x[CH];
  const uint32_t y = seed ^ threadIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) { acc[c] = c; x[c] = seed + c * 77 + threadIdx.x; }
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[c]) : "r"(x[c]), "r"(y));
      asm volatile("add.u32 %0, %0, 0x9e3779b9;" : "+r"(x[c]));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

// IMAD.HI: acc_c = hi(x_c * y) + acc_c
__global__ void k_hi(uint64_t *out, uint32_t seed) {
  uint32_t acc[CH]; uint32_t x[CH];
  const uint32_t y = seed ^ threadIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) { acc[c] = c; x[c] = seed + c * 77 + threadIdx.x; }
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(acc[c]) : "r"(x[c]), "r"(y));
      asm volatile("add.u32 %0, %0, 0x9e3779b9;" : "+r"(x[c]));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

// DFMA: acc_c = x_c * y + acc_c   (x_c advanced by an FP add each iteration)
__global__ void k_dfma(uint64_t *out, uint32_t seed) {
  double acc[CH], x[CH];
  const double y = 1.0 + 1e-9 * (seed ^ threadIdx.x);
#pragma unroll
  for (int c = 0; c < CH; c++) { acc[c] = c; x[c] = 1.0 + c * 1e-3 + threadIdx.x * 1e-7; }
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc[c]) : "d"(x[c]), "d"(y));
      asm volatile("add.rn.f64 %0, %0, 0d3ff0000000000000;" : "+d"(x[c]));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += acc[c];
  if (s == 0.5) out[0] = 1;
}

// IADD3 only (ALU pipe reference): x_c += const
__global__ void k_add(uint64_t *out, uint32_t seed) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) x[c] = seed + c * 77 + threadIdx.x;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("add.u32 %0, %0, 0x9e3779b9;" : "+r"(x[c]));
      asm volatile("add.u32 %0, %0, 0x7f4a7c15;" : "+r"(x[c]));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= x[c];
  if (s == 0x12345) out[0] = s;
}

typedef void (*kern_t)(uint64_t *, uint32_t);

void run(const char *name, kern_t k, double ops_per_thread_iter, int blocks_per_sm, int threads) {
  uint64_t *d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * blocks_per_sm;
  for (int w = 0; w < 2; w++) k<<<blocks, threads>>>(d, 12345u);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; r++) k<<<blocks, threads>>>(d, 12345u);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)reps * blocks * threads * ITERS * ops_per_thread_iter;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double gops = ops / (ms * 1e-3) / 1e9;
  printf("%-8s warps/SM %3d  %9.1f Gop/s  %6.2f op/clk/SM @ %d MHz\n", name, blocks_per_sm * threads / 32, gops,
         gops * 1e9 / ((double)sms * clk * 1e3), clk / 1000);
  cudaFree(d);
}

int main() {
  for (int bps : {2, 8}) {
    run("imadwide", k_wide, CH, bps, 256);
    run("imadlo", k_lo, CH, bps, 256);
    run("imadhi", k_hi, CH, bps, 256);
    run("dfma", k_dfma, CH, bps, 256);
    run("iadd", k_add, 2 * CH, bps, 256);
  }
  return 0;
}
