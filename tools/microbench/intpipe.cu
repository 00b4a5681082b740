// Integer-pipe throughput microbenchmark for sm_100a (B200).
// Measures issue rate of the instructions the modular MAC / NTT kernels are built from.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

__global__ void k_madwide(uint64_t* out, uint32_t a0, uint32_t b0) {
  uint64_t acc[CH];
  uint32_t a = a0 + threadIdx.x, b = b0 ^ blockIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[c]) : "r"(a + c), "r"(b));
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_madlo(uint64_t* out, uint32_t a0, uint32_t b0) {
  uint32_t acc[CH];
  uint32_t a = a0 + threadIdx.x, b = b0 ^ blockIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[c]) : "r"(a + c), "r"(b));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_madhi(uint64_t* out, uint32_t a0, uint32_t b0) {
  uint32_t acc[CH];
  uint32_t a = a0 + threadIdx.x, b = b0 ^ blockIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(acc[c]) : "r"(a + c), "r"(b));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_iadd3(uint64_t* out, uint32_t a0, uint32_t b0) {
  uint32_t acc[CH];
  uint32_t a = a0 + threadIdx.x, b = b0 ^ blockIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("add.u32 %0, %0, %1;" : "+r"(acc[c]) : "r"(a + c));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s + b;
}

__global__ void k_dfma(uint64_t* out, double a0, double b0) {
  double acc[CH];
  double a = a0 + threadIdx.x, b = b0 + blockIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc[c]) : "d"(a + c), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += acc[c];
  if (s == 0.5) out[0] = 1;
}

__global__ void k_ffma(uint64_t* out, float a0, float b0) {
  float acc[CH];
  float a = a0 + threadIdx.x, b = b0 + blockIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[c]) : "f"(a + c), "f"(b));
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += acc[c];
  if (s == 0.5f) out[0] = 1;
}

// 64x64 -> high 64 (what __umul64hi costs)
__global__ void k_mulhi64(uint64_t* out, uint64_t a0, uint64_t b0) {
  uint64_t acc[CH];
  uint64_t a = a0 + threadIdx.x, b = b0 ^ blockIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      acc[c] = __umul64hi(acc[c] + a, b);
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

// 64x64 -> low 64
__global__ void k_mullo64(uint64_t* out, uint64_t a0, uint64_t b0) {
  uint64_t acc[CH];
  uint64_t a = a0 + threadIdx.x, b = b0 ^ blockIdx.x;
#pragma unroll
  for (int c = 0; c < CH; c++) acc[c] = c + 1;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      acc[c] = acc[c] * b + a;
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

template <typename K, typename A>
void run(const char* name, K kern, A a, A b, double ops_per_iter_per_thread) {
  uint64_t* d; cudaMalloc(&d, 64);
  int blocks = 148 * 8, threads = 256;
  for (int w = 0; w < 2; w++) kern<<<blocks, threads>>>(d, a, b);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; r++) kern<<<blocks, threads>>>(d, a, b);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)reps * blocks * threads * ITERS * ops_per_iter_per_thread;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double gops = ops / (ms * 1e-3) / 1e9;
  printf("%-10s %10.1f Gop/s   %7.2f op/clk/SM @max-clock %d MHz   (%.3f ms)\n", name, gops,
         gops * 1e9 / (148.0 * clk * 1e3), clk / 1000, ms / reps);
  cudaFree(d);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(err));
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  run("madwide", k_madwide, 3u, 5u, CH);
  run("madlo", k_madlo, 3u, 5u, CH);
  run("madhi", k_madhi, 3u, 5u, CH);
  run("add32", k_iadd3, 3u, 5u, CH);
  run("dfma", k_dfma, 1.0, 1.0000001, CH);
  run("ffma", k_ffma, 1.0f, 1.0000001f, CH);
  run("mulhi64", k_mulhi64, (uint64_t)3, (uint64_t)0x123456789abcdefull, CH);
  run("mullo64+add", k_mullo64, (uint64_t)3, (uint64_t)0x123456789abcdefull, CH);
  run("madwide", k_madwide, 3u, 5u, CH);
  return 0;
}
