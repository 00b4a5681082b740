// chacha.h -- ChaCha20 block function (RFC 8439 §2.3) as the library's PRF (reading C10).
// Host and device.  Independent of oracle/oracle.c (written separately; parity is tested).
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define HL_HD __host__ __device__ __forceinline__
#else
#define HL_HD inline
#endif

namespace hl {

enum : uint32_t { kDomSK = 1, kDomA = 2, kDomE = 3, kDomMask = 4,
                  kDomPkA = 5, kDomPkE = 6, kDomRrU = 7, kDomRrE = 8, kDomRrF = 9,   // 5-9: row f4 (reading C22)
                  kDomPub = 10 };                                                     // reading C28

HL_HD uint32_t rotl(uint32_t x, int n) {
#ifdef __CUDA_ARCH__
  return __funnelshift_l(x, x, n);
#else
  return (x << n) | (x >> (32 - n));
#endif
}

#define HL_QR(a, b, c, d)              \
  a += b; d ^= a; d = rotl(d, 16);     \
  c += d; b ^= c; b = rotl(b, 12);     \
  a += b; d ^= a; d = rotl(d, 8);      \
  c += d; b ^= c; b = rotl(b, 7);

// 64-byte keystream block for key = LE64(seed) || 0^24, nonce = LE32(domain) || LE64(stream),
// block counter `ctr`; returned as 8 little-endian u64 words.
HL_HD void chacha_block_u64(uint64_t seed, uint32_t domain, uint64_t stream, uint32_t ctr,
                            uint64_t out[8]) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const uint32_t n0 = domain, n1 = (uint32_t)stream, n2 = (uint32_t)(stream >> 32);
  uint32_t x0 = 0x61707865u, x1 = 0x3320646eu, x2 = 0x79622d32u, x3 = 0x6b206574u;
  uint32_t x4 = k0, x5 = k1, x6 = 0, x7 = 0, x8 = 0, x9 = 0, x10 = 0, x11 = 0;
  uint32_t x12 = ctr, x13 = n0, x14 = n1, x15 = n2;
#pragma unroll 1
  for (int i = 0; i < 10; i++) {   // not unrolled: keeps the fused INTT+mask kernel within the I-cache
    HL_QR(x0, x4, x8, x12) HL_QR(x1, x5, x9, x13) HL_QR(x2, x6, x10, x14) HL_QR(x3, x7, x11, x15)
    HL_QR(x0, x5, x10, x15) HL_QR(x1, x6, x11, x12) HL_QR(x2, x7, x8, x13) HL_QR(x3, x4, x9, x14)
  }
  x0 += 0x61707865u; x1 += 0x3320646eu; x2 += 0x79622d32u; x3 += 0x6b206574u;
  x4 += k0; x5 += k1; x12 += ctr; x13 += n0; x14 += n1; x15 += n2;
  out[0] = (uint64_t)x0 | ((uint64_t)x1 << 32);
  out[1] = (uint64_t)x2 | ((uint64_t)x3 << 32);
  out[2] = (uint64_t)x4 | ((uint64_t)x5 << 32);
  out[3] = (uint64_t)x6 | ((uint64_t)x7 << 32);
  out[4] = (uint64_t)x8 | ((uint64_t)x9 << 32);
  out[5] = (uint64_t)x10 | ((uint64_t)x11 << 32);
  out[6] = (uint64_t)x12 | ((uint64_t)x13 << 32);
  out[7] = (uint64_t)x14 | ((uint64_t)x15 << 32);
}
#undef HL_QR

// Single u64 word `idx` of a stream.
HL_HD uint64_t prf_u64(uint64_t seed, uint32_t domain, uint64_t stream, uint64_t idx) {
  uint64_t w[8];
  chacha_block_u64(seed, domain, stream, (uint32_t)(idx >> 3), w);
  uint64_t r = w[0];
#pragma unroll
  for (int i = 1; i < 8; i++) r = ((idx & 7) == (uint64_t)i) ? w[i] : r;
  return r;
}

// Reading C28: the A domain (the public c1 = a_hat) is keyed by a public seed derived one-way from
// the client's private encryption seed; the E domain (the errors) by the private seed itself.
HL_HD uint64_t public_seed(uint64_t enc_seed) {
  uint64_t w[8];
  chacha_block_u64(enc_seed, kDomPub, 0, 0, w);
  return w[0];
}

}  // namespace hl
