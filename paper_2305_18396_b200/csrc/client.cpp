// client.cpp -- client side of Alg. 1 on the host: keygen, pi_B + secret-key
// BFV encryption (step 2), decryption + pi_C^-1 decoding of the compressed response (step 4,
// PAPER.md:154 "m = s*c1 + c0").  Host memory; OpenMP over ciphertexts.  Independent of oracle/.
#include <omp.h>

#include <cstring>
#include <vector>

#include "chacha.h"
#include "hl_internal.h"

using hl::prf_u64;

// ---- 50-bit wire format (include/helinear.h) ------------------------------------------------
extern "C" int64_t hl_packed50_words(int64_t words) { return words <= 0 ? 0 : (words + 31) / 32 * 25; }

extern "C" int hl_pack50(const uint64_t *in, int64_t words, uint64_t *out) {
  if (!in || !out || words < 0) return hl_fail(HL_EINVAL, "hl_pack50: bad arguments");
  const int64_t ng = (words + 31) / 32;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t g = 0; g < ng; g++) {
    uint64_t w[25] = {0};
    for (int i = 0; i < 32; i++) {
      const int64_t e = g * 32 + i;
      const uint64_t v = e < words ? in[e] : 0;
      bad |= (v >> 50) != 0;
      const int b = 50 * i, q = b >> 6, r = b & 63;
      w[q] |= v << r;
      if (r > 14) w[q + 1] |= v >> (64 - r);
    }
    memcpy(out + g * 25, w, sizeof(w));
  }
  return bad ? hl_fail(HL_ERANGE, "hl_pack50: word >= 2^50") : HL_OK;
}

extern "C" int hl_unpack50(const uint64_t *in, int64_t words, uint64_t *out) {
  if (!in || !out || words < 0) return hl_fail(HL_EINVAL, "hl_unpack50: bad arguments");
  const int64_t ng = (words + 31) / 32;
#pragma omp parallel for schedule(static)
  for (int64_t g = 0; g < ng; g++) {
    const uint64_t *w = in + g * 25;
    for (int i = 0; i < 32; i++) {
      const int64_t e = g * 32 + i;
      if (e >= words) break;
      const int b = 50 * i, q = b >> 6, r = b & 63;
      uint64_t v = w[q] >> r;
      if (r > 14) v |= w[q + 1] << (64 - r);
      out[e] = v & ((1ull << 50) - 1);
    }
  }
  return HL_OK;
}

extern "C" uint64_t hl_public_seed(uint64_t enc_seed) { return hl::public_seed(enc_seed); }

extern "C" int hl_keygen(const hl_ctx *c, uint64_t seed, int8_t *sk) {
  if (!c || !sk) return hl_fail(HL_EINVAL, "hl_keygen: NULL argument");
  // s_i = (u64_SK[i] mod 3) - 1  (reading C7); one ChaCha block serves 8 coefficients
  for (uint32_t b = 0; b < c->N / 8; b++) {
    uint64_t w[8];
    hl::chacha_block_u64(seed, hl::kDomSK, 0, b, w);
    for (int i = 0; i < 8; i++) sk[8 * b + i] = (int8_t)((int)(w[i] % 3) - 1);
  }
  return HL_OK;
}

static int check_sk(const hl_ctx *c, const int8_t *sk) {
  for (uint32_t i = 0; i < c->N; i++)
    if (sk[i] < -1 || sk[i] > 1) return hl_fail(HL_ERANGE, "secret key must be ternary");
  return HL_OK;
}

// NTT of the ternary secret per prime (bit-reversed NTT order, host)
static void sk_ntt(const hl_ctx *c, const int8_t *sk, std::vector<uint64_t> &out) {
  const uint32_t N = c->N;
  out.assign((size_t)c->L * N, 0);
  for (uint32_t l = 0; l < c->L; l++) {
    uint64_t p = c->primes[l], *s = &out[(size_t)l * N];
    for (uint32_t i = 0; i < N; i++) s[i] = sk[i] > 0 ? 1 : (sk[i] < 0 ? p - 1 : 0);
    hl_host_ntt_fwd(c, (int)l, s);
  }
}

extern "C" int hl_encrypt(const hl_ctx *c, const int8_t *sk, hl_tile tile, const uint64_t *X,
                          int64_t Nb, int64_t R, uint64_t seed, uint64_t *ct_in) {
  if (!c || !sk || !X || !ct_in) return hl_fail(HL_EINVAL, "hl_encrypt: NULL argument");
  Geo g;
  int rc = hl_geometry(c, tile, 1, R, Nb, 0, -1, &g);
  if (rc) return rc;
  if ((rc = check_sk(c, sk))) return rc;
  const uint64_t tmask = (1ull << c->log2_t) - 1;
  for (int64_t i = 0; i < Nb * R; i++)
    if (X[i] & ~tmask) return hl_fail(HL_ERANGE, "hl_encrypt: X value >= 2^log2_t");
  const uint32_t N = c->N, L = c->L;
  const int m = g.m, r = g.r, n = g.n;
  std::vector<uint64_t> shat;
  sk_ntt(c, sk, shat);
  const int64_t nct = g.nJ * g.nK;
  const uint64_t a_seed = hl::public_seed(seed);     // reading C28: a is keyed by the public seed
#pragma omp parallel
  {
    std::vector<uint64_t> b(N), a(N), as(N);
    std::vector<int64_t> e(N);
#pragma omp for schedule(dynamic)
    for (int64_t gi = 0; gi < nct; gi++) {
      const int64_t J = gi / g.nK, K = gi % g.nK;
      // pi_B: b[k*m*r + j] = B[j][k] = X[K*n+k][J*r+j], zero padded
      std::fill(b.begin(), b.end(), 0);
      for (int k = 0; k < n; k++)
        for (int j = 0; j < r; j++) {
          int64_t row = K * n + k, col = J * (int64_t)r + j;
          if (row < Nb && col < R) b[(size_t)k * m * r + j] = X[row * R + col];
        }
      // e: discrete Gaussian by CDT from stream (E, g): sign = u>>63, |e| = min{k : v < T[k]}
      for (uint32_t blk = 0; blk < N / 8; blk++) {
        uint64_t w[8];
        hl::chacha_block_u64(seed, hl::kDomE, (uint64_t)gi, blk, w);
        for (int i = 0; i < 8; i++) {
          uint64_t v = w[i] & 0x7fffffffffffffffull;
          int k = 0;
          while (k < 41 && v >= c->cdt[k]) k++;
          e[8 * blk + i] = (w[i] >> 63) ? -(int64_t)k : (int64_t)k;
        }
      }
      for (uint32_t l = 0; l < L; l++) {
        const uint64_t p = c->primes[l];
        // a_hat_l[k] = (u[2k] + 2^64 u[2k+1]) mod p, stream (a_seed, A, g*L + l): the evaluation form of
        // a (reading C26), natural order k; it is c1 as sent
        for (uint32_t blk = 0; blk < N / 4; blk++) {
          uint64_t w[8];
          hl::chacha_block_u64(a_seed, hl::kDomA, (uint64_t)gi * L + l, blk, w);
          for (int i = 0; i < 4; i++)
            a[4 * blk + i] = (uint64_t)((((hl_u128)w[2 * i + 1] << 64) | w[2 * i]) % p);
        }
        // a * s = INTT(a_hat . s_hat); the host NTT order is bit-reversed: index i <-> k = brv(i)
        const uint64_t *sh = &shat[(size_t)l * N];
        for (uint32_t i = 0; i < N; i++) as[i] = h_mulmod(a[c->brv[i]], sh[i], p);
        hl_host_ntt_inv(c, (int)l, as.data());
        uint64_t *c0 = ct_in + ((size_t)gi * 2 + 0) * L * N + (size_t)l * N;
        uint64_t *c1 = ct_in + ((size_t)gi * 2 + 1) * L * N + (size_t)l * N;
        const uint64_t dl = c->delta_mod[l];
        for (uint32_t i = 0; i < N; i++) {
          uint64_t v = as[i] ? p - as[i] : 0;                                  // -a*s
          uint64_t ev = e[i] >= 0 ? (uint64_t)e[i] : p - (uint64_t)(-e[i]);    // e mod p
          v += ev; if (v >= p) v -= p;
          v += h_mulmod(dl, b[i] % p, p); if (v >= p) v -= p;                   // + Delta*b
          c0[i] = v;
          c1[i] = a[i];
        }
      }
    }
  }
  return HL_OK;
}

// Public key (row f4, reading C22): pk1 = a (domain 5, stream l), pk0 = -a*s + e (e: domain 6,
// stream 0), layout [2][L][N], coefficient form.
extern "C" int hl_pk_gen(const hl_ctx *c, const int8_t *sk, uint64_t seed, uint64_t *pk) {
  if (!c || !sk || !pk) return hl_fail(HL_EINVAL, "hl_pk_gen: NULL argument");
  int rc;
  if ((rc = check_sk(c, sk))) return rc;
  const uint32_t N = c->N, L = c->L;
  std::vector<uint64_t> shat;
  sk_ntt(c, sk, shat);
  std::vector<int64_t> e(N);
  for (uint32_t blk = 0; blk < N / 8; blk++) {
    uint64_t w[8];
    hl::chacha_block_u64(seed, hl::kDomPkE, 0, blk, w);
    for (int i = 0; i < 8; i++) {
      uint64_t v = w[i] & 0x7fffffffffffffffull;
      int k = 0;
      while (k < 41 && v >= c->cdt[k]) k++;
      e[8 * blk + i] = (w[i] >> 63) ? -(int64_t)k : (int64_t)k;
    }
  }
  std::vector<uint64_t> a(N), as(N);
  for (uint32_t l = 0; l < L; l++) {
    const uint64_t p = c->primes[l];
    for (uint32_t blk = 0; blk < N / 4; blk++) {
      uint64_t w[8];
      hl::chacha_block_u64(seed, hl::kDomPkA, l, blk, w);
      for (int i = 0; i < 4; i++) a[4 * blk + i] = (uint64_t)((((hl_u128)w[2 * i + 1] << 64) | w[2 * i]) % p);
    }
    memcpy(as.data(), a.data(), 8ull * N);
    hl_host_ntt_fwd(c, (int)l, as.data());
    for (uint32_t i = 0; i < N; i++) as[i] = h_mulmod(as[i], shat[(size_t)l * N + i], p);
    hl_host_ntt_inv(c, (int)l, as.data());
    for (uint32_t i = 0; i < N; i++) {
      uint64_t v = as[i] ? p - as[i] : 0;
      uint64_t ev = e[i] >= 0 ? (uint64_t)e[i] : p - (uint64_t)(-e[i]);
      v += ev; if (v >= p) v -= p;
      pk[(size_t)l * N + i] = v;
      pk[(size_t)(L + l) * N + i] = a[i];
    }
  }
  return HL_OK;
}

// --- 256-bit helpers for the CRT and the rounding of decryption ---------------------------
struct U256 { uint64_t w[4]; };

static inline void u256_add(U256 &a, const U256 &b) {
  hl_u128 cy = 0;
  for (int i = 0; i < 4; i++) { cy += (hl_u128)a.w[i] + b.w[i]; a.w[i] = (uint64_t)cy; cy >>= 64; }
}
static inline void u256_sub(U256 &a, const U256 &b) {   // a >= b
  uint64_t br = 0;
  for (int i = 0; i < 4; i++) {
    uint64_t bi = b.w[i] + br;
    uint64_t nb = (bi < br) || (a.w[i] < bi);
    a.w[i] -= bi; br = nb;
  }
}
static inline bool u256_ge(const U256 &a, const U256 &b) {
  for (int i = 3; i >= 0; i--) if (a.w[i] != b.w[i]) return a.w[i] > b.w[i];
  return true;
}
static inline U256 u256_mul_u64(const uint64_t *a, uint64_t m) {
  U256 r; hl_u128 cy = 0;
  for (int i = 0; i < 4; i++) { cy += (hl_u128)a[i] * m; r.w[i] = (uint64_t)cy; cy >>= 64; }
  return r;
}
static inline U256 u256_shl(const U256 &a, int s) {   // 0 < s < 64
  U256 r;
  for (int i = 3; i >= 0; i--) r.w[i] = (a.w[i] << s) | (i ? a.w[i - 1] >> (64 - s) : 0);
  return r;
}

// y = floor((t*x + floor(q/2)) / q) mod t with x = CRT(res)  (PAPER.md:65 BFV decryption)
static uint64_t crt_round(const hl_ctx *c, const uint64_t *res) {
  U256 x = {{0, 0, 0, 0}}, q, hq;
  memcpy(q.w, c->q_limbs, 32); memcpy(hq.w, c->half_q_limbs, 32);
  for (uint32_t l = 0; l < c->L; l++) {
    uint64_t z = h_mulmod(res[l], c->Ml_inv[l], c->primes[l]);
    u256_add(x, u256_mul_u64(c->Ml_limbs[l], z));
  }
  while (u256_ge(x, q)) u256_sub(x, q);
  U256 num = u256_shl(x, (int)c->log2_t);
  u256_add(num, hq);
  // long division by q: quotient < 2^(log2_t + 1)
  uint64_t y = 0;
  for (int b = (int)c->log2_t; b >= 0; b--) {
    U256 qs = b ? u256_shl(q, b) : q;
    if (u256_ge(num, qs)) { u256_sub(num, qs); y |= 1ull << b; }
  }
  return y & ((1ull << c->log2_t) - 1);
}

extern "C" int hl_decrypt_share(const hl_ctx *c, const int8_t *sk, hl_tile tile,
                                const uint64_t *ct, int compress, int64_t Ma, int64_t Nb,
                                uint64_t *share) {
  if (!c || !sk || !ct || !share) return hl_fail(HL_EINVAL, "hl_decrypt_share: NULL argument");
  Geo g;
  int rc = hl_geometry(c, tile, Ma, 1, Nb, 0, -1, &g);
  if (rc) return rc;
  if ((rc = check_sk(c, sk))) return rc;
  const uint32_t N = c->N, L = c->L;
  const int m = g.m, r = g.r, n = g.n;
  const int64_t per = compress ? (int64_t)L * ((int64_t)m * n + N) : 2ll * L * N;
  std::vector<uint64_t> shat;
  sk_ntt(c, sk, shat);
  const int64_t nct = g.nI * g.nK;
#pragma omp parallel
  {
    std::vector<uint64_t> cs((size_t)L * N);
    std::vector<uint64_t> res(L);
#pragma omp for schedule(dynamic)
    for (int64_t o = 0; o < nct; o++) {
      const int64_t I = o / g.nK, K = o % g.nK;
      const uint64_t *base = ct + o * per;
      for (uint32_t l = 0; l < L; l++) {
        const uint64_t p = c->primes[l];
        // c1 arrives in evaluation form (reading C26): c1 * s = INTT(c1_hat . s_hat)
        const uint64_t *c1 = compress ? base + (size_t)L * m * n + (size_t)l * N : base + (size_t)(L + l) * N;
        uint64_t *v = &cs[(size_t)l * N];
        const uint64_t *sh = &shat[(size_t)l * N];
        for (uint32_t i = 0; i < N; i++) v[i] = h_mulmod(c1[c->brv[i]], sh[i], p);
        hl_host_ntt_inv(c, (int)l, v);
      }
      for (int k = 0; k < n; k++) {
        int64_t row = K * n + k;
        if (row >= Nb) continue;
        for (int i = 0; i < m; i++) {
          int64_t col = I * m + i;
          if (col >= Ma) continue;
          size_t pos = (size_t)k * m * r + (size_t)i * r + r - 1;
          for (uint32_t l = 0; l < L; l++) {
            uint64_t c0 = compress ? base[(size_t)l * m * n + (size_t)k * m + i] : base[(size_t)l * N + pos];
            uint64_t x = cs[(size_t)l * N + pos] + c0;
            if (x >= c->primes[l]) x -= c->primes[l];
            res[l] = x;
          }
          share[row * Ma + col] = crt_round(c, res.data());
        }
      }
    }
  }
  return HL_OK;
}
