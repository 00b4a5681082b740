/*
 * oracle.c -- plain, slow CPU ORACLE for the server-side homomorphic linear layer of
 * arxiv 2305.18396 (Algorithm 1; compression PAPER.md:153-154).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` legs may load this library.  It shares no code,
 * header, table or constant generator with paper_2305_18396_b200/ (the CUDA path) and
 * never includes anything from it.  All arithmetic is exact integer arithmetic with
 * `unsigned __int128` and the `%` operator -- no Shoup/Barrett, no blocking, no NTT
 * tricks on the he_matmul path (that path is the sparse schoolbook product of its
 * definition).  The readings of the paper it follows are SURVEY.md §8(c) O1-O11 and
 * the ambiguity register C1-C21, restated in DESIGN.md §3.
 *
 * Layouts (all row-major, uint64 residues canonical in [0, p_l)):
 *   X      [Nb][R]                 client share, values < 2^t_bits
 *   W      [R][Ma]                 server weights, values < 2^t_bits (two's complement)
 *   ct_in  [nJ][nK][2][L][N]       fresh ciphertexts (c0, c1) of pi_B tiles
 *   ct_out [nI][nK][2][L][N]       Enc(c) = sum_J a_IJ * ct_in[J][K]
 *   masked, compressed: [nI][nK]{ c0_kept[L][m*n], c1[L][N] }  (c0 kept index k*m+i)
 * Every ciphertext carries c0 in coefficient form and c1 in EVALUATION form (reading C26):
 *   c1_hat[k] = c1(psi_l^(2k+1)) mod p_l, k = 0..N-1 natural order = or_ntt(c1); psi_l is the
 *   oracle's root (ref.primitive_2n_root: g^((p-1)/2N), g the smallest primitive root).  The
 *   arithmetic below converts with the oracle's own or_ntt / or_intt at the boundary and keeps
 *   the definitions themselves in coefficient form.
 *   masked, full:       [nI][nK][2][L][N]
 *   share  [Nb][Ma]                server share S (the mask at the decoded positions)
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC oracle/oracle.c -o oracle/liboracle.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------------------
 * ChaCha20 block function, RFC 8439 §2.3 (the PRF of reading C10).
 * ---------------------------------------------------------------------------------- */
static uint32_t rotl32(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }

static void quarter_round(uint32_t *s, int a, int b, int c, int d) {
  s[a] += s[b]; s[d] ^= s[a]; s[d] = rotl32(s[d], 16);
  s[c] += s[d]; s[b] ^= s[c]; s[b] = rotl32(s[b], 12);
  s[a] += s[b]; s[d] ^= s[a]; s[d] = rotl32(s[d], 8);
  s[c] += s[d]; s[b] ^= s[c]; s[b] = rotl32(s[b], 7);
}

void or_chacha20_block(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3],
                       uint32_t out[16]) {
  uint32_t init[16], s[16];
  init[0] = 0x61707865u; init[1] = 0x3320646eu; init[2] = 0x79622d32u; init[3] = 0x6b206574u;
  for (int i = 0; i < 8; i++) init[4 + i] = key[i];
  init[12] = counter;
  init[13] = nonce[0]; init[14] = nonce[1]; init[15] = nonce[2];
  memcpy(s, init, sizeof(s));
  for (int round = 0; round < 10; round++) {      /* 20 rounds = 10 double rounds */
    quarter_round(s, 0, 4, 8, 12);
    quarter_round(s, 1, 5, 9, 13);
    quarter_round(s, 2, 6, 10, 14);
    quarter_round(s, 3, 7, 11, 15);
    quarter_round(s, 0, 5, 10, 15);
    quarter_round(s, 1, 6, 11, 12);
    quarter_round(s, 2, 7, 8, 13);
    quarter_round(s, 3, 4, 9, 14);
  }
  for (int i = 0; i < 16; i++) out[i] = s[i] + init[i];
}

/* u64 word `idx` of PRF stream (seed, domain, stream):
 *   key = LE64(seed) || 24 zero bytes; nonce = LE32(domain) || LE64(stream);
 *   block counter = idx / 8; u64 = LE64(keystream bytes [8*(idx%8), +8)).          (O2) */
static uint64_t prf_word(uint64_t seed, uint32_t domain, uint64_t stream, uint64_t idx) {
  uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), 0, 0, 0, 0, 0, 0};
  uint32_t nonce[3] = {domain, (uint32_t)stream, (uint32_t)(stream >> 32)};
  uint32_t blk[16];
  or_chacha20_block(key, (uint32_t)(idx / 8), nonce, blk);
  int w = (int)(idx % 8);
  return (uint64_t)blk[2 * w] | ((uint64_t)blk[2 * w + 1] << 32);
}

void or_prf_u64(uint64_t seed, uint32_t domain, uint64_t stream, uint64_t first,
                uint64_t count, uint64_t *out) {
  for (uint64_t i = 0; i < count; i++) out[i] = prf_word(seed, domain, stream, first + i);
}

enum { DOM_SK = 1, DOM_A = 2, DOM_E = 3, DOM_MASK = 4, DOM_PUB = 10 };

/* Reading C28 (the paper is silent on how the client draws its randomness,
 * PAPER.md:99): the uniform polynomials a are public (they are c1), the errors e are not.  The
 * A domain is therefore keyed by a PUBLIC seed derived one-way from the client's private
 * encryption seed, a_seed = u64 word 0 of stream (seed, PUB = 10, 0); the E domain stays keyed by
 * the private seed.  A seeded upload ships a_seed only, which does not determine e.           */
uint64_t or_public_seed(uint64_t seed) { return prf_word(seed, DOM_PUB, 0, 0); }

/* ------------------------------------------------------------------------------------
 * Samplers (O3, O4; readings C7, C8)
 * ---------------------------------------------------------------------------------- */
/* ternary secret s_i = (u64_SK[i] mod 3) - 1                                         (O3) */
void or_keygen(uint32_t N, uint64_t seed, int8_t *sk) {
  for (uint32_t i = 0; i < N; i++) sk[i] = (int8_t)((int)(prf_word(seed, DOM_SK, 0, i) % 3) - 1);
}

/* uniform a_l[i] = (u64_A[2i] + 2^64 u64_A[2i+1]) mod p_l, stream g*L + l, keyed by the
 * public seed a_seed (O4, reading C28)                                                      */
void or_sample_a(uint32_t N, uint64_t a_seed, uint64_t g, uint32_t l, uint32_t L, uint64_t p,
                 uint64_t *a) {
  for (uint32_t i = 0; i < N; i++) {
    uint64_t lo = prf_word(a_seed, DOM_A, g * L + l, 2ull * i);
    uint64_t hi = prf_word(a_seed, DOM_A, g * L + l, 2ull * i + 1);
    a[i] = (uint64_t)((((u128)hi << 64) | lo) % p);
  }
}

/* discrete Gaussian by CDT (C8): sign = u>>63, v = u & (2^63-1),
 * |e| = min{k : v < T[k]}; T[41] = 2^63 closes the table.                           (O4) */
int64_t or_cdt_sample_one(uint64_t u, const uint64_t *cdt, int ncdt) {
  uint64_t v = u & 0x7fffffffffffffffull;
  int k = 0;
  while (k < ncdt - 1 && !(v < cdt[k])) k++;
  return (u >> 63) ? -(int64_t)k : (int64_t)k;
}

void or_sample_e(uint32_t N, uint64_t seed, uint64_t g, const uint64_t *cdt, int ncdt,
                 int64_t *e) {
  for (uint32_t i = 0; i < N; i++) e[i] = or_cdt_sample_one(prf_word(seed, DOM_E, g, i), cdt, ncdt);
}

/* ------------------------------------------------------------------------------------
 * Negacyclic schoolbook product in Z_p[X]/(X^N+1)  (definition)
 *   out[k] = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j  (mod p)
 * ---------------------------------------------------------------------------------- */
void or_negacyclic_mul(uint32_t N, uint64_t p, const uint64_t *a, const uint64_t *b,
                       uint64_t *out) {
  u128 *pos = (u128 *)calloc(N, sizeof(u128));
  u128 *neg = (u128 *)calloc(N, sizeof(u128));
  for (uint32_t i = 0; i < N; i++)
    for (uint32_t j = 0; j < N; j++) {
      u128 prod = (u128)a[i] * b[j];
      if (i + j < N) pos[i + j] += prod; else neg[i + j - N] += prod;
    }
  for (uint32_t k = 0; k < N; k++) {
    uint64_t P = (uint64_t)(pos[k] % p), Q = (uint64_t)(neg[k] % p);
    out[k] = P >= Q ? P - Q : P + (p - Q);
  }
  free(pos); free(neg);
}

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)(((u128)a * b) % p); }
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t p) { uint64_t s = a + b; return s >= p ? s - p : s; }
static uint64_t submod(uint64_t a, uint64_t b, uint64_t p) { return a >= b ? a - b : a + (p - b); }
static uint64_t powmod(uint64_t b, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p; b %= p;
  while (e) { if (e & 1) r = mulmod(r, b, p); b = mulmod(b, b, p); e >>= 1; }
  return r;
}

/* ------------------------------------------------------------------------------------
 * The oracle's own scalar NTT (north_star: "a separate scalar NTT"), textbook form:
 *   NTT(a)_k = a(psi^(2k+1)) = sum_i a_i psi^i (psi^2)^(ik),  natural order.
 * Fast version: twist by psi^i, then an iterative radix-2 cyclic DFT with omega = psi^2
 * (bit-reversal permutation + butterflies).  Naive version: the defining sum, O(N^2).
 * ---------------------------------------------------------------------------------- */
void or_ntt_naive(uint32_t N, uint64_t p, uint64_t psi, const uint64_t *a, uint64_t *out) {
  for (uint32_t k = 0; k < N; k++) {
    uint64_t x = powmod(psi, 2ull * k + 1, p), acc = 0, xi = 1;
    for (uint32_t i = 0; i < N; i++) { acc = addmod(acc, mulmod(a[i], xi, p), p); xi = mulmod(xi, x, p); }
    out[k] = acc;
  }
}

static void cyclic_dft(uint32_t N, uint64_t p, uint64_t omega, uint64_t *a) {
  /* bit-reversal permutation */
  for (uint32_t i = 1, j = 0; i < N; i++) {
    uint32_t bit = N >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) { uint64_t t = a[i]; a[i] = a[j]; a[j] = t; }
  }
  for (uint32_t len = 2; len <= N; len <<= 1) {
    uint64_t wl = powmod(omega, N / len, p);
    for (uint32_t i = 0; i < N; i += len) {
      uint64_t w = 1;
      for (uint32_t j = 0; j < len / 2; j++) {
        uint64_t u = a[i + j], v = mulmod(a[i + j + len / 2], w, p);
        a[i + j] = addmod(u, v, p);
        a[i + j + len / 2] = submod(u, v, p);
        w = mulmod(w, wl, p);
      }
    }
  }
}

void or_ntt(uint32_t N, uint64_t p, uint64_t psi, const uint64_t *a, uint64_t *out) {
  uint64_t t = 1;
  for (uint32_t i = 0; i < N; i++) { out[i] = mulmod(a[i], t, p); t = mulmod(t, psi, p); }
  cyclic_dft(N, p, mulmod(psi, psi, p), out);
}

void or_intt(uint32_t N, uint64_t p, uint64_t psi, const uint64_t *ahat, uint64_t *out) {
  uint64_t psi_inv = powmod(psi, p - 2, p), n_inv = powmod(N, p - 2, p);
  memcpy(out, ahat, sizeof(uint64_t) * N);
  cyclic_dft(N, p, mulmod(psi_inv, psi_inv, p), out);
  uint64_t t = n_inv;
  for (uint32_t i = 0; i < N; i++) { out[i] = mulmod(out[i], t, p); t = mulmod(t, psi_inv, p); }
}

void or_negacyclic_mul_ntt(uint32_t N, uint64_t p, uint64_t psi, const uint64_t *a,
                           const uint64_t *b, uint64_t *out) {
  uint64_t *A = (uint64_t *)malloc(8ull * N), *B = (uint64_t *)malloc(8ull * N);
  or_ntt(N, p, psi, a, A);
  or_ntt(N, p, psi, b, B);
  for (uint32_t i = 0; i < N; i++) A[i] = mulmod(A[i], B[i], p);
  or_intt(N, p, psi, A, out);
  free(A); free(B);
}

/* ------------------------------------------------------------------------------------
 * Encodings of Alg. 1 step 1 with tile (m, r, n), padded with zeros (C2).
 * pi_B: b[k*m*r + j] = B[j][k] with B = X^T, i.e. X[K*n+k][J*r+j]        (C1, O4)
 * pi_A: a[i*r + r-1-j] = lift(A[i][j]) with A = W^T, i.e. W[J*r+j][I*m+i] (C1, C6, O5)
 * ---------------------------------------------------------------------------------- */
static int64_t lift(uint64_t w, uint32_t t_bits) {       /* centered [-t/2, t/2)  (C6) */
  uint64_t half = 1ull << (t_bits - 1);
  return w < half ? (int64_t)w : (int64_t)w - (int64_t)(1ull << t_bits);
}

static uint64_t signed_mod(int64_t v, uint64_t p) {
  return v >= 0 ? (uint64_t)v % p : (p - ((uint64_t)(-v)) % p) % p;
}

/* Secret-key BFV encryption of every pi_B tile (O4, readings C26, C28):
 *   a_hat_l = PRF keyed by or_public_seed(seed) (or_sample_a, evaluation form),  a_l = INTT(a_hat_l),
 *   e = CDT(PRF keyed by seed itself)
 *   c1 = a_hat_l (evaluation form),  c0 = -a_l * s + e + Delta_l * b   (mod p_l)             */
void or_encrypt(uint32_t N, uint32_t L, const uint64_t *primes, const uint64_t *psis,
                const uint64_t *delta_mod, uint32_t m, uint32_t r, uint32_t n, const uint64_t *X,
                int64_t Nb, int64_t R, const int8_t *sk, uint64_t seed, const uint64_t *cdt, int ncdt,
                uint64_t *ct_in) {
  int64_t nJ = (R + r - 1) / r, nK = (Nb + n - 1) / n;
  const uint64_t a_seed = or_public_seed(seed);
#pragma omp parallel for schedule(dynamic)
  for (int64_t g = 0; g < nJ * nK; g++) {
    int64_t J = g / nK, K = g % nK;
    uint64_t *b = (uint64_t *)calloc(N, 8);
    int64_t *e = (int64_t *)malloc(8ull * N);
    uint64_t *a = (uint64_t *)malloc(8ull * N), *a_hat = (uint64_t *)malloc(8ull * N);
    u128 *pos = (u128 *)malloc(sizeof(u128) * N), *neg = (u128 *)malloc(sizeof(u128) * N);
    for (uint32_t k = 0; k < n; k++)
      for (uint32_t j = 0; j < r; j++) {
        int64_t row = K * n + k, col = J * (int64_t)r + j;
        if (row < Nb && col < R) b[(uint64_t)k * m * r + j] = X[row * R + col];
      }
    or_sample_e(N, seed, (uint64_t)g, cdt, ncdt, e);
    for (uint32_t l = 0; l < L; l++) {
      uint64_t p = primes[l];
      or_sample_a(N, a_seed, (uint64_t)g, l, L, p, a_hat);
      or_intt(N, p, psis[l], a_hat, a);
      /* a * s, schoolbook over the ternary s */
      memset(pos, 0, sizeof(u128) * N); memset(neg, 0, sizeof(u128) * N);
      for (uint32_t j = 0; j < N; j++) {
        if (sk[j] == 0) continue;
        for (uint32_t i = 0; i < N; i++) {
          int up = (i + j < N);
          uint32_t k = up ? i + j : i + j - N;
          int plus = (sk[j] > 0) == up;        /* sign of a_i s_j x^{i+j} after x^N = -1 */
          if (plus) pos[k] += a[i]; else neg[k] += a[i];
        }
      }
      uint64_t *c0 = ct_in + ((uint64_t)g * 2 + 0) * L * N + (uint64_t)l * N;
      uint64_t *c1 = ct_in + ((uint64_t)g * 2 + 1) * L * N + (uint64_t)l * N;
      for (uint32_t k = 0; k < N; k++) {
        uint64_t as = submod((uint64_t)(pos[k] % p), (uint64_t)(neg[k] % p), p);
        uint64_t v = submod(0, as, p);
        v = addmod(v, signed_mod(e[k], p), p);
        v = addmod(v, mulmod(delta_mod[l], b[k] % p, p), p);
        c0[k] = v;
        c1[k] = a_hat[k];
      }
    }
    free(b); free(e); free(a); free(a_hat); free(pos); free(neg);
  }
}

/* he_matmul, definition (i) of SURVEY.md §8(c):
 *   ct_out[I][K][c] = sum_J a_IJ * ct_in[J][K][c]  mod (X^N+1, p_l)
 * as a sparse schoolbook product: a_IJ has at most m*r nonzero coefficients.   (O6)   */
void or_he_matmul(uint32_t N, uint32_t L, const uint64_t *primes, const uint64_t *psis, uint32_t m,
                  uint32_t r, uint32_t n, uint32_t t_bits, const uint64_t *W, int64_t R, int64_t Ma,
                  int64_t Nb, const uint64_t *ct_in_eval, uint64_t *ct_out) {
  int64_t nI = (Ma + m - 1) / m, nJ = (R + r - 1) / r, nK = (Nb + n - 1) / n;
  /* boundary (reading C26): c1 halves to coefficient form */
  uint64_t *ct_in = (uint64_t *)malloc(8ull * nJ * nK * 2 * L * N);
  memcpy(ct_in, ct_in_eval, 8ull * nJ * nK * 2 * L * N);
#pragma omp parallel for schedule(dynamic)
  for (int64_t w = 0; w < nJ * nK * (int64_t)L; w++) {
    uint64_t *x = ct_in + ((uint64_t)(w / L) * 2 + 1) * L * N + (uint64_t)(w % L) * N;
    or_intt(N, primes[w % L], psis[w % L], ct_in_eval + (x - ct_in), x);
  }
  /* independent work items: (output tile (I, K), component c, prime l) */
#pragma omp parallel for schedule(dynamic)
  for (int64_t w = 0; w < nI * nK * 2 * (int64_t)L; w++) {
    int64_t o = w / (2 * L), I = o / nK, K = o % nK;
    int c = (int)((w / L) % 2);
    uint32_t l = (uint32_t)(w % L);
    uint64_t p = primes[l];
    u128 *pos = (u128 *)calloc(N, sizeof(u128)), *neg = (u128 *)calloc(N, sizeof(u128));
    for (int64_t J = 0; J < nJ; J++) {
      const uint64_t *x = ct_in + ((uint64_t)(J * nK + K) * 2 + c) * L * N + (uint64_t)l * N;
      for (uint32_t i = 0; i < m; i++)
        for (uint32_t j = 0; j < r; j++) {
          int64_t row = J * (int64_t)r + j, col = I * (int64_t)m + i;
          if (row >= R || col >= Ma) continue;
          uint64_t val = signed_mod(lift(W[row * Ma + col], t_bits), p);
          if (val == 0) continue;
          uint32_t e = i * r + r - 1 - j;          /* exponent of a_ij in pi_A */
          for (uint32_t s = 0; s < N; s++) {
            u128 prod = (u128)val * x[s];
            if (s + e < N) pos[s + e] += prod; else neg[s + e - N] += prod;
          }
        }
    }
    uint64_t *y = ct_out + ((uint64_t)(I * nK + K) * 2 + c) * L * N + (uint64_t)l * N;
    for (uint32_t k = 0; k < N; k++)
      y[k] = submod((uint64_t)(pos[k] % p), (uint64_t)(neg[k] % p), p);
    if (c == 1) {                                  /* boundary (C26): c1 to evaluation form */
      uint64_t *tmp = (uint64_t *)malloc(8ull * N);
      or_ntt(N, p, psis[l], y, tmp);
      memcpy(y, tmp, 8ull * N);
      free(tmp);
    }
    free(pos); free(neg);
  }
  free(ct_in);
}

/* Same definition evaluated through the oracle's own scalar NTT (or_ntt / or_intt):
 * used to cross-check the schoolbook path and to time larger samples.  Only the output
 * tiles listed in `tiles` (pairs I, K) are computed, written in list order to ct_out. */
void or_he_matmul_ntt_tiles(uint32_t N, uint32_t L, const uint64_t *primes, const uint64_t *psis,
                            uint32_t m, uint32_t r, uint32_t n, uint32_t t_bits,
                            const uint64_t *W, int64_t R, int64_t Ma, int64_t Nb,
                            const uint64_t *ct_in, const int64_t *tiles, int64_t ntiles,
                            uint64_t *ct_out) {
  int64_t nJ = (R + r - 1) / r, nK = (Nb + n - 1) / n;
#pragma omp parallel for schedule(dynamic)
  for (int64_t o = 0; o < ntiles; o++) {
    int64_t I = tiles[2 * o], K = tiles[2 * o + 1];
    uint64_t *apoly = (uint64_t *)malloc(8ull * N), *ahat = (uint64_t *)malloc(8ull * N);
    uint64_t *xhat = (uint64_t *)malloc(8ull * N), *acc = (uint64_t *)malloc(8ull * N);
    for (int c = 0; c < 2; c++)
      for (uint32_t l = 0; l < L; l++) {
        uint64_t p = primes[l];
        memset(acc, 0, 8ull * N);
        for (int64_t J = 0; J < nJ; J++) {
          memset(apoly, 0, 8ull * N);
          for (uint32_t i = 0; i < m; i++)
            for (uint32_t j = 0; j < r; j++) {
              int64_t row = J * (int64_t)r + j, col = I * (int64_t)m + i;
              if (row < R && col < Ma)
                apoly[i * r + r - 1 - j] = signed_mod(lift(W[row * Ma + col], t_bits), p);
            }
          or_ntt(N, p, psis[l], apoly, ahat);
          const uint64_t *x = ct_in + ((uint64_t)(J * nK + K) * 2 + c) * L * N + (uint64_t)l * N;
          if (c == 0) or_ntt(N, p, psis[l], x, xhat);
          else memcpy(xhat, x, 8ull * N);            /* c1 is in evaluation form (C26) */
          for (uint32_t k = 0; k < N; k++) acc[k] = addmod(acc[k], mulmod(ahat[k], xhat[k], p), p);
        }
        uint64_t *y = ct_out + ((uint64_t)o * 2 + c) * L * N + (uint64_t)l * N;
        if (c == 0) or_intt(N, p, psis[l], acc, y);
        else memcpy(y, acc, 8ull * N);
      }
    free(apoly); free(ahat); free(xhat); free(acc);
  }
}

/* Reading C27: the mask word of coefficient position pos.  The kept positions
 * pos(i,k) = (k*m + i)*r + r-1 (all p < m*r*n with p = r-1 mod r) take words 0 .. m*n-1 in
 * kept-index order k*m + i; every other position takes the next word in increasing position
 * order, i.e. m*n + (pos - #kept positions below pos).  A permutation of [0, N).             */
uint64_t or_mask_word(uint32_t m, uint32_t r, uint32_t n, uint64_t pos) {
  uint64_t mn = (uint64_t)m * n, mrn = mn * r;
  if (pos < mrn && pos % r == r - 1) return pos / r;
  return mn + pos - (pos < mrn ? pos / r : mn);
}

/* Alg. 1 step 3 + §3.1.3 (O7-O9; readings C3, C10-C12, C27) for ONE output ciphertext (I, K):
 *   sigma[pos] = u64_MASK(stream I*nK+K)[or_mask_word(pos)] & (2^t_bits - 1)
 *   c0 <- c0 - Delta_l * sigma (mod p_l);  keep c1, keep c0 at pos(i,k) = k*m*r + i*r + r-1
 * Writes the masked ciphertext to dst and sigma at the kept positions (index k*m+i) to kept. */
static void mask_one(uint32_t N, uint32_t L, const uint64_t *primes, const uint64_t *delta_mod,
                     uint32_t t_bits, uint32_t m, uint32_t r, uint32_t n, uint64_t stream,
                     const uint64_t *src, uint64_t seed, int compress, uint64_t *dst, uint64_t *kept) {
  uint64_t tmask = (t_bits == 64) ? ~0ull : ((1ull << t_bits) - 1);
  uint64_t *sigma = (uint64_t *)malloc(8ull * N), *words = (uint64_t *)malloc(8ull * N);
  or_prf_u64(seed, DOM_MASK, stream, 0, N, words);
  for (uint32_t i = 0; i < N; i++) sigma[i] = words[or_mask_word(m, r, n, i)] & tmask;
  free(words);
  for (uint32_t l = 0; l < L; l++) {
    uint64_t p = primes[l];
    const uint64_t *c0 = src + (uint64_t)l * N, *c1 = src + (uint64_t)(L + l) * N;
    if (compress) {
      for (uint32_t k = 0; k < n; k++)
        for (uint32_t i = 0; i < m; i++) {
          uint32_t pos = k * m * r + i * r + r - 1;
          dst[(uint64_t)l * m * n + k * m + i] = submod(c0[pos], mulmod(delta_mod[l], sigma[pos] % p, p), p);
        }
      memcpy(dst + (uint64_t)L * m * n + (uint64_t)l * N, c1, 8ull * N);
    } else {
      for (uint32_t s = 0; s < N; s++)
        dst[(uint64_t)l * N + s] = submod(c0[s], mulmod(delta_mod[l], sigma[s] % p, p), p);
      memcpy(dst + (uint64_t)(L + l) * N, c1, 8ull * N);
    }
  }
  for (uint32_t k = 0; k < n; k++)
    for (uint32_t i = 0; i < m; i++) kept[k * m + i] = sigma[k * m * r + i * r + r - 1];
  free(sigma);
}

/* Whole problem: every (I, K); server share S[K*n+k][I*m+i] = sigma[pos(i,k)] in range. */
void or_mask_and_share(uint32_t N, uint32_t L, const uint64_t *primes, const uint64_t *delta_mod,
                       uint32_t t_bits, uint32_t m, uint32_t r, uint32_t n, int64_t Ma, int64_t Nb,
                       const uint64_t *ct_out, uint64_t seed, int compress, uint64_t *ct_masked,
                       uint64_t *share) {
  int64_t nI = (Ma + m - 1) / m, nK = (Nb + n - 1) / n;
  uint64_t per_ct = compress ? (uint64_t)L * (m * n + N) : 2ull * L * N;
#pragma omp parallel for schedule(dynamic)
  for (int64_t o = 0; o < nI * nK; o++) {
    int64_t I = o / nK, K = o % nK;
    uint64_t *kept = (uint64_t *)malloc(8ull * m * n);
    mask_one(N, L, primes, delta_mod, t_bits, m, r, n, (uint64_t)o, ct_out + (uint64_t)o * 2 * L * N,
             seed, compress, ct_masked + (uint64_t)o * per_ct, kept);
    for (uint32_t k = 0; k < n; k++)
      for (uint32_t i = 0; i < m; i++) {
        int64_t row = K * n + k, col = I * (int64_t)m + i;
        if (row < Nb && col < Ma) share[row * Ma + col] = kept[k * m + i];
      }
    free(kept);
  }
}

/* Selected output tiles only (for sampled parity at full size): tiles = pairs (I, K) with
 * global I; ct [ntiles][2][L][N] -> masked [ntiles][per_ct], kept sigma [ntiles][m*n].       */
void or_mask_tiles(uint32_t N, uint32_t L, const uint64_t *primes, const uint64_t *delta_mod,
                   uint32_t t_bits, uint32_t m, uint32_t r, uint32_t n, int64_t nK,
                   const uint64_t *ct, const int64_t *tiles, int64_t ntiles, uint64_t seed,
                   int compress, uint64_t *masked, uint64_t *kept) {
  uint64_t per_ct = compress ? (uint64_t)L * (m * n + N) : 2ull * L * N;
#pragma omp parallel for schedule(dynamic)
  for (int64_t o = 0; o < ntiles; o++)
    mask_one(N, L, primes, delta_mod, t_bits, m, r, n, (uint64_t)(tiles[2 * o] * nK + tiles[2 * o + 1]),
             ct + (uint64_t)o * 2 * L * N, seed, compress, masked + (uint64_t)o * per_ct,
             kept + (uint64_t)o * m * n);
}

/* Decryption core ("m = s*c1 + c0"), per prime, at the decoded positions
 * pos(i,k) only: x_l = c0[pos] + (c1 * s)[pos]  (mod p_l).  The CRT and the rounding
 * y = floor((t*x + floor(q/2)) / q) mod t are done with Python integers (oracle/ref.py). (O10)
 * Output layout: x [nI][nK][L][m*n] (index k*m + i).                                     */
void or_decrypt_residues(uint32_t N, uint32_t L, const uint64_t *primes, const uint64_t *psis, uint32_t m,
                         uint32_t r, uint32_t n, int64_t Ma, int64_t Nb, const int8_t *sk,
                         const uint64_t *ct_masked, int compress, uint64_t *x) {
  int64_t nI = (Ma + m - 1) / m, nK = (Nb + n - 1) / n;
  uint64_t per_ct = compress ? (uint64_t)L * (m * n + N) : 2ull * L * N;
#pragma omp parallel for schedule(dynamic)
  for (int64_t o = 0; o < nI * nK; o++) {
    const uint64_t *ct = ct_masked + (uint64_t)o * per_ct;
    uint64_t *c1 = (uint64_t *)malloc(8ull * N);
    for (uint32_t l = 0; l < L; l++) {
      uint64_t p = primes[l];
      /* c1 from evaluation form (C26) */
      or_intt(N, p, psis[l], compress ? ct + (uint64_t)L * m * n + (uint64_t)l * N : ct + (uint64_t)(L + l) * N, c1);
      for (uint32_t k = 0; k < n; k++)
        for (uint32_t i = 0; i < m; i++) {
          uint32_t pos = k * m * r + i * r + r - 1;
          uint64_t c0 = compress ? ct[(uint64_t)l * m * n + k * m + i] : ct[(uint64_t)l * N + pos];
          /* (c1 * s)[pos] = sum_{j<=pos} c1[j] s[pos-j] - sum_{j>pos} c1[j] s[pos-j+N] */
          u128 P = 0, Q = 0;
          for (uint32_t j = 0; j < N; j++) {
            int sv; int up = (j <= pos);
            sv = up ? sk[pos - j] : sk[pos + N - j];
            if (sv == 0) continue;
            if ((sv > 0) == up) P += c1[j]; else Q += c1[j];
          }
          uint64_t v = submod((uint64_t)(P % p), (uint64_t)(Q % p), p);
          x[((uint64_t)o * L + l) * m * n + k * m + i] = addmod(v, c0, p);
        }
    }
    free(c1);
  }
}

/* Full decryption residues of every coefficient (for noise measurements and the
 * "compressed decrypt equals full decrypt" pin): x [nct][L][N] = c0 + c1*s (mod p_l). */
void or_decrypt_full_residues(uint32_t N, uint32_t L, const uint64_t *primes, const uint64_t *psis,
                              const int8_t *sk, const uint64_t *ct, int64_t nct, uint64_t *x) {
#pragma omp parallel for schedule(dynamic)
  for (int64_t o = 0; o < nct; o++)
    for (uint32_t l = 0; l < L; l++) {
      uint64_t p = primes[l];
      const uint64_t *c0 = ct + ((uint64_t)o * 2 + 0) * L * N + (uint64_t)l * N;
      uint64_t *c1 = (uint64_t *)malloc(8ull * N);      /* c1 from evaluation form (C26) */
      or_intt(N, p, psis[l], ct + ((uint64_t)o * 2 + 1) * L * N + (uint64_t)l * N, c1);
      u128 *pos = (u128 *)calloc(N, sizeof(u128)), *neg = (u128 *)calloc(N, sizeof(u128));
      for (uint32_t j = 0; j < N; j++) {
        if (sk[j] == 0) continue;
        for (uint32_t i = 0; i < N; i++) {
          int up = (i + j < N);
          uint32_t k = up ? i + j : i + j - N;
          if ((sk[j] > 0) == up) pos[k] += c1[i]; else neg[k] += c1[i];
        }
      }
      for (uint32_t k = 0; k < N; k++)
        x[((uint64_t)o * L + l) * N + k] =
            addmod(submod((uint64_t)(pos[k] % p), (uint64_t)(neg[k] % p), p), c0[k], p);
      free(pos); free(neg); free(c1);
    }
}
