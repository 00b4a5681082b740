// client_dev.cuh -- SURVEY.md §8(f) row f3: the client side of Alg. 1 on the GPU (PAPER.md:99, 101,
// 154; the paper's GPU BFV also covered "Encryption" and "Decryption").
// Included by kernels.cu (uses the NTT rounds, mm_d/red_d and the ChaCha PRF).  Bit-identical to
// the host client (client.cpp) and the oracle: same randomness (reading C10), same encodings.
//
//   k_encrypt   one CTA per input ciphertext g = J*nK + K, loop over the primes:
//               e = CDT(u64_E(g)) once (reading C8), a_hat_l[k] = (u[2k] + 2^64 u[2k+1]) mod p_l from
//               u64_A(g*L + l) -- the evaluation form of a (reading C26), sent as c1 --,
//               c0 = -a_l*s + e + Delta_l*pi_B(X), a_l*s = INTT(a_hat . NTT(s)).
//   k_decrypt   one CTA per output ciphertext (compressed response, "m = s c1 + c0"):
//               c1*s = INTT(c1_hat . NTT(s)) per prime (c1 arrives in evaluation form), m_l = c0 + c1*s
//               at the kept positions, then the RNS
//               rounding y = round(t x / q) mod t with x = CRT(m_l):  t x / q = sum_l m_l theta_l
//               (mod t), theta_l = t ((q/p_l)^-1 mod p_l) / p_l = I_l + F_l 2^-64 precomputed; the
//               truncation of F_l costs < L 2^-14, far inside the decryption margin (|t v / q| <
//               2^-9 for the noise v of SURVEY Appendix C), so the rounding is exact.
#pragma once

struct EncArgs {
  const uint64_t *X;            // [Nb][R] < 2^t
  int64_t Nb, R, nK;
  int m, r, n, lm, lr;
  uint64_t seed;                // private encryption seed: keys the errors (domain E)
  uint64_t a_seed;              // hl::public_seed(seed): keys the public a_hat (domain A, reading C28)
  const uint64_t *s_hat;        // [L][N] NTT(s) in slot order (hl_sk_prepare)
};

// u128 (hi, lo) mod p, canonical
__device__ __forceinline__ uint64_t mod_u128(uint64_t hi, uint64_t lo, const PrimeConsts &pc) {
  const uint64_t r1 = shoup_mul(hi, pc.r64, pc.r64_sh, pc.p);     // hi 2^64 mod p, [0, 2p)
  const uint64_t r2 = lo - __umul64hi(lo, pc.mu) * pc.p;          // lo mod p, [0, 2p)
  uint64_t r = r1 + r2;
  r = r >= pc.two_p ? r - pc.two_p : r;
  return r >= pc.p ? r - pc.p : r;
}

template <int LOGN>
__global__ void __launch_bounds__(Geom<LOGN>::NT)
k_encrypt(EncArgs E, uint64_t *__restrict__ ct, DevParams P, const uint64_t *__restrict__ cdt, uint32_t *flags) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  int8_t *e_sm = reinterpret_cast<int8_t *>(sm + Gm::SMEM_WORDS);
  uint64_t *a_nat = reinterpret_cast<uint64_t *>(sm);            // natural-order a (aliases the NTT scratch)
  const int t = threadIdx.x, L = P.L;
  const int64_t gi = blockIdx.x, J = gi / E.nK, K = gi % E.nK;
  const int mr = E.m * E.r;
  const uint64_t tmask = (1ull << P.t_bits) - 1;
  // e: discrete Gaussian by CDT from stream (E, g), 8 words per ChaCha block
#pragma unroll 1
  for (int blk = t; blk < Gm::N / 8; blk += Gm::NT) {
    uint64_t w[8];
    hl::chacha_block_u64(E.seed, hl::kDomE, (uint64_t)gi, (uint32_t)blk, w);
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const uint64_t v = w[i] & 0x7fffffffffffffffull;
      int k = 0;
      while (k < 41 && v >= __ldg(&cdt[k])) k++;
      e_sm[8 * blk + i] = (int8_t)((w[i] >> 63) ? -k : k);
    }
  }
  for (int l = 0; l < L; l++) {
    const PrimeConsts pc = pick(P, l);
    uint64_t *c0 = ct + ((size_t)gi * 2 * L + l) * Gm::N, *c1 = ct + ((size_t)gi * 2 * L + L + l) * Gm::N;
    // a_l = (u[2i] + 2^64 u[2i+1]) mod p from stream (A, g*L + l), 4 coefficients per block
#pragma unroll 1
    for (int blk = t; blk < Gm::N / 4; blk += Gm::NT) {
      uint64_t w[8];
      hl::chacha_block_u64(E.a_seed, hl::kDomA, (uint64_t)gi * L + l, (uint32_t)blk, w);
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const uint64_t a = mod_u128(w[2 * i + 1], w[2 * i], pc);
        a_nat[pad_idx(4 * blk + i)] = a;
        c1[4 * blk + i] = a;
      }
    }
    __syncthreads();
    double a[16];
    constexpr int K0 = Gm::k(0), G = 16 >> K0;
#pragma unroll
    for (int u = 0; u < 16; u++) a[u] = u2d(a_nat[pad_idx(nat_of<LOGN>(t, u))]);   // a_hat in slot order
    __syncthreads();                                   // the inverse NTT reuses the smem
    const uint64_t *sh = E.s_hat + (size_t)l * Gm::N;
#pragma unroll
    for (int u = 0; u < 16; u++)
      a[u] = red_d(mm_d(a[u], u2d(__ldg(&sh[slot_of<LOGN>(t, u)])), pc.pd, pc.pinv), pc.pd, pc.pinv);
    inv_rounds_from<LOGN, Gm::NR - 1>(a, sm, t, P.twd_inv + (size_t)l * Gm::N, pc);
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
      for (int u = 0; u < (1 << K0); u++) {
        const int idx = elem_idx<LOGN, 0>(t, g, u);
        const uint64_t as = d2u(canon_d(a[g * (1 << K0) + u], pc.pd, pc.pinv));
        // pi_B: b[k m r + j] = X[K n + k][J r + j], zero padded
        uint64_t b = 0;
        const int k = idx >> (E.lm + E.lr), j = idx & (mr - 1);
        if (k < E.n && j < E.r) {
          const int64_t row = K * E.n + k, col = J * E.r + j;
          if (row < E.Nb && col < E.R) {
            b = E.X[row * E.R + col];
            if (b & ~tmask) atomicOr(&flags[0], 1u);
          }
        }
        uint64_t v = as ? pc.p - as : 0;                              // -a*s
        const int ev = e_sm[idx];
        v += ev >= 0 ? (uint64_t)ev : pc.p - (uint64_t)(-ev);         // + e
        v = v >= pc.p ? v - pc.p : v;
        uint64_t db = shoup_mul(b & tmask, pc.delta, pc.delta_sh, pc.p);
        db = db >= pc.p ? db - pc.p : db;
        v += db;                                                      // + Delta_l b
        c0[idx] = v >= pc.p ? v - pc.p : v;
      }
    __syncthreads();                                   // smem reuse by the next prime
  }
}

struct DecArgs {
  int64_t Ma, Nb, nK;
  int m, r, n, lm, lr;
  const uint64_t *s_hat;
};

template <int LOGN>
__global__ void __launch_bounds__(Geom<LOGN>::NT)
k_decrypt(const uint64_t *__restrict__ masked, uint64_t *__restrict__ share, DecArgs D, DevParams P) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  const int L = P.L, t = threadIdx.x;
  const int mn = D.m * D.n, mr = D.m * D.r;
  uint64_t *res = reinterpret_cast<uint64_t *>(sm + Gm::SMEM_WORDS);   // [L][m n]
  const int64_t o = blockIdx.x, I = o / D.nK, K = o % D.nK;
  const uint64_t *base = masked + (size_t)o * L * (mn + Gm::N);
  for (int l = 0; l < L; l++) {
    const PrimeConsts pc = pick(P, l);
    const uint64_t *c1 = base + (size_t)L * mn + (size_t)l * Gm::N;
    double a[16];
    constexpr int K0 = Gm::k(0), G = 16 >> K0;
    load_eval_slots<LOGN>(a, c1, reinterpret_cast<uint64_t *>(sm), t, -1);   // c1_hat in slot order (C26)
    const uint64_t *sh = D.s_hat + (size_t)l * Gm::N;
#pragma unroll
    for (int u = 0; u < 16; u++)
      a[u] = red_d(mm_d(a[u], u2d(__ldg(&sh[slot_of<LOGN>(t, u)])), pc.pd, pc.pinv), pc.pd, pc.pinv);
    inv_rounds_from<LOGN, Gm::NR - 1>(a, sm, t, P.twd_inv + (size_t)l * Gm::N, pc);
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
      for (int u = 0; u < (1 << K0); u++) {
        const int idx = elem_idx<LOGN, 0>(t, g, u);
        if (idx < mr * D.n && (idx & (D.r - 1)) == D.r - 1) {        // kept position pos(i, k)
          const int kk = idx >> D.lr;                                  // = k m + i
          uint64_t x = d2u(canon_d(a[g * (1 << K0) + u], pc.pd, pc.pinv)) + base[(size_t)l * mn + kk];
          res[(size_t)l * mn + kk] = x >= pc.p ? x - pc.p : x;         // m_l = c0 + c1*s
        }
      }
    __syncthreads();
  }
  const uint64_t tmask = (1ull << P.t_bits) - 1;
  for (int kk = t; kk < mn; kk += Gm::NT) {
    const int k = kk >> D.lm, i = kk & (D.m - 1);
    const int64_t row = K * D.n + k, col = I * D.m + i;
    if (row >= D.Nb || col >= D.Ma) continue;
    uint64_t s = 0;
    hl_u128 frac = 0;
    for (int l = 0; l < L; l++) {
      const PrimeConsts pc = pick(P, l);
      const uint64_t ml = res[(size_t)l * mn + kk];
      const hl_u128 pf = (hl_u128)ml * pc.dec_F;
      s += ml * pc.dec_I + (uint64_t)(pf >> 64);
      frac += (uint64_t)pf;
    }
    s += (uint64_t)(frac >> 64) + (((uint64_t)frac) >> 63);           // carry + round half up
    share[row * D.Ma + col] = s & tmask;
  }
}

// Seeded ciphertext upload (hl_expand_seeded): c1 = a_hat_l (evaluation form, C26) of every input ciphertext regenerated from
// the client's PUBLIC seed a_seed = hl::public_seed(enc_seed) (reading C28; the private seed never reaches the server) -- the same PRF stream (A, g*L + l) and the same reduction as
// k_encrypt / the host client / the oracle (reading C10), so the expanded ciphertext is
// bit-identical to the one the client encrypted.  One thread per ChaCha block (4 coefficients).
__global__ void k_expand_a(uint64_t *__restrict__ ct, int64_t nct, int logn, uint64_t a_seed, DevParams P) {
  const int L = P.L, N = 1 << logn;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)L * (N / 4);
  if (tid >= nct * per) return;
  const int64_t gi = tid / per;
  const int l = (int)((tid % per) / (N / 4)), blk = (int)(tid % (N / 4));
  const PrimeConsts pc = pick(P, l);
  uint64_t w[8];
  hl::chacha_block_u64(a_seed, hl::kDomA, (uint64_t)gi * L + l, (uint32_t)blk, w);
  uint64_t a[4];
#pragma unroll
  for (int i = 0; i < 4; i++) a[i] = mod_u128(w[2 * i + 1], w[2 * i], pc);
  ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(ct + ((size_t)gi * 2 * L + L + l) * N + 4 * blk);
  dst[0] = make_ulonglong2(a[0], a[1]);
  dst[1] = make_ulonglong2(a[2], a[3]);
}
