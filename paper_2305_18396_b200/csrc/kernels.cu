// kernels.cu -- sm_100a kernels and device entry points of libhelinear.
//
// The server path of Alg. 1 with the GPU cipher-plain multiply of
// PAPER.md:155-156 ("Multiplication of polynomials is done by NTT and elementwise
// multiplication"), redesigned for B200 integer pipes:
//
//   encode_weights : pi_A scatter + centered lift + forward NTT  -> wcache (25-bit limb pairs)
//   he_matmul      : forward NTT of ct_in -> slot-parallel modular MAC over J -> inverse NTT
//   mask_and_share : ChaCha20 mask, c0 -= Delta*sigma, drop unused c0, shares
//   he_matmul_share: the inverse NTT fused with the masking/compression epilogue
//
// NTT: negacyclic, merged-psi Cooley-Tukey forward / Gentleman-Sande inverse on the FP64
// pipe (exact modular products by error-free DFMA transformations, signed lazy residues,
// reductions every second stage; see mm_d / red_d).  One CTA per
// polynomial, N/16 threads holding 16 coefficients each; radix-16 rounds in registers with
// padded shared-memory transposes between rounds.  NTT-domain slot order is internal:
// slot P(idx) = (idx & 15) * (N/16) + (idx >> 4) of the bit-reversed CT output index, which
// makes both the last forward round and the first inverse round fully coalesced.
//
// MAC: per (prime, slot) a small GEMM out[I][col] = sum_J W[I][J] * X[J][col] mod p.
// Operands are stored as 25-bit limb pairs (x = x0 + 2^25 x1); each modular MAC costs three
// IMAD.WIDE.U32 (Karatsuba: x0*y0, x1*y1, (x0+x1)(y0+y1)) into three exact 64-bit lazy
// accumulators; one 128-bit reduction per output.
#include <cuda.h>   // CUtensorMap (the MAC's c1 loads; encoded through the runtime's driver entry point)
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: named ranges for nsys / Nsight timelines

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>
#include <string>
#include <vector>

#include "chacha.h"
#include "hl_internal.h"

namespace {

constexpr uint32_t kLimbBits = 25;
constexpr uint32_t kLimbMask = (1u << kLimbBits) - 1;
constexpr int kMacJChunk = 4096;   // (2^26)^2 * 4096 = 2^64: exact 64-bit lazy accumulation bound

// ---------------------------------------------------------------------------------------
// modular helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t shoup_mul(uint64_t x, uint64_t w, uint64_t wsh, uint64_t p) {
  const uint64_t q = __umul64hi(x, wsh);
  return x * w - q * p;   // in [0, 2p) for any x < 2^64
}

// ---------------------------------------------------------------------------------------
// Exact modular arithmetic on the FP64 pipe (DFMA 57 /clk/SM vs 24 for the
// IMAD.WIDE a 64-bit Shoup product needs).  Residues are integer-valued doubles, signed and
// lazily reduced; every intermediate below is an integer of magnitude < 2^53, hence exact.
//   mm_d(y, w):  h = y w (rounded), l = fma(y, w, -h) (exact: y w = h + l),
//                q = rint(h / p) via the 1.5*2^52 magic, r = fma(-q, p, h) (exact), return r + l.
//                Requires |y| < 2^51 and 0 <= w < p; |h/p - q| <= 0.75 so |result| < p.
//   red_d(v):    v - p * rint(v / p), |result| <= p/2 (+ tiny) for |v| < 2^51.
// ---------------------------------------------------------------------------------------
constexpr double kMagic = 6755399441055744.0;            // 1.5 * 2^52
constexpr double kTwo52 = 4503599627370496.0;            // 2^52

__device__ __forceinline__ double mm_d(double y, double w, double p, double pinv) {
  const double h = __dmul_rn(y, w);
  const double l = __fma_rn(y, w, -h);
  const double q = __dsub_rn(__fma_rn(h, pinv, kMagic), kMagic);
  const double r = __fma_rn(-q, p, h);
  return __dadd_rn(r, l);
}

__device__ __forceinline__ double red_d(double v, double p, double pinv) {
  const double q = __dsub_rn(__fma_rn(v, pinv, kMagic), kMagic);
  return __fma_rn(-q, p, v);
}

// [0, 2^52) integer <-> double without the conversion unit
__device__ __forceinline__ double u2d(uint64_t x) {
  return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), kTwo52);
}
__device__ __forceinline__ uint64_t d2u(double v) {      // v integer-valued in [0, 2^52)
  return (uint64_t)__double_as_longlong(__dadd_rn(v, kTwo52)) - 0x4330000000000000ull;
}
// canonical residue in [0, p) as an integer-valued double, from |v| < 2^51
__device__ __forceinline__ double canon_d(double v, double p, double pinv) {
  const double r = red_d(v, p, pinv);
  return r < 0.0 ? __dadd_rn(r, p) : r;
}

__device__ __forceinline__ PrimeConsts pick(const DevParams &P, int l) {
  PrimeConsts c = P.pc[0];
  if (l == 1) c = P.pc[1];
  if (l == 2) c = P.pc[2];
  return c;
}

// mbarrier / bulk-copy (TMA) helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// bulk prefetch of [src, src + bytes) into L2 (no completion tracking; bytes a multiple of 16)
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------------------------------
// NTT round geometry.  Rounds cover the stages [S0, S0+K) of the log2(N) CT stages; round 0
// is the short one when log2(N) is not a multiple of 4.  A thread holds G = 16 >> K groups of
// 2^K coefficients; the coefficient (g, u) of thread t has bit-reversed-order index idx.
// ---------------------------------------------------------------------------------------
template <int LOGN>
struct Geom {
  static constexpr int N = 1 << LOGN;
  static constexpr int NT = N / 16;
  static constexpr int K0 = (LOGN % 4) ? (LOGN % 4) : 4;
  static constexpr int NR = (LOGN - K0) / 4 + 1;
  static constexpr int SMEM_WORDS = N + N / 16;
  __host__ __device__ static constexpr int s0(int r) { return r == 0 ? 0 : K0 + 4 * (r - 1); }
  __host__ __device__ static constexpr int k(int r) { return r == 0 ? K0 : 4; }
  __host__ __device__ static constexpr int lo(int r) { return LOGN - s0(r) - k(r); }
};

template <int LOGN, int R>
__device__ __forceinline__ int elem_idx(int t, int g, int u) {
  using Gm = Geom<LOGN>;
  constexpr int K = Gm::k(R), LO = Gm::lo(R);
  const int gid = t + g * Gm::NT;
  return ((gid >> LO) << (LO + K)) | (u << LO) | (gid & ((1 << LO) - 1));
}

__device__ __forceinline__ int pad_idx(int idx) { return idx + (idx >> 4); }

template <int LOGN, int R>
__device__ __forceinline__ void to_smem(const double (&a)[16], double *sm, int t) {
  constexpr int K = Geom<LOGN>::k(R), G = 16 >> K;
#pragma unroll
  for (int g = 0; g < G; g++)
#pragma unroll
    for (int u = 0; u < (1 << K); u++) sm[pad_idx(elem_idx<LOGN, R>(t, g, u))] = a[g * (1 << K) + u];
}

template <int LOGN, int R>
__device__ __forceinline__ void from_smem(double (&a)[16], const double *sm, int t) {
  constexpr int K = Geom<LOGN>::k(R), G = 16 >> K;
#pragma unroll
  for (int g = 0; g < G; g++)
#pragma unroll
    for (int u = 0; u < (1 << K); u++) a[g * (1 << K) + u] = sm[pad_idx(elem_idx<LOGN, R>(t, g, u))];
}

// All twiddles of round R for thread t, loaded up front (issued before the round's smem exchange
// so that their L1/L2 latency overlaps it): wv[g (2^K - 1) + 2^ls - 1 + (u >> (K - ls))].
template <int LOGN, int R>
__device__ __forceinline__ void load_round_tw(double (&wv)[15], int t, const double *tw) {
  using Gm = Geom<LOGN>;
  constexpr int S0 = Gm::s0(R), K = Gm::k(R), LO = Gm::lo(R), G = 16 >> K;
#pragma unroll
  for (int g = 0; g < G; g++) {
    const int gid_high = (t + g * Gm::NT) >> LO;
#pragma unroll
    for (int ls = 0; ls < K; ls++)
#pragma unroll
      for (int j = 0; j < (1 << ls); j++)
        wv[g * ((1 << K) - 1) + (1 << ls) - 1 + j] = __ldg(&tw[(1 << (S0 + ls)) + (gid_high << ls) + j]);
  }
}

// Forward CT stages of round R.  Twiddle of a pair whose lower index is idx at stage st:
// psi^bitrev((1<<st) + (idx >> (LOGN - st))); within a round that is
// (1<<st) + (gid_high << ls) + (u >> (K - ls)).
// Values: |v| <= p at entry of stage 0 (canonical input) or <= p/2 after a reduction; a CT
// stage adds < p, so every value is reduced (red_d) after each odd stage: multiplicands stay
// below 2p < 2^51 as mm_d requires.
template <int LOGN, int R>
__device__ __forceinline__ void fwd_round(double (&a)[16], const double (&wv)[15], double p, double pinv) {
  using Gm = Geom<LOGN>;
  constexpr int S0 = Gm::s0(R), K = Gm::k(R), G = 16 >> K;
#pragma unroll
  for (int ls = 0; ls < K; ls++) {
    const int st = S0 + ls;
    const int half = 1 << (K - 1 - ls);
#pragma unroll
    for (int g = 0; g < G; g++) {
#pragma unroll
      for (int u = 0; u < (1 << K); u++) {
        if (u & half) continue;
        const double w = wv[g * ((1 << K) - 1) + (1 << ls) - 1 + (u >> (K - ls))];
        double &X = a[g * (1 << K) + u], &Y = a[g * (1 << K) + u + half];
        const double T = mm_d(Y, w, p, pinv);
        Y = __dsub_rn(X, T);
        X = __dadd_rn(X, T);
      }
    }
    if (st & 1) {
#pragma unroll
      for (int i = 0; i < 16; i++) a[i] = red_d(a[i], p, pinv);
    }
  }
}

// Inverse GS stages of round R (stages descending); N^-1 is folded into stage 0.  Inputs must
// satisfy |v| <= p/2; a GS stage keeps |Y'| < p and |X'| <= 2 max|v|, so values are reduced
// after every second stage (counted from the top, stage LOGN-1) -- differences stay < 2p.
template <int LOGN, int R>
__device__ __forceinline__ void inv_round(double (&a)[16], const double (&wv)[15], const PrimeConsts &pc) {
  using Gm = Geom<LOGN>;
  constexpr int S0 = Gm::s0(R), K = Gm::k(R), G = 16 >> K;
  const double p = pc.pd, pinv = pc.pinv;
#pragma unroll
  for (int ls = K - 1; ls >= 0; ls--) {
    const int st = S0 + ls;
    const int half = 1 << (K - 1 - ls);
#pragma unroll
    for (int g = 0; g < G; g++) {
#pragma unroll
      for (int u = 0; u < (1 << K); u++) {
        if (u & half) continue;
        double &X = a[g * (1 << K) + u], &Y = a[g * (1 << K) + u + half];
        const double s = __dadd_rn(X, Y), d = __dsub_rn(X, Y);
        if (st == 0) {
          // last stage: (X, Y) -> ((X+Y) N^-1, (X-Y) psi^-bitrev(1) N^-1)
          X = mm_d(s, pc.ninv_d, p, pinv);
          Y = mm_d(d, pc.ninv_w1_d, p, pinv);
        } else {
          const double w = wv[g * ((1 << K) - 1) + (1 << ls) - 1 + (u >> (K - ls))];
          X = s;
          Y = mm_d(d, w, p, pinv);
        }
      }
    }
    if (st > 0 && ((LOGN - 1 - st) & 1)) {
#pragma unroll
      for (int i = 0; i < 16; i++) a[i] = red_d(a[i], p, pinv);
    }
  }
}

// exchange barrier of one transform: the whole CTA (bar < 0) or named barrier `bar` over the
// transform's NT threads (several transforms per CTA synchronise independently)
template <int LOGN>
__device__ __forceinline__ void xsync(int bar) {
  if (bar < 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(Geom<LOGN>::NT) : "memory");
}

template <int LOGN, int R>
__device__ __forceinline__ void fwd_rounds_from(double (&a)[16], double *sm, int t, const double *tw,
                                                double p, double pinv, int bar = -1) {
  if constexpr (R < Geom<LOGN>::NR) {
    double wv[15];
    load_round_tw<LOGN, R>(wv, t, tw);               // in flight during the smem exchange
    if constexpr (R > 0) {
      to_smem<LOGN, R - 1>(a, sm, t);
      xsync<LOGN>(bar);
      from_smem<LOGN, R>(a, sm, t);
      xsync<LOGN>(bar);
    }
    fwd_round<LOGN, R>(a, wv, p, pinv);
    fwd_rounds_from<LOGN, R + 1>(a, sm, t, tw, p, pinv, bar);
  }
}

// two independent transforms (same prime) in the same threads: shared twiddles, one pair of
// barriers per exchange for both, twice the independent butterflies per stage
template <int LOGN, int R>
__device__ __forceinline__ void fwd_rounds_from2(double (&a)[16], double (&b)[16], double *sma, double *smb, int t,
                                                 const double *tw, double p, double pinv) {
  if constexpr (R < Geom<LOGN>::NR) {
    double wv[15];
    load_round_tw<LOGN, R>(wv, t, tw);
    if constexpr (R > 0) {
      to_smem<LOGN, R - 1>(a, sma, t);
      to_smem<LOGN, R - 1>(b, smb, t);
      __syncthreads();
      from_smem<LOGN, R>(a, sma, t);
      from_smem<LOGN, R>(b, smb, t);
      __syncthreads();
    }
    fwd_round<LOGN, R>(a, wv, p, pinv);
    fwd_round<LOGN, R>(b, wv, p, pinv);
    fwd_rounds_from2<LOGN, R + 1>(a, b, sma, smb, t, tw, p, pinv);
  }
}

template <int LOGN, int R>
__device__ __forceinline__ void inv_rounds_from(double (&a)[16], double *sm, int t, const double *tw,
                                                const PrimeConsts &pc) {
  if constexpr (R >= 0) {
    double wv[15];
    if constexpr (R < Geom<LOGN>::NR - 1) {
      to_smem<LOGN, R + 1>(a, sm, t);
      __syncthreads();
      from_smem<LOGN, R>(a, sm, t);
      __syncthreads();
    }
    load_round_tw<LOGN, R>(wv, t, tw);
    inv_round<LOGN, R>(a, wv, pc);
    inv_rounds_from<LOGN, R - 1>(a, sm, t, tw, pc);
  }
}

// slot position of the bit-reversed CT index held by the last forward round (lo = 0, K = 4)
template <int LOGN>
__device__ __forceinline__ int slot_of(int t, int u) { return u * Geom<LOGN>::NT + t; }

// Evaluation form at the boundary (reading C26): register u of thread t in slot order holds the
// CT index idx = 16 t + u, i.e. the evaluation at psi^(2k+1) with natural k = bitrev(idx).
template <int LOGN>
__device__ __forceinline__ int nat_of(int t, int u) { return (int)(__brev((unsigned)(16 * t + u)) >> (32 - LOGN)); }

// c1 of a ciphertext (evaluation form, natural order, canonical) -> registers in slot order:
// coalesced copy through shared memory `stg` (N + N/16 u64, padded, free on entry), then the bit-reversal
// gather; `stg` is free again on return.  `bar` as xsync.
template <int LOGN>
__device__ __forceinline__ void load_eval_slots(double (&a)[16], const uint64_t *src, uint64_t *stg, int t, int bar) {
  using Gm = Geom<LOGN>;
#pragma unroll
  for (int j = 0; j < 16; j++) stg[pad_idx(t + j * Gm::NT)] = __ldcs(src + t + j * Gm::NT);
  xsync<LOGN>(bar);
#pragma unroll
  for (int u = 0; u < 16; u++) a[u] = u2d(stg[pad_idx(nat_of<LOGN>(t, u))]);   // padded: no bank conflicts
  xsync<LOGN>(bar);
}

// registers in slot order (canonical residues) -> natural evaluation order in global memory
// (reading C26), through `stg` (N u64, free on entry and on return)
template <int LOGN>
__device__ __forceinline__ void store_eval_slots(const uint64_t (&x)[16], uint64_t *dst, uint64_t *stg, int t, int bar) {
  using Gm = Geom<LOGN>;
#pragma unroll
  for (int u = 0; u < 16; u++) stg[pad_idx(nat_of<LOGN>(t, u))] = x[u];
  xsync<LOGN>(bar);
#pragma unroll
  for (int j = 0; j < 16; j++) dst[t + j * Gm::NT] = stg[pad_idx(t + j * Gm::NT)];
  xsync<LOGN>(bar);
}

// ---------------------------------------------------------------------------------------
// MAC operand layouts in HBM (NTT domain, 25-bit limb pairs).  Both are blocked
// so that the operands of one (tile, J) step of the MAC kernel are ONE contiguous chunk each,
// fetched by a single bulk (TMA) copy:
//   W cache   [nIb][nSb][nJ][32 slots][16 rows] uint2            nIb = ceil(nIs/16), nSb = L*N/32
//   X (ct_in) [nSb][nCg][nJ]{ [32 slots][CW cols] uint2 limb pairs, [32 slots][CW cols] u32 x0+x1 }
//             CW in {8,4,2} divides nC, nCg = nC/CW; the limb sums of X (Karatsuba middle term)
//             are stored so that the MAC's integer-multiply pipe only multiplies.
// slot s = l*N + P(idx) (prime-major), rows = I tiles of the shard, cols = K*2 + c.
// ---------------------------------------------------------------------------------------
struct MacGeom {
  int nIs, nIb, nJ, nC, CW, nCg, nSb, LN;
  int f64;       // MAC engine: 0 = IMAD.WIDE on 25-bit limbs, 1 = exact FP64 (DFMA) products
  int engine;    // 0 IMAD, 1 FP64, 2 int8 tensor cores (mac_tc.cuh)
  int nIp, nIt, RT, nJp, nJc;   // engine 2: rows padded to 16, nIt balanced I tiles of RT rows, J padded to 32, 32-J steps
  int cperm;     // MAC column of (K, c): 0 -> 2K + c (the API layout [nK][2]), 1 -> c nK + K (c0 columns
                 // first: the fused paths, so that the forward NTTs of c0 pair up and the c1 copies do too)
  int c1_in;     // 1: the MAC loads the c1 halves straight from the ciphertexts (tensor-map TMA, quad
                 // order) and the forward kernel transforms c0 only
  int pf;        // forward kernels: L2 prefetch distance in CTAs (one wave), 0: off
  int xw;        // X row width (u64 per (slot, J)): CW, or nK when c1_in with one column group (X then
                 // holds only the c0 columns)
};

__host__ __device__ __forceinline__ size_t w_index(const MacGeom &g, int iloc, int J, int s) {
  return ((((size_t)(iloc >> 4) * g.nSb + (s >> 5)) * g.nJ + J) * 32 + (s & 31)) * 16 + (iloc & 15);
}

// u32-word offset of the X chunk of (J, column group cg, slot block sb):
//   IMAD engine: 96*CW words ([32][CW] limb pairs + [32][CW] limb sums, 3 KB at CW = 8)
//   FP64 engine: 64*CW words ([32][CW] doubles, 2 KB at CW = 8)
__host__ __device__ __forceinline__ int x_chunk_words(const MacGeom &g) { return (g.f64 ? 64 : 96) * g.CW; }
__host__ __device__ __forceinline__ size_t x_chunk(const MacGeom &g, int J, int cg, int sb) {
  return (((size_t)sb * g.nCg + cg) * g.nJ + J) * (size_t)x_chunk_words(g);
}

MacGeom mac_geom(const hl_ctx *c, int64_t nIs, int64_t nJ, int64_t nC) {
  MacGeom g;
  g.nIs = (int)nIs; g.nIb = (int)((nIs + 15) / 16); g.nJ = (int)nJ; g.nC = (int)nC;
  g.engine = c->mac_engine;
  if (g.engine == 2)
    g.CW = (nC % 16 == 0) ? 16 : ((nC % 8 == 0) ? 8 : ((nC % 4 == 0) ? 4 : 2));
  else
    g.CW = (nC % 8 == 0) ? 8 : ((nC % 4 == 0) ? 4 : 2);
  g.nCg = (int)(nC / g.CW);
  g.LN = (int)(c->L * c->N);
  g.nSb = g.LN / 32;
  g.f64 = c->mac_engine == 1;
  g.nIp = g.nIb * 16;
  // tile rows per MMA: <= 128 (M = 128; tiles of <= 64 rows use M = 64), balanced tiles in multiples
  // of 8 (UMMA core rows).  Measured alternatives: tiles of <= 64 rows, and full
  // 128-row tiles + one short last tile, were both slower on c2 (the latter re-measured in round 2:
  // c2 0.867 -> 0.904 ms, c3 43.2 -> 43.9 ms per stack).
  constexpr int rt_max = 128;
  g.nIt = (g.nIp + rt_max - 1) / rt_max;
  g.RT = ((g.nIp + g.nIt - 1) / g.nIt + 7) / 8 * 8;
  if ((int64_t)g.RT * (g.nIt - 1) >= nIs) g.RT = rt_max;   // never an empty last tile
  g.nJp = (int)((nJ + 31) / 32 * 32);
  g.nJc = g.nJp / 32;
  g.cperm = 0;
  g.c1_in = 0;
  g.pf = 0;
  g.xw = g.CW;
  return g;
}

// ---------------------------------------------------------------------------------------
// Forward NTT kernels
// ---------------------------------------------------------------------------------------
// (a) ciphertext polynomials: in [npoly][L][N] coefficient form ->
//     MODE 0: u64 [npoly][L][N] in slot order (diagnostics)
//     MODE 1: limb pairs in the blocked X layout (poly = J*nC + col), the MAC operand
template <int LOGN, int MODE>
__global__ void __launch_bounds__(Geom<LOGN>::NT)
k_ntt_fwd(const uint64_t *__restrict__ in, void *__restrict__ out, DevParams P, MacGeom mg) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  const int t = threadIdx.x, l = blockIdx.y;
  const size_t base = ((size_t)blockIdx.x * P.L + l) * Gm::N;
  const PrimeConsts pc = pick(P, l);
  const double *tw = P.twd_fwd + (size_t)l * Gm::N;
  double a[16];
  constexpr int K = Gm::k(0), G = 16 >> K;
  const int J = (int)(blockIdx.x / (unsigned)max(mg.nC, 1)), col = (int)(blockIdx.x % (unsigned)max(mg.nC, 1));
  if (MODE == 1 && (col & 1)) {
    load_eval_slots<LOGN>(a, in + base, reinterpret_cast<uint64_t *>(sm), t, -1);   // c1: evaluation form (C26)
  } else {
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
      for (int u = 0; u < (1 << K); u++) a[g * (1 << K) + u] = u2d(__ldcs(in + base + elem_idx<LOGN, 0>(t, g, u)));
    fwd_rounds_from<LOGN, 0>(a, sm, t, tw, pc.pd, pc.pinv);
  }
#pragma unroll
  for (int u = 0; u < 16; u++) {
    const double xd = canon_d(a[u], pc.pd, pc.pinv);
    if constexpr (MODE == 1) {
      const int s = l * Gm::N + slot_of<LOGN>(t, u);
      uint32_t *ch = reinterpret_cast<uint32_t *>(out) + x_chunk(mg, J, col / mg.CW, s >> 5);
      const int e = (s & 31) * mg.CW + col % mg.CW;
      if (mg.engine == 2) {
        const int cg = col / mg.CW, c = col % mg.CW;
        reinterpret_cast<uint64_t *>(out)[(((size_t)cg * mg.LN + s) * mg.nJp + J) * mg.CW + c] = d2u(xd);
      } else if (mg.f64) {
        reinterpret_cast<double *>(ch)[e] = xd;
      } else {
        const uint64_t x = d2u(xd);
        const uint32_t x0 = (uint32_t)x & kLimbMask, x1 = (uint32_t)(x >> kLimbBits);
        reinterpret_cast<uint2 *>(ch)[e] = make_uint2(x0, x1);
        ch[64 * mg.CW + e] = x0 + x1;
      }
    } else {
      reinterpret_cast<uint64_t *>(out)[base + slot_of<LOGN>(t, u)] = d2u(xd);
    }
  }
}

// (a') ciphertext polynomials for the tensor-core MAC (engine 2): G consecutive polynomials
//      (same J, columns col0 .. col0+G-1 of one CW group) per CTA, canonical residues staged in
//      shared memory as [slot][G] so that every (slot, J) store is G consecutive u64 of the X
//      layout [cg][LN][nJp][CW] (a 16-B half sector for G = 2, a full 32-B sector for G = 4).
template <int LOGN, int G>
__global__ void __launch_bounds__(Geom<LOGN>::NT * G)
k_ntt_fwd_x(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, DevParams P, MacGeom mg) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  const int sub = threadIdx.x / Gm::NT, t = threadIdx.x % Gm::NT, l = blockIdx.y;
  const int64_t poly0 = (int64_t)blockIdx.x * G;
  const size_t base = ((size_t)(poly0 + sub) * P.L + l) * Gm::N;
  const PrimeConsts pc = pick(P, l);
  const double *tw = P.twd_fwd + (size_t)l * Gm::N;
  double a[16];
  constexpr int K = Gm::k(0), GG = 16 >> K;
  if ((poly0 + sub) % mg.nC & 1) {
    // c1 (column 2K+1) arrives in evaluation form (reading C26): no transform, only the
    // permutation from natural order to slots
    load_eval_slots<LOGN>(a, in + base, reinterpret_cast<uint64_t *>(sm + sub * Gm::SMEM_WORDS), t,
                          G > 1 ? 1 + sub : -1);
  } else {
#pragma unroll
    for (int g = 0; g < GG; g++)
#pragma unroll
      for (int u = 0; u < (1 << K); u++) a[g * (1 << K) + u] = u2d(__ldcs(in + base + elem_idx<LOGN, 0>(t, g, u)));
    fwd_rounds_from<LOGN, 0>(a, sm + sub * Gm::SMEM_WORDS, t, tw, pc.pd, pc.pinv, G > 1 ? 1 + sub : -1);
  }
  __syncthreads();                                     // every sub-NTT is done with its smem
  uint64_t *xs = reinterpret_cast<uint64_t *>(sm);     // [N][G] canonical residues
#pragma unroll
  for (int u = 0; u < 16; u++) xs[slot_of<LOGN>(t, u) * G + sub] = d2u(canon_d(a[u], pc.pd, pc.pinv));
  __syncthreads();
  const int J = (int)(poly0 / mg.nC), col0 = (int)(poly0 % mg.nC);
  const int cg = col0 / mg.CW, c0 = col0 % mg.CW;
  uint64_t *dst0 = out + ((size_t)cg * mg.LN + (size_t)l * Gm::N) * mg.nJp * mg.CW + (size_t)J * mg.CW + c0;
#pragma unroll 2
  for (int sl = threadIdx.x; sl < Gm::N; sl += Gm::NT * G) {
    uint64_t *dst = dst0 + (size_t)sl * mg.nJp * mg.CW;
    if constexpr (G == 4) {
      const ulonglong2 v0 = *reinterpret_cast<const ulonglong2 *>(xs + sl * 4);
      const ulonglong2 v1 = *reinterpret_cast<const ulonglong2 *>(xs + sl * 4 + 2);
      reinterpret_cast<ulonglong2 *>(dst)[0] = v0;
      reinterpret_cast<ulonglong2 *>(dst)[1] = v1;
    } else if constexpr (G == 2) {
      *reinterpret_cast<ulonglong2 *>(dst) = *reinterpret_cast<const ulonglong2 *>(xs + sl * 2);
    } else {
      *dst = xs[sl];
    }
  }
}

// (a'') the fused paths' X layout (MacGeom::cperm = 1, c0 columns first): the forward NTTs of the
//       c0 halves of two adjacent columns (K0, K0+1) in the SAME threads (fwd_rounds_from2): the
//       pair's values for a slot sit in one thread, so the 16-B (slot, J) chunks are stored
//       straight from registers (no staging, no output barrier)
template <int LOGN, bool C1, int MB = 1>
__global__ void __launch_bounds__(Geom<LOGN>::NT, MB)
k_ntt_fwd_c0x2(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, DevParams P, MacGeom mg) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  __shared__ __align__(8) uint64_t c1bar;
  const int t = threadIdx.x, l = blockIdx.y;
  const int nK = mg.nC / 2, nKh = (nK + 1) / 2;
  const int J = (int)(blockIdx.x / (unsigned)nKh), K0 = 2 * (int)(blockIdx.x % (unsigned)nKh);
  const bool pair = K0 + 1 < nK;
  const PrimeConsts pc = pick(P, l);
  double a[16], b[16];
  const size_t base0 = (((size_t)J * nK + K0) * 2 * P.L + l) * Gm::N;       // c0 of (J, K0)
  const size_t base1 = base0 + (pair ? (size_t)2 * P.L * Gm::N : 0);       // c0 of (J, K0 + 1)
  if (t == 0 && mg.pf > 0) {
    // the inputs of the CTA one wave ahead (CTAs are dispatched x fastest) into L2: its loads at
    // start-up no longer wait for DRAM.  N = 8192 only (launch_fwd_cperm): one 512-thread CTA per
    // SM exposes that latency (c4 forward 238 -> 227 ms per stack); at N = 4096 (2-3 CTAs per SM)
    // it measured slower (c3 11.2 -> 11.6 ms)
    const unsigned lin = blockIdx.y * gridDim.x + blockIdx.x + (unsigned)mg.pf;
    if (lin < gridDim.x * gridDim.y) {
      const int x2 = (int)(lin % gridDim.x), l2 = (int)(lin / gridDim.x);
      const int J2 = x2 / nKh, K2 = 2 * (x2 % nKh);
      const uint64_t *b2 = in + (((size_t)J2 * nK + K2) * 2 * P.L + l2) * Gm::N;
      prefetch_l2(b2, Gm::N * 8);
      if (K2 + 1 < nK) prefetch_l2(b2 + (size_t)2 * P.L * Gm::N, Gm::N * 8);
    }
  }
  constexpr int KK = Gm::k(0), GG = 16 >> KK;
#pragma unroll
  for (int g = 0; g < GG; g++)
#pragma unroll
    for (int u = 0; u < (1 << KK); u++) {
      const int e = elem_idx<LOGN, 0>(t, g, u);
      a[g * (1 << KK) + u] = u2d(__ldcs(in + base0 + e));
      b[g * (1 << KK) + u] = u2d(__ldcs(in + base1 + e));
    }
  fwd_rounds_from2<LOGN, 0>(a, b, sm, sm + Gm::SMEM_WORDS, t, P.twd_fwd + (size_t)l * Gm::N, pc.pd, pc.pinv);
  if constexpr (C1) {
    // fused c1 pair (evaluation form, C26): the exchange buffers are free once every thread is
    // past the last exchange; the bulk copies land while the c0 results are stored
    __syncthreads();
    if (t == 0) {
      mbar_init(&c1bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&c1bar, (pair ? 2 : 1) * Gm::N * 8);
      const uint64_t *c1src = in + (((size_t)J * nK + K0) * 2 * P.L + P.L + l) * Gm::N;
      bulk_g2s(sm, c1src, Gm::N * 8, &c1bar);
      if (pair) bulk_g2s(reinterpret_cast<uint64_t *>(sm) + Gm::N, c1src + (size_t)2 * P.L * Gm::N, Gm::N * 8, &c1bar);
    }
  }
  const int cg = K0 / mg.CW, cc = K0 % mg.CW;
  uint64_t *dst0 = out + ((size_t)cg * mg.LN + (size_t)l * Gm::N) * mg.nJp * mg.xw + (size_t)J * mg.xw + cc;
#pragma unroll
  for (int u = 0; u < 16; u++) {
    uint64_t *dst = dst0 + (size_t)slot_of<LOGN>(t, u) * mg.nJp * mg.xw;
    const uint64_t x0 = d2u(canon_d(a[u], pc.pd, pc.pinv)), x1 = d2u(canon_d(b[u], pc.pd, pc.pinv));
    if (pair) *reinterpret_cast<ulonglong2 *>(dst) = make_ulonglong2(x0, x1);
    else *dst = x0;
  }
  if constexpr (C1) {
    __syncthreads();                                  // the barrier init is visible to every thread
    mbar_wait(&c1bar, 0);
    const uint64_t *stg = reinterpret_cast<const uint64_t *>(sm);
    const int lane = t & 31, warp = t >> 5;
    const int tr = ((lane & 15) << (LOGN - 8)) | ((lane >> 4) << (LOGN - 9)) | warp;   // conflict-free gather
    const int col = nK + K0, cg1 = col / mg.CW, cc1 = col % mg.CW;
    uint64_t *d1 = out + ((size_t)cg1 * mg.LN + (size_t)l * Gm::N) * mg.nJp * mg.CW + (size_t)J * mg.CW + cc1;
#pragma unroll 4
    for (int u = 0; u < 16; u++) {
      const int k = nat_of<LOGN>(tr, u);
      uint64_t *dst = d1 + (size_t)slot_of<LOGN>(tr, u) * mg.nJp * mg.CW;
      if (pair) *reinterpret_cast<ulonglong2 *>(dst) = make_ulonglong2(stg[k], stg[Gm::N + k]);
      else *dst = stg[k];
    }
  }
}

// c1 halves (evaluation form, reading C26) into the permuted X layout: no transform, only the
// natural -> slot reordering.  G1 consecutive K (adjacent columns nK + K) per CTA, so that every
// (slot, J) store is 8 G1 contiguous bytes (a full 32-B sector for G1 = 4).  The G1 natural-order
// polynomials arrive by bulk copies (TMA); the gather is bank-conflict free because the 16 low
// lanes of a warp differ in the top bits of t, i.e. in the low bits of the natural index.
// c1 halves (evaluation form, natural order, reading C26) of whole CW = 16 column groups into the
// X layout for the tensor-core MAC (the c1 columns of the fat products c3/c4, where the MAC's own
// gather of c1 through a tensor-map box moves 16-B pieces): a CTA takes one J, one c1 column group
// (16 ciphertexts K0 .. K0+15) and 256 natural points of one prime; coalesced 8-B loads of the 16
// rows into shared memory (rows padded to 257 words: conflict-free both ways), then every point's
// 16 columns as one 128-B line X[cg][l N + slot(k)][J][0..16) -- full lines, 4 sectors each.
template <int LOGN>
__global__ void __launch_bounds__(256)
k_c1_tx16(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, DevParams P, MacGeom mg) {
  constexpr int N = 1 << LOGN, PTS = 256, ROW = PTS + 1;
  __shared__ uint64_t stg[16 * ROW];
  const int t = threadIdx.x, l = blockIdx.z;
  const int nK = mg.nC / 2, ncg1 = nK / 16;
  const int J = (int)(blockIdx.y / (unsigned)ncg1), g1 = (int)(blockIdx.y % (unsigned)ncg1);
  const int k0 = blockIdx.x * PTS, K0 = g1 * 16;
#pragma unroll
  for (int c = 0; c < 16; c++)
    stg[c * ROW + t] = __ldcs(in + (((size_t)J * nK + K0 + c) * 2 * P.L + P.L + l) * N + k0 + t);
  __syncthreads();
  const int cg = (nK + K0) / 16, c = t & 15;
  uint64_t *dst0 = out + ((size_t)cg * mg.LN + (size_t)l * N) * mg.nJp * 16 + (size_t)J * 16 + c;
#pragma unroll 4
  for (int it = 0; it < PTS / 16; it++) {
    const int kk = it * 16 + (t >> 4), k = k0 + kk;
    const int idx = (int)(__brev((unsigned)k) >> (32 - LOGN));          // CT index of natural point k
    const int s = (idx & 15) * (N / 16) + (idx >> 4);                    // its slot (slot_of)
    dst0[(size_t)s * mg.nJp * 16] = stg[c * ROW + kk];
  }
}

template <int LOGN, int G1>
__global__ void __launch_bounds__(Geom<LOGN>::NT)
k_c1_to_x(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, DevParams P, MacGeom mg) {
  using Gm = Geom<LOGN>;
  extern __shared__ __align__(128) unsigned char smc[];
  const uint64_t *stg = reinterpret_cast<const uint64_t *>(smc);          // [G1][N] natural order
  __shared__ __align__(8) uint64_t bar;
  const int l = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nK = mg.nC / 2, nKg = nK / G1;
  const int J = (int)(blockIdx.x / (unsigned)nKg), K0 = G1 * (int)(blockIdx.x % (unsigned)nKg);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar, G1 * Gm::N * 8);
#pragma unroll
    for (int g = 0; g < G1; g++)
      bulk_g2s(smc + g * Gm::N * 8, in + (((size_t)J * nK + K0 + g) * 2 * P.L + P.L + l) * Gm::N, Gm::N * 8, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int t = ((lane & 15) << (LOGN - 8)) | ((lane >> 4) << (LOGN - 9)) | warp;
  const int col = nK + K0, cg = col / mg.CW, cc = col % mg.CW;
  uint64_t *dst0 = out + ((size_t)cg * mg.LN + (size_t)l * Gm::N) * mg.nJp * mg.CW + (size_t)J * mg.CW + cc;
#pragma unroll 4
  for (int u = 0; u < 16; u++) {
    const int k = nat_of<LOGN>(t, u);
    uint64_t *dst = dst0 + (size_t)slot_of<LOGN>(t, u) * mg.nJp * mg.CW;
    if constexpr (G1 == 4) {
      reinterpret_cast<ulonglong2 *>(dst)[0] = make_ulonglong2(stg[k], stg[Gm::N + k]);
      reinterpret_cast<ulonglong2 *>(dst)[1] = make_ulonglong2(stg[2 * Gm::N + k], stg[3 * Gm::N + k]);
    } else if constexpr (G1 == 2) {
      *reinterpret_cast<ulonglong2 *>(dst) = make_ulonglong2(stg[k], stg[Gm::N + k]);
    } else {
      *dst = stg[k];
    }
  }
}

// (b) weights: pi_A of tile (I, J), centered lift (reading C6), mod p_l, NTT.
//     poly index = I_loc * nJ + J over the 16-padded shard; wcache in the blocked W layout.
struct EncodeArgs {
  const uint64_t *W;
  int64_t R, Ma, nJ, nIs, i_begin;
  int m, r;
  MacGeom mg;
  int64_t ld_r, ld_c;      // element (row, col) of W at W[row * ld_r + col * ld_c]
};

template <int LOGN>
__global__ void __launch_bounds__(Geom<LOGN>::NT)
k_encode_weights(EncodeArgs A, uint2 *__restrict__ wcache, DevParams P, uint32_t *flags, uint64_t *__restrict__ scratch) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  const int t = threadIdx.x, l = blockIdx.y;
  const int64_t poly = blockIdx.x, Iloc = poly / A.nJ, J = poly % A.nJ, I = A.i_begin + Iloc;
  const PrimeConsts pc = pick(P, l);
  const double *tw = P.twd_fwd + (size_t)l * Gm::N;
  const uint64_t tmask = (P.t_bits >= 64) ? ~0ull : ((1ull << P.t_bits) - 1);
  const uint64_t half = 1ull << (P.t_bits - 1);
  const int mr = A.m * A.r;
  double a[16];
  uint32_t maxabs = 0, bad = 0;
  constexpr int K = Gm::k(0), G = 16 >> K;
#pragma unroll
  for (int g = 0; g < G; g++)
#pragma unroll
    for (int u = 0; u < (1 << K); u++) {
      const int e = elem_idx<LOGN, 0>(t, g, u);
      uint64_t v = 0;
      if (e < mr && Iloc < A.nIs) {          // rows padded up to 16 are zero polynomials
        const int i = e / A.r, j = A.r - 1 - e % A.r;
        const int64_t row = J * A.r + j, col = I * A.m + i;
        if (row < A.R && col < A.Ma) {
          const uint64_t w = A.W[row * A.ld_r + col * A.ld_c];
          bad |= (w & ~tmask) != 0;
          const uint64_t wm = w & tmask;
          if (wm < half) {                      // lift(w) = w
            v = wm % pc.p;
            maxabs = max(maxabs, (uint32_t)min(wm, (uint64_t)0xffffffffu));
          } else {                              // lift(w) = w - t  (negative)
            const uint64_t mag = (tmask - wm) + 1;
            const uint64_t mm = mag % pc.p;
            v = mm ? pc.p - mm : 0;
            maxabs = max(maxabs, (uint32_t)min(mag, (uint64_t)0xffffffffu));
          }
        }
      }
      a[g * (1 << K) + u] = u2d(v);
    }
  if (l == 0) {
    if (bad) atomicOr(&flags[0], 1u);
    if (maxabs) atomicMax(&flags[1], maxabs);
  }
  fwd_rounds_from<LOGN, 0>(a, sm, t, tw, pc.pd, pc.pinv);
#pragma unroll
  for (int u = 0; u < 16; u++) {
    const double xd = canon_d(a[u], pc.pd, pc.pinv);
    const uint64_t x = d2u(xd);
    const int s = l * Gm::N + slot_of<LOGN>(t, u);
    if (scratch) {                      // engine 2, two-pass: u64 residues now, byte planes by k_wplanes
      if (Iloc < A.nIs) scratch[((size_t)Iloc * A.nJ + J) * A.mg.LN + s] = x;
    } else if (A.mg.engine == 2) {
      // 7 byte planes, UMMA canonical K-major: [I tile][slot][32-J step][plane][K half][row][16 B]
      const int tt = (int)(Iloc / A.mg.RT), row = (int)(Iloc % A.mg.RT);
      const int rows = min(A.mg.RT, A.mg.nIp - A.mg.RT * tt);
      uint8_t *wb = reinterpret_cast<uint8_t *>(wcache) + (size_t)tt * A.mg.RT * A.mg.LN * A.mg.nJp * 7 +
                    ((size_t)s * A.mg.nJc + (J >> 5)) * 224 * rows + ((J >> 4) & 1) * rows * 16 + row * 16 + (J & 15);
#pragma unroll
      for (int a = 0; a < 7; a++) wb[a * 32 * rows] = (uint8_t)(x >> (8 * a));
    } else if (A.mg.f64)
      reinterpret_cast<double *>(wcache)[w_index(A.mg, (int)Iloc, (int)J, s)] = xd;
    else
      wcache[w_index(A.mg, (int)Iloc, (int)J, s)] = make_uint2((uint32_t)x & kLimbMask, (uint32_t)(x >> kLimbBits));
  }
}

// ---------------------------------------------------------------------------------------
// Inverse NTT kernel: in u64 [npoly][L][N] (NTT domain, slot order) -> out [npoly][L][N]
// coefficient form, canonical.  in may alias out.
// ---------------------------------------------------------------------------------------
// residues in [0, 2^52) (canonical, or the MAC's lazy outputs < 4p), reduced to |v| <= p/2 (the inverse rounds' entry bound)
template <int LOGN>
__device__ __forceinline__ void load_ntt_domain(double (&a)[16], const uint64_t *src, int t, const PrimeConsts &pc) {
#pragma unroll
  for (int u = 0; u < 16; u++) a[u] = red_d(u2d(__ldcs(src + slot_of<LOGN>(t, u))), pc.pd, pc.pinv);
}
// Quad order of the MAC output (MacTcArgs::qperm): position 4 q + i of a row holds slot
// u NT + t' + {0, 2, 1, 3}[i] NT/4 (q = u NT/4 + t'), so that the 4 slots of a MAC work item are 4
// consecutive natural evaluation points (k_mac_tc's direct c1 store).  Slot u NT + t is therefore
// read from u NT + 4 (t mod NT/4) + brev2(t / (NT/4)); a warp's 32 loads touch 32 sectors that the
// CTA's other three quarter-warps complete (L1-cached loads).
template <int LOGN>
__device__ __forceinline__ void load_ntt_domain_q(double (&a)[16], const uint64_t *src, int t, const PrimeConsts &pc) {
  constexpr int NT = Geom<LOGN>::NT, Q = NT / 4;
  const int h = t / Q, off = 4 * (t % Q) + ((h & 1) << 1 | (h >> 1));
#pragma unroll
  for (int u = 0; u < 16; u++) a[u] = red_d(u2d(__ldg(src + u * NT + off)), pc.pd, pc.pinv);
}

template <int LOGN>
__global__ void __launch_bounds__(Geom<LOGN>::NT)
k_ntt_inv(const uint64_t *in, uint64_t *out, DevParams P, int ct_mode) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  const int t = threadIdx.x, l = blockIdx.y;
  const size_t base = ((size_t)blockIdx.x * P.L + l) * Gm::N;
  const PrimeConsts pc = pick(P, l);
  const double *tw = P.twd_inv + (size_t)l * Gm::N;
  double a[16];
  load_ntt_domain<LOGN>(a, in + base, t, pc);
  if (ct_mode && (blockIdx.x & 1)) {        // ciphertexts: c1 stays in evaluation form (reading C26)
    uint64_t x[16];
#pragma unroll
    for (int u = 0; u < 16; u++) x[u] = d2u(canon_d(a[u], pc.pd, pc.pinv));
    store_eval_slots<LOGN>(x, out + base, reinterpret_cast<uint64_t *>(sm), t, -1);
    return;
  }
  inv_rounds_from<LOGN, Gm::NR - 1>(a, sm, t, tw, pc);
  constexpr int K = Gm::k(0), G = 16 >> K;
#pragma unroll
  for (int g = 0; g < G; g++)
#pragma unroll
    for (int u = 0; u < (1 << K); u++)
      out[base + elem_idx<LOGN, 0>(t, g, u)] = d2u(canon_d(a[g * (1 << K) + u], pc.pd, pc.pinv));
}

// Second pass of the two-pass weight encoding (hl_encode_weights_scratch): u64 NTT-domain
// residues scratch [nIs][nJ][LN] -> the 7 byte planes of the tensor-core MAC's A operand
// ([I tile][slot][32-J step][plane][K half][row][16 B]).  A tiled transpose: one CTA per
// (I tile, 32-J step, block of 16 rows, block of 16 slots) stages [slot][row][J] in shared memory
// (reads: 128-B runs of consecutive slots), then writes each slot's 16 rows x 14 pieces of 16 B
// (256-B runs per (plane, K half)); padded rows and J are zero, so no memset is needed.
constexpr int kWpS = 16, kWpR = 16;
__global__ void __launch_bounds__(256) k_wplanes(const uint64_t *__restrict__ scratch, uint8_t *__restrict__ wcache,
                                                 MacGeom g) {
  extern __shared__ uint64_t vsd[];                                // [kWpS][kWpR][33] (+1: bank spread)
  auto vs = [&](int si, int r, int j) -> uint64_t & { return vsd[(si * kWpR + r) * 33 + j]; };
  const int nsb = g.LN / kWpS, nrb = (g.RT + kWpR - 1) / kWpR;
  int b = blockIdx.x;
  const int sb = b % nsb; b /= nsb;
  const int rb = b % nrb; b /= nrb;
  const int jc = b % g.nJc, tt = b / g.nJc;
  const int rows = min(g.RT, g.nIp - g.RT * tt);
  if (rb * kWpR >= rows) return;
  const int s0 = sb * kWpS;
  for (int e = threadIdx.x; e < kWpR * 32 * kWpS; e += blockDim.x) {
    const int si = e % kWpS, j = (e / kWpS) % 32, r = e / kWpS / 32;
    const int row = rb * kWpR + r, Iloc = tt * g.RT + row, J = jc * 32 + j;
    vs(si, r, j) = (row < rows && Iloc < g.nIs && J < g.nJ) ? __ldcs(scratch + ((size_t)Iloc * g.nJ + J) * g.LN + s0 + si) : 0;
  }
  __syncthreads();
  const int rr = min(kWpR, rows - rb * kWpR);
  for (int e = threadIdx.x; e < kWpS * 14 * rr; e += blockDim.x) {
    const int r = e % rr, ah = (e / rr) % 14, si = e / rr / 14;
    const int a = ah >> 1, h = ah & 1;
    const uint32_t bb = a & 3, sel = bb | ((bb + 4) << 4);
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      uint32_t x[4];
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const uint64_t v = vs(si, r, h * 16 + 4 * q + t);
        x[t] = a < 4 ? (uint32_t)v : (uint32_t)(v >> 32);
      }
      w[q] = __byte_perm(__byte_perm(x[0], x[1], sel), __byte_perm(x[2], x[3], sel), 0x5410);
    }
    uint8_t *chunk = wcache + (size_t)tt * g.RT * g.LN * g.nJp * 7 + ((size_t)(s0 + si) * g.nJc + jc) * 224 * rows;
    *reinterpret_cast<uint4 *>(chunk + (size_t)a * 32 * rows + h * rows * 16 + (rb * kWpR + r) * 16) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// ---------------------------------------------------------------------------------------
// Fused inverse NTT + mask + compression + server share (compressed mode only).
// One CTA per (output ct o = I_loc*nK + K, component c); loops over the L primes.
//   c = 1: c1 copied to the compressed response
//   c = 0: sigma at the kept positions (ChaCha20, once for all primes), c0 - Delta_l*sigma
//          written at index k*m+i; share_server[K*n+k][I*m+i] = sigma (in-range only).
// ---------------------------------------------------------------------------------------
struct MaskArgs {
  int64_t Ma, Nb, nK, i_begin;
  int m, r, n;
  int lm, lr;          // log2 m, log2 r (tiles are powers of two: divisions become shifts)
  uint64_t seed;
  // row f4 (reading C22): re-randomisation c += Enc_pk(0) + (F, 0); pk_hat == nullptr: off
  const uint64_t *pk_hat;   // [2][L][N] NTT(pk) in slot order
  const uint64_t *u_hat;    // [nout][L][N] NTT(u) in slot order (k_rr_u)
  const uint64_t *cdt;      // device CDT table
  int flood_bits;
  int nC, cperm;            // MAC output columns and their order (MacGeom::cperm)
  int c1_done;              // the MAC already wrote the c1 halves of the response (MacTcArgs::c1_out)
};

// index of the NTT-domain polynomial (component c of output ciphertext o = I_loc nK + K) in the
// MAC output [nI_s][nC][L][N]
__device__ __forceinline__ size_t ct_poly(const MaskArgs &M, int64_t o, int c) {
  return M.cperm ? (size_t)(o / M.nK) * M.nC + (size_t)c * M.nK + (size_t)(o % M.nK) : (size_t)o * 2 + c;
}

// e (reading C8) from one PRF word
__device__ __forceinline__ int cdt_sample(uint64_t w, const uint64_t *cdt) {
  const uint64_t v = w & 0x7fffffffffffffffull;
  int k = 0;
  while (k < 41 && v >= __ldg(&cdt[k])) k++;
  return (w >> 63) ? -k : k;
}
// signed value mod p (|v| < 2^63)
__device__ __forceinline__ uint64_t smod(int64_t v, const PrimeConsts &pc) {
  if (v >= 0) return (uint64_t)v % pc.p;
  const uint64_t m = (uint64_t)(-v) % pc.p;
  return m ? pc.p - m : 0;
}
// c0 extra of re-randomisation at position pos: e1[pos] + F[pos] (domains 8 and 9)
__device__ __forceinline__ int64_t rr_c0_extra(const MaskArgs &M, uint64_t stream, int pos) {
  int64_t ext = cdt_sample(hl::prf_u64(M.seed, hl::kDomRrE, 2 * stream, (uint64_t)pos), M.cdt);
  if (M.flood_bits > 0)
    ext += (int64_t)(hl::prf_u64(M.seed, hl::kDomRrF, stream, (uint64_t)pos) & ((1ull << M.flood_bits) - 1)) -
           (1ll << (M.flood_bits - 1));
  return ext;
}
// Reading C27: the MASK-stream word order puts the kept positions first, so the m n masks of a
// compressed response are the stream's first m n words: (m n)/8 ChaCha blocks, not one per kept
// position.  sigma (kept-index order kk = k m + i) -> sig_sm, the server share, and for row f4
// the c0 extras e1 + F at the kept positions.
template <bool RR>
__device__ __forceinline__ void mask_kept(const MaskArgs &M, uint64_t stream, int64_t I, int64_t K, uint64_t tmask,
                                          uint64_t *sig_sm, int64_t *ext_sm, uint64_t *share, int t, int nthr) {
  const int mn = M.m * M.n;
#pragma unroll 1
  for (int blk = t; blk < (mn + 7) / 8; blk += nthr) {
    uint64_t w[8];
    hl::chacha_block_u64(M.seed, hl::kDomMask, stream, (uint32_t)blk, w);
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int kk = 8 * blk + q;
      if (kk >= mn) break;
      const uint64_t sg = w[q] & tmask;
      sig_sm[kk] = sg;
      const int64_t row = K * M.n + (kk >> M.lm), col = I * M.m + (kk & (M.m - 1));
      if (row < M.Nb && col < M.Ma) share[row * M.Ma + col] = sg;
    }
  }
  if constexpr (RR) {
#pragma unroll 1
    for (int kk = t; kk < mn; kk += nthr) ext_sm[kk] = rr_c0_extra(M, stream, (kk << M.lr) + M.r - 1);
  }
}

// coefficient position of MASK word w (inverse of the C27 order)
__device__ __forceinline__ int mask_pos(const MaskArgs &M, int w) {
  const int mn = M.m * M.n;
  if (w < mn) return (w << M.lr) + M.r - 1;
  const int rho = w - mn;
  if (M.r == 1 || rho >= mn * (M.r - 1)) return rho + mn;
  return rho + rho / (M.r - 1);
}

// re-randomisation of a loaded NTT-domain polynomial: a += pk_hat[c] * u_hat  (slot order)
template <int LOGN>
__device__ __forceinline__ void rr_add_ntt(double (&a)[16], const MaskArgs &M, int64_t o, int c, int l, int L, int t,
                                           const PrimeConsts &pc) {
  const uint64_t *pk = M.pk_hat + ((size_t)c * L + l) * Geom<LOGN>::N;
  const uint64_t *uh = M.u_hat + ((size_t)o * L + l) * Geom<LOGN>::N;
#pragma unroll
  for (int u = 0; u < 16; u++) {
    const int sl = slot_of<LOGN>(t, u);
    a[u] = red_d(__dadd_rn(a[u], mm_d(u2d(__ldg(&uh[sl])), u2d(__ldg(&pk[sl])), pc.pd, pc.pinv)), pc.pd, pc.pinv);
  }
}

// u_hat[o][l] = NTT(u) (slot order) of the ternary u of every output ciphertext (domain 7,
// stream (i_begin + I) nK + K)
template <int LOGN>
__global__ void __launch_bounds__(Geom<LOGN>::NT)
k_rr_u(uint64_t *__restrict__ u_hat, MaskArgs M, DevParams P) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  int8_t *u_sm = reinterpret_cast<int8_t *>(sm + Gm::SMEM_WORDS);
  const int t = threadIdx.x, L = P.L;
  const int64_t o = blockIdx.x, I = M.i_begin + o / M.nK, K = o % M.nK;
#pragma unroll 1
  for (int blk = t; blk < Gm::N / 8; blk += Gm::NT) {
    uint64_t w[8];
    hl::chacha_block_u64(M.seed, hl::kDomRrU, (uint64_t)(I * M.nK + K), (uint32_t)blk, w);
#pragma unroll
    for (int i = 0; i < 8; i++) u_sm[8 * blk + i] = (int8_t)((int)(w[i] % 3) - 1);
  }
  __syncthreads();
  constexpr int K0 = Gm::k(0), G = 16 >> K0;
  for (int l = 0; l < L; l++) {
    const PrimeConsts pc = pick(P, l);
    double a[16];
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
      for (int u = 0; u < (1 << K0); u++) a[g * (1 << K0) + u] = (double)u_sm[elem_idx<LOGN, 0>(t, g, u)];
    fwd_rounds_from<LOGN, 0>(a, sm, t, P.twd_fwd + (size_t)l * Gm::N, pc.pd, pc.pinv);
    uint64_t *dst = u_hat + ((size_t)o * L + l) * Gm::N;
#pragma unroll
    for (int u = 0; u < 16; u++) dst[slot_of<LOGN>(t, u)] = d2u(canon_d(a[u], pc.pd, pc.pinv));
    __syncthreads();
  }
}


template <int LOGN, bool RR>
__global__ void __launch_bounds__(Geom<LOGN>::NT, LOGN == 12 ? 2 : 1)
k_ntt_inv_mask(const uint64_t *__restrict__ ct_ntt, uint64_t *__restrict__ masked, uint64_t *__restrict__ share,
               MaskArgs M, DevParams P, int c1_only) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  uint64_t *sig_sm = reinterpret_cast<uint64_t *>(sm + Gm::SMEM_WORDS);   // sigma at kept positions
  const int t = threadIdx.x;
  const int c = c1_only ? 1 : (blockIdx.x & 1);
  const int64_t o = c1_only ? blockIdx.x : (blockIdx.x >> 1);   // I_loc * nK + K
  const int64_t Iloc = o / M.nK, K = o % M.nK, I = M.i_begin + Iloc;
  const int mn = M.m * M.n, mr = M.m * M.r;
  const int L = P.L;
  const uint64_t tmask = (P.t_bits >= 64) ? ~0ull : ((1ull << P.t_bits) - 1);
  const size_t per = (size_t)L * (mn + Gm::N);
  uint64_t *dst = masked + (size_t)o * per;
  constexpr bool rr = RR;                                         // row f4 (compile-time: lean plain kernel)
  int64_t *ext_sm = reinterpret_cast<int64_t *>(sig_sm + mn);    // c0: e1 + F at the kept positions
  int8_t *e2_sm = reinterpret_cast<int8_t *>(sig_sm);             // c1: e2 at every position
  const uint64_t stream = (uint64_t)(I * M.nK + K);
  if (c == 0) {
    mask_kept<RR>(M, stream, I, K, tmask, sig_sm, ext_sm, share, t, Gm::NT);
    __syncthreads();
  } else if (rr) {
#pragma unroll 1
    for (int blk = t; blk < Gm::N / 8; blk += Gm::NT) {
      uint64_t w[8];
      hl::chacha_block_u64(M.seed, hl::kDomRrE, 2 * stream + 1, (uint32_t)blk, w);
#pragma unroll
      for (int i = 0; i < 8; i++) e2_sm[8 * blk + i] = (int8_t)cdt_sample(w[i], M.cdt);
    }
    __syncthreads();
  }
  for (int l = 0; l < L; l++) {
    const PrimeConsts pc = pick(P, l);
    const double *tw = P.twd_inv + (size_t)l * Gm::N;
    double a[16];
    load_ntt_domain<LOGN>(a, ct_ntt + (ct_poly(M, o, c) * L + l) * Gm::N, t, pc);
    if (rr) rr_add_ntt<LOGN>(a, M, o, c, l, L, t, pc);
    constexpr int K0 = Gm::k(0), G = 16 >> K0;
    if (c == 1) {
      // c1 leaves in evaluation form (reading C26): no inverse transform, only the reordering
      // to natural order -- except for re-randomisation, whose e2 is a coefficient-domain term
      if (rr) {
        inv_rounds_from<LOGN, Gm::NR - 1>(a, sm, t, tw, pc);
#pragma unroll
        for (int g = 0; g < G; g++)
#pragma unroll
          for (int u = 0; u < (1 << K0); u++) {
            double &v = a[g * (1 << K0) + u];
            v = red_d(__dadd_rn(v, (double)e2_sm[elem_idx<LOGN, 0>(t, g, u)]), pc.pd, pc.pinv);
          }
        fwd_rounds_from<LOGN, 0>(a, sm, t, P.twd_fwd + (size_t)l * Gm::N, pc.pd, pc.pinv);
        __syncthreads();                           // the exchange buffer becomes the staging buffer
      }
      uint64_t x[16];
#pragma unroll
      for (int u = 0; u < 16; u++) x[u] = d2u(canon_d(a[u], pc.pd, pc.pinv));
      store_eval_slots<LOGN>(x, dst + (size_t)L * mn + (size_t)l * Gm::N, reinterpret_cast<uint64_t *>(sm), t, -1);
      continue;
    }
    inv_rounds_from<LOGN, Gm::NR - 1>(a, sm, t, tw, pc);
#pragma unroll
    for (int g = 0; g < G; g++)
#pragma unroll
      for (int u = 0; u < (1 << K0); u++) {
        uint64_t x = d2u(canon_d(a[g * (1 << K0) + u], pc.pd, pc.pinv));
        const int idx = elem_idx<LOGN, 0>(t, g, u);
        if (idx < mr * M.n && (idx & (M.r - 1)) == M.r - 1) {
          const int kk = idx >> M.lr;               // = k*m + i for pos(i, k) = (k m + i) r + r - 1
          if (rr) { x += smod(ext_sm[kk], pc); x = x >= pc.p ? x - pc.p : x; }
          uint64_t d = shoup_mul(sig_sm[kk], pc.delta, pc.delta_sh, pc.p);
          d = d >= pc.p ? d - pc.p : d;
          dst[(size_t)l * mn + kk] = x >= d ? x - d : x + pc.p - d;
        }
      }
    __syncthreads();   // smem reuse by the next prime
  }
}

// c1 of the compressed response (plain responses, reading C26): the MAC output reordered from
// slot order to natural evaluation order and reduced from the MAC's lazy range (< 4p); no
// transform, so a light kernel (few registers, one staging buffer) instead of k_ntt_inv_mask
template <int LOGN>
__global__ void __launch_bounds__(Geom<LOGN>::NT)
k_c1_out(const uint64_t *__restrict__ ct_ntt, uint64_t *__restrict__ masked, MaskArgs M, DevParams P) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  const int t = threadIdx.x, L = P.L;
  const int64_t o = blockIdx.x;
  const int mn = M.m * M.n;
  uint64_t *dst = masked + (size_t)o * L * (mn + Gm::N) + (size_t)L * mn;
  for (int l = 0; l < L; l++) {
    const uint64_t p = pick(P, l).p;
    const uint64_t *src = ct_ntt + (ct_poly(M, o, 1) * L + l) * Gm::N;
    uint64_t x[16];
#pragma unroll
    for (int u = 0; u < 16; u++) {
      uint64_t v = __ldcs(src + slot_of<LOGN>(t, u));
      v = v >= 2 * p ? v - 2 * p : v;
      x[u] = v >= p ? v - p : v;
    }
    store_eval_slots<LOGN>(x, dst + (size_t)l * Gm::N, reinterpret_cast<uint64_t *>(sm), t, -1);
  }
}

// ---------------------------------------------------------------------------------------
// c0 of the compressed response, pruned (k_ntt_inv_mask computes c1).  Only the coefficients
// pos(i,k) = (k m + i) r + r - 1, the residue class r-1 mod r, are kept.  The
// first inverse round (distances 1..8) mixes every class; every later stage pairs indices >= 16
// apart, i.e. within a class when r <= 16.  Phase A: all threads run the first round of every
// prime and park the values in shared memory.  Phase B: per prime, NT/r threads -- the live
// "virtual threads" tv = 16 h + (r j + r - 1) of the remaining rounds -- finish the transform on
// their own warps, all primes concurrently: 1/r of the remaining butterflies.
// ---------------------------------------------------------------------------------------
template <int LOGN, int R>
__device__ __forceinline__ void inv_rounds_live(double (&a)[16], double *sm, int tv, bool act, int bar, int nbar,
                                                const double *tw, const PrimeConsts &pc) {
  if constexpr (R >= 0) {
    double wv[15];
    if (act) to_smem<LOGN, R + 1>(a, sm, tv);
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nbar) : "memory");
    if (act) from_smem<LOGN, R>(a, sm, tv);
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nbar) : "memory");
    if (act) load_round_tw<LOGN, R>(wv, tv, tw);
    if (act) inv_round<LOGN, R>(a, wv, pc);
    inv_rounds_live<LOGN, R - 1>(a, sm, tv, act, bar, nbar, tw, pc);
  }
}

// compact parking of the live class (q = idx >> log2 r, padded every 16): N/r words per prime
// instead of a full exchange buffer, so more CTAs fit per SM (and beside a co-resident MAC)
__device__ __forceinline__ int cpad(int q) { return q + (q >> 4); }
template <int LOGN, int R>
__device__ __forceinline__ void c_to_smem(const double (&a)[16], double *cv, int tv, int lr) {
  constexpr int K = Geom<LOGN>::k(R), G = 16 >> K;
#pragma unroll
  for (int g = 0; g < G; g++)
#pragma unroll
    for (int u = 0; u < (1 << K); u++) cv[cpad(elem_idx<LOGN, R>(tv, g, u) >> lr)] = a[g * (1 << K) + u];
}
template <int LOGN, int R>
__device__ __forceinline__ void c_from_smem(double (&a)[16], const double *cv, int tv, int lr) {
  constexpr int K = Geom<LOGN>::k(R), G = 16 >> K;
#pragma unroll
  for (int g = 0; g < G; g++)
#pragma unroll
    for (int u = 0; u < (1 << K); u++) a[g * (1 << K) + u] = cv[cpad(elem_idx<LOGN, R>(tv, g, u) >> lr)];
}
template <int LOGN, int R>
__device__ __forceinline__ void inv_rounds_live_c(double (&a)[16], double *cv, int tv, int lr, bool act, int bar,
                                                  int nbar, const double *tw, const PrimeConsts &pc) {
  if constexpr (R >= 0) {
    double wv[15];
    if (act) c_to_smem<LOGN, R + 1>(a, cv, tv, lr);
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nbar) : "memory");
    if (act) c_from_smem<LOGN, R>(a, cv, tv, lr);
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nbar) : "memory");
    if (act) load_round_tw<LOGN, R>(wv, tv, tw);
    if (act) inv_round<LOGN, R>(a, wv, pc);
    inv_rounds_live_c<LOGN, R - 1>(a, cv, tv, lr, act, bar, nbar, tw, pc);
  }
}

template <int LOGN, bool RR, bool CMP = false>
// (N = 8192 with compact parking: 2 CTAs per SM at 64 registers, a few bytes of spill -- phase B runs
// on 1/re of the threads, so a second CTA's phase A fills the SM: c4 inverse 126 -> 102 ms per stack)
__global__ void __launch_bounds__(Geom<LOGN>::NT, (CMP && LOGN == 12) ? 4 : (LOGN == 12 || CMP ? 2 : 1))
k_intt_c0_pruned(const uint64_t *__restrict__ ct_ntt, uint64_t *__restrict__ masked, uint64_t *__restrict__ share,
                 MaskArgs M, DevParams P) {
  using Gm = Geom<LOGN>;
  extern __shared__ double sm[];
  const int L = P.L;
  // the live class: r-1 mod re with re = min(r, 16) -- every stage after the first round pairs
  // indices >= 16 apart, so for r = 32 the kept class r-1 mod 32 needs its distance-16 partners
  // (class 15 mod 32) through the next stage: the class 15 mod 16 covers both
  const int re = M.r < 16 ? M.r : 16, lre = M.lr < 4 ? M.lr : 4;
  const int cw = cpad(Gm::N >> lre);                   // compact words per prime (CMP)
  uint64_t *sig_sm = reinterpret_cast<uint64_t *>(sm + (size_t)L * (CMP ? cw : Gm::SMEM_WORDS));
  int64_t *ext_sm = reinterpret_cast<int64_t *>(sig_sm + M.m * M.n);   // row f4: e1 + F at the kept positions
  const int t = threadIdx.x, warp = t >> 5;
  const int64_t o = blockIdx.x;                        // I_loc * nK + K
  const int64_t Iloc = o / M.nK, K = o % M.nK, I = M.i_begin + Iloc;
  const int mn = M.m * M.n, mr = M.m * M.r;
  const uint64_t tmask = (P.t_bits >= 64) ? ~0ull : ((1ull << P.t_bits) - 1);
  uint64_t *dst = masked + (size_t)o * L * (mn + Gm::N);
  const uint64_t stream = (uint64_t)(I * M.nK + K);
  mask_kept<RR>(M, stream, I, K, tmask, sig_sm, ext_sm, share, t, Gm::NT);
  // phase A: first inverse round of every prime (all threads)
  for (int l = 0; l < L; l++) {
    const PrimeConsts pc = pick(P, l);
    double a[16];
    if (M.c1_done) load_ntt_domain_q<LOGN>(a, ct_ntt + (ct_poly(M, o, 0) * L + l) * Gm::N, t, pc);
    else load_ntt_domain<LOGN>(a, ct_ntt + (ct_poly(M, o, 0) * L + l) * Gm::N, t, pc);
    if constexpr (RR) rr_add_ntt<LOGN>(a, M, o, 0, l, L, t, pc);
    { double wv[15]; load_round_tw<LOGN, Gm::NR - 1>(wv, t, P.twd_inv + (size_t)l * Gm::N); inv_round<LOGN, Gm::NR - 1>(a, wv, pc); }
    if constexpr (CMP) {                                // only the live class r-1 mod r is parked
      constexpr int K1 = Gm::k(Gm::NR - 1), G1 = 16 >> K1;
#pragma unroll
      for (int g = 0; g < G1; g++)
#pragma unroll
        for (int v = 0; v < (1 << K1); v++) {
          const int idx = elem_idx<LOGN, Gm::NR - 1>(t, g, v);
          if ((idx & (re - 1)) == re - 1) sm[(size_t)l * cw + cpad(idx >> lre)] = a[g * (1 << K1) + v];
        }
    } else {
      to_smem<LOGN, Gm::NR - 1>(a, sm + (size_t)l * Gm::SMEM_WORDS, t);
    }
  }
  __syncthreads();
  // phase B: prime l on warps [l*wpp, (l+1)*wpp)
  const int nlive = 16 / re, nact = Gm::NT / re, wpp = (nact + 31) / 32;
  if (warp >= L * wpp) return;
  const int l = warp / wpp, p = (warp % wpp) * 32 + (t & 31);
  const bool act = p < nact;
  const int tv = ((p / nlive) << 4) | (re * (p % nlive) + re - 1);
  const PrimeConsts pc = pick(P, l);
  const double *tw = P.twd_inv + (size_t)l * Gm::N;
  double *sml = sm + (size_t)l * (CMP ? cw : Gm::SMEM_WORDS);
  double a[16];
  if (act) {
    double wv[15];
    load_round_tw<LOGN, Gm::NR - 2>(wv, tv, tw);
    if constexpr (CMP) c_from_smem<LOGN, Gm::NR - 2>(a, sml, tv, lre);
    else from_smem<LOGN, Gm::NR - 2>(a, sml, tv);
    inv_round<LOGN, Gm::NR - 2>(a, wv, pc);
  }
  if constexpr (CMP) inv_rounds_live_c<LOGN, Gm::NR - 3>(a, sml, tv, lre, act, 1 + l, wpp * 32, tw, pc);
  else inv_rounds_live<LOGN, Gm::NR - 3>(a, sml, tv, act, 1 + l, wpp * 32, tw, pc);
  if (!act) return;
  constexpr int K0 = Gm::k(0), G = 16 >> K0;
#pragma unroll
  for (int g = 0; g < G; g++)
#pragma unroll
    for (int u = 0; u < (1 << K0); u++) {
      const int idx = elem_idx<LOGN, 0>(tv, g, u);
      if (idx < mr * M.n && (idx & (M.r - 1)) == M.r - 1) {   // r-1 mod re by construction; kept: r-1 mod r
        uint64_t x = d2u(canon_d(a[g * (1 << K0) + u], pc.pd, pc.pinv));
        const int kk = idx >> M.lr;
        if constexpr (RR) { x += smod(ext_sm[kk], pc); x = x >= pc.p ? x - pc.p : x; }
        uint64_t d = shoup_mul(sig_sm[kk], pc.delta, pc.delta_sh, pc.p);
        d = d >= pc.p ? d - pc.p : d;
        dst[(size_t)l * mn + kk] = x >= d ? x - d : x + pc.p - d;
      }
    }
}

// ---------------------------------------------------------------------------------------
// Unfused mask_and_share: CTA per output ct, one thread per ChaCha block: MASK words 8b .. 8b+7
// (reading C27 order: positions mask_pos(w)) for c0 and the share, positions 8b .. 8b+7 for c1.
// ---------------------------------------------------------------------------------------
__global__ void k_mask(const uint64_t *__restrict__ ct_out, uint64_t *__restrict__ masked,
                       uint64_t *__restrict__ share, MaskArgs M, DevParams P, int compress) {
  const int N = P.N, L = P.L;
  const int64_t o = blockIdx.y;
  const int64_t Iloc = o / M.nK, K = o % M.nK, I = M.i_begin + Iloc;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= N / 8) return;
  const int mn = M.m * M.n;
  const uint64_t tmask = (P.t_bits >= 64) ? ~0ull : ((1ull << P.t_bits) - 1);
  const size_t per = compress ? (size_t)L * (mn + N) : (size_t)2 * L * N;
  const uint64_t *src = ct_out + (size_t)o * 2 * L * N;
  uint64_t *dst = masked + (size_t)o * per;
  const bool words = !compress || 8 * b < mn;
  uint64_t sig[8];
  if (words) {
    hl::chacha_block_u64(M.seed, hl::kDomMask, (uint64_t)(I * M.nK + K), (uint32_t)b, sig);
#pragma unroll
    for (int q = 0; q < 8; q++) sig[q] &= tmask;
  }
  for (int l = 0; l < L; l++) {
    const PrimeConsts pc = pick(P, l);
    const uint64_t *c0 = src + (size_t)l * N, *c1 = src + (size_t)(L + l) * N;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int w = 8 * b + q;
      if (words && (!compress || w < mn)) {
        const int pos = mask_pos(M, w);
        uint64_t d = shoup_mul(sig[q], pc.delta, pc.delta_sh, pc.p);
        d = d >= pc.p ? d - pc.p : d;
        const uint64_t x = c0[pos];
        const uint64_t y = x >= d ? x - d : x + pc.p - d;
        if (compress) dst[(size_t)l * mn + w] = y;            // kept word w = kept index k m + i
        else dst[(size_t)l * N + pos] = y;
      }
      const int pos = 8 * b + q;                                // c1 (evaluation form) passes through
      if (compress) dst[(size_t)L * mn + (size_t)l * N + pos] = c1[pos];
      else dst[(size_t)(L + l) * N + pos] = c1[pos];
    }
  }
#pragma unroll
  for (int q = 0; q < 8; q++) {
    const int w = 8 * b + q;
    if (words && w < mn) {
      const int64_t row = K * M.n + (w >> M.lm), col = I * M.m + (w & (M.m - 1));
      if (row < M.Nb && col < M.Ma) share[row * M.Ma + col] = sig[q];
    }
  }
}

// ---------------------------------------------------------------------------------------
// Slot-parallel modular MAC (the dominant kernel), persistent and warp-specialised.
//   out[I][col][s] (+)= sum_{J in [j0, j1)} W[I][J][s] * X[J][col][s]  mod p_{s / N}
// A tile is 16 rows (I) x 32 slots x CW columns.  Warp 8 (producer) streams, for every J, the
// tile's W chunk (4 KB) and X chunk (256*CW B) into a NST-deep shared-memory ring with
// cp.async.bulk (TMA bulk copies completing on mbarriers).  Warps 0-7 (consumers) each own 4
// slots: lane = (row = lane & 15, slot pair half = lane >> 4), 2 slots x CW columns per thread,
// three IMAD.WIDE.U32 per modular MAC (Karatsuba on 25-bit limbs) into exact 64-bit lazy
// accumulators.  The epilogue reduces mod p (one 128-bit reduction per output), transposes
// through shared memory and stores 256-B rows of out[I][col][LN] (the inverse NTT's input).
// ---------------------------------------------------------------------------------------
struct MacArgs {
  const uint2 *W;
  const uint32_t *X;
  uint64_t *out;
  MacGeom g;
  int N, j0, j1, accumulate;
};

template <int CW>
struct MacSmem {
  static constexpr int W_BYTES = 32 * 16 * 8;
  static constexpr int X_BYTES = 32 * CW * 12;
  static constexpr int STAGE = W_BYTES + X_BYTES;
  static constexpr int E_STRIDE = CW * 32 + 1;               // odd row stride: conflict-free transpose
  static constexpr int E_BYTES = 16 * E_STRIDE * 8;
};

constexpr int kMacStages = 16;                     // IMAD engine ring depth (16 x 7 KB in flight per SM)
constexpr int kMacConsumerWarps = 16;                      // one slot per thread, 2 slots per warp
constexpr int kMacThreads = (kMacConsumerWarps + 1) * 32;  // + 1 producer warp

template <int CW, int LN, int NST>
__global__ void __launch_bounds__(kMacThreads, 1)
k_mac(MacArgs A, DevParams P) {
  using S = MacSmem<CW>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + NST * S::STAGE + S::E_BYTES);
  uint64_t *empty = full + NST;
  uint64_t *ebuf = reinterpret_cast<uint64_t *>(smem + NST * S::STAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const MacGeom &g = A.g;
  const int ntiles = g.nIb * g.nCg * g.nSb;
  const int nj = A.j1 - A.j0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], kMacConsumerWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kMacConsumerWarps) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      int st = 0;
      uint32_t phase = 1;                 // a fresh empty barrier completes "phase -1" (parity 1)
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int ib = tile % g.nIb, cg = (tile / g.nIb) % g.nCg, sb = tile / (g.nIb * g.nCg);
        const uint2 *wsrc = A.W + (((size_t)ib * g.nSb + sb) * g.nJ + A.j0) * 512;
        const uint32_t *xsrc = A.X + x_chunk(g, A.j0, cg, sb);
        for (int j = 0; j < nj; j++) {
          mbar_wait(&empty[st], phase);
          unsigned char *dst = smem + st * S::STAGE;
          mbar_expect_tx(&full[st], S::STAGE);
          bulk_g2s(dst, wsrc + (size_t)j * 512, S::W_BYTES, &full[st]);
          bulk_g2s(dst + S::W_BYTES, xsrc + (size_t)j * 96 * CW, S::X_BYTES, &full[st]);
          if (++st == NST) { st = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  const int row = lane & 15;
  const int sl = 2 * warp + (lane >> 4);            // this thread's slot within the 32-slot block
  constexpr int NCT = kMacConsumerWarps * 32;
  int st = 0;
  uint32_t phase = 0;
  const int woff = (sl * 16 + row) * 8, xoff = S::W_BYTES + sl * CW * 8, soff = S::W_BYTES + 32 * CW * 8 + sl * CW * 4;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int ib = tile % g.nIb, cg = (tile / g.nIb) % g.nCg, sb = tile / (g.nIb * g.nCg);
    uint64_t lo[CW], hi[CW], md[CW];
#pragma unroll
    for (int b = 0; b < CW; b++) lo[b] = hi[b] = md[b] = 0;

#pragma unroll 1
    for (int j = 0; j < nj; j++) {
      mbar_wait(&full[st], phase);
      const unsigned char *stage = smem + st * S::STAGE;
      const uint2 w = *reinterpret_cast<const uint2 *>(stage + woff);
      uint2 x[CW];
      uint32_t xs[CW];
#pragma unroll
      for (int q = 0; q < CW / 2; q++) {
        const uint4 v = *reinterpret_cast<const uint4 *>(stage + xoff + 16 * q);
        x[2 * q] = make_uint2(v.x, v.y); x[2 * q + 1] = make_uint2(v.z, v.w);
      }
      if constexpr (CW >= 4) {
#pragma unroll
        for (int q = 0; q < CW / 4; q++) {
          const uint4 v = *reinterpret_cast<const uint4 *>(stage + soff + 16 * q);
          xs[4 * q] = v.x; xs[4 * q + 1] = v.y; xs[4 * q + 2] = v.z; xs[4 * q + 3] = v.w;
        }
      } else {
        const uint2 v = *reinterpret_cast<const uint2 *>(stage + soff);
        xs[0] = v.x; xs[1] = v.y;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);       // operands are in registers: release the stage
      if (++st == NST) { st = 0; phase ^= 1; }
      const uint32_t ws = w.x + w.y;
#pragma unroll
      for (int b = 0; b < CW; b++) {
        lo[b] += (uint64_t)w.x * x[b].x;
        hi[b] += (uint64_t)w.y * x[b].y;
        md[b] += (uint64_t)ws * xs[b];
      }
    }

    // ---------------- epilogue: reduce, transpose through smem, coalesced stores
    const int l = (sb * 32) / A.N;
    const PrimeConsts pc = pick(P, l);
    asm volatile("bar.sync 1, %0;" ::"r"(NCT) : "memory");     // previous tile's ebuf reads are done
#pragma unroll
    for (int b = 0; b < CW; b++) {
      const uint64_t mid = md[b] - lo[b] - hi[b];                      // exact: x0 y1 + x1 y0
      const hl_u128 V = ((hl_u128)hi[b] << (2 * kLimbBits)) + ((hl_u128)mid << kLimbBits) + lo[b];
      const uint64_t vh = (uint64_t)(V >> 64), vl = (uint64_t)V;
      const uint64_t r1 = shoup_mul(vh, pc.r64, pc.r64_sh, pc.p);    // vh * 2^64 mod p, [0, 2p)
      const uint64_t r2 = vl - __umul64hi(vl, pc.mu) * pc.p;         // vl mod p, [0, 2p)
      uint64_t r = r1 + r2;
      r = r >= pc.two_p ? r - pc.two_p : r;
      r = r >= pc.p ? r - pc.p : r;
      ebuf[row * S::E_STRIDE + b * 32 + sl] = r;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NCT) : "memory");
    const int I0 = ib * 16;
    for (int e = threadIdx.x; e < 16 * CW * 32; e += NCT) {
      const int rr = e / (CW * 32), b = (e / 32) % CW, s2 = e % 32;
      if (I0 + rr >= g.nIs) continue;
      uint64_t v = ebuf[rr * S::E_STRIDE + b * 32 + s2];
      uint64_t *dst = A.out + ((size_t)(I0 + rr) * g.nC + cg * CW + b) * LN + sb * 32 + s2;
      if (A.accumulate) {
        v += *dst;
        v = v >= pc.p ? v - pc.p : v;
      }
      *dst = v;
    }
  }
}

// ---------------------------------------------------------------------------------------
// FP64 MAC engine (default).  Same tiling, ring and epilogue as k_mac; the exact product of
// two residues a = W, b = X < 2^50 (held as doubles, exact) is formed with error-free FP64
// transformations on the DFMA pipe (57 /clk/SM vs 24 for IMAD.WIDE, profiles/r01):
//   t  = fma(a * 2^-49, b, C)            C = 1.5 * 2^52:  t = C + hi, hi = round(a b / 2^49) < 2^51
//   c  = fma(t, -2^49, C * 2^49)         = -hi * 2^49   (exact: 51 significant bits)
//   r  = fma(a, b, c)                    = a b - hi 2^49, |r| <= 2^48, exact
//   H += bits(t)  (u64; subtract nj*bits(C) at the end)     R += r  (exact for 32 terms)
// R is flushed to an int64 every 32 J.  sum_J a b = (H - nj bits(C)) * 2^49 + R_total exactly.
// ---------------------------------------------------------------------------------------
template <int CW, int JPS>
struct MacSmemF64 {
  static constexpr int W_BYTES = 32 * 16 * 8;             // per J
  static constexpr int X_BYTES = 32 * CW * 8;             // per J
  static constexpr int STAGE = JPS * (W_BYTES + X_BYTES); // JPS consecutive J per stage
  static constexpr int E_STRIDE = CW * 32 + 1;
  static constexpr int E_BYTES = 16 * E_STRIDE * 8;
};

template <int CW, int LN, int NST, int JPS>
__global__ void __launch_bounds__(kMacThreads, 1)
k_mac_f64(MacArgs A, DevParams P) {
  using S = MacSmemF64<CW, JPS>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + NST * S::STAGE + S::E_BYTES);
  uint64_t *empty = full + NST;
  uint64_t *ebuf = reinterpret_cast<uint64_t *>(smem + NST * S::STAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const MacGeom &g = A.g;
  const int ntiles = g.nIb * g.nCg * g.nSb;
  const int nj = A.j1 - A.j0;
  const int nstage = (nj + JPS - 1) / JPS;                // stages per tile

  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], kMacConsumerWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kMacConsumerWarps) {
    if (lane == 0) {
      int st = 0;
      uint32_t phase = 1;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int ib = tile % g.nIb, cg = (tile / g.nIb) % g.nCg, sb = tile / (g.nIb * g.nCg);
        const double *wsrc = reinterpret_cast<const double *>(A.W) + (((size_t)ib * g.nSb + sb) * g.nJ + A.j0) * 512;
        const uint32_t *xsrc = A.X + x_chunk(g, A.j0, cg, sb);
        for (int k = 0; k < nstage; k++) {
          const int jn = min(JPS, nj - k * JPS);
          mbar_wait(&empty[st], phase);
          unsigned char *dst = smem + st * S::STAGE;
          mbar_expect_tx(&full[st], jn * (S::W_BYTES + S::X_BYTES));
          bulk_g2s(dst, wsrc + (size_t)k * JPS * 512, jn * S::W_BYTES, &full[st]);
          bulk_g2s(dst + JPS * S::W_BYTES, xsrc + (size_t)k * JPS * 64 * CW, jn * S::X_BYTES, &full[st]);
          if (++st == NST) { st = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  const int row = lane & 15;
  const int sl = 2 * warp + (lane >> 4);
  constexpr int NCT = kMacConsumerWarps * 32;
  constexpr double kC = 6755399441055744.0;                          // 1.5 * 2^52
  constexpr double kC49 = 6755399441055744.0 * 562949953421312.0;   // C * 2^49
  constexpr double kM49 = -562949953421312.0;                       // -2^49
  constexpr double kS49 = 1.7763568394002505e-15;                   // 2^-49
  const uint64_t kCbits = 0x4338000000000000ull;                    // bit pattern of C
  int st = 0;
  uint32_t phase = 0;
  const int woff = (sl * 16 + row) * 8, xoff = JPS * S::W_BYTES + sl * CW * 8;

  // one J step: t = C + round(w x / 2^49) -> H; r = w x - (t - C) 2^49 -> R  (all exact)
  auto mac_step = [&](const unsigned char *wp, const unsigned char *xp, uint64_t (&H)[CW], double (&R)[CW]) {
    const double w = *reinterpret_cast<const double *>(wp);
    double x[CW];
#pragma unroll
    for (int q = 0; q < CW / 2; q++) {
      const double2 v = *reinterpret_cast<const double2 *>(xp + 16 * q);
      x[2 * q] = v.x; x[2 * q + 1] = v.y;
    }
    const double ws = w * kS49;                                       // exact
    double t[CW];
#pragma unroll
    for (int b = 0; b < CW; b++) t[b] = __fma_rn(ws, x[b], kC);
#pragma unroll
    for (int b = 0; b < CW; b++) H[b] += (uint64_t)__double_as_longlong(t[b]);
#pragma unroll
    for (int b = 0; b < CW; b++) t[b] = __fma_rn(t[b], kM49, kC49);    // -hi * 2^49
#pragma unroll
    for (int b = 0; b < CW; b++) t[b] = __fma_rn(w, x[b], t[b]);       // w x - hi 2^49
#pragma unroll
    for (int b = 0; b < CW; b++) R[b] = __dadd_rn(R[b], t[b]);
  };
  // |R| <= 32 * 2^48: move round(R / 2^49) into H (same magic), keep the exact remainder in R
  auto flush = [&](uint64_t (&H)[CW], double (&R)[CW]) {
#pragma unroll
    for (int b = 0; b < CW; b++) {
      const double t2 = __fma_rn(R[b], kS49, kC);
      H[b] += (uint64_t)__double_as_longlong(t2);
      R[b] = __dadd_rn(R[b], __fma_rn(t2, kM49, kC49));
    }
  };

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int ib = tile % g.nIb, cg = (tile / g.nIb) % g.nCg, sb = tile / (g.nIb * g.nCg);
    uint64_t H[CW];
    double R[CW];
#pragma unroll
    for (int b = 0; b < CW; b++) { H[b] = 0; R[b] = 0.0; }
    int nmagic = 0;                                   // number of C offsets added into H

#pragma unroll 1
    for (int k = 0; k < nstage; k++) {
      const int jn = min(JPS, nj - k * JPS);
      mbar_wait(&full[st], phase);
      const unsigned char *stage = smem + st * S::STAGE;
      if (jn == JPS) {
#pragma unroll
        for (int jj = 0; jj < JPS; jj++)
          mac_step(stage + jj * S::W_BYTES + woff, stage + xoff + jj * S::X_BYTES, H, R);
      } else {
#pragma unroll 1
        for (int jj = 0; jj < jn; jj++)
          mac_step(stage + jj * S::W_BYTES + woff, stage + xoff + jj * S::X_BYTES, H, R);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == NST) { st = 0; phase ^= 1; }
      nmagic += jn;
      if (((k + 1) * JPS) % 32 == 0) { flush(H, R); nmagic++; }
    }
    flush(H, R);                                      // |R| <= 2^48 afterwards
    nmagic++;

    const int l = (sb * 32) / A.N;
    const PrimeConsts pc = pick(P, l);
    asm volatile("bar.sync 1, %0;" ::"r"(NCT) : "memory");
#pragma unroll
    for (int b = 0; b < CW; b++) {
      const uint64_t hi = H[b] - (uint64_t)nmagic * kCbits;            // sum of the rounded 2^49 parts
      const int64_t lo = __double2ll_rn(R[b]);                         // exact remainder, |lo| <= 2^48
      const hl_u128 V = ((hl_u128)hi << 49) + (hl_u128)(__int128)lo;  // exact sum_J a b >= 0
      const uint64_t vh = (uint64_t)(V >> 64), vl = (uint64_t)V;
      const uint64_t r1 = shoup_mul(vh, pc.r64, pc.r64_sh, pc.p);
      const uint64_t r2 = vl - __umul64hi(vl, pc.mu) * pc.p;
      uint64_t r = r1 + r2;
      r = r >= pc.two_p ? r - pc.two_p : r;
      r = r >= pc.p ? r - pc.p : r;
      ebuf[row * S::E_STRIDE + b * 32 + sl] = r;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NCT) : "memory");
    const int I0 = ib * 16;
    for (int e = threadIdx.x; e < 16 * CW * 32; e += NCT) {
      const int rr = e / (CW * 32), b = (e / 32) % CW, s2 = e % 32;
      if (I0 + rr >= g.nIs) continue;
      uint64_t v = ebuf[rr * S::E_STRIDE + b * 32 + s2];
      uint64_t *dst = A.out + ((size_t)(I0 + rr) * g.nC + cg * CW + b) * LN + sb * 32 + s2;
      if (A.accumulate) {
        v += *dst;
        v = v >= pc.p ? v - pc.p : v;
      }
      *dst = v;
    }
  }
}

#include "mac_tc.cuh"
#include "fc.cuh"
#include "client_dev.cuh"

// pointwise product in the NTT domain (diagnostics only)
__global__ void k_pointwise(const uint64_t *a, const uint64_t *b, uint64_t *out, int64_t n, DevParams P) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int l = (int)((i / P.N) % P.L);
  const uint64_t p = pick(P, l).p;
  out[i] = (uint64_t)(((hl_u128)a[i] * b[i]) % p);
}

// ---------------------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------------------
// one-time kernel attribute setup per DEVICE (cudaFuncSetAttribute applies to the current device):
// a second context on another device in the same process sets its own
struct PerDevice {
  std::atomic<uint64_t> done{0};
  bool first() {
    int d = 0;
    cudaGetDevice(&d);
    const uint64_t b = 1ull << (d & 63);
    return (done.fetch_or(b) & b) == 0;
  }
};

template <typename Kern>
void set_smem(Kern k, size_t bytes) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int LOGN>
constexpr size_t ntt_smem() { return (size_t)Geom<LOGN>::SMEM_WORDS * 8; }

template <int LOGN, int MODE>
void launch_fwd(const hl_ctx *c, const uint64_t *in, void *out, int64_t npoly, const MacGeom &mg, cudaStream_t st) {
  static PerDevice init;
  if (init.first()) { set_smem(k_ntt_fwd<LOGN, MODE>, ntt_smem<LOGN>()); }
  dim3 grid((unsigned)npoly, c->L);
  KTimer kt(c, MODE ? HL_K_NTT_FWD : HL_K_OTHER, st);
  k_ntt_fwd<LOGN, MODE><<<grid, Geom<LOGN>::NT, ntt_smem<LOGN>(), st>>>(in, out, c->dp, mg);
}

template <int LOGN>
void launch_inv(const hl_ctx *c, const uint64_t *in, uint64_t *out, int64_t npoly, cudaStream_t st, int ct_mode) {
  static PerDevice init;
  if (init.first()) { set_smem(k_ntt_inv<LOGN>, ntt_smem<LOGN>()); }
  dim3 grid((unsigned)npoly, c->L);
  KTimer kt(c, HL_K_INTT, st);
  k_ntt_inv<LOGN><<<grid, Geom<LOGN>::NT, ntt_smem<LOGN>(), st>>>(in, out, c->dp, ct_mode);
}

template <int LOGN, int G>
void launch_fwd_x(const hl_ctx *c, const uint64_t *in, void *out, int64_t npoly, const MacGeom &mg, cudaStream_t st) {
  constexpr size_t smem = ntt_smem<LOGN>() * G;
  static PerDevice init;
  if (init.first()) { set_smem(k_ntt_fwd_x<LOGN, G>, smem); }
  dim3 grid((unsigned)(npoly / G), c->L);
  KTimer kt(c, HL_K_NTT_FWD, st);
  k_ntt_fwd_x<LOGN, G><<<grid, Geom<LOGN>::NT * G, smem, st>>>(in, (uint64_t *)out, c->dp, mg);
}


// CTAs of kernel k resident on the device at once (one wave): the L2 prefetch distance of the NTT kernels
template <typename Kern>
int wave_ctas(const hl_ctx *c, Kern k, int threads, size_t smem) {
  if (threads < 512) return 0;             // N = 4096 kernels: off (see k_ntt_fwd_c0x2)
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, threads, smem) != cudaSuccess) { cudaGetLastError(); return 0; }
  return n * c->num_sms;
}

template <int LOGN>
void launch_fwd_cperm(const hl_ctx *c, const uint64_t *in, uint64_t *out, int64_t npoly, const MacGeom &mg_in,
                      cudaStream_t st) {
  MacGeom mg = mg_in;
  const int nK = mg.nC / 2;
  const int64_t nJ = npoly / mg.nC;
  constexpr size_t smem2 = ntt_smem<LOGN>() * 2;
  constexpr int MB2 = LOGN == 12 ? 2 : 1;             // explicit: minBlocks 1 lets the kernel grow to 1 CTA/SM
  static PerDevice init;
  if (init.first()) {
    set_smem(k_ntt_fwd_c0x2<LOGN, false, MB2>, smem2); set_smem(k_ntt_fwd_c0x2<LOGN, true>, smem2);
    if constexpr (LOGN == 12) {
      set_smem(k_ntt_fwd_c0x2<LOGN, true, 3>, smem2);
      set_smem(k_ntt_fwd_c0x2<LOGN, false, 3>, smem2);
    }
    set_smem(k_c1_to_x<LOGN, 4>, 4 * (size_t)Geom<LOGN>::N * 8); set_smem(k_c1_to_x<LOGN, 2>, 2 * (size_t)Geom<LOGN>::N * 8);
    set_smem(k_c1_to_x<LOGN, 1>, (size_t)Geom<LOGN>::N * 8);
  }
  KTimer kt(c, HL_K_NTT_FWD, st);
  if (mg.c1_in) {                                  // c1 is read by the MAC itself: c0 pairs only
    const dim3 gx((unsigned)(nJ * ((nK + 1) / 2)), c->L);
    if constexpr (LOGN == 12) {
      mg.pf = wave_ctas(c, k_ntt_fwd_c0x2<LOGN, false, 3>, Geom<LOGN>::NT, smem2);
      k_ntt_fwd_c0x2<LOGN, false, 3><<<gx, Geom<LOGN>::NT, smem2, st>>>(in, out, c->dp, mg);
    }
    else {
      mg.pf = wave_ctas(c, k_ntt_fwd_c0x2<LOGN, false, MB2>, Geom<LOGN>::NT, smem2);
      k_ntt_fwd_c0x2<LOGN, false, MB2><<<gx, Geom<LOGN>::NT, smem2, st>>>(in, out, c->dp, mg);
    }
    return;
  }
  // c1 pairs (K0, K0+1) adjacent in the c1 column range, copied by the c0 kernel; whole 16-column
  // c1 groups go to k_c1_tx16 instead (128-B line stores)
  const bool fused = nK % 2 == 0 && !(mg.CW == 16 && nK % 16 == 0);
  kt.nk = fused ? 1 : 2;
  if constexpr (LOGN == 12) {
    if (fused) {   // N = 4096: 3 CTAs per SM (80 registers, a few bytes of spill; measured best)
      const dim3 gx((unsigned)(nJ * ((nK + 1) / 2)), c->L);
      {
        mg.pf = wave_ctas(c, k_ntt_fwd_c0x2<LOGN, true, 3>, Geom<LOGN>::NT, smem2);
        k_ntt_fwd_c0x2<LOGN, true, 3><<<gx, Geom<LOGN>::NT, smem2, st>>>(in, out, c->dp, mg);
      }
      return;
    }
  }
  if (fused) {
    {
      mg.pf = wave_ctas(c, k_ntt_fwd_c0x2<LOGN, true>, Geom<LOGN>::NT, smem2);
      k_ntt_fwd_c0x2<LOGN, true><<<dim3((unsigned)(nJ * ((nK + 1) / 2)), c->L), Geom<LOGN>::NT, smem2, st>>>(in, out, c->dp, mg);
    }
    return;
  }
  // odd nK (or whole 16-column c1 groups): the c0 pairs without their c1, then the c1 reordering
  {
    mg.pf = wave_ctas(c, k_ntt_fwd_c0x2<LOGN, false, MB2>, Geom<LOGN>::NT, smem2);
    k_ntt_fwd_c0x2<LOGN, false, MB2><<<dim3((unsigned)(nJ * ((nK + 1) / 2)), c->L), Geom<LOGN>::NT, smem2, st>>>(in, out, c->dp, mg);
  }
  if (mg.CW == 16 && nK % 16 == 0) {
    k_c1_tx16<LOGN><<<dim3((unsigned)(Geom<LOGN>::N / 256), (unsigned)(nJ * (nK / 16)), c->L), 256, 0, st>>>(in, out, c->dp, mg);
    return;
  }
  // G1 = 4 needs 4 | nK and 4 | CW (the 4 columns in one group); 4 x 64 KB does not fit at N = 8192
  const int G1 = (nK % 4 == 0 && mg.CW % 4 == 0 && LOGN == 12) ? 4 : (nK % 2 == 0 ? 2 : 1);
  const dim3 g1((unsigned)(nJ * (nK / G1)), c->L);
  constexpr size_t pb = (size_t)Geom<LOGN>::N * 8;
  if (G1 == 4) k_c1_to_x<LOGN, 4><<<g1, Geom<LOGN>::NT, 4 * pb, st>>>(in, out, c->dp, mg);
  else if (G1 == 2) k_c1_to_x<LOGN, 2><<<g1, Geom<LOGN>::NT, 2 * pb, st>>>(in, out, c->dp, mg);
  else k_c1_to_x<LOGN, 1><<<g1, Geom<LOGN>::NT, pb, st>>>(in, out, c->dp, mg);
}

// MODE 0 (u64, slot order) when mg == nullptr, else MODE 1 (the MAC engine's X layout)
void fwd_ntt(const hl_ctx *c, const uint64_t *in, void *out, int64_t npoly, const MacGeom *mg, cudaStream_t st) {
  if (mg && mg->engine == 2 && mg->cperm) {
    if (c->N == 4096) launch_fwd_cperm<12>(c, in, (uint64_t *)out, npoly, *mg, st);
    else launch_fwd_cperm<13>(c, in, (uint64_t *)out, npoly, *mg, st);
    return;
  }
  if (mg && mg->engine == 2) {
    // G consecutive polynomials share J and a column group (G divides CW)
    // (CW >= 2 always, so 2 divides it)
    if (c->N == 4096) launch_fwd_x<12, 2>(c, in, out, npoly, *mg, st);
    else launch_fwd_x<13, 2>(c, in, out, npoly, *mg, st);
    return;
  }
  MacGeom z{};
  if (c->N == 4096) { if (mg) launch_fwd<12, 1>(c, in, out, npoly, *mg, st); else launch_fwd<12, 0>(c, in, out, npoly, z, st); }
  else { if (mg) launch_fwd<13, 1>(c, in, out, npoly, *mg, st); else launch_fwd<13, 0>(c, in, out, npoly, z, st); }
}

// ct_mode: the polynomials are ciphertext halves (c0, c1, c0, ...): c1 is only reordered to the
// boundary's evaluation form (reading C26)
void inv_ntt(const hl_ctx *c, const uint64_t *in, uint64_t *out, int64_t npoly, cudaStream_t st, int ct_mode = 0) {
  if (c->N == 4096) launch_inv<12>(c, in, out, npoly, st, ct_mode); else launch_inv<13>(c, in, out, npoly, st, ct_mode);
}

template <int CW, int LN>
void launch_mac_t(const hl_ctx *c, const MacArgs &A, cudaStream_t st) {
  using S = MacSmem<CW>;
  constexpr size_t smem = (size_t)kMacStages * S::STAGE + S::E_BYTES + 2 * kMacStages * 8;
  static PerDevice init;
  if (init.first()) { set_smem(k_mac<CW, LN, kMacStages>, smem); }
  const int ntiles = A.g.nIb * A.g.nCg * A.g.nSb;
  const int grid = std::min(ntiles, c->num_sms);
  KTimer kt(c, HL_K_MAC, st);
  k_mac<CW, LN, kMacStages><<<grid, kMacThreads, smem, st>>>(A, c->dp);
}

constexpr int kMacF64Jps = 4;                    // J steps per ring stage (one bulk copy pair)
constexpr int kMacF64Stages = 6;                 // 6 x 4 x 6 KB = 144 KB in flight per SM at CW = 8

template <int CW, int LN>
void launch_mac_f64_t(const hl_ctx *c, const MacArgs &A, cudaStream_t st) {
  using S = MacSmemF64<CW, kMacF64Jps>;
  constexpr size_t smem = (size_t)kMacF64Stages * S::STAGE + S::E_BYTES + 2 * kMacF64Stages * 8;
  static PerDevice init;
  if (init.first()) { set_smem(k_mac_f64<CW, LN, kMacF64Stages, kMacF64Jps>, smem); }
  const int ntiles = A.g.nIb * A.g.nCg * A.g.nSb;
  const int grid = std::min(ntiles, c->num_sms);
  KTimer kt(c, HL_K_MAC, st);
  k_mac_f64<CW, LN, kMacF64Stages, kMacF64Jps><<<grid, kMacThreads, smem, st>>>(A, c->dp);
}

template <int LN>
void launch_mac_ln(const hl_ctx *c, const MacArgs &A, cudaStream_t st) {
  if (A.g.f64) {
    if (A.g.CW == 8) launch_mac_f64_t<8, LN>(c, A, st);
    else if (A.g.CW == 4) launch_mac_f64_t<4, LN>(c, A, st);
    else launch_mac_f64_t<2, LN>(c, A, st);
  } else {
    if (A.g.CW == 8) launch_mac_t<8, LN>(c, A, st);
    else if (A.g.CW == 4) launch_mac_t<4, LN>(c, A, st);
    else launch_mac_t<2, LN>(c, A, st);
  }
}

template <int CW>
void launch_mac_tc_t(const hl_ctx *c, MacTcArgs A, int smem_budget, int grid, cudaStream_t st) {
  using T = TcGeom<CW>;
  static PerDevice init;
  if (init.first()) { set_smem(k_mac_tc<CW, true>, T::SMEM_MAX); set_smem(k_mac_tc<CW, false>, T::SMEM_MAX); }
  bool fast = true;             // the fast epilogue recombination needs 2^50 - p < 2^27 for every prime
  for (uint32_t l = 0; l < c->L; l++) fast = fast && c->dp.pc[l].mc != 0 && c->dp.pc[l].mc < (1ull << 27);
  // pure column groups (every group all c0 or all c1): a stage holds the X residues or the c1 box
  A.ring = tc_ring<CW>(A.g.RT, smem_budget, A.c1_bytes, A.c1_in && A.c1_nK % CW == 0);
  // diagnostics: HELINEAR_MAC_PROF=1 with a -DHL_MAC_PROF build (HELINEAR_NVCC_EXTRA) prints, per
  // launch, the average cycles per CTA each role waits (mac_tc.cuh)
#ifdef HL_MAC_PROF
  static const bool prof = getenv("HELINEAR_MAC_PROF") != nullptr;
#else
  constexpr bool prof = false;
#endif
  A.prof = nullptr;
  if (prof) cudaMalloc(&A.prof, 10 * sizeof(unsigned long long)), cudaMemsetAsync(A.prof, 0, 80, st);
  {
  KTimer kt(c, HL_K_MAC, st);
  if (fast) k_mac_tc<CW, true><<<grid, T::THREADS, A.ring.smem, st>>>(A, c->dp);
  else k_mac_tc<CW, false><<<grid, T::THREADS, A.ring.smem, st>>>(A, c->dp);
  }
  if (prof) {   // diagnostics: average cycles per CTA waiting, by role
    unsigned long long h[10];
    cudaMemcpyAsync(h, A.prof, 80, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const double n = c->num_sms;
    fprintf(stderr, "[mac_tc CW=%d nIs=%d nJ=%d RT=%d nst=%d sb=%d] total %.0f | prod.empty %.0f | mma.tempty %.0f "
            "mma.full %.0f mma.zfull %.0f mma.issue %.0f | conv.full %.0f | epi.tfull %.0f epi.drain %.0f epi.fold_store %.0f (cycles/CTA)\n", CW, A.g.nIs,
            A.g.nJ, A.g.RT, A.ring.nst, A.ring.sbytes, h[7] / n, h[0] / n, h[1] / n, h[2] / n, h[3] / n, h[6] / n,
            h[4] / n, h[5] / n, h[8] / n, h[9] / n);
    cudaFree(A.prof);
  }
}

// the tensor-core engine's workspace = X residues [nCg][LN][nJp][CW] u64 + 256 B of scheduler state
inline size_t tc_sched_offset(const MacGeom &g) { return (size_t)g.nJp * g.nC * g.LN * 8; }

// cuTensorMapEncodeTiled through the runtime (no -lcuda): nullptr if the driver lacks it
using TmapEncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncodeFn tmap_encode() {
  static TmapEncodeFn fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (TmapEncodeFn)p;
  }();
  return fn;
}
// the c1 halves of ct_in [nJ][nK][2][L][N] as a 3-D tensor (k over all primes, K, J) of u64; a box
// is {2 natural points, the group's c1 columns, 32 J} -> shared [J][K][2] (rows J >= nJ zero-filled)
static bool c1_tmap(CUtensorMap *m, const uint64_t *ct_in, int64_t LN, int64_t nK, int64_t nJ, int cols) {
  const TmapEncodeFn enc = tmap_encode();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)LN, (cuuint64_t)nK, (cuuint64_t)nJ};
  const cuuint64_t strides[2] = {(cuuint64_t)(2 * LN * 8), (cuuint64_t)(nK * 2 * LN * 8)};
  const cuuint32_t box[3] = {2, (cuuint32_t)cols, 32}, es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint64_t *>(ct_in + LN), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_mac_tc(const hl_ctx *c, const void *W, const void *X, uint64_t *out, const MacGeom &g, int smem_budget,
                   int grid, cudaStream_t st, const MaskArgs *c1m = nullptr, uint64_t *c1_masked = nullptr,
                   const uint64_t *ct_in = nullptr) {
  MacTcArgs A;
  A.c1_in = 0; A.c1_cols = 0; A.c1_bytes = 0;
  if (g.c1_in && c1m && ct_in) {
    A.c1_cols = (int)std::min<int64_t>(g.CW, c1m->nK);
    A.c1_bytes = 2 * A.c1_cols * 32 * 8;
    c1_tmap(&A.c1map, ct_in, g.LN, c1m->nK, g.nJ, A.c1_cols);   // validated by c1_in_ok
    A.c1_in = 1;
  }
  A.W = (const uint8_t *)W; A.X = (const uint64_t *)X; A.out = out; A.g = g; A.N = (int)c->N;
  A.c1_out = c1m ? c1_masked : nullptr;
  A.c1_nK = c1m ? (int)c1m->nK : 0;
  A.c1_mn = c1m ? c1m->m * c1m->n : 0;
  A.c1_lognt = (c->N == 4096 ? 12 : 13) - 4;
  A.qperm = A.c1_out != nullptr;
  A.out_v4 = ((uintptr_t)out % 32) == 0;
  A.c1_v4 = A.c1_out && ((uintptr_t)A.c1_out % 32) == 0 && (A.c1_mn % 4 == 0 || c->L % 4 == 0);
  A.sched = (int *)((char *)X + tc_sched_offset(g));
  for (int64_t j0 = 0; j0 < g.nJp; j0 += kMacJChunk) {     // S_d < 7 * 4096 * 255^2 < 2^31 per launch
    A.jc0 = (int)(j0 / 32);
    A.njc = (int)((std::min<int64_t>(g.nJp, j0 + kMacJChunk) - j0) / 32);
    A.accumulate = j0 > 0;
    A.lazy_out = g.nJp <= kMacJChunk;                       // single launch: nobody adds to the outputs
    cudaMemsetAsync(A.sched, 0, sizeof(int), st);
    switch (g.CW) {
      case 16: launch_mac_tc_t<16>(c, A, smem_budget, grid, st); break;
      case 8: launch_mac_tc_t<8>(c, A, smem_budget, grid, st); break;
      case 4: launch_mac_tc_t<4>(c, A, smem_budget, grid, st); break;
      default: launch_mac_tc_t<2>(c, A, smem_budget, grid, st); break;
    }
  }
}

constexpr int kMacSmemAlone = 232448;        // the MAC alone on the SM: the deepest ring that fits
// the batch's MAC ring: since the c1 TMA path (c0-only forward kernels) the full ring wins again
// (tools/gpu/ring_sweep3.sh: 155 KB, one forward CTA beside the MAC, 0.911 ms; 227 KB, the forward
// NTTs fill the SMs between MAC launches and beside the inverse, 0.905 ms)
constexpr int kMacSmemShared = 232448;

void launch_mac(const hl_ctx *c, const uint2 *W, const uint32_t *X, uint64_t *out, const MacGeom &g, cudaStream_t st,
                int smem_budget = kMacSmemAlone, int grid = 0, const MaskArgs *c1m = nullptr, uint64_t *c1_masked = nullptr,
                const uint64_t *ct_in = nullptr) {
  if (g.engine == 2) {
    launch_mac_tc(c, W, X, out, g, smem_budget, grid > 0 ? grid : c->num_sms, st, c1m, c1_masked, ct_in);
    return;
  }
  MacArgs A;
  A.W = W; A.X = X; A.out = out; A.g = g; A.N = (int)c->N;
  for (int64_t j0 = 0; j0 < g.nJ; j0 += kMacJChunk) {
    A.j0 = (int)j0; A.j1 = (int)std::min<int64_t>(g.nJ, j0 + kMacJChunk);
    A.accumulate = j0 > 0;
    switch (g.LN) {
      case 4096: launch_mac_ln<4096>(c, A, st); break;
      case 8192: launch_mac_ln<8192>(c, A, st); break;
      case 12288: launch_mac_ln<12288>(c, A, st); break;
      case 16384: launch_mac_ln<16384>(c, A, st); break;
      case 24576: launch_mac_ln<24576>(c, A, st); break;
      default: break;
    }
  }
}

// the pruned c0 transform needs r >= 2 and one warp group per prime within the CTA
template <int LOGN, bool RR>
bool inv_prunes(const hl_ctx *c, const MaskArgs &M) {
  using Gm = Geom<LOGN>;
  const int re = std::min(M.r, 16);                   // the pruned kernel's live class (see there)
  const int wpp = (Gm::NT / std::max(re, 1) + 31) / 32;
  const size_t ext = RR ? 16 : 8;                      // sigma (+ row f4: e1 + F) per kept position
  const size_t smem_c0 = ntt_smem<LOGN>() * c->L + (size_t)M.m * M.n * ext;
  return M.r >= 2 && (int)c->L * wpp <= Gm::NT / 32 && smem_c0 <= 232448;
}
// May the MAC write the c1 halves of the response itself (MacTcArgs::c1_out)?  Only where the
// inverse would otherwise just reorder them (k_c1_out): pruned c0 inverse, no re-randomisation,
// tensor-core MAC in one launch with c0 columns first.
template <int LOGN>
bool c1_direct_ok(const hl_ctx *c, const MacGeom &g, const MaskArgs &M) {
  return g.engine == 2 && g.cperm && g.nJp <= kMacJChunk && !M.pk_hat &&
         inv_prunes<LOGN, false>(c, M);
}
inline bool c1_direct(const hl_ctx *c, const MacGeom &g, const MaskArgs &M) {
  return c->N == 4096 ? c1_direct_ok<12>(c, g, M) : c1_direct_ok<13>(c, g, M);
}
// May the MAC also READ c1 from the ciphertexts (MacGeom::c1_in)?  With the quad order (c1_direct)
// a work item's slots are 4 consecutive natural points; the column groups must be pure c0 / pure c1
// or a single group.
inline bool c1_in_ok(const MacGeom &g, const MaskArgs &M, const uint64_t *ct_in) {
  // whole 16-column c1 groups: the forward stage transposes c1 into X (k_c1_tx16, full 128-B lines)
  // -- the MAC's box gather would move 16-B pieces (and twice: a box carries 2 points per stage)
  if (g.CW == 16 && M.nK % 16 == 0) return false;
  if (!(M.c1_done && (g.nCg == 1 || M.nK % g.CW == 0))) return false;
  CUtensorMap probe;                                    // the launch re-encodes the same map
  return c1_tmap(&probe, ct_in, g.LN, M.nK, g.nJ, (int)std::min<int64_t>(g.CW, M.nK));
}

template <int LOGN, bool RR>
void launch_inv_mask_t(const hl_ctx *c, const uint64_t *ct_ntt, uint64_t *masked, uint64_t *share, MaskArgs M,
                       int64_t nout, cudaStream_t st) {
  using Gm = Geom<LOGN>;
  static PerDevice init;
  if (init.first()) {
    set_smem(k_ntt_inv_mask<LOGN, RR>, ntt_smem<LOGN>() + (size_t)Gm::N * 16);
    set_smem(k_intt_c0_pruned<LOGN, RR, true>, 232448);
    set_smem(k_c1_out<LOGN>, ntt_smem<LOGN>());
  }
  const int re = std::min(M.r, 16);
  const size_t ext = RR ? 16 : 8;
  const bool prune = inv_prunes<LOGN, RR>(c, M);
  const size_t smem = ntt_smem<LOGN>() + (RR ? std::max((size_t)M.m * M.n * 16, (size_t)Gm::N) : (size_t)M.m * M.n * 8);
  KTimer kt(c, HL_K_INTT_MASK, st);
  kt.nk = prune && !M.c1_done ? 2 : 1;
  if (prune) {   // compact parking of the live class (4 CTAs/SM; the full-size parking measured slower)
    const size_t cwords = (size_t)(Gm::N / re) + (size_t)(Gm::N / re) / 16;
    const size_t smem_cmp = cwords * 8 * c->L + (size_t)M.m * M.n * ext;
    k_intt_c0_pruned<LOGN, RR, true><<<(unsigned)nout, Gm::NT, smem_cmp, st>>>(ct_ntt, masked, share, M, c->dp);
    if (M.c1_done) return;                             // the MAC wrote c1 (c1_direct_ok)
    if (!RR) k_c1_out<LOGN><<<(unsigned)nout, Gm::NT, ntt_smem<LOGN>(), st>>>(ct_ntt, masked, M, c->dp);
    else k_ntt_inv_mask<LOGN, RR><<<(unsigned)nout, Gm::NT, smem, st>>>(ct_ntt, masked, share, M, c->dp, 1);
  } else {
    k_ntt_inv_mask<LOGN, RR><<<(unsigned)(nout * 2), Gm::NT, smem, st>>>(ct_ntt, masked, share, M, c->dp, 0);
  }
}

template <int LOGN>
void launch_inv_mask(const hl_ctx *c, const uint64_t *ct_ntt, uint64_t *masked, uint64_t *share, MaskArgs M,
                     int64_t nout, cudaStream_t st) {
  if (M.pk_hat) launch_inv_mask_t<LOGN, true>(c, ct_ntt, masked, share, M, nout, st);
  else launch_inv_mask_t<LOGN, false>(c, ct_ntt, masked, share, M, nout, st);
}

}  // namespace

// =========================================================================================
// entry points
// =========================================================================================
// NVTX range over a host-side scope (an API call or one pipeline stage of it): nsys / Nsight Systems
// show the library's phases on the CPU timeline and correlate the launches inside them.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Every device entry point runs on the context's device and restores the caller's current device.
struct DeviceGuard {
  int prev = -1, dev = -1;
  explicit DeviceGuard(const hl_ctx *c) {
    if (!c || c->device < 0) return;
    cudaGetDevice(&prev);
    if (prev != c->device) { dev = c->device; cudaSetDevice(dev); }
  }
  ~DeviceGuard() { if (dev >= 0) cudaSetDevice(prev); }
};

// the first pointer must be the context
static int check_ptrs(std::initializer_list<const void *> ps, const char *who) {
  for (const void *p : ps)
    if (!p) return hl_fail(HL_EINVAL, std::string(who) + ": NULL argument");
  const hl_ctx *c = (const hl_ctx *)*ps.begin();
  if (c->device < 0) return hl_fail(HL_EINVAL, std::string(who) + ": host-only context (device < 0)");
  return HL_OK;
}

static int encode_weights_impl(const hl_ctx *c, hl_tile tile, const uint64_t *W, int64_t R, int64_t Ma, int64_t ld_r,
                               int64_t ld_c, int64_t i_begin, int64_t i_end, void *wcache, uint64_t *scratch, int check,
                               void *stream);

extern "C" int hl_encode_weights(const hl_ctx *c, hl_tile tile, const uint64_t *W, int64_t R, int64_t Ma,
                                 int64_t i_begin, int64_t i_end, void *wcache, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_encode_weights");
  return encode_weights_impl(c, tile, W, R, Ma, Ma, 1, i_begin, i_end, wcache, nullptr, 1, stream);
}

extern "C" int hl_encode_weights_strided(const hl_ctx *c, hl_tile tile, const uint64_t *W, int64_t R, int64_t Ma,
                                         int64_t ld_row, int64_t ld_col, int64_t i_begin, int64_t i_end, void *wcache,
                                         void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_encode_weights_strided");
  return encode_weights_impl(c, tile, W, R, Ma, ld_row, ld_col, i_begin, i_end, wcache, nullptr, 1, stream);
}

extern "C" int hl_encode_weights_scratch(const hl_ctx *c, hl_tile tile, const uint64_t *W, int64_t R, int64_t Ma,
                                         int64_t ld_row, int64_t ld_col, int64_t i_begin, int64_t i_end, void *wcache,
                                         uint64_t *scratch, int check, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_encode_weights_scratch");
  if (!scratch) return hl_fail(HL_EINVAL, "hl_encode_weights_scratch: scratch is NULL");
  return encode_weights_impl(c, tile, W, R, Ma, ld_row, ld_col, i_begin, i_end, wcache, scratch, check, stream);
}

static int encode_weights_impl(const hl_ctx *c, hl_tile tile, const uint64_t *W, int64_t R, int64_t Ma, int64_t ld_r,
                               int64_t ld_c, int64_t i_begin, int64_t i_end, void *wcache, uint64_t *scratch, int check,
                               void *stream) {
  int rc;
  if ((rc = check_ptrs({c, W, wcache}, "hl_encode_weights"))) return rc;
  Geo g;
  if ((rc = hl_geometry(c, tile, Ma, R, 1, i_begin, i_end, &g))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(c->d_flags, 0, 8, st);
  const MacGeom mg = mac_geom(c, g.nIs, g.nJ, 2 * g.nK);
  if (mg.engine != 2) scratch = nullptr;       // the two-pass form is the tensor-core cache's
  if (mg.engine == 2 && mg.nJp != mg.nJ && !scratch)   // J padded to the 32-J MMA step: zero weight planes
    cudaMemsetAsync(wcache, 0, (size_t)mg.nIp * mg.LN * mg.nJp * 7, st);
  EncodeArgs A{W, R, Ma, g.nJ, g.nIs, g.i_begin, g.m, g.r, mg, ld_r, ld_c};
  dim3 grid((unsigned)((int64_t)(scratch ? g.nIs : (int64_t)mg.nIb * 16) * g.nJ), c->L);
  {
  KTimer kt(c, HL_K_ENCODE, st);
  if (c->N == 4096) {
    static PerDevice init;
    if (init.first()) { set_smem(k_encode_weights<12>, ntt_smem<12>()); }
    k_encode_weights<12><<<grid, Geom<12>::NT, ntt_smem<12>(), st>>>(A, (uint2 *)wcache, c->dp, c->d_flags, scratch);
  } else {
    static PerDevice init;
    if (init.first()) { set_smem(k_encode_weights<13>, ntt_smem<13>()); }
    k_encode_weights<13><<<grid, Geom<13>::NT, ntt_smem<13>(), st>>>(A, (uint2 *)wcache, c->dp, c->d_flags, scratch);
  }
  if (scratch) {
    const int64_t nb = (int64_t)mg.nIt * mg.nJc * ((mg.RT + kWpR - 1) / kWpR) * (mg.LN / kWpS);
    constexpr size_t wsm = (size_t)kWpS * kWpR * 33 * 8;
    static PerDevice winit;
    if (winit.first()) { set_smem(k_wplanes, wsm); }
    k_wplanes<<<(unsigned)nb, 256, wsm, st>>>(scratch, (uint8_t *)wcache, mg);
  }
  }
  if ((rc = hl_cuda_check("hl_encode_weights: launch"))) return rc;
  if (!check) return HL_OK;                    // the caller vouches for the range and the noise bound
  uint32_t flags[2];
  if (cudaMemcpyAsync(flags, c->d_flags, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return hl_cuda_check("hl_encode_weights: status readback");
  if (flags[0]) return hl_fail(HL_ERANGE, "hl_encode_weights: W value >= 2^log2_t");
  // Appendix C of SURVEY.md: |noise| <= 2R max|w| (r_t + e_max) must stay below Delta/2
  const double bound = log2(2.0 * (double)R) + log2((double)flags[1] + 1.0) + log2((double)c->r_t + 41.0);
  if (bound >= c->log2_delta - 1.0)
    return hl_fail(HL_ENOISE, "hl_encode_weights: worst-case noise bound 2R*max|w|*(r_t+41) >= Delta/2");
  return HL_OK;
}

extern "C" int hl_he_matmul(const hl_ctx *c, hl_tile tile, const void *wcache, int64_t Ma, int64_t R, int64_t Nb,
                            int64_t i_begin, int64_t i_end, const uint64_t *ct_in, void *workspace,
                            uint64_t *ct_out, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_he_matmul");
  int rc;
  if ((rc = check_ptrs({c, wcache, ct_in, workspace, ct_out}, "hl_he_matmul"))) return rc;
  Geo g;
  if ((rc = hl_geometry(c, tile, Ma, R, Nb, i_begin, i_end, &g))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nC = 2 * g.nK;
  const MacGeom mg = mac_geom(c, g.nIs, g.nJ, nC);
  fwd_ntt(c, ct_in, workspace, g.nJ * nC, &mg, st);
  launch_mac(c, (const uint2 *)wcache, (const uint32_t *)workspace, ct_out, mg, st);
  inv_ntt(c, ct_out, ct_out, g.nIs * nC, st, 1);
  return hl_cuda_check("hl_he_matmul: launch");
}

static MaskArgs mask_args(const Geo &g, int64_t Ma, int64_t Nb, uint64_t seed) {
  MaskArgs M;
  M.Ma = Ma; M.Nb = Nb; M.nK = g.nK; M.i_begin = g.i_begin;
  M.m = g.m; M.r = g.r; M.n = g.n; M.seed = seed;
  M.lm = __builtin_ctz((unsigned)g.m); M.lr = __builtin_ctz((unsigned)g.r);
  M.pk_hat = nullptr; M.u_hat = nullptr; M.cdt = nullptr; M.flood_bits = 0;
  M.nC = (int)(2 * g.nK); M.cperm = 0; M.c1_done = 0;
  return M;
}

extern "C" int hl_mask_and_share(const hl_ctx *c, hl_tile tile, int64_t Ma, int64_t Nb, int64_t i_begin,
                                 int64_t i_end, const uint64_t *ct_out, uint64_t seed, int compress,
                                 uint64_t *ct_masked, uint64_t *share, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_mask_and_share");
  int rc;
  if ((rc = check_ptrs({c, ct_out, ct_masked, share}, "hl_mask_and_share"))) return rc;
  Geo g;
  if ((rc = hl_geometry(c, tile, Ma, 1, Nb, i_begin, i_end, &g))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)((c->N / 8 + 127) / 128), (unsigned)(g.nIs * g.nK));
  KTimer kt(c, HL_K_MASK, st);
  k_mask<<<grid, 128, 0, st>>>(ct_out, ct_masked, share, mask_args(g, Ma, Nb, seed), c->dp, compress ? 1 : 0);
  return hl_cuda_check("hl_mask_and_share: launch");
}

extern "C" int hl_he_matmul_share(const hl_ctx *c, hl_tile tile, const void *wcache, int64_t Ma, int64_t R,
                                  int64_t Nb, int64_t i_begin, int64_t i_end, const uint64_t *ct_in,
                                  void *workspace, uint64_t *ct_out_ntt, uint64_t seed, int compress,
                                  uint64_t *ct_masked, uint64_t *share, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_he_matmul_share");
  int rc;
  if ((rc = check_ptrs({c, wcache, ct_in, workspace, ct_out_ntt, ct_masked, share}, "hl_he_matmul_share")))
    return rc;
  Geo g;
  if ((rc = hl_geometry(c, tile, Ma, R, Nb, i_begin, i_end, &g))) return rc;
  if (!compress) {   // full responses: the unfused pair (the mask needs every coefficient)
    if ((rc = hl_he_matmul(c, tile, wcache, Ma, R, Nb, i_begin, i_end, ct_in, workspace, ct_out_ntt, stream)))
      return rc;
    return hl_mask_and_share(c, tile, Ma, Nb, i_begin, i_end, ct_out_ntt, seed, 0, ct_masked, share, stream);
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nC = 2 * g.nK;
  MacGeom mg = mac_geom(c, g.nIs, g.nJ, nC);
  mg.cperm = mg.engine == 2;
  MaskArgs M = mask_args(g, Ma, Nb, seed);
  M.cperm = mg.cperm;
  M.c1_done = c1_direct(c, mg, M);
  mg.c1_in = c1_in_ok(mg, M, ct_in);
  if (mg.c1_in && mg.nCg == 1) mg.xw = (int)g.nK;
  fwd_ntt(c, ct_in, workspace, g.nJ * nC, &mg, st);
  launch_mac(c, (const uint2 *)wcache, (const uint32_t *)workspace, ct_out_ntt, mg, st, kMacSmemAlone, 0,
             M.c1_done ? &M : nullptr, ct_masked, ct_in);
  if (c->N == 4096) launch_inv_mask<12>(c, ct_out_ntt, ct_masked, share, M, g.nIs * g.nK, st);
  else launch_inv_mask<13>(c, ct_out_ntt, ct_masked, share, M, g.nIs * g.nK, st);
  return hl_cuda_check("hl_he_matmul_share: launch");
}

// ---------------------------------------------------------------------------------------
// Pipelined batch of compressed he_matmul_share calls (e.g. the four products of an encoder
// block).  The MAC is HBM-bound (weight cache) while the NTT kernels are bound by the FP64 pipe
// and latency, so they share SMs: the MACs run in entry order on the context's high-priority
// stream, every forward NTT is issued up front on the low-priority forward stream and the
// inverse NTT + mask of entry i on the low-priority auxiliary stream once MAC(i) is done;
// `stream` is joined to all of them at the start and at the end.
// ---------------------------------------------------------------------------------------
// n events of the context's pool `which` (grown on demand, never destroyed before the context)
static cudaEvent_t *ctx_events(const hl_ctx *c, int which, size_t n) {
  std::vector<void *> &pool = *c->ev_pool[which];
  while (pool.size() < n) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    pool.push_back((void *)e);
  }
  return reinterpret_cast<cudaEvent_t *>(pool.data());
}

// ready[i] (optional): event the forward NTT of entry i waits for (its input upload);
// done[i] (optional): recorded on the auxiliary stream once entry i's results are written.
// expand_seed (optional, with ready): per entry, the c1 halves are regenerated from this seed on the
// forward stream before the forward NTT, and every forward NTT is issued up front on the context's
// upload-side NTT stream so that no entry's inverse NTT queues behind a later entry's upload.
static void expand_seeded(const hl_ctx *c, int64_t nct, uint64_t a_seed, uint64_t *ct_in, cudaStream_t st);
static int linear_batch_run(const hl_ctx *c, hl_tile tile, int n, const hl_linear_desc *d, void *stream,
                            const cudaEvent_t *ready, const cudaEvent_t *done, const uint64_t *expand_seed) {
  int rc;
  struct Entry { Geo g; MacGeom mg; MaskArgs M; };
  std::vector<Entry> E(n);
  std::vector<int> ord;     // compute order = entry order of the non-empty entries (the caller's choice:
                            // the bench submits the order measured fastest, synth Config.batch_order)
  for (int i = 0; i < n; i++) {
    if (d[i].i_end >= 0 && d[i].i_begin == d[i].i_end) {        // an empty I-tile shard: nothing to do
      if (ready || done) return hl_fail(HL_EINVAL, "hl_he_linear_batch_host: empty shards are not supported");
      continue;
    }
    if ((rc = check_ptrs({c, d[i].wcache, d[i].ct_in, d[i].workspace, d[i].ct_out_ntt, d[i].ct_masked, d[i].share},
                         "hl_he_linear_batch")))
      return rc;
    if ((rc = hl_geometry(c, d[i].tile.m ? d[i].tile : tile, d[i].Ma, d[i].R, d[i].Nb, d[i].i_begin, d[i].i_end,
                          &E[i].g)))
      return rc;
    ord.push_back(i);
    E[i].mg = mac_geom(c, E[i].g.nIs, E[i].g.nJ, 2 * E[i].g.nK);
    E[i].mg.cperm = E[i].mg.engine == 2;
    E[i].M = mask_args(E[i].g, d[i].Ma, d[i].Nb, d[i].seed);
    E[i].M.cperm = E[i].mg.cperm;
    E[i].M.c1_done = c1_direct(c, E[i].mg, E[i].M);
    E[i].mg.c1_in = c1_in_ok(E[i].mg, E[i].M, d[i].ct_in);
    if (E[i].mg.c1_in && E[i].mg.nCg == 1) E[i].mg.xw = (int)E[i].g.nK;
  }
  cudaStream_t sc = (cudaStream_t)stream, s0 = (cudaStream_t)c->mac_stream, s1 = (cudaStream_t)c->aux_stream;
  cudaEvent_t *ev = ctx_events(c, 0, 2 * (size_t)n + 3);
  if (!ev) return hl_cuda_check("hl_he_linear_batch: events");
  cudaEvent_t *e_fwd = ev, *e_mac = ev + n, e_in = ev[2 * n], e_done = ev[2 * n + 1];
  cudaEvent_t e_macs = ev[2 * n + 2];
  // every forward NTT is issued up front on the forward stream (measured: 1.082 -> 1.060 ms per c2
  // block vs interleaving them with the MACs)
  // adaptive policy: with many columns per weight byte (nK >= 8, e.g. c3/c4: 8-16x c2's NTT work per
  // byte) a MAC sharing its SMs with NTT kernels slows down more than the overlap gains -- run every
  // MAC alone and overlap only the NTT stages of neighbouring products (serial branch below)
  constexpr int serial_nk = 8;
  bool serial = !ready;
  for (int i : ord) serial = serial && E[i].g.nK >= serial_nk;
  cudaStream_t sf = (cudaStream_t)c->fwd_stream;
  auto fwd = [&](int i) {
    NvtxRange nr("hl.batch.forward_ntt");
    if (ready) cudaStreamWaitEvent(sf, ready[i], 0);
    if (expand_seed)
      expand_seeded(c, E[i].g.nJ * E[i].g.nK, expand_seed[i], const_cast<uint64_t *>(d[i].ct_in), sf);
    fwd_ntt(c, d[i].ct_in, d[i].workspace, E[i].g.nJ * 2 * E[i].g.nK, &E[i].mg, sf);
    cudaEventRecord(e_fwd[i], sf);
  };
  auto inv = [&](int i) {
    NvtxRange nr("hl.batch.inverse_ntt_mask");
    if (c->N == 4096) launch_inv_mask<12>(c, d[i].ct_out_ntt, d[i].ct_masked, d[i].share, E[i].M, E[i].g.nIs * E[i].g.nK, s1);
    else launch_inv_mask<13>(c, d[i].ct_out_ntt, d[i].ct_masked, d[i].share, E[i].M, E[i].g.nIs * E[i].g.nK, s1);
  };
  const int na = (int)ord.size();
  if (na == 0) return HL_OK;
  cudaEventRecord(e_in, sc);                      // inputs written on `stream` are visible to both streams
  cudaStreamWaitEvent(s0, e_in, 0);
  cudaStreamWaitEvent(s1, e_in, 0);
  cudaStreamWaitEvent(sf, e_in, 0);
  if (serial) {
    // every MAC alone on the device (it takes every SM's shared memory and registers), and the two
    // NTT stages of neighbouring products side by side: the forward NTT of product k+1 starts when
    // MAC(k) is done, beside the inverse NTT + mask of product k (both FP64- and latency-bound at
    // low occupancy).  MAC(k+1) waits for its forward NTT only.
    for (int k = 0; k < na; k++) {
      const int i = ord[k];
      if (k == 0) fwd(i);
      cudaStreamWaitEvent(s0, e_fwd[i], 0);
      {
        NvtxRange nr("hl.batch.mac");
        launch_mac(c, (const uint2 *)d[i].wcache, (const uint32_t *)d[i].workspace, d[i].ct_out_ntt, E[i].mg, s0,
                   kMacSmemAlone, 0, E[i].M.c1_done ? &E[i].M : nullptr, d[i].ct_masked, d[i].ct_in);
      }
      cudaEventRecord(e_mac[i], s0);
      if (k + 1 < na) {
        cudaStreamWaitEvent(sf, e_mac[i], 0);
        fwd(ord[k + 1]);
      }
      cudaStreamWaitEvent(s1, e_mac[i], 0);
      inv(i);
    }
  } else {
  for (int k = 0; k < na; k++) fwd(ord[k]);
  for (int k = 0; k < na; k++) {
    const int i = ord[k];
    cudaStreamWaitEvent(s0, e_fwd[i], 0);
    NvtxRange nr("hl.batch.mac");
    launch_mac(c, (const uint2 *)d[i].wcache, (const uint32_t *)d[i].workspace, d[i].ct_out_ntt, E[i].mg, s0,
               kMacSmemShared, 0, E[i].M.c1_done ? &E[i].M : nullptr, d[i].ct_masked, d[i].ct_in);
    cudaEventRecord(e_mac[i], s0);
    cudaStreamWaitEvent(s1, e_mac[i], 0);
    inv(i);                                                               // overlaps MAC(i+1)
    if (done) cudaEventRecord(done[i], s1);
  }
  }
  cudaEventRecord(e_done, s1);
  cudaEventRecord(e_macs, s0);
  cudaStreamWaitEvent(sc, e_done, 0);
  cudaStreamWaitEvent(sc, e_macs, 0);
  // (every forward NTT precedes a MAC, so sf is joined through s0)
  return hl_cuda_check("hl_he_linear_batch: launch");
}

extern "C" int hl_he_linear_batch(const hl_ctx *c, hl_tile tile, int n, const hl_linear_desc *d, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_he_linear_batch");
  int rc;
  if ((rc = check_ptrs({c, d}, "hl_he_linear_batch"))) return rc;
  if (n <= 0) return hl_fail(HL_EINVAL, "hl_he_linear_batch: n must be positive");
  return linear_batch_run(c, tile, n, d, stream, nullptr, nullptr, nullptr);
}

// ---------------------------------------------------------------------------------------
// Seeded ciphertext upload: c1 = a is PRF output of the client's
// encryption seed (reading C10), so only c0 crosses PCIe and the device regenerates c1.
// ---------------------------------------------------------------------------------------
static void expand_seeded(const hl_ctx *c, int64_t nct, uint64_t a_seed, uint64_t *ct_in, cudaStream_t st) {
  const int64_t nth = nct * c->L * (c->N / 4);
  KTimer kt(c, HL_K_OTHER, st);
  k_expand_a<<<(unsigned)((nth + 255) / 256), 256, 0, st>>>(ct_in, nct, __builtin_ctz((unsigned)c->N), a_seed, c->dp);
}

extern "C" int hl_expand_seeded(const hl_ctx *c, hl_tile tile, int64_t R, int64_t Nb, uint64_t a_seed,
                                uint64_t *ct_in, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_expand_seeded");
  int rc;
  if ((rc = check_ptrs({c, ct_in}, "hl_expand_seeded"))) return rc;
  Geo g;
  if ((rc = hl_geometry(c, tile, 1, R, Nb, 0, -1, &g))) return rc;
  expand_seeded(c, g.nJ * g.nK, a_seed, ct_in, (cudaStream_t)stream);
  return hl_cuda_check("hl_expand_seeded: launch");
}

// 50-bit wire format on the device (include/helinear.h hl_pack50).  Coalesced both ways: one
// thread per packed word (gathers the <= 3 residues overlapping its 64 bits) / per residue
// (reads the <= 2 packed words holding its 50 bits).
__global__ void k_pack50(const uint64_t *__restrict__ in, int64_t words, uint64_t *__restrict__ out) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;     // packed word
  const int64_t g = o / 25, q = o % 25;
  if (g * 32 >= words) return;
  const int lo = (int)(64 * q), hi = lo + 64;                            // bit range in the group
  uint64_t w = 0;
  for (int i = lo / 50; i < 32 && 50 * i < hi; i++) {
    const int64_t e = g * 32 + i;
    const uint64_t v = e < words ? __ldg(in + e) : 0;
    const int sh = 50 * i - lo;                                          // in (-50, 64)
    w |= sh >= 0 ? v << sh : v >> -sh;
  }
  out[o] = w;
}
// unpack into the c0 halves of ciphertexts [nct][2][L][N] (ln = L*N words per half)
__global__ void k_unpack50_c0(const uint64_t *__restrict__ in, int64_t words, uint64_t *__restrict__ ct, int64_t ln) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;     // residue
  if (e >= words) return;
  const int64_t g = e / 32;
  const int b = 50 * (int)(e % 32), q = b >> 6, r = b & 63;
  const uint64_t *w = in + g * 25;
  uint64_t v = __ldg(w + q) >> r;
  if (r > 14) v |= __ldg(w + q + 1) << (64 - r);
  ct[(e / ln) * 2 * ln + e % ln] = v & ((1ull << 50) - 1);
}

// End-to-end batch on host buffers: a three-stage pipeline over the entries -- upload of entry
// i+1 (c0 halves, strided H2D on the context's upload stream, then the c1 expansion) while entry
// i computes (hl_he_linear_batch's streams) while entry i-1's results download (download stream).
extern "C" int hl_he_linear_batch_host(const hl_ctx *c, hl_tile tile, int n, const hl_linear_host_desc *h,
                                       void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_he_linear_batch_host");
  int rc;
  if ((rc = check_ptrs({c, h}, "hl_he_linear_batch_host"))) return rc;
  if (n <= 0) return hl_fail(HL_EINVAL, "hl_he_linear_batch_host: n must be positive");
  std::vector<hl_linear_desc> d(n);
  std::vector<hl_layout> lay(n);
  for (int i = 0; i < n; i++) {
    if ((rc = check_ptrs({c, h[i].c0_host, h[i].ct_masked_host, h[i].share_host, h[i].dev.ct_in},
                         "hl_he_linear_batch_host")))
      return rc;
    if ((rc = hl_layout_query(c, h[i].dev.tile.m ? h[i].dev.tile : tile, h[i].dev.Ma, h[i].dev.R, h[i].dev.Nb, 0,
                              -1, &lay[i])))
      return rc;
    if (!(h[i].dev.i_begin == 0 && (h[i].dev.i_end == -1 || h[i].dev.i_end == lay[i].nI)))
      return hl_fail(HL_EINVAL, "hl_he_linear_batch_host: whole products only (i_begin = 0, i_end = -1 or nI)");
    d[i] = h[i].dev;
  }
  cudaStream_t sc = (cudaStream_t)stream, su = (cudaStream_t)c->up_stream, sd = (cudaStream_t)c->down_stream;
  cudaEvent_t *ev = ctx_events(c, 1, 2 * (size_t)n + 2);
  if (!ev) return hl_cuda_check("hl_he_linear_batch_host: events");
  cudaEvent_t *e_up = ev, *e_res = ev + n, e_in = ev[2 * n], e_down = ev[2 * n + 1];
  cudaEventRecord(e_in, sc);                      // the buffers are free once earlier work on `stream` is done
  cudaStreamWaitEvent(su, e_in, 0);
  cudaStreamWaitEvent(sd, e_in, 0);
  const size_t half = (size_t)c->L * c->N * 8;
  std::vector<uint64_t> seeds(n);
  for (int i = 0; i < n; i++) {
    const int64_t nct = lay[i].ct_in_words / (2 * c->L * c->N);
    if (h[i].packed) {            // 50-bit stream of the c0 halves -> workspace -> unpacked into ct_in
      const int64_t words = nct * c->L * c->N, pw = hl_packed50_words(words);
      uint64_t *stage = reinterpret_cast<uint64_t *>(d[i].workspace);
      if (cudaMemcpyAsync(stage, h[i].c0_host, (size_t)pw * 8, cudaMemcpyHostToDevice, su) != cudaSuccess)
        return hl_cuda_check("hl_he_linear_batch_host: H2D");
      k_unpack50_c0<<<(unsigned)((words + 255) / 256), 256, 0, su>>>(stage, words, const_cast<uint64_t *>(d[i].ct_in),
                                                                   (int64_t)c->L * c->N);
    } else if (cudaMemcpy2DAsync(const_cast<uint64_t *>(d[i].ct_in), 2 * half, h[i].c0_host, half, half, (size_t)nct,
                                 cudaMemcpyHostToDevice, su) != cudaSuccess) {
      return hl_cuda_check("hl_he_linear_batch_host: H2D");
    }
    cudaEventRecord(e_up[i], su);
    seeds[i] = h[i].a_seed;
  }
  if ((rc = linear_batch_run(c, tile, n, d.data(), stream, e_up, e_res, seeds.data()))) return rc;
  for (int i = 0; i < n; i++) {
    cudaStreamWaitEvent(sd, e_res[i], 0);
    const uint64_t *resp = d[i].ct_masked;
    size_t resp_bytes = (size_t)lay[i].ct_masked_words * 8;
    if (h[i].packed) {            // packed on the device into the (now free) NTT-domain scratch
      const int64_t words = lay[i].ct_masked_words, pw = hl_packed50_words(words);
      k_pack50<<<(unsigned)((pw + 255) / 256), 256, 0, sd>>>(d[i].ct_masked, words, d[i].ct_out_ntt);
      resp = d[i].ct_out_ntt;
      resp_bytes = (size_t)hl_packed50_words(words) * 8;
    }
    if (cudaMemcpyAsync(h[i].ct_masked_host, resp, resp_bytes, cudaMemcpyDeviceToHost, sd) != cudaSuccess ||
        cudaMemcpyAsync(h[i].share_host, d[i].share, (size_t)lay[i].share_words * 8, cudaMemcpyDeviceToHost,
                        sd) != cudaSuccess)
      return hl_cuda_check("hl_he_linear_batch_host: D2H");
  }
  cudaEventRecord(e_down, sd);
  cudaStreamWaitEvent(sc, e_down, 0);
  return hl_cuda_check("hl_he_linear_batch_host: launch");
}

// ---------------------------------------------------------------------------------------
// the client side on the GPU (client_dev.cuh)
// ---------------------------------------------------------------------------------------
extern "C" int hl_sk_prepare(const hl_ctx *c, const int8_t *sk, uint64_t *s_hat, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_sk_prepare");
  int rc;
  if ((rc = check_ptrs({c, sk, s_hat}, "hl_sk_prepare"))) return rc;
  std::vector<uint64_t> res((size_t)c->L * c->N);
  for (uint32_t i = 0; i < c->N; i++)
    if (sk[i] < -1 || sk[i] > 1) return hl_fail(HL_ERANGE, "hl_sk_prepare: secret key must be ternary");
  for (uint32_t l = 0; l < c->L; l++)
    for (uint32_t i = 0; i < c->N; i++)
      res[(size_t)l * c->N + i] = sk[i] > 0 ? 1 : (sk[i] < 0 ? c->primes[l] - 1 : 0);
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(s_hat, res.data(), res.size() * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return hl_cuda_check("hl_sk_prepare: upload");
  fwd_ntt(c, s_hat, s_hat, 1, nullptr, st);            // in place: NTT(s) per prime, slot order
  if (cudaStreamSynchronize(st) != cudaSuccess) return hl_cuda_check("hl_sk_prepare: sync");
  return hl_cuda_check("hl_sk_prepare: launch");
}

extern "C" int hl_encrypt_device(const hl_ctx *c, const uint64_t *s_hat, hl_tile tile, const uint64_t *X, int64_t Nb,
                                 int64_t R, uint64_t seed, uint64_t *ct_in, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_encrypt_device");
  int rc;
  if ((rc = check_ptrs({c, s_hat, X, ct_in}, "hl_encrypt_device"))) return rc;
  Geo g;
  if ((rc = hl_geometry(c, tile, 1, R, Nb, 0, -1, &g))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(c->d_flags, 0, 8, st);
  EncArgs E{X, Nb, R, g.nK, g.m, g.r, g.n, __builtin_ctz((unsigned)g.m), __builtin_ctz((unsigned)g.r), seed, hl::public_seed(seed), s_hat};
  const unsigned nct = (unsigned)(g.nJ * g.nK);
  {
    KTimer kt(c, HL_K_OTHER, st);
    if (c->N == 4096) {
      constexpr size_t sm = ntt_smem<12>() + 4096;
      static PerDevice init;
      if (init.first()) { set_smem(k_encrypt<12>, sm); }
      k_encrypt<12><<<nct, Geom<12>::NT, sm, st>>>(E, ct_in, c->dp, c->d_cdt, c->d_flags);
    } else {
      constexpr size_t sm = ntt_smem<13>() + 8192;
      static PerDevice init;
      if (init.first()) { set_smem(k_encrypt<13>, sm); }
      k_encrypt<13><<<nct, Geom<13>::NT, sm, st>>>(E, ct_in, c->dp, c->d_cdt, c->d_flags);
    }
  }
  if ((rc = hl_cuda_check("hl_encrypt_device: launch"))) return rc;
  uint32_t flags[2];
  if (cudaMemcpyAsync(flags, c->d_flags, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return hl_cuda_check("hl_encrypt_device: status readback");
  if (flags[0]) return hl_fail(HL_ERANGE, "hl_encrypt_device: X value >= 2^log2_t");
  return HL_OK;
}

extern "C" int hl_decrypt_share_device(const hl_ctx *c, const uint64_t *s_hat, hl_tile tile, const uint64_t *ct_masked,
                                       int64_t Ma, int64_t Nb, uint64_t *share_client, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_decrypt_share_device");
  int rc;
  if ((rc = check_ptrs({c, s_hat, ct_masked, share_client}, "hl_decrypt_share_device"))) return rc;
  Geo g;
  if ((rc = hl_geometry(c, tile, Ma, 1, Nb, 0, -1, &g))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  DecArgs D{Ma, Nb, g.nK, g.m, g.r, g.n, __builtin_ctz((unsigned)g.m), __builtin_ctz((unsigned)g.r), s_hat};
  const size_t res = (size_t)c->L * g.m * g.n * 8;
  const unsigned nout = (unsigned)(g.nI * g.nK);
  KTimer kt(c, HL_K_OTHER, st);
  if (c->N == 4096) {
    const size_t sm = ntt_smem<12>() + res;
    static PerDevice init;
    if (init.first()) { set_smem(k_decrypt<12>, 232448); }
    k_decrypt<12><<<nout, Geom<12>::NT, sm, st>>>(ct_masked, share_client, D, c->dp);
  } else {
    const size_t sm = ntt_smem<13>() + res;
    static PerDevice init;
    if (init.first()) { set_smem(k_decrypt<13>, 232448); }
    k_decrypt<13><<<nout, Geom<13>::NT, sm, st>>>(ct_masked, share_client, D, c->dp);
  }
  return hl_cuda_check("hl_decrypt_share_device: launch");
}

// ---------------------------------------------------------------------------------------
// Share arithmetic: dst[rows][cols] += src (or src^T, src being [cols][rows]) mod 2^t.  The
// attention cross terms add shares of (X1 Y0)^T after the transposition of
// footnote 3.  32x32 tiles through shared memory (coalesced both ways).
// ---------------------------------------------------------------------------------------
__global__ void k_share_acc(uint64_t *__restrict__ dst, const uint64_t *__restrict__ src, int64_t rows, int64_t cols,
                            int transpose, uint64_t tmask) {
  __shared__ uint64_t tl[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;           // 32 x 8
  if (transpose) {
    for (int k = ty; k < 32; k += 8) {                     // src row = c0 + k (a dst column), src col = r0 + tx
      const int64_t sr = c0 + k, sc = r0 + tx;
      tl[k][tx] = (sr < cols && sc < rows) ? src[sr * rows + sc] : 0;
    }
    __syncthreads();
  }
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + k, cc = c0 + tx;
    if (r < rows && cc < cols) {
      const uint64_t v = transpose ? tl[tx][k] : src[r * cols + cc];
      dst[r * cols + cc] = (dst[r * cols + cc] + v) & tmask;
    }
  }
}

extern "C" int hl_share_accumulate(const hl_ctx *c, uint64_t *dst, const uint64_t *src, int64_t rows, int64_t cols,
                                   int transpose, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_share_accumulate");
  int rc;
  if ((rc = check_ptrs({c, dst, src}, "hl_share_accumulate"))) return rc;
  if (rows <= 0 || cols <= 0) return hl_fail(HL_EINVAL, "hl_share_accumulate: rows, cols must be positive");
  const uint64_t tmask = c->log2_t >= 64 ? ~0ull : ((1ull << c->log2_t) - 1);
  KTimer kt(c, HL_K_OTHER, (cudaStream_t)stream);
  k_share_acc<<<dim3((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32)), dim3(32, 8), 0,
                (cudaStream_t)stream>>>(dst, src, rows, cols, transpose ? 1 : 0, tmask);
  return hl_cuda_check("hl_share_accumulate: launch");
}

// ---------------------------------------------------------------------------------------
// FC-layer share assembly, fc.cuh
// ---------------------------------------------------------------------------------------
static int fc_geom(const hl_ctx *c, int64_t Nb, int64_t R, int64_t Ma, FcGeom *g) {
  if (!c) return hl_fail(HL_EINVAL, "ctx is NULL");
  if (Nb <= 0 || R <= 0 || Ma <= 0) return hl_fail(HL_EINVAL, "Nb, R, Ma must be positive");
  if (R > 6400) return hl_fail(HL_ENOTSUP, "FC local share: R > 6400 (s32 limb accumulators)");
  if (c->log2_t > 40) return hl_fail(HL_ENOTSUP, "FC local share: log2_t > 40 (5 byte limbs)");
  g->Nb = Nb; g->R = R; g->Ma = Ma;
  g->nMt = (int)((Nb + kFcMT - 1) / kFcMT);
  g->nNt = (int)((Ma + kFcNT - 1) / kFcNT);
  g->nKc = (int)((R + 31) / 32);
  // split K so that the grid covers ~2 CTAs per SM (partial sums meet by wrapping atomic adds)
  const int tiles = g->nMt * g->nNt;
  const int splits = std::max(1, std::min(g->nKc, (2 * c->num_sms + tiles - 1) / tiles));
  g->kps = (g->nKc + splits - 1) / splits;
  g->tmask = (1ull << c->log2_t) - 1;
  return HL_OK;
}

extern "C" int hl_fc_layout(const hl_ctx *c, int64_t Nb, int64_t R, int64_t Ma, int64_t *wplanes_bytes,
                            int64_t *workspace_bytes) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_fc_layout");
  FcGeom g;
  int rc;
  if ((rc = fc_geom(c, Nb, R, Ma, &g))) return rc;
  if (wplanes_bytes) *wplanes_bytes = (int64_t)g.nNt * g.nKc * kFcBStage;
  if (workspace_bytes) *workspace_bytes = (int64_t)g.nMt * g.nKc * kFcAStage;
  return HL_OK;
}

extern "C" int hl_fc_encode_weights(const hl_ctx *c, const uint64_t *W, int64_t R, int64_t Ma, void *wplanes,
                                    void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_fc_encode_weights");
  return hl_fc_encode_weights_chk(c, W, R, Ma, wplanes, 1, stream);
}

extern "C" int hl_fc_encode_weights_chk(const hl_ctx *c, const uint64_t *W, int64_t R, int64_t Ma, void *wplanes,
                                        int check, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_fc_encode_weights_chk");
  int rc;
  if ((rc = check_ptrs({c, W, wplanes}, "hl_fc_encode_weights"))) return rc;
  FcGeom g;
  if ((rc = fc_geom(c, 1, R, Ma, &g))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(c->d_flags, 0, 8, st);
  const int64_t n = (int64_t)g.nNt * kFcNT * g.nKc * 32;
  {
    KTimer kt(c, HL_K_ENCODE, st);
    k_fc_w_planes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(W, (uint8_t *)wplanes, g, c->d_flags);
  }
  if ((rc = hl_cuda_check("hl_fc_encode_weights: launch"))) return rc;
  if (!check) return HL_OK;
  uint32_t flags[2];
  if (cudaMemcpyAsync(flags, c->d_flags, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return hl_cuda_check("hl_fc_encode_weights: status readback");
  if (flags[0]) return hl_fail(HL_ERANGE, "hl_fc_encode_weights: W value >= 2^log2_t");
  return HL_OK;
}

extern "C" int hl_fc_local_share(const hl_ctx *c, const uint64_t *X1, const void *wplanes, const uint64_t *bias,
                                 int64_t Nb, int64_t R, int64_t Ma, void *workspace, uint64_t *share, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_fc_local_share");
  int rc;
  if ((rc = check_ptrs({c, X1, wplanes, workspace, share}, "hl_fc_local_share"))) return rc;
  FcGeom g;
  if ((rc = fc_geom(c, Nb, R, Ma, &g))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  static PerDevice init;
  if (init.first()) { set_smem(k_fc_gemm, kFcSmem); }
  KTimer kt(c, HL_K_FC, st);
  const int64_t n = (int64_t)g.nMt * kFcMT * g.nKc * 8;
  k_fc_x_planes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(X1, (uint8_t *)workspace, g);
  const unsigned nsplit = (unsigned)((g.nKc + g.kps - 1) / g.kps);
  k_fc_gemm<<<dim3(g.nNt, g.nMt, nsplit), 256, kFcSmem, st>>>((const uint8_t *)workspace, (const uint8_t *)wplanes,
                                                              bias, share, g);
  k_fc_mask<<<(unsigned)((Nb * Ma + 255) / 256), 256, 0, st>>>(share, Nb * Ma, g.tmask);
  return hl_cuda_check("hl_fc_local_share: launch");
}

// ---------------------------------------------------------------------------------------
// re-randomised responses (reading C22)
// ---------------------------------------------------------------------------------------
extern "C" int hl_pk_prepare(const hl_ctx *c, const uint64_t *pk, uint64_t *pk_hat, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_pk_prepare");
  int rc;
  if ((rc = check_ptrs({c, pk, pk_hat}, "hl_pk_prepare"))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(pk_hat, pk, (size_t)2 * c->L * c->N * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return hl_cuda_check("hl_pk_prepare: upload");
  fwd_ntt(c, pk_hat, pk_hat, 2, nullptr, st);          // NTT(pk0), NTT(pk1) per prime, slot order
  if (cudaStreamSynchronize(st) != cudaSuccess) return hl_cuda_check("hl_pk_prepare: sync");
  return hl_cuda_check("hl_pk_prepare: launch");
}

extern "C" int hl_he_matmul_share_rr(const hl_ctx *c, hl_tile tile, const void *wcache, int64_t Ma, int64_t R,
                                     int64_t Nb, int64_t i_begin, int64_t i_end, const uint64_t *ct_in,
                                     void *workspace, uint64_t *ct_out_ntt, const uint64_t *pk_hat, int flood_bits,
                                     uint64_t *rr_ws, uint64_t seed, uint64_t *ct_masked, uint64_t *share,
                                     void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_he_matmul_share_rr");
  int rc;
  if ((rc = check_ptrs({c, wcache, ct_in, workspace, ct_out_ntt, pk_hat, rr_ws, ct_masked, share},
                       "hl_he_matmul_share_rr")))
    return rc;
  Geo g;
  if ((rc = hl_geometry(c, tile, Ma, R, Nb, i_begin, i_end, &g))) return rc;
  if (flood_bits < 0 || flood_bits > std::min(62, (int)c->log2_delta - 1))
    return hl_fail(HL_ERANGE, "hl_he_matmul_share_rr: flood_bits must be in [0, min(62, log2(Delta) - 1)]");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nC = 2 * g.nK, nout = g.nIs * g.nK;
  MacGeom mg = mac_geom(c, g.nIs, g.nJ, nC);
  mg.cperm = mg.engine == 2;
  fwd_ntt(c, ct_in, workspace, g.nJ * nC, &mg, st);
  launch_mac(c, (const uint2 *)wcache, (const uint32_t *)workspace, ct_out_ntt, mg, st);
  MaskArgs M = mask_args(g, Ma, Nb, seed);
  M.cperm = mg.cperm;
  M.pk_hat = pk_hat; M.u_hat = rr_ws; M.cdt = c->d_cdt; M.flood_bits = flood_bits;
  {
    KTimer kt(c, HL_K_INTT_MASK, st);
    if (c->N == 4096) {
      static PerDevice init;
      if (init.first()) { set_smem(k_rr_u<12>, ntt_smem<12>() + 4096); }
      k_rr_u<12><<<(unsigned)nout, Geom<12>::NT, ntt_smem<12>() + 4096, st>>>(rr_ws, M, c->dp);
    } else {
      static PerDevice init;
      if (init.first()) { set_smem(k_rr_u<13>, ntt_smem<13>() + 8192); }
      k_rr_u<13><<<(unsigned)nout, Geom<13>::NT, ntt_smem<13>() + 8192, st>>>(rr_ws, M, c->dp);
    }
  }
  if (c->N == 4096) launch_inv_mask<12>(c, ct_out_ntt, ct_masked, share, M, nout, st);
  else launch_inv_mask<13>(c, ct_out_ntt, ct_masked, share, M, nout, st);
  return hl_cuda_check("hl_he_matmul_share_rr: launch");
}

extern "C" int hl_he_linear_host(const hl_ctx *c, hl_tile tile, const void *wcache, int64_t Ma, int64_t R,
                                 int64_t Nb, const uint64_t *ct_in_host, uint64_t seed, int compress,
                                 uint64_t *ct_masked_host, uint64_t *share_host, uint64_t *dev_ct_in,
                                 void *workspace, uint64_t *dev_ct_out_ntt, uint64_t *dev_ct_masked,
                                 uint64_t *dev_share, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_he_linear_host");
  int rc;
  if ((rc = check_ptrs({c, wcache, ct_in_host, ct_masked_host, share_host, dev_ct_in, workspace,
                        dev_ct_out_ntt, dev_ct_masked, dev_share}, "hl_he_linear_host")))
    return rc;
  hl_layout lay;
  if ((rc = hl_layout_query(c, tile, Ma, R, Nb, 0, -1, &lay))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(dev_ct_in, ct_in_host, (size_t)lay.ct_in_words * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return hl_cuda_check("hl_he_linear_host: H2D");
  if ((rc = hl_he_matmul_share(c, tile, wcache, Ma, R, Nb, 0, -1, dev_ct_in, workspace, dev_ct_out_ntt, seed,
                               compress, dev_ct_masked, dev_share, stream)))
    return rc;
  const size_t mw = compress ? (size_t)lay.ct_masked_words : (size_t)lay.ct_full_words;
  if (cudaMemcpyAsync(ct_masked_host, dev_ct_masked, mw * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(share_host, dev_share, (size_t)lay.share_words * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return hl_cuda_check("hl_he_linear_host: D2H");
  return HL_OK;
}

extern "C" int hl_poly_mul(const hl_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *out, int64_t npoly,
                           void *scratch, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_poly_mul");
  int rc;
  if ((rc = check_ptrs({c, a, b, out, scratch}, "hl_poly_mul"))) return rc;
  if (npoly <= 0) return hl_fail(HL_EINVAL, "hl_poly_mul: npoly must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = npoly * c->L * c->N;
  uint64_t *s1 = (uint64_t *)scratch, *s2 = s1 + n;
  fwd_ntt(c, a, s1, npoly, nullptr, st);
  fwd_ntt(c, b, s2, npoly, nullptr, st);
  { KTimer kt(c, HL_K_OTHER, st);
  k_pointwise<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s1, s2, s1, n, c->dp); }
  inv_ntt(c, s1, out, npoly, st);
  return hl_cuda_check("hl_poly_mul: launch");
}

extern "C" int hl_ntt_roundtrip(const hl_ctx *c, uint64_t *x, int64_t npoly, void *scratch, void *stream) {
  DeviceGuard dg_(c);
  NvtxRange nvtx_("hl_ntt_roundtrip");
  int rc;
  if ((rc = check_ptrs({c, x, scratch}, "hl_ntt_roundtrip"))) return rc;
  if (npoly <= 0) return hl_fail(HL_EINVAL, "hl_ntt_roundtrip: npoly must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  fwd_ntt(c, x, scratch, npoly, nullptr, st);
  inv_ntt(c, (uint64_t *)scratch, x, npoly, st);
  return hl_cuda_check("hl_ntt_roundtrip: launch");
}
