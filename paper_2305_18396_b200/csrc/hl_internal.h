// hl_internal.h -- private declarations of libhelinear (the CUDA path).
// Nothing here is shared with oracle/ (the CPU oracle is an independent implementation).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <vector_types.h>   // ulonglong2 (CUDA vector type; host-side include only)

#include "../../include/helinear.h"

#define HL_MAX_L 3

typedef unsigned __int128 hl_u128;

// Per-prime constants used by the device kernels (passed by value as kernel parameters).
struct PrimeConsts {
  uint64_t p;         // prime, 2^49 < p < 2^50, p = 1 mod 2N
  uint64_t two_p;     // 2p
  uint64_t mu;        // floor(2^64 / p)              (Barrett for 64-bit inputs)
  uint64_t r64;       // 2^64 mod p
  uint64_t r64_sh;    // floor(r64 * 2^64 / p)        (Shoup companion)
  uint64_t c40, c40_sh, c72, c72_sh;   // 2^40, 2^72 mod p (tensor-core MAC recombination) + Shoup
  uint64_t dec_I, dec_F;   // theta_l = t ((q/p)^-1 mod p) / p = dec_I + dec_F 2^-64 (RNS decryption, row f3)
  uint64_t mc;             // 2^50 - p if < 2^32 (pseudo-Mersenne fold 2^50 = mc mod p), else 0
  // tensor-core MAC epilogue (mac_tc.cuh): k_d = 2^(8d) mod p for the diagonals d = 7..12 as two
  // 25-bit limbs (k_d = ek0 + ek1 2^25); the fast recombination needs mc < 2^27
  uint32_t ek0[6], ek1[6];
  uint64_t delta;     // Delta mod p, Delta = floor(q / t)
  uint64_t delta_sh;  // Shoup companion of delta
  uint64_t ninv;      // N^-1 mod p
  uint64_t ninv_sh;
  uint64_t ninv_w1;   // N^-1 * psi^-bitrev(1) mod p (last inverse stage, folded)
  uint64_t ninv_w1_sh;
  // FP64 NTT constants (exact integer-valued doubles; pinv = 1/p rounded to nearest)
  double pd, pinv, ninv_d, ninv_w1_d;
};

struct DevParams {
  int N, logN, L, t_bits;
  PrimeConsts pc[HL_MAX_L];
  const double *twd_fwd;      // [L][N] psi^bitrev(i) as exact doubles
  const double *twd_inv;      // [L][N] psi^-bitrev(i)
};

// CUDA-event timing of kernel launches (hl_timing_enable / hl_timing_read)
struct TimingState {
  bool on = false;
  std::vector<void *> pool;                        // free cudaEvent_t
  std::vector<std::pair<int, std::pair<void *, void *>>> rec;   // (kernel class, (start, stop))
  int64_t kernels = 0;                             // kernel launches inside the timed sections
};

struct hl_ctx {
  uint32_t N, L, log2_t;
  int device;
  int num_sms = 148;
  int mac_engine = 2;                 // 0 = IMAD.WIDE limbs, 1 = exact FP64 products, 2 = int8 tensor cores (default)
  std::vector<uint64_t> primes;
  std::vector<uint64_t> psi;          // primitive 2N-th roots: g^((p-1)/2N), g the smallest primitive root (C26)
  std::vector<uint32_t> brv;          // bit reversal of log2(N) bits: natural evaluation index <-> NTT order
  std::vector<uint64_t> delta_mod;    // Delta mod p_l
  // big-integer constants for host decryption (little-endian u64 limbs, 4 limbs)
  uint64_t q_limbs[4];
  uint64_t half_q_limbs[4];
  uint64_t Ml_limbs[HL_MAX_L][4];     // q / p_l
  uint64_t Ml_inv[HL_MAX_L];          // (q / p_l)^-1 mod p_l
  uint64_t r_t;                       // q mod t  (noise-bound check)
  double log2_delta;
  // host twiddles (same tables as the device copy)
  std::vector<uint64_t> h_tw_fwd, h_tw_fwd_sh, h_tw_inv, h_tw_inv_sh;
  std::vector<uint64_t> cdt;          // 42 entries, floor(2^63 * P(|E| <= k))
  DevParams dp;
  void *d_tw = nullptr;               // device allocation holding tw_fwd + tw_inv
  uint32_t *d_flags = nullptr;        // device scratch: [0] range flag, [1] max |w| (as u32 bits)
  uint64_t *d_cdt = nullptr;          // device copy of the CDT table (device encryption, row f3)
  void *aux_stream = nullptr;         // cudaStream_t (non-blocking, lowest priority): hl_he_linear_batch's NTT stages
  void *mac_stream = nullptr;         // cudaStream_t (non-blocking, highest priority): hl_he_linear_batch's MACs
  void *fwd_stream = nullptr;         // cudaStream_t (non-blocking, lowest priority): hl_he_linear_batch_host's forward NTTs
  void *up_stream = nullptr;          // cudaStream_t (non-blocking): hl_he_linear_batch_host's uploads
  void *down_stream = nullptr;        // cudaStream_t (non-blocking): hl_he_linear_batch_host's downloads
  TimingState *timing = nullptr;      // owned; mutable through const hl_ctx*
  // cached cudaEvent_t of the batch calls (0: hl_he_linear_batch's pipeline, 1: the host batch's
  // copy stages), created on first use and reused: a call records and waits on them in stream order
  std::vector<void *> *ev_pool[2] = {nullptr, nullptr};   // owned; mutable through const hl_ctx*
};

// RAII event pair around one kernel launch when timing is on
struct KTimer {
  const hl_ctx *c; int kid; void *stream; void *ev0 = nullptr, *ev1 = nullptr;
  int nk = 1;                                      // kernels launched inside this section
  KTimer(const hl_ctx *c_, int kid_, void *stream_);
  ~KTimer();
};

// ---- error handling ------------------------------------------------------------------
void hl_set_error(const std::string &msg);
int hl_fail(int code, const std::string &msg);
int hl_cuda_check(const char *what);

// ---- host modular helpers --------------------------------------------------------------
static inline uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)(((hl_u128)a * b) % p); }
static inline uint64_t h_powmod(uint64_t b, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p; b %= p;
  while (e) { if (e & 1) r = h_mulmod(r, b, p); b = h_mulmod(b, b, p); e >>= 1; }
  return r;
}
static inline uint64_t h_shoup(uint64_t w, uint64_t p) { return (uint64_t)(((hl_u128)w << 64) / p); }

// tile geometry
struct Geo {
  int64_t nI, nJ, nK, nIs, i_begin, i_end;
  int m, r, n;
};
int hl_geometry(const hl_ctx *ctx, hl_tile tile, int64_t Ma, int64_t R, int64_t Nb, int64_t i_begin,
                int64_t i_end, Geo *g);

// host NTT (client side): natural-order in, bit-reversed out / inverse, canonical outputs
void hl_host_ntt_fwd(const hl_ctx *ctx, int l, uint64_t *a);
void hl_host_ntt_inv(const hl_ctx *ctx, int l, uint64_t *a);
