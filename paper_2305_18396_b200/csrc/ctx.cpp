// ctx.cpp -- context, parameters, twiddle tables, layouts and error reporting of libhelinear.
//
// Parameters follow PAPER.md:65 (§2.2: BFV-RNS with {N, t, q}, t = 2^l) with the readings of
// primes = the L largest p < 2^50 with p = 1 mod 2N (C4), Delta = floor(q/t) (C5),
// discrete Gaussian sigma = 3.2 by a CDT table (C8).  Independent of oracle/.
#include <cuda_runtime.h>
#include <quadmath.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "hl_internal.h"

// ---------------------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------------------
static thread_local std::string g_last_error;

void hl_set_error(const std::string &msg) { g_last_error = msg; }
int hl_fail(int code, const std::string &msg) { g_last_error = msg; return code; }
int hl_cuda_check(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return hl_fail(HL_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return HL_OK;
}

extern "C" const char *hl_last_error(void) { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------------------
// primes (reading C4) and roots
// ---------------------------------------------------------------------------------------
static bool is_prime_u64(uint64_t n) {
  if (n < 2) return false;
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (uint64_t b : bases) if (n % b == 0) return n == b;
  uint64_t d = n - 1; int s = 0;
  while (!(d & 1)) { d >>= 1; s++; }
  for (uint64_t a : bases) {      // deterministic for n < 3.3e24 with these 12 bases
    uint64_t x = h_powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < s; i++) { x = h_mulmod(x, x, n); if (x == n - 1) { comp = false; break; } }
    if (comp) return false;
  }
  return true;
}

// psi = g^((p-1)/2N) with g the smallest primitive root mod p (reading C26: the evaluation
// points psi^(2k+1) of the boundary's evaluation form are ordered by this psi).  p - 1 is
// factored by trial division: p - 1 = 2N * m with m < 2^38, so divisors up to 2^19 suffice.
static uint64_t find_psi(uint64_t p, uint32_t N) {
  std::vector<uint64_t> fac;
  uint64_t m = p - 1;
  for (uint64_t d = 2; d * d <= m; d++)
    if (m % d == 0) { fac.push_back(d); while (m % d == 0) m /= d; }
  if (m > 1) fac.push_back(m);
  for (uint64_t g = 2; g < 1000000; g++) {
    bool gen = true;
    for (uint64_t f : fac) if (h_powmod(g, (p - 1) / f, p) == 1) { gen = false; break; }
    if (!gen) continue;
    uint64_t psi = h_powmod(g, (p - 1) / (2ull * N), p);
    return h_powmod(psi, N, p) == p - 1 ? psi : 0;
  }
  return 0;
}

static uint32_t bitrev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

// ---------------------------------------------------------------------------------------
// small unsigned big integers (4 x u64, little endian) for q, q/p_l
// ---------------------------------------------------------------------------------------
static void big_mul_u64(uint64_t *a, uint64_t m) {   // a *= m (a has 4 limbs, no overflow)
  hl_u128 c = 0;
  for (int i = 0; i < 4; i++) { c += (hl_u128)a[i] * m; a[i] = (uint64_t)c; c >>= 64; }
}
static uint64_t big_mod_u64(const uint64_t *a, uint64_t m) {
  hl_u128 r = 0;
  for (int i = 3; i >= 0; i--) r = ((r << 64) | a[i]) % m;
  return (uint64_t)r;
}
static void big_div_u64(const uint64_t *a, uint64_t m, uint64_t *q) {
  hl_u128 r = 0;
  for (int i = 3; i >= 0; i--) { hl_u128 cur = (r << 64) | a[i]; q[i] = (uint64_t)(cur / m); r = cur % m; }
}
static void big_shr(const uint64_t *a, int s, uint64_t *out) {  // s < 64
  for (int i = 0; i < 4; i++) {
    uint64_t hi = (i + 1 < 4) ? a[i + 1] : 0;
    out[i] = s ? ((a[i] >> s) | (hi << (64 - s))) : a[i];
  }
}
static double big_log2(const uint64_t *a) {
  double v = 0;
  for (int i = 3; i >= 0; i--) v = v * 18446744073709551616.0 + (double)a[i];
  return log2(v);
}

// ---------------------------------------------------------------------------------------
// discrete Gaussian CDT (reading C8): T[k] = floor(2^63 * P(|E| <= k)), sigma = 3.2, |E| <= 41
// ---------------------------------------------------------------------------------------
static void build_cdt(std::vector<uint64_t> &T) {
  const int tail = 41;
  __float128 sigma = strtoflt128("3.2", nullptr), two_s2 = 2 * sigma * sigma;
  __float128 rho[tail + 1], Z = 0;
  for (int k = 0; k <= tail; k++) { rho[k] = expq(-(__float128)(k * k) / two_s2); Z += (k ? 2 : 1) * rho[k]; }
  T.assign(tail + 1, 0);
  __float128 acc = 0, two63 = ldexpq((__float128)1, 63);
  for (int k = 0; k <= tail; k++) {
    acc += (k ? 2 : 1) * rho[k];
    T[k] = (uint64_t)floorq(two63 * acc / Z);
  }
  T[tail] = 1ull << 63;
}

// ---------------------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------------------
extern "C" int hl_ctx_create(uint32_t N, uint32_t L, uint32_t log2_t, const uint64_t *primes,
                             int device, hl_ctx **out) {
  if (!out) return hl_fail(HL_EINVAL, "hl_ctx_create: out is NULL");
  *out = nullptr;
  if (N != 4096 && N != 8192) return hl_fail(HL_ENOTSUP, "hl_ctx_create: N must be 4096 or 8192");
  if (L < 1 || L > HL_MAX_L) return hl_fail(HL_ENOTSUP, "hl_ctx_create: 1 <= L <= 3 required");
  if (log2_t < 1 || log2_t > 62) return hl_fail(HL_ENOTSUP, "hl_ctx_create: 1 <= log2_t <= 62 required");
  hl_ctx *c = new hl_ctx();
  c->N = N; c->L = L; c->log2_t = log2_t; c->device = device;
  int logN = 0; while ((1u << logN) < N) logN++;
  if (primes) {
    for (uint32_t l = 0; l < L; l++) {
      uint64_t p = primes[l];
      if (p <= (1ull << 49) || p >= (1ull << 50) || (p - 1) % (2ull * N) != 0 || !is_prime_u64(p)) {
        delete c;
        return hl_fail(HL_ENOTSUP, "hl_ctx_create: primes must be primes in (2^49, 2^50) with p = 1 mod 2N");
      }
      for (uint32_t k = 0; k < l; k++)
        if (primes[k] == p) { delete c; return hl_fail(HL_EINVAL, "hl_ctx_create: primes must be distinct"); }
      c->primes.push_back(p);
    }
  } else {
    uint64_t step = 2ull * N, p = ((1ull << 50) - 1) / step * step + 1;
    while (c->primes.size() < L) { if (is_prime_u64(p)) c->primes.push_back(p); p -= step; }
  }
  // q, Delta = floor(q / t), Delta mod p_l, q / p_l, (q / p_l)^-1 mod p_l, r_t = q mod t
  uint64_t q[4] = {1, 0, 0, 0};
  for (uint64_t p : c->primes) big_mul_u64(q, p);
  memcpy(c->q_limbs, q, sizeof(q));
  big_shr(q, 1, c->half_q_limbs);
  uint64_t delta[4];
  {
    // Delta = q >> log2_t
    uint64_t tmp[4];
    int s = (int)log2_t;
    memcpy(tmp, q, sizeof(tmp));
    while (s >= 63) { big_shr(tmp, 63, delta); memcpy(tmp, delta, sizeof(tmp)); s -= 63; }
    big_shr(tmp, s, delta);
  }
  c->r_t = q[0] & ((1ull << log2_t) - 1);
  c->log2_delta = big_log2(delta);
  for (uint32_t l = 0; l < L; l++) {
    uint64_t p = c->primes[l];
    c->delta_mod.push_back(big_mod_u64(delta, p));
    big_div_u64(q, p, c->Ml_limbs[l]);
    c->Ml_inv[l] = h_powmod(big_mod_u64(c->Ml_limbs[l], p), p - 2, p);
  }
  // roots and twiddles: tw_fwd[i] = psi^bitrev(i), tw_inv[i] = psi^-bitrev(i)
  c->h_tw_fwd.resize((size_t)L * N); c->h_tw_fwd_sh.resize((size_t)L * N);
  c->h_tw_inv.resize((size_t)L * N); c->h_tw_inv_sh.resize((size_t)L * N);
  c->brv.resize(N);
  for (uint32_t i = 0; i < N; i++) c->brv[i] = bitrev(i, logN);
  std::vector<double> tw((size_t)2 * L * N);
  DevParams &dp = c->dp;
  dp.N = (int)N; dp.logN = logN; dp.L = (int)L; dp.t_bits = (int)log2_t;
  for (uint32_t l = 0; l < L; l++) {
    uint64_t p = c->primes[l];
    uint64_t psi = find_psi(p, N);
    if (!psi) { delete c; return hl_fail(HL_ENOTSUP, "hl_ctx_create: no 2N-th root of unity"); }
    c->psi.push_back(psi);
    uint64_t psi_inv = h_powmod(psi, p - 2, p);
    for (uint32_t i = 0; i < N; i++) {
      uint32_t br = bitrev(i, logN);
      uint64_t wf = h_powmod(psi, br, p), wi = h_powmod(psi_inv, br, p);
      size_t o = (size_t)l * N + i;
      c->h_tw_fwd[o] = wf; c->h_tw_fwd_sh[o] = h_shoup(wf, p);
      c->h_tw_inv[o] = wi; c->h_tw_inv_sh[o] = h_shoup(wi, p);
      tw[o] = (double)wf;                       // exact: w < 2^50
      tw[(size_t)L * N + o] = (double)wi;
    }
    PrimeConsts &pc = dp.pc[l];
    pc.p = p; pc.two_p = 2 * p;
    pc.mu = (uint64_t)((~(hl_u128)0 >> 64) / p);                 // floor((2^64 - 1) / p) = floor(2^64/p)
    pc.r64 = (uint64_t)(((hl_u128)1 << 64) % p);
    pc.r64_sh = h_shoup(pc.r64, p);
    pc.c40 = h_powmod(2, 40, p); pc.c40_sh = h_shoup(pc.c40, p);
    pc.mc = ((1ull << 50) - p) < (1ull << 32) ? (1ull << 50) - p : 0;
    for (int d = 7; d <= 12; d++) {
      const uint64_t k = h_powmod(2, 8 * d, p);
      pc.ek0[d - 7] = (uint32_t)(k & ((1u << 25) - 1));
      pc.ek1[d - 7] = (uint32_t)(k >> 25);
    }
    {   // RNS decryption constants: theta_l = t * inv_l / p_l = I + F / 2^64  (inv_l = (q/p_l)^-1 mod p_l)
      const hl_u128 ti = ((hl_u128)1 << log2_t) * c->Ml_inv[l];
      pc.dec_I = (uint64_t)(ti / p);
      pc.dec_F = (uint64_t)((((hl_u128)(uint64_t)(ti % p)) << 64) / p);
    }
    pc.c72 = h_powmod(2, 72, p); pc.c72_sh = h_shoup(pc.c72, p);
    pc.delta = c->delta_mod[l]; pc.delta_sh = h_shoup(pc.delta, p);
    pc.ninv = h_powmod(N, p - 2, p); pc.ninv_sh = h_shoup(pc.ninv, p);
    pc.ninv_w1 = h_mulmod(pc.ninv, c->h_tw_inv[(size_t)l * N + 1], p);
    pc.ninv_w1_sh = h_shoup(pc.ninv_w1, p);
    pc.pd = (double)p; pc.pinv = 1.0 / (double)p;
    pc.ninv_d = (double)pc.ninv; pc.ninv_w1_d = (double)pc.ninv_w1;
  }
  build_cdt(c->cdt);
  // device tables (device < 0: host-only context for the client calls; no CUDA needed)
  if (device < 0) {
    dp.twd_fwd = dp.twd_inv = nullptr;
    *out = c;
    return HL_OK;
  }
  if (cudaSetDevice(device) != cudaSuccess) { delete c; return hl_cuda_check("hl_ctx_create: cudaSetDevice"); }
  size_t bytes = tw.size() * sizeof(double);
  if (cudaMalloc(&c->d_tw, bytes) != cudaSuccess ||
      cudaMemcpy(c->d_tw, tw.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMalloc((void **)&c->d_flags, 64) != cudaSuccess) {
    int rc = hl_cuda_check("hl_ctx_create: device tables");
    if (c->d_tw) cudaFree(c->d_tw);
    delete c;
    return rc ? rc : hl_fail(HL_ECUDA, "hl_ctx_create: device allocation failed");
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc((void **)&c->d_cdt, c->cdt.size() * 8) != cudaSuccess ||
      cudaMemcpy(c->d_cdt, c->cdt.data(), c->cdt.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(c->d_tw); cudaFree(c->d_flags); delete c;
    return hl_cuda_check("hl_ctx_create: CDT table");
  }
  {
    // the batch pipeline's streams: MACs at the highest priority so that their persistent CTAs
    // are placed before queued NTT blocks of the concurrent low-priority stream
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const int fprio = lo;     // forward NTTs at the lowest priority (middle / highest measured no better)
    cudaStream_t aux, mac, up, down, fwd;
    if (cudaStreamCreateWithPriority(&aux, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&fwd, cudaStreamNonBlocking, fprio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&mac, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking) != cudaSuccess) {
      cudaFree(c->d_tw); cudaFree(c->d_flags); delete c;
      return hl_cuda_check("hl_ctx_create: pipeline streams");
    }
    c->ev_pool[0] = new std::vector<void *>();
    c->ev_pool[1] = new std::vector<void *>();
    c->aux_stream = (void *)aux;
    c->mac_stream = (void *)mac;
    c->up_stream = (void *)up;
    c->fwd_stream = (void *)fwd;
    c->down_stream = (void *)down;
  }
  dp.twd_fwd = (const double *)c->d_tw;
  dp.twd_inv = (const double *)c->d_tw + (size_t)L * N;
  *out = c;
  return HL_OK;
}

// ---------------------------------------------------------------------------------------
// kernel timing
// ---------------------------------------------------------------------------------------
static void *take_event(TimingState *ts) {
  if (!ts->pool.empty()) { void *e = ts->pool.back(); ts->pool.pop_back(); return e; }
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return (void *)e;
}

KTimer::KTimer(const hl_ctx *c_, int kid_, void *stream_) : c(c_), kid(kid_), stream(stream_) {
  if (!c->timing || !c->timing->on) return;
  ev0 = take_event(c->timing); ev1 = take_event(c->timing);
  if (ev0) cudaEventRecord((cudaEvent_t)ev0, (cudaStream_t)stream);
}

KTimer::~KTimer() {
  if (!ev0 || !ev1) return;
  cudaEventRecord((cudaEvent_t)ev1, (cudaStream_t)stream);
  c->timing->rec.push_back({kid, {ev0, ev1}});
  c->timing->kernels += nk;
}

extern "C" int hl_timing_kernels(hl_ctx *c, int64_t *n) {
  if (!c || !n) return hl_fail(HL_EINVAL, "hl_timing_kernels: NULL argument");
  *n = c->timing ? c->timing->kernels : 0;
  if (c->timing) c->timing->kernels = 0;
  return HL_OK;
}

extern "C" int hl_timing_enable(hl_ctx *c, int on) {
  if (!c) return hl_fail(HL_EINVAL, "hl_timing_enable: ctx is NULL");
  if (!c->timing) c->timing = new TimingState();
  c->timing->on = on != 0;
  return HL_OK;
}

extern "C" int hl_timing_read(hl_ctx *c, double *ms, int64_t *count) {
  if (!c || !ms || !count) return hl_fail(HL_EINVAL, "hl_timing_read: NULL argument");
  if (!c->timing) return HL_OK;
  // diagnostics: HELINEAR_TIMELINE=1 prints every section's (class, start, end) in ms relative to
  // the first recorded start (tools/gpu/timeline.py)
  static const bool timeline = getenv("HELINEAR_TIMELINE") != nullptr;
  for (auto &r : c->timing->rec) {
    float t = 0;
    if (cudaEventSynchronize((cudaEvent_t)r.second.second) != cudaSuccess ||
        cudaEventElapsedTime(&t, (cudaEvent_t)r.second.first, (cudaEvent_t)r.second.second) != cudaSuccess)
      return hl_cuda_check("hl_timing_read");
    if (timeline && !c->timing->rec.empty()) {
      float t0 = 0;
      cudaEventElapsedTime(&t0, (cudaEvent_t)c->timing->rec[0].second.first, (cudaEvent_t)r.second.first);
      fprintf(stderr, "[timeline] %d %.4f %.4f\n", r.first, t0, t0 + t);
    }
    if (r.first >= 0 && r.first < HL_K_COUNT) { ms[r.first] += t; count[r.first] += 1; }
    c->timing->pool.push_back(r.second.first);
    c->timing->pool.push_back(r.second.second);
  }
  c->timing->rec.clear();
  return HL_OK;
}

extern "C" int hl_ctx_destroy(hl_ctx *c) {
  if (!c) return HL_OK;
  if (c->timing) {
    for (void *e : c->timing->pool) cudaEventDestroy((cudaEvent_t)e);
    for (auto &r : c->timing->rec) { cudaEventDestroy((cudaEvent_t)r.second.first); cudaEventDestroy((cudaEvent_t)r.second.second); }
    delete c->timing;
  }
  for (auto *pool : c->ev_pool) {
    if (!pool) continue;
    for (void *e : *pool) cudaEventDestroy((cudaEvent_t)e);
    delete pool;
  }
  if (c->aux_stream) cudaStreamDestroy((cudaStream_t)c->aux_stream);
  if (c->mac_stream) cudaStreamDestroy((cudaStream_t)c->mac_stream);
  if (c->up_stream) cudaStreamDestroy((cudaStream_t)c->up_stream);
  if (c->fwd_stream) cudaStreamDestroy((cudaStream_t)c->fwd_stream);
  if (c->down_stream) cudaStreamDestroy((cudaStream_t)c->down_stream);
  if (c->d_tw) cudaFree(c->d_tw);
  if (c->d_flags) cudaFree(c->d_flags);
  if (c->d_cdt) cudaFree(c->d_cdt);
  delete c;
  return HL_OK;
}

extern "C" int hl_ctx_set_mac_engine(hl_ctx *c, int engine) {
  if (!c) return hl_fail(HL_EINVAL, "hl_ctx_set_mac_engine: ctx is NULL");
  if (engine < 0 || engine > 2) return hl_fail(HL_EINVAL, "hl_ctx_set_mac_engine: engine must be 0, 1 or 2");
  c->mac_engine = engine;
  return HL_OK;
}

extern "C" int hl_ctx_params(const hl_ctx *c, uint64_t *primes_out, uint64_t *delta_mod_out) {
  if (!c) return hl_fail(HL_EINVAL, "hl_ctx_params: ctx is NULL");
  for (uint32_t l = 0; l < c->L; l++) {
    if (primes_out) primes_out[l] = c->primes[l];
    if (delta_mod_out) delta_mod_out[l] = c->delta_mod[l];
  }
  return HL_OK;
}

int hl_geometry(const hl_ctx *c, hl_tile tile, int64_t Ma, int64_t R, int64_t Nb, int64_t i_begin,
                int64_t i_end, Geo *g) {
  if (!c) return hl_fail(HL_EINVAL, "ctx is NULL");
  if (tile.m <= 0 || tile.r <= 0 || tile.n <= 0 ||
      (int64_t)tile.m * tile.r * tile.n > (int64_t)c->N)
    return hl_fail(HL_EDIM, "tile (m, r, n) must be positive with m*r*n <= N");
  if ((tile.m & (tile.m - 1)) || (tile.r & (tile.r - 1)) || (tile.n & (tile.n - 1)))
    return hl_fail(HL_EDIM, "tile (m, r, n) must be powers of two (reading C2)");
  if (Ma <= 0 || R <= 0 || Nb <= 0) return hl_fail(HL_EINVAL, "Ma, R, Nb must be positive");
  g->m = tile.m; g->r = tile.r; g->n = tile.n;
  g->nI = (Ma + tile.m - 1) / tile.m;
  g->nJ = (R + tile.r - 1) / tile.r;
  g->nK = (Nb + tile.n - 1) / tile.n;
  if (i_end < 0) i_end = g->nI;
  if (i_begin < 0 || i_begin >= i_end || i_end > g->nI)
    return hl_fail(HL_EINVAL, "shard [i_begin, i_end) must be a non-empty sub-range of [0, nI)");
  g->i_begin = i_begin; g->i_end = i_end; g->nIs = i_end - i_begin;
  return HL_OK;
}

extern "C" int hl_layout_query(const hl_ctx *c, hl_tile tile, int64_t Ma, int64_t R, int64_t Nb,
                               int64_t i_begin, int64_t i_end, hl_layout *out) {
  Geo g;
  int rc = hl_geometry(c, tile, Ma, R, Nb, i_begin, i_end, &g);
  if (rc) return rc;
  if (!out) return hl_fail(HL_EINVAL, "hl_layout_query: out is NULL");
  int64_t LN = (int64_t)c->L * c->N;
  out->nI = g.nI; out->nJ = g.nJ; out->nK = g.nK; out->nI_shard = g.nIs;
  out->ct_in_words = g.nJ * g.nK * 2 * LN;
  out->ct_out_words = g.nIs * g.nK * 2 * LN;
  out->ct_masked_words = g.nIs * g.nK * (int64_t)c->L * ((int64_t)g.m * g.n + c->N);
  out->ct_full_words = g.nIs * g.nK * 2 * LN;
  out->share_words = Nb * Ma;
  const int64_t nIp = (g.nIs + 15) / 16 * 16;                     // I rows padded to 16 (MAC tiles)
  if (c->mac_engine == 2) {            // int8 tensor cores: 7 byte planes per residue, J padded to 32
    const int64_t nJp = (g.nJ + 31) / 32 * 32;
    out->wcache_bytes = nIp * nJp * LN * 7;
    out->workspace_bytes = nJp * g.nK * 2 * LN * 8 + 256;          // residues [cg][LN][nJp][CW] + MAC scheduler
  } else {
    out->wcache_bytes = nIp * g.nJ * LN * 8;
    out->workspace_bytes = g.nJ * g.nK * 2 * LN * 12;              // limb pairs + limb sums (MAC operand X)
  }
  return HL_OK;
}

// Tile planner: the cost model of include/helinear.h (constants from the B200 tile sweep,
// tools/gpu/tile_sweep.py).  Candidates: powers of two with m*r*n <= N and
// m <= Ma, r <= R, n <= Nb rounded up to a power of two (padded tiles cost what they move).
extern "C" int hl_plan_tile(const hl_ctx *c, int64_t Ma, int64_t R, int64_t Nb, hl_tile *out) {
  return hl_plan_tile_budget(c, Ma, R, Nb, 0, out);
}

// Effective rate of the tensor-core MAC on fat products (u8 limb MACs per second over the issued
// M = 64 / 128 rows), measured on c3/c4
static constexpr double kMacTcRate = 1.4e15;

extern "C" int hl_plan_tile_budget(const hl_ctx *c, int64_t Ma, int64_t R, int64_t Nb, int64_t max_wcache_bytes,
                                   hl_tile *out) {
  if (!c || !out) return hl_fail(HL_EINVAL, "hl_plan_tile: ctx or out is NULL");
  if (Ma <= 0 || R <= 0 || Nb <= 0) return hl_fail(HL_EINVAL, "hl_plan_tile: Ma, R, Nb must be positive");
  // transform cost per ciphertext relative to the calibration point N = 4096, L = 2
  const double ntt_scale = (double)c->N * c->L * (31 - __builtin_clz(c->N)) / (4096.0 * 2 * 12);
  auto ceil_pow2 = [](int64_t v) { int64_t p = 1; while (p < v) p <<= 1; return p; };
  const int64_t N = c->N, mmax = std::min<int64_t>(ceil_pow2(Ma), N), rmax = std::min<int64_t>(ceil_pow2(R), N),
                nmax = std::min<int64_t>(ceil_pow2(Nb), N);
  double best = 0;
  bool found = false;
  for (int64_t m = mmax; m >= 1; m >>= 1)
    for (int64_t r = rmax; r >= 1; r >>= 1)
      for (int64_t n = nmax; n >= 1; n >>= 1) {
      if (m * r * n > N) continue;
      hl_tile t{(int32_t)m, (int32_t)r, (int32_t)n};
      hl_layout lay;
      if (hl_layout_query(c, t, Ma, R, Nb, 0, -1, &lay) != HL_OK) continue;
      if (max_wcache_bytes > 0 && lay.wcache_bytes > max_wcache_bytes) continue;
      const double nC = 2.0 * lay.nK;
      const double e_mac = (nC <= 4 ? 1.0 : nC <= 8 ? 0.85 : 0.5) * std::min(1.0, (double)lay.nI / 96.0);
      // tensor-core work of the MAC as issued: balanced row tiles of <= 128 rows at M = 64 / 128,
      // J padded to the 32-J step, 49 limb products per modular MAC
      const int64_t nIp = (lay.nI + 15) / 16 * 16, nIt = (nIp + 127) / 128;
      const int64_t rt = ((nIp + nIt - 1) / nIt + 7) / 8 * 8;
      const double rows = (double)nIt * (rt <= 64 ? 64 : 128), nJp = (double)((lay.nJ + 31) / 32 * 32);
      const double t_tc = 49.0 * 2 * c->L * c->N * rows * nJp * (double)lay.nK / kMacTcRate;
      // the c0 inverse is pruned (to the class 15 mod 16 for r > 16, k_intt_c0_pruned)
      const double cost = std::max((double)lay.wcache_bytes / (6.2e12 * e_mac), t_tc) +
                          ntt_scale * (0.14e-6 * (double)(lay.nJ * lay.nK) + 0.10e-6 * (double)(lay.nI * lay.nK));
      if (!found || cost < best) { best = cost; *out = t; found = true; }
    }
  if (!found) return hl_fail(HL_EDIM, "hl_plan_tile: no tile fits the problem (or the weight-cache budget)");
  return HL_OK;
}

// ---------------------------------------------------------------------------------------
// host NTT (client side).  Same transform as the device kernels: merged-psi Cooley-Tukey
// forward (natural -> bit-reversed), Gentleman-Sande inverse (bit-reversed -> natural).
// ---------------------------------------------------------------------------------------
static inline uint64_t h_shoup_mul(uint64_t x, uint64_t w, uint64_t wsh, uint64_t p) {
  uint64_t qq = (uint64_t)(((hl_u128)x * wsh) >> 64);
  return x * w - qq * p;   // [0, 2p)
}

void hl_host_ntt_fwd(const hl_ctx *c, int l, uint64_t *a) {
  const uint32_t N = c->N;
  const uint64_t p = c->primes[l], p2 = 2 * p;
  const uint64_t *w = &c->h_tw_fwd[(size_t)l * N], *ws = &c->h_tw_fwd_sh[(size_t)l * N];
  for (uint32_t m = 1, t = N / 2; m < N; m <<= 1, t >>= 1)
    for (uint32_t i = 0; i < m; i++) {
      uint32_t j1 = 2 * i * t;
      for (uint32_t j = j1; j < j1 + t; j++) {
        uint64_t X = a[j]; if (X >= p2) X -= p2;
        uint64_t T = h_shoup_mul(a[j + t], w[m + i], ws[m + i], p);
        a[j] = X + T; a[j + t] = X - T + p2;
      }
    }
  for (uint32_t j = 0; j < N; j++) { uint64_t x = a[j]; if (x >= p2) x -= p2; if (x >= p) x -= p; a[j] = x; }
}

void hl_host_ntt_inv(const hl_ctx *c, int l, uint64_t *a) {
  const uint32_t N = c->N;
  const uint64_t p = c->primes[l], p2 = 2 * p;
  const uint64_t *w = &c->h_tw_inv[(size_t)l * N], *ws = &c->h_tw_inv_sh[(size_t)l * N];
  for (uint32_t m = N, t = 1; m > 1; m >>= 1, t <<= 1) {
    uint32_t h = m / 2;
    for (uint32_t i = 0; i < h; i++) {
      uint32_t j1 = 2 * i * t;
      for (uint32_t j = j1; j < j1 + t; j++) {
        uint64_t X = a[j], Y = a[j + t];
        uint64_t S = X + Y; if (S >= p2) S -= p2;
        a[j] = S;
        a[j + t] = h_shoup_mul(X - Y + p2, w[h + i], ws[h + i], p);
      }
    }
  }
  const PrimeConsts &pc = c->dp.pc[l];
  for (uint32_t j = 0; j < N; j++) {
    uint64_t x = h_shoup_mul(a[j], pc.ninv, pc.ninv_sh, p);
    if (x >= p) x -= p;
    a[j] = x;
  }
}
