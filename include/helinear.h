/*
 * helinear.h -- C ABI of the B200-native server-side homomorphic linear layer of
 * arxiv 2305.18396 ("Privacy-Computing-Friendly Transformer Inference"), Algorithm 1
 * (Pi_MatMul), with the response compression of §3.1.3
 * and the GPU cipher-plain multiply of PAPER.md:155-156.
 *
 * Roles (reading C1 of DESIGN.md §3): the server holds W (R x Ma), the
 * client holds its share X (Nb x R).  Alg. 1 is run on A = W^T (server, left operand) and
 * B = X^T (client, right operand); shares of C = A.B = (X.W)^T are emitted in the layout
 * of X.W, i.e. [Nb][Ma] (the transposition trick of PAPER.md:115, footnote).
 *
 * Ring and parameters (§2.2): BFV-RNS over R_q = Z_q[X]/(X^N+1),
 * q = p_0 ... p_{L-1}, plaintext modulus t = 2^log2_t, Delta = floor(q/t).
 *
 * Tiles (reading C2): an explicit (m, r, n) with m*r*n <= N.  Counts
 *   nI = ceil(Ma/m), nJ = ceil(R/r), nK = ceil(Nb/n); partial tiles are zero-padded.
 * Encodings (Alg. 1 step 1):
 *   pi_A: a_IJ[i*r + r-1-j] = lift(W[J*r+j][I*m+i]),  lift = centered [-t/2, t/2) (reading C6)
 *   pi_B: b_JK[k*m*r + j]   = X[K*n+k][J*r+j]
 * Decoding (Alg. 1 step 4): C[i][k] = c[pos(i,k)], pos(i,k) = k*m*r + i*r + r-1.
 *
 * Memory layouts (uint64 words; residues canonical in [0, p_l); little-endian hosts):
 *   X          [Nb][R]                      values < 2^log2_t
 *   W          [R][Ma]                      values < 2^log2_t (two's complement of the lift)
 *   sk         int8 [N]                     ternary {-1, 0, 1}
 *   ct_in      [nJ][nK][2][L][N]            (c0, c1) of Enc(pi_B(X^T tile JK))
 *   ct_out     [nI_s][nK][2][L][N]          Enc(c_IK) = sum_J a_IJ * ct_in[J][K]
 * Every ciphertext (input, output, masked) carries c0 in COEFFICIENT form and c1 in EVALUATION
 * form (reading C26 of DESIGN.md §3): c1_hat[k] = c1(psi_l^(2k+1)) mod p_l, k = 0..N-1 natural
 * order, psi_l = g_l^((p_l - 1)/2N) with g_l the smallest primitive root mod p_l.  Fresh c1 is
 * the PRF output itself (uniform in either form), so neither side transforms c1: the server
 * multiplies it pointwise and the client's decryption needs c1_hat . NTT(s) only.
 *   ct_masked  compressed: [nI_s][nK][ L*m*n (c0 at pos(i,k), index k*m+i) | L*N (c1) ]
 *              full:       [nI_s][nK][2][L][N]
 *   share      [Nb][Ma]                     (server share; a shard writes only its columns)
 *   wcache     opaque device bytes          NTT-domain pi_A polynomials of a shard of I tiles
 *   workspace  opaque device bytes          NTT-domain copy of ct_in
 * where a shard is the I-tile range [i_begin, i_end) (i_end = -1 means nI) and nI_s = i_end - i_begin.
 *
 * Randomness (reading C10): a ChaCha20 PRF (RFC 8439 block function), key = LE64(seed) || 0^24,
 * nonce = LE32(domain) || LE64(stream), block counter from 0; u64 word i = LE64(keystream[8i, 8i+8)).
 * Domains: 1 secret key (stream 0), 2 uniform a_hat (stream g*L + l), 3 error (stream g),
 * 4 mask (stream I*nK + K, I global).  g = J*nK + K.  Reading C28: domain 2 (the public a_hat = c1)
 * is keyed by the PUBLIC seed hl_public_seed(seed) = word 0 of stream (seed, domain 10, 0); domain 3
 * (the errors) by the client's private encryption seed itself, which never leaves the client.
 *
 * Ownership: the caller allocates and owns every buffer (host or device as stated per call).
 * The library owns only the context: parameters, per-prime constants and twiddle tables
 * (uploaded once to `device` at create) plus a few bytes of device scratch for status flags.
 * The library performs no device allocation after hl_ctx_create.
 *
 * Errors: every call returns HL_OK (0) or a negative code; hl_last_error() returns a
 * thread-local message describing the last failure on the calling thread.  Device calls
 * are enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy default stream)
 * and return after launch: asynchronous faults surface at the next synchronisation.
 * Contexts are immutable after creation and may be used concurrently from several threads
 * on different streams.
 */
#ifndef HELINEAR_H_
#define HELINEAR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HL_OK = 0,
  HL_EINVAL = -1,   /* null pointer, bad shard range, shape mismatch          */
  HL_EDIM = -2,     /* m*r*n > N or a non-positive tile dimension ("dims too large")        */
  HL_ERANGE = -3,   /* an input value >= 2^log2_t, or a secret key not ternary             */
  HL_ENOISE = -4,   /* static worst-case noise bound 2R*max|w|*(r_t + 41) >= Delta/2       */
  HL_ECUDA = -5,    /* a CUDA runtime error; the message carries cudaGetErrorString         */
  HL_ENOTSUP = -6   /* (N, L, log2_t) outside the built kernels: N in {4096, 8192},
                       1 <= L <= 3, primes in (2^49, 2^50), 1 <= log2_t <= 62              */
};

typedef struct hl_ctx hl_ctx;

typedef struct { int32_t m, r, n; } hl_tile;

typedef struct {
  int64_t nI, nJ, nK;         /* tile counts of the full problem                              */
  int64_t nI_shard;           /* i_end - i_begin                                              */
  int64_t ct_in_words;        /* nJ*nK*2*L*N                                                  */
  int64_t ct_out_words;       /* nI_shard*nK*2*L*N                                            */
  int64_t ct_masked_words;    /* compressed: nI_shard*nK*L*(m*n + N)                          */
  int64_t ct_full_words;      /* uncompressed masked: nI_shard*nK*2*L*N                       */
  int64_t share_words;        /* Nb*Ma                                                        */
  int64_t wcache_bytes;       /* engine 2 (default): ceil(nI_shard/16)*16 * ceil(nJ/32)*32 * L*N*7
                                 engines 0/1: ceil(nI_shard/16)*16 * nJ * L*N*8               */
  int64_t workspace_bytes;    /* engine 2: ceil(nJ/32)*32 * nK*2*L*N*8 + 256; engines 0/1: nJ*nK*2*L*N*12 */
} hl_layout;

/* ---- context ---------------------------------------------------------------------------- */

/* Thread-local description of the last error on this thread ("" if none). */
const char *hl_last_error(void);

/* Create a context for N, L primes, t = 2^log2_t on CUDA device `device`.
 * primes == NULL selects the L largest primes below 2^50 with p = 1 (mod 2N), descending
 * (reading C4); otherwise primes[0..L) must be distinct primes in (2^49, 2^50), p = 1 mod 2N.
 * device < 0 creates a host-only context: the client calls (keygen, encrypt, decrypt_share)
 * and the queries work, the device calls fail with HL_EINVAL. */
int hl_ctx_create(uint32_t N, uint32_t L, uint32_t log2_t, const uint64_t *primes, int device,
                  hl_ctx **out);
int hl_ctx_destroy(hl_ctx *ctx);

/* Select the MAC engine of he_matmul: 0 = IMAD.WIDE.U32 on 25-bit limbs,
 * 1 = exact FP64 products (error-free DFMA transformations), 2 = exact products on the int8
 * tensor cores (tcgen05.mma kind::i8, 7 byte limbs, TMEM accumulators; default).  Results are
 * bit-identical; the NTT-domain weight cache and workspace formats (and sizes, see
 * hl_layout_query) differ, so a cache must be encoded and used under the same engine.
 * Not thread-safe against concurrent calls on ctx. */
int hl_ctx_set_mac_engine(hl_ctx *ctx, int engine);

/* Copy the primes and Delta mod p_l (Delta = floor(q/t), reading C5) into caller arrays of L. */
int hl_ctx_params(const hl_ctx *ctx, uint64_t *primes_out, uint64_t *delta_mod_out);

/* Tile planner (reading C2: the tile is an explicit protocol parameter; the client encrypts and
 * decrypts with the tile the server announces).  Among the power-of-two tiles with m*r*n <= N,
 * m <= Ma, r <= R, n <= Nb (each rounded up to a power of two) it returns the one minimising a
 * cost model of the GPU path, calibrated on B200:
 *   T = Wbytes / (6.2 TB/s * e_mac) + 0.14 us * nJ*nK + 0.10 us * nI*nK
 * Wbytes = the padded weight cache (layout.wcache_bytes), nJ*nK forward and nI*nK inverse
 * transforms (ciphertexts; the c0 inverse is pruned), e_mac = (nC <= 4 ? 1 : nC <= 8 ? 0.85 : 0.5) * min(1, nI/96), nC = 2 nK
 * the MAC's columns.  Ties keep the first candidate (m, then r, then n descending).
 * c2 (BERT-base): QKV, FF1 -> (16, 8, 32); O -> (8, 8, 64); FF2 -> (4, 32, 32). */
int hl_plan_tile(const hl_ctx *ctx, int64_t Ma, int64_t R, int64_t Nb, hl_tile *out);

/* hl_plan_tile under a weight-cache budget: only tiles whose layout.wcache_bytes <= max_wcache_bytes
 * (<= 0: unlimited) are candidates -- a stack of layers must keep every layer's cache resident
 * (c4 on one GPU: 24 x 4.2 GB at n = 16 fits, the unconstrained choice at n = 32/64 does not).  The
 * cost model adds, for products with many columns per weight byte (c3, c4), the tensor-core time of
 * the MAC as issued (balanced row tiles at M = 64 / 128, J padded to 32, 49 limb products per
 * modular MAC) and scales the transform terms by N L log N relative to N = 4096, L = 2:
 *   T = max(Wbytes / (6.2 TB/s e_mac), T_tensor) + s (0.14 us nJ nK + 0.10 us nI nK).
 * HL_EDIM if no tile fits the budget. */
int hl_plan_tile_budget(const hl_ctx *ctx, int64_t Ma, int64_t R, int64_t Nb, int64_t max_wcache_bytes,
                        hl_tile *out);

/* Sizes of every buffer of one matmul (Ma x R weights, Nb tokens) for I-tile shard [i_begin, i_end). */
int hl_layout_query(const hl_ctx *ctx, hl_tile tile, int64_t Ma, int64_t R, int64_t Nb,
                    int64_t i_begin, int64_t i_end, hl_layout *out);

/* ---- client side (host memory; the boundary of the server path) ------------------------- */

/* Reading C28: the public seed of the A domain derived one-way from the private encryption seed
 * (u64 word 0 of the ChaCha20 stream (enc_seed, domain 10, stream 0)).  The seeded upload ships it. */
uint64_t hl_public_seed(uint64_t enc_seed);

/* Secret key s_i = (u64_SK[i] mod 3) - 1 (reading C7).  sk: host int8[N]. */
int hl_keygen(const hl_ctx *ctx, uint64_t seed, int8_t *sk);

/* Alg. 1 step 2: encode every tile with pi_B and encrypt with the secret key:
 *   c1 = a_hat_l (evaluation form, PRF domain 2 keyed by hl_public_seed(seed)),
 *   c0 = -a_l*s + e + Delta_l*b (mod p_l) with
 *   a_l = INTT(a_hat_l), e discrete Gaussian sigma=3.2 (CDT, reading C8; domain 3 keyed by seed).  X: host [Nb][R]; ct_in: host [nJ][nK][2][L][N] (layout.ct_in_words).
 * Errors: HL_ERANGE if some X >= 2^log2_t or sk is not ternary. */
int hl_encrypt(const hl_ctx *ctx, const int8_t *sk, hl_tile tile, const uint64_t *X, int64_t Nb,
               int64_t R, uint64_t seed, uint64_t *ct_in);

/* Alg. 1 step 4 on the client: m = c0 + c1*s, x = CRT(m) in [0, q),
 * y = floor((t*x + floor(q/2)) / q) mod t at pos(i,k); share_client[K*n+k][I*m+i] = y.
 * ct_masked: host, whole problem (shard [0, nI)); share_client: host [Nb][Ma]. */
int hl_decrypt_share(const hl_ctx *ctx, const int8_t *sk, hl_tile tile, const uint64_t *ct_masked,
                     int compress, int64_t Ma, int64_t Nb, uint64_t *share_client);

/* ---- client side on the GPU (device memory) ------------------------ */

/* NTT(s) per prime (slot order, device [L][N]) of the ternary secret sk (host int8[N]); the
 * device client calls take it instead of sk.  Synchronises `stream`.  HL_ERANGE if not ternary. */
int hl_sk_prepare(const hl_ctx *ctx, const int8_t *sk, uint64_t *s_hat, void *stream);

/* hl_encrypt on the GPU, bit-identical: X device [Nb][R] (< 2^log2_t, HL_ERANGE otherwise; the
 * check synchronises `stream`), ct_in device [nJ][nK][2][L][N]. */
int hl_encrypt_device(const hl_ctx *ctx, const uint64_t *s_hat, hl_tile tile, const uint64_t *X, int64_t Nb,
                      int64_t R, uint64_t seed, uint64_t *ct_in, void *stream);

/* hl_decrypt_share of a COMPRESSED response on the GPU, bit-identical (RNS rounding, see
 * client_dev.cuh): ct_masked device (whole problem), share_client device [Nb][Ma]. */
int hl_decrypt_share_device(const hl_ctx *ctx, const uint64_t *s_hat, hl_tile tile, const uint64_t *ct_masked,
                            int64_t Ma, int64_t Nb, uint64_t *share_client, void *stream);

/* ---- re-randomised responses (reading C22 of DESIGN.md) ---------- */

/* Client: public key pk = (pk0, pk1) = (-a s + e, a), host [2][L][N] coefficient form; a from
 * PRF domain 5 (stream l), e from domain 6 (stream 0). */
int hl_pk_gen(const hl_ctx *ctx, const int8_t *sk, uint64_t seed, uint64_t *pk);

/* Server: NTT(pk) per prime (device [2][L][N], slot order) from the host pk.  Synchronises. */
int hl_pk_prepare(const hl_ctx *ctx, const uint64_t *pk, uint64_t *pk_hat, void *stream);

/* hl_he_matmul_share (compressed) with every output ciphertext re-randomised before masking:
 *   c0 += pk0*u + e1 + F,  c1 += pk1*u + e2
 * u ternary (domain 7, stream I*nK+K), e1, e2 CDT (domain 8, streams 2(I*nK+K) and +1),
 * F[i] = (u64_RR_F[i] mod 2^flood_bits) - 2^(flood_bits-1) (domain 9; none for flood_bits = 0),
 * all from `seed` (the mask seed).  Closes the weight leak of reading C13 (the client no longer
 * sees sum_J pi_A(W) * a_J in c1); flooding hides the W-dependent noise up to the budget.  The
 * caller keeps the HE noise + 2^(flood_bits-1) below Delta/2 (HL_ERANGE unless
 * 0 <= flood_bits <= min(62, log2(Delta) - 1): F comes from one PRF word per coefficient).
 * rr_ws: device scratch of nI_shard*nK*L*N words. */
int hl_he_matmul_share_rr(const hl_ctx *ctx, hl_tile tile, const void *wcache, int64_t Ma, int64_t R,
                          int64_t Nb, int64_t i_begin, int64_t i_end, const uint64_t *ct_in, void *workspace,
                          uint64_t *ct_out_ntt, const uint64_t *pk_hat, int flood_bits, uint64_t *rr_ws,
                          uint64_t seed, uint64_t *ct_masked, uint64_t *share_server, void *stream);

/* ---- server side (device memory, stream-ordered) ----------------------------------------- */

/* hl_encode_weights_strided in two passes with a caller-provided device scratch of
 * nI_shard * nJ * L * N u64 words (layout.nI_shard, layout.nJ): the forward NTTs write u64
 * residues to scratch with coalesced stores, then one pass writes the tensor-core cache's byte
 * planes in 16-B chunks (the one-pass form scatters single bytes).  Bit-identical cache.
 * check = 0 skips the range / noise-bound verification and its stream synchronisation (online
 * encodings of operands the caller already bounds, e.g. the server's 37-bit shares of row f2);
 * check != 0 behaves as hl_encode_weights.  Other MAC engines ignore scratch. */
int hl_encode_weights_scratch(const hl_ctx *ctx, hl_tile tile, const uint64_t *W, int64_t R, int64_t Ma,
                              int64_t ld_row, int64_t ld_col, int64_t i_begin, int64_t i_end, void *wcache,
                              uint64_t *scratch, int check, void *stream);

/* Alg. 1 step 1 for the server + the NTT of PAPER.md:156 fn: pi_A of every
 * (I, J) tile with I in [i_begin, i_end), lifted (C6), reduced mod p_l, forward-NTT'd into
 * `wcache` (layout.wcache_bytes, device).  W: device [R][Ma].  Synchronises `stream` once to
 * check the input range and the static noise bound (offline call).
 * Errors: HL_ERANGE (W >= 2^log2_t), HL_ENOISE (worst-case noise >= Delta/2). */
int hl_encode_weights(const hl_ctx *ctx, hl_tile tile, const uint64_t *W, int64_t R, int64_t Ma,
                      int64_t i_begin, int64_t i_end, void *wcache, void *stream);

/* hl_encode_weights for a strided W: element (row k, column j) at W[k*ld_row + j*ld_col], e.g.
 * ld_row = 1, ld_col = R encodes the transpose of a row-major [Ma][R] matrix (the server operand
 * X1^T of the attention cross term X1 Y0, PAPER.md:115 footnote). */
int hl_encode_weights_strided(const hl_ctx *ctx, hl_tile tile, const uint64_t *W, int64_t R, int64_t Ma,
                              int64_t ld_row, int64_t ld_col, int64_t i_begin, int64_t i_end, void *wcache,
                              void *stream);

/* Alg. 1 step 3, homomorphic part: for every I in the shard and every K,
 *   ct_out[I][K][c] = sum_J a_IJ * ct_in[J][K][c]  mod (X^N + 1, p_l),  c in {0, 1}
 * computed as forward NTT of ct_in -> pointwise multiply-accumulate over J against the cached
 * NTT-domain weights -> inverse NTT (c0; c1 stays in evaluation form, reading C26).  ct_in: device
 * [nJ][nK][2][L][N]; workspace: device, layout.workspace_bytes; ct_out: device [nI_s][nK][2][L][N],
 * canonical residues. */
int hl_he_matmul(const hl_ctx *ctx, hl_tile tile, const void *wcache, int64_t Ma, int64_t R,
                 int64_t Nb, int64_t i_begin, int64_t i_end, const uint64_t *ct_in,
                 void *workspace, uint64_t *ct_out, void *stream);

/* Alg. 1 step 3, masking + §3.1.3 compression:
 *   sigma[pos] = u64_MASK(stream I*nK+K)[w(pos)] & (t-1), with the word order of reading C27: the
 *   kept positions pos(i,k) = k*m*r + i*r + r-1 take words 0 .. m*n-1 in kept-index order k*m+i,
 *   every other position the next word in position order (a permutation of [0, N));
 *   c0 <- c0 - Delta_l*sigma (mod p_l);
 *   compress != 0: keep c1 and c0 at pos(i,k) only;  share_server[K*n+k][I*m+i] = sigma[pos(i,k)].
 * ct_out: device [nI_s][nK][2][L][N]; ct_masked: device (layout.ct_masked_words or
 * ct_full_words); share_server: device [Nb][Ma], only the shard's columns are written. */
int hl_mask_and_share(const hl_ctx *ctx, hl_tile tile, int64_t Ma, int64_t Nb, int64_t i_begin,
                      int64_t i_end, const uint64_t *ct_out, uint64_t seed, int compress,
                      uint64_t *ct_masked, uint64_t *share_server, void *stream);

/* he_matmul followed by mask_and_share in one call: the inverse NTT and the masking /
 * compression / share extraction run as one fused kernel, so the coefficient-form ct_out is
 * never written.  Results are bit-identical to the two calls.  ct_out_ntt: device scratch of
 * layout.ct_out_words (holds the NTT-domain accumulators). */
int hl_he_matmul_share(const hl_ctx *ctx, hl_tile tile, const void *wcache, int64_t Ma, int64_t R,
                       int64_t Nb, int64_t i_begin, int64_t i_end, const uint64_t *ct_in,
                       void *workspace, uint64_t *ct_out_ntt, uint64_t seed, int compress,
                       uint64_t *ct_masked, uint64_t *share_server, void *stream);

/* One entry of hl_he_linear_batch: a product or an I-tile shard [i_begin, i_end) of it (the column
 * split of SURVEY.md §8(e): wcache holds that shard, ct_masked its nI_shard x nK responses, share
 * only its columns are written; mask streams use the global I, so shards are bit-identical slices
 * of the whole product), compressed responses.  i_end = -1 means nI; i_begin == i_end: the entry
 * is skipped (an empty shard of a rank when nI < ranks). */
typedef struct {
  const void *wcache;         /* hl_encode_weights output for this (Ma, R), device                */
  int64_t Ma, R, Nb;
  const uint64_t *ct_in;      /* device [nJ][nK][2][L][N]                                          */
  void *workspace;            /* device, layout.workspace_bytes -- distinct for every entry        */
  uint64_t *ct_out_ntt;       /* device, layout.ct_out_words    -- distinct for every entry        */
  uint64_t seed;              /* mask seed (as hl_mask_and_share)                                  */
  uint64_t *ct_masked;        /* device, layout.ct_masked_words (compressed response)              */
  uint64_t *share;            /* device [Nb][Ma] server share                                      */
  hl_tile tile;               /* this product's tile; m == 0: the tile argument of the batch call  */
  int64_t i_begin, i_end;     /* I-tile shard (0, -1: the whole product)                           */
} hl_linear_desc;

/* n compressed hl_he_matmul_share calls, e.g. the four products of an encoder block; results are
 * bit-identical to the calls made one after the other on `stream`.  The calls are pipelined over
 * the context's internal streams (joined to `stream` at entry and exit, so the call is ordered on
 * `stream` like a single kernel): the MACs in entry order on a high-priority stream, the forward
 * NTTs on a forward stream and each inverse NTT + mask on an auxiliary stream behind its MAC.  Two
 * schedules: with few columns per weight byte (some entry with nK < 8, e.g. c2)
 * every forward NTT is issued up front and shares SMs with the MACs; otherwise (c3/c4 token
 * counts) every MAC runs alone and only the forward NTT of entry i+1 overlaps the inverse of entry
 * i.  The internal streams are per context: batches issued concurrently on one context from
 * different caller streams serialise on them (use one context per concurrent caller). */
int hl_he_linear_batch(const hl_ctx *ctx, hl_tile tile, int n, const hl_linear_desc *descs, void *stream);

/* End-to-end server call on HOST buffers (the e2e path of bench.py): copies ct_in_host
 * (pinned host, [nJ][nK][2][L][N]) to dev_ct_in, runs hl_he_matmul_share, and copies the
 * masked response and the server share back to ct_masked_host / share_host (pinned host).
 * All device buffers are caller-owned; the call is stream-ordered (synchronise before reading). */
int hl_he_linear_host(const hl_ctx *ctx, hl_tile tile, const void *wcache, int64_t Ma, int64_t R,
                      int64_t Nb, const uint64_t *ct_in_host, uint64_t seed, int compress,
                      uint64_t *ct_masked_host, uint64_t *share_host, uint64_t *dev_ct_in,
                      void *workspace, uint64_t *dev_ct_out_ntt, uint64_t *dev_ct_masked,
                      uint64_t *dev_share, void *stream);

/* ---- Seeded ciphertext upload ------------------------------------ */

/* The c1 half of every input ciphertext is a_hat = PRF(a_seed, A, g*L + l) reduced mod p_l with
 * a_seed = hl_public_seed(enc_seed) (readings C10, C26, C28; the same stream hl_encrypt /
 * hl_encrypt_device draw), i.e. public randomness the client need not send: it uploads the c0 halves
 * and a_seed, and the server regenerates c1.  a_seed does not determine the error stream (keyed by
 * the private enc_seed), so the server learns nothing it could not read from the full ciphertext.
 * hl_expand_seeded writes the c1 halves of ct_in (device [nJ][nK][2][L][N] for (R, Nb)),
 * leaving the c0 halves untouched; the result is bit-identical to the client's ciphertext.
 * Stream-ordered; errors: HL_EINVAL (bad tile / sizes / null). */
int hl_expand_seeded(const hl_ctx *ctx, hl_tile tile, int64_t R, int64_t Nb, uint64_t a_seed,
                     uint64_t *ct_in, void *stream);

/* One entry of hl_he_linear_batch_host: the device buffers of a hl_he_linear_batch entry
 * (dev.ct_in is the upload target) plus pinned host buffers. */
typedef struct {
  hl_linear_desc dev;
  const uint64_t *c0_host;    /* pinned host [nJ][nK][L][N]: the c0 halves of the input ciphertexts */
  uint64_t a_seed;            /* hl_public_seed(client's encryption seed): c1 regenerated on device */
  uint64_t *ct_masked_host;   /* pinned host, layout.ct_masked_words (compressed response)         */
  uint64_t *share_host;       /* pinned host [Nb][Ma] server share                                 */
  int32_t packed;             /* 1: 50-bit wire format (hl_pack50) for c0_host and ct_masked_host  */
} hl_linear_host_desc;

/* 50-bit wire format for residues (every residue is < p_l < 2^50): each group of 32 words becomes
 * 25 words, residue i of a group at bit 50 i of the group's 1600-bit little-endian block; a last
 * partial group is zero-filled.  Packed length of w words: hl_packed50_words(w) = ceil(w/32)*25.
 * Host memory, OpenMP.  hl_pack50: HL_ERANGE if a word is >= 2^50. */
int64_t hl_packed50_words(int64_t words);
int hl_pack50(const uint64_t *in, int64_t words, uint64_t *out);
int hl_unpack50(const uint64_t *in, int64_t words, uint64_t *out);

/* The end-to-end form of hl_he_linear_batch (bench.py's e2e leg): for every entry, the c0 halves
 * are copied host->device (strided into dev.ct_in; packed = 1: the 50-bit stream of the c0 halves,
 * unpacked on the device through dev.workspace) and c1 is expanded from a_seed, the product
 * runs as in hl_he_linear_batch, and the compressed response + share are copied back to the host
 * buffers (packed = 1: the response in the 50-bit format, packed on the device through
 * dev.ct_out_ntt, hl_packed50_words(layout.ct_masked_words) words; the share stays u64).  The
 * packed format moves 25/32 of the bytes over PCIe, which bounds this call.  Entry i+1 uploads and entry i-1 downloads while entry i computes (the context's upload
 * / download streams).  Stream-ordered on `stream`: synchronise it before reading the host
 * outputs.  Results are bit-identical to hl_he_matmul_share on the client's full ciphertexts.
 * Do not run two batches on one context concurrently. */
int hl_he_linear_batch_host(const hl_ctx *ctx, hl_tile tile, int n, const hl_linear_host_desc *descs,
                            void *stream);

/* ---- FC layer, server side --------------------- */

/* With the layer input shared as x = <x>_0 + <x>_1 (client, server), the server's share of
 * y = W x + b is <y>_1 = <W<x>_0>_1 + W<x>_1 + b (mod 2^l), <W<x>_0>_1 being its share from
 * hl_mask_and_share / hl_he_matmul_share.  In the layout of X.W (reading C1):
 *   share[Nb][Ma] <- share + X1 . W + b   (mod 2^log2_t; b per output column)
 * computed exactly on the int8 tensor cores (5 byte limbs, only limb pairs a+b <= 4 survive
 * mod 2^37).  Supports log2_t <= 40 and R <= 6400 (HL_ENOTSUP otherwise). */

/* Buffer sizes: wplanes_bytes (hl_fc_encode_weights output), workspace_bytes (per call scratch). */
int hl_fc_layout(const hl_ctx *ctx, int64_t Nb, int64_t R, int64_t Ma, int64_t *wplanes_bytes,
                 int64_t *workspace_bytes);

/* Offline: W device [R][Ma] (< 2^log2_t, HL_ERANGE otherwise; synchronises `stream` once) ->
 * wplanes (device, opaque byte planes). */
int hl_fc_encode_weights(const hl_ctx *ctx, const uint64_t *W, int64_t R, int64_t Ma, void *wplanes,
                         void *stream);
/* Same, with the range check optional: check = 0 skips the status readback and its stream
 * synchronisation (the caller vouches for W < 2^log2_t, e.g. the server's own shares, which are
 * reduced mod 2^log2_t by construction -- row f2's online encodings); values
 * out of range then give unspecified (but memory-safe) results.  check != 0: hl_fc_encode_weights. */
int hl_fc_encode_weights_chk(const hl_ctx *ctx, const uint64_t *W, int64_t R, int64_t Ma, void *wplanes,
                             int check, void *stream);

/* Online: X1 device [Nb][R] (the server's share of the input, taken mod 2^log2_t), bias device [Ma]
 * or NULL, share device [Nb][Ma] (in/out), workspace device (hl_fc_layout). Stream-ordered. */
int hl_fc_local_share(const hl_ctx *ctx, const uint64_t *X1, const void *wplanes, const uint64_t *bias,
                      int64_t Nb, int64_t R, int64_t Ma, void *workspace, uint64_t *share, void *stream);

/* Share arithmetic (attention cross terms):
 * dst[rows][cols] <- dst + src (mod 2^log2_t), or dst + src^T when transpose != 0 (src then
 * [cols][rows]: the shares of (X1 Y0)^T returned by Pi_MatMul in the footnote-3 form).
 * Device buffers, stream-ordered. */
int hl_share_accumulate(const hl_ctx *ctx, uint64_t *dst, const uint64_t *src, int64_t rows, int64_t cols,
                        int transpose, void *stream);

/* ---- diagnostics (used by the parity tests and the NTT microbenchmark) -------------------- */

/* out[p] = a[p] * b[p] in Z_{p_l}[X]/(X^N+1) for p < npoly, through the device NTT/INTT
 * kernels.  a, b, out: device [npoly][L][N] canonical residues; out may alias a or b.
 * scratch: device, npoly*L*N*8*2 bytes. */
int hl_poly_mul(const hl_ctx *ctx, const uint64_t *a, const uint64_t *b, uint64_t *out,
                int64_t npoly, void *scratch, void *stream);

/* Forward NTT then inverse NTT of x in place (identity on canonical residues): exercises the
 * two transforms alone.  x: device [npoly][L][N]; scratch: device npoly*L*N*8 bytes. */
int hl_ntt_roundtrip(const hl_ctx *ctx, uint64_t *x, int64_t npoly, void *scratch, void *stream);

/* ---- per-kernel timing (bench.py's roofline evidence) ------------------------------------- */

enum {
  HL_K_NTT_FWD = 0,     /* forward NTT of ct_in (he_matmul step 1)                              */
  HL_K_MAC = 1,         /* slot-parallel modular multiply-accumulate over J (step 2)             */
  HL_K_INTT_MASK = 2,   /* fused inverse NTT + mask + compression + share (he_matmul_share)      */
  HL_K_INTT = 3,        /* inverse NTT (he_matmul step 3)                                        */
  HL_K_MASK = 4,        /* mask_and_share                                                        */
  HL_K_ENCODE = 5,      /* encode_weights (pi_A + forward NTT)                                   */
  HL_K_OTHER = 6,       /* diagnostics                                                           */
  HL_K_FC = 7,          /* FC local share (hl_fc_local_share)                                    */
  HL_K_COUNT = 8
};

/* on != 0: record a CUDA event pair on the launching stream around every kernel launch made
 * through ctx (adds ~2 event records per launch); on == 0: stop recording.  Mutates the
 * context's timing record: do not enable while other threads use the context. */
int hl_timing_enable(hl_ctx *ctx, int on);

/* Wait for the recorded events, ADD the summed durations (ms) and launch counts per kernel
 * class into ms[HL_K_COUNT] and count[HL_K_COUNT], then clear the record.  A timed section may
 * hold several kernels (e.g. the pruned c0 inverse + the c1 reorder): count[] counts sections. */
int hl_timing_read(hl_ctx *ctx, double *ms, int64_t *count);

/* Number of kernel launches inside the timed sections since the last call (then reset). */
int hl_timing_kernels(hl_ctx *ctx, int64_t *n);

#ifdef __cplusplus
}
#endif

#endif /* HELINEAR_H_ */
