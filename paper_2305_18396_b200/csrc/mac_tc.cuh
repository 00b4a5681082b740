// mac_tc.cuh -- the slot-parallel modular MAC on the 5th-generation tensor cores (tcgen05,
// kind::i8, accumulators in TMEM).  Included by kernels.cu inside its anonymous namespace.
//
// What it computes (the "elementwise multiplication" of PAPER.md:156 fn
// accumulated over the shared dimension, reading C3): for every prime l and NTT slot s,
//     out[I][col][s] = sum_J W[I][J][s] * X[J][col][s]  mod p_l          (W, X < p_l < 2^50)
// i.e. one small GEMM (nI x nJ) . (nJ x nC) per slot.  Exact integer products on int8 tensor
// cores: residues are split into 7 unsigned bytes, W = sum_a w_a 2^(8a), X = sum_b x_b 2^(8b),
//     sum_J W X = sum_{d=0..12} 2^(8d) S_d,   S_d = sum_{a+b=d} sum_J w_a x_b   (S_d < 2^31 for nJ <= 4096)
// and the tensor core forms every S_d directly: for limb plane a, MMA a multiplies A_a = w_a
// [128 I rows x 32 J] by the X limbs (B operand, row b*CW + c = x_b[c], N = 7 CW) and
// accumulates into the TMEM column window starting at a*CW, so column (a+b)*CW + c = d*CW + c
// collects S_d -- the Toeplitz structure lives in the accumulator address, not in a zero-padded
// B image (half the B operand, the MMA at its issue floor).  7 MMAs per 32-J step; the epilogue
// forms sum_d S_d 2^(8d) (< 2^124) and reduces it mod p_l once per output.
//
// Kernel roles (384 threads, one persistent CTA per SM):
//   warp 0      TMA producer: per (slot, 32-J step) one cp.async.bulk of the 7 weight planes
//               (224 B per I row, pre-laid-out by encode_weights in UMMA canonical K-major
//               no-swizzle form) and one of the X residues (u64, written by the forward NTT)
//   warp 1      TMEM allocator + single-thread MMA issuer (tcgen05.mma, tcgen05.commit)
//   warps 2-3   converters: u64 residues -> byte rows of the Toeplitz image Z (generic stores,
//               fence.proxy.async before release to the tensor core)
//   warps 4-11  epilogue (2 warps per TMEM lane quadrant, each half of the columns): tcgen05.ld
//               of S_d, recombination sum_d S_d 2^(8d) mod p, staging of 4 slots, full 32-B
//               sector stores of out[I][col][s..s+3]
// Work item = (I tile of RT <= 128 rows, column group of CW, 4 consecutive slots); the nI rows are
// split into balanced tiles (e.g. 144 = 2 x 72) and the ring depth is sized to the tile (more
// stages for short tiles, so that enough bytes stay in flight).  TMEM holds two accumulators so the
// epilogue of slot s overlaps the MMAs of slot s+1.
#pragma once

template <int CW>
struct TcGeom {
  static constexpr int NM = ((7 * CW + 15) / 16) * 16;   // MMA N: the 7 limbs x CW columns of X (+ zero pad)
  static constexpr int N = 6 * CW + NM;                  // accumulator width: columns d*CW + c, d < 13 (+ pad)
  static constexpr int ZR = NM;                          // rows of the X-limb B image: row b*CW + c = x_b[c]
  static constexpr int Z_BYTES = 2 * ZR * 16;            // one B image (Z ring entry)
  static constexpr int NZ = 4;                           // Z ring depth (decoupled from the TMA ring)
  static constexpr int RAW_BYTES = 32 * CW * 8;          // X residues of one 32-J step
  static constexpr int A_OFF = RAW_BYTES;                // TMA stage layout: [RAW][A (224 B per I row)]
  static constexpr int SPI = 4;                          // slots per work item (32-B output sectors)
  static constexpr int STG_STRIDE = CW * SPI + 1;        // u64 per staged row (+1: bank spread)
  // CW = 16: the epilogue keeps 2 slots x 8 columns of its row in registers and stores them
  // directly (16-B halves of the 32-B sectors, merged in L2) -- the 48 KB staging buffer would cost
  // the ring a stage; 4 slots in registers would exceed the 128 registers of 14 warps per SM
  static constexpr bool REG_EPI = CW >= 16;
  static constexpr int NBUF = 4 * N <= 512 ? 4 : 2;      // TMEM accumulators in flight (MMA runs ahead of the epilogue)
  static constexpr int TCOLS = NBUF * N <= 64 ? 64 : (NBUF * N <= 128 ? 128 : (NBUF * N <= 256 ? 256 : 512));
  static constexpr int MAX_NST = 24;
  static constexpr int BAR_BYTES = (2 * MAX_NST + 2 * NZ + 2 * NBUF + 2 * 4) * 8 + 4 * 4 + 16;
  // converter warps: each converts whole stages, the warps taking turns (stage z to warp z mod
  // NCONV), so NCONV stages are converted concurrently.  2 (12 warps per CTA: 3 per SM
  // sub-partition, so up to 168 registers per thread -- 4 converters would cap them at 128 and spill)
  static constexpr int NCONV = 2;
  // CW = 16: the converter warps take turns (one warp converts a whole stage, 2 stages in flight);
  // CW <= 8: both warps convert each stage (its conversion is short; measured faster on c2)
  static constexpr bool ALT_CONV = CW >= 16;
  // CW = 16: the accumulator columns [NM, N) that the a = 0 MMA does not initialise are zeroed by
  // one extra MMA per slot (A x a zero B image of N - NM = 96 rows, accumulate off) instead of
  // tcgen05.st by the epilogue warps (a 96-column store + wait per warp and slot)
  static constexpr bool ZMMA = CW >= 16;
  static constexpr int ZZ_BYTES = ZMMA ? 2 * (N - NM) * 16 : 0;   // the zero B image
  static constexpr int EPI0 = 2 + NCONV;                 // first epilogue warp
  // epilogue warps: 2 per TMEM lane quadrant (4 per quadrant measured: c4 -4 %, c3 +9 %: more warps
  // share the MMA warp's scheduler)
  static constexpr int NEPI = 8;
  static constexpr int CH = CW * 4 / NEPI;               // columns per epilogue warp
  static constexpr int THREADS = 32 * (EPI0 + NEPI);     // producer + MMA + converters + epilogue warps
  static constexpr int SMEM_MAX = 232448;                // 227 KB opt-in per CTA
  static_assert(A_OFF % 16 == 0 && Z_BYTES % 128 == 0, "alignment");
};

// ring geometry for a launch: rt rows per I tile (balanced tiles, multiple of 8)
struct TcRing { int nst, sbytes, a_off, c1_off, z_off, stg_off, bar_off, smem; };
template <int CW>
TcRing tc_ring(int rt, int smem_budget, int c1_bytes = 0, bool x_union = false) {
  using T = TcGeom<CW>;
  TcRing r;
  // the M = 128 MMA reads 128 rows of every plane (rows >= rt are don't-care): plane 6 starts at
  // 192 rt, row 127 of its second K half ends 2048 + 16 rt later -> 208 rt + 2048 >= 224 rt bytes.
  // Stage layout [X residues][A planes][c1 box]; x_union (every column group is pure c0 or pure c1,
  // so a stage holds either the X residues or the c1 box): [X residues | c1 box][A planes]
  const int a_end = 208 * rt + 2048;
  if (x_union) {
    r.c1_off = 0;
    r.a_off = (std::max(T::RAW_BYTES, c1_bytes) + 127) / 128 * 128;
    r.sbytes = (r.a_off + a_end + 127) / 128 * 128;
  } else {
    r.a_off = T::A_OFF;
    r.c1_off = (T::A_OFF + a_end + 127) / 128 * 128;
    r.sbytes = r.c1_off + (c1_bytes + 127) / 128 * 128;
  }
  const int stg = T::REG_EPI ? 0 : (rt * T::STG_STRIDE * 8 + 127) / 128 * 128;
  const int fixed = T::NZ * T::Z_BYTES + T::ZZ_BYTES + stg + T::BAR_BYTES;
  r.nst = std::max(2, std::min(T::MAX_NST, (std::min(smem_budget, T::SMEM_MAX) - fixed) / r.sbytes));
  r.z_off = r.nst * r.sbytes;
  r.stg_off = r.z_off + T::NZ * T::Z_BYTES + T::ZZ_BYTES;
  r.bar_off = r.stg_off + stg;
  r.smem = r.bar_off + T::BAR_BYTES;
  return r;
}

struct MacTcArgs {
  // c1 halves read straight from the ciphertexts (MacGeom::c1_in): 3-D tensor map over ct_in's c1
  // (natural evaluation points of all primes, K, J); per stage a box {2 points, c1_cols, 32 J}
  CUtensorMap c1map;
  const uint8_t *W;       // weight planes (encode_weights, engine 2 layout)
  const uint64_t *X;      // NTT-domain ct_in residues [nCg][LN][nJp][CW]
  uint64_t *out;          // [nIs][nC][LN] canonical residues
  MacGeom g;
  TcRing ring;
  int N, jc0, njc, accumulate;
  unsigned long long *prof;   // diagnostics (HELINEAR_MAC_PROF): per-CTA cycles spent waiting, by role
  int *sched;                 // work counter (zeroed before the launch; in the caller's workspace)
  int lazy_out;               // 1: outputs only < 2^52 (= residue + k p, k < 4): fine for the inverse NTT's input
  // c1 straight into the compressed response (fused paths, cperm, one launch): columns C >= c1_nK
  // (the c1 halves) are written canonical, in natural evaluation order (reading C26), at
  // c1_out + o L (mn + N) + L mn + l N + k, o = row nK + (C - nK) -- k_c1_out's result, without the
  // NTT-domain round trip through `out`.  c1_out == nullptr: off.
  uint64_t *c1_out;
  int c1_nK, c1_mn, c1_lognt;
  int qperm;                  // quad order (load_ntt_domain_q): set with c1_out
  int c1_in, c1_cols, c1_bytes;   // c1 from c1map (requires qperm): columns per c1 group, box bytes
  int out_v4, c1_v4;          // the output sectors (out / c1_out) are 32-B aligned: 256-bit stores
};

// one 32-B output sector: a single 256-bit store (STG.256, sm_100) when 32-B aligned, else two 16-B
// halves.  The epilogue's stores are scattered sectors (one per output row and column of an item):
// one instruction per sector instead of two halved its store-side stall (c4 MAC 707 -> 445 ms per
// stack, c3 27.0 -> 25.2 ms, c2 0.780 -> 0.766 ms per block)
__device__ __forceinline__ void st_sector(uint64_t *dst, uint64_t v0, uint64_t v1, uint64_t v2, uint64_t v3, int v4) {
  if (v4) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "l"(v0), "l"(v1), "l"(v2), "l"(v3) : "memory");
  } else {
    reinterpret_cast<ulonglong2 *>(dst)[0] = make_ulonglong2(v0, v1);
    reinterpret_cast<ulonglong2 *>(dst)[1] = make_ulonglong2(v2, v3);
  }
}

// natural evaluation point (prime offset l N included) of the first slot of quad sq (quad order)
__device__ __forceinline__ int tc_quad_k0(const MacTcArgs &A, int sq) {
  const int pos = sq * 4, l = pos / A.N, rem = pos - l * A.N;
  const int nt = 1 << A.c1_lognt, u = rem >> A.c1_lognt, tq = (rem & (nt - 1)) >> 2;
  return l * A.N + (int)(__brev((unsigned)u) >> 28) * nt + (int)(__brev((unsigned)tq) >> (32 - A.c1_lognt));
}
// first c1 column of column group cg (CW columns; c1 columns are those >= nK), CW if none
template <int CW>
__device__ __forceinline__ int tc_c1_lo(const MacTcArgs &A, int cg) {
  return A.c1_in ? max(0, min(CW, A.c1_nK - cg * CW)) : CW;
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
               : "memory");
}

// slot of the si-th output of slot quad sq: consecutive slots, or (qperm) the quad order
// u NT + t' + {0, 2, 1, 3}[si] NT/4 whose natural evaluation points are 4 consecutive k
__device__ __forceinline__ int tc_slot(const MacTcArgs &A, int sq, int si) {
  if (!A.qperm) return sq * 4 + si;
  const int pos = sq * 4, l = pos / A.N, rem = pos - l * A.N;
  const int nt = 1 << A.c1_lognt, u = rem >> A.c1_lognt, tq = (rem & (nt - 1)) >> 2;
  return l * A.N + u * nt + tq + ((si & 1) << 1 | (si >> 1)) * (nt >> 2);
}

// UMMA shared-memory descriptor: K-major, no swizzle; core matrix = 8 rows x 16 B contiguous.
// lbo = byte distance between the two 16-B K halves, sbo = between 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
// instruction descriptor kind::i8: A, B unsigned 8-bit K-major, D s32, M x N
__host__ __device__ constexpr uint32_t umma_idesc_u8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
// Role profiling (HELINEAR_MAC_PROF=1 at run time) is compiled in only with -DHL_MAC_PROF
// (HELINEAR_NVCC_EXTRA): the MMA warp's per-stage path is sensitive to every instruction (the
// checks alone cost c2 1.5 %).
#ifdef HL_MAC_PROF
constexpr bool kProf = true;
#else
constexpr bool kProf = false;
#endif
// mbarrier wait that, when profiling, adds the cycles spent waiting to *acc
__device__ __forceinline__ void mbar_wait_p(uint64_t *bar, uint32_t parity, unsigned long long *acc) {
  if (acc) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    *acc += (unsigned long long)(clock64() - t0);
  } else {
    mbar_wait(bar, parity);
  }
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

template <int CW>
__device__ __forceinline__ void tmem_ld_cw(uint32_t addr, uint32_t (&v)[CW]) {
  if constexpr (CW == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v[0]) : "r"(addr));
  } else if constexpr (CW == 2) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(addr));
  } else if constexpr (CW == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
  } else if constexpr (CW == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(addr));
  }
}

// zero CH consecutive accumulator columns of the warp's 32 lanes
template <int CH>
__device__ __forceinline__ void tmem_zero_cw(uint32_t addr) {
  if constexpr (CH == 1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(addr), "r"(0u));
  } else if constexpr (CH == 2) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%1};" ::"r"(addr), "r"(0u));
  } else if constexpr (CH == 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(addr), "r"(0u));
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(addr), "r"(0u));
  }
}

// Dynamic work schedule: the producer takes the next item from a global counter (in the caller's
// workspace, zeroed before the launch) and hands it to the other roles through a 4-deep ring in
// shared memory, so CTAs that start late (e.g. behind NTT blocks of a concurrent kernel) simply
// take fewer items.  Consecutive items share a slot quad (kind fastest): the X residues of the
// quad are re-read from L2 by the CTAs working on its other (I tile, column group) kinds.
struct TcItem { int t, cg, sq; };
__device__ __forceinline__ TcItem tc_decode(const MacGeom &g, int item) {
  const int kinds = g.nIt * g.nCg, kind = item % kinds;
  TcItem it;
  it.sq = item / kinds;
  it.t = kind / g.nCg;
  it.cg = kind % g.nCg;
  return it;
}
constexpr int kItemRing = 4;
// consumers of an item: the MMA warp + the converter warps + 8 epilogue warps (lane 0 each)
// consumer side: wait for item number `seq`, read it, release the ring slot; returns -1 at the end
__device__ __forceinline__ int tc_next_item(uint64_t *ifull, uint64_t *iempty, const volatile int *itm, uint32_t seq) {
  const int slot = seq % kItemRing;
  mbar_wait(&ifull[slot], (seq / kItemRing) & 1);
  const int item = itm[slot];
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&iempty[slot]);
  return item;
}

// one converter unit: the limb rows b*CW + c and b*CW + c + 1 (b < 7) for the 4 consecutive J of
// 32-bit word gq in K half h of the Toeplitz image z, from the 4 x 2 residues x0 (column c) and x1
// (column c+1).  Lanes of a warp cover the column pairs fastest: with the two stores in a lane-
// dependent order (swap = column pair >= 4) a warp's 32 stores hit 32 distinct banks.
template <int CW, int ZR>
__device__ __forceinline__ void conv_unit(unsigned char *z, int h, int c, int gq, const uint64_t (&x0)[4],
                                          const uint64_t (&x1)[4], bool swap) {
  uint32_t *row = reinterpret_cast<uint32_t *>(z + ((size_t)h * ZR + c) * 16) + gq;
  const uint32_t l0[4] = {(uint32_t)x0[0], (uint32_t)x0[1], (uint32_t)x0[2], (uint32_t)x0[3]};
  const uint32_t h0[4] = {(uint32_t)(x0[0] >> 32), (uint32_t)(x0[1] >> 32), (uint32_t)(x0[2] >> 32), (uint32_t)(x0[3] >> 32)};
  const uint32_t l1[4] = {(uint32_t)x1[0], (uint32_t)x1[1], (uint32_t)x1[2], (uint32_t)x1[3]};
  const uint32_t h1[4] = {(uint32_t)(x1[0] >> 32), (uint32_t)(x1[1] >> 32), (uint32_t)(x1[2] >> 32), (uint32_t)(x1[3] >> 32)};
  const int f = swap ? 4 : 0;                            // u32 offset of the first store (column c+1 if swap)
#pragma unroll
  for (int b = 0; b < 7; b++) {
    const uint32_t *s0 = b < 4 ? l0 : h0, *s1 = b < 4 ? l1 : h1;
    const uint32_t bb = b & 3, sel = bb | ((bb + 4) << 4);
    const uint32_t w0 = __byte_perm(__byte_perm(s0[0], s0[1], sel), __byte_perm(s0[2], s0[3], sel), 0x5410);
    const uint32_t w1 = __byte_perm(__byte_perm(s1[0], s1[1], sel), __byte_perm(s1[2], s1[3], sel), 0x5410);
    row[b * CW * 4 + f] = swap ? w1 : w0;
    row[b * CW * 4 + (4 - f)] = swap ? w0 : w1;
  }
}

// FAST: every prime has 2^50 - p < 2^27 (the fast epilogue recombination; the launch checks)
template <int CW, bool FAST>
// <= 80 registers for CW <= 8 (minBlocks 2): leaves room for NTT CTAs on the same SM when the
// MAC of one matmul runs concurrently with the NTTs of its neighbours (hl_he_linear_batch)
__global__ void __launch_bounds__(TcGeom<CW>::THREADS, (CW <= 8 ? 2 : 1))
k_mac_tc(const __grid_constant__ MacTcArgs A, DevParams P) {
  using T = TcGeom<CW>;
  const int NST = A.ring.nst, SB = A.ring.sbytes;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *stg = reinterpret_cast<uint64_t *>(smem + A.ring.stg_off);
  unsigned char *zring = smem + A.ring.z_off;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + A.ring.bar_off);
  uint64_t *empty = full + NST, *zfull = empty + NST, *zempty = zfull + T::NZ;
  uint64_t *tfull = zempty + T::NZ, *tempty = tfull + T::NBUF;
  uint64_t *ifull = tempty + T::NBUF, *iempty = ifull + kItemRing;
  int *itm = reinterpret_cast<int *>(iempty + kItemRing);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(itm + kItemRing);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const MacGeom &g = A.g;
  const int total_items = g.nIt * g.nCg * (g.LN / 4);

  // ---- setup: zero the Toeplitz images (only data rows are rewritten), barriers, TMEM
  for (int i = threadIdx.x; i < (T::NZ * T::Z_BYTES + T::ZZ_BYTES) / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(zring)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < T::NZ; i++) { mbar_init(&zfull[i], T::ALT_CONV ? 32 : 64); mbar_init(&zempty[i], 1); }
    for (int i = 0; i < T::NBUF; i++) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], T::NEPI); }
    for (int i = 0; i < kItemRing; i++) { mbar_init(&ifull[i], 1); mbar_init(&iempty[i], 1 + T::NCONV + T::NEPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "n"(T::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // The limb-plane MMA a accumulates into the column window [a*CW, a*CW + NM) of its buffer (the
  // Toeplitz shift lives in the accumulator address): columns [NM, N) must start at zero.  The
  // epilogue re-zeroes them after draining a buffer; here every buffer is zeroed once.
  if (!T::ZMMA && warp >= T::EPI0) {
    const uint32_t lanes = (uint32_t)(32 * (warp & 3)) << 16;
    for (int b = 0; b < T::NBUF; b++)
      for (int col = T::NM + ((warp - T::EPI0) >> 2); col < T::N; col += 2)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lanes + b * T::N + col), "r"(0u));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  unsigned long long pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // profiling accumulators (registers, kProf)
  const long long t_start = clock64();

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 1;
      uint64_t pol_w;                     // the weight cache is streamed once: evict it from L2 first
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
      for (uint32_t seq = 0;; seq++) {
        const int slot = seq % kItemRing;
        mbar_wait(&iempty[slot], ((seq / kItemRing) & 1) ^ 1);
        const int item = atomicAdd(A.sched, 1);
        itm[slot] = item < total_items ? item : -1;
        mbar_arrive(&ifull[slot]);
        if (item >= total_items) break;
        const TcItem it = tc_decode(g, item);
        const int rows = min(g.RT, g.nIp - g.RT * it.t);
        const uint32_t abytes = 224u * rows;
        const uint8_t *wt = A.W + (size_t)it.t * g.RT * g.LN * g.nJp * 7;
        const int c1lo = tc_c1_lo<CW>(A, it.cg);
        const bool xraw = c1lo > 0, xc1 = c1lo < CW;             // this group's c0 / c1 columns
        const int kq0 = xc1 ? tc_quad_k0(A, it.sq) : 0;
        const int K1 = xc1 ? it.cg * CW + c1lo - A.c1_nK : 0;     // first c1 column's K
        const uint32_t rawb = 256u * g.xw;                        // 32 J x xw u64
        const uint32_t tx = abytes + (xraw ? rawb : 0) + (xc1 ? A.c1_bytes : 0);
        for (int si = 0; si < T::SPI; si++) {
          const int s = tc_slot(A, it.sq, si);
          for (int kk = 0; kk < A.njc; kk++) {
            const int jc = A.jc0 + kk;
            mbar_wait_p(&empty[st], ph, (kProf && A.prof) ? &pw[0] : nullptr);
            unsigned char *dst = smem + st * SB;
            mbar_expect_tx(&full[st], tx);
            bulk_g2s_hint(dst + A.ring.a_off, wt + ((size_t)s * g.nJc + jc) * abytes, abytes, &full[st], pol_w);
            if (xraw)
              bulk_g2s(dst, A.X + (((size_t)it.cg * g.LN + s) * g.nJp + (size_t)jc * 32) * g.xw, rawb, &full[st]);
            if (xc1)   // natural points k0 + (si & 2) .. +1 of the group's c1 columns, 32 J
              tma_load_3d(dst + A.ring.c1_off, &A.c1map, kq0 + (si & 2), K1, jc * 32, &full[st]);
            if (++st == NST) { st = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (every value is warp-uniform, so descriptors live in uniform
    // registers) and one elected lane issues: a per-MMA register->uniform conversion in a
    // single-lane branch costs more than the MMA itself (profiles/r01/microbench_umma_i8_cost.log).
    // tiles of <= 64 rows use M = 64 (half the A-operand shared-memory reads per MMA); the
    // accumulator rows then sit in lanes 32(r/16) + r%16 (profiles/r01/microbench_umma_i8.log)
    // M per item: tiles of <= 64 rows (also a short last tile of uneven tiling) use M = 64
    const uint32_t zdesc128 = umma_idesc_u8(128, T::ZMMA ? T::N - T::NM : 16);
    const uint32_t zdesc64 = umma_idesc_u8(64, T::ZMMA ? T::N - T::NM : 16);
    const uint32_t zz = smem_u32(zring + T::NZ * T::Z_BYTES);     // the zero B image (ZMMA)
    const uint32_t idesc128 = umma_idesc_u8(128, T::NM);
    const uint32_t idesc64 = umma_idesc_u8(64, T::NM);
    int st = 0;
    uint32_t ph = 0;
    uint32_t tile_no = 0, zseq = 0;
    for (uint32_t seq = 0;; seq++) {
      const int item = tc_next_item(ifull, iempty, itm, seq);
      if (item < 0) break;
      const TcItem it = tc_decode(g, item);
      const int rows = min(g.RT, g.nIp - g.RT * it.t);
      const uint32_t plane = 32u * rows, lbo_a = 16u * rows;
      const uint32_t idesc = rows <= 64 ? idesc64 : idesc128;
      for (int si = 0; si < T::SPI; si++, tile_no++) {
        const uint32_t buf = tile_no % T::NBUF, tph = (tile_no / T::NBUF) & 1;
        mbar_wait_p(&tempty[buf], tph ^ 1, (kProf && A.prof && lane == 0) ? &pw[1] : nullptr);
        tc_fence_after();
        const uint32_t dcol = tmem + buf * T::N;
        for (int kk = 0; kk < A.njc; kk++, zseq++) {
          const uint32_t zi = zseq % T::NZ, zph = (zseq / T::NZ) & 1;
          // Only zfull: the converter arrives on zfull after it observed full[st] (the stage's TMA
          // bytes, the A planes included, complete), so the acquire on zfull orders the MMA's reads
          // of the stage after the TMA writes (mbarrier arrive = release, try_wait = acquire) -- one
          // mbarrier poll less on the MMA warp's per-stage path (c3: MAC -3 %)
          mbar_wait_p(&zfull[zi], zph, (kProf && A.prof && lane == 0) ? &pw[3] : nullptr);
          tc_fence_after();
          const long long ti0 = (kProf && A.prof) ? clock64() : 0;
          const uint32_t a0 = smem_u32(smem + st * SB) + A.ring.a_off;
          const uint32_t z0 = smem_u32(zring + zi * T::Z_BYTES);
          if (elect_one()) {
            if constexpr (T::ZMMA) {
              if (kk == 0)       // zero the columns [NM, N) the a = 0 MMA does not write
                umma_i8(dcol + T::NM, umma_sdesc(a0, lbo_a, 128), umma_sdesc(zz, (T::N - T::NM) * 16, 128),
                        rows <= 64 ? zdesc64 : zdesc128, 0u);
            }
#pragma unroll
            for (int a = 0; a < 7; a++) {
              const uint64_t ad = umma_sdesc(a0 + a * plane, lbo_a, 128);
              const uint64_t bd = umma_sdesc(z0, T::ZR * 16, 128);
              umma_i8(dcol + a * CW, ad, bd, idesc, (kk | a) ? 1u : 0u);   // D window shifted by a*CW
            }
            umma_commit(&empty[st]);
            umma_commit(&zempty[zi]);
          }
          __syncwarp();
          if (kProf && A.prof && lane == 0) pw[6] += (unsigned long long)(clock64() - ti0);
          if (++st == NST) { st = 0; ph ^= 1; }
        }
        if (elect_one()) umma_commit(&tfull[buf]);
        __syncwarp();
      }
    }
  } else if (warp < T::EPI0) {
    // ------------------------------------------------------------------ converters
    // CW <= 8: both converter warps convert every stage, one column of 4 J per thread
    if constexpr (!T::ALT_CONV) {
    const int ct = threadIdx.x - 64;
    int st = 0;
    uint32_t ph = 0, zseq = 0;
    for (uint32_t seq = 0;; seq++) {
      const int item = tc_next_item(ifull, iempty, itm, seq);
      if (item < 0) break;
      const int c1lo = tc_c1_lo<CW>(A, tc_decode(g, item).cg);
      for (int si = 0; si < T::SPI; si++) {
        for (int kk = 0; kk < A.njc; kk++, zseq++) {
          const uint32_t zi = zseq % T::NZ, zph = (zseq / T::NZ) & 1;
          mbar_wait_p(&full[st], ph, (kProf && A.prof && ct == 0) ? &pw[4] : nullptr);
          mbar_wait(&zempty[zi], zph ^ 1);
          const uint64_t *raw = reinterpret_cast<const uint64_t *>(smem + st * SB);
          const uint64_t *c1b = reinterpret_cast<const uint64_t *>(smem + st * SB + A.ring.c1_off) + (si & 1);
          unsigned char *z = zring + zi * T::Z_BYTES;
          constexpr int QIT = (CW * 8 + 63) / 64;
#pragma unroll
          for (int qi = 0; qi < QIT; qi++) {
            const int q = ct + qi * 64;
            if (q >= CW * 8) break;
            const int c = q >> 3, h = (q >> 2) & 1, gq = q & 3;
            const int j0 = h * 16 + gq * 4;
            uint32_t lo[4], hi[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
              // c0 columns from the forward NTT's X chunk [J][CW]; c1 columns from the box [J][K][2]
              const uint64_t x = c < c1lo ? raw[(j0 + j) * g.xw + c] : c1b[((j0 + j) * A.c1_cols + (c - c1lo)) * 2];
              lo[j] = (uint32_t)x; hi[j] = (uint32_t)(x >> 32);
            }
            uint32_t *zrow = reinterpret_cast<uint32_t *>(z + ((size_t)h * T::ZR + c) * 16) + gq;
#pragma unroll
            for (int b = 0; b < 7; b++) {
              const uint32_t *src = b < 4 ? lo : hi;
              const uint32_t bb = b & 3;
              const uint32_t sel = bb | ((bb + 4) << 4);
              const uint32_t t01 = __byte_perm(src[0], src[1], sel);
              const uint32_t t23 = __byte_perm(src[2], src[3], sel);
              zrow[b * CW * 4] = __byte_perm(t01, t23, 0x5410);   // row b*CW + c
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&zfull[zi]);
          if (++st == NST) { st = 0; ph ^= 1; }
        }
      }
    }
    } else {
    // Converter warp cw converts the stages z = cw, cw + NCONV, ... of the sequence: the u64 residues
    // of 32 J x CW columns -> the byte rows of the Toeplitz image (row b*CW + c, 32 J bytes split
    // in two 16-B K halves).  A unit = 2 columns x 4 J (one u32 word per limb row and column):
    // CW*4 units per stage over the warp's 32 lanes, column pairs fastest so that the 16-B loads of
    // a warp cover whole 128-B rows of the stage's [J][xw] residues (no bank conflicts at xw = 16).
    const int cw = warp - 2;
    constexpr int NPAIR = CW / 2, UNITS = NPAIR * 8, UIT = (UNITS + 31) / 32;
    uint32_t zseq = 0;
    for (uint32_t seq = 0;; seq++) {
      const int item = tc_next_item(ifull, iempty, itm, seq);
      if (item < 0) break;
      const int c1lo = tc_c1_lo<CW>(A, tc_decode(g, item).cg);
      for (int si = 0; si < T::SPI; si++) {
        for (int kk = 0; kk < A.njc; kk++, zseq++) {
          if ((int)(zseq % T::NCONV) != cw) continue;
          const int st = (int)(zseq % (uint32_t)NST);
          const uint32_t ph = (zseq / (uint32_t)NST) & 1;
          const uint32_t zi = zseq % T::NZ, zph = (zseq / T::NZ) & 1;
          mbar_wait_p(&full[st], ph, (kProf && A.prof && lane == 0 && cw == 0) ? &pw[4] : nullptr);
          mbar_wait(&zempty[zi], zph ^ 1);
          const uint64_t *raw = reinterpret_cast<const uint64_t *>(smem + st * SB);
          const uint64_t *c1b = reinterpret_cast<const uint64_t *>(smem + st * SB + A.ring.c1_off) + (si & 1);
          const ulonglong2 *c1q = reinterpret_cast<const ulonglong2 *>(smem + st * SB + A.ring.c1_off);
          unsigned char *z = zring + zi * T::Z_BYTES;
#pragma unroll
          for (int ui = 0; ui < UIT; ui++) {
            const int u = lane + 32 * ui;
            if (u >= UNITS) break;
            const int cp = u % NPAIR, hg = u / NPAIR, h = hg >> 2, gq = hg & 3;
            const int c = 2 * cp, j0 = h * 16 + gq * 4;
            uint64_t x0[4], x1[4];
            if (c + 1 < c1lo && !(g.xw & 1)) {                  // both c0: one 16-B load per J
#pragma unroll
              for (int j = 0; j < 4; j++) {
                const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(raw + (j0 + j) * g.xw + c);
                x0[j] = v.x; x1[j] = v.y;
              }
            } else if (c >= c1lo) {
              // both c1, from the box [J][K][2 points]: the 16-B (point 0, point 1) pair of each
              // column, the two loads in a lane-dependent order so that a warp's loads cover all
              // 32 banks; the stage's point is si & 1
              const int k0 = c - c1lo, f = (cp & 4) ? 1 : 0;
#pragma unroll
              for (int j = 0; j < 4; j++) {
                const ulonglong2 *rw = c1q + (j0 + j) * A.c1_cols + k0;
                const ulonglong2 va = rw[f], vb = rw[1 - f];
                const ulonglong2 v0 = f ? vb : va, v1 = f ? va : vb;
                x0[j] = (si & 1) ? v0.y : v0.x;
                x1[j] = (si & 1) ? v1.y : v1.x;
              }
            } else {                                           // a c0 / c1 boundary pair (odd nK)
#pragma unroll
              for (int j = 0; j < 4; j++) {
                x0[j] = c < c1lo ? raw[(j0 + j) * g.xw + c] : c1b[((j0 + j) * A.c1_cols + (c - c1lo)) * 2];
                x1[j] = c + 1 < c1lo ? raw[(j0 + j) * g.xw + c + 1]
                                     : c1b[((j0 + j) * A.c1_cols + (c + 1 - c1lo)) * 2];
              }
            }
            conv_unit<CW, T::ZR>(z, h, c, gq, x0, x1, (cp & 4) != 0);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&zfull[zi]);                             // every lane (count 32)
        }
      }
    }
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    // warp w (4..11): TMEM lanes 32*(w&3).. (the hardware quadrant of w), columns c in half hh.
    // Recombination: L = sum_{d<5} S_d 2^(8d) < 2^64, M = sum_{d=5..8} S_d 2^(8(d-5)) < 2^56,
    // H = sum_{d=9..12} S_d 2^(8(d-9)) < 2^56 (S_d < 2^31), sum_J W X = L + M 2^40 + H 2^72,
    // reduced as Barrett(L) + Shoup(M, 2^40 mod p) + Shoup(H, 2^72 mod p), each in [0, 2p).
    constexpr int CH = T::CH;
    const int q = warp & 3, hh = (warp - T::EPI0) >> 2;
    const int et = threadIdx.x - 32 * T::EPI0;
    uint32_t tile_no = 0;
    for (uint32_t seq = 0;; seq++) {
      const int item = tc_next_item(ifull, iempty, itm, seq);
      if (item < 0) break;
      const TcItem it = tc_decode(g, item);
      const int l = (it.sq * T::SPI) / A.N;
      const PrimeConsts pc = pick(P, l);
      const int rows_valid = min(g.RT, g.nIs - g.RT * it.t);
      const bool m64 = min(g.RT, g.nIp - g.RT * it.t) <= 64;   // this item's MMA M (as the MMA warp)
      const int row = m64 ? (lane < 16 ? 16 * q + lane : 1 << 20) : 32 * q + lane;   // tile row held by this lane
      const bool active = (m64 ? 16 : 32) * q < rows_valid;   // warp-uniform: this quadrant holds outputs
      const size_t s0 = (size_t)it.sq * T::SPI;
      // full 32-B sector stores of out[I][col][s0 .. s0+3] (c1 columns: into the response)
      auto store4 = [&](int rr, int c, uint64_t v0, uint64_t v1, uint64_t v2, uint64_t v3) {
        const int col = it.cg * CW + c;
        if (A.c1_out && col >= A.c1_nK) {
          // quad order (tc_slot): slot u NT + t' + {0,2,1,3}[i] NT/4 holds natural k = k0 + i,
          // k0 = brev4(u) NT + brev(t') (nat_of) -- one 32-B sector of the response's c1
          const int sl = (int)(s0 - (size_t)l * A.N), nt = 1 << A.c1_lognt;
          const int u = sl >> A.c1_lognt, tq = (sl & (nt - 1)) >> 2;
          const int k0 = (int)(__brev((unsigned)u) >> 28) * nt + (int)(__brev((unsigned)tq) >> (32 - A.c1_lognt));
          const int64_t o = (int64_t)(g.RT * it.t + rr) * A.c1_nK + (col - A.c1_nK);
          uint64_t *dst = A.c1_out + (size_t)o * P.L * (A.c1_mn + A.N) + (size_t)P.L * A.c1_mn + (size_t)l * A.N + k0;
          v0 = v0 >= pc.two_p ? v0 - pc.two_p : v0; v0 = v0 >= pc.p ? v0 - pc.p : v0;
          v1 = v1 >= pc.two_p ? v1 - pc.two_p : v1; v1 = v1 >= pc.p ? v1 - pc.p : v1;
          v2 = v2 >= pc.two_p ? v2 - pc.two_p : v2; v2 = v2 >= pc.p ? v2 - pc.p : v2;
          v3 = v3 >= pc.two_p ? v3 - pc.two_p : v3; v3 = v3 >= pc.p ? v3 - pc.p : v3;
          st_sector(dst, v0, v1, v2, v3, A.c1_v4);
          return;
        }
        uint64_t *dst = A.out + ((size_t)(g.RT * it.t + rr) * g.nC + it.cg * CW + c) * g.LN + s0;
        if (A.accumulate) {
          const ulonglong2 o0 = reinterpret_cast<const ulonglong2 *>(dst)[0], o1 = reinterpret_cast<const ulonglong2 *>(dst)[1];
          v0 += o0.x; v1 += o0.y; v2 += o1.x; v3 += o1.y;
          v0 = v0 >= pc.p ? v0 - pc.p : v0; v1 = v1 >= pc.p ? v1 - pc.p : v1;
          v2 = v2 >= pc.p ? v2 - pc.p : v2; v3 = v3 >= pc.p ? v3 - pc.p : v3;
        }
        st_sector(dst, v0, v1, v2, v3, A.out_v4);
      };
      uint64_t acc[T::REG_EPI ? CH : 1][4];                     // REG_EPI: the item's 4 slots of this lane's outputs
#pragma unroll
      for (int si = 0; si < T::SPI; si++, tile_no++) {
        const uint32_t buf = tile_no % T::NBUF, tph = (tile_no / T::NBUF) & 1;
        mbar_wait_p(&tfull[buf], tph, (kProf && A.prof && et == 0) ? &pw[5] : nullptr);
        const long long te0 = (kProf && A.prof) ? clock64() : 0;
        tc_fence_after();
        // Fast recombination (pc.mc < 2^27, every prime of reading C4): with k_d = 2^(8d) mod p in
        // 25-bit limbs, sum_d S_d 2^(8d) = A0 + A1 2^25 (mod p), accumulated from the diagonals as
        // they are loaded:  A0 = S_0 + S_1 2^8 + S_2 2^16 + S_3 2^24 + sum_{d>=7} S_d k_d0 < 2^59,
        // A1 = S_4 2^7 + S_5 2^15 + S_6 2^23 + sum_{d>=7} S_d k_d1 < 2^60 (2^(8d) < p for d <= 6);
        // then two pseudo-Mersenne folds (2^50 = mc mod p) -- one third of the integer multiplies of
        // the general path (L + M 2^40 + H 2^72 as a 124-bit value, Shoup + Barrett), which made this
        // epilogue the bottleneck of the fat products (c3, c4).
        // General path: three column groups (d < 5 -> L, 5..8 -> M, 9..12 -> H), one at a time.
        constexpr bool fastr = FAST;
        uint64_t L[CH], M[CH], H[CH];
        if (active && fastr && CW >= 16) {
          // the 13 diagonals of 4 of the warp's columns in flight at once (one wait per half)
          const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + buf * T::N + hh * CH;
#pragma unroll
          for (int c0 = 0; c0 < CH; c0 += 4) {
            uint32_t v[13][4];
#pragma unroll
            for (int d = 0; d < 13; d++) tmem_ld_cw<4>(base + d * CW + c0, v[d]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int c = 0; c < 4; c++) {
              L[c0 + c] = (uint64_t)v[0][c] + ((uint64_t)v[1][c] << 8) + ((uint64_t)v[2][c] << 16) + ((uint64_t)v[3][c] << 24);
              M[c0 + c] = ((uint64_t)v[4][c] << 7) + ((uint64_t)v[5][c] << 15) + ((uint64_t)v[6][c] << 23);
#pragma unroll
              for (int d = 7; d < 13; d++) {
                L[c0 + c] += (uint64_t)v[d][c] * pc.ek0[d - 7];
                M[c0 + c] += (uint64_t)v[d][c] * pc.ek1[d - 7];
              }
            }
          }
        } else if (active && fastr) {
          const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + buf * T::N + hh * CH;
          uint32_t v[5][CH];
#pragma unroll
          for (int d = 0; d < 5; d++) tmem_ld_cw<CH>(base + d * CW, v[d]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int c = 0; c < CH; c++) {
            L[c] = (uint64_t)v[0][c] + ((uint64_t)v[1][c] << 8) + ((uint64_t)v[2][c] << 16) + ((uint64_t)v[3][c] << 24);
            M[c] = (uint64_t)v[4][c] << 7;
          }
#pragma unroll
          for (int d = 0; d < 4; d++) tmem_ld_cw<CH>(base + (5 + d) * CW, v[d]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int c = 0; c < CH; c++) {
            M[c] += ((uint64_t)v[0][c] << 15) + ((uint64_t)v[1][c] << 23);
            L[c] += (uint64_t)v[2][c] * pc.ek0[0] + (uint64_t)v[3][c] * pc.ek0[1];
            M[c] += (uint64_t)v[2][c] * pc.ek1[0] + (uint64_t)v[3][c] * pc.ek1[1];
          }
#pragma unroll
          for (int d = 0; d < 4; d++) tmem_ld_cw<CH>(base + (9 + d) * CW, v[d]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int c = 0; c < CH; c++) {
#pragma unroll
            for (int d = 0; d < 4; d++) {
              L[c] += (uint64_t)v[d][c] * pc.ek0[2 + d];
              M[c] += (uint64_t)v[d][c] * pc.ek1[2 + d];
            }
          }
        } else if (active) {
          const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + buf * T::N + hh * CH;
          uint32_t v[5][CH];
#pragma unroll
          for (int d = 0; d < 5; d++) tmem_ld_cw<CH>(base + d * CW, v[d]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int c = 0; c < CH; c++) {
            L[c] = v[0][c];
#pragma unroll
            for (int d = 1; d < 4; d++) L[c] += (uint64_t)v[d][c] << (8 * d);
            L[c] += (uint64_t)v[4][c] << 32;
          }
#pragma unroll
          for (int d = 0; d < 4; d++) tmem_ld_cw<CH>(base + (5 + d) * CW, v[d]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int c = 0; c < CH; c++) {
            M[c] = v[0][c];
#pragma unroll
            for (int d = 1; d < 4; d++) M[c] += (uint64_t)v[d][c] << (8 * d);
          }
#pragma unroll
          for (int d = 0; d < 4; d++) tmem_ld_cw<CH>(base + (9 + d) * CW, v[d]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int c = 0; c < CH; c++) {
            H[c] = v[0][c];
#pragma unroll
            for (int d = 1; d < 4; d++) H[c] += (uint64_t)v[d][c] << (8 * d);
          }
        }
        if constexpr (!T::ZMMA) {   // re-zero the columns no a = 0 MMA initialises (see the setup) -- only columns of this
            // warp's own half (c / CH == hh): the other warp of the quadrant may still be reading its half
          const uint32_t zb = tmem + ((uint32_t)(32 * q) << 16) + buf * T::N + hh * CH;
#pragma unroll
          for (int d = T::NM / CW; d < T::N / CW; d++) tmem_zero_cw<CH>(zb + d * CW);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        const long long te1 = (kProf && A.prof) ? clock64() : 0;
        if (kProf && A.prof && et == 0) pw[2] += (unsigned long long)(te1 - te0);   // TMEM drain + accumulate
        if (active) {
#pragma unroll
          for (int c = 0; c < CH; c++) {
            uint64_t r;
            if (fastr) {
              // T = A0 + A1 2^25 < 2^86 = th 2^50 + tl;  T = tl + th mc (mod p) < 2^50 + 2^63;
              // fold once more: < 2^50 + 2^41 < 2p
              const uint64_t lo = L[c] + (M[c] << 25);
              const uint64_t hi = (M[c] >> 39) + (lo < L[c] ? 1 : 0);
              const uint64_t th = (lo >> 50) | (hi << 14);
              uint64_t t = (lo & ((1ull << 50) - 1)) + th * pc.mc;
              r = (t & ((1ull << 50) - 1)) + (t >> 50) * pc.mc;          // [0, 2p)
            } else {
            // V = L + M 2^40 + H 2^72 < 2^124 exactly; V mod p = Shoup(V_hi, 2^64 mod p) + (V_lo mod p)
            const hl_u128 V = (hl_u128)L[c] + ((hl_u128)M[c] << 40) + ((hl_u128)H[c] << 72);
            const uint64_t vh = (uint64_t)(V >> 64), vl = (uint64_t)V;
            r = shoup_mul(vh, pc.r64, pc.r64_sh, pc.p);                    // [0, 2p)
            if (pc.mc) {
              // pseudo-Mersenne fold, 2^50 = mc (mod p): vl = a 2^50 + b -> b + a mc < 2^50 + 2^46 < 2p
              r += (vl & ((1ull << 50) - 1)) + (vl >> 50) * pc.mc;
            } else {
              r += vl - __umul64hi(vl, pc.mu) * pc.p;                      // [0, 2p)
            }                                                              // r in [0, 4p) < 2^52
            }
            if (!A.lazy_out) {
              r = r >= pc.two_p ? r - pc.two_p : r;
              r = r >= pc.p ? r - pc.p : r;
            }
            if constexpr (T::REG_EPI) acc[c][si] = r;
            else if (row < rows_valid) stg[row * T::STG_STRIDE + (hh * CH + c) * T::SPI + si] = r;
          }
        }
        if constexpr (T::REG_EPI) {
          if (si == 3 && active && row < rows_valid) {      // full 32-B sectors (no partial-sector writes)
#pragma unroll
            for (int c = 0; c < CH; c++) store4(row, hh * CH + c, acc[c][0], acc[c][1], acc[c][2], acc[c][3]);
          }
        }
        if (kProf && A.prof && et == 0) pw[3] += (unsigned long long)(clock64() - te1);   // folds + stores
      }
      if constexpr (!T::REG_EPI) {
        asm volatile("bar.sync 2, 256;" ::: "memory");      // 4 slots staged
        for (int e = et; e < rows_valid * CW; e += 256) {
          const int rr = e / CW, c = e % CW;
          const uint64_t *sv = stg + rr * T::STG_STRIDE + c * T::SPI;
          store4(rr, c, sv[0], sv[1], sv[2], sv[3]);
        }
        asm volatile("bar.sync 2, 256;" ::: "memory");
      }
    }
  }

  // ---- teardown
  if (kProf && A.prof) {
    const unsigned long long tot = (unsigned long long)(clock64() - t_start);
    if (threadIdx.x == 0) { atomicAdd(&A.prof[0], pw[0]); atomicAdd(&A.prof[7], tot); }
    if (threadIdx.x == 32) { atomicAdd(&A.prof[1], pw[1]); atomicAdd(&A.prof[2], pw[2]); atomicAdd(&A.prof[3], pw[3]); atomicAdd(&A.prof[6], pw[6]); }
    if (threadIdx.x == 64) atomicAdd(&A.prof[4], pw[4]);
    if (threadIdx.x == 32 * T::EPI0) { atomicAdd(&A.prof[5], pw[5]); atomicAdd(&A.prof[8], pw[2]); atomicAdd(&A.prof[9], pw[3]); }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(T::TCOLS));
}
