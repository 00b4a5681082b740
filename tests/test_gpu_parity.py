"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit for bit (-m gpu).

Every expected value comes from oracle/ (or from brute-force numpy matmul for the
reconstruction property); inputs come from synth/ (seeded) or the oracle's encrypt.
Integer work, so the bar is bit-exact equality everywhere.
"""
import numpy as np
import pytest

import synth
from oracle import ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hl():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2305_18396_b200 as hl
    hl.load_library()
    return hl


@pytest.fixture(scope="module")
def ctx4096(hl):
    return hl.Context(4096, 2, 37, device=0)


@pytest.fixture(scope="module")
def ctx8192(hl):
    return hl.Context(8192, 3, 37, device=0)


def _P(ctx):
    return ref.bfv_params(ctx.N, ctx.L, ctx.t_bits)


def _sync():
    import torch
    torch.cuda.synchronize()


# ------------------------------------------------------------------------- NTT kernels
@pytest.mark.parametrize("which", ["4096", "8192"])
def test_ntt_roundtrip_identity(hl, ctx4096, ctx8192, which):
    ctx = ctx4096 if which == "4096" else ctx8192
    P = _P(ctx)
    x = synth.uniform_below(1, (7, ctx.L, ctx.N), P.primes)
    # extreme residues: 0 and p-1 everywhere in one polynomial
    x[0, :, :] = 0
    for l, p in enumerate(P.primes):
        x[1, l, :] = p - 1
    d = hl.to_device(x)
    ctx.ntt_roundtrip(d)
    _sync()
    assert np.array_equal(hl.to_host(d).reshape(x.shape), x)


@pytest.mark.parametrize("which", ["4096", "8192"])
def test_poly_mul_vs_oracle_schoolbook(hl, ctx4096, ctx8192, which):
    ctx = ctx4096 if which == "4096" else ctx8192
    P = _P(ctx)
    a = synth.uniform_below(2, (3, ctx.L, ctx.N), P.primes)
    b = synth.uniform_below(3, (3, ctx.L, ctx.N), P.primes)
    # special case x^(N-1) * x = -1 in polynomial 0
    a[0] = 0; a[0, :, ctx.N - 1] = 1
    b[0] = 0; b[0, :, 1] = 1
    out = hl.to_host(ctx.poly_mul(hl.to_device(a), hl.to_device(b))).reshape(a.shape)
    for i in range(3):
        for l, p in enumerate(P.primes):
            assert np.array_equal(out[i, l], ref.negacyclic_mul(ctx.N, p, a[i, l], b[i, l])), (i, l)
    assert all(out[0, l, 0] == p - 1 for l, p in enumerate(P.primes)) and not out[0, :, 1:].any()


# ------------------------------------------------------------------------- he_matmul / mask
CASES = [
    # (N, shape (Nb, R, Ma), tile)                          what it covers
    (4096, (8, 64, 64), (16, 32, 8)),      # config c0
    (4096, (40, 24, 40), (16, 8, 32)),     # ragged in every dimension, several tiles
    (4096, (64, 48, 100), (4, 8, 16)),     # nC = 8, ragged I tail (nI = 25)
    (4096, (3, 5, 7), (1, 1, 1)),          # degenerate 1x1x1 tile, nC = 6
    (4096, (6, 10, 7), (1, 4, 2)),         # m n = 2: the fused MAC's c1 sectors in the response are only
                                           # 16-B aligned (two 16-B stores instead of one 256-bit store)
    (8192, (32, 48, 40), (32, 16, 16)),    # c4 parameters (N=8192, L=3) at small size
    (4096, (256, 40, 50), (16, 8, 32)),    # nC = 16: the MAC's 16-column groups (CW = 16)
    (4096, (520, 24, 40), (16, 8, 32)),    # nC = 34 -> CW = 2, 17 column groups, ragged K tail
    (8192, (288, 48, 40), (32, 16, 16)),   # c4 tile, nC = 36 (CW = 4, 9 groups), N=8192 L=3
    (8192, (256, 48, 40), (32, 16, 16)),   # c4 tile, nK = 16: whole 16-column groups at N = 8192 (the
                                           # single-column forward kernel, c1 by k_c1_tx16)
    (4096, (512, 24, 40), (16, 8, 32)),    # nK = 16: pure c0 / c1 column groups (CW = 16, 2 groups;
                                           # the fused MAC reads c1 by tensor-map TMA, group 1 has no X)
]


def _case_inputs(ctx, shape, tile, seed):
    P = _P(ctx)
    Nb, R, Ma = shape
    nI, nJ, nK = ref.tile_counts(tile, Ma, R, Nb)
    ct_in = synth.uniform_below(seed, (nJ, nK, 2, ctx.L, ctx.N), P.primes)
    W = synth.weights(seed + 1, R, Ma)
    return P, ct_in, W


@pytest.mark.parametrize("N,shape,tile", CASES)
def test_he_matmul_bit_exact(hl, ctx4096, ctx8192, N, shape, tile):
    ctx = ctx4096 if N == 4096 else ctx8192
    Nb, R, Ma = shape
    P, ct_in, W = _case_inputs(ctx, shape, tile, 200 + N + Ma)
    wc = ctx.encode_weights(tile, hl.to_device(W))
    out = ctx.he_matmul(tile, wc, Ma, R, Nb, hl.to_device(ct_in))
    got = hl.to_host(out).reshape(-1, 2, ctx.L, ctx.N)
    exp = ref.he_matmul(P, tile, W, ct_in, Nb).reshape(-1, 2, ctx.L, ctx.N)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("N,shape,tile", CASES)
@pytest.mark.parametrize("compress", [True, False])
def test_mask_and_share_bit_exact(hl, ctx4096, ctx8192, N, shape, tile, compress):
    ctx = ctx4096 if N == 4096 else ctx8192
    Nb, R, Ma = shape
    P = _P(ctx)
    nI, _, nK = ref.tile_counts(tile, Ma, R, Nb)
    ct_out = synth.uniform_below(300 + N, (nI, nK, 2, ctx.L, ctx.N), P.primes)
    masked, share = ctx.mask_and_share(tile, Ma, Nb, hl.to_device(ct_out), seed=77, compress=compress)
    em, es = ref.mask_and_share(P, tile, ct_out, Ma, Nb, 77, compress)
    assert np.array_equal(hl.to_host(masked).reshape(em.shape), em)
    assert np.array_equal(hl.to_host(share).reshape(es.shape), es)


@pytest.mark.parametrize("N,shape,tile", CASES)
def test_fused_he_matmul_share_bit_exact(hl, ctx4096, ctx8192, N, shape, tile):
    ctx = ctx4096 if N == 4096 else ctx8192
    Nb, R, Ma = shape
    P, ct_in, W = _case_inputs(ctx, shape, tile, 400 + N + Ma)
    wc = ctx.encode_weights(tile, hl.to_device(W))
    masked, share = ctx.he_matmul_share(tile, wc, Ma, R, Nb, hl.to_device(ct_in), seed=91)
    exp_ct = ref.he_matmul(P, tile, W, ct_in, Nb)
    em, es = ref.mask_and_share(P, tile, exp_ct, Ma, Nb, 91, True)
    assert np.array_equal(hl.to_host(masked).reshape(em.shape), em)
    assert np.array_equal(hl.to_host(share).reshape(es.shape), es)


def test_sharded_outputs_equal_slices(hl, ctx4096):
    """I-tile shards [i0, i1) produce exactly the slice of the unsharded result (mask streams
    are indexed by the global tile), so any GPU count gives identical outputs."""
    ctx = ctx4096
    tile, (Nb, R, Ma) = (16, 8, 32), (64, 32, 160)
    P, ct_in, W = _case_inputs(ctx, (Nb, R, Ma), tile, 501)
    dW, dct = hl.to_device(W), hl.to_device(ct_in)
    full_m, full_s = ctx.he_matmul_share(tile, ctx.encode_weights(tile, dW), Ma, R, Nb, dct, seed=5)
    full_m = hl.to_host(full_m).reshape(10, 2, -1)
    full_s = hl.to_host(full_s).reshape(Nb, Ma)
    for i0, i1 in [(0, 3), (3, 4), (4, 10)]:
        wc = ctx.encode_weights(tile, dW, i0, i1)
        m, s = ctx.he_matmul_share(tile, wc, Ma, R, Nb, dct, seed=5, i_begin=i0, i_end=i1)
        assert np.array_equal(hl.to_host(m).reshape(i1 - i0, 2, -1), full_m[i0:i1])
        s = hl.to_host(s).reshape(Nb, Ma)
        cols = slice(i0 * 16, i1 * 16)
        assert np.array_equal(s[:, cols], full_s[:, cols])


# ------------------------------------------------------------------------- end to end (Alg. 1)
@pytest.mark.parametrize("N,shape,tile", [
    (4096, (8, 64, 64), (16, 32, 8)),
    (4096, (37, 50, 45), (8, 8, 32)),
    (8192, (16, 40, 24), (32, 16, 16)),
])
def test_end_to_end_reconstructs_XW(hl, ctx4096, ctx8192, N, shape, tile):
    """Oracle client (keygen, encrypt, decrypt) around the GPU server: shares sum to X.W mod 2^37,
    and the GPU's response equals the oracle server's response."""
    ctx = ctx4096 if N == 4096 else ctx8192
    P = _P(ctx)
    Nb, R, Ma = shape
    X, W = synth.activations(601, Nb, R), synth.weights(602, R, Ma)
    sk = ref.keygen(P, 603)
    ct_in = ref.encrypt(P, tile, sk, X, 604)
    wc = ctx.encode_weights(tile, hl.to_device(W))
    masked, share_s = ctx.he_matmul_share(tile, wc, Ma, R, Nb, hl.to_device(ct_in), seed=605)
    masked = hl.to_host(masked).reshape(-1, P.L * (tile[0] * tile[2] + P.N))
    share_s = hl.to_host(share_s).reshape(Nb, Ma)
    share_c = ref.decrypt_share(P, tile, sk, masked, Ma, Nb, True)
    got = (share_c + share_s) & np.uint64((1 << 37) - 1)
    assert np.array_equal(got, ref.matmul_mod_t(X, W))
    em, es = ref.mask_and_share(P, tile, ref.he_matmul(P, tile, W, ct_in, Nb), Ma, Nb, 605, True)
    assert np.array_equal(masked.reshape(em.shape), em) and np.array_equal(share_s, es)


def test_bert_tiny_block_c1(hl, ctx4096):
    """Config c1 (BERT-Tiny block, the four matmuls) end to end against the oracle server."""
    ctx = ctx4096
    cfg = synth.CONFIGS["c1"]
    P = _P(ctx)
    for mi, mm in enumerate(cfg.matmuls):
        X = synth.activations(synth.seed_for(0, mi, "x"), mm.Nb, mm.R)
        W = synth.weights(synth.seed_for(0, mi, "w"), mm.R, mm.Ma)
        nI, nJ, nK = ref.tile_counts(cfg.tile, mm.Ma, mm.R, mm.Nb)
        ct_in = synth.uniform_below(synth.seed_for(0, mi, "enc"), (nJ, nK, 2, P.L, P.N), P.primes)
        wc = ctx.encode_weights(cfg.tile, hl.to_device(W))
        seed = synth.seed_for(0, mi, "mask")
        m, s = ctx.he_matmul_share(cfg.tile, wc, mm.Ma, mm.R, mm.Nb, hl.to_device(ct_in), seed=seed)
        em, es = ref.mask_and_share(P, cfg.tile, ref.he_matmul(P, cfg.tile, W, ct_in, mm.Nb), mm.Ma, mm.Nb, seed)
        assert np.array_equal(hl.to_host(m).reshape(em.shape), em), mm.name
        assert np.array_equal(hl.to_host(s).reshape(es.shape), es), mm.name


def _block_inputs(ctx, cfg, block=0, tiles=None):
    P = _P(ctx)
    out = []
    for mi, mm in enumerate(cfg.matmuls):
        tile = tiles[mi] if tiles else cfg.tile
        W = synth.weights(synth.seed_for(block, mi, "w"), mm.R, mm.Ma)
        nI, nJ, nK = ref.tile_counts(tile, mm.Ma, mm.R, mm.Nb)
        ct_in = synth.uniform_below(synth.seed_for(block, mi, "enc"), (nJ, nK, 2, P.L, P.N), P.primes)
        out.append((mm, W, ct_in, synth.seed_for(block, mi, "mask")))
    return out


def test_linear_batch_c1_vs_oracle(hl, ctx4096):
    """hl_he_linear_batch (the bench's call: the four products pipelined over two streams) on
    config c1, bit-exact against the oracle server for every product."""
    ctx = ctx4096
    cfg = synth.CONFIGS["c1"]
    P = _P(ctx)
    ins = _block_inputs(ctx, cfg)
    entries = [dict(wcache=ctx.encode_weights(cfg.tile, hl.to_device(W)), Ma=mm.Ma, R=mm.R, Nb=mm.Nb,
                    ct_in=hl.to_device(ct_in), seed=seed) for mm, W, ct_in, seed in ins]
    exp = [ref.mask_and_share(P, cfg.tile, ref.he_matmul(P, cfg.tile, W, ct_in, mm.Nb), mm.Ma, mm.Nb, seed)
           for mm, W, ct_in, seed in ins]
    for rep in range(4):                  # repeated: the two streams race if any ordering is missing
        outs = ctx.he_linear_batch(cfg.tile, entries)
        _sync()
        for (mm, *_), (m, sh), (em, es) in zip(ins, outs, exp):
            assert np.array_equal(hl.to_host(m).reshape(em.shape), em), (rep, mm.name)
            assert np.array_equal(hl.to_host(sh).reshape(es.shape), es), (rep, mm.name)


def test_linear_batch_mixed_tiles_vs_oracle(hl, ctx4096):
    """hl_he_linear_batch with a different tile per product (hl_linear_desc.tile, as bench.py runs
    c2 with the planner's tiles) on config c1's shapes, bit-exact against the oracle."""
    ctx = ctx4096
    cfg = synth.CONFIGS["c1"]
    P = _P(ctx)
    tiles = [(16, 8, 32), (8, 8, 64), (4, 32, 32), (32, 4, 32)]
    ins = _block_inputs(ctx, cfg, tiles=tiles)
    entries = [dict(wcache=ctx.encode_weights(t, hl.to_device(W)), Ma=mm.Ma, R=mm.R, Nb=mm.Nb, tile=t,
                    ct_in=hl.to_device(ct_in), seed=seed) for t, (mm, W, ct_in, seed) in zip(tiles, ins)]
    exp = [ref.mask_and_share(P, t, ref.he_matmul(P, t, W, ct_in, mm.Nb), mm.Ma, mm.Nb, seed)
           for t, (mm, W, ct_in, seed) in zip(tiles, ins)]
    for rep in range(3):
        outs = ctx.he_linear_batch((1, 1, 1), entries)   # the call's tile is overridden by every entry
        _sync()
        for (mm, *_), (m, sh), (em, es) in zip(ins, outs, exp):
            assert np.array_equal(hl.to_host(m).reshape(em.shape), em), (rep, mm.name)
            assert np.array_equal(hl.to_host(sh).reshape(es.shape), es), (rep, mm.name)


def test_linear_batch_pipelined_with_fat_product_vs_oracle(hl, ctx4096):
    """The pipelined schedule (some entry has nK < 8, so every forward NTT is issued up front and
    shares SMs with the MACs) with a fat CW = 16 entry among thin ones: the c1 transposition
    (k_c1_tx16), the CW = 16 MAC and the CW = 4/8 MACs with the c1 tensor-map path interleaved
    over the context's streams; bit-exact against the oracle, three times over."""
    ctx = ctx4096
    P = _P(ctx)
    ins = []
    for k, (Nb, R, Ma, tile) in enumerate([(128, 40, 72, (8, 8, 32)), (512, 24, 40, (16, 8, 32)),
                                           (64, 48, 40, (4, 16, 32))]):
        W = synth.weights(1400 + k, R, Ma)
        nI, nJ, nK = ref.tile_counts(tile, Ma, R, Nb)
        ct_in = synth.uniform_below(1410 + k, (nJ, nK, 2, P.L, P.N), P.primes)
        ins.append((Nb, R, Ma, tile, W, ct_in, 1420 + k))
    assert min(ref.tile_counts(t, Ma, R, Nb)[2] for Nb, R, Ma, t, *_ in ins) < 8
    entries = [dict(wcache=ctx.encode_weights(t, hl.to_device(W)), Ma=Ma, R=R, Nb=Nb, tile=t,
                    ct_in=hl.to_device(ct), seed=sd) for Nb, R, Ma, t, W, ct, sd in ins]
    exp = [ref.mask_and_share(P, t, ref.he_matmul(P, t, W, ct, Nb), Ma, Nb, sd) for Nb, R, Ma, t, W, ct, sd in ins]
    for rep in range(3):
        outs = ctx.he_linear_batch((1, 1, 1), entries)
        _sync()
        for (em, es), (m, sh) in zip(exp, outs):
            assert np.array_equal(hl.to_host(m).reshape(em.shape), em), rep
            assert np.array_equal(hl.to_host(sh).reshape(es.shape), es), rep


def test_linear_batch_serial_policy_vs_oracle(hl, ctx4096):
    """hl_he_linear_batch with nK >= 8 for every entry (c3/c4-sized token counts) takes the
    adaptive serial policy (every MAC alone; the forward NTT of entry k+1 beside the inverse NTT +
    mask of entry k): bit-exact against the oracle, twice over (the cross-stream ordering is
    re-exercised), including a CW = 16 entry with whole c1 column groups (k_c1_tx16)."""
    ctx = ctx4096
    P = _P(ctx)
    ins = []
    for k, (Nb, R, Ma, tile) in enumerate([(256, 48, 40, (16, 8, 16)), (512, 24, 40, (16, 8, 32)),
                                           (160, 40, 72, (8, 8, 16))]):
        nI, nJ, nK = ref.tile_counts(tile, Ma, R, Nb)
        assert nK >= 8
        W = synth.weights(1200 + k, R, Ma)
        ct_in = synth.uniform_below(1210 + k, (nJ, nK, 2, P.L, P.N), P.primes)
        ins.append((Nb, R, Ma, tile, W, ct_in, 1220 + k))
    entries = [dict(wcache=ctx.encode_weights(t, hl.to_device(W)), Ma=Ma, R=R, Nb=Nb, tile=t,
                    ct_in=hl.to_device(ct), seed=sd) for Nb, R, Ma, t, W, ct, sd in ins]
    exp = [ref.mask_and_share(P, t, ref.he_matmul(P, t, W, ct, Nb), Ma, Nb, sd) for Nb, R, Ma, t, W, ct, sd in ins]
    for _ in range(2):
        outs = ctx.he_linear_batch((1, 1, 1), entries)
        _sync()
        for (em, es), (m, sh) in zip(exp, outs):
            assert np.array_equal(hl.to_host(m).reshape(em.shape), em)
            assert np.array_equal(hl.to_host(sh).reshape(es.shape), es)


def _sample_tiles(nI, nK, mac_rows):
    """Output tiles (I, K) covering the MAC's row-tile boundaries (first / last row of every MAC
    I tile of `mac_rows` rows), both ends of K and an interior point."""
    Is = {0, nI - 1, nI // 2, (17 * nI) // 29}
    for t0 in range(0, nI, mac_rows):
        Is |= {t0, min(nI, t0 + mac_rows) - 1}
    out = []
    for n, I in enumerate(sorted(Is)):
        out.append((I, n % nK))
    out += [(0, nK - 1), (nI - 1, 0)]
    return sorted(set(out))


def test_linear_batch_c2_vs_oracle_sampled(hl, ctx4096):
    """The bench's call on the bench's workload: the four c2 products (QKV, O, FF1, FF2) at the
    planner's tiles through hl_he_linear_batch in the bench's submission order, with uniform
    full-range ciphertext residues.  For every product, sampled output ciphertexts (compressed
    response + server share) bit-exact against the oracle's scalar-NTT path + mask, at both sides of
    every MAC row tile (QKV: nI = 144 in two 72-row M = 128 tiles; FF1: 192 = 2 x 96; O, FF2: one
    48/192-row tile), every K; repeated twice to catch cross-stream races."""
    ctx = ctx4096
    cfg = synth.CONFIGS["c2"]
    P = _P(ctx)
    tiles = [tuple(ctx.plan_tile(mm.Ma, mm.R, mm.Nb)) for mm in cfg.matmuls]
    assert tiles == [cfg.tile_of(mi) for mi in range(len(cfg.matmuls))]
    ins = _block_inputs(ctx, cfg, tiles=tiles)
    entries = [dict(wcache=ctx.encode_weights(t, hl.to_device(W)), Ma=mm.Ma, R=mm.R, Nb=mm.Nb, tile=t,
                    ct_in=hl.to_device(ct_in), seed=seed) for t, (mm, W, ct_in, seed) in zip(tiles, ins)]
    order = list(cfg.batch_order)
    exp = []
    for t, (mm, W, ct_in, seed) in zip(tiles, ins):
        nI, nJ, nK = ref.tile_counts(t, mm.Ma, mm.R, mm.Nb)
        nIp = (nI + 15) // 16 * 16
        rows = (nIp + (nIp + 127) // 128 - 1) // ((nIp + 127) // 128)       # balanced MAC row tiles
        smp = _sample_tiles(nI, nK, (rows + 7) // 8 * 8)
        ect = ref.he_matmul_ntt_tiles(P, t, W, ct_in, mm.Nb, smp)
        em, kept = ref.mask_tiles(P, t, ect, nK, smp, seed, True)
        exp.append((smp, em, kept, nI, nK))
    for rep in range(2):
        outs = ctx.he_linear_batch(cfg.tile, [entries[i] for i in order])
        _sync()
        for k, i in enumerate(order):
            (mm, *_), t, (smp, em, kept, nI, nK) = ins[i], tiles[i], exp[i]
            m_, r_, n_ = t
            masked = hl.to_host(outs[k][0]).reshape(nI, nK, -1)
            share = hl.to_host(outs[k][1]).reshape(mm.Nb, mm.Ma)
            for o, (I, K) in enumerate(smp):
                assert np.array_equal(masked[I, K], em[o]), (rep, mm.name, I, K)
                for kk in range(n_):
                    for ii in range(m_):
                        if K * n_ + kk < mm.Nb and I * m_ + ii < mm.Ma:
                            assert share[K * n_ + kk, I * m_ + ii] == kept[o, kk * m_ + ii], (rep, mm.name, I, K)


def test_linear_batch_c2_equals_single_calls(hl, ctx4096):
    """Config c2 at full size in the bench's launch configuration (batch of the four products, each
    with its planned tile): bit-identical to four he_matmul_share calls, repeated twice to catch
    cross-stream races (the batch itself is checked against the oracle by
    test_linear_batch_c2_vs_oracle_sampled)."""
    ctx = ctx4096
    cfg = synth.CONFIGS["c2"]
    tiles = [cfg.tile_of(mi) for mi in range(len(cfg.matmuls))]
    ins = _block_inputs(ctx, cfg, tiles=tiles)
    entries = [dict(wcache=ctx.encode_weights(t, hl.to_device(W)), Ma=mm.Ma, R=mm.R, Nb=mm.Nb, tile=t,
                    ct_in=hl.to_device(ct_in), seed=seed) for t, (mm, W, ct_in, seed) in zip(tiles, ins)]
    single = []
    for t, e in zip(tiles, entries):
        m, sh = ctx.he_matmul_share(t, e["wcache"], e["Ma"], e["R"], e["Nb"], e["ct_in"], seed=e["seed"])
        single.append((hl.to_host(m), hl.to_host(sh)))
    for _ in range(2):
        outs = ctx.he_linear_batch(cfg.tile, entries)
        _sync()
        for (mm, *_), (m, sh), (em, es) in zip(ins, outs, single):
            assert np.array_equal(hl.to_host(m), em), mm.name
            assert np.array_equal(hl.to_host(sh), es), mm.name


@pytest.mark.parametrize("N", [4096, 8192])
def test_expand_seeded_vs_oracle_encrypt(hl, ctx4096, ctx8192, N):
    """Seeded upload: c1 regenerated on the device from the PUBLIC seed (reading C28: the oracle's
    public_seed of the encryption seed) equals the oracle client's c1 = a bit for bit (both PRF
    streams, reading C10); c0 halves are left untouched."""
    import torch
    ctx = ctx4096 if N == 4096 else ctx8192
    P = _P(ctx)
    tile = (16, 8, 32) if N == 4096 else (32, 16, 16)
    Nb, R, seed = 40, 72, 4242 + N
    X = synth.activations(seed, Nb, R)
    sk = ref.keygen(P, seed + 1)
    ct = ref.encrypt(P, tile, sk, X, seed + 2)
    up = ct.copy()
    up[:, :, 1] = 0x5a5a5a5a                       # garbage where c1 will be regenerated
    dev = hl.to_device(up)
    assert hl.public_seed(seed + 2) == ref.public_seed(seed + 2)
    ctx.expand_seeded(tile, R, Nb, ref.public_seed(seed + 2), dev)
    _sync()
    assert np.array_equal(hl.to_host(dev).reshape(ct.shape), ct)


@pytest.mark.parametrize("packed", [False, True])
def test_linear_batch_host_seeded_c1_vs_oracle(hl, ctx4096, packed):
    """hl_he_linear_batch_host (bench.py's e2e call): only the c0 halves + the PUBLIC seed (C28) go
    host->device, results come back to pinned host buffers; every product's compressed response
    and share bit-exact against the oracle client + server, repeated to catch stream races.
    packed: c0 halves up and responses down in the 50-bit wire format (hl_pack50)."""
    import torch
    ctx = ctx4096
    cfg = synth.CONFIGS["c1"]
    P = _P(ctx)
    entries, exp = [], []
    for mi, mm in enumerate(cfg.matmuls):
        X = synth.activations(synth.seed_for(0, mi, "x"), mm.Nb, mm.R)
        W = synth.weights(synth.seed_for(0, mi, "w"), mm.R, mm.Ma)
        sk = ref.keygen(P, synth.seed_for(0, mi, "key"))
        es = synth.seed_for(0, mi, "enc")
        ct = ref.encrypt(P, cfg.tile, sk, X, es)
        seed = synth.seed_for(0, mi, "mask")
        lay = ctx.layout(cfg.tile, mm.Ma, mm.R, mm.Nb)
        c0 = hl.Context.c0_halves(ct)
        c0 = hl.Context.pack50(c0) if packed else c0
        c0 = torch.from_numpy(c0.view(np.int64).reshape(-1)).pin_memory()
        mw = hl.Context.pack50(np.zeros(lay.ct_masked_words, np.uint64)).size if packed else lay.ct_masked_words
        entries.append(dict(wcache=ctx.encode_weights(cfg.tile, hl.to_device(W)), Ma=mm.Ma, R=mm.R, Nb=mm.Nb,
                            ct_in=torch.full((lay.ct_in_words,), 7, dtype=torch.int64, device="cuda"),
                            seed=seed, c0_host=c0, a_seed=ref.public_seed(es), packed=packed,
                            masked_host=torch.zeros(mw, dtype=torch.int64).pin_memory(),
                            share_host=torch.zeros(lay.share_words, dtype=torch.int64).pin_memory()))
        exp.append(ref.mask_and_share(P, cfg.tile, ref.he_matmul(P, cfg.tile, W, ct, mm.Nb), mm.Ma, mm.Nb, seed))
    for rep in range(3):
        for e in entries:
            e["masked_host"].zero_()
            e["share_host"].zero_()
        ctx.he_linear_batch_host(cfg.tile, entries)
        _sync()
        for mm, e, (em, es_) in zip(cfg.matmuls, entries, exp):
            got = e["masked_host"].numpy().view(np.uint64)
            got = hl.Context.unpack50(got, em.size) if packed else got
            assert np.array_equal(got.reshape(em.shape), em), (rep, mm.name)
            assert np.array_equal(e["share_host"].numpy().view(np.uint64).reshape(es_.shape), es_), (rep, mm.name)


@pytest.mark.parametrize("mi,tile", [
    (3, (16, 8, 32)),     # FF2 (R = 3072, the longest J reduction) at the default tile
    (3, (8, 16, 32)),     # FF2, r = 16, nI = 96, nJ = 192
    (3, (4, 32, 32)),     # FF2 at the planner's tile (bench): r = 32, c0 inverse pruned to 15 mod 16, nI = 192
    (1, (8, 8, 64)),      # O at the planner's tile (bench): nK = 2, 4 MAC columns (CW = 4)
])
def test_bert_base_full_size_sampled(hl, ctx4096, mi, tile):
    """Config c2 at full size in the bench's launch configuration (fused call): sampled output
    tiles bit-exact against the oracle (its own scalar NTT), and for the whole matmul the
    reconstruction property (library decrypt + brute-force X.W mod 2^37)."""
    ctx = ctx4096
    cfg = synth.CONFIGS["c2"]
    P = _P(ctx)
    mm = cfg.matmuls[mi]
    X = synth.activations(synth.seed_for(0, mi, "x"), mm.Nb, mm.R)
    W = synth.weights(synth.seed_for(0, mi, "w"), mm.R, mm.Ma)
    sk = ctx.keygen(synth.seed_for(0, mi, "key"))
    ct_in = ctx.encrypt(sk, tile, X, synth.seed_for(0, mi, "enc"))
    assert np.array_equal(ct_in[:1, :1], ref.encrypt(P, tile, sk, X[:tile[2], :tile[1]],
                                                     synth.seed_for(0, mi, "enc")))
    wc = ctx.encode_weights(tile, hl.to_device(W))
    seed = synth.seed_for(0, mi, "mask")
    masked, share = ctx.he_matmul_share(tile, wc, mm.Ma, mm.R, mm.Nb, hl.to_device(ct_in), seed=seed)
    nI, nJ, nK = ref.tile_counts(tile, mm.Ma, mm.R, mm.Nb)
    masked = hl.to_host(masked).reshape(nI, nK, -1)
    share = hl.to_host(share).reshape(mm.Nb, mm.Ma)
    tiles = [(0, 0), (nI - 1, nK - 1), (17 % nI, 2 % nK)]
    exp_ct = ref.he_matmul_ntt_tiles(P, tile, W, ct_in, mm.Nb, tiles)
    em, kept = ref.mask_tiles(P, tile, exp_ct, nK, tiles, seed, True)
    for o, (I, K) in enumerate(tiles):
        assert np.array_equal(masked[I, K], em[o]), (I, K)
    share_c = ctx.decrypt_share(sk, tile, masked, mm.Ma, mm.Nb, True)
    got = (share_c + share) & np.uint64((1 << 37) - 1)
    assert np.array_equal(got, ref.matmul_mod_t(X, W))


@pytest.mark.parametrize("N,shape,tile,shard", [
    (4096, (768, 768), (16, 8, 32), (0, -1)),        # c2 O/QKV-like, no padding
    (4096, (40, 50), (16, 8, 32), (0, -1)),          # ragged: J padded to 32, rows to 16
    (4096, (64, 160), (16, 8, 32), (3, 9)),          # I-tile shard
    (8192, (64, 128), (8, 8, 128), (0, -1)),         # row f2 shape, N=8192 L=3
])
def test_encode_two_pass_equals_one_pass(hl, ctx4096, ctx8192, N, shape, tile, shard):
    """hl_encode_weights_scratch (u64 scratch + byte-plane pass, the binding's encode) writes the
    same tensor-core weight cache, byte for byte, as the one-pass hl_encode_weights."""
    import ctypes
    ctx = ctx4096 if N == 4096 else ctx8192
    R, Ma = shape
    W = hl.to_device(synth.weights(777 + R, R, Ma))
    i0, i1 = shard
    lay = ctx.layout(tile, Ma, R, 1, i0, i1)
    one = hl._dev_empty(lay.wcache_bytes // 8, W.device)
    one.fill_(0x5A)
    rc = hl._lib.hl_encode_weights(ctx._h, hl._tile(tile), hl._dptr(W), R, Ma, i0, i1, hl._dptr(one), None)
    assert rc == 0, hl._lib.hl_last_error()
    two = ctx.encode_weights(tile, W, i0, i1)
    _sync()
    assert hl.to_host(one).tobytes() == hl.to_host(two).tobytes()


@pytest.mark.parametrize("mc_bits", [30, 45])
def test_mac_general_epilogue_non_pseudo_mersenne_primes(hl, mc_bits):
    """Primes far below 2^50 (2^50 - p >= 2^27): the tensor-core MAC's general epilogue
    (124-bit recombination, Shoup + Barrett / pseudo-Mersenne with a 30-bit fold constant) instead of
    the fast 25-bit-limb one, through the fused batch call on a ragged shape, CW = 16 and CW = 4:
    bit-exact against the oracle with the same explicit primes (reading C4 allows any NTT-friendly
    primes in (2^49, 2^50) through hl_ctx_create)."""
    N, L = 4096, 2
    primes, p = [], (((1 << 50) - (1 << mc_bits)) // (2 * N)) * (2 * N) + 1
    while len(primes) < L:
        if ref._is_prime(p):
            primes.append(p)
        p -= 2 * N
    ctx = hl.Context(N, L, 37, primes=primes, device=0)
    P = ref.bfv_params(N, L, 37, primes=primes)
    for (Nb, R, Ma, tile) in [(256, 48, 40, (16, 8, 16)), (40, 24, 40, (16, 8, 32))]:
        nI, nJ, nK = ref.tile_counts(tile, Ma, R, Nb)
        W = synth.weights(1300 + Nb, R, Ma)
        ct_in = synth.uniform_below(1310 + Nb, (nJ, nK, 2, P.L, P.N), P.primes)
        e = dict(wcache=ctx.encode_weights(tile, hl.to_device(W)), Ma=Ma, R=R, Nb=Nb, tile=tile,
                 ct_in=hl.to_device(ct_in), seed=1320)
        (m, sh), = ctx.he_linear_batch(tile, [e])
        _sync()
        em, es = ref.mask_and_share(P, tile, ref.he_matmul(P, tile, W, ct_in, Nb), Ma, Nb, 1320)
        assert np.array_equal(hl.to_host(m).reshape(em.shape), em)
        assert np.array_equal(hl.to_host(sh).reshape(es.shape), es)


# ------------------------------------------------------------------------- errors
def test_encode_weights_errors(hl, ctx4096):
    ctx = ctx4096
    W = synth.weights(1, 64, 64)
    W[3, 5] = 1 << 37
    with pytest.raises(hl.HLError) as e:
        ctx.encode_weights((16, 32, 8), hl.to_device(W))
    assert e.value.code == hl.HL_ERANGE
    Wbig = synth.stressed_weights(2, 64, 64, bound=1 << 30)     # 2R max|w| r_t >> Delta/2
    with pytest.raises(hl.HLError) as e:
        ctx.encode_weights((16, 32, 8), hl.to_device(Wbig))
    assert e.value.code == hl.HL_ENOISE


# ------------------------------------------------------------------------- both MAC engines
@pytest.mark.parametrize("engine", [0, 1, 2])
@pytest.mark.parametrize("N,shape,tile", [
    (4096, (40, 24, 40), (16, 8, 32)),
    (4096, (64, 48, 100), (4, 8, 16)),
    (4096, (3, 5, 7), (1, 1, 1)),
    (8192, (32, 48, 40), (32, 16, 16)),
])
def test_mac_engines_bit_exact(hl, ctx4096, ctx8192, engine, N, shape, tile):
    """IMAD.WIDE (engine 0), exact-FP64 (engine 1) and int8 tensor-core (engine 2, the default)
    MACs all equal the oracle."""
    ctx = ctx4096 if N == 4096 else ctx8192
    Nb, R, Ma = shape
    P, ct_in, W = _case_inputs(ctx, shape, tile, 700 + N + Ma + engine)
    ctx.set_mac_engine(engine)
    try:
        wc = ctx.encode_weights(tile, hl.to_device(W))
        out = ctx.he_matmul(tile, wc, Ma, R, Nb, hl.to_device(ct_in))
        got = hl.to_host(out).reshape(-1, 2, ctx.L, ctx.N)
    finally:
        ctx.set_mac_engine(2)
    exp = ref.he_matmul(P, tile, W, ct_in, Nb).reshape(-1, 2, ctx.L, ctx.N)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("engine", [0, 1, 2])
def test_mac_extreme_residues(hl, ctx4096, engine):
    """All weights and ciphertext residues = p - 1 (the largest products and sums) over a long
    J reduction (R = 3072 -> nJ = 384), every engine."""
    ctx = ctx4096
    P = _P(ctx)
    tile, (Nb, R, Ma) = (16, 8, 32), (32, 3072, 16)
    nI, nJ, nK = ref.tile_counts(tile, Ma, R, Nb)
    ct_in = np.empty((nJ, nK, 2, P.L, P.N), dtype=np.uint64)
    for l, p in enumerate(P.primes):
        ct_in[:, :, :, l, :] = p - 1
    W = synth.weights(801, R, Ma)
    ctx.set_mac_engine(engine)
    try:
        wc = ctx.encode_weights(tile, hl.to_device(W))
        out = ctx.he_matmul(tile, wc, Ma, R, Nb, hl.to_device(ct_in))
        got = hl.to_host(out).reshape(-1, 2, ctx.L, ctx.N)
    finally:
        ctx.set_mac_engine(2)
    exp = ref.he_matmul(P, tile, W, ct_in, Nb).reshape(-1, 2, ctx.L, ctx.N)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("engine", [1, 2])
def test_mac_long_j_chunked(hl, ctx4096, engine):
    """nJ = 4100 > 4096: the MAC splits J into launches of <= 4096 (the exact-accumulation bound
    of every engine) and adds the partial results mod p; the 4-J ragged tail also exercises the
    tensor-core engine's zero padding of J up to its 32-J MMA step."""
    ctx = ctx4096
    tile, (Nb, R, Ma) = (1, 2, 1), (1, 8200, 2)
    P, ct_in, W = _case_inputs(ctx, (Nb, R, Ma), tile, 900 + engine)
    ctx.set_mac_engine(engine)
    try:
        wc = ctx.encode_weights(tile, hl.to_device(W))
        out = ctx.he_matmul(tile, wc, Ma, R, Nb, hl.to_device(ct_in))
        got = hl.to_host(out).reshape(-1, 2, ctx.L, ctx.N)
    finally:
        ctx.set_mac_engine(2)
    exp = ref.he_matmul(P, tile, W, ct_in, Nb).reshape(-1, 2, ctx.L, ctx.N)
    assert np.array_equal(got, exp)


# ------------------------------------------------------------------------- FC layer (row f1)
@pytest.mark.parametrize("Nb,R,Ma", [(128, 768, 768), (5, 40, 50), (200, 100, 97), (1, 1, 1), (128, 3072, 96)])
def test_fc_local_share_vs_oracle(hl, ctx4096, Nb, R, Ma):
    """hl_fc_local_share (int8 tensor cores, 5 byte limbs) == oracle <W<x>_0>_1 + W<x>_1 + b mod 2^37:
    several M/N/K tiles with ragged tails (Nb > 128, Ma not a multiple of 48, R not of 32), the
    degenerate 1x1x1 product, and extreme limbs (all-ones 37-bit values)."""
    ctx = ctx4096
    S = synth.activations(901 + Nb, Nb, Ma)
    X1 = synth.activations(902 + R, Nb, R)
    W = synth.weights(903 + Ma, R, Ma)
    b = synth.activations(904, 1, Ma)[0]
    if Nb == 200:
        X1[:] = (1 << 37) - 1
        W[:7] = (1 << 37) - 1
    wp = ctx.fc_encode_weights(hl.to_device(W))
    # the unchecked online form (hl_fc_encode_weights_chk, check = 0) writes the same planes
    assert np.array_equal(hl.to_host(ctx.fc_encode_weights(hl.to_device(W), check=False)), hl.to_host(wp))
    share = hl.to_device(S)
    ctx.fc_local_share(hl.to_device(X1), wp, Ma, share, bias=hl.to_device(b))
    _sync()
    assert np.array_equal(hl.to_host(share).reshape(Nb, Ma), ref.fc_server_share(S, X1, W, b))


def test_fc_protocol_end_to_end(hl, ctx4096):
    """The FC protocol of PAPER.md:106-111 with the GPU server: the client encrypts its share X0,
    the server runs he_matmul_share and adds W X1 + b; client + server shares = X.W + b mod 2^37."""
    ctx = ctx4096
    P = _P(ctx)
    tile, (Nb, R, Ma) = (16, 8, 32), (40, 48, 72)
    X = synth.activations(911, Nb, R)
    X1 = synth.activations(912, Nb, R)
    X0 = (X - X1) & np.uint64((1 << 37) - 1)
    W = synth.weights(913, R, Ma)
    b = synth.activations(914, 1, Ma)[0]
    sk = ctx.keygen(915)
    ct_in = ctx.encrypt(sk, tile, X0, 916)
    wc = ctx.encode_weights(tile, hl.to_device(W))
    masked, share = ctx.he_matmul_share(tile, wc, Ma, R, Nb, hl.to_device(ct_in), seed=917)
    ctx.fc_local_share(hl.to_device(X1), ctx.fc_encode_weights(hl.to_device(W)), Ma, share, bias=hl.to_device(b))
    _sync()
    share_c = ctx.decrypt_share(sk, tile, hl.to_host(masked), Ma, Nb, True)
    got = (share_c + hl.to_host(share).reshape(Nb, Ma)) & np.uint64((1 << 37) - 1)
    want = (ref.matmul_mod_t(X, W) + b[None, :]) & np.uint64((1 << 37) - 1)
    assert np.array_equal(got, want)


# ------------------------------------------------------------------------- attention (row f2)
@pytest.mark.parametrize("n,d,n2,tiles", [
    (24, 20, 24, None), (128, 64, 128, None),
    (128, 128, 64, "plan"),       # the bench's per-term planner tiles (A V of one head)
])
def test_attention_cross_terms_vs_oracle(hl, ctx8192, n, d, n2, tiles):
    """Server side of Z = X.Y with both inputs shared: the responses and the
    server share equal the oracle's bit for bit, and with the client's decryptions plus its local
    product X0.Y0 the shares reconstruct X.Y mod 2^37 (N=8192, L=3; (128, 64, 128) = one BERT
    head's Q K^T)."""
    from paper_2305_18396_b200 import attention
    ctx = ctx8192
    P = _P(ctx)
    tile = (32, 16, 16) if tiles is None else (ctx.plan_tile(n, d, n2), ctx.plan_tile(n2, d, n))
    t1, t2 = (tile, tile) if tiles is None else tile
    X0, X1 = synth.activations(921, n, d), synth.activations(922, n, d)
    Y0, Y1 = synth.activations(923, d, n2), synth.activations(924, d, n2)
    seeds = (931, 932, 933, 934, 935, 936)          # (key, enc, mask) of term 1, then of term 2
    sk1, sk2 = ref.keygen(P, seeds[0]), ref.keygen(P, seeds[3])
    ct1 = ref.encrypt(P, t1, sk1, np.ascontiguousarray(Y0.T), seeds[1])
    ct2 = ref.encrypt(P, t2, sk2, X0, seeds[4])
    m1, m2, z1 = attention.server_cross_product(ctx, tile, hl.to_device(X1), hl.to_device(Y1), hl.to_device(ct1),
                                                hl.to_device(ct2), (seeds[2], seeds[5]))
    _sync()
    Z0, Z1 = ref.attention_protocol(P, tile, X0, X1, Y0, Y1, seeds)
    assert np.array_equal(hl.to_host(z1).reshape(n, n2), Z1)
    c1 = ctx.decrypt_share(sk1, t1, hl.to_host(m1), n, n2, True)          # [n2][n]
    c2 = ctx.decrypt_share(sk2, t2, hl.to_host(m2), n2, n, True)          # [n][n2]
    tm = np.uint64((1 << 37) - 1)
    z0 = (c1.T + c2 + ref.matmul_mod_t(X0, Y0)) & tm
    assert np.array_equal(z0, Z0)
    assert np.array_equal((z0 + hl.to_host(z1).reshape(n, n2)) & tm, ref.matmul_mod_t((X0 + X1) & tm, (Y0 + Y1) & tm))


def test_attention_batched_equals_single(hl, ctx8192):
    """server_cross_products (every head's two Pi_MatMul in one hl_he_linear_batch, the bench's
    row-f2 call) is bit-identical to server_cross_product per item (itself checked against the
    oracle above), for a mix of head shapes and tiles."""
    from paper_2305_18396_b200 import attention
    ctx = ctx8192
    items = []
    for h, (n, d, n2) in enumerate([(128, 64, 128), (128, 128, 64), (24, 20, 24)]):
        tiles = (ctx.plan_tile(n, d, n2), ctx.plan_tile(n2, d, n)) if h != 2 else (32, 16, 16)
        t1, t2 = (tiles, tiles) if h == 2 else tiles
        sd = 950 + 10 * h
        X0, X1 = synth.activations(sd, n, d), synth.activations(sd + 1, n, d)
        Y0, Y1 = synth.activations(sd + 2, d, n2), synth.activations(sd + 3, d, n2)
        sk1, sk2 = ctx.keygen(sd + 4), ctx.keygen(sd + 5)
        items.append(dict(tile=tiles, X1=hl.to_device(X1), Y1=hl.to_device(Y1),
                          ct_Y0T=hl.to_device(ctx.encrypt(sk1, t1, np.ascontiguousarray(Y0.T), sd + 6)),
                          ct_X0=hl.to_device(ctx.encrypt(sk2, t2, X0, sd + 7)), seeds=(sd + 8, sd + 9)))
    single = [tuple(hl.to_host(x) for x in attention.server_cross_product(
        ctx, it["tile"], it["X1"], it["Y1"], it["ct_Y0T"], it["ct_X0"], it["seeds"])) for it in items]
    for _ in range(2):
        batched = attention.server_cross_products(ctx, items)
        _sync()
        for k, (b, s_) in enumerate(zip(batched, single)):
            for x, y in zip(b, s_):
                assert np.array_equal(hl.to_host(x), y), k


def test_share_accumulate_transpose(hl, ctx4096):
    """hl_share_accumulate: dst += src^T (and src) mod 2^37 on ragged 32x32 tiles."""
    ctx = ctx4096
    a = synth.activations(941, 45, 70)
    b = synth.activations(942, 70, 45)
    c = synth.activations(943, 45, 70)
    d = hl.to_device(a)
    ctx.share_accumulate(d, hl.to_device(b), 45, 70, transpose=True)
    ctx.share_accumulate(d, hl.to_device(c), 45, 70)
    _sync()
    assert np.array_equal(hl.to_host(d).reshape(45, 70), (a + b.T + c) & np.uint64((1 << 37) - 1))


# ------------------------------------------------------------------------- client on the GPU (row f3)
@pytest.mark.parametrize("N,shape,tile", [(4096, (8, 64, 64), (16, 32, 8)), (4096, (40, 24, 40), (16, 8, 32)),
                                          (8192, (32, 48, 40), (32, 16, 16)), (4096, (3, 5, 7), (1, 1, 1))])
def test_device_client_encrypt_decrypt(hl, ctx4096, ctx8192, N, shape, tile):
    """hl_encrypt_device == the oracle's encrypt (and the host client), bit for bit; the GPU server
    then runs, and hl_decrypt_share_device (RNS rounding) == the oracle's decrypt (exact CRT)."""
    ctx = ctx4096 if N == 4096 else ctx8192
    P = _P(ctx)
    Nb, R, Ma = shape
    X = synth.activations(951 + N, Nb, R)
    W = synth.weights(952 + N, R, Ma)
    sk = ref.keygen(P, 953)
    s_hat = ctx.sk_prepare(sk)
    ct_dev = ctx.encrypt_device(s_hat, tile, hl.to_device(X), 954)
    _sync()
    exp = ref.encrypt(P, tile, sk, X, 954)
    assert np.array_equal(hl.to_host(ct_dev).reshape(exp.shape), exp)
    wc = ctx.encode_weights(tile, hl.to_device(W))
    masked, share_s = ctx.he_matmul_share(tile, wc, Ma, R, Nb, ct_dev, seed=955)
    share_c = ctx.decrypt_share_device(s_hat, tile, masked, Ma, Nb)
    _sync()
    exp_c = ref.decrypt_share(P, tile, sk, hl.to_host(masked), Ma, Nb, True)
    assert np.array_equal(hl.to_host(share_c).reshape(Nb, Ma), exp_c)
    assert np.array_equal((exp_c + hl.to_host(share_s).reshape(Nb, Ma)) & np.uint64((1 << 37) - 1),
                          ref.matmul_mod_t(X, W))



def test_bert_base_c3_shape_sampled(hl, ctx4096):
    """Config c3's product shape (8 sequences: Nb = 1024 -> nC = 64, four 16-column groups) for
    W_o (768 x 768) at full size in the bench's launch configuration: sampled output ciphertexts
    bit-exact vs the oracle's scalar NTT path, and the whole product's reconstruction vs X.W."""
    ctx = ctx4096
    cfg = synth.CONFIGS["c3"]
    P = _P(ctx)
    tile = cfg.tile
    mm = cfg.matmuls[1]
    assert (mm.Nb, mm.R, mm.Ma) == (1024, 768, 768)
    X = synth.activations(961, mm.Nb, mm.R)
    W = synth.weights(962, mm.R, mm.Ma)
    sk = ctx.keygen(963)
    s_hat = ctx.sk_prepare(sk)
    ct_in = ctx.encrypt_device(s_hat, tile, hl.to_device(X), 964)
    wc = ctx.encode_weights(tile, hl.to_device(W))
    masked, share = ctx.he_linear_batch(tile, [dict(wcache=wc, Ma=mm.Ma, R=mm.R, Nb=mm.Nb, ct_in=ct_in, seed=965)])[0]
    share_c = ctx.decrypt_share_device(s_hat, tile, masked, mm.Ma, mm.Nb)
    _sync()
    nI, nJ, nK = ref.tile_counts(tile, mm.Ma, mm.R, mm.Nb)
    mh = hl.to_host(masked).reshape(nI, nK, -1)
    tiles = [(0, 0), (nI - 1, nK - 1), (13, 17), (47, 31)]
    exp_ct = ref.he_matmul_ntt_tiles(P, tile, W, hl.to_host(ct_in).reshape(nJ, nK, 2, P.L, P.N), mm.Nb, tiles)
    em, _ = ref.mask_tiles(P, tile, exp_ct, nK, tiles, 965, True)
    for o, (I, K) in enumerate(tiles):
        assert np.array_equal(mh[I, K], em[o]), (I, K)
    got = (hl.to_host(share_c).reshape(mm.Nb, mm.Ma) + hl.to_host(share).reshape(mm.Nb, mm.Ma)) & np.uint64((1 << 37) - 1)
    assert np.array_equal(got, ref.matmul_mod_t(X, W))


def test_bert_large_c4_shape_sampled(hl, ctx8192):
    """Config c4's parameters and product shape (N=8192, L=3, tile (32,16,16); 4 sequences of 512:
    Nb = 2048 -> nC = 256, sixteen 16-column groups) for W_o (1024 x 1024) at full size: sampled
    output ciphertexts bit-exact vs the oracle's scalar NTT path, whole-product reconstruction."""
    ctx = ctx8192
    cfg = synth.CONFIGS["c4"]
    P = _P(ctx)
    tile = cfg.tile
    mm = cfg.matmuls[1]
    assert (mm.Nb, mm.R, mm.Ma) == (2048, 1024, 1024) and tile == (32, 16, 16)
    X = synth.activations(971, mm.Nb, mm.R)
    W = synth.weights(972, mm.R, mm.Ma)
    sk = ctx.keygen(973)
    s_hat = ctx.sk_prepare(sk)
    ct_in = ctx.encrypt_device(s_hat, tile, hl.to_device(X), 974)
    wc = ctx.encode_weights(tile, hl.to_device(W))
    masked, share = ctx.he_linear_batch(tile, [dict(wcache=wc, Ma=mm.Ma, R=mm.R, Nb=mm.Nb, ct_in=ct_in, seed=975)])[0]
    share_c = ctx.decrypt_share_device(s_hat, tile, masked, mm.Ma, mm.Nb)
    _sync()
    nI, nJ, nK = ref.tile_counts(tile, mm.Ma, mm.R, mm.Nb)
    mh = hl.to_host(masked).reshape(nI, nK, -1)
    tiles = [(0, 0), (nI - 1, nK - 1), (17, 100)]
    ct_h = hl.to_host(ct_in).reshape(nJ, nK, 2, P.L, P.N)
    exp_ct = ref.he_matmul_ntt_tiles(P, tile, W, ct_h, mm.Nb, tiles)
    em, _ = ref.mask_tiles(P, tile, exp_ct, nK, tiles, 975, True)
    for o, (I, K) in enumerate(tiles):
        assert np.array_equal(mh[I, K], em[o]), (I, K)
    got = (hl.to_host(share_c).reshape(mm.Nb, mm.Ma) + hl.to_host(share).reshape(mm.Nb, mm.Ma)) & np.uint64((1 << 37) - 1)
    assert np.array_equal(got, ref.matmul_mod_t(X, W))


# ------------------------------------------------------------------------- re-randomisation (row f4)
@pytest.mark.parametrize("N,shape,tile,fb", [
    (4096, (24, 16, 40), (16, 8, 32), 0),          # pruned c0 path (r = 8), no flooding
    (4096, (24, 16, 40), (16, 8, 32), 58),         # with flooding
    (4096, (8, 64, 64), (16, 32, 8), 40),          # r = 32: unpruned c0 path
    (8192, (32, 48, 40), (32, 16, 16), 62),        # N=8192, L=3, the largest flood (one PRF word)
])
def test_rerandomized_response_vs_oracle(hl, ctx4096, ctx8192, N, shape, tile, fb):
    """hl_he_matmul_share_rr == oracle rerandomize + mask_and_share bit for bit; the client's
    decryption of the re-randomised (and flooded) response still reconstructs X.W mod 2^37."""
    ctx = ctx4096 if N == 4096 else ctx8192
    P = _P(ctx)
    Nb, R, Ma = shape
    X, W = synth.activations(981 + fb, Nb, R), synth.weights(982, R, Ma)
    sk = ref.keygen(P, 983)
    pk = ref.pk_gen(P, sk, 984)
    ct_in = ref.encrypt(P, tile, sk, X, 985)
    wc = ctx.encode_weights(tile, hl.to_device(W))
    masked, share = ctx.he_matmul_share_rr(tile, wc, Ma, R, Nb, hl.to_device(ct_in), 986, ctx.pk_prepare(pk), fb)
    _sync()
    nI, nJ, nK = ref.tile_counts(tile, Ma, R, Nb)
    ct_rr = ref.rerandomize(P, tile, pk, ref.he_matmul(P, tile, W, ct_in, Nb), nK, 986, fb)
    em, es = ref.mask_and_share(P, tile, ct_rr, Ma, Nb, 986, True)
    assert np.array_equal(hl.to_host(masked).reshape(em.shape), em)
    assert np.array_equal(hl.to_host(share).reshape(es.shape), es)
    share_c = ctx.decrypt_share(sk, tile, hl.to_host(masked), Ma, Nb, True)
    assert np.array_equal((share_c + es) & np.uint64((1 << 37) - 1), ref.matmul_mod_t(X, W))


# ------------------------------------------------------------------------- write bounds (memcheck stand-in)
_GUARD = 8192          # words of guard band before and after every buffer


def _guarded(nwords, fill=None):
    """A device buffer of nwords with guard bands of a known pattern on both sides; returns
    (full tensor, view).  compute-sanitizer is refused on this pool (profiles/r02), so the tests
    check the library's writes against buffer bounds this way."""
    import torch
    full = torch.full((nwords + 2 * _GUARD,), 0x5A5A5A5A5A5A5A5A - (1 << 63), dtype=torch.int64, device="cuda")
    view = full[_GUARD:_GUARD + nwords]
    if fill is not None:
        view.copy_(fill)
    return full, view


def _guards_intact(full, nwords):
    g = 0x5A5A5A5A5A5A5A5A - (1 << 63)
    return bool((full[:_GUARD] == g).all()) and bool((full[_GUARD + nwords:] == g).all())


@pytest.mark.parametrize("case", ["c1_batch", "fat_cw16", "c0_fused", "c1_host_seeded", "ragged_shard"])
def test_writes_stay_in_bounds(hl, ctx4096, case):
    """Every buffer the server calls write (workspace, NTT-domain scratch, compressed responses,
    share) sits between guard bands that must come back untouched, the read-only inputs (ct_in,
    weight caches) must come back unchanged, and the results must still equal the oracle's; the
    calls cover the batch (two streams), the CW = 16 MAC with the c1 transposition, the fused single
    call, the host batch with the seeded upload and an I-tile shard of a ragged product."""
    import torch
    ctx = ctx4096
    P = _P(ctx)
    if case == "c1_batch":
        cfg = synth.CONFIGS["c1"]
        specs = [(mm.Nb, mm.R, mm.Ma, cfg.tile, 0, -1) for mm in cfg.matmuls]
    elif case == "fat_cw16":
        specs = [(256, 48, 40, (16, 8, 16), 0, -1)]
    elif case == "c0_fused":
        specs = [(8, 64, 64, (16, 32, 8), 0, -1)]
    elif case == "c1_host_seeded":
        cfg = synth.CONFIGS["c1"]
        specs = [(mm.Nb, mm.R, mm.Ma, cfg.tile, 0, -1) for mm in cfg.matmuls[:2]]
    else:
        specs = [(40, 72, 168, (16, 8, 32), 3, 8)]
    ents, checks = [], []
    for k, (Nb, R, Ma, tile, i0, i1) in enumerate(specs):
        lay = ctx.layout(tile, Ma, R, Nb, i0, i1)
        W = synth.weights(1500 + k, R, Ma)
        X = synth.activations(1510 + k, Nb, R)
        sk = ref.keygen(P, 1520 + k)
        ct = ref.encrypt(P, tile, sk, X, 1530 + k)
        wc = ctx.encode_weights(tile, hl.to_device(W), i0, i1)
        wc_sum = wc.clone()
        ct_dev = hl.to_device(ct)
        bufs = {name: _guarded(n) for name, n in (("ws", lay.workspace_bytes // 8), ("co", lay.ct_out_words),
                                                  ("cm", lay.ct_masked_words), ("sh", lay.share_words))}
        e = dict(wcache=wc, Ma=Ma, R=R, Nb=Nb, tile=tile, ct_in=ct_dev, seed=1540 + k, i_begin=i0, i_end=i1,
                 workspace=bufs["ws"][1], ct_out_ntt=bufs["co"][1], ct_masked=bufs["cm"][1], share=bufs["sh"][1])
        if case == "c1_host_seeded":
            up = _guarded(lay.ct_in_words)
            bufs["up"] = up
            c0 = torch.from_numpy(hl.Context.c0_halves(ct).view(np.int64).reshape(-1)).pin_memory()
            e.update(ct_in=up[1], c0_host=c0, a_seed=ref.public_seed(1530 + k), packed=False,
                     masked_host=torch.zeros(lay.ct_masked_words, dtype=torch.int64).pin_memory(),
                     share_host=torch.zeros(lay.share_words, dtype=torch.int64).pin_memory())
        ents.append(e)
        nI = lay.nI
        ct_full = ref.he_matmul(P, tile, W, ct, Nb)
        em, es = ref.mask_and_share(P, tile, ct_full, Ma, Nb, 1540 + k)
        checks.append((lay, bufs, wc, wc_sum, ct_dev, ct.copy(), em[i0:(i1 if i1 >= 0 else nI)], es, i0, i1, tile, Ma))
    if case == "c0_fused":
        e = ents[0]
        ctx.he_matmul_share(e["tile"], e["wcache"], e["Ma"], e["R"], e["Nb"], e["ct_in"], e["seed"], True,
                            workspace=e["workspace"], ct_out_ntt=e["ct_out_ntt"], ct_masked=e["ct_masked"],
                            share=e["share"])
    elif case == "c1_host_seeded":
        ctx.he_linear_batch_host(specs[0][3], ents)
    else:
        ctx.he_linear_batch(specs[0][3], ents)
    _sync()
    for (lay, bufs, wc, wc_sum, ct_dev, ct_h, em, es, i0, i1, tile, Ma) in checks:
        for name, (full, view) in bufs.items():
            assert _guards_intact(full, view.numel()), (case, name)
        assert torch.equal(wc, wc_sum), (case, "weight cache written")
        assert np.array_equal(hl.to_host(ct_dev).reshape(ct_h.shape), ct_h), (case, "ct_in written")
        got = hl.to_host(bufs["cm"][1]).reshape(em.shape)
        assert np.array_equal(got, em), case
        m = tile[0]
        c0_, c1_ = i0 * m, min((i1 if i1 >= 0 else lay.nI) * m, Ma)
        sh = hl.to_host(bufs["sh"][1]).reshape(es.shape)
        assert np.array_equal(sh[:, c0_:c1_], es[:, c0_:c1_]), case
