"""C-ABI library checks that need no GPU (-m "not gpu").

* libhelinear.so loads and exports every function include/helinear.h declares;
* the library's host-side client (keygen, encrypt, decrypt_share) is bit-exact against the
  oracle on the same seeds (host-only context, device = -1);
* parameter derivation, layouts and error codes.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import synth
from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hl():
    from paper_2305_18396_b200 import build
    build.build()
    import paper_2305_18396_b200 as hl
    hl.load_library()
    return hl


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "helinear.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hl_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(hl):
    declared = _declared_functions()
    assert len(declared) >= 14
    lib = ctypes.CDLL(hl.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(hl.EXPORTS) == declared


@pytest.mark.parametrize("N,L", [(4096, 2), (8192, 3)])
def test_params_match_oracle(hl, N, L):
    ctx = hl.Context(N, L, 37, device=-1)
    P = ref.bfv_params(N, L, 37)
    assert ctx.primes == P.primes
    assert ctx.delta_mod == tuple(P.delta_mod)


def test_explicit_primes_and_errors(hl):
    P = ref.bfv_params(4096, 2, 37)
    ctx = hl.Context(4096, 2, 37, primes=P.primes[::-1], device=-1)
    assert ctx.primes == P.primes[::-1]
    with pytest.raises(hl.HLError) as e:
        hl.Context(2048, 2, 37, device=-1)
    assert e.value.code == hl.HL_ENOTSUP
    with pytest.raises(hl.HLError) as e:
        hl.Context(4096, 2, 37, primes=[P.primes[0] + 2, P.primes[1]], device=-1)
    assert e.value.code == hl.HL_ENOTSUP
    with pytest.raises(hl.HLError) as e:
        hl.Context(4096, 4, 37, device=-1)
    assert e.value.code == hl.HL_ENOTSUP


def test_layout_and_dims(hl):
    ctx = hl.Context(4096, 2, 37, device=-1)
    lay = ctx.layout((16, 8, 32), 2304, 768, 128)
    assert (lay.nI, lay.nJ, lay.nK) == (144, 96, 4)
    assert lay.ct_in_words == 96 * 4 * 2 * 2 * 4096
    assert lay.ct_masked_words == 144 * 4 * 2 * (16 * 32 + 4096)
    # default engine 2 (int8 tensor cores): 7 byte limbs per NTT-domain weight residue
    assert lay.wcache_bytes == 144 * 96 * 2 * 4096 * 7
    assert lay.workspace_bytes == 96 * 4 * 2 * 2 * 4096 * 8 + 256
    sh = ctx.layout((16, 8, 32), 2304, 768, 128, 10, 20)
    assert sh.nI_shard == 10 and sh.wcache_bytes == 16 * 96 * 2 * 4096 * 7   # rows padded to 16
    odd = ctx.layout((16, 8, 32), 64, 40, 64)                    # nJ = 5 padded to the 32-J MMA step
    assert odd.wcache_bytes == 16 * 32 * 2 * 4096 * 7 and odd.workspace_bytes == 32 * 2 * 2 * 2 * 4096 * 8 + 256
    ctx.set_mac_engine(1)                                        # FP64 engine: one double per residue
    assert ctx.layout((16, 8, 32), 2304, 768, 128).wcache_bytes == 144 * 96 * 2 * 4096 * 8
    with pytest.raises(hl.HLError) as e:
        ctx.layout((16, 16, 32), 64, 64, 64)          # m*r*n = 8192 > N
    assert e.value.code == hl.HL_EDIM
    with pytest.raises(hl.HLError) as e:
        ctx.layout((3, 8, 32), 64, 64, 64)            # tiles are powers of two (reading C2)
    assert e.value.code == hl.HL_EDIM
    with pytest.raises(hl.HLError) as e:
        ctx.layout((16, 8, 32), 64, 64, 64, 3, 9)     # shard beyond nI = 4
    assert e.value.code == hl.HL_EINVAL


def test_plan_tile(hl):
    """hl_plan_tile (host logic, no GPU): valid power-of-two tiles with m*r*n = N, the c2 choices
    that synth.CONFIGS['c2'].tiles (the bench's tiles) records, and the argument checks."""
    ctx = hl.Context(4096, 2, 37, device=-1)
    cfg = synth.CONFIGS["c2"]
    for mi, mm in enumerate(cfg.matmuls):
        t = ctx.plan_tile(mm.Ma, mm.R, mm.Nb)
        assert t == cfg.tile_of(mi), (mm.name, t)
    for shape in [(1, 1, 1), (7, 300, 5), (4096, 4096, 4096), (128, 3072, 768)]:
        m, r, n = ctx.plan_tile(*shape)
        assert m * r * n <= 4096 and all(v & (v - 1) == 0 for v in (m, r, n))
        assert m <= 2 * shape[0] and r <= 2 * shape[1] and n <= 2 * shape[2]
        assert m * r * n == 4096 or (m >= shape[0] and r >= shape[1] and n >= shape[2])
        ctx.layout((m, r, n), *shape)                   # accepted by the geometry check
    assert hl.Context(8192, 3, 37, device=-1).plan_tile(1024, 1024, 2048)[0] > 0
    with pytest.raises(hl.HLError) as e:
        ctx.plan_tile(0, 8, 8)
    assert e.value.code == hl.HL_EINVAL


def test_pack50_roundtrip(hl):
    """50-bit wire format: exact round trip (full and partial last group, residues up to 2^50-1),
    25/32 of the words, HL_ERANGE for a word >= 2^50."""
    rng = np.random.default_rng(5)
    for words in (32, 96, 1000, 1, 0):
        v = rng.integers(0, 1 << 50, size=words, dtype=np.uint64)
        if words:
            v[0] = (1 << 50) - 1
        p = hl.Context.pack50(v)
        assert p.size == -(-words // 32) * 25
        assert np.array_equal(hl.Context.unpack50(p, words), v)
    # bit layout: residue i of a group starts at bit 50 i
    v = np.zeros(32, np.uint64); v[1] = 1; v[31] = 3
    p = hl.Context.pack50(v)
    assert int(p[0]) == 1 << 50 and int(p[24]) == 3 << (1550 - 1536)
    with pytest.raises(hl.HLError) as e:
        hl.Context.pack50(np.array([1 << 50], dtype=np.uint64))
    assert e.value.code == hl.HL_ERANGE


def test_keygen_matches_oracle(hl):
    ctx = hl.Context(4096, 2, 37, device=-1)
    P = ref.bfv_params(4096, 2, 37)
    for seed in (0, 7, 2**63 + 5):
        assert np.array_equal(ctx.keygen(seed), ref.keygen(P, seed))


@pytest.mark.parametrize("N,L", [(4096, 2), (8192, 3)])
def test_pk_gen_matches_oracle(hl, N, L):
    """Row f4: the library's public key (host client) equals the oracle's, bit for bit."""
    ctx = hl.Context(N, L, 37, device=-1)
    P = ref.bfv_params(N, L, 37)
    sk = ref.keygen(P, 41)
    assert np.array_equal(ctx.pk_gen(sk, 42), ref.pk_gen(P, sk, 42))


@pytest.mark.parametrize("N,L,shape,tile", [
    (4096, 2, (8, 64), (16, 32, 8)),
    (4096, 2, (37, 21), (4, 8, 16)),           # ragged
    (8192, 3, (16, 40), (32, 16, 16)),
])
def test_encrypt_bit_exact_vs_oracle(hl, N, L, shape, tile):
    ctx = hl.Context(N, L, 37, device=-1)
    P = ref.bfv_params(N, L, 37)
    X = synth.activations(101, *shape)
    sk = ref.keygen(P, 102)
    assert np.array_equal(ctx.encrypt(sk, tile, X, 103), ref.encrypt(P, tile, sk, X, 103))


def test_public_seed_matches_oracle(hl):
    """Reading C28: the library's public seed (shipped by the seeded upload) equals the oracle's."""
    for s in (0, 103, 0x230518396 + 3, 2**64 - 1):
        assert hl.public_seed(s) == ref.public_seed(s)


@pytest.mark.parametrize("compress", [True, False])
def test_decrypt_share_matches_oracle(hl, compress):
    ctx = hl.Context(4096, 2, 37, device=-1)
    P = ref.bfv_params(4096, 2, 37)
    tile, Nb, R, Ma = (8, 16, 16), 20, 40, 24
    X, W = synth.activations(111, Nb, R), synth.weights(112, R, Ma)
    out = ref.matmul_protocol(P, tile, X, W, 113, 114, 115, compress)
    got = ctx.decrypt_share(out["sk"], tile, out["masked"], Ma, Nb, compress)
    assert np.array_equal(got, out["share_client"])


def test_client_errors(hl):
    ctx = hl.Context(4096, 2, 37, device=-1)
    sk = ctx.keygen(1)
    bad = sk.copy(); bad[5] = 2
    X = synth.activations(1, 8, 64)
    with pytest.raises(hl.HLError) as e:
        ctx.encrypt(bad, (16, 32, 8), X, 1)
    assert e.value.code == hl.HL_ERANGE
    X2 = X.copy(); X2[0, 0] = 1 << 37
    with pytest.raises(hl.HLError) as e:
        ctx.encrypt(sk, (16, 32, 8), X2, 1)
    assert e.value.code == hl.HL_ERANGE
    with pytest.raises(hl.HLError) as e:
        ctx.encrypt(sk, (16, 32, 16), X, 1)
    assert e.value.code == hl.HL_EDIM
