"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test pins an oracle function to something other than itself: a closed form, a
special case, an independent library routine (cryptography's ChaCha20, mpmath, numpy),
brute force on tiny inputs, or the SPEC/paper worked example under tests/golden/.
"""
import json
import os
import random

import numpy as np
import pytest

import synth
from oracle import ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------------------ params (O1)
def _miller_rabin(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (first 13 prime bases) -- independent of sympy."""
    if n < 2:
        return False
    bases = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41]
    for b in bases:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in bases:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = pow(x, 2, n)
            if x == n - 1:
                break
        else:
            return False
    return True


@pytest.mark.parametrize("N,L", [(4096, 2), (8192, 3)])
def test_primes_are_the_largest_ntt_friendly(N, L):
    P = ref.bfv_params(N, L, 37)
    assert len(P.primes) == L
    # largest first; every candidate p = 1 mod 2N between 2^50 and the last prime is checked
    cand = ((1 << 50) - 1) // (2 * N) * (2 * N) + 1
    found = []
    while len(found) < L:
        if _miller_rabin(cand):
            found.append(cand)
        cand -= 2 * N
    assert tuple(found) == P.primes
    for p, psi in zip(P.primes, P.psis):
        assert p < (1 << 50) and p % (2 * N) == 1
        assert pow(psi, N, p) == p - 1          # psi is a primitive 2N-th root: psi^N = -1
        assert pow(psi, 2 * N, p) == 1


def test_delta_closed_form(P4096, P8192):
    for P in (P4096, P8192):
        q, t = P.q, P.t
        assert P.delta * t <= q < (P.delta + 1) * t
        assert P.r_t == q - P.delta * t
        assert all(dm == P.delta % p for dm, p in zip(P.delta_mod, P.primes))
    # N=4096/L=2 shares its primes with N=8192/L=3 (both are = 1 mod 16384?) -- only if so:
    assert 99 < P4096.q.bit_length() <= 100


# ------------------------------------------------------------------------------ PRF (O2, C10)
def _lib_chacha_u64(seed, domain, stream, count, first=0):
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms
    key = int(seed).to_bytes(8, "little") + bytes(24)
    nonce12 = int(domain).to_bytes(4, "little") + int(stream).to_bytes(8, "little")
    blk0 = first // 8
    nblk = (first + count + 7) // 8 - blk0
    nonce16 = blk0.to_bytes(4, "little") + nonce12
    ks = Cipher(algorithms.ChaCha20(key, nonce16), mode=None).encryptor().update(bytes(64 * nblk))
    words = np.frombuffer(ks, dtype="<u8")
    off = first - 8 * blk0
    return words[off:off + count].astype(np.uint64)


@pytest.mark.parametrize("seed,domain,stream,count,first", [
    (0, 1, 0, 64, 0), (0x230518396, 2, 5, 100, 3), (2**64 - 1, 4, 2**40 + 7, 37, 1001),
    (12345, 3, 17, 8, 8 * 300)])
def test_prf_matches_cryptography_chacha20(seed, domain, stream, count, first):
    ours = ref.prf_u64(seed, domain, stream, count, first)
    assert np.array_equal(ours, _lib_chacha_u64(seed, domain, stream, count, first))


# ------------------------------------------------------------------------------ CDT (C8)
def test_cdt_table_closed_form():
    import mpmath
    T = ref.cdt_table()
    assert len(T) == 42 and T[-1] == 1 << 63
    assert all(T[k] < T[k + 1] for k in range(20))          # strictly increasing in the bulk
    assert all(T[k] <= T[k + 1] for k in range(41))         # saturates at 2^63 - 1 in the far tail
    # moments of the table's distribution vs the closed-form discrete Gaussian
    probs = [T[0]] + [T[k] - T[k - 1] for k in range(1, 42)]
    var = sum(k * k * p for k, p in enumerate(probs)) / 2**63
    mpmath.mp.dps = 40
    rho = [mpmath.e ** (-(k * k) / mpmath.mpf("20.48")) for k in range(-41, 42)]
    var_exact = sum((k - 41) ** 2 * r for k, r in enumerate(rho)) / sum(rho)
    assert abs(var - float(var_exact)) < 1e-12
    assert abs(var ** 0.5 - 3.2) < 0.01          # a discrete Gaussian of width 3.2 has std ~3.2
    # P(E = 0) = 1/Z
    assert abs(T[0] / 2**63 - float(1 / sum(rho))) < 1e-15


def test_cdt_sampler_boundaries_and_moments(P4096):
    import ctypes
    T = ref._u64arr(ref.cdt_table())
    one = ref.lib().or_cdt_sample_one
    one.restype = ctypes.c_int64
    for k in (0, 1, 5, 20):           # distinct table entries (the far tail saturates)
        for sign in (0, 1):
            u_in = (sign << 63) | (int(T[k]) - 1)
            u_next = (sign << 63) | int(T[k])
            s = -1 if sign else 1
            assert one(ctypes.c_uint64(u_in), ref._p(T), 42) == s * k
            assert one(ctypes.c_uint64(u_next), ref._p(T), 42) == s * (k + 1)
    e = np.concatenate([ref.sample_e(P4096, 99, g) for g in range(25)]).astype(np.float64)
    assert abs(e.mean()) < 0.05 and abs(e.std() - 3.2) < 0.04 and np.abs(e).max() <= 41


# ------------------------------------------------------------------------------ encodings
def test_encodings_golden():
    g = json.load(open(os.path.join(GOLDEN, "encodings.json")))
    N = g["N"]
    for case in g["piA"]:
        a = ref.encode_A(case["A"], N, case["r"])
        assert a[:len(case["poly"])] == case["poly"] and not any(a[len(case["poly"]):])
    for case in g["piB"]:
        b = ref.encode_B(case["B"], N, case["m"])
        assert b[:len(case["poly"])] == case["poly"] and not any(b[len(case["poly"]):])
    pr = g["product"]
    c = ref.negacyclic_mul_int(ref.encode_A(pr["A"], N, pr["r"]), ref.encode_B(pr["B"], N, pr["m"]), N)
    assert c[:len(pr["poly"])] == pr["poly"]
    assert ref.decode_C(c, pr["m"], pr["r"], pr["n"]) == pr["C"]


@pytest.mark.parametrize("N,tile", [(64, (2, 4, 8)), (64, (4, 4, 4)), (64, (1, 64, 1)),
                                    (64, (64, 1, 1)), (64, (1, 1, 64)), (128, (3, 5, 7))])
def test_encodings_reconstruct_matmul_bruteforce(N, tile):
    """No-collision property of Alg. 1: decode(pi_A(A) * pi_B(B)) = A.B over Z (brute force)."""
    m, r, n = tile
    rng = random.Random(N * 1000 + m * 100 + r * 10 + n)
    for _ in range(5):
        A = [[rng.randint(-50, 50) for _ in range(r)] for _ in range(m)]
        B = [[rng.randint(-50, 50) for _ in range(n)] for _ in range(r)]
        c = ref.negacyclic_mul_int(ref.encode_A(A, N, r), ref.encode_B(B, N, m), N)
        AB = [[sum(A[i][j] * B[j][k] for j in range(r)) for k in range(n)] for i in range(m)]
        assert ref.decode_C(c, m, r, n) == AB


# ------------------------------------------------------------------------------ negacyclic products, NTT
def test_negacyclic_special_cases(P4096):
    N, p = P4096.N, P4096.primes[0]
    a = np.zeros(N, np.uint64); a[N - 1] = 1
    x = np.zeros(N, np.uint64); x[1] = 1
    out = ref.negacyclic_mul(N, p, a, x)                       # x^(N-1) * x = -1
    assert out[0] == p - 1 and not out[1:].any()
    rng = np.random.default_rng(1)
    b = rng.integers(0, p, N, dtype=np.uint64)
    one = np.zeros(N, np.uint64); one[0] = 1
    assert np.array_equal(ref.negacyclic_mul(N, p, one, b), b)   # 1 * b = b


def test_schoolbook_vs_python_vs_numpy_fold():
    N, p = 64, ref.ntt_primes(64, 1)[0]
    rng = np.random.default_rng(2)
    for _ in range(10):
        a = rng.integers(0, p, N, dtype=np.uint64)
        b = rng.integers(0, p, N, dtype=np.uint64)
        c = ref.negacyclic_mul(N, p, a, b)
        full = np.convolve(a.astype(object), b.astype(object))          # numpy, exact ints
        fold = [(int(full[k]) - (int(full[k + N]) if k + N < len(full) else 0)) % p for k in range(N)]
        assert [int(v) for v in c] == fold
        assert [int(v) for v in c] == ref.negacyclic_mul_int([int(v) for v in a], [int(v) for v in b], N, p)


@pytest.mark.parametrize("N", [16, 64])
def test_oracle_ntt_fast_equals_definition(N):
    p = ref.ntt_primes(N, 1)[0]
    psi = ref.primitive_2n_root(p, N)
    rng = np.random.default_rng(N)
    a = rng.integers(0, p, N, dtype=np.uint64)
    assert np.array_equal(ref.ntt(N, p, psi, a), ref.ntt_naive(N, p, psi, a))
    x = np.zeros(N, np.uint64); x[1] = 1                    # NTT(x)_k = psi^(2k+1)
    assert [int(v) for v in ref.ntt(N, p, psi, x)] == [pow(psi, 2 * k + 1, p) for k in range(N)]


@pytest.mark.parametrize("N", [64, 1024, 4096])
def test_oracle_ntt_roundtrip_and_convolution(N):
    rng = np.random.default_rng(N + 7)
    for p in ref.ntt_primes(N, 2):
        psi = ref.primitive_2n_root(p, N)
        a = rng.integers(0, p, N, dtype=np.uint64)
        b = rng.integers(0, p, N, dtype=np.uint64)
        assert np.array_equal(ref.intt(N, p, psi, ref.ntt(N, p, psi, a)), a)     # INTT o NTT = id
        assert np.array_equal(ref.negacyclic_mul_ntt(N, p, psi, a, b), ref.negacyclic_mul(N, p, a, b))


# ------------------------------------------------------------------------------ BFV encrypt / decrypt (O3, O4, O10)
def test_keygen_ternary_and_balanced(P4096):
    sk = ref.keygen(P4096, 7)
    assert set(np.unique(sk)) <= {-1, 0, 1}
    counts = [(sk == v).sum() for v in (-1, 0, 1)]
    assert min(counts) > 1200      # (u mod 3) - 1 is near-uniform
    assert np.array_equal(sk, ref.keygen(P4096, 7))   # deterministic per seed


def test_keygen_is_the_sk_stream(P4096, P8192):
    """O3 recomputed from the library ChaCha20: s_i = (u64_SK[i] mod 3) - 1, stream (seed, 1, 0)."""
    for P, seed in ((P4096, 7), (P8192, 2**64 - 3)):
        u = _lib_chacha_u64(seed, 1, 0, P.N)
        assert np.array_equal(ref.keygen(P, seed), ((u % np.uint64(3)).astype(np.int64) - 1).astype(np.int8))


def test_public_seed_is_the_pub_stream_and_hides_the_error_key():
    """Reading C28: a_seed = word 0 of the library ChaCha20 stream (seed, 10, 0); distinct seeds give
    distinct public seeds, and the public seed is not the private one."""
    seeds = [0, 1, 5, 0x230518396 + 3, 2**64 - 1]
    pubs = [ref.public_seed(s) for s in seeds]
    for s, a in zip(seeds, pubs):
        assert a == int(_lib_chacha_u64(s, 10, 0, 1)[0]) and a != s
    assert len(set(pubs)) == len(pubs)


@pytest.mark.parametrize("NL", [(4096, 2), (8192, 3)])
def test_encrypt_c1_is_the_a_stream(NL, P4096, P8192):
    """O4 + C26 + C28 recomputed from the library ChaCha20: the c1 half of input ciphertext g for
    prime l is a_hat[i] = (u[2i] + 2^64 u[2i+1]) mod p_l over stream (public_seed(seed), 2, g*L + l),
    computed with Python integers.  A short word (u[2i] alone), a wrong stream index or the private
    seed as key would all fail."""
    P = P4096 if NL[0] == 4096 else P8192
    tile = (16, 32, 8) if P.N == 4096 else (32, 16, 16)
    X = synth.activations(41, 2 * tile[2], 2 * tile[1])        # nJ = nK = 2: g = 0..3
    seed = 0x5EED
    ct = ref.encrypt(P, tile, ref.keygen(P, 1), X, seed)
    a_seed = int(_lib_chacha_u64(seed, 10, 0, 1)[0])
    for J in range(2):
        for K in range(2):
            g = J * 2 + K
            for l, p in enumerate(P.primes):
                u = _lib_chacha_u64(a_seed, 2, g * P.L + l, 2 * P.N)
                want = [(int(u[2 * i]) + (int(u[2 * i + 1]) << 64)) % p for i in range(P.N)]
                assert [int(v) for v in ct[J, K, 1, l]] == want
                assert np.array_equal(ref.sample_a(P, a_seed, g, l), np.array(want, dtype=np.uint64))


def test_sample_a_uniform_chi_squared(P4096):
    """a mod p_l is uniform on [0, p_l): 64 equal-width buckets, chi^2_63 < 103.4 (p = 0.001), and
    the top bit of the 50-bit residues is set about (p - 2^49)/p of the time (a 64-bit or 32-bit
    reduction would skew both)."""
    for l, p in enumerate(P4096.primes):
        a = np.concatenate([ref.sample_a(P4096, 77, g, l) for g in range(8)]).astype(object)
        assert max(a) < p
        counts = np.bincount(np.array([(int(v) * 64) // p for v in a], dtype=np.int64), minlength=64)
        exp = len(a) / 64
        assert ((counts - exp) ** 2 / exp).sum() < 103.4
        top = sum(1 for v in a if int(v) >= (1 << 49)) / len(a)
        assert abs(top - (p - (1 << 49)) / p) < 0.02


def test_sample_e_is_the_error_stream(P4096):
    """O4 + C8 recomputed: e[i] = sign(u) * min{k : (u & (2^63-1)) < T[k]} over the library ChaCha20
    stream (seed, 3, g) keyed by the PRIVATE seed (C28); T is the closed-form-pinned CDT table."""
    T = np.array(ref.cdt_table(), dtype=np.uint64)
    for seed, g in ((99, 0), (99, 17), (2**63 + 5, 3)):
        u = _lib_chacha_u64(seed, 3, g, P4096.N)
        mag = np.array([int(np.searchsorted(T, v & np.uint64((1 << 63) - 1), side="right")) for v in u])
        want = np.where((u >> np.uint64(63)) != 0, -mag, mag)
        assert np.array_equal(ref.sample_e(P4096, seed, g), want)
    # the encryption noise is that stream: fresh ct decrypts to Delta*b + e exactly (below)


def test_psi_matches_appendix_a(P4096, P8192):
    """psi_l = g_l^((p_l - 1)/2N) with g_l the SMALLEST primitive root (reading C26).  The N=4096
    values are the ones SURVEY.md Appendix A prints; g_l itself is re-derived here from the
    factorisation of p - 1 (g is a primitive root iff g^((p-1)/f) != 1 for every prime f | p-1) and
    no smaller g qualifies."""
    import sympy
    assert P4096.psis == (990116967873799, 702736788773885)
    for P, gens in ((P4096, (22, 10)), (P8192, (22, 10, 7))):
        for p, psi, g in zip(P.primes, P.psis, gens):
            fs = list(sympy.factorint(p - 1))
            is_gen = lambda x: all(pow(x, (p - 1) // f, p) != 1 for f in fs)
            assert is_gen(g) and not any(is_gen(x) for x in range(2, g))
            assert psi == pow(g, (p - 1) // (2 * P.N), p)


def test_encrypt_decrypt_roundtrip_exact_noise(P4096):
    """Fresh ct: c0 + c1*s = Delta*b + e exactly, so Dec = pi_B(X tile) and the measured
    noise equals the sampled error polynomial e (reading C8)."""
    P, tile = P4096, (16, 32, 8)
    X = synth.activations(11, 8, 64)
    sk = ref.keygen(P, 3)
    ct = ref.encrypt(P, tile, sk, X, 5)
    pts, noise = ref.decrypt_full(P, sk, ct)
    m, r, n = tile
    for J in range(2):
        g = J          # nK = 1
        b = ref.encode_B([[int(X[k, J * r + j]) for k in range(n)] for j in range(r)], P.N, m)
        assert pts[g] == b
        assert noise[g] == [int(v) for v in ref.sample_e(P, 5, g)]
    # encrypt(0) -> 0
    ct0 = ref.encrypt(P, tile, sk, np.zeros((8, 64), np.uint64), 6)
    pts0, _ = ref.decrypt_full(P, sk, ct0)
    assert all(v == 0 for row in pts0 for v in row)


def test_c1_travels_in_evaluation_form(P4096):
    """Reading C26: a ciphertext's c1 is carried as c1_hat[k] = c1(psi^(2k+1)) (natural k).  The
    fresh c1_hat is the evaluation, by the defining O(N^2) sum, of the polynomial a with
    c0 + a*s = e + Delta*b over the schoolbook product, and decryption of the response is
    unchanged (the response's c1_hat evaluates sum_J pi_A * a_J)."""
    P, tile = P4096, (16, 32, 8)
    X = synth.activations(61, 8, 64)
    sk = ref.keygen(P, 62)
    ct = ref.encrypt(P, tile, sk, X, 63)
    e = ref.sample_e(P, 63, 0)
    b = ref.encode_B([[int(X[k, j]) for k in range(8)] for j in range(32)], P.N, 16)
    for l, (p, psi) in enumerate(zip(P.primes, P.psis)):
        a_hat = ct[0, 0, 1, l]
        a = ref.intt(P.N, p, psi, a_hat)
        assert np.array_equal(ref.ntt_naive(P.N, p, psi, a), a_hat)      # the defining sum
        s_l = np.array([int(v) % p for v in sk], dtype=np.uint64)
        lhs = (ct[0, 0, 0, l].astype(object) + ref.negacyclic_mul(P.N, p, a, s_l).astype(object)) % p
        rhs = [(int(ev) + P.delta_mod[l] * bv) % p for ev, bv in zip(e, b)]
        assert [int(v) for v in lhs] == rhs


def test_he_matmul_homomorphism_and_noise(P4096):
    """Dec(he_matmul) = [sum_J pi_A(A_IJ) * pi_B(B_JK)]_t over Z and the
    noise fits the Appendix C bound 2R*max|w|*(r_t + e_max) < Delta/2."""
    P, tile = P4096, (16, 32, 8)
    m, r, n = tile
    X = synth.activations(21, 8, 64)
    W = synth.stressed_weights(22, 64, 32, bound=1500)
    sk = ref.keygen(P, 23)
    ct_in = ref.encrypt(P, tile, sk, X, 24)
    ct_out = ref.he_matmul(P, tile, W, ct_in, 8)
    pts, noise = ref.decrypt_full(P, sk, ct_out)
    lift = lambda w: int(w) - (1 << 37) if int(w) >= (1 << 36) else int(w)
    nI, nJ, nK = ref.tile_counts(tile, 32, 64, 8)
    maxw = max(abs(lift(w)) for w in W.reshape(-1))
    bound = 2 * 64 * maxw * (P.r_t + 41)
    assert bound < P.delta // 2
    for I in range(nI):
        acc = [0] * P.N
        for J in range(nJ):
            A = [[lift(W[J * r + j, I * m + i]) for j in range(r)] for i in range(m)]
            B = [[int(X[k, J * r + j]) for k in range(n)] for j in range(r)]
            prod = ref.negacyclic_mul_int(ref.encode_A(A, P.N, r), ref.encode_B(B, P.N, m), P.N)
            acc = [u + v for u, v in zip(acc, prod)]
        assert pts[I * nK] == [v % P.t for v in acc]
        assert max(abs(v) for v in noise[I * nK]) < bound


def test_he_matmul_schoolbook_equals_oracle_ntt(P4096):
    P, tile = P4096, (16, 8, 32)
    Nb, R, Ma = 40, 24, 40          # ragged: nI=3, nJ=3, nK=2, partial tiles everywhere
    ct_in = synth.uniform_below(31, (3, 2, 2, P.L, P.N), P.primes)
    W = synth.weights(32, R, Ma)
    sb = ref.he_matmul(P, tile, W, ct_in, Nb)
    tiles = [(I, K) for I in range(3) for K in range(2)]
    nt = ref.he_matmul_ntt_tiles(P, tile, W, ct_in, Nb, tiles)
    for o, (I, K) in enumerate(tiles):
        assert np.array_equal(sb[I, K], nt[o])


# ------------------------------------------------------------------------------ end to end (Alg. 1; O7-O11)
@pytest.mark.parametrize("shape,tile,compress", [
    ((8, 64, 64), (16, 32, 8), True),      # config c0
    ((8, 64, 64), (16, 32, 8), False),
    ((5, 37, 19), (4, 8, 4), True),        # ragged in every dimension
    ((3, 1, 2), (1, 1, 1), True),          # degenerate 1x1x1 tile
])
def test_protocol_reconstructs_XW_mod_t(P4096, shape, tile, compress):
    Nb, R, Ma = shape
    X = synth.activations(41, Nb, R)
    W = synth.weights(42, R, Ma)
    out = ref.matmul_protocol(P4096, tile, X, W, 43, 44, 45, compress)
    got = (out["share_client"] + out["share_server"]) & np.uint64((1 << 37) - 1)
    assert np.array_equal(got, ref.matmul_mod_t(X, W))


def test_compressed_decrypt_equals_full_and_size(P4096):
    P, tile = P4096, (16, 32, 8)
    m, r, n = tile
    X = synth.activations(51, 8, 64)
    W = synth.weights(52, 64, 64)
    sk = ref.keygen(P, 53)
    ct_out = ref.he_matmul(P, tile, W, ref.encrypt(P, tile, sk, X, 54), 8)
    mc, sc = ref.mask_and_share(P, tile, ct_out, 64, 8, 55, True)
    mf, sf = ref.mask_and_share(P, tile, ct_out, 64, 8, 55, False)
    assert np.array_equal(sc, sf)
    assert np.array_equal(ref.decrypt_share(P, tile, sk, mc, 64, 8, True),
                          ref.decrypt_share(P, tile, sk, mf, 64, 8, False))
    # response size ratio (N + m*n) / 2N exactly ("roughly reduces half")
    assert mc.shape[-1] * 2 * P.N == mf.shape[-1] * (P.N + m * n)


@pytest.mark.parametrize("tile", [(16, 8, 32), (4, 32, 32), (8, 8, 64), (16, 32, 8), (1, 1, 1), (32, 16, 16)])
def test_mask_word_order(P4096, tile):
    """Reading C27: the mask word order is a permutation of [0, N) that puts the kept positions
    pos(i,k) first, at word k*m + i, and the other positions after it in increasing order."""
    m, r, n = tile
    N = 8192 if m * r * n > 4096 else 4096
    words = [ref.mask_word(tile, p) for p in range(N)]
    assert sorted(words) == list(range(N))
    for k in range(n):
        for i in range(m):
            assert words[(k * m + i) * r + r - 1] == k * m + i
    rest = [w for p, w in enumerate(words) if w >= m * n]
    assert rest == sorted(rest)


def test_mask_share_is_the_stream_prefix(P4096):
    """Reading C27 end to end: the server share of output ciphertext (I, K) is the first m*n words
    of its MASK stream (library ChaCha20, pinned above), masked to 37 bits, in kept-index order."""
    P, tile, (Nb, Ma) = P4096, (16, 8, 32), (64, 32)
    m, r, n = tile
    nI, _, nK = ref.tile_counts(tile, Ma, 1, Nb)
    ct = synth.uniform_below(71, (nI, nK, 2, P.L, P.N), P.primes)
    _, share = ref.mask_and_share(P, tile, ct, Ma, Nb, 72, True)
    for I in range(nI):
        for K in range(nK):
            w = ref.prf_u64(72, ref.DOM_MASK, I * nK + K, m * n) & np.uint64((1 << 37) - 1)
            for k in range(n):
                for i in range(m):
                    assert share[K * n + k, I * m + i] == w[k * m + i]


def test_mask_uniform_chi_squared(P4096):
    """The server share is the mask at the decoded positions: uniform on Z_{2^37}."""
    P, tile = P4096, (16, 8, 32)
    ct = synth.uniform_below(61, (4, 4, 2, P.L, P.N), P.primes)
    _, share = ref.mask_and_share(P, tile, ct, 64, 128, 62, True)
    top = (share >> np.uint64(33)).astype(np.int64).reshape(-1)     # 16 buckets of the top 4 bits
    counts = np.bincount(top, minlength=16)
    exp = len(top) / 16
    chi2 = ((counts - exp) ** 2 / exp).sum()
    assert chi2 < 37.7        # chi^2_{15} at p = 0.001


# ----------------------------------------------------------------------------- FC layer (row f1)
@pytest.mark.parametrize("shape,tile", [((8, 64, 64), (16, 32, 8)), ((5, 24, 40), (16, 8, 32))])
def test_fc_protocol_reconstructs_XW_plus_b(P4096, shape, tile):
    """with x = <x>_0 + <x>_1, the client's decrypted Pi_MatMul share of
    W<x>_0 plus the server's <W<x>_0>_1 + W<x>_1 + b reconstruct W x + b (mod 2^l) -- checked
    against brute force with Python integers (no numpy wrapping)."""
    import synth
    Nb, R, Ma = shape
    X = synth.activations(71, Nb, R)
    X1 = synth.activations(72, Nb, R)           # the server's share: uniform, independent of X
    W = synth.weights(73, R, Ma)
    b = synth.activations(74, 1, Ma)[0]
    sc, ss = ref.fc_protocol(P4096, tile, X, X1, W, b, 75, 76, 77)
    t = 1 << 37
    for i in range(Nb):
        for j in range(Ma):
            want = (sum(int(X[i, k]) * int(W[k, j]) for k in range(R)) + int(b[j])) % t
            assert (int(sc[i, j]) + int(ss[i, j])) % t == want


def test_fc_server_share_special_cases(P4096):
    """X1 = 0 and b = 0 leave the HE share unchanged; the local term is X1.W mod 2^37 (Python
    integers) and the bias is added per output column."""
    import synth
    S = synth.activations(81, 4, 6)
    X1 = synth.activations(82, 4, 3)
    W = synth.weights(83, 3, 6)
    b = synth.activations(84, 1, 6)[0]
    assert np.array_equal(ref.fc_server_share(S, np.zeros_like(X1), W, None), S)
    got = ref.fc_server_share(S, X1, W, b)
    for i in range(4):
        for j in range(6):
            want = (int(S[i, j]) + sum(int(X1[i, k]) * int(W[k, j]) for k in range(3)) + int(b[j])) % (1 << 37)
            assert int(got[i, j]) == want


# ----------------------------------------------------------------------------- attention (row f2)
def test_attention_cross_terms_reconstruct_XY(P8192):
    """PAPER.md:113-118 (Eq. 2): with X and Y both shared, two Pi_MatMul invocations on the cross
    terms plus each party's local product give shares of X.Y mod 2^l -- checked against brute
    force with Python integers.  Shares are uniform in Z_(2^37), so the server operand is not
    small: the N=8192, L=3 set (q ~ 2^150) keeps the noise below Delta/2."""
    import synth
    tile = (32, 16, 16)
    n, d = 24, 20                                   # Q K^T shape: (n x d) . (d x n)
    X0, X1 = synth.activations(61, n, d), synth.activations(62, n, d)
    Y0, Y1 = synth.activations(63, d, n), synth.activations(64, d, n)
    Z0, Z1 = ref.attention_protocol(P8192, tile, X0, X1, Y0, Y1)
    t = 1 << 37
    X = [[(int(X0[i, k]) + int(X1[i, k])) % t for k in range(d)] for i in range(n)]
    Y = [[(int(Y0[k, j]) + int(Y1[k, j])) % t for j in range(n)] for k in range(d)]
    for i in range(n):
        for j in range(n):
            assert (int(Z0[i, j]) + int(Z1[i, j])) % t == sum(X[i][k] * Y[k][j] for k in range(d)) % t


def test_attention_noise_needs_the_large_modulus(P4096):
    """At N=4096, L=2 (q ~ 2^100) a uniform 37-bit server operand breaks decryption (the
    r_t * K term of SURVEY Appendix C, ~2^75, exceeds Delta/2 ~ 2^62): the reconstruction fails,
    which is why row f2 uses the q ~ 2^150 parameter set."""
    import synth
    tile = (16, 8, 32)
    X0, X1 = synth.activations(65, 8, 24), synth.activations(66, 8, 24)
    Y0, Y1 = synth.activations(67, 24, 8), synth.activations(68, 24, 8)
    Z0, Z1 = ref.attention_protocol(P4096, tile, X0, X1, Y0, Y1)
    want = ref.matmul_mod_t((X0 + X1) & np.uint64((1 << 37) - 1), (Y0 + Y1) & np.uint64((1 << 37) - 1))
    assert not np.array_equal((Z0 + Z1) & np.uint64((1 << 37) - 1), want)


# ----------------------------------------------------------------------------- re-randomisation (row f4)
def test_rerandomized_response_reconstructs_and_floods(P4096):
    """Row f4 (reading C22): a fresh public-key encryption of zero plus a flooding term of
    fb = log2(Delta) - 3 bits keeps decryption exact (shares reconstruct X.W mod 2^37), and the
    decryption noise of the response is then dominated by the flood (|noise| ~ 2^(fb-1))."""
    import synth
    tile, (Nb, R, Ma) = (16, 8, 32), (24, 16, 40)
    X, W = synth.activations(101, Nb, R), synth.weights(102, R, Ma)
    sk = ref.keygen(P4096, 103)
    pk = ref.pk_gen(P4096, sk, 104)
    ct_in = ref.encrypt(P4096, tile, sk, X, 105)
    nI, nJ, nK = ref.tile_counts(tile, Ma, R, Nb)
    fb = int(np.floor(np.log2(float(P4096.delta)))) - 3
    ct = ref.rerandomize(P4096, tile, pk, ref.he_matmul(P4096, tile, W, ct_in, Nb), nK, 106, fb)
    masked, share_s = ref.mask_and_share(P4096, tile, ct, Ma, Nb, 106, True)
    share_c = ref.decrypt_share(P4096, tile, sk, masked, Ma, Nb, True)
    assert np.array_equal((share_c + share_s) & np.uint64((1 << 37) - 1), ref.matmul_mod_t(X, W))
    pts, noise = ref.decrypt_full(P4096, sk, ct[0, 0])
    assert max(abs(int(v)) for v in noise[0]) > 1 << (fb - 3)    # flood-sized, not HE-noise-sized


def test_rerandomization_defeats_weight_recovery(P4096):
    """Without re-randomisation (the paper's Alg. 1 as stated, reading C13) the client recovers W
    from the response: with nJ = 1, c1_out = pi_A(W) * a in R_q, so NTT(pi_A(W)) = NTT(c1_out)/NTT(a)
    coefficient-wise.  After re-randomisation the same computation no longer yields pi_A(W)."""
    import synth
    tile, (Nb, R, Ma) = (16, 8, 32), (32, 8, 16)          # nI = nJ = nK = 1
    X, W = synth.activations(111, Nb, R), synth.weights(112, R, Ma)
    sk = ref.keygen(P4096, 113)
    ct_in = ref.encrypt(P4096, tile, sk, X, 114)
    ct_out = ref.he_matmul(P4096, tile, W, ct_in, Nb)
    pk = ref.pk_gen(P4096, sk, 115)
    ct_rr = ref.rerandomize(P4096, tile, pk, ct_out, 1, 116, 0)
    p, psi, N = P4096.primes[0], P4096.psis[0], P4096.N
    a_hat = ct_in[0, 0, 1, 0]                   # c1 travels in evaluation form (reading C26)
    inv = np.array([pow(int(v), p - 2, p) for v in a_hat], dtype=object)

    def recover(c_hat):
        return ref.intt(N, p, psi, np.array([(int(x) * int(y)) % p for x, y in zip(c_hat, inv)], dtype=np.uint64))

    wpoly = ref.encode_A([[int(W[j, i]) for j in range(R)] for i in range(Ma)], N, tile[1])
    lift = np.array([(int(v) - (1 << 37)) % p if int(v) >= (1 << 36) else int(v) for v in wpoly], dtype=np.uint64)
    assert np.array_equal(recover(ct_out[0, 0, 1, 0]), lift)            # the leak: pi_A(W) mod p, centered lift
    assert not np.array_equal(recover(ct_rr[0, 0, 1, 0]), lift)         # closed
