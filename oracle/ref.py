"""CPU ORACLE for the server-side homomorphic linear layer (arxiv 2305.18396, Alg. 1).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this module.  It never imports the
CUDA package (paper_2305_18396_b200) and shares no code, table or constant generator
with it; the only shared module is `synth` (seeded input generation, no HE arithmetic).

Heavy loops live in oracle.c (plain C, exact `unsigned __int128` arithmetic); this file
holds parameter derivation with Python integers, the CDT table with mpmath, the CRT and
rounding of decryption with Python integers, and pure-Python encoders for tiny cases.

Every function cites the passage it follows.  Readings of silent/ambiguous passages are
SURVEY.md §8(c) C1-C21, restated in DESIGN.md §3.

Parity status per function (DESIGN.md §3 lists the pins):
  params/primes/Delta      pinned (closed form, independent Miller-Rabin in tests)
  chacha20 / prf           pinned (cryptography's ChaCha20)
  keygen / sample_a /      pinned (each stream recomputed from cryptography's ChaCha20 with the
    sample_e / public_seed   formula of O3/O4/C28; chi-squared uniformity of a mod p_l)
  cdt_table                pinned (closed-form moments, monotonicity, tail)
  encode_A/B, decode_C     pinned (SPEC.md worked values; brute-force matmul)
  negacyclic products/NTT  pinned (special cases, schoolbook vs NTT vs numpy fold)
  encrypt/decrypt          pinned (round trip, enc(0), homomorphism)
  he_matmul                pinned (decrypt = sum_J a_IJ*b_JK over Z; reconstruction)
  mask_and_share           pinned (reconstruction = X.W mod 2^37; compressed = full)
  exact ciphertext coefficient values: parity unpinned by the paper (depend on the
    randomness choices C4-C12); pinned only by the invariants above.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

DOM_SK, DOM_A, DOM_E, DOM_MASK = 1, 2, 3, 4   # PRF domains
DOM_PUB = 10                                  # public-seed derivation (reading C28)
SIGMA = 3.2                                   # error std (BASELINE.json)
CDT_TAIL = 41                                 # support [-41, 41]  (reading C8)


# ----------------------------------------------------------------------------------------
# build / load the C part
# ----------------------------------------------------------------------------------------
def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, OpenMP over output tiles)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", _SRC, "-o", _LIB_PATH])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        L.or_chacha20_block.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint32,
                                        ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]
        L.or_prf_u64.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_uint64, u64p]
        L.or_mask_word.restype = ctypes.c_uint64
        L.or_public_seed.restype = ctypes.c_uint64
        L.or_public_seed.argtypes = [ctypes.c_uint64]
        _lib = L
    return _lib


def _p(a: np.ndarray, ctype=ctypes.c_uint64):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def _u64arr(xs) -> np.ndarray:
    return np.ascontiguousarray(np.array(xs, dtype=np.uint64))


# ----------------------------------------------------------------------------------------
# O1: parameters  ("{N, t, q}", t = 2^l; readings C4, C5)
# ----------------------------------------------------------------------------------------
def _is_prime(n: int) -> bool:
    import sympy
    return bool(sympy.isprime(n))


def ntt_primes(N: int, L: int, bits: int = 50) -> list:
    """The L largest primes p < 2^bits with p = 1 (mod 2N), descending (reading C4)."""
    out, p = [], ((1 << bits) - 1) // (2 * N) * (2 * N) + 1
    while len(out) < L:
        if p < (1 << bits) and _is_prime(p):
            out.append(p)
        p -= 2 * N
    return out


def primitive_2n_root(p: int, N: int) -> int:
    """Smallest generator g of Z_p^*, psi = g^((p-1)/2N): a primitive 2N-th root of unity."""
    import sympy
    g = int(sympy.primitive_root(p))
    return pow(g, (p - 1) // (2 * N), p)


@dataclass(frozen=True)
class Params:
    N: int
    L: int
    t_bits: int
    primes: tuple
    psis: tuple

    @property
    def t(self) -> int:
        return 1 << self.t_bits

    @property
    def q(self) -> int:
        q = 1
        for p in self.primes:
            q *= p
        return q

    @property
    def delta(self) -> int:          # Delta = floor(q / t)   (reading C5)
        return self.q // self.t

    @property
    def delta_mod(self) -> list:
        return [self.delta % p for p in self.primes]

    @property
    def r_t(self) -> int:
        return self.q % self.t


def bfv_params(N: int = 4096, L: int = 2, t_bits: int = 37, primes=None) -> Params:
    primes = tuple(int(p) for p in (primes if primes is not None else ntt_primes(N, L)))
    psis = tuple(primitive_2n_root(p, N) for p in primes)
    return Params(N, L, t_bits, primes, psis)


# ----------------------------------------------------------------------------------------
# O2: PRF = ChaCha20 block function (RFC 8439 §2.3) -- reading C10
# ----------------------------------------------------------------------------------------
def chacha20_block(key: bytes, counter: int, nonce: bytes) -> bytes:
    k = np.frombuffer(key, dtype="<u4").astype(np.uint32).copy()
    nn = np.frombuffer(nonce, dtype="<u4").astype(np.uint32).copy()
    out = np.zeros(16, dtype=np.uint32)
    lib().or_chacha20_block(_p(k, ctypes.c_uint32), counter, _p(nn, ctypes.c_uint32), _p(out, ctypes.c_uint32))
    return out.astype("<u4").tobytes()


def prf_u64(seed: int, domain: int, stream: int, count: int, first: int = 0) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint64)
    lib().or_prf_u64(seed, domain, stream, first, count, _p(out))
    return out


# ----------------------------------------------------------------------------------------
# CDT table of the discrete Gaussian (reading C8)
# ----------------------------------------------------------------------------------------
def cdt_table(sigma: float = SIGMA, tail: int = CDT_TAIL) -> list:
    """T[k] = floor(2^63 * P(|E| <= k)), P(E = k) ~ exp(-k^2 / (2 sigma^2)) on [-tail, tail]."""
    import mpmath
    mpmath.mp.dps = 60
    s = mpmath.mpf(str(sigma))   # the decimal 3.2, not the binary double nearest to it
    rho = [mpmath.e ** (-(mpmath.mpf(k) ** 2) / (2 * s * s)) for k in range(tail + 1)]
    Z = rho[0] + 2 * sum(rho[1:])
    T, acc = [], mpmath.mpf(0)
    for k in range(tail + 1):
        acc += rho[0] if k == 0 else 2 * rho[k]
        T.append(int(mpmath.floor(mpmath.mpf(2) ** 63 * acc / Z)))
    T[tail] = 1 << 63      # P(|E| <= tail) = 1 exactly
    return T


# ----------------------------------------------------------------------------------------
# tile counts (reading C2: explicit (m, r, n), zero padding of partial tiles)
# ----------------------------------------------------------------------------------------
def tile_counts(tile, Ma: int, R: int, Nb: int):
    m, r, n = tile
    return -(-Ma // m), -(-R // r), -(-Nb // n)


def mask_word(tile, pos: int) -> int:
    """Reading C27: index of the MASK-stream word used at coefficient position pos (kept
    positions first, in kept-index order; the others after, in position order)."""
    m, r, n = tile
    return int(lib().or_mask_word(ctypes.c_uint32(m), ctypes.c_uint32(r), ctypes.c_uint32(n), ctypes.c_uint64(pos)))


def kept_positions(tile) -> list:
    """pos(i,k) = k*m*r + i*r + r-1 in index order k*m + i (reading C12)."""
    m, r, n = tile
    return [k * m * r + i * r + r - 1 for k in range(n) for i in range(m)]


# ----------------------------------------------------------------------------------------
# pure-Python encoders (tiny cases)
# ----------------------------------------------------------------------------------------
def encode_A(A, N: int, r: int) -> list:
    """pi_A: a = sum_ij A[i][j] x^(i*r + r-1-j)  (Alg. 1 step 1)."""
    a = [0] * N
    for i, row in enumerate(A):
        for j, v in enumerate(row):
            a[i * r + r - 1 - j] += int(v)
    return a


def encode_B(B, N: int, m: int) -> list:
    """pi_B: b = sum_jk B[j][k] x^(k*m*r + j)  (Alg. 1 step 1)."""
    r = len(B)
    b = [0] * N
    for j, row in enumerate(B):
        for k, v in enumerate(row):
            b[k * m * r + j] += int(v)
    return b


def decode_C(c, m: int, r: int, n: int) -> list:
    """pi_C^-1: C[i][k] = c[k*m*r + i*r + r-1]  (Alg. 1 step 4)."""
    return [[c[k * m * r + i * r + r - 1] for k in range(n)] for i in range(m)]


def negacyclic_mul_int(a, b, N: int, mod=None) -> list:
    """Schoolbook product in Z[X]/(X^N+1) (optionally reduced mod `mod`), pure Python."""
    out = [0] * N
    for i, ai in enumerate(a):
        if ai == 0:
            continue
        for j, bj in enumerate(b):
            if i + j < N:
                out[i + j] += ai * bj
            else:
                out[i + j - N] -= ai * bj
    return [x % mod for x in out] if mod else out


# ----------------------------------------------------------------------------------------
# C-backed pieces
# ----------------------------------------------------------------------------------------
def keygen(P: Params, seed: int) -> np.ndarray:
    """O3: s_i = (u64_SK[i] mod 3) - 1  (reading C7: ternary secret)."""
    sk = np.zeros(P.N, dtype=np.int8)
    lib().or_keygen(ctypes.c_uint32(P.N), ctypes.c_uint64(seed), _p(sk, ctypes.c_int8))
    return sk


def public_seed(seed: int) -> int:
    """Reading C28: the public seed of the A domain, u64 word 0 of stream (seed, PUB, 0).  A seeded
    upload (c1 regenerated by the server) ships this value, never `seed`, which keys the errors."""
    return int(lib().or_public_seed(ctypes.c_uint64(seed)))


def sample_a(P: Params, a_seed: int, g: int, l: int) -> np.ndarray:
    """O4: a_hat_l[i] = (u64_A[2i] + 2^64 u64_A[2i+1]) mod p_l, stream g*L + l, key a_seed (C28)."""
    a = np.zeros(P.N, dtype=np.uint64)
    lib().or_sample_a(ctypes.c_uint32(P.N), ctypes.c_uint64(a_seed), ctypes.c_uint64(g), ctypes.c_uint32(l),
                      ctypes.c_uint32(P.L), ctypes.c_uint64(P.primes[l]), _p(a))
    return a


def sample_e(P: Params, seed: int, g: int) -> np.ndarray:
    T = _u64arr(cdt_table())
    e = np.zeros(P.N, dtype=np.int64)
    lib().or_sample_e(ctypes.c_uint32(P.N), ctypes.c_uint64(seed), ctypes.c_uint64(g), _p(T),
                      ctypes.c_int(len(T)), _p(e, ctypes.c_int64))
    return e


def negacyclic_mul(N: int, p: int, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a, b = _u64arr(a), _u64arr(b)
    out = np.zeros(N, dtype=np.uint64)
    lib().or_negacyclic_mul(ctypes.c_uint32(N), ctypes.c_uint64(p), _p(a), _p(b), _p(out))
    return out


def ntt(N: int, p: int, psi: int, a) -> np.ndarray:
    a = _u64arr(a); out = np.zeros(N, dtype=np.uint64)
    lib().or_ntt(ctypes.c_uint32(N), ctypes.c_uint64(p), ctypes.c_uint64(psi), _p(a), _p(out))
    return out


def ntt_naive(N: int, p: int, psi: int, a) -> np.ndarray:
    a = _u64arr(a); out = np.zeros(N, dtype=np.uint64)
    lib().or_ntt_naive(ctypes.c_uint32(N), ctypes.c_uint64(p), ctypes.c_uint64(psi), _p(a), _p(out))
    return out


def intt(N: int, p: int, psi: int, a) -> np.ndarray:
    a = _u64arr(a); out = np.zeros(N, dtype=np.uint64)
    lib().or_intt(ctypes.c_uint32(N), ctypes.c_uint64(p), ctypes.c_uint64(psi), _p(a), _p(out))
    return out


def negacyclic_mul_ntt(N: int, p: int, psi: int, a, b) -> np.ndarray:
    a, b = _u64arr(a), _u64arr(b)
    out = np.zeros(N, dtype=np.uint64)
    lib().or_negacyclic_mul_ntt(ctypes.c_uint32(N), ctypes.c_uint64(p), ctypes.c_uint64(psi),
                                _p(a), _p(b), _p(out))
    return out


def encrypt(P: Params, tile, sk: np.ndarray, X: np.ndarray, seed: int) -> np.ndarray:
    """O4: pi_B tiles of X^T, secret-key BFV: c1 = a, c0 = -a*s + e + Delta*b (mod p_l); a keyed by
    public_seed(seed), e by seed (reading C28).
    Returns ct_in uint64 [nJ][nK][2][L][N]."""
    m, r, n = tile
    Nb, R = X.shape
    _, nJ, nK = tile_counts(tile, 1, R, Nb)
    X = np.ascontiguousarray(X, dtype=np.uint64)
    ct = np.zeros((nJ, nK, 2, P.L, P.N), dtype=np.uint64)
    T = _u64arr(cdt_table())
    lib().or_encrypt(ctypes.c_uint32(P.N), ctypes.c_uint32(P.L), _p(_u64arr(P.primes)), _p(_u64arr(P.psis)),
                     _p(_u64arr(P.delta_mod)), ctypes.c_uint32(m), ctypes.c_uint32(r),
                     ctypes.c_uint32(n), _p(X), ctypes.c_int64(Nb), ctypes.c_int64(R),
                     _p(np.ascontiguousarray(sk), ctypes.c_int8), ctypes.c_uint64(seed), _p(T),
                     ctypes.c_int(len(T)), _p(ct))
    return ct


def he_matmul(P: Params, tile, W: np.ndarray, ct_in: np.ndarray, Nb: int) -> np.ndarray:
    """O6 / definition (i): ct_out[I][K][c] = sum_J pi_A(W^T tile IJ) * ct_in[J][K][c].
    Returns uint64 [nI][nK][2][L][N] (sparse schoolbook)."""
    m, r, n = tile
    R, Ma = W.shape
    nI, nJ, nK = tile_counts(tile, Ma, R, Nb)
    assert ct_in.shape == (nJ, nK, 2, P.L, P.N), ct_in.shape
    out = np.zeros((nI, nK, 2, P.L, P.N), dtype=np.uint64)
    lib().or_he_matmul(ctypes.c_uint32(P.N), ctypes.c_uint32(P.L), _p(_u64arr(P.primes)), _p(_u64arr(P.psis)),
                       ctypes.c_uint32(m), ctypes.c_uint32(r), ctypes.c_uint32(n),
                       ctypes.c_uint32(P.t_bits), _p(np.ascontiguousarray(W, dtype=np.uint64)),
                       ctypes.c_int64(R), ctypes.c_int64(Ma), ctypes.c_int64(Nb),
                       _p(np.ascontiguousarray(ct_in)), _p(out))
    return out


def he_matmul_ntt_tiles(P: Params, tile, W: np.ndarray, ct_in: np.ndarray, Nb: int, tiles) -> np.ndarray:
    """Definition (i) through the oracle's scalar NTT, only for output tiles [(I, K), ...].
    Returns uint64 [len(tiles)][2][L][N]."""
    m, r, n = tile
    R, Ma = W.shape
    tl = np.ascontiguousarray(np.array(tiles, dtype=np.int64).reshape(-1, 2))
    out = np.zeros((len(tl), 2, P.L, P.N), dtype=np.uint64)
    lib().or_he_matmul_ntt_tiles(ctypes.c_uint32(P.N), ctypes.c_uint32(P.L), _p(_u64arr(P.primes)),
                                 _p(_u64arr(P.psis)), ctypes.c_uint32(m), ctypes.c_uint32(r),
                                 ctypes.c_uint32(n), ctypes.c_uint32(P.t_bits),
                                 _p(np.ascontiguousarray(W, dtype=np.uint64)), ctypes.c_int64(R),
                                 ctypes.c_int64(Ma), ctypes.c_int64(Nb), _p(np.ascontiguousarray(ct_in)),
                                 _p(tl, ctypes.c_int64), ctypes.c_int64(len(tl)), _p(out))
    return out


def mask_and_share(P: Params, tile, ct_out: np.ndarray, Ma: int, Nb: int, seed: int, compress: bool = True):
    """O7-O9: c0 -= Delta_l*sigma, drop unused c0, server share S[Nb][Ma]."""
    m, r, n = tile
    nI, _, nK = tile_counts(tile, Ma, 1, Nb)
    per = P.L * (m * n + P.N) if compress else 2 * P.L * P.N
    masked = np.zeros((nI, nK, per), dtype=np.uint64)
    share = np.zeros((Nb, Ma), dtype=np.uint64)
    lib().or_mask_and_share(ctypes.c_uint32(P.N), ctypes.c_uint32(P.L), _p(_u64arr(P.primes)),
                            _p(_u64arr(P.delta_mod)), ctypes.c_uint32(P.t_bits), ctypes.c_uint32(m),
                            ctypes.c_uint32(r), ctypes.c_uint32(n), ctypes.c_int64(Ma), ctypes.c_int64(Nb),
                            _p(np.ascontiguousarray(ct_out)), ctypes.c_uint64(seed), ctypes.c_int(int(compress)),
                            _p(masked), _p(share))
    return masked, share


def mask_tiles(P: Params, tile, ct: np.ndarray, nK: int, tiles, seed: int, compress: bool = True):
    """O7-O9 for selected output tiles [(I, K), ...] (global I): ct [ntiles][2][L][N] ->
    (masked [ntiles][per_ct], sigma at the kept positions [ntiles][m*n], index k*m+i)."""
    m, r, n = tile
    tl = np.ascontiguousarray(np.array(tiles, dtype=np.int64).reshape(-1, 2))
    per = P.L * (m * n + P.N) if compress else 2 * P.L * P.N
    masked = np.zeros((len(tl), per), dtype=np.uint64)
    kept = np.zeros((len(tl), m * n), dtype=np.uint64)
    lib().or_mask_tiles(ctypes.c_uint32(P.N), ctypes.c_uint32(P.L), _p(_u64arr(P.primes)),
                        _p(_u64arr(P.delta_mod)), ctypes.c_uint32(P.t_bits), ctypes.c_uint32(m),
                        ctypes.c_uint32(r), ctypes.c_uint32(n), ctypes.c_int64(nK),
                        _p(np.ascontiguousarray(ct)), _p(tl, ctypes.c_int64), ctypes.c_int64(len(tl)),
                        ctypes.c_uint64(seed), ctypes.c_int(int(compress)), _p(masked), _p(kept))
    return masked, kept


def crt_round(P: Params, residues) -> int:
    """O10: x = CRT(residues) in [0, q); y = floor((t*x + floor(q/2)) / q) mod t."""
    q = P.q
    x = 0
    for xl, p in zip(residues, P.primes):
        Ml = q // p
        x += int(xl) * Ml * pow(Ml, -1, p)
    x %= q
    return ((P.t * x + q // 2) // q) % P.t


def decrypt_share(P: Params, tile, sk: np.ndarray, masked: np.ndarray, Ma: int, Nb: int,
                  compress: bool = True) -> np.ndarray:
    """O10: client share C0[K*n+k][I*m+i] = Dec(masked ct)[pos(i,k)]  (Alg. 1 step 4)."""
    m, r, n = tile
    nI, _, nK = tile_counts(tile, Ma, 1, Nb)
    x = np.zeros((nI, nK, P.L, m * n), dtype=np.uint64)
    lib().or_decrypt_residues(ctypes.c_uint32(P.N), ctypes.c_uint32(P.L), _p(_u64arr(P.primes)),
                              _p(_u64arr(P.psis)), ctypes.c_uint32(m), ctypes.c_uint32(r), ctypes.c_uint32(n),
                              ctypes.c_int64(Ma), ctypes.c_int64(Nb), _p(np.ascontiguousarray(sk), ctypes.c_int8),
                              _p(np.ascontiguousarray(masked)), ctypes.c_int(int(compress)), _p(x))
    out = np.zeros((Nb, Ma), dtype=np.uint64)
    for I in range(nI):
        for K in range(nK):
            for k in range(n):
                row = K * n + k
                if row >= Nb:
                    continue
                for i in range(m):
                    col = I * m + i
                    if col >= Ma:
                        continue
                    out[row, col] = crt_round(P, x[I, K, :, k * m + i])
    return out


def decrypt_full(P: Params, sk: np.ndarray, ct: np.ndarray):
    """Decrypt every coefficient of full ciphertexts [nct][2][L][N]; returns
    (plaintexts [nct][N] as Python ints mod t, centered noise [nct][N] as Python ints)."""
    nct = ct.reshape(-1, 2, P.L, P.N).shape[0]
    x = np.zeros((nct, P.L, P.N), dtype=np.uint64)
    lib().or_decrypt_full_residues(ctypes.c_uint32(P.N), ctypes.c_uint32(P.L), _p(_u64arr(P.primes)),
                                   _p(_u64arr(P.psis)), _p(np.ascontiguousarray(sk), ctypes.c_int8),
                                   _p(np.ascontiguousarray(ct.reshape(-1))), ctypes.c_int64(nct), _p(x))
    q, t, D = P.q, P.t, P.delta
    pts, noise = [], []
    Ms = [(q // p) * pow(q // p, -1, p) for p in P.primes]
    for o in range(nct):
        row_pt, row_nz = [], []
        for k in range(P.N):
            xv = sum(int(x[o, l, k]) * Ms[l] for l in range(P.L)) % q
            y = ((t * xv + q // 2) // q) % t
            v = (xv - D * y) % q
            if v > q // 2:
                v -= q
            row_pt.append(y)
            row_nz.append(v)
        pts.append(row_pt)
        noise.append(row_nz)
    return pts, noise


# ----------------------------------------------------------------------------------------
# end-to-end protocol (Alg. 1) for one matmul, all on the oracle
# ----------------------------------------------------------------------------------------
def matmul_protocol(P: Params, tile, X: np.ndarray, W: np.ndarray, key_seed: int, enc_seed: int,
                    mask_seed: int, compress: bool = True):
    """Client share, server share and all intermediates of Pi_MatMul(W^T, X^T) (reading C1)."""
    Nb, R = X.shape
    Ma = W.shape[1]
    sk = keygen(P, key_seed)
    ct_in = encrypt(P, tile, sk, X, enc_seed)
    ct_out = he_matmul(P, tile, W, ct_in, Nb)
    masked, share_s = mask_and_share(P, tile, ct_out, Ma, Nb, mask_seed, compress)
    share_c = decrypt_share(P, tile, sk, masked, Ma, Nb, compress)
    return dict(sk=sk, ct_in=ct_in, ct_out=ct_out, masked=masked, share_server=share_s,
                share_client=share_c)


def matmul_mod_t(X: np.ndarray, W: np.ndarray, t_bits: int = 37) -> np.ndarray:
    """Brute force (X.W) mod 2^t_bits with wrapping uint64 arithmetic (2^t | 2^64)."""
    with np.errstate(over="ignore"):
        acc = np.zeros((X.shape[0], W.shape[1]), dtype=np.uint64)
        for j in range(X.shape[1]):
            acc += np.outer(X[:, j].astype(np.uint64), W[j, :].astype(np.uint64))
    return acc & np.uint64((1 << t_bits) - 1)


# ----------------------------------------------------------------------------------------
# FC layer (§3.1.1 "fully connected layer"): with the input shared as
# x = <x>_0 + <x>_1 (client, server), the client's share of y = W x + b is the decrypted
# Pi_MatMul output <W<x>_0>_0 and the server's is <y>_1 = <W<x>_0>_1 + W<x>_1 + b.  In the
# layout of X.W (reading C1): Y = X W + b, server share = share_server + X1.W + b mod 2^t.
# ----------------------------------------------------------------------------------------
def fc_server_share(share_server: np.ndarray, X1: np.ndarray, W: np.ndarray, bias, t_bits: int = 37) -> np.ndarray:
    """<y>_1 = <W<x>_0>_1 + W<x>_1 + b, all mod 2^t_bits; bias per output
    column (broadcast over the Nb rows) or None."""
    out = share_server.astype(np.uint64) + matmul_mod_t(X1, W, 64 if t_bits >= 64 else t_bits)
    if bias is not None:
        with np.errstate(over="ignore"):
            out = out + np.asarray(bias, dtype=np.uint64)[None, :]
    return out & np.uint64((1 << t_bits) - 1)


def fc_protocol(P: Params, tile, X: np.ndarray, X1: np.ndarray, W: np.ndarray, bias, key_seed: int,
                enc_seed: int, mask_seed: int):
    """The FC protocol of PAPER.md:106-111 on the oracle: X = X0 + X1 mod 2^t with X0 the
    client's share; returns (client share, server share) of X.W + b."""
    tmask = np.uint64((1 << P.t_bits) - 1)
    with np.errstate(over="ignore"):
        X0 = (X.astype(np.uint64) - X1.astype(np.uint64)) & tmask
    r = matmul_protocol(P, tile, X0, W, key_seed, enc_seed, mask_seed, True)
    return r["share_client"], fc_server_share(r["share_server"], X1, W, bias, P.t_bits)


# ----------------------------------------------------------------------------------------
# Attention cross terms (Eq. 2): Z = X Y with both inputs shared,
# X = X0 + X1, Y = Y0 + Y1 (client 0, server 1).  Two Pi_MatMul invocations give shares of
# the cross terms X1 Y0 + X0 Y1 -- in the form of footnote 3 so that the client
# always encrypts: Pi_MatMul(Y0^T -> client, X1^T -> server) yields shares of (X1 Y0)^T, which
# both parties transpose -- and each party adds its local product (client X0 Y0, server X1 Y1).
# ----------------------------------------------------------------------------------------
def attention_protocol(P: Params, tile, X0: np.ndarray, X1: np.ndarray, Y0: np.ndarray, Y1: np.ndarray,
                       seeds=(1, 2, 3, 4, 5, 6)):
    """Returns (client share Z0, server share Z1) of Z = (X0+X1)(Y0+Y1) mod 2^t.
    tile: one (m, r, n) for both Pi_MatMul invocations, or a pair (term 1, term 2)."""
    tmask = np.uint64((1 << P.t_bits) - 1)
    tile1, tile2 = (tile[0], tile[1]) if isinstance(tile[0], (tuple, list)) else (tile, tile)
    # term 1: X1 Y0 = (Y0^T X1^T)^T -- client operand Y0^T, server operand X1^T
    t1 = matmul_protocol(P, tile1, np.ascontiguousarray(Y0.T), np.ascontiguousarray(X1.T), *seeds[0:3])
    # term 2: X0 Y1 -- client operand X0, server operand Y1
    t2 = matmul_protocol(P, tile2, X0, Y1, *seeds[3:6])
    with np.errstate(over="ignore"):
        Z0 = (t1["share_client"].T + t2["share_client"] + matmul_mod_t(X0, Y0, P.t_bits)) & tmask
        Z1 = (t1["share_server"].T + t2["share_server"] + matmul_mod_t(X1, Y1, P.t_bits)) & tmask
    return Z0, Z1


# ----------------------------------------------------------------------------------------
# Response re-randomisation (reading C22 of DESIGN.md).  The paper is
# silent (C13); without it the client, who knows its own c1 = a_J, learns sum_J pi_A(W_IJ) * a_J
# from the response's c1 and so W (linear algebra).  Standard fix: add a fresh public-key
# encryption of zero, c' = c + (pk0 u + e1 + F, pk1 u + e2), with u ternary, e1, e2 discrete
# Gaussian and F a uniform "flooding" term of flood_bits bits (|F| <= 2^(flood_bits-1)) that hides
# the W-dependent noise as far as the noise budget allows.
#   pk  = (pk0, pk1) = (-a s + e, a): a from PRF domain 5 (stream l), e from domain 6 (stream 0)
#   u   = (u64_RR_U[i] mod 3) - 1          domain 7, stream I*nK + K
#   e1, e2 = CDT(u64_RR_E)                  domain 8, streams 2(I*nK+K) and 2(I*nK+K)+1
#   F[i] = (u64_RR_F[i] mod 2^fb) - 2^(fb-1)  domain 9, stream I*nK + K  (F = 0 when fb = 0; fb <= 62)
# ----------------------------------------------------------------------------------------
DOM_PK_A, DOM_PK_E, DOM_RR_U, DOM_RR_E, DOM_RR_F = 5, 6, 7, 8, 9


def _cdt_sample(words: np.ndarray) -> np.ndarray:
    """Reading C8 on given PRF words: sign = u>>63, |e| = min{k : (u & (2^63-1)) < T[k]}."""
    T = np.array(cdt_table(), dtype=np.uint64)
    v = words & np.uint64((1 << 63) - 1)
    mag = np.searchsorted(T, v, side="right").astype(np.int64)
    return np.where((words >> np.uint64(63)) != 0, -mag, mag)


def _to_mod(v: np.ndarray, p: int) -> np.ndarray:
    return np.array([int(x) % p for x in v], dtype=np.uint64)


def pk_gen(P: Params, sk: np.ndarray, seed: int) -> np.ndarray:
    """Public key pk [2][L][N]: pk1 = a, pk0 = -a*s + e (mod p_l)."""
    N = P.N
    e = _cdt_sample(prf_u64(seed, DOM_PK_E, 0, N))
    pk = np.zeros((2, P.L, N), dtype=np.uint64)
    for l, p in enumerate(P.primes):
        u = prf_u64(seed, DOM_PK_A, l, 2 * N)
        a = np.array([(int(u[2 * i]) + (int(u[2 * i + 1]) << 64)) % p for i in range(N)], dtype=np.uint64)
        s_l = _to_mod(sk.astype(np.int64), p)
        as_ = negacyclic_mul(N, p, a, s_l)
        e_l = _to_mod(e, p)
        pk[0, l] = np.array([(p - int(x) + int(y)) % p for x, y in zip(as_, e_l)], dtype=np.uint64)
        pk[1, l] = a
    return pk


def rerandomize(P: Params, tile, pk: np.ndarray, ct_out: np.ndarray, nK: int, seed: int, flood_bits: int,
                i_begin: int = 0) -> np.ndarray:
    """c' = c + Enc_pk(0) + (F, 0) for every output ciphertext of ct_out [nI][nK][2][L][N]
    (c0 coefficient form, c1 evaluation form -- reading C26; global tile index (i_begin + I) nK + K)."""
    N = P.N
    out = ct_out.copy()
    for I in range(ct_out.shape[0]):
        for K in range(nK):
            st = (i_begin + I) * nK + K
            u = (prf_u64(seed, DOM_RR_U, st, N) % np.uint64(3)).astype(np.int64) - 1
            e1 = _cdt_sample(prf_u64(seed, DOM_RR_E, 2 * st, N))
            e2 = _cdt_sample(prf_u64(seed, DOM_RR_E, 2 * st + 1, N))
            if flood_bits > 0:
                w = prf_u64(seed, DOM_RR_F, st, N) & np.uint64((1 << flood_bits) - 1)
                F = w.astype(np.int64) - (1 << (flood_bits - 1))
            else:
                F = np.zeros(N, dtype=np.int64)
            for l, p in enumerate(P.primes):
                u_l = _to_mod(u, p)
                a0 = negacyclic_mul(N, p, pk[0, l], u_l)
                a1 = negacyclic_mul(N, p, pk[1, l], u_l)
                add0 = _to_mod(e1 + F, p)
                add1 = _to_mod(e2, p)
                out[I, K, 0, l] = [(int(c) + int(x) + int(y)) % p for c, x, y in zip(out[I, K, 0, l], a0, add0)]
                c1 = intt(N, p, P.psis[l], out[I, K, 1, l])
                c1 = np.array([(int(c) + int(x) + int(y)) % p for c, x, y in zip(c1, a1, add1)], dtype=np.uint64)
                out[I, K, 1, l] = ntt(N, p, P.psis[l], c1)
    return out
