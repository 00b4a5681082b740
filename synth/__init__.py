"""Seeded synthetic workloads for the homomorphic linear layer (shared by oracle tests and bench).

This module holds NO arithmetic of the method: it only names the configurations of
BASELINE.json (shapes, RLWE sizes, tiles) and draws seeded numpy inputs with the
value distributions those configurations state.  Both the CPU oracle (`oracle/`) and
the CUDA path (`paper_2305_18396_b200/`) consume what it produces; neither is imported here.

Value distributions (BASELINE.json configs; SURVEY.md §8(d) "Synthetic inputs"):
  * activations X: the client's additive share, uniform in Z_{2^37}
  * weights W: round(N(0, 0.02) * 2^12) mod 2^37  (12 fractional bits; BASELINE.json)
The paper's GLUE/pretrained-checkpoint workloads are replaced by these
seeded inputs with the same shapes (seq 128, hidden 128/768/1024, FFN 4E).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

T_BITS = 37           # plaintext modulus t = 2^37 (BASELINE.json)
FRAC_BITS = 12        # fixed-point fractional bits f (BASELINE.json)
W_STD = 0.02          # weight std (BASELINE.json "N(0,0.02)")
BASE_SEED = 0x230518396


@dataclass(frozen=True)
class MatmulShape:
    """One encrypted product X(Nb x R) . W(R x Ma)."""
    name: str
    Nb: int   # tokens (rows of X)
    R: int    # shared dimension
    Ma: int   # output features


@dataclass(frozen=True)
class Config:
    name: str
    N: int
    L: int
    tile: tuple          # (m, r, n), m*r*n <= N   (SURVEY.md §8 reading C2)
    matmuls: tuple       # tuple[MatmulShape]
    blocks: int = 1      # independent encoder blocks (c3/c4)
    note: str = ""
    tiles: tuple = ()    # per-product tiles (the library's hl_plan_tile choice); () = `tile` for all
    batch_order: tuple = ()   # bench submission order of the products to hl_he_linear_batch; () = as listed
    e2e_order: tuple = ()     # the same for the end-to-end (host buffers, PCIe-bound) call; () = batch_order
    seqs: int = 1             # independent sequences per block (c3: 8, c4: 4); Nb = seqs * seq_len
    seq_len: int = 128

    def block_shapes(self, nseq: int) -> tuple:
        """The block's products over `nseq` of its sequences (Nb = nseq * seq_len)."""
        return tuple(MatmulShape(mm.name, nseq * self.seq_len, mm.R, mm.Ma) for mm in self.matmuls)

    def tile_of(self, mi: int) -> tuple:
        return self.tiles[mi] if self.tiles else self.tile


def _block(seq: int, hidden: int, ffn: int, qkv: bool = True):
    return (
        MatmulShape("qkv", seq, hidden, 3 * hidden),
        MatmulShape("o", seq, hidden, hidden),
        MatmulShape("ff1", seq, hidden, ffn),
        MatmulShape("ff2", seq, ffn, hidden),
    )


CONFIGS = {
    # c0: single 8x64 . 64x64 encrypted matmul, N=4096, L=2
    "c0": Config("c0", 4096, 2, (16, 32, 8), (MatmulShape("single", 8, 64, 64),),
                 note="single encrypted matmul X(8x64).W(64x64)"),
    # c1: BERT-Tiny block, seq 128, hidden 128, FFN 512
    "c1": Config("c1", 4096, 2, (16, 8, 32), _block(128, 128, 512),
                 note="BERT-Tiny-shaped encoder block, seq 128"),
    # c2: BERT-base block, seq 128, hidden 768, FFN 3072  (the bench workload)
    "c2": Config("c2", 4096, 2, (16, 8, 32), _block(128, 768, 3072),
                 note="BERT-base-shaped encoder block, seq 128",
                 tiles=((16, 8, 32), (8, 8, 64), (16, 8, 32), (4, 32, 32)), batch_order=(3, 1, 2, 0), e2e_order=(2, 0, 3, 1)),
    # c3: 12 BERT-base blocks x 8 sequences (Nb = 8*128)
    "c3": Config("c3", 4096, 2, (16, 8, 32), _block(1024, 768, 3072), blocks=12,
                 note="12 BERT-base blocks, 8 sequences x 128 tokens", seqs=8, seq_len=128),
    # c4: BERT-large 24 blocks, seq 512 x batch 4, N=8192, L=3
    "c4": Config("c4", 8192, 3, (32, 16, 16), _block(2048, 1024, 4096), blocks=24,
                 note="24 BERT-large blocks, 4 sequences x 512 tokens", seqs=4, seq_len=512),
}


def seed_for(block: int, matmul: int, what: str) -> int:
    """Seed recipe of SURVEY.md §8(d): BASE + 1000*block + 10*matmul + offset."""
    off = {"x": 0, "w": 1, "key": 2, "enc": 3, "mask": 4}[what]
    return BASE_SEED + 1000 * block + 10 * matmul + off


def activations(seed: int, Nb: int, R: int, t_bits: int = T_BITS) -> np.ndarray:
    """Client share X: uint64 [Nb][R], uniform in [0, 2^t_bits)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 1 << t_bits, size=(Nb, R), dtype=np.uint64)


def activations_seq(seed: int, seq0: int, seq1: int, seq_len: int, R: int, t_bits: int = T_BITS) -> np.ndarray:
    """Client shares X [(seq1 - seq0) * seq_len][R] of sequences [seq0, seq1) of a stacked block
    (c3, c4): sequence s's rows are activations(seed + 7919 * (s + 1), seq_len, R), so any
    sequence range of a block is generated without materialising the others."""
    out = np.empty(((seq1 - seq0) * seq_len, R), dtype=np.uint64)
    for s in range(seq0, seq1):
        out[(s - seq0) * seq_len:(s - seq0 + 1) * seq_len] = activations(seed + 7919 * (s + 1), seq_len, R, t_bits)
    return out


def weights(seed: int, R: int, Ma: int, t_bits: int = T_BITS, frac_bits: int = FRAC_BITS,
            std: float = W_STD) -> np.ndarray:
    """Server weights W: uint64 [R][Ma] = round(N(0,std) * 2^f) mod 2^t_bits (two's complement)."""
    rng = np.random.default_rng(seed)
    w = np.rint(rng.normal(0.0, std, size=(R, Ma)) * (1 << frac_bits)).astype(np.int64)
    return (w & ((1 << t_bits) - 1)).astype(np.uint64)


def stressed_weights(seed: int, R: int, Ma: int, bound: int, t_bits: int = T_BITS) -> np.ndarray:
    """Edge-case weights: uniform signed integers in [-bound, bound] mod 2^t_bits."""
    rng = np.random.default_rng(seed)
    w = rng.integers(-bound, bound + 1, size=(R, Ma), dtype=np.int64)
    return (w & ((1 << t_bits) - 1)).astype(np.uint64)


def uniform_below(seed: int, shape, bounds) -> np.ndarray:
    """uint64 array whose slice [..., l, :] is uniform in [0, bounds[l]).

    Used for random ciphertext residues (he_matmul is linear, so parity on uniform
    residues exercises every coefficient).  `shape[-2]` must equal len(bounds).
    """
    rng = np.random.default_rng(seed)
    out = np.empty(shape, dtype=np.uint64)
    for l, b in enumerate(bounds):
        out[..., l, :] = rng.integers(0, int(b), size=out[..., l, :].shape, dtype=np.uint64)
    return out
