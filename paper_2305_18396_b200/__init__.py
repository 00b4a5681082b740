"""paper_2305_18396_b200 -- B200-native homomorphic linear layer of arxiv 2305.18396 (Alg. 1).

Thin Python binding of libhelinear (C ABI declared in include/helinear.h): argument
marshalling only.  Every step of the server path (encode_weights, he_matmul,
mask_and_share) runs in the sm_100a kernels of csrc/kernels.cu; the client calls
(keygen, encrypt, decrypt_share) run in the library's host C++.  PyTorch supplies device
memory and streams.  There is no CPU fallback: if libhelinear.so is missing or no CUDA
device is present, the device calls raise.

Arrays are uint64 bit patterns.  Host arguments are numpy uint64 arrays; device arguments
are torch CUDA tensors of dtype int64 or uint64 (same bits) -- see include/helinear.h for
every layout.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libhelinear.so")

HL_OK, HL_EINVAL, HL_EDIM, HL_ERANGE, HL_ENOISE, HL_ECUDA, HL_ENOTSUP = 0, -1, -2, -3, -4, -5, -6
_CODES = {HL_EINVAL: "HL_EINVAL", HL_EDIM: "HL_EDIM", HL_ERANGE: "HL_ERANGE", HL_ENOISE: "HL_ENOISE",
          HL_ECUDA: "HL_ECUDA", HL_ENOTSUP: "HL_ENOTSUP"}

# every symbol include/helinear.h declares (checked by tests/test_abi.py)
EXPORTS = ("hl_last_error", "hl_ctx_create", "hl_ctx_destroy", "hl_ctx_params", "hl_ctx_set_mac_engine", "hl_plan_tile",
           "hl_layout_query",
           "hl_keygen", "hl_encrypt", "hl_decrypt_share", "hl_encode_weights", "hl_he_matmul",
           "hl_mask_and_share", "hl_he_matmul_share", "hl_he_linear_batch", "hl_he_linear_host", "hl_poly_mul",
           "hl_ntt_roundtrip", "hl_timing_enable", "hl_timing_read", "hl_fc_layout", "hl_fc_encode_weights", "hl_fc_encode_weights_chk",
           "hl_fc_local_share", "hl_encode_weights_strided", "hl_encode_weights_scratch", "hl_share_accumulate", "hl_sk_prepare",
           "hl_encrypt_device", "hl_decrypt_share_device", "hl_pk_gen", "hl_pk_prepare", "hl_he_matmul_share_rr",
           "hl_expand_seeded", "hl_he_linear_batch_host", "hl_packed50_words", "hl_pack50", "hl_unpack50",
           "hl_timing_kernels", "hl_public_seed", "hl_plan_tile_budget")
KERNELS = ("ntt_fwd", "mac", "intt_mask", "intt", "mask", "encode", "other", "fc")   # HL_K_* order


class HLError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_CODES.get(code, code)}: {msg}")
        self.code = code


class Tile(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("r", ctypes.c_int32), ("n", ctypes.c_int32)]

    def __repr__(self):
        return f"Tile({self.m}, {self.r}, {self.n})"


class _Layout(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in (
        "nI", "nJ", "nK", "nI_shard", "ct_in_words", "ct_out_words", "ct_masked_words",
        "ct_full_words", "share_words", "wcache_bytes", "workspace_bytes")]


class LinearDesc(ctypes.Structure):
    """hl_linear_desc: one product of hl_he_linear_batch (device pointers)."""
    _fields_ = [("wcache", ctypes.c_void_p), ("Ma", ctypes.c_int64), ("R", ctypes.c_int64), ("Nb", ctypes.c_int64),
                ("ct_in", ctypes.c_void_p), ("workspace", ctypes.c_void_p), ("ct_out_ntt", ctypes.c_void_p),
                ("seed", ctypes.c_uint64), ("ct_masked", ctypes.c_void_p), ("share", ctypes.c_void_p),
                ("tile", Tile), ("i_begin", ctypes.c_int64), ("i_end", ctypes.c_int64)]


class LinearHostDesc(ctypes.Structure):
    """hl_linear_host_desc: one product of hl_he_linear_batch_host (device + pinned host pointers)."""
    _fields_ = [("dev", LinearDesc), ("c0_host", ctypes.c_void_p), ("a_seed", ctypes.c_uint64),
                ("ct_masked_host", ctypes.c_void_p), ("share_host", ctypes.c_void_p), ("packed", ctypes.c_int32)]


@dataclass(frozen=True)
class Layout:
    nI: int
    nJ: int
    nK: int
    nI_shard: int
    ct_in_words: int
    ct_out_words: int
    ct_masked_words: int
    ct_full_words: int
    share_words: int
    wcache_bytes: int
    workspace_bytes: int


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libhelinear.so (built by `python -m paper_2305_18396_b200.build`); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libhelinear.so not built at {path}: run `python -m paper_2305_18396_b200.build`")
    L = ctypes.CDLL(path)
    vp, i64, u64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
    L.hl_last_error.restype = ctypes.c_char_p
    L.hl_last_error.argtypes = []
    sig = {
        "hl_ctx_create": [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, vp, i32, ctypes.POINTER(vp)],
        "hl_ctx_destroy": [vp],
        "hl_ctx_params": [vp, vp, vp],
        "hl_ctx_set_mac_engine": [vp, i32],
        "hl_layout_query": [vp, Tile, i64, i64, i64, i64, i64, ctypes.POINTER(_Layout)],
        "hl_plan_tile": [vp, i64, i64, i64, ctypes.POINTER(Tile)],
        "hl_plan_tile_budget": [vp, i64, i64, i64, i64, ctypes.POINTER(Tile)],
        "hl_keygen": [vp, u64, vp],
        "hl_public_seed": [u64],
        "hl_encrypt": [vp, vp, Tile, vp, i64, i64, u64, vp],
        "hl_decrypt_share": [vp, vp, Tile, vp, i32, i64, i64, vp],
        "hl_encode_weights": [vp, Tile, vp, i64, i64, i64, i64, vp, vp],
        "hl_he_matmul": [vp, Tile, vp, i64, i64, i64, i64, i64, vp, vp, vp, vp],
        "hl_mask_and_share": [vp, Tile, i64, i64, i64, i64, vp, u64, i32, vp, vp, vp],
        "hl_he_matmul_share": [vp, Tile, vp, i64, i64, i64, i64, i64, vp, vp, vp, u64, i32, vp, vp, vp],
        "hl_he_linear_batch": [vp, Tile, i32, ctypes.POINTER(LinearDesc), vp],
        "hl_he_linear_host": [vp, Tile, vp, i64, i64, i64, vp, u64, i32, vp, vp, vp, vp, vp, vp, vp, vp],
        "hl_poly_mul": [vp, vp, vp, vp, i64, vp, vp],
        "hl_ntt_roundtrip": [vp, vp, i64, vp, vp],
        "hl_timing_enable": [vp, i32],
        "hl_fc_layout": [vp, i64, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)],
        "hl_encode_weights_strided": [vp, Tile, vp, i64, i64, i64, i64, i64, i64, vp, vp],
        "hl_encode_weights_scratch": [vp, Tile, vp, i64, i64, i64, i64, i64, i64, vp, vp, ctypes.c_int, vp],
        "hl_share_accumulate": [vp, vp, vp, i64, i64, i32, vp],
        "hl_sk_prepare": [vp, vp, vp, vp],
        "hl_encrypt_device": [vp, vp, Tile, vp, i64, i64, u64, vp, vp],
        "hl_decrypt_share_device": [vp, vp, Tile, vp, i64, i64, vp, vp],
        "hl_pk_gen": [vp, vp, u64, vp],
        "hl_pk_prepare": [vp, vp, vp, vp],
        "hl_he_matmul_share_rr": [vp, Tile, vp, i64, i64, i64, i64, i64, vp, vp, vp, vp, i32, vp, u64, vp, vp, vp],
        "hl_fc_encode_weights": [vp, vp, i64, i64, vp, vp],
        "hl_fc_encode_weights_chk": [vp, vp, i64, i64, vp, ctypes.c_int, vp],
        "hl_fc_local_share": [vp, vp, vp, vp, i64, i64, i64, vp, vp, vp],
        "hl_timing_read": [vp, vp, vp],
        "hl_expand_seeded": [vp, Tile, i64, i64, u64, vp, vp],
        "hl_pack50": [vp, i64, vp],
        "hl_timing_kernels": [vp, ctypes.POINTER(i64)],
        "hl_unpack50": [vp, i64, vp],
        "hl_he_linear_batch_host": [vp, Tile, i32, ctypes.POINTER(LinearHostDesc), vp],
    }
    missing = set(EXPORTS) - set(sig) - {"hl_last_error", "hl_packed50_words"}
    if missing:     # an entry point without a prototype would be called with C-int arguments
        raise ImportError(f"libhelinear binding: no signature for {sorted(missing)}")
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.hl_packed50_words.argtypes = [i64]
    L.hl_packed50_words.restype = i64
    L.hl_public_seed.restype = u64
    _lib = L
    return L


def _check(rc: int):
    if rc != HL_OK:
        raise HLError(rc, _lib.hl_last_error().decode())


def _tile(t) -> Tile:
    return t if isinstance(t, Tile) else Tile(*[int(v) for v in t])


def _hptr(a: np.ndarray, dtype) -> int:
    assert isinstance(a, np.ndarray) and a.dtype == dtype and a.flags["C_CONTIGUOUS"], (a.dtype, dtype)
    return a.ctypes.data


def _dptr(t) -> int:
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
        raise HLError(HL_EINVAL, "expected a contiguous CUDA tensor")
    return t.data_ptr()


def _stream(stream) -> int:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev_empty(nwords: int, device):
    import torch
    return torch.empty(int(nwords), dtype=torch.int64, device=device)


class Context:
    """A BFV-RNS parameter set {N, t = 2^t_bits, q = p_0..p_{L-1}} bound to one CUDA device."""

    def __init__(self, N: int = 4096, L: int = 2, t_bits: int = 37, primes=None, device: int = 0):
        lib = load_library()
        self.N, self.L, self.t_bits, self.device = int(N), int(L), int(t_bits), int(device)
        h = ctypes.c_void_p()
        pr = None
        if primes is not None:
            pr = np.ascontiguousarray(np.array(primes, dtype=np.uint64))
        _check(lib.hl_ctx_create(self.N, self.L, self.t_bits, pr.ctypes.data if pr is not None else None,
                                 self.device, ctypes.byref(h)))
        self._h = h
        p = np.zeros(self.L, np.uint64)
        d = np.zeros(self.L, np.uint64)
        _check(lib.hl_ctx_params(h, p.ctypes.data, d.ctypes.data))
        self.primes = tuple(int(v) for v in p)
        self.delta_mod = tuple(int(v) for v in d)

    MAC_IMAD, MAC_F64, MAC_TC = 0, 1, 2

    def set_mac_engine(self, engine: int):
        """0 = IMAD.WIDE limbs, 1 = exact FP64 products, 2 = int8 tensor cores (default).
        Re-encode weights after (cache formats differ)."""
        _check(_lib.hl_ctx_set_mac_engine(self._h, int(engine)))

    def close(self):
        if getattr(self, "_h", None):
            _lib.hl_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def device_str(self) -> str:
        return f"cuda:{self.device}"

    def layout(self, tile, Ma: int, R: int, Nb: int, i_begin: int = 0, i_end: int = -1) -> Layout:
        out = _Layout()
        _check(_lib.hl_layout_query(self._h, _tile(tile), Ma, R, Nb, i_begin, i_end, ctypes.byref(out)))
        return Layout(*[getattr(out, f) for f, _ in _Layout._fields_])

    # ---------------------------------------------------------------- client (host memory)
    def plan_tile(self, Ma: int, R: int, Nb: int, max_wcache_bytes: int = 0) -> tuple:
        """hl_plan_tile(_budget): the planner's (m, r, n) for an Nb x R . R x Ma product, optionally
        under a weight-cache budget in bytes."""
        t = Tile()
        if max_wcache_bytes > 0:
            _check(_lib.hl_plan_tile_budget(self._h, Ma, R, Nb, int(max_wcache_bytes), ctypes.byref(t)))
        else:
            _check(_lib.hl_plan_tile(self._h, Ma, R, Nb, ctypes.byref(t)))
        return (t.m, t.r, t.n)

    def keygen(self, seed: int) -> np.ndarray:
        sk = np.zeros(self.N, dtype=np.int8)
        _check(_lib.hl_keygen(self._h, seed, sk.ctypes.data))
        return sk

    def encrypt(self, sk: np.ndarray, tile, X: np.ndarray, seed: int) -> np.ndarray:
        X = np.ascontiguousarray(X, dtype=np.uint64)
        Nb, R = X.shape
        lay = self.layout(tile, 1, R, Nb)
        ct = np.zeros((lay.nJ, lay.nK, 2, self.L, self.N), dtype=np.uint64)
        _check(_lib.hl_encrypt(self._h, _hptr(np.ascontiguousarray(sk), np.int8), _tile(tile), X.ctypes.data,
                               Nb, R, seed, ct.ctypes.data))
        return ct

    def decrypt_share(self, sk: np.ndarray, tile, ct_masked: np.ndarray, Ma: int, Nb: int,
                      compress: bool = True) -> np.ndarray:
        ct_masked = np.ascontiguousarray(ct_masked, dtype=np.uint64)
        lay = self.layout(tile, Ma, 1, Nb)
        need = lay.ct_masked_words if compress else lay.ct_full_words
        if ct_masked.size != need:
            raise HLError(HL_EINVAL, f"ct_masked has {ct_masked.size} words, expected {need}")
        out = np.zeros((Nb, Ma), dtype=np.uint64)
        _check(_lib.hl_decrypt_share(self._h, _hptr(np.ascontiguousarray(sk), np.int8), _tile(tile),
                                     ct_masked.ctypes.data, int(bool(compress)), Ma, Nb, out.ctypes.data))
        return out

    # ---------------------------------------------------------------- client on the GPU (row f3)
    def sk_prepare(self, sk: np.ndarray, device=None, stream=None):
        """NTT(s) per prime on the device (the device client's key form)."""
        import torch
        dev = device if device is not None else torch.device("cuda", self.device)
        s_hat = _dev_empty(self.L * self.N, dev)
        _check(_lib.hl_sk_prepare(self._h, _hptr(np.ascontiguousarray(sk), np.int8), _dptr(s_hat), _stream(stream)))
        return s_hat

    def encrypt_device(self, s_hat, tile, X, seed: int, ct_in=None, stream=None):
        """X: CUDA tensor [Nb][R] (< 2^t) -> ct_in CUDA tensor [nJ][nK][2][L][N] (== encrypt())."""
        Nb, R = X.shape
        lay = self.layout(tile, 1, R, Nb)
        if ct_in is None:
            ct_in = _dev_empty(lay.ct_in_words, X.device)
        _check(_lib.hl_encrypt_device(self._h, _dptr(s_hat), _tile(tile), _dptr(X), Nb, R, seed, _dptr(ct_in),
                                      _stream(stream)))
        return ct_in

    def decrypt_share_device(self, s_hat, tile, ct_masked, Ma: int, Nb: int, share=None, stream=None):
        """Compressed response (CUDA tensor) -> client share [Nb][Ma] (== decrypt_share())."""
        if share is None:
            share = _dev_empty(Nb * Ma, ct_masked.device)
        _check(_lib.hl_decrypt_share_device(self._h, _dptr(s_hat), _tile(tile), _dptr(ct_masked), Ma, Nb,
                                            _dptr(share), _stream(stream)))
        return share

    # ---------------------------------------------------------------- re-randomisation (row f4)
    def pk_gen(self, sk: np.ndarray, seed: int) -> np.ndarray:
        pk = np.zeros((2, self.L, self.N), dtype=np.uint64)
        _check(_lib.hl_pk_gen(self._h, _hptr(np.ascontiguousarray(sk), np.int8), seed, pk.ctypes.data))
        return pk

    def pk_prepare(self, pk: np.ndarray, device=None, stream=None):
        import torch
        dev = device if device is not None else torch.device("cuda", self.device)
        pk_hat = _dev_empty(2 * self.L * self.N, dev)
        _check(_lib.hl_pk_prepare(self._h, _hptr(np.ascontiguousarray(pk, dtype=np.uint64), np.uint64),
                                  _dptr(pk_hat), _stream(stream)))
        return pk_hat

    def he_matmul_share_rr(self, tile, wcache, Ma: int, R: int, Nb: int, ct_in, seed: int, pk_hat, flood_bits: int,
                           i_begin: int = 0, i_end: int = -1, stream=None):
        """Compressed he_matmul_share with re-randomised responses (hl_he_matmul_share_rr)."""
        import torch
        lay = self.layout(tile, Ma, R, Nb, i_begin, i_end)
        dev = ct_in.device
        ws = _dev_empty(lay.workspace_bytes // 8, dev)
        co = _dev_empty(lay.ct_out_words, dev)
        rr = _dev_empty(lay.nI_shard * lay.nK * self.L * self.N, dev)
        cm = _dev_empty(lay.ct_masked_words, dev)
        sh = torch.zeros(Nb * Ma, dtype=torch.int64, device=dev)
        _check(_lib.hl_he_matmul_share_rr(self._h, _tile(tile), _dptr(wcache), Ma, R, Nb, i_begin, i_end, _dptr(ct_in),
                                          _dptr(ws), _dptr(co), _dptr(pk_hat), int(flood_bits), _dptr(rr), seed,
                                          _dptr(cm), _dptr(sh), _stream(stream)))
        self._rr_keep = (ws, co, rr)
        return cm, sh

    # ---------------------------------------------------------------- server (device memory)
    def encode_weights(self, tile, W, i_begin: int = 0, i_end: int = -1, wcache=None, stream=None,
                       check: bool = True):
        """W: CUDA tensor [R][Ma] (int64/uint64 bits).  Returns the opaque NTT-domain cache
        (hl_encode_weights_scratch: two passes through a scratch buffer allocated here).
        check=False skips the range / noise-bound check and its synchronisation."""
        R, Ma = W.shape
        return self._encode(tile, W, R, Ma, Ma, 1, i_begin, i_end, wcache, stream, check)

    def encode_weights_T(self, tile, M, i_begin: int = 0, i_end: int = -1, wcache=None, stream=None,
                         check: bool = True):
        """Encode W = M^T for a CUDA tensor M [Ma][R] without materialising the transpose."""
        Ma, R = M.shape
        return self._encode(tile, M, R, Ma, 1, R, i_begin, i_end, wcache, stream, check)

    def _encode(self, tile, W, R, Ma, ld_row, ld_col, i_begin, i_end, wcache, stream, check):
        lay = self.layout(tile, Ma, R, 1, i_begin, i_end)
        if wcache is None:
            wcache = _dev_empty(lay.wcache_bytes // 8, W.device)
        scratch = _dev_empty(lay.nI_shard * lay.nJ * self.L * self.N, W.device)
        _check(_lib.hl_encode_weights_scratch(self._h, _tile(tile), _dptr(W), R, Ma, ld_row, ld_col, i_begin, i_end,
                                              _dptr(wcache), _dptr(scratch), int(bool(check)), _stream(stream)))
        self._enc_scratch = scratch          # alive until the next encode (stream-ordered use)
        return wcache

    def share_accumulate(self, dst, src, rows: int, cols: int, transpose: bool = False, stream=None):
        """dst[rows][cols] += src (or src^T) mod 2^t, in place."""
        _check(_lib.hl_share_accumulate(self._h, _dptr(dst), _dptr(src), rows, cols, int(bool(transpose)),
                                        _stream(stream)))
        return dst

    def he_matmul(self, tile, wcache, Ma: int, R: int, Nb: int, ct_in, i_begin: int = 0, i_end: int = -1,
                  workspace=None, ct_out=None, stream=None):
        lay = self.layout(tile, Ma, R, Nb, i_begin, i_end)
        if workspace is None:
            workspace = _dev_empty(lay.workspace_bytes // 8, ct_in.device)
        if ct_out is None:
            ct_out = _dev_empty(lay.ct_out_words, ct_in.device)
        _check(_lib.hl_he_matmul(self._h, _tile(tile), _dptr(wcache), Ma, R, Nb, i_begin, i_end, _dptr(ct_in),
                                 _dptr(workspace), _dptr(ct_out), _stream(stream)))
        return ct_out

    def mask_and_share(self, tile, Ma: int, Nb: int, ct_out, seed: int, compress: bool = True,
                       i_begin: int = 0, i_end: int = -1, ct_masked=None, share=None, stream=None):
        lay = self.layout(tile, Ma, 1, Nb, i_begin, i_end)
        if ct_masked is None:
            ct_masked = _dev_empty(lay.ct_masked_words if compress else lay.ct_full_words, ct_out.device)
        if share is None:
            import torch
            share = torch.zeros(Nb * Ma, dtype=torch.int64, device=ct_out.device)
        _check(_lib.hl_mask_and_share(self._h, _tile(tile), Ma, Nb, i_begin, i_end, _dptr(ct_out), seed,
                                      int(bool(compress)), _dptr(ct_masked), _dptr(share), _stream(stream)))
        return ct_masked, share

    def he_matmul_share(self, tile, wcache, Ma: int, R: int, Nb: int, ct_in, seed: int, compress: bool = True,
                        i_begin: int = 0, i_end: int = -1, workspace=None, ct_out_ntt=None, ct_masked=None,
                        share=None, stream=None):
        lay = self.layout(tile, Ma, R, Nb, i_begin, i_end)
        dev = ct_in.device
        if workspace is None:
            workspace = _dev_empty(lay.workspace_bytes // 8, dev)
        if ct_out_ntt is None:
            ct_out_ntt = _dev_empty(lay.ct_out_words, dev)
        if ct_masked is None:
            ct_masked = _dev_empty(lay.ct_masked_words if compress else lay.ct_full_words, dev)
        if share is None:
            import torch
            share = torch.zeros(Nb * Ma, dtype=torch.int64, device=dev)
        _check(_lib.hl_he_matmul_share(self._h, _tile(tile), _dptr(wcache), Ma, R, Nb, i_begin, i_end,
                                       _dptr(ct_in), _dptr(workspace), _dptr(ct_out_ntt), seed,
                                       int(bool(compress)), _dptr(ct_masked), _dptr(share), _stream(stream)))
        return ct_masked, share

    def he_linear_batch(self, tile, entries, stream=None):
        """Pipelined compressed he_matmul_share over several products (hl_he_linear_batch).
        entries: dicts with wcache, Ma, R, Nb, ct_in, seed and optionally tile (this product's tile;
        default: `tile`), i_begin / i_end (an I-tile shard, default the whole product), workspace,
        ct_out_ntt, ct_masked, share (allocated here if absent; every entry gets its own buffers).
        Returns [(ct_masked, share), ...]."""
        descs = (LinearDesc * len(entries))()
        keep, outs = [], []
        for d, e in zip(descs, entries):
            self._fill_desc(tile, d, e, keep, outs)
        _check(_lib.hl_he_linear_batch(self._h, _tile(tile), len(entries), descs, _stream(stream)))
        self._batch_keep = keep        # scratch stays alive until the next batch call
        return outs

    def _fill_desc(self, tile, d, e, keep, outs):
        import torch
        Ma, R, Nb = int(e["Ma"]), int(e["R"]), int(e["Nb"])
        tile = tuple(e["tile"]) if e.get("tile") is not None else tuple(tile)
        i0, i1 = int(e.get("i_begin", 0)), int(e.get("i_end", -1))
        lay = self.layout(tile, Ma, R, Nb, i0, i1)
        dev = e["ct_in"].device
        ws = e.get("workspace") if e.get("workspace") is not None else _dev_empty(lay.workspace_bytes // 8, dev)
        co = e.get("ct_out_ntt") if e.get("ct_out_ntt") is not None else _dev_empty(lay.ct_out_words, dev)
        cm = e.get("ct_masked") if e.get("ct_masked") is not None else _dev_empty(lay.ct_masked_words, dev)
        sh = e.get("share") if e.get("share") is not None else torch.zeros(Nb * Ma, dtype=torch.int64, device=dev)
        d.wcache, d.Ma, d.R, d.Nb = _dptr(e["wcache"]), Ma, R, Nb
        d.ct_in, d.workspace, d.ct_out_ntt = _dptr(e["ct_in"]), _dptr(ws), _dptr(co)
        d.seed, d.ct_masked, d.share = int(e["seed"]), _dptr(cm), _dptr(sh)
        d.tile = _tile(tile)
        d.i_begin, d.i_end = i0, i1
        keep += [ws, co]
        outs.append((cm, sh))

    def expand_seeded(self, tile, R: int, Nb: int, a_seed: int, ct_in, stream=None):
        """hl_expand_seeded: regenerate the c1 = a halves of ct_in (CUDA int64 [nJ][nK][2][L][N])
        from the client's PUBLIC seed a_seed = public_seed(enc_seed) (reading C28)."""
        _check(_lib.hl_expand_seeded(self._h, _tile(tile), R, Nb, a_seed, _dptr(ct_in), _stream(stream)))
        return ct_in

    def he_linear_batch_host(self, tile, entries, stream=None):
        """End-to-end pipelined batch on pinned host buffers (hl_he_linear_batch_host).  entries:
        the he_linear_batch dicts (ct_in = the device upload buffer, distinct per entry) plus
        c0_host (pinned CPU int64 [nJ][nK][L][N], see c0_halves), a_seed (= public_seed(enc seed),
        reading C28: the private encryption seed never crosses the boundary), masked_host and
        share_host (pinned CPU int64), and optionally packed=True (c0_host and masked_host in the
        50-bit wire format of pack50).  Stream-ordered: synchronise before reading the host outputs."""
        descs = (LinearHostDesc * len(entries))()
        keep, outs = [], []
        for d, e in zip(descs, entries):
            self._fill_desc(tile, d.dev, e, keep, outs)
            d.c0_host, d.a_seed = e["c0_host"].data_ptr(), int(e["a_seed"])
            d.packed = int(bool(e.get("packed", False)))
            d.ct_masked_host, d.share_host = e["masked_host"].data_ptr(), e["share_host"].data_ptr()
            keep += [e["c0_host"], e["masked_host"], e["share_host"]] + [o for o in outs[-1]]
        _check(_lib.hl_he_linear_batch_host(self._h, _tile(tile), len(entries), descs, _stream(stream)))
        self._batch_keep = keep

    @staticmethod
    def pack50(words: np.ndarray) -> np.ndarray:
        """50-bit wire format (hl_pack50) of uint64 words < 2^50."""
        w = np.ascontiguousarray(words, dtype=np.uint64).reshape(-1)
        out = np.zeros(int(_lib.hl_packed50_words(w.size)), dtype=np.uint64)
        _check(_lib.hl_pack50(w.ctypes.data, w.size, out.ctypes.data))
        return out

    @staticmethod
    def unpack50(packed: np.ndarray, words: int) -> np.ndarray:
        """Inverse of pack50: the first `words` residues."""
        p = np.ascontiguousarray(packed, dtype=np.uint64).reshape(-1)
        out = np.zeros(words, dtype=np.uint64)
        _check(_lib.hl_unpack50(p.ctypes.data, words, out.ctypes.data))
        return out

    @staticmethod
    def c0_halves(ct):
        """The c0 halves of input ciphertexts [nJ][nK][2][L][N] (what a seeded upload sends):
        a contiguous [nJ][nK][L][N] array."""
        return np.ascontiguousarray(np.asarray(ct)[:, :, 0])

    def he_linear_host(self, tile, wcache, Ma: int, R: int, Nb: int, ct_in_host, seed: int, ct_masked_host,
                       share_host, dev_ct_in, workspace, dev_ct_out_ntt, dev_ct_masked, dev_share,
                       compress: bool = True, stream=None):
        """End-to-end server call on pinned host buffers (torch CPU tensors, pin_memory=True)."""
        _check(_lib.hl_he_linear_host(self._h, _tile(tile), _dptr(wcache), Ma, R, Nb, ct_in_host.data_ptr(), seed,
                                      int(bool(compress)), ct_masked_host.data_ptr(), share_host.data_ptr(),
                                      _dptr(dev_ct_in), _dptr(workspace), _dptr(dev_ct_out_ntt),
                                      _dptr(dev_ct_masked), _dptr(dev_share), _stream(stream)))

    # ---------------------------------------------------------------- FC layer (row f1)
    def fc_layout(self, Nb: int, R: int, Ma: int):
        wb, ws = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.hl_fc_layout(self._h, Nb, R, Ma, ctypes.byref(wb), ctypes.byref(ws)))
        return wb.value, ws.value

    def fc_encode_weights(self, W, stream=None, check: bool = True):
        """W: CUDA tensor [R][Ma] (< 2^t).  Returns the opaque byte-plane form.  check=False skips
        the range check and its stream synchronisation (hl_fc_encode_weights_chk)."""
        R, Ma = W.shape
        wb, _ = self.fc_layout(1, R, Ma)
        wp = _dev_empty(-(-wb // 8), W.device)
        _check(_lib.hl_fc_encode_weights_chk(self._h, _dptr(W), R, Ma, _dptr(wp), int(bool(check)),
                                             _stream(stream)))
        return wp

    def fc_local_share(self, X1, wplanes, Ma: int, share, bias=None, workspace=None, stream=None):
        """share[Nb][Ma] += X1.W + bias (mod 2^t), in place."""
        Nb, R = X1.shape
        _, ws = self.fc_layout(Nb, R, Ma)
        if workspace is None:
            workspace = _dev_empty(-(-ws // 8), X1.device)
        _check(_lib.hl_fc_local_share(self._h, _dptr(X1), _dptr(wplanes), _dptr(bias) if bias is not None else None,
                                      Nb, R, Ma, _dptr(workspace), _dptr(share), _stream(stream)))
        return share

    # ---------------------------------------------------------------- timing
    def timing_enable(self, on: bool = True):
        _check(_lib.hl_timing_enable(self._h, int(bool(on))))

    def timing_kernels(self) -> int:
        """Kernel launches inside the timed sections since the last call (hl_timing_kernels)."""
        n = ctypes.c_int64()
        _check(_lib.hl_timing_kernels(self._h, ctypes.byref(n)))
        return n.value

    def timing_read(self) -> dict:
        """{kernel: (total_ms, launches)} since the last read (synchronises the recorded events)."""
        ms = np.zeros(len(KERNELS), np.float64)
        cnt = np.zeros(len(KERNELS), np.int64)
        _check(_lib.hl_timing_read(self._h, ms.ctypes.data, cnt.ctypes.data))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNELS)}

    # ---------------------------------------------------------------- diagnostics
    def poly_mul(self, a, b, out=None, scratch=None, stream=None):
        npoly = a.numel() // (self.L * self.N)
        if out is None:
            out = _dev_empty(a.numel(), a.device)
        if scratch is None:
            scratch = _dev_empty(2 * a.numel(), a.device)
        _check(_lib.hl_poly_mul(self._h, _dptr(a), _dptr(b), _dptr(out), npoly, _dptr(scratch), _stream(stream)))
        return out

    def ntt_roundtrip(self, x, scratch=None, stream=None):
        npoly = x.numel() // (self.L * self.N)
        if scratch is None:
            scratch = _dev_empty(x.numel(), x.device)
        _check(_lib.hl_ntt_roundtrip(self._h, _dptr(x), npoly, _dptr(scratch), _stream(stream)))
        return x


def public_seed(enc_seed: int) -> int:
    """hl_public_seed (reading C28): the public A-domain seed of a private encryption seed."""
    return int(load_library().hl_public_seed(enc_seed))


def to_device(a: np.ndarray, device="cuda"):
    """numpy uint64 -> CUDA int64 tensor with the same bits."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(device)


def to_host(t) -> np.ndarray:
    """CUDA/CPU int64 tensor -> numpy uint64 with the same bits."""
    return t.detach().cpu().numpy().view(np.uint64)
