"""the server side of the attention cross terms (Eq. 2).

For Z = X Y with both inputs secret-shared (X = X0 + X1, Y = Y0 + Y1; client 0, server 1), e.g.
Q K^T and A V of multi-head attention, the parties invoke Pi_MatMul twice on the cross terms and
add their local products:
    term 1  X1 Y0 = (Y0^T X1^T)^T   client encrypts Y0^T, server operand X1^T  (footnote 3,
                                     PAPER.md:115: the client always encrypts; both transpose)
    term 2  X0 Y1                    client encrypts X0,   server operand Y1
    server  Z1 = <X1 Y0>_1^T + <X0 Y1>_1 + X1 Y1
Every step runs in libhelinear's kernels (online pi_A encoding of the server's shares, the fused
he_matmul_share, the transposed share accumulation, the FC-style local product); this module
only sequences the calls.  The server operands are uniform 37-bit shares, so the noise budget
needs the N=8192, L=3 parameter set (q ~ 2^150, tests/test_oracle.py).
"""
from __future__ import annotations


def server_cross_product(ctx, tile, X1, Y1, ct_Y0T, ct_X0, seeds, stream=None):
    """X1 [n][d], Y1 [d][n2]: the server's shares (CUDA int64 tensors, values < 2^t);
    ct_Y0T: the client's encryption of Y0^T ([n2][d], pi_B layout of hl_encrypt);
    ct_X0: the client's encryption of X0 ([n][d]); seeds: the two mask seeds.
    Returns (masked_1, masked_2, Z1): the compressed responses of term 1 ((X1 Y0)^T, layout
    [n2][n] after decryption) and term 2 (X0 Y1, [n][n2]) for the client, and the server's share
    Z1 [n][n2] of X Y (mod 2^t).  tile: one (m, r, n) for both terms, or a pair (term 1, term 2)
    (e.g. hl_plan_tile's choices for (n, d, n2) and (n2, d, n)); the client encrypts with the same."""
    n, d = X1.shape
    n2 = Y1.shape[1]
    t1, t2 = (tile[0], tile[1]) if isinstance(tile[0], (tuple, list)) else (tile, tile)
    # the server's shares are < 2^t by construction and the N=8192/L=3 set bounds the noise of any
    # 37-bit operand (reading C23): online encodings skip the range check and its sync
    w1 = ctx.encode_weights_T(t1, X1, stream=stream, check=False)          # W = X1^T: R = d, Ma = n
    m1, s1 = ctx.he_matmul_share(t1, w1, n, d, n2, ct_Y0T, seed=seeds[0], stream=stream)     # s1 [n2][n]
    w2 = ctx.encode_weights(t2, Y1, stream=stream, check=False)            # W = Y1: R = d, Ma = n2
    m2, z1 = ctx.he_matmul_share(t2, w2, n2, d, n, ct_X0, seed=seeds[1], stream=stream)      # z1 [n][n2]
    ctx.share_accumulate(z1, s1, n, n2, transpose=True, stream=stream)     # + <X1 Y0>_1^T
    ctx.fc_local_share(X1, ctx.fc_encode_weights(Y1, stream=stream, check=False), n2, z1, stream=stream)   # + X1 Y1
    return m1, m2, z1


def server_cross_products(ctx, items, stream=None):
    """Many cross products at once (e.g. every head of a block): items = dicts with tile (one or a
    pair, as server_cross_product), X1, Y1, ct_Y0T, ct_X0, seeds.  The 2 len(items) Pi_MatMul
    products run as ONE pipelined hl_he_linear_batch (each entry with its own tile), then the
    transposed share accumulation and the local products.  Results equal server_cross_product's
    item by item; returns [(masked_1, masked_2, Z1), ...]."""
    entries, meta = [], []
    for it in items:
        tile = it["tile"]
        t1, t2 = (tile[0], tile[1]) if isinstance(tile[0], (tuple, list)) else (tile, tile)
        X1, Y1 = it["X1"], it["Y1"]
        n, d = X1.shape
        n2 = Y1.shape[1]
        w1 = ctx.encode_weights_T(t1, X1, stream=stream, check=False)
        entries.append(dict(wcache=w1, Ma=n, R=d, Nb=n2, ct_in=it["ct_Y0T"], seed=it["seeds"][0], tile=t1))
        w2 = ctx.encode_weights(t2, Y1, stream=stream, check=False)
        entries.append(dict(wcache=w2, Ma=n2, R=d, Nb=n, ct_in=it["ct_X0"], seed=it["seeds"][1], tile=t2))
        meta.append((n, n2))
    outs = ctx.he_linear_batch(entries[0]["tile"], entries, stream=stream)
    res = []
    for k, it in enumerate(items):
        n, n2 = meta[k]
        (m1, s1), (m2, z1) = outs[2 * k], outs[2 * k + 1]
        ctx.share_accumulate(z1, s1, n, n2, transpose=True, stream=stream)
        ctx.fc_local_share(it["X1"], ctx.fc_encode_weights(it["Y1"], stream=stream, check=False), n2, z1,
                           stream=stream)
        res.append((m1, m2, z1))
    return res
