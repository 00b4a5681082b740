"""Break down the row-f2 cross-product time (one QK^T-shaped head): per call host+device time."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2305_18396_b200 as hl  # noqa
from paper_2305_18396_b200 import attention  # noqa
import synth  # noqa

ctx = hl.Context(8192, 3, 37, device=0)
dev = torch.device("cuda", 0)
for (n, d, n2) in ((128, 64, 128), (128, 128, 64)):
    for tile in [(32, 16, 16), tuple(ctx.plan_tile(n, d, n2)), tuple(ctx.plan_tile(n2, d, n))]:
        sd = 1234
        X0, X1 = synth.activations(sd, n, d), synth.activations(sd + 1, n, d)
        Y0, Y1 = synth.activations(sd + 2, d, n2), synth.activations(sd + 3, d, n2)
        sk1, sk2 = ctx.keygen(sd + 4), ctx.keygen(sd + 5)
        dX1, dY1 = hl.to_device(X1, dev), hl.to_device(Y1, dev)
        ct1 = hl.to_device(ctx.encrypt(sk1, tile, np.ascontiguousarray(Y0.T), sd + 6), dev)
        ct2 = hl.to_device(ctx.encrypt(sk2, tile, X0, sd + 7), dev)
        for _ in range(3):
            attention.server_cross_product(ctx, tile, dX1, dY1, ct1, ct2, (1, 2))
        torch.cuda.synchronize()
        steps = {}
        def T(name, f):
            torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
            steps[name] = steps.get(name, 0) + (time.perf_counter() - t0) * 1e3
            return r
        for _ in range(5):
            w1 = T("encode_T", lambda: ctx.encode_weights_T(tile, dX1))
            m1, s1 = T("he_matmul_share1", lambda: ctx.he_matmul_share(tile, w1, n, d, n2, ct1, seed=1))
            w2 = T("encode", lambda: ctx.encode_weights(tile, dY1))
            m2, z1 = T("he_matmul_share2", lambda: ctx.he_matmul_share(tile, w2, n2, d, n, ct2, seed=2))
            T("accumulate", lambda: ctx.share_accumulate(z1, s1, n, n2, transpose=True))
            wp = T("fc_encode", lambda: ctx.fc_encode_weights(dY1))
            T("fc_local", lambda: ctx.fc_local_share(dX1, wp, n2, z1))
        t0 = time.perf_counter()
        for _ in range(10):
            attention.server_cross_product(ctx, tile, dX1, dY1, ct1, ct2, (1, 2))
        torch.cuda.synchronize()
        tot = (time.perf_counter() - t0) * 100
        print((n, d, n2), tile, "whole ms", round(tot, 3), {k: round(v / 5, 3) for k, v in steps.items()},
              "wcache MB", ctx.layout(tile, n, d, n2).wcache_bytes / 1e6, flush=True)
