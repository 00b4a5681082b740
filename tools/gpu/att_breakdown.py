"""Row f2 time split by kernel class (library CUDA events) for the bench's batched call."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2305_18396_b200 as hl, synth  # noqa
from paper_2305_18396_b200 import attention  # noqa
ctx = hl.Context(8192, 3, 37, device=0)
dev = torch.device("cuda", 0)
items = []
for h in range(12):
    for (n, d, n2) in ((128, 64, 128), (128, 128, 64)):
        at = (ctx.plan_tile(n, d, n2), ctx.plan_tile(n2, d, n))
        sd = 77 + h * 100 + d
        X0, X1 = synth.activations(sd, n, d), synth.activations(sd + 1, n, d)
        Y0, Y1 = synth.activations(sd + 2, d, n2), synth.activations(sd + 3, d, n2)
        sk1, sk2 = ctx.keygen(sd + 4), ctx.keygen(sd + 5)
        items.append(dict(tile=at, X1=hl.to_device(X1, dev), Y1=hl.to_device(Y1, dev),
                          ct_Y0T=hl.to_device(ctx.encrypt(sk1, at[0], np.ascontiguousarray(Y0.T), sd + 6), dev),
                          ct_X0=hl.to_device(ctx.encrypt(sk2, at[1], X0, sd + 7), dev), seeds=(sd + 8, sd + 9)))
for _ in range(2):
    attention.server_cross_products(ctx, items)
torch.cuda.synchronize()
ctx.timing_enable(True); ctx.timing_read()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
attention.server_cross_products(ctx, items)
e1.record(); torch.cuda.synchronize()
print("total ms", round(e0.elapsed_time(e1), 3), {k: (round(v[0], 3), v[1]) for k, v in ctx.timing_read().items() if v[1]})
print("wcache MB per term:", {str(it["tile"]): ctx.layout(it["tile"][0], it["X1"].shape[0], it["X1"].shape[1], it["Y1"].shape[1]).wcache_bytes / 1e6 for it in items[:2]})
