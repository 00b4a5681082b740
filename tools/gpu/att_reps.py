"""Row f2: per-rep device time and host dispatch time of the bench's batched call (is it host-bound?)."""
import os, sys, time
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
attention.server_cross_products(ctx, items)
torch.cuda.synchronize()
for rep in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    attention.server_cross_products(ctx, items)
    t1 = time.perf_counter()
    e1.record(); torch.cuda.synchronize()
    print(f"rep {rep}: device {e0.elapsed_time(e1):.3f} ms, host dispatch {1e3 * (t1 - t0):.3f} ms")
