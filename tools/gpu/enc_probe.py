"""Offline weight encoding of the c2 block: per-call wall time (synchronised), repeated."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2305_18396_b200 as hl, synth  # noqa
cfg = synth.CONFIGS["c2"]
ctx = hl.Context(cfg.N, cfg.L, 37, device=0)
dev = torch.device("cuda", 0)
for mi, mm in enumerate(cfg.matmuls):
    tile = cfg.tile_of(mi)
    dW = hl.to_device(synth.weights(synth.seed_for(0, mi, "w"), mm.R, mm.Ma), dev)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        wc = ctx.encode_weights(tile, dW)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(mm.name, tile, rep, f"{1e3 * (t1 - t0):.3f} ms", flush=True)
        del wc
