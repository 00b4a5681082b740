import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2305_18396_b200 as hl, synth
ctx = hl.Context(8192, 3, 37, device=0)
dev = torch.device("cuda", 0)
for tile in [(32,16,16),(8,8,128)]:
    dY1 = hl.to_device(synth.activations(5, 64, 128), dev)
    for _ in range(3): ctx.encode_weights(tile, dY1)
    torch.cuda.synchronize()
    ctx.timing_enable(True); ctx.timing_read()
    t0=time.perf_counter()
    for _ in range(10): ctx.encode_weights(tile, dY1)
    torch.cuda.synchronize(); dt=(time.perf_counter()-t0)*100
    print(tile, 'host ms per encode', round(dt,3), {k:(round(v[0]/10,4),v[1]) for k,v in ctx.timing_read().items() if v[1]})
    ctx.timing_enable(False)
