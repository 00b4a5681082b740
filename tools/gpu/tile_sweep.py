"""Per-product tile sweep on the GPU (experiment): time hl_he_matmul_share of each product of a
config's block under candidate tiles (m, r, n), per kernel (library CUDA events), sequential, after
warm-up.

    python tools/gpu/tile_sweep.py [steps] [config] ["m,r,n;m,r,n;..."]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2305_18396_b200 as hl  # noqa: E402
import synth  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = synth.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c2"]
ctx = hl.Context(cfg.N, cfg.L, synth.T_BITS, device=0)
dev = torch.device("cuda", 0)
cands = [(16, 8, 32), (8, 16, 32), (32, 8, 16), (4, 32, 32), (8, 8, 64), (16, 16, 16), (32, 4, 32)]
if len(sys.argv) > 3:
    cands = [tuple(int(v) for v in t.split(",")) for t in sys.argv[3].split(";")]
for mi, mm in enumerate(cfg.block_shapes(cfg.seqs) if hasattr(cfg, "block_shapes") else cfg.matmuls):
    X = synth.activations(synth.seed_for(0, mi, "x"), mm.Nb, mm.R)
    W = synth.weights(synth.seed_for(0, mi, "w"), mm.R, mm.Ma)
    sk = ctx.keygen(synth.seed_for(0, mi, "key"))
    s_hat = ctx.sk_prepare(sk, dev)
    dX, dW = hl.to_device(X, dev), hl.to_device(W, dev)
    for tile in cands:
        m, r, n = tile
        if mm.R % r or mm.Ma % m or mm.Nb % n:
            continue
        try:
            ct = ctx.encrypt_device(s_hat, tile, dX, 5)
            wc = ctx.encode_weights(tile, dW)
        except hl.HLError as e:
            print(mm, tile, "skip", e)
            continue
        lay = ctx.layout(tile, mm.Ma, mm.R, mm.Nb)
        ws = torch.empty(lay.workspace_bytes // 8, dtype=torch.int64, device=dev)
        co = torch.empty(lay.ct_out_words, dtype=torch.int64, device=dev)
        cm = torch.empty(lay.ct_masked_words, dtype=torch.int64, device=dev)
        sh = torch.zeros(lay.share_words, dtype=torch.int64, device=dev)

        def run():
            ctx.he_matmul_share(tile, wc, mm.Ma, mm.R, mm.Nb, ct, 7, True, workspace=ws, ct_out_ntt=co,
                                ct_masked=cm, share=sh)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        ctx.timing_enable(True)
        ctx.timing_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            run()
        e1.record()
        torch.cuda.synchronize()
        tm = ctx.timing_read()
        ctx.timing_enable(False)
        ks = {k: round(1000 * v[0] / steps, 1) for k, v in tm.items() if v[1]}
        print(f"Ma={mm.Ma} R={mm.R} tile={tile} nI={lay.nI} nJ={lay.nJ} nK={lay.nK} wcache={lay.wcache_bytes/1e9:.2f}GB "
              f"total={1000 * e0.elapsed_time(e1) / steps:.1f}us {ks}", flush=True)
        del ws, co, cm, sh, wc, ct
        torch.cuda.empty_cache()
