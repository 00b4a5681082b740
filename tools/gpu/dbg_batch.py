import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, synth, sys
import paper_2305_18396_b200 as hl
from oracle import ref
ctx = hl.Context(4096, 2, 37, device=0)
cfg = synth.CONFIGS["c1"]; P = ref.bfv_params(4096, 2, 37)
ins = []
for mi, mm in enumerate(cfg.matmuls):
    W = synth.weights(synth.seed_for(0, mi, "w"), mm.R, mm.Ma)
    nI, nJ, nK = ref.tile_counts(cfg.tile, mm.Ma, mm.R, mm.Nb)
    ct_in = synth.uniform_below(synth.seed_for(0, mi, "enc"), (nJ, nK, 2, P.L, P.N), P.primes)
    ins.append((mm, W, ct_in, synth.seed_for(0, mi, "mask")))
entries = [dict(wcache=ctx.encode_weights(cfg.tile, hl.to_device(W)), Ma=mm.Ma, R=mm.R, Nb=mm.Nb, ct_in=hl.to_device(ct), seed=sd) for mm, W, ct, sd in ins]
for rep in range(3):
    outs = ctx.he_linear_batch(cfg.tile, entries); torch.cuda.synchronize()
    single = [ctx.he_matmul_share(cfg.tile, e["wcache"], e["Ma"], e["R"], e["Nb"], e["ct_in"], seed=e["seed"]) for e in entries]
    torch.cuda.synchronize()
    res = []
    for (mm, W, ct, sd), (m, s), (m2, s2) in zip(ins, outs, single):
        em, es = ref.mask_and_share(P, cfg.tile, ref.he_matmul(P, cfg.tile, W, ct, mm.Nb), mm.Ma, mm.Nb, sd)
        a = hl.to_host(m).reshape(em.shape); b = hl.to_host(m2).reshape(em.shape)
        res.append((mm.name, int((a != em).sum()), int((b != em).sum()), em.size))
    print(rep, res, flush=True)
