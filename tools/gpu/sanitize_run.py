"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck), SURVEY.md §5.

    compute-sanitizer --tool memcheck python tools/gpu/sanitize_run.py [c0|c1|all]

Runs configs c0 and c1 through the server calls a user makes -- hl_he_matmul_share,
hl_he_linear_batch (the bench's call, two streams) and hl_he_linear_batch_host (seeded upload,
50-bit wire format), plus one fat product (CW = 16, k_c1_tx16) -- and checks every result bit for
bit against the oracle, so a sanitizer run is also a parity run.  Prints one line per check.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import ref  # noqa: E402


def main(which: str):
    import torch
    import paper_2305_18396_b200 as hl
    ctx = hl.Context(4096, 2, synth.T_BITS, device=0)
    P = ref.bfv_params(4096, 2, synth.T_BITS)
    cases = []
    if which in ("c0", "all"):
        cases.append(("c0", synth.CONFIGS["c0"], [synth.CONFIGS["c0"].tile]))
    if which in ("c1", "all"):
        cfg = synth.CONFIGS["c1"]
        cases.append(("c1", cfg, [cfg.tile] * len(cfg.matmuls)))
    for name, cfg, tiles in cases:
        entries, exp, hosts = [], [], []
        for mi, (mm, tile) in enumerate(zip(cfg.matmuls, tiles)):
            X = synth.activations(synth.seed_for(0, mi, "x"), mm.Nb, mm.R)
            W = synth.weights(synth.seed_for(0, mi, "w"), mm.R, mm.Ma)
            sk = ref.keygen(P, synth.seed_for(0, mi, "key"))
            es = synth.seed_for(0, mi, "enc")
            ct = ref.encrypt(P, tile, sk, X, es)
            seed = synth.seed_for(0, mi, "mask")
            wc = ctx.encode_weights(tile, hl.to_device(W))
            em, esh = ref.mask_and_share(P, tile, ref.he_matmul(P, tile, W, ct, mm.Nb), mm.Ma, mm.Nb, seed)
            exp.append((em, esh))
            # single fused call
            m, sh = ctx.he_matmul_share(tile, wc, mm.Ma, mm.R, mm.Nb, hl.to_device(ct), seed=seed)
            torch.cuda.synchronize()
            ok = np.array_equal(hl.to_host(m).reshape(em.shape), em) and np.array_equal(hl.to_host(sh).reshape(esh.shape), esh)
            print(f"{name} {mm.name} he_matmul_share {'ok' if ok else 'MISMATCH'}", flush=True)
            entries.append(dict(wcache=wc, Ma=mm.Ma, R=mm.R, Nb=mm.Nb, tile=tile, ct_in=hl.to_device(ct), seed=seed))
            lay = ctx.layout(tile, mm.Ma, mm.R, mm.Nb)
            c0 = torch.from_numpy(hl.Context.pack50(hl.Context.c0_halves(ct)).view(np.int64)).pin_memory()
            mw = hl.Context.pack50(np.zeros(lay.ct_masked_words, np.uint64)).size
            hosts.append(dict(entries[-1], ct_in=torch.empty(lay.ct_in_words, dtype=torch.int64, device="cuda"),
                              c0_host=c0, a_seed=ref.public_seed(es), packed=True,
                              masked_host=torch.zeros(mw, dtype=torch.int64).pin_memory(),
                              share_host=torch.zeros(lay.share_words, dtype=torch.int64).pin_memory()))
        outs = ctx.he_linear_batch(tiles[0], entries)
        torch.cuda.synchronize()
        ok = all(np.array_equal(hl.to_host(m).reshape(em.shape), em) and np.array_equal(hl.to_host(sh).reshape(es_.shape), es_)
                 for (m, sh), (em, es_) in zip(outs, exp))
        print(f"{name} he_linear_batch {'ok' if ok else 'MISMATCH'}", flush=True)
        ctx.he_linear_batch_host(tiles[0], hosts)
        torch.cuda.synchronize()
        ok = all(np.array_equal(hl.Context.unpack50(h["masked_host"].numpy().view(np.uint64), em.size).reshape(em.shape), em)
                 and np.array_equal(h["share_host"].numpy().view(np.uint64).reshape(es_.shape), es_)
                 for h, (em, es_) in zip(hosts, exp))
        print(f"{name} he_linear_batch_host {'ok' if ok else 'MISMATCH'}", flush=True)
    if which in ("fat", "all"):          # CW = 16 MAC + the c1 transposition (c3-like columns, small)
        Nb, R, Ma, tile = 256, 48, 40, (16, 8, 16)
        nI, nJ, nK = ref.tile_counts(tile, Ma, R, Nb)
        W = synth.weights(1200, R, Ma)
        ct_in = synth.uniform_below(1210, (nJ, nK, 2, P.L, P.N), P.primes)
        e = dict(wcache=ctx.encode_weights(tile, hl.to_device(W)), Ma=Ma, R=R, Nb=Nb, tile=tile,
                 ct_in=hl.to_device(ct_in), seed=1220)
        (m, sh), = ctx.he_linear_batch(tile, [e])
        torch.cuda.synchronize()
        em, es_ = ref.mask_and_share(P, tile, ref.he_matmul(P, tile, W, ct_in, Nb), Ma, Nb, 1220)
        ok = np.array_equal(hl.to_host(m).reshape(em.shape), em) and np.array_equal(hl.to_host(sh).reshape(es_.shape), es_)
        print(f"fat CW=16 he_linear_batch {'ok' if ok else 'MISMATCH'}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
