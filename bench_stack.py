"""bench_stack.py -- BASELINE configs 3 and 4: stacks of encoder blocks x sequences (bench.py --config c3|c4).

c3: 12 BERT-base blocks (hidden 768, FFN 3072), 8 sequences x 128 tokens, N = 4096, L = 2.
c4: 24 BERT-large blocks (hidden 1024, FFN 4096), 4 sequences x 512 tokens, N = 8192, L = 3.
Every block has independently seeded weights (synth.seed_for(block, product, "w")).

A step is the whole stack: every (layer, sequence) item's four encrypted products (SURVEY.md §8(a)
rows a3-a6).  The items are split layer-major over the ranks (dist.stack_plan); a rank merges its
items of one layer into one product set over their concatenated sequences (Nb = seq_len x #seqs)
and runs it with hl_he_linear_batch; every sequence's compressed responses go to its client-facing
rank (dist.StackRouter, P2P) inside the timed region.

Memory (180 GB HBM): the weight caches of a rank's layers stay resident (c3: 12 x 3.2 GB, c4:
24 x 4.2 GB at one GPU).  c3's input ciphertexts are resident too (12 x 2.8 GB).  c4's inputs are
22.5 GB per block (541 GB for the stack), so they are generated per item on the device (client
encryption, hl_encrypt_device) OUTSIDE the timed region: the step time is the sum of the items'
CUDA-event-timed server sections (bracketed by barriers).
"""
from __future__ import annotations

import os
import time

import numpy as np

import synth


def run_stack(args, rank, world, local_rank, B):
    """B: the bench module (shared helpers: ClockSampler, counts, path_roofline, mac_roofline, ...)."""
    import torch
    import paper_2305_18396_b200 as hl
    from paper_2305_18396_b200 import dist as hd

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = synth.CONFIGS[args.config]
    ctx = hl.Context(cfg.N, cfg.L, synth.T_BITS, device=local_rank)
    stream = torch.cuda.current_stream()
    plan = hd.stack_plan(cfg.blocks, cfg.seqs, world)
    mine = plan[rank]
    n_client = cfg.seqs                               # every sequence has its own client-facing rank
    router = hd.StackRouter(plan, world, rank, n_client) if world > 1 else None
    resident = cfg.name != "c4"                       # c4's inputs do not fit: generated per item
    LN = cfg.L * cfg.N

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([x], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    # ---------------- setup (untimed): weights of this rank's layers, keys, inputs
    items = []
    t_enc = 0.0
    # one tile per product for every item (the planner's choice at the block's full Nb): a sequence's
    # responses then have the same shape whichever rank produced them
    # The planner's tiles trade weight-cache bytes for fewer transforms; the rank's layers' caches
    # must stay resident, so above a budget of 55 % of HBM the config's default tile is used (c4 at
    # 1-2 GPUs: the planner's caches are 9.2 GB per block, 24 x 9.2 GB does not fit)
    full_shapes = cfg.block_shapes(cfg.seqs)
    tiles, tile_choice = choose_tiles(ctx, cfg, len({it.block for it in mine}),
                                      torch.cuda.get_device_properties(dev).total_memory, args.tile)
    for it in mine:
        shapes = cfg.block_shapes(it.nseq)
        prods = []
        for mi, (mm, tile) in enumerate(zip(shapes, tiles)):
            lay = ctx.layout(tile, mm.Ma, mm.R, mm.Nb)
            W = hl.to_device(synth.weights(synth.seed_for(it.block, mi, "w"), mm.R, mm.Ma), dev)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            wc = ctx.encode_weights(tile, W)
            torch.cuda.synchronize()
            t_enc += time.perf_counter() - t0
            del W
            sk = ctx.keygen(synth.seed_for(it.block, mi, "key"))
            X = hl.to_device(synth.activations_seq(synth.seed_for(it.block, mi, "x"), it.seq0, it.seq1, cfg.seq_len,
                                                   mm.R), dev)
            enc_seed = synth.seed_for(it.block, mi, "enc") + 7919 * it.seq0
            prods.append(dict(mm=mm, tile=tile, lay=lay, wc=wc, s_hat=ctx.sk_prepare(sk, dev), X=X, enc_seed=enc_seed,
                              seed=synth.seed_for(it.block, mi, "mask") + 7919 * it.seq0,
                              kps=cfg.seq_len // tile[2], per_ct=cfg.L * (tile[0] * tile[2] + cfg.N)))
        items.append(dict(it=it, prods=prods))
    # the batch runs the products one after the other at these sizes (nK >= 8: the adaptive serial
    # policy of hl_he_linear_batch), so the scratch is shared by the products and the items
    ws_words = max(p["lay"].workspace_bytes // 8 for i in items for p in i["prods"]) if items else 1
    co_words = max(p["lay"].ct_out_words for i in items for p in i["prods"]) if items else 1
    workspace = torch.empty(ws_words, dtype=torch.int64, device=dev)
    ct_out_ntt = torch.empty(co_words, dtype=torch.int64, device=dev)
    # c4: one input buffer per product (regenerated per item) and two alternating output sets per
    # product (a whole stack's responses, 185 GB, do not fit either); c3: everything resident
    nprod = len(cfg.matmuls)
    words_of = lambda f: [max((f(i["prods"][pi]) for i in items), default=1) for pi in range(nprod)]   # noqa: E731
    gen_in = None if resident else [torch.empty(w, dtype=torch.int64, device=dev)
                                    for w in words_of(lambda p: p["lay"].ct_in_words)]
    nout = 2 if world > 1 else 1        # alternate while the router may still read the previous item's
    out_sets = None if resident else [[(torch.empty(wm, dtype=torch.int64, device=dev),
                                        torch.zeros(ws_, dtype=torch.int64, device=dev))
                                       for wm, ws_ in zip(words_of(lambda p: p["lay"].ct_masked_words),
                                                          words_of(lambda p: p["lay"].share_words))]
                                      for _ in range(nout)]
    for k_, i in enumerate(items):
        for pi, p in enumerate(i["prods"]):
            if resident:
                p["ct"] = ctx.encrypt_device(p["s_hat"], p["tile"], p["X"], p["enc_seed"])
                p["masked"] = torch.empty(p["lay"].ct_masked_words, dtype=torch.int64, device=dev)
                p["share"] = torch.zeros(p["lay"].share_words, dtype=torch.int64, device=dev)
            else:
                p["ct"] = gen_in[pi][: p["lay"].ct_in_words]
                p["masked"] = out_sets[k_ % nout][pi][0][: p["lay"].ct_masked_words]
                p["share"] = out_sets[k_ % nout][pi][1][: p["lay"].share_words]
        if resident:
            for p in i["prods"]:
                del p["X"]            # the inputs are encrypted once (c3); c4 keeps X to encrypt per step
    torch.cuda.synchronize()
    rings = None
    if router is not None:                  # receive rings of this rank (its client-facing sequences)
        rings = []
        for mi in range(len(cfg.matmuls)):
            mm, t0_ = full_shapes[mi], tiles[mi]
            nI = -(-mm.Ma // t0_[0])
            words = nI * (cfg.seq_len // t0_[2]) * cfg.L * (t0_[0] * t0_[2] + cfg.N)
            rings.append(torch.empty(max(router.slots(), 1), words, dtype=torch.int64, device=dev))

    def gen_inputs(i):
        for p in i["prods"]:
            ctx.encrypt_device(p["s_hat"], p["tile"], p["X"], p["enc_seed"], ct_in=p["ct"], stream=stream)

    def run_item(i):
        ents = [dict(wcache=p["wc"], Ma=p["mm"].Ma, R=p["mm"].R, Nb=p["mm"].Nb, ct_in=p["ct"], seed=p["seed"],
                     tile=p["tile"], workspace=workspace, ct_out_ntt=ct_out_ntt, ct_masked=p["masked"],
                     share=p["share"]) for p in i["prods"]]
        ctx.he_linear_batch(i["prods"][0]["tile"], ents, stream=stream)

    def route(k):
        if router is None:
            return []
        works = []
        i = items[k] if k < len(items) else None
        for mi in range(len(cfg.matmuls)):
            p = i["prods"][mi] if i else None
            nI = p["lay"].nI if p else 0
            w, _ = router.route(k, mi, p["masked"] if p else None, nI, p["kps"] if p else 0,
                                p["per_ct"] if p else 0, rings[mi])
            works += w
        return works

    rounds = router.rounds if router else len(items)

    def step(timed_sections=None):
        """One stack pass; resident inputs: one timed region; else per item: generate (untimed) then
        time the server section with events (appended to timed_sections)."""
        works = []
        for k in range(rounds):
            if not resident:
                if k < len(items):
                    if timed_sections is not None:     # the client's encryption is not a server kernel
                        ctx.timing_enable(False)
                    gen_inputs(items[k])
                    if timed_sections is not None:
                        ctx.timing_enable(True)
                torch.cuda.synchronize()
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            if k < len(items):
                run_item(items[k])
            works += route(k)
            if not resident:
                for w in works:
                    w.wait()
                works = []
                e1.record(stream)
                torch.cuda.synchronize()
                if timed_sections is not None:
                    timed_sections.append(e0.elapsed_time(e1))
        for w in works:
            w.wait()

    for _ in range(args.warmup if resident else 1):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region
    clocks = B.ClockSampler(local_rank) if rank == 0 else None
    if clocks:
        clocks.start()
    ctx.timing_enable(True)
    ctx.timing_kernels()
    barrier()
    torch.cuda.synchronize()
    sections = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(sections)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ctx.timing_enable(False)
    if resident:
        elapsed = max_over_ranks(ev0.elapsed_time(ev1))
    else:   # per-section maxima over ranks (every section is bracketed by barriers)
        elapsed = sum(max_over_ranks(s) for s in sections)
    ktimes = ctx.timing_read()
    launches = ctx.timing_kernels()
    clk = clocks.stop() if clocks else None
    ms_step = elapsed / args.steps

    # ---------------- end to end on pinned host buffers (hl_he_linear_batch_host per item: the c0
    # halves + public seeds up in the 50-bit wire format, responses + shares down), over the first
    # e2e items of the rank, scaled to the rank's items (c4: pinned memory for the whole stack's
    # inputs would be 211 GB)
    n_e2e = len(items) if resident else min(len(items), max(1, args.e2e_items))
    e2e_ms = None
    h2d = d2h = 0
    if items:
        host = []
        for i in items[:n_e2e]:
            if not resident:
                gen_inputs(i)
                torch.cuda.synchronize()
            ents = []
            for pi, p in enumerate(i["prods"]):
                lay = p["lay"]
                v = p["ct"].view(-1, 2, LN)
                c0 = np.concatenate([v[a:a + 2048, 0].cpu().numpy() for a in range(0, v.shape[0], 2048)]).view(np.uint64)
                c0p = torch.from_numpy(hl.Context.pack50(c0).view(np.int64)).pin_memory()
                mw = int(hl._lib.hl_packed50_words(lay.ct_masked_words))
                # c4: the upload lands in the product's input buffer, the products share the scratch
                ents.append(dict(wcache=p["wc"], Ma=p["mm"].Ma, R=p["mm"].R, Nb=p["mm"].Nb,
                                 ct_in=(torch.empty(lay.ct_in_words, dtype=torch.int64, device=dev) if resident
                                        else p["ct"]), seed=p["seed"], tile=p["tile"],
                                 c0_host=c0p, a_seed=hl.public_seed(p["enc_seed"]), packed=True,
                                 masked_host=torch.empty(mw, dtype=torch.int64).pin_memory(),
                                 share_host=torch.empty(lay.share_words, dtype=torch.int64).pin_memory(),
                                 **({} if resident else dict(workspace=workspace, ct_out_ntt=ct_out_ntt,
                                                             ct_masked=p["masked"], share=p["share"]))))
                h2d += c0p.numel() * 8
                d2h += (mw + lay.share_words) * 8
            host.append(ents)

        def e2e_item(ents):
            if resident:     # the item's products pipelined (upload / compute / download)
                ctx.he_linear_batch_host(ents[0]["tile"], ents, stream=stream)
            else:            # c4: one product at a time (shared scratch)
                for e in ents:
                    ctx.he_linear_batch_host(e["tile"], [e], stream=stream)
        e2e_item(host[0])                   # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for ents in host:
            e2e_item(ents)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) * len(items) / n_e2e
        h2d = h2d * len(items) // n_e2e
        d2h = d2h * len(items) // n_e2e
        del host
    e2e_ms = max_over_ranks(e2e_ms or 0.0)

    if rank != 0:
        return None
    peaks = B._peaks()
    hbm = peaks.get("hbm_gbs") or 6650.0
    # algorithmic counts of the whole stack (all ranks' items): the per-block products at the full
    # Nb (the ranks' merged items partition them exactly)
    full_tiles = tiles
    lays = [ctx.layout(t, mm.Ma, mm.R, mm.Nb) for t, mm in zip(full_tiles, full_shapes)]
    cfg_full = synth.Config(cfg.name, cfg.N, cfg.L, cfg.tile, full_shapes)
    cnt_block = B.counts(cfg_full, lays, full_tiles)
    cnt = [dict(c, **{k: v * cfg.blocks for k, v in c.items() if isinstance(v, int)}) for c in cnt_block]
    roof = B.mac_roofline(B.counts(cfg_full, lays, full_tiles), ktimes, peaks) if ktimes["mac"][1] else None
    if roof:      # per launch at the planner's full-Nb tiles (a rank's merged items may be smaller)
        roof["note"] = ("per-launch algorithmic counts of the full-Nb products; this rank's "
                        f"{len(items)} item(s) x 4 products = {ktimes['mac'][1] // args.steps} MAC launches per step")
    total_k = sum(v[0] for v in ktimes.values())
    path_bytes = sum(c["path_bytes"] for c in cnt)
    products = sum(c["products"] for c in cnt)
    value = ms_step
    line = {
        "metric": f"ms per {cfg.name} stack step ({cfg.blocks} encoder blocks' encrypted matmuls x {cfg.seqs} sequences)",
        "value": round(value, 3), "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.note}", "N": cfg.N, "L": cfg.L, "t_bits": synth.T_BITS,
                   "blocks": cfg.blocks, "sequences": cfg.seqs, "seq_len": cfg.seq_len,
                   "tile": [list(t) for t in full_tiles],
                   "tile_choice": tile_choice,
                   "matmuls_per_block": [[mm.Nb, mm.R, mm.Ma] for mm in full_shapes],
                   "items_per_rank": [[(it.block, it.seq0, it.seq1) for it in p] for p in plan],
                   "inputs": ("resident in HBM" if resident else
                              "generated per item on the device (hl_encrypt_device) outside the timed sections; "
                              "the step = sum of the items' event-timed server sections"),
                   "l2": "inputs larger than L2 (weight caches of GBs per block)",
                   "parallelism": (f"{world} rank(s): layer-major (layer, sequence) items, responses routed to each "
                                   f"sequence's client-facing rank (P2P)" if world > 1 else "1 GPU, all items")},
        "ms_per_block": round(value / cfg.blocks, 3),
        "poly_products_per_s": products * args.steps / (elapsed * 1e-3),
        "path_bytes_per_step": path_bytes,
        "path_hbm_frac": path_bytes / (value * 1e-3) / (hbm * 1e9),
        "path_roofline": B.path_roofline(cnt, value, peaks),
        "roofline": roof,
        "kernels": {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps,
                        "share": v[0] / total_k if total_k else None} for k, v in ktimes.items() if v[1]},
        "gpu_launches": launches,
        "encode_weights_ms": round(t_enc * 1e3, 1),
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "call": ("hl_he_linear_batch_host per item" if resident else "hl_he_linear_batch_host per product") +
                        " (c0 halves + public seed up, 50-bit wire format both ways, responses + shares down)" +
                        ("" if n_e2e == len(items) else f"; measured on {n_e2e} of the rank's {len(items)} items, "
                         "scaled linearly (extrapolated)")},
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = stack_oracle_baseline(cfg, full_tiles, args.cpu_frac)
    return line


def choose_tiles(ctx, cfg, nblocks: int, hbm_bytes: float, override=None):
    """Per-product tiles of a stack: the planner's (hl_plan_tile at the block's full Nb) under a
    weight-cache budget (hl_plan_tile_budget) -- the caches of the rank's `nblocks` layers must stay
    resident in 55 % of HBM, shared by the products in proportion to their weights (c4 on one GPU:
    ~4 GB per block, where the unconstrained choice would take 22 GB)."""
    shapes = cfg.block_shapes(cfg.seqs)
    if override:
        return [tuple(override)] * len(shapes), "--tile override"
    per_block = 0.55 * hbm_bytes / max(nblocks, 1)
    tot = sum(mm.Ma * mm.R for mm in shapes)
    tiles = [tuple(ctx.plan_tile(mm.Ma, mm.R, mm.Nb, int(per_block * mm.Ma * mm.R / tot))) for mm in shapes]
    cache = sum(ctx.layout(t, mm.Ma, mm.R, mm.Nb).wcache_bytes for t, mm in zip(tiles, shapes))
    return tiles, (f"per product, hl_plan_tile_budget (DESIGN.md §5): weight caches {cache / 1e9:.2f} GB per block "
                   f"within 55 % of HBM over {nblocks} layer(s)")


def stack_oracle_baseline(cfg, tiles, frac: float, seed: int = 5):
    """The CPU oracle as it stands on a uniformly random sample of `frac` of one block's output
    ciphertexts per product (oracle he_matmul through its own scalar NTT -- SURVEY.md §8(d): the
    c3/c4 oracle path -- plus the mask), scaled by total / sampled output ciphertexts (oracle work is
    linear in them; every block of the stack has the same shapes): extrapolated."""
    from oracle import ref
    P = ref.bfv_params(cfg.N, cfg.L, synth.T_BITS)
    rng = np.random.default_rng(seed)
    total_s, sampled, total = 0.0, 0, 0
    for mi, (mm, tile) in enumerate(zip(cfg.block_shapes(cfg.seqs), tiles)):
        nI, nJ, nK = ref.tile_counts(tile, mm.Ma, mm.R, mm.Nb)
        ns = max(1, int(round(frac * nI * nK)))
        pick = rng.choice(nI * nK, size=ns, replace=False)
        smp = [(int(o) // nK, int(o) % nK) for o in pick]
        W = synth.weights(synth.seed_for(0, mi, "w"), mm.R, mm.Ma)
        ct_in = synth.uniform_below(synth.seed_for(0, mi, "enc"), (nJ, nK, 2, P.L, P.N), P.primes)
        t0 = time.perf_counter()
        ct = ref.he_matmul_ntt_tiles(P, tile, W, ct_in, mm.Nb, smp)
        ref.mask_tiles(P, tile, ct, nK, smp, 1, True)
        total_s += (time.perf_counter() - t0) * (nI * nK) / ns
        sampled += ns
        total += nI * nK
    cores = len(os.sched_getaffinity(0))
    return {"value": round(total_s * 1e3 * cfg.blocks, 1), "unit": "ms", "cores": cores, "kind": "oracle",
            "sample": f"{sampled} of {total} output ciphertexts of one block ({100 * frac:.2g} % per product, uniform "
                      f"random), oracle scalar-NTT he_matmul + mask, scaled to the block and x {cfg.blocks} blocks "
                      "(extrapolated)",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None
