"""bench.py -- the server's homomorphic linear layers of one BERT-base encoder block (config c2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step is one pass of the whole hot path over one BERT-base
block: for each of the four encrypted products X.W_qkv, X.W_o, X.W_1, H.W_2 -- forward NTT
of the client's ciphertexts, modular MAC against the cached NTT-domain weights, inverse NTT,
mask + compression + server share (hl_he_linear_batch).  Weights are encoded once before
timing (offline, reported separately); input ciphertexts are resident in HBM.  Multi-GPU
(default for N > 1, BASELINE config 2 "sharded by output columns"): strong scaling -- the I
tiles of every product are split over the ranks and the compressed responses are gathered to
rank 0 point to point inside the timed region (paper_2305_18396_b200/dist.py); `--mode weak`
runs one independent block per rank instead.  `--config c3|c4` runs the stacks of BASELINE
configs 3 and 4 (bench_stack.py).

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (oracle/) on a
bounded sample of the same workload instead (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "ms per BERT-base encoder block's encrypted matmuls"
IMAD_WIDE_PER_CLK_SM = 24.4      # measured peak, profiles/r01/microbench_intpipe3.log
DFMA_PER_CLK_SM = 57.3           # measured peak (same run): the FP64 pipe of the default MAC engine
FP64_OPS_PER_MAC = 4.125         # 3 DFMA + 1 DADD per modular MAC + 1 DMUL per 8 (k_mac_f64)
FP64_OPS_PER_BFLY = 10.0         # exact modular butterfly (mm_d 6 + add/sub 2) + reductions (2 amortised)
UNIT = "ms"


def ref_primes(cfg):
    """The primes of the config (reading C4) from the library's own context -- for input ranges only."""
    import paper_2305_18396_b200 as hl
    c = hl.Context(cfg.N, cfg.L, synth.T_BITS, device=-1)
    return c.primes


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ----------------------------------------------------------------------------- algorithmic counts
def counts(cfg, lay_by_mm, tiles):
    """Per-matmul algorithmic work: MACs, butterflies, bytes of each kernel."""
    N, L = cfg.N, cfg.L
    out = []
    logN = N.bit_length() - 1
    for mm, lay, (m, r, n) in zip(cfg.matmuls, lay_by_mm, tiles):
        nI, nJ, nK = lay.nI_shard, lay.nJ, lay.nK     # this rank's I tiles
        nC = 2 * nK
        P = nI * nJ * nK
        out.append(dict(
            name=mm.name, products=P,
            mac=P * 2 * L * N,                                   # modular MACs
            bfly_fwd=nJ * nC * L * (N // 2) * logN,
            bfly_inv=nI * nC * L * (N // 2) * logN,
            # MAC kernel bytes: weight cache + NTT-domain ct_in (read once) + NTT-domain output
            mac_bytes=8 * (-(-nI // 16) * 16 * nJ * L * N + nJ * nC * L * N + nI * nC * L * N),
            # tensor-core engine: weight residues as 7 byte limbs (the least whole bytes of a
            # 50-bit residue), ct_in residues and outputs as u64, each read/written once
            mac_bytes_tc=(7 * nI * nJ + 8 * nJ * nC + 8 * nI * nC) * L * N,
            fwd_bytes=8 * 2 * nJ * nC * L * N,                   # coefficient ct_in in, limb pairs out
            inv_bytes=8 * (nI * nC * L * N + nI * nK * L * (m * n + N) + mm.Nb * mm.Ma),
            # whole-path algorithmic bytes (SURVEY.md §8(d) "Bytes")
            path_bytes=8 * (nJ * nK * 2 * L * N + nI * nJ * L * N + nI * nK * L * (N + m * n) + mm.Nb * mm.Ma),
            # the method's transforms (reading C26: c1 travels in evaluation form, so only the c0
            # halves are transformed, forward for the inputs, inverse for the outputs)
            bfly_c0=(nJ * nK + nI * nK) * L * (N // 2) * logN,
        ))
    return out


U8_PER_MAC = 49                  # 7 x 7 byte-limb products per modular MAC on the int8 tensor cores
INT8_PER_BF16 = 2.0              # nominal dense ratio int8 / bf16 (B200_PROFILING.md: 4.5 vs 2.25 PFLOP/s)


def peak_rates(peaks):
    """(HBM B/s, int8 tensor op/s, FP64 butterflies/s) and their sources."""
    hbm = peaks.get("hbm_gbs")
    hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if hbm else "fallback 6650 GB/s (B200_PROFILING.md)"
    hbm = (hbm or 6650.0) * 1e9
    bf16 = peaks.get("bf16_tflops")
    tc = (bf16 or 2250.0) * INT8_PER_BF16 * 1e12
    tc_src = ("MEASURED_PEAKS.json bf16_tflops (burst) x 2 (nominal int8/bf16 ratio)" if bf16
              else "fallback 4.5 POPS int8 dense (B200_PROFILING.md)")
    sm_max = peaks.get("sm_max_mhz") or 1965.0
    bfly = DFMA_PER_CLK_SM * 148 * sm_max * 1e6 / FP64_OPS_PER_BFLY
    return hbm, tc, bfly, {"hbm": hbm_src, "tc": tc_src,
                           "fp64": f"DFMA {DFMA_PER_CLK_SM}/clk/SM (tools/microbench/intpipe3.cu) x 148 x sm_max / "
                                   f"{FP64_OPS_PER_BFLY} FP64 ops per butterfly"}


def path_roofline(cnt, ms, peaks):
    """Whole-path roofline: the slowest of HBM (algorithmic bytes), the int8
    tensor cores (49 u8 MACs per modular MAC, 2 ops each) and the FP64 pipe (c0 transforms) bounds
    the step; frac = that bound / the measured time."""
    hbm, tc, bfly, _ = peak_rates(peaks)
    t = {"hbm": sum(c["path_bytes"] for c in cnt) / hbm,
         "tensor": 2 * U8_PER_MAC * sum(c["mac"] for c in cnt) / tc,
         "fp64": sum(c["bfly_c0"] for c in cnt) / bfly}
    bound = max(t, key=t.get)
    return {"t_hbm_ms": t["hbm"] * 1e3, "t_tensor_ms": t["tensor"] * 1e3, "t_fp64_ms": t["fp64"] * 1e3,
            "bound": bound, "frac": t[bound] * 1e3 / ms,
            "note": "max(T_hbm, T_tensor, T_fp64) / measured ms per block; the three overlap in the pipeline"}


def mac_roofline(cnt, ktimes, peaks):
    """Roofline object of the dominant kernel k_mac_tc: the binding one of HBM (weight planes +
    NTT-domain inputs + outputs, per launch) and the int8 tensor cores (49 u8 MACs per modular MAC)."""
    hbm, tc, _, src = peak_rates(peaks)
    mac_ms, mac_n = ktimes["mac"]
    mac_avg_s = mac_ms / max(mac_n, 1) * 1e-3
    n = len(cnt)
    per_bytes = sum(c["mac_bytes_tc"] for c in cnt) / n
    per_ops = 2 * U8_PER_MAC * sum(c["mac"] for c in cnt) / n
    if per_ops / tc > per_bytes / hbm:
        roof = {"bound": "tensor", "achieved": per_ops / mac_avg_s / 1e12, "peak": tc / 1e12, "unit": "TOPS (int8)",
                "peak_source": src["tc"]}
    else:
        roof = {"bound": "hbm", "achieved": per_bytes / mac_avg_s / 1e9, "peak": hbm / 1e9, "unit": "GB/s",
                "peak_source": src["hbm"]}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["hbm_frac_same_kernel"] = per_bytes / mac_avg_s / hbm
    roof["tensor_frac_same_kernel"] = per_ops / mac_avg_s / tc
    roof["algorithmic_bytes_per_launch"] = per_bytes
    roof["algorithmic_int8_ops_per_launch"] = per_ops
    roof["kernel"] = "k_mac_tc (slot-parallel modular MAC, int8 tensor cores)"
    roof["traffic"] = None
    return roof


# ----------------------------------------------------------------------------- clocks sampler
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2305_18396_b200 as hl

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = synth.CONFIGS[args.config]
    tiles = _tiles(cfg, args)
    ctx = hl.Context(cfg.N, cfg.L, synth.T_BITS, device=local_rank)
    if args.plan:                        # every product at the planner's tile (configs without recorded tiles)
        tiles = [tuple(ctx.plan_tile(mm.Ma, mm.R, mm.Nb)) for mm in cfg.matmuls]
    elif not args.tile and not args.tiles and cfg.tiles:    # the bench's tiles are the library planner's choices (hl_plan_tile)
        assert all(ctx.plan_tile(mm.Ma, mm.R, mm.Nb) == t for mm, t in zip(cfg.matmuls, tiles)), 'planner drift'
    # shard (the default for N > 1, BASELINE config 2 "sharded by output columns"): one block; the I
    #   tiles (output columns) of its four products are split over the ranks, every
    #   rank runs hl_he_linear_batch on its shards and the compressed responses are gathered to rank 0
    #   point to point, overlapped with the next step's compute (two alternating output sets).
    # weak (--mode weak): every rank owns one independently seeded block, no data-path collective.
    shard = args.mode == "shard" or (args.mode == "auto" and world > 1)
    block = 0 if shard else rank
    stream = torch.cuda.current_stream()

    # ---------------- setup (untimed): client encryption on the host, weight encoding on device
    mats = []
    t_enc = 0.0
    from paper_2305_18396_b200 import dist as hd
    for mi, mm in enumerate(cfg.matmuls):
        tile = tiles[mi]
        nI_full = ctx.layout(tile, mm.Ma, mm.R, mm.Nb).nI
        i0, i1 = hd.shard_range(nI_full, world, rank) if shard else (0, nI_full)
        lay = ctx.layout(tile, mm.Ma, mm.R, mm.Nb, i0, i1)
        X = synth.activations(synth.seed_for(block, mi, "x"), mm.Nb, mm.R)
        W = synth.weights(synth.seed_for(block, mi, "w"), mm.R, mm.Ma)
        sk = ctx.keygen(synth.seed_for(block, mi, "key"))
        s_hat = ctx.sk_prepare(sk, dev)
        dX = hl.to_device(X, dev)
        ct_dev = ctx.encrypt_device(s_hat, tile, dX, synth.seed_for(block, mi, "enc"))   # row f3, == encrypt()
        ct_host = hl.to_host(ct_dev)
        dW = hl.to_device(W, dev)
        # offline encoding, timed warm: the first call pays one-off costs (lazy module loading, the
        # allocation of the cache), so it is repeated and the second call timed
        del_wc = ctx.encode_weights(tile, dW, i0, i1)
        torch.cuda.synchronize()
        del del_wc                    # its blocks return to torch's allocator cache for the timed calls
        best = None
        for _ in range(3):            # best of 3 (host-side allocation jitter)
            t0 = time.perf_counter()
            wc = ctx.encode_weights(tile, dW, i0, i1)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
            if _ < 2:
                del wc
        t_enc += best
        del dW
        mats.append(dict(mm=mm, tile=tile, lay=lay, wc=wc, ct=ct_dev, i0=i0, i1=i1, nI_full=nI_full, s_hat=s_hat, dX=dX,
                         ct_host=torch.from_numpy(ct_host.view(np.int64).reshape(-1)).pin_memory(),
                         c0_host=torch.from_numpy(hl.Context.c0_halves(ct_host.reshape(lay.nJ, lay.nK, 2, -1)).view(np.int64).reshape(-1)).pin_memory(),
                         a_seed=hl.public_seed(synth.seed_for(block, mi, "enc")),   # reading C28
                         seed=synth.seed_for(block, mi, "mask")))
    ws_words = max(m["lay"].workspace_bytes // 8 for m in mats)
    out_words = max(m["lay"].ct_out_words for m in mats)
    workspace = torch.empty(ws_words, dtype=torch.int64, device=dev)
    ct_out_ntt = torch.empty(out_words, dtype=torch.int64, device=dev)
    nsets = 2 if shard and world > 1 else 1          # output sets alternate between steps when gathering
    gathers, full = [], [[None] * len(mats) for _ in range(nsets)]
    for mi, m in enumerate(mats):
        mm, tile = m["mm"], m["tile"]
        per_ct = cfg.L * (tile[0] * tile[2] + cfg.N)
        m["per_ct"] = per_ct
        m["sets"] = []
        if shard and world > 1:
            g = hd.ResponseGather(m["nI_full"], m["lay"].nK, per_ct, dst=0)
            gathers.append(g)
        for si in range(nsets):
            if shard and world > 1 and rank == 0:       # rank 0 computes its rows in place in the full buffer
                full[si][mi] = torch.empty(m["nI_full"] * m["lay"].nK * per_ct, dtype=torch.int64, device=dev)
                w0, w1 = gathers[-1].words(0)
                masked = full[si][mi][w0:w1]
            else:
                masked = torch.empty(max(m["lay"].ct_masked_words, 1), dtype=torch.int64, device=dev)
            m["sets"].append((masked, torch.zeros(m["lay"].share_words, dtype=torch.int64, device=dev)))
        m["masked"], m["share"] = m["sets"][0]

    # every product gets its own scratch: the batch call pipelines them over two streams
    for m in mats:
        m["ws"] = torch.empty(m["lay"].workspace_bytes // 8, dtype=torch.int64, device=dev)
        m["co"] = torch.empty(m["lay"].ct_out_words, dtype=torch.int64, device=dev)
    entries = [dict(wcache=m["wc"], Ma=m["mm"].Ma, R=m["mm"].R, Nb=m["mm"].Nb, ct_in=m["ct"], seed=m["seed"], tile=m["tile"],
                    workspace=m["ws"], ct_out_ntt=m["co"], ct_masked=m["masked"], share=m["share"],
                    i_begin=m["i0"], i_end=m["i1"]) for m in mats]

    # the four products are independent: submit them in the order measured fastest for the pipeline
    # (tools/gpu/order_sweep.sh, all 24 orders; synth Config.batch_order)
    order = list(cfg.batch_order) if cfg.batch_order else list(range(len(entries)))
    batch = [entries[i] for i in order]
    # e2e: PCIe-bound (the downloads start once the first product is done): experiment knob
    e2e_order = ([int(x) for x in os.environ["BENCH_E2E_ORDER"].split(",")] if os.environ.get("BENCH_E2E_ORDER")
                 else list(cfg.e2e_order) if cfg.e2e_order else order)

    pending = [[] for _ in range(nsets)]
    nstep = [0]

    def step():
        if shard:
            si = nstep[0] % nsets
            nstep[0] += 1
            for w in pending[si]:          # the gather that last read this output set is done
                w.wait()
            ents = [dict(entries[i], ct_masked=mats[i]["sets"][si][0], share=mats[i]["sets"][si][1]) for i in order]
            ctx.he_linear_batch(tiles[0], ents, stream=stream)
            if world > 1:                  # P2P to rank 0 on NCCL's stream, overlapping the next step
                pending[si] = [w for i in order for w in gathers[i].post(mats[i]["sets"][si][0], full[si][i])]
        elif args.sequential:
            for m in mats:
                mm, tile = m["mm"], m["tile"]
                ctx.he_matmul_share(tile, m["wc"], mm.Ma, mm.R, mm.Nb, m["ct"], m["seed"], True,
                                    workspace=workspace, ct_out_ntt=ct_out_ntt, ct_masked=m["masked"],
                                    share=m["share"], stream=stream)
        else:
            ctx.he_linear_batch(tiles[0], batch, stream=stream)

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

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region (device events on the launching stream)
    clocks = ClockSampler(local_rank) if rank == 0 else None
    if clocks:
        clocks.start()
    ctx.timing_enable(True)
    ctx.timing_kernels()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    for ws_ in pending:                    # the timed region ends when rank 0 holds every response
        for w in ws_:
            w.wait()
    pending = [[] for _ in range(nsets)]
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ctx.timing_enable(False)
    elapsed = max_over_ranks(ev0.elapsed_time(ev1))
    # the device path's results, kept for the e2e check (rows f1/f4 below write into m["share"])
    dev_results = [(m["masked"].clone(), m["share"].clone()) for m in mats]
    ktimes = ctx.timing_read()
    kernels_launched = ctx.timing_kernels()
    clk = clocks.stop() if clocks else None

    # ---------------- standalone batched NTT microbenchmark: forward + inverse
    # negacyclic transforms of 4096 polynomials x L primes in place (hl_ntt_roundtrip), CUDA events
    ntt_info = None
    if not shard:
        npoly = 4096
        xs = hl.to_device(synth.uniform_below(77, (npoly, cfg.L, cfg.N), ref_primes(cfg)), dev)
        scratch = torch.empty_like(xs)
        for _ in range(3):
            ctx.ntt_roundtrip(xs, scratch, stream=stream)
        torch.cuda.synchronize()
        ctx.timing_enable(True)
        ctx.timing_read()
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nrep = 10
        n0.record(stream)
        for _ in range(nrep):
            ctx.ntt_roundtrip(xs, scratch, stream=stream)
        n1.record(stream)
        torch.cuda.synchronize()
        kt = ctx.timing_read()
        ctx.timing_enable(False)
        transforms = 2 * npoly * cfg.L * nrep
        logn = cfg.N.bit_length() - 1
        bfly = transforms * (cfg.N // 2) * logn
        sec = n0.elapsed_time(n1) * 1e-3
        peak_bfly = DFMA_PER_CLK_SM * 148 * (_peaks().get("sm_max_mhz") or 1965.0) * 1e6 / FP64_OPS_PER_BFLY
        ntt_info = {"what": f"forward + inverse negacyclic NTT, {npoly} polynomials x {cfg.L} primes, N={cfg.N}, "
                            "exact FP64 butterflies (hl_ntt_roundtrip)",
                    "transforms_per_s": round(transforms / sec, 1), "butterflies_per_s": round(bfly / sec, 1),
                    "fp64_roofline_frac": round(bfly / sec / peak_bfly, 3),
                    "roofline_note": f"peak = DFMA {DFMA_PER_CLK_SM}/clk/SM x 148 SMs x max clock / "
                                     f"{FP64_OPS_PER_BFLY} FP64 ops per butterfly (8 for the exact modular "
                                     "butterfly + 2 for the lazy reductions every other stage)",
                    "kernel_ms": {k: round(v[0] / nrep, 4) for k, v in kt.items() if v[1]}}
        del xs, scratch

    # ---------------- row f1: the server's FC share assembly, share += X1.W + b,
    # timed separately (it is not part of the Pi_MatMul metric): device-resident inputs, events
    fc_info = None
    if not shard:
        fc_in = []
        for mi, m in enumerate(mats):
            mm = m["mm"]
            W = synth.weights(synth.seed_for(block, mi, "w"), mm.R, mm.Ma)
            fc_in.append(dict(X1=hl.to_device(synth.activations(synth.seed_for(block, mi, "x") + 7, mm.Nb, mm.R), dev),
                              wp=ctx.fc_encode_weights(hl.to_device(W, dev)),
                              b=hl.to_device(synth.activations(synth.seed_for(block, mi, "x") + 8, 1, mm.Ma)[0], dev),
                              mm=mm, share=m["share"]))

        def fc_step():
            for f in fc_in:
                ctx.fc_local_share(f["X1"], f["wp"], f["mm"].Ma, f["share"], bias=f["b"], stream=stream)
        for _ in range(3):
            fc_step()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            fc_step()
        f1.record(stream)
        torch.cuda.synchronize()
        fc_ms = f0.elapsed_time(f1) / args.steps
        fc_macs = sum(f["mm"].Nb * f["mm"].R * f["mm"].Ma for f in fc_in)
        fc_info = {"what": "server FC share assembly share += X1.W + b mod 2^37 (row f1, PAPER.md:106-111), "
                           "4 products of the block, int8 tensor cores (15 limb MMAs per 32-K step)",
                   "ms_per_block": round(fc_ms, 4), "plaintext_macs": fc_macs,
                   "gmacs_per_s": round(fc_macs / (fc_ms * 1e-3) / 1e9, 1)}

    # ---------------- row f3: the client side of the block on the GPU -- encryption of the four
    # inputs (pi_B + secret-key BFV) and decryption of the four compressed responses
    # (PAPER.md:101, 154); CUDA events, device-resident buffers
    cli_info = None
    if not shard:
        cts = [torch.empty_like(m["ct"]) for m in mats]
        shc = [torch.empty(m["lay"].share_words, dtype=torch.int64, device=dev) for m in mats]

        def enc_step():
            for m, ct in zip(mats, cts):
                ctx.encrypt_device(m["s_hat"], m["tile"], m["dX"], synth.seed_for(block, 0, "enc") + 99, ct_in=ct,
                                   stream=stream)

        def dec_step():
            for m, sh in zip(mats, shc):
                ctx.decrypt_share_device(m["s_hat"], m["tile"], m["masked"], m["mm"].Ma, m["mm"].Nb, share=sh,
                                         stream=stream)
        enc_step(); dec_step()
        torch.cuda.synchronize()
        nrep = max(2, min(args.steps, 10))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        for _ in range(nrep):
            enc_step()
        ev[1].record(stream)
        for _ in range(nrep):
            dec_step()
        ev[2].record(stream)
        torch.cuda.synchronize()
        cli_info = {"what": "client side of the block on the GPU (row f3): encrypt the 4 inputs (2688 ciphertexts), "
                            "decrypt the 4 compressed responses (1728), bit-identical to the host client / oracle",
                    "encrypt_ms_per_block": round(ev[0].elapsed_time(ev[1]) / nrep, 3),
                    "decrypt_ms_per_block": round(ev[1].elapsed_time(ev[2]) / nrep, 3)}

    # ---------------- row f4 (reading C22): the block with re-randomised, flooded responses
    # (fresh pk-encryption of zero + 2^57 flood per response), sequential calls
    rr_info = None
    if not shard:
        sk_rr = ctx.keygen(synth.seed_for(block, 0, "key") + 11)
        pk_hat = ctx.pk_prepare(ctx.pk_gen(sk_rr, synth.seed_for(block, 0, "key") + 12))

        def rr_step():
            for m in mats:
                mm = m["mm"]
                ctx.he_matmul_share_rr(m["tile"], m["wc"], mm.Ma, mm.R, mm.Nb, m["ct"], m["seed"], pk_hat, 58, stream=stream)
        rr_step()
        torch.cuda.synchronize()
        nrep = max(2, min(args.steps, 10))
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(nrep):
            rr_step()
        r1.record(stream)
        torch.cuda.synchronize()
        rr_info = {"what": "the block's 4 products with re-randomised responses (row f4: + Enc_pk(0), 58-bit flood), "
                           "sequential hl_he_matmul_share_rr", "ms_per_block": round(r0.elapsed_time(r1) / nrep, 4)}

    # ---------------- row f2: the server side of one BERT-base block's attention
    # cross terms, 12 heads x (Q K^T: 128x64 . 64x128, A V: 128x128 . 128x64), both inputs shared;
    # N=8192, L=3 (uniform shares as server operands need q ~ 2^150), per-term planner tiles.
    att_info = None
    if not shard and not args.no_attention:
        from paper_2305_18396_b200 import attention
        actx = hl.Context(8192, 3, synth.T_BITS, device=local_rank)
        heads = []
        atiles = {}
        for h in range(12):
            for (n, d, n2) in ((128, 64, 128), (128, 128, 64)):
                # per-term tiles from the planner (term 1: Ma = n, R = d, Nb = n2; term 2: Ma = n2, Nb = n)
                at = atiles.setdefault((n, d, n2), (actx.plan_tile(n, d, n2), actx.plan_tile(n2, d, n)))
                sd = synth.seed_for(block, 50 + h, "x") + 10 * d
                X0, X1 = synth.activations(sd, n, d), synth.activations(sd + 1, n, d)
                Y0, Y1 = synth.activations(sd + 2, d, n2), synth.activations(sd + 3, d, n2)
                sk1, sk2 = actx.keygen(sd + 4), actx.keygen(sd + 5)
                heads.append(dict(X1=hl.to_device(X1, dev), Y1=hl.to_device(Y1, dev), tiles=at,
                                  ct1=hl.to_device(actx.encrypt(sk1, at[0], np.ascontiguousarray(Y0.T), sd + 6), dev),
                                  ct2=hl.to_device(actx.encrypt(sk2, at[1], X0, sd + 7), dev), seeds=(sd + 8, sd + 9)))

        items = [dict(tile=hd_["tiles"], X1=hd_["X1"], Y1=hd_["Y1"], ct_Y0T=hd_["ct1"], ct_X0=hd_["ct2"],
                      seeds=hd_["seeds"]) for hd_ in heads]

        def att_step():      # the block's 48 Pi_MatMul products as one pipelined batch
            attention.server_cross_products(actx, items, stream=stream)
        for _ in range(2):   # warm-up: the first calls pay module loading and allocator growth
            att_step()
        torch.cuda.synchronize()
        nrep = max(2, min(args.steps, 5))
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(nrep):
            att_step()
        a1.record(stream)
        torch.cuda.synchronize()
        att_info = {"what": "server side of the attention cross terms of one BERT-base block (row f2, "
                            "PAPER.md:113-118): 12 heads x (QK^T, AV), 2 Pi_MatMul + local product each (the 48 "
                            "products as one hl_he_linear_batch), online "
                            "pi_A encoding of the server's shares (two-pass, no sync), N=8192 L=3, per-term "
                            "tiles from hl_plan_tile: " + "; ".join(f"{k}: {v}" for k, v in atiles.items()),
                    "ms_per_block": round(a0.elapsed_time(a1) / nrep, 3), "cross_products": len(heads)}
        del actx

    # ---------------- end to end through the public API on pinned host buffers
    # weak mode: the 50-bit wire format (hl_pack50) both ways -- the client packs its c0 halves
    # (untimed, like its encryption) and unpacks the responses when it decrypts
    packed = not shard and not os.environ.get("BENCH_E2E_UNPACKED")
    mwords = [int(hl._lib.hl_packed50_words(m["lay"].ct_masked_words)) if packed else m["lay"].ct_masked_words
              for m in mats]
    host_masked = [torch.empty(w, dtype=torch.int64).pin_memory() for w in mwords]
    host_share = [torch.empty(m["lay"].share_words, dtype=torch.int64).pin_memory() for m in mats]
    dev_ct_in = torch.empty(max(m["lay"].ct_in_words for m in mats), dtype=torch.int64, device=dev)

    # weak mode: the pipelined seeded batch (hl_he_linear_batch_host): c0 halves + public seeds
    # up, c1 regenerated on the device, compressed responses + shares down, overlapped per product
    up_bufs = [torch.empty(m["lay"].ct_in_words, dtype=torch.int64, device=dev) for m in mats]
    c0_up = [torch.from_numpy(hl.Context.pack50(m["c0_host"].numpy().view(np.uint64)).view(np.int64)).pin_memory()
             if packed else m["c0_host"] for m in mats]
    # own device output buffers: the check below compares the e2e results with the device batch's
    host_entries = [dict(e, ct_in=u, c0_host=c0, a_seed=m["a_seed"], masked_host=hm, share_host=hs, packed=packed,
                         ct_masked=torch.empty_like(m["masked"]), share=torch.zeros_like(m["share"]))
                    for e, m, u, c0, hm, hs in zip(entries, mats, up_bufs, c0_up, host_masked, host_share)]

    # shard mode: every rank uploads the c0 halves into its ct_in and regenerates c1 from the public
    # seed (hl_expand_seeded), runs its shards (hl_he_linear_batch), the responses are gathered to
    # rank 0 (P2P) and rank 0 downloads the whole block's responses; every rank downloads the server
    # share of its own columns (the server's output share stays on its rank)
    if shard:
        host_full = [torch.empty(m["nI_full"] * m["lay"].nK * m["per_ct"], dtype=torch.int64).pin_memory()
                     if rank == 0 else None for m in mats]
        mwords = [m["nI_full"] * m["lay"].nK * m["per_ct"] if rank == 0 else 0 for m in mats]

    def e2e_step():
        if not shard:
            ctx.he_linear_batch_host(tiles[0], [host_entries[i] for i in e2e_order], stream=stream)
            return
        LN = cfg.L * cfg.N
        for i in order:
            m, u = mats[i], up_bufs[i]
            u.view(-1, 2, LN)[:, 0].copy_(m["c0_host"].view(-1, LN), non_blocking=True)
            ctx.expand_seeded(m["tile"], m["mm"].R, m["mm"].Nb, m["a_seed"], u, stream=stream)
        ents = [dict(entries[i], ct_in=up_bufs[i], ct_masked=mats[i]["sets"][0][0], share=mats[i]["sets"][0][1])
                for i in order]
        ctx.he_linear_batch(tiles[0], ents, stream=stream)
        works = [w for i in order for w in gathers[i].post(mats[i]["sets"][0][0], full[0][i])] if world > 1 else []
        for w in works:
            w.wait()
        for i in order:
            if rank == 0:
                host_full[i].copy_(full[0][i] if world > 1 else mats[i]["sets"][0][0], non_blocking=True)
            host_share[i].copy_(mats[i]["sets"][0][1], non_blocking=True)

    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e2e_checked = False
    if not shard:       # the host results are the device path's, bit for bit (the e2e leg does the real work)
        for m, hm, hs, (dm, ds) in zip(mats, host_masked, host_share, dev_results):
            got = hm.numpy().view(np.uint64)
            if packed:
                got = hl.Context.unpack50(got, m["lay"].ct_masked_words)
            assert np.array_equal(got, dm.cpu().numpy().view(np.uint64)) and torch.equal(hs, ds.cpu()), \
                "e2e results differ"
        e2e_checked = True
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / e2e_steps
    h2d = sum(c0.numel() * 8 for c0 in c0_up) if not shard else sum(m["c0_host"].numel() * 8 for m in mats)
    d2h = sum((w + m["lay"].share_words) * 8 for w, m in zip(mwords, mats))

    if rank != 0:
        return None

    # ---------------- numbers
    ms_step = elapsed / args.steps
    value = ms_step if shard else elapsed / (args.steps * world)   # ms per block (all ranks' blocks)
    cnt = counts(cfg, [m["lay"] for m in mats], tiles)
    products = sum(c["products"] for c in cnt)
    peaks = _peaks()
    hbm = (peaks.get("hbm_gbs") or 6650.0)
    roof = mac_roofline(cnt, ktimes, peaks)
    try:   # per-launch DRAM bytes of the same kernel from the committed ncu --set full capture
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        if tr.get("kernel") == "k_mac_tc" and tr.get("config", "c2") == cfg.name:
            roof["traffic"] = tr["per_launch_bytes"]
            roof["traffic_source"] = tr["source"]
    except Exception:
        pass
    total_k = sum(v[0] for v in ktimes.values())
    kernel_share = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps,
                        "share": v[0] / total_k if total_k else None} for k, v in ktimes.items() if v[1]}
    launches = kernels_launched          # our kernels inside the timed region (hl_timing_kernels)
    path_bytes = sum(c["path_bytes"] for c in cnt)

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": False,
        "scaling": "strong" if shard else "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.note}", "N": cfg.N, "L": cfg.L, "t_bits": synth.T_BITS,
                   "tile": [list(t) for t in tiles],
                   "tile_choice": ("--tile/--tiles override" if (args.tile or args.tiles) else "per product, hl_plan_tile (DESIGN.md §5)"
                                   if args.plan or cfg.tiles else "config default tile"),
                   "batch_order": [cfg.matmuls[i].name for i in order],
                   "matmuls": [[mm.Nb, mm.R, mm.Ma] for mm in cfg.matmuls],
                   "blocks_per_step_per_rank": 1, "compress": True,
                   "l2": (f"inputs larger than L2: {sum(m['lay'].wcache_bytes for m in mats) / 1e9:.2f} GB NTT-domain "
                          f"weight cache + {sum(m['ct'].numel() for m in mats) * 8 / 1e6:.0f} MB ct_in per block"),
                   "parallelism": (f"shard x{world} (I tiles of one block per rank, responses gathered to rank 0)"
                                   if shard else f"weak x{world} (one block per rank)")},
        "poly_products_per_s": (sum(m["nI_full"] * m["lay"].nJ * m["lay"].nK for m in mats) if shard
                                else products * world) * args.steps / (elapsed * 1e-3),
        "path_bytes_per_block": path_bytes,
        "path_hbm_frac": path_bytes / (value * 1e-3) / (hbm * 1e9),
        "path_roofline": path_roofline(cnt, value, peaks),
        "roofline": roof,
        "kernels": kernel_share,
        "gpu_launches": launches,
        "encode_weights_ms": round(t_enc * 1e3, 3),
        "e2e": {"value": round(e2e_ms, 4), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "call": ("shard mode: c0 halves H2D into every rank's ct_in + hl_expand_seeded (public seed), "
                         "hl_he_linear_batch on the rank's I shards, P2P gather of the responses to rank 0, D2H of "
                         "the whole block's responses on rank 0 and of each rank's share") if shard else
                        "hl_he_linear_batch_host: seeded upload (c0 halves + public seed; c1 = a regenerated on "
                        "the device), upload / compute / download pipelined per product" +
                        (", 50-bit wire format both ways (hl_pack50)" if packed else ""),
                "checked_equal_to_device_path": e2e_checked},
        "clocks": clk,
    }
    if ntt_info:
        line["ntt_microbench"] = ntt_info
    if fc_info:
        line["fc_local_share"] = fc_info
    if att_info:
        line["attention_cross_terms"] = att_info
    if cli_info:
        line["client_gpu"] = cli_info
    if rr_info:
        line["rerandomized"] = rr_info
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = oracle_baseline(cfg, tiles, args.cpu_itiles)
    return line


# ----------------------------------------------------------------------------- the oracle arm
def oracle_baseline(cfg, tiles, itiles: int, ktiles: int = 0):
    """The CPU oracle as it stands (sparse schoolbook he_matmul + mask; OpenMP over output
    ciphertext x component x prime) on a bounded sample: the first `itiles` I tiles and the first
    `ktiles` K tiles (0 = all) of each matmul, all J, extrapolated linearly to the whole block
    (oracle work is exactly linear in the number of output ciphertexts)."""
    from oracle import ref
    P = ref.bfv_params(cfg.N, cfg.L, synth.T_BITS)
    total_s = 0.0
    sampled = total = 0
    for mi, mm in enumerate(cfg.matmuls):
        tile = tiles[mi]
        m, r, n = tile
        nI, nJ, nK = ref.tile_counts(tile, mm.Ma, mm.R, mm.Nb)
        s = min(itiles, nI)
        kk = nK if ktiles <= 0 else min(ktiles, nK)
        Nb = min(mm.Nb, kk * n)
        W = synth.weights(synth.seed_for(0, mi, "w"), mm.R, mm.Ma)[:, : s * m].copy()
        ct_in = synth.uniform_below(synth.seed_for(0, mi, "enc"), (nJ, kk, 2, P.L, P.N), P.primes)
        t0 = time.perf_counter()
        ct_out = ref.he_matmul(P, tile, W, ct_in, Nb)
        ref.mask_and_share(P, tile, ct_out, W.shape[1], Nb, 1, True)
        dt = time.perf_counter() - t0
        total_s += dt * (nI * nK) / (s * kk)
        sampled += s * kk
        total += nI * nK
    cores = len(os.sched_getaffinity(0))
    return {"value": round(total_s * 1e3, 1), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{sampled} of {total} output ciphertexts (first {itiles} I-tile(s) x "
                      f"{'all' if ktiles <= 0 else ktiles} K-tile(s) of each of the 4 matmuls, all J), "
                      f"extrapolated linearly to the block",
            "cpu": _cpu_model()}


def _tiles(cfg, args):
    """Per-product tiles: --tile for all, else the config's (synth: hl_plan_tile's choices for c2)."""
    if getattr(args, "tiles", None):    # experiment: per-product tiles "m,r,n;m,r,n;..."
        return [tuple(int(v) for v in t.split(",")) for t in args.tiles.split(";")]
    return [tuple(args.tile)] * len(cfg.matmuls) if args.tile else [cfg.tile_of(i) for i in range(len(cfg.matmuls))]


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, rank, world):
    if rank != 0:
        return None
    cfg = synth.CONFIGS[args.config]
    tiles = _tiles(cfg, args)
    vals = []
    if cfg.blocks > 1:      # c3 / c4: the stack sampler of our arm's cpu_baseline (bench_stack.py)
        import bench_stack
        import paper_2305_18396_b200 as hl
        hctx = hl.Context(cfg.N, cfg.L, synth.T_BITS, device=-1)
        tiles, _ = bench_stack.choose_tiles(hctx, cfg, cfg.blocks, 178.35 * 2**30, args.tile)   # ours at N = 1
        sample = lambda: bench_stack.stack_oracle_baseline(cfg, tiles, args.cpu_frac)   # noqa: E731
        base = bench_stack.stack_oracle_baseline.__doc__
    else:
        # the same bounded sample as our arm's cpu_baseline (first 2 I tiles x all K tiles of each product:
        # 32 output ciphertexts, enough OpenMP tasks for the host's cores), extrapolated to the block
        sample = lambda: oracle_baseline(cfg, tiles, 2, 0)       # noqa: E731
        base = oracle_baseline.__doc__
    for _ in range(min(args.warmup, 1)):
        sample()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s_ = sample()
        vals.append(s_["value"])
    wall = time.perf_counter() - t0
    v = float(np.mean(vals))
    cores = len(os.sched_getaffinity(0))
    return {"metric": METRIC, "value": round(v, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(v, 1), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "N": cfg.N, "L": cfg.L, "t_bits": synth.T_BITS,
                       "tile": [list(t) for t in tiles], "parallelism": "CPU oracle, OpenMP over output tiles"},
            "cpu_baseline": {"value": round(v, 1), "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": s_["sample"],
                             "cpu": _cpu_model(),
                             "wall_s": round(wall, 2)},
            "e2e": {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0, "note": base.split("\n")[0] if base else ""}


def main():
    # the stacks allocate tens of GB in few large buffers: avoid allocator fragmentation (c4 fills HBM)
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--tile", type=int, nargs=3, default=None)
    ap.add_argument("--tiles", default=None, help='per-product tiles, e.g. "32,8,16;8,8,64;32,8,16;8,16,32"')
    ap.add_argument("--plan", action="store_true", help="every product at hl_plan_tile's tile")
    ap.add_argument("--cpu-itiles", type=int, default=2)
    ap.add_argument("--cpu-frac", type=float, default=None,
                    help="c3/c4: sampled fraction of one block's output ciphertexts for the oracle baseline "
                         "(default c3 1 %%, c4 0.2 %%)")
    ap.add_argument("--e2e-items", type=int, default=1, help="c4: items measured end to end (scaled to the stack)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sequential", action="store_true", help="one he_matmul_share per product (no 2-stream pipeline)")
    ap.add_argument("--no-attention", action="store_true", help="skip the row-f2 attention measurement")
    ap.add_argument("--mode", choices=["auto", "weak", "shard"], default="auto",
                    help="auto: shard for N > 1 (BASELINE config 2: sharded by output columns), the whole block "
                         "at N = 1; weak: one block per rank; shard: one block split by I tiles + gather to rank 0")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    stack = synth.CONFIGS[args.config].blocks > 1
    if args.cpu_frac is None:
        args.cpu_frac = 0.002 if args.config == "c4" else 0.01
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    elif stack:
        import bench_stack
        line = bench_stack.run_stack(args, rank, world, local_rank, sys.modules[__name__])
    else:
        line = run_ours(args, rank, world, local_rank)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
