"""Multi-process (gloo, CPU, world_size 2-4) tests of the multi-GPU server path's host logic
(SURVEY.md §8(e)): the I-tile shard plan and the point-to-point gather of compressed responses to
the client-facing rank (c2's column split), the layer-major (layer, sequence) item plan of the
stacks (c3, c4) and the routing of every sequence's responses to its client-facing rank.

Column split: each rank produces its shard's responses with the oracle (tests may use oracle/),
using the GLOBAL tile index for the mask streams, exactly as hl_he_matmul_share /
hl_he_linear_batch do with [i_begin, i_end); rank 0 checks that the gathered responses are the
unsharded oracle result bit for bit and that the client's decrypted share plus the server shares
(which stay on their ranks; collected here for the check only) reconstruct X.W.
"""
import os
import socket

import numpy as np
import pytest

from paper_2305_18396_b200 import dist as hd


def test_shard_range_partition():
    for nI in (1, 2, 5, 48, 144, 191):
        for world in (1, 2, 3, 4, 8):
            spans = [hd.shard_range(nI, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nI
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    from oracle import ref
    import synth
    try:
        _init(rank, world, port)
        (Nb, R, Ma), tile, seed = case
        m, r, n = tile
        P = ref.bfv_params(4096, 2, 37)
        X = synth.activations(seed, Nb, R)
        W = synth.weights(seed + 1, R, Ma)
        sk = ref.keygen(P, seed + 2)
        ct_in = ref.encrypt(P, tile, sk, X, seed + 3)
        nI, nJ, nK = ref.tile_counts(tile, Ma, R, Nb)
        i0, i1 = hd.shard_range(nI, world, rank)
        c0, c1 = hd.shard_columns(i0, i1, m, Ma)
        per = P.L * (m * n + P.N)
        masked_s = np.zeros((max(i1 - i0, 0), nK, per), np.uint64)
        share_s = np.zeros((Nb, Ma), np.uint64)
        if i1 > i0:
            ct = ref.he_matmul(P, tile, W[:, c0:c1].copy(), ct_in, Nb)          # local I tiles
            tiles = [(I, K) for I in range(i0, i1) for K in range(nK)]          # global indices
            mk, kept = ref.mask_tiles(P, tile, ct.reshape(-1, 2, P.L, P.N), nK, tiles, seed + 4, True)
            masked_s[:] = mk.reshape(i1 - i0, nK, per)
            for o, (I, K) in enumerate(tiles):                                   # S[Kn+k][Im+i]
                for k in range(n):
                    for i in range(m):
                        row, col = K * n + k, I * m + i
                        if row < Nb and col < Ma:
                            share_s[row, col] = kept[o, k * m + i]
        t = lambda a: torch.from_numpy(a.view(np.int64).reshape(-1).copy())
        g = hd.ResponseGather(nI, nK, per, dst=0)
        full = torch.full((nI * nK * per,), -1, dtype=torch.int64) if rank == 0 else None
        for w in g.post(t(masked_s), full):
            w.wait()
        shares = [None] * world                      # the check only: the server shares stay put
        dist.all_gather_object(shares, (c0, c1, share_s[:, c0:c1]))
        if rank == 0:
            em, es = ref.mask_and_share(P, tile, ref.he_matmul(P, tile, W, ct_in, Nb), Ma, Nb, seed + 4, True)
            gm = full.numpy().view(np.uint64).reshape(em.shape)
            assert np.array_equal(gm, em), "gathered responses differ from the unsharded oracle"
            gs = np.zeros_like(es)
            for a, b, cols in shares:
                gs[:, a:b] = cols
            assert np.array_equal(gs, es), "server shares differ from the unsharded oracle"
            share_c = ref.decrypt_share(P, tile, sk, gm, Ma, Nb, True)
            assert np.array_equal((share_c + gs) & np.uint64((1 << 37) - 1), ref.matmul_mod_t(X, W))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()[-800:]))


def _spawn(target, world, *args):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("world,case", [
    (2, ((16, 32, 80), (16, 8, 32), 11)),      # nI = 5 over 2 ranks: ragged shards 3 + 2
    (2, ((8, 64, 64), (16, 32, 8), 12)),       # config c0 shape, nI = 4
    (3, ((40, 24, 112), (16, 8, 32), 13)),     # nI = 7 over 3 ranks: 3 + 2 + 2, nK = 2
    (4, ((8, 64, 48), (16, 32, 8), 14)),       # nI = 3 over 4 ranks: rank 3's shard is empty
])
def test_sharded_gather(world, case):
    res = _spawn(_worker, world, case)
    assert res == {r: "ok" for r in range(world)}, res


# ---------------------------------------------------------------------------------------- stacks
@pytest.mark.parametrize("blocks,seqs,world", [(12, 8, 1), (12, 8, 2), (12, 8, 8), (24, 4, 8), (24, 4, 3), (2, 3, 4)])
def test_stack_plan_partition(blocks, seqs, world):
    """Every (layer, sequence) item exactly once, layer-major contiguous chunks of balanced size,
    merged per layer; at 8 GPUs c3 gives every rank <= 2 layers and c4 3 layers."""
    plan = hd.stack_plan(blocks, seqs, world)
    flat = [(it.block, s) for p in plan for it in p for s in range(it.seq0, it.seq1)]
    assert flat == [(b, s) for b in range(blocks) for s in range(seqs)]
    sizes = [sum(it.nseq for it in p) for p in plan]
    assert max(sizes) - min(sizes) <= 1
    for p in plan:
        assert all(a.block != b.block for a, b in zip(p, p[1:]))       # merged per layer
    if world == 8 and (blocks, seqs) == (12, 8):
        assert max(len(p) for p in plan) <= 2
    if world == 8 and (blocks, seqs) == (24, 4):
        assert all(len(p) == 3 for p in plan)


def _router_worker(rank, world, port, blocks, seqs, n_client, q):
    """Synthetic responses: value = block * 1e6 + seq * 1e3 + product * 100 + position % 97 -- every
    client-facing rank must receive exactly its sequences' responses, in its ring slots."""
    import torch
    import torch.distributed as dist
    try:
        _init(rank, world, port)
        plan = hd.stack_plan(blocks, seqs, world)
        router = hd.StackRouter(plan, world, rank, n_client)
        nI, kps, per = 3, 2, 5
        rings = [torch.full((max(router.slots(), 1), nI * kps * per), -1, dtype=torch.int64) for _ in range(2)]
        pat = torch.arange(nI * kps * per, dtype=torch.int64).view(nI, kps, per) % 97
        seen = []
        for k in range(router.rounds):
            mine = plan[rank][k] if k < len(plan[rank]) else None
            for prod in range(2):
                out = None
                if mine is not None:
                    out = torch.empty(nI, mine.nseq * kps, per, dtype=torch.int64)
                    for s in range(mine.seq0, mine.seq1):
                        out[:, (s - mine.seq0) * kps:(s - mine.seq0 + 1) * kps] = \
                            pat + mine.block * 1_000_000 + s * 1000 + prod * 100
                works, got = router.route(k, prod, out, nI, kps, per, rings[prod])
                for w in works:
                    w.wait()
                for blk, s, p_, slot in got:
                    want = pat + blk * 1_000_000 + s * 1000 + p_ * 100
                    assert torch.equal(rings[p_][slot].view(nI, kps, per), want), (rank, k, blk, s, p_)
                    assert hd.client_rank(s, world, n_client) == rank
                    seen.append((blk, s, p_))
        allseen = [None] * world
        dist.all_gather_object(allseen, seen)
        if rank == 0:
            flat = sorted(x for v in allseen for x in v)
            assert flat == sorted((b, s, p) for b in range(blocks) for s in range(seqs) for p in range(2))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()[-800:]))


@pytest.mark.parametrize("world,blocks,seqs,n_client", [(3, 4, 8, 0), (4, 6, 4, 4), (2, 3, 5, 1)])
def test_stack_router_delivers_every_sequence(world, blocks, seqs, n_client):
    res = _spawn(_router_worker, world, blocks, seqs, n_client)
    assert res == {r: "ok" for r in range(world)}, res
