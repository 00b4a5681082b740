"""Multi-process (world_size 2, gloo, CPU) tests of the sharded server path's host logic
(SURVEY.md §8(e)): the I-tile shard plan, and the gather of compressed responses + share
columns to the client-facing rank.  Each rank produces its shard's responses with the oracle
(tests may use oracle/), using the GLOBAL tile index for the mask streams, exactly as
hl_he_matmul_share does with [i_begin, i_end); rank 0 checks that the gathered result is the
unsharded oracle result bit for bit, and that the client's decrypted share reconstructs X.W.
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


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    from oracle import ref
    import synth
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
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
        masked, share = hd.gather_responses(t(masked_s), t(share_s), nI, nK, per, tile, Ma, Nb, dst=0)
        if rank == 0:
            em, es = ref.mask_and_share(P, tile, ref.he_matmul(P, tile, W, ct_in, Nb), Ma, Nb, seed + 4, True)
            gm = masked.numpy().view(np.uint64).reshape(em.shape)
            gs = share.numpy().view(np.uint64).reshape(es.shape)
            assert np.array_equal(gm, em), "gathered responses differ from the unsharded oracle"
            assert np.array_equal(gs, es), "gathered share differs from the unsharded oracle"
            share_c = ref.decrypt_share(P, tile, sk, gm, Ma, Nb, True)
            assert np.array_equal((share_c + gs) & np.uint64((1 << 37) - 1), ref.matmul_mod_t(X, W))
        else:
            assert masked is None and share is None
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("case", [
    ((16, 32, 80), (16, 8, 32), 11),      # nI = 5 over 2 ranks: ragged shards 3 + 2
    ((8, 64, 64), (16, 32, 8), 12),       # config c0 shape, nI = 4
])
def test_sharded_gather_world2(case):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
