"""Multi-GPU plumbing of the server path: one process per GPU.

Partition ("larger matrices could be split into smaller blocks"; reading C2):
the output ciphertexts (I, K) of a product are independent given the inputs, so the I tiles
(output-column blocks of X.W) are split into contiguous shards, one per rank.  Each rank encodes
only its shard of the weights (hl_encode_weights with [i_begin, i_end)), receives the whole
ct_in, and produces the compressed responses of its shard plus the server share of its columns.
The mask streams use the GLOBAL tile index I*nK + K, so the shards are bit-identical slices of
the unsharded result.  The one exchange step is gathering the responses to the client-facing
rank (north_star: "NCCL over NVLink only to gather output ciphertexts").

This module is host logic only (shard plan, gather, assembly) on torch.distributed; it works
with the nccl backend on CUDA tensors and with gloo on CPU tensors (tests/test_dist.py).
"""
from __future__ import annotations


def shard_range(nI: int, world: int, rank: int):
    """Contiguous, balanced I-tile shard [i_begin, i_end) of rank `rank` (empty shards only when
    nI < world)."""
    q, r = divmod(nI, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def shard_columns(i_begin: int, i_end: int, m: int, Ma: int):
    """Columns of X.W (rows of W^T) covered by I tiles [i_begin, i_end) of width m."""
    return i_begin * m, min(i_end * m, Ma)


def gather_responses(masked_shard, share_shard, nI: int, nK: int, per_ct: int, tile, Ma: int, Nb: int,
                     dst: int = 0, group=None):
    """Gather every rank's compressed responses and share columns to rank `dst`.

    masked_shard: tensor [nI_s * nK * per_ct] (this rank's I tiles, [I_loc][K][per_ct]);
    share_shard: tensor [Nb * Ma] holding this rank's columns (others arbitrary).
    Returns (masked [nI][nK][per_ct], share [Nb][Ma]) on rank dst, (None, None) elsewhere.
    Shards are zero-padded to the largest one so that a single all_gather moves everything
    (gather is not implemented by every backend); rank dst assembles the rows and columns."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m = tile[0]
    qmax = -(-nI // world)
    dev = masked_shard.device
    i0, i1 = shard_range(nI, world, rank)
    buf = torch.zeros(qmax * nK * per_ct, dtype=masked_shard.dtype, device=dev)
    buf[: (i1 - i0) * nK * per_ct] = masked_shard.reshape(-1)[: (i1 - i0) * nK * per_ct]
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    c0, c1 = shard_columns(i0, i1, m, Ma)
    cols = torch.zeros(Nb * qmax * m, dtype=share_shard.dtype, device=dev)
    cols.view(Nb, qmax * m)[:, : c1 - c0] = share_shard.view(Nb, Ma)[:, c0:c1]
    souts = [torch.empty_like(cols) for _ in range(world)]
    dist.all_gather(souts, cols, group=group)
    if rank != dst:
        return None, None
    masked = torch.empty(nI, nK, per_ct, dtype=masked_shard.dtype, device=dev)
    share = torch.empty(Nb, Ma, dtype=share_shard.dtype, device=dev)
    for r_ in range(world):
        j0, j1 = shard_range(nI, world, r_)
        masked[j0:j1] = outs[r_][: (j1 - j0) * nK * per_ct].view(j1 - j0, nK, per_ct)
        k0, k1 = shard_columns(j0, j1, m, Ma)
        share[:, k0:k1] = souts[r_].view(Nb, qmax * m)[:, : k1 - k0]
    return masked, share
