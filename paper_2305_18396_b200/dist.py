"""Multi-GPU plumbing of the server path: one process per GPU.

Partitions ("larger matrices could be split into smaller blocks"; reading C2):

* c2, one block, column split.  The output ciphertexts (I, K) of a product are independent given
  the inputs, so the I tiles (output-column blocks of X.W) are split into contiguous shards, one
  per rank (`shard_range`).  Each rank encodes only its shard of the weights (hl_encode_weights
  with [i_begin, i_end)), receives the whole ct_in, runs hl_he_linear_batch on its shards of the
  four products and produces their compressed responses plus the server share of its columns.
  The mask streams use the GLOBAL tile index I*nK + K, so the shards are bit-identical slices of
  the unsharded result.  The forward NTT of ct_in is NOT sharded: every rank transforms all of
  ct_in (its MAC needs every J); exchanging NTT-domain ciphertexts instead would move more bytes
  than the transform costs.
* c3 / c4, stacks of blocks x sequences: the blocks*seqs (layer, sequence) items in layer-major
  order, split into contiguous balanced chunks (`stack_plan`), so a rank holds the weight caches of
  few layers; consecutive items of one layer are merged into one product set over their
  concatenated sequences (Nb = 128 * #sequences), keeping the weight reuse of the batched columns.

The one exchange step is moving the responses to the client (north_star: "NCCL over NVLink only to
gather output ciphertexts"; "Server sends [[c]] - s to client"):

* `ResponseGather` (column split): rank r's responses are rows [i0, i1) of the I-major response
  array [nI][nK][per_ct], i.e. ONE contiguous block, sent point-to-point straight into those rows
  of the client-facing rank's buffer (no padding, no all-gather: rank dst ingests (G-1)/G of the
  responses once).  The server share S stays with the rank that owns its columns: it is the
  server's own share of the output (Alg. 1 step 3), not sent to the client.
* `StackRouter` (stacks): every sequence has a client-facing rank (`client_rank`); after each round
  of items the producing ranks send each sequence's responses (its K tiles, packed contiguous) to
  that rank, which receives them into a ring of buffers.

All transfers are asynchronous torch.distributed P2P operations (NCCL on CUDA tensors, gloo on
CPU tensors in tests/test_dist.py); they run on the backend's own stream, so a caller overlaps them
with the next step's compute by alternating two sets of output buffers.
"""
from __future__ import annotations

from dataclasses import dataclass


def shard_range(nI: int, world: int, rank: int):
    """Contiguous, balanced I-tile shard [i_begin, i_end) of rank `rank` (empty shards only when
    nI < world)."""
    q, r = divmod(nI, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def shard_columns(i_begin: int, i_end: int, m: int, Ma: int):
    """Columns of X.W (rows of W^T) covered by I tiles [i_begin, i_end) of width m."""
    return i_begin * m, min(i_end * m, Ma)


def _p2p(ops):
    """Issue a list of P2POp as one batch (NCCL groups them); returns the works."""
    import torch.distributed as dist
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


class ResponseGather:
    """Point-to-point gather of the compressed responses of an I-tile column split to rank `dst`.

    post(masked_shard, full) issues, on every rank, the transfers of one product: rank r != dst
    sends masked_shard ([nI_r * nK * per_ct] words, its rows [i0, i1)); rank dst receives every
    other rank's block into full[i0 * nK * per_ct : i1 * nK * per_ct] and copies its own rows
    (skipped when masked_shard already aliases them).  Returns the works (wait() them, or let the
    backend stream order them before later collectives)."""

    def __init__(self, nI: int, nK: int, per_ct: int, dst: int = 0, group=None):
        import torch.distributed as dist
        self.nI, self.nK, self.per_ct, self.dst, self.group = nI, nK, per_ct, dst, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranges = [shard_range(nI, self.world, r) for r in range(self.world)]

    def words(self, r: int) -> tuple:
        i0, i1 = self.ranges[r]
        row = self.nK * self.per_ct
        return i0 * row, i1 * row

    def post(self, masked_shard, full=None):
        import torch.distributed as dist
        ops = []
        w0, w1 = self.words(self.rank)
        if self.rank == self.dst:
            assert full is not None and full.numel() >= self.nI * self.nK * self.per_ct
            if w1 > w0 and masked_shard.data_ptr() != full[w0:w1].data_ptr():
                full[w0:w1].copy_(masked_shard.reshape(-1)[: w1 - w0])
            for r in range(self.world):
                a, b = self.words(r)
                if r != self.dst and b > a:
                    ops.append(dist.P2POp(dist.irecv, full[a:b], dist.get_global_rank(self.group, r)
                                          if self.group is not None else r, self.group))
        elif w1 > w0:
            ops.append(dist.P2POp(dist.isend, masked_shard.reshape(-1)[: w1 - w0],
                                  dist.get_global_rank(self.group, self.dst) if self.group is not None else self.dst,
                                  self.group))
        return _p2p(ops)


# ----------------------------------------------------------------------------------------- stacks
@dataclass(frozen=True)
class Item:
    """Sequences [seq0, seq1) of block (layer) `block`: one product set over their concatenated tokens."""
    block: int
    seq0: int
    seq1: int

    @property
    def nseq(self) -> int:
        return self.seq1 - self.seq0


def stack_plan(blocks: int, seqs: int, world: int):
    """Per rank, its items: the blocks*seqs (layer, sequence) items in layer-major order split into
    contiguous balanced chunks, consecutive items of one block merged."""
    plan = []
    for rank in range(world):
        a, b = shard_range(blocks * seqs, world, rank)
        items = []
        for it in range(a, b):
            blk, s = divmod(it, seqs)
            if items and items[-1].block == blk and items[-1].seq1 == s:
                items[-1] = Item(blk, items[-1].seq0, s + 1)
            else:
                items.append(Item(blk, s, s + 1))
        plan.append(items)
    return plan


def client_rank(seq: int, world: int, n_client: int = 0) -> int:
    """The client-facing rank of a sequence: sequences are spread round-robin over the first
    min(world, n_client) ranks (n_client = 0: all ranks)."""
    k = min(world, n_client) if n_client else world
    return seq % k


class StackRouter:
    """Moves every sequence's compressed responses to its client-facing rank, round by round.

    Round k consists of the k-th item of every rank (ranks with fewer items idle).  For an item and
    product with nI output tiles, kps K tiles per sequence and per_ct words per response, the
    producing rank packs sequence s's responses [nI][kps][per_ct] (its K tiles of the item's
    [nI][nK_item][per_ct] array) and sends them to client_rank(s), which receives them into its
    ring: `slots()` buffers of nI*kps*per_ct words per product, two halves used by alternate rounds
    (round k writes half k mod 2 after the transfers of round k-2 into it completed), so round k+1's
    compute and transfers overlap round k's.  route() returns the works and the list of
    (block, seq, product, slot) received."""

    def __init__(self, plan, world: int, rank: int, n_client: int = 0, group=None):
        self.plan, self.world, self.rank, self.n_client, self.group = plan, world, rank, n_client, group
        self.rounds = max(len(p) for p in plan)
        per = [sum(1 for p in plan if k < len(p) for s in range(p[k].seq0, p[k].seq1) if self.dest(s) == rank)
               for k in range(self.rounds)]
        self.per_round = max(per) if per else 0
        self._works = {}           # (half, product) -> works of the round that last wrote that half

    def dest(self, seq: int) -> int:
        return client_rank(seq, self.world, self.n_client)

    def slots(self) -> int:
        return 2 * self.per_round

    def route(self, k: int, product: int, out, nI: int, kps: int, per_ct: int, ring):
        """Round k, product `product`: `out` is this rank's response array of its k-th item
        ([nI][nseq*kps][per_ct] words; ignored when the rank has no k-th item); ring: this rank's
        slots() receive buffers of nI*kps*per_ct words for this product."""
        import torch.distributed as dist
        half = k % 2
        for w in self._works.pop((half, product), []):      # the half's previous transfers are done
            w.wait()
        ops, got, idx = [], [], 0
        mine = self.plan[self.rank][k] if k < len(self.plan[self.rank]) else None
        if mine is not None:
            o = out.reshape(nI, mine.nseq * kps, per_ct)
            for s in range(mine.seq0, mine.seq1):
                part = o[:, (s - mine.seq0) * kps:(s - mine.seq0 + 1) * kps]
                d = self.dest(s)
                if d == self.rank:
                    slot = half * self.per_round + idx
                    idx += 1
                    ring[slot].view(nI, kps, per_ct).copy_(part)
                    got.append((mine.block, s, product, slot))
                else:
                    ops.append(dist.P2POp(dist.isend, part.contiguous().view(-1), d, self.group))
        for r in range(self.world):
            if r == self.rank or k >= len(self.plan[r]):
                continue
            it = self.plan[r][k]
            for s in range(it.seq0, it.seq1):
                if self.dest(s) == self.rank:
                    slot = half * self.per_round + idx
                    idx += 1
                    ops.append(dist.P2POp(dist.irecv, ring[slot].view(-1), r, self.group))
                    got.append((it.block, s, product, slot))
        works = _p2p(ops)
        self._works[(half, product)] = works
        return works, got
