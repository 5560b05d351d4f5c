"""Sequence-sharded decode attention across GPUs (one process per GPU).

The compressed cache of a long context is partitioned by contiguous token
range: rank r owns tokens [r*ceil(T/P), min(T, (r+1)*ceil(T/P))) of every
(batch, kv head) stream — exactly the chunking of the reference's
attention_decode(..., n_splits = P) (attention.hpp:60-69), whose result is
independent of the split count.  Each rank runs the fused attention kernel on
its slice and produces one SoftmaxState (m, l, acc) per (batch, query head);
ONE all-gather (NCCL over NVLink) moves those partials, and every rank merges
them in rank order (SoftmaxState::merge, attention.hpp:36-44) with the
combine kernel, so all ranks hold bit-identical outputs.  Compress and decode
need no collective (independent per token).

The orchestration is written against plain callables so the same code runs
with the GPU kernels (production) and with CPU stand-ins (gloo tests).
"""
from __future__ import annotations

import math


def shard_bounds(T: int, world: int, rank: int):
    """Token range [t0, t1) owned by `rank` (ceil chunking, attention.hpp:61)."""
    if T < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad sharding arguments")
    chunk = math.ceil(T / world) if T else 0
    t0 = min(T, rank * chunk)
    return t0, min(T, t0 + chunk)


def gather_partials(partial, group=None):
    """All-gather one [rows, W] partial per rank -> [world, rows, W] in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rows = partial.shape[0]
    out = torch.empty((world * rows,) + tuple(partial.shape[1:]), dtype=partial.dtype,
                      device=partial.device)
    dist.all_gather_into_tensor(out, partial.contiguous(), group=group)
    return out.view((world,) + tuple(partial.shape))


def sharded_decode(local_partial, combine, group=None):
    """local_partial: [rows, W] SoftmaxState of this rank's token range.
    combine(gathered [world, rows, W]) merges in token order and finalizes."""
    return combine(gather_partials(local_partial, group))


class ShardedAttention:
    """GPU production path: partials (K5+K3) -> NCCL all-gather -> combine (K4)."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, q, cache, n_splits=None, out=None):
        import paper_2605_21226_b200 as oq
        B, Hq, D = q.shape
        rows = B * Hq
        part = oq.attention_partials(q, cache, 0, cache.tokens, n_splits=n_splits)

        def combine(g):
            world = g.shape[0]
            return oq.attention_combine(cache.enc_v, g, rows, world, g.shape[2],
                                        rows * g.shape[2],
                                        out=None if out is None else out.view(rows, D))

        return sharded_decode(part, combine, self.group).view(B, Hq, D)
