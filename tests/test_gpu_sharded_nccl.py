"""GPU: the native sequence-sharded entry point (oq_attention_decode_sharded).

One process per GPU; this rank's partials -> ONE ncclAllGather through the
library's own NCCL loader -> rank-ordered merge.  The GPU pool gives one GPU
per call, so the collective is exercised with a 1-rank communicator (the
all-gather is then an in-place no-op, every other step is the multi-rank
code path); the rank-ordered merge over several ranks is checked by
emulating the ranks' token ranges on this GPU and merging them with the same
combine kernel, against the reference's attention_decode(..., n_splits = P)
(attention.hpp:60-69).  The torch.distributed variant is covered by
tests/test_dist.py (gloo, world size 2).
"""
import numpy as np
import pytest

import paper_2605_21226_b200 as oq

pytestmark = pytest.mark.gpu


def _cache(cuda, B, Hkv, T, bits=3):
    import torch
    bd, bn = oq.default_bit_split(bits)
    ek = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=31))
    ev = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=32))
    g = torch.Generator(device=cuda).manual_seed(3)
    k = torch.randn((B * Hkv * T, 128), device=cuda, generator=g)
    v = torch.randn((B * Hkv * T, 128), device=cuda, generator=g)
    cache = oq.KVCache(ek, ev, B, Hkv, T)
    cache.pack(ek.compress(k), ev.compress(v), T)
    q = torch.randn((B, 7 * Hkv, 128), device=cuda, generator=g)
    return cache, q


@pytest.mark.parametrize("bits", [3, 2])
def test_single_rank_nccl_equals_decode(cuda, bits):
    B, Hkv, T = 2, 2, 3000
    cache, q = _cache(cuda, B, Hkv, T, bits)
    comm = oq.NcclComm(1, oq.NcclComm.unique_id(), 0)
    try:
        got = oq.attention_decode_sharded(q, cache, 0, T, comm)
    finally:
        comm.close()
    want = oq.attention_decode(q, cache)
    err = ((got - want).norm(dim=-1) / want.norm(dim=-1)).max().item()
    assert err < 1e-5, err


@pytest.mark.parametrize("bits", [3, 2])
@pytest.mark.parametrize("P", [2, 3, 8])
def test_rank_ordered_merge_matches_n_splits(cuda, P, bits):
    import torch
    B, Hkv, T = 1, 2, 2500
    cache, q = _cache(cuda, B, Hkv, T, bits)
    rows = B * 7 * Hkv
    chunk = -(-T // P)
    parts = []
    for r in range(P):  # what rank r computes on its own GPU
        t0, t1 = min(T, r * chunk), min(T, (r + 1) * chunk)
        parts.append(oq.attention_partials(q, cache, t0, t1))
    gathered = torch.stack(parts)  # the all-gather's [rank][rows][4 + dim] layout
    merged = oq.attention_combine(cache.enc_v, gathered, rows, P, gathered.shape[2],
                                  rows * gathered.shape[2])
    want = oq.attention_decode(q, cache, n_splits=P).reshape(rows, 128)
    err = ((merged - want).norm(dim=-1) / want.norm(dim=-1)).max().item()
    # both are within 1e-3 of the fp64 reference (test_gpu_attention.py); the
    # P fragments are rounded to fp16 against different running maxima when
    # the split points differ, hence the same 1e-3 bound between them
    assert err < 1e-3, err


def test_empty_rank_range_is_an_empty_partial(cuda):
    """A rank whose token range is empty contributes an empty (l = 0) partial
    (attention.hpp:40-41 skips it in the merge)."""
    import torch
    B, Hkv, T = 1, 2, 65
    cache, q = _cache(cuda, B, Hkv, T)
    rows = B * 7 * Hkv
    ranges = [(0, 40), (40, 65), (65, 65)]
    parts = [oq.attention_partials(q, cache, t0, t1) for t0, t1 in ranges]
    assert float(parts[2][:, 1].abs().max()) == 0.0  # l = 0 on every row
    gathered = torch.stack(parts)
    merged = oq.attention_combine(cache.enc_v, gathered, rows, len(ranges), gathered.shape[2],
                                  rows * gathered.shape[2])
    want = oq.attention_decode(q, cache).reshape(rows, 128)
    err = ((merged - want).norm(dim=-1) / want.norm(dim=-1)).max().item()
    assert err < 1e-3, err
