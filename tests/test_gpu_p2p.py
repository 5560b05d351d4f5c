"""Fused P2P sequence sharding (oq_attention_decode_p2p) — the exchange
protocol exercised on ONE GPU.

Each "rank" is a concurrent launch on its own stream with its own token slice
of the context in its own cache, its own workspace and its own exchange
buffer; the buffers are ordinary device allocations here (across GPUs they
are CUDA-IPC mappings of the peers' buffers, P2PExchange).  Every launch gets
a share of the SMs (max_ctas) so all of them are resident at once, as the
ranks' kernels are on their own GPUs.  Checked: every rank's output equals the
single-GPU attention_decode over the whole context (the chunk merge of
attention_decode(..., n_splits = nranks), attention.hpp:60-69, so within the
fp16 tolerance of the kernels, 1e-3), all ranks' outputs are bit-identical,
and consecutive calls (epochs; the two halves of the exchange buffer) keep
working with fresh queries.  The kernel traps instead of hanging if a rank
never arrives (20 s); this file runs the protocol only with all ranks present.
"""
import pytest

import paper_2605_21226_b200 as oq

pytestmark = pytest.mark.gpu


def _ranks_setup(cuda, bits, B, Hkv, T, P, qjl=False):
    import torch
    bd, bn = oq.default_bit_split(bits)
    ek = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=51, qjl=qjl, qjl_seed=53))
    ev = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=52))
    g = torch.Generator(device=cuda).manual_seed(7)
    k = torch.randn((B * Hkv, T, 128), device=cuda, generator=g)
    v = torch.randn((B * Hkv, T, 128), device=cuda, generator=g)
    kr = ek.compress(k.reshape(-1, 128)).reshape(B * Hkv, T, -1)
    vr = ev.compress(v.reshape(-1, 128)).reshape(B * Hkv, T, -1)
    full = oq.KVCache(ek, ev, B, Hkv, T)
    full.pack(kr, vr, T)
    per = T // P
    caches = []
    for r in range(P):
        c = oq.KVCache(ek, ev, B, Hkv, per)
        c.pack(kr[:, r * per:(r + 1) * per].contiguous(), vr[:, r * per:(r + 1) * per].contiguous(),
               per)
        caches.append(c)
    return full, caches, per


@pytest.mark.parametrize("bits,P,qjl", [(3, 2, False), (2, 3, False), (3, 4, False), (2, 2, True),
                                        (3, 3, True)])
def test_p2p_exchange_emulated_ranks(cuda, bits, P, qjl):
    import torch
    B, Hq, Hkv, T = 2, 14, 2, 6144
    full, caches, per = _ranks_setup(cuda, bits, B, Hkv, T, P, qjl)
    sms = torch.cuda.get_device_properties(cuda).multi_processor_count
    nbytes = oq.p2p_exchange_bytes(caches[0], Hq, P)
    xbufs = [torch.zeros(nbytes, dtype=torch.uint8, device=cuda) for _ in range(P)]
    streams = [torch.cuda.Stream(device=cuda) for _ in range(P)]
    g = torch.Generator(device=cuda).manual_seed(11)
    for epoch in (1, 2, 3):  # both halves of the exchange buffers, twice
        q = torch.randn((B, Hq, 128), device=cuda, generator=g)
        torch.cuda.synchronize()
        outs = []
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                outs.append(oq.attention_decode_p2p(q, caches[r], 0, per, r, P, xbufs, epoch,
                                                    max_ctas=sms // P, stream=streams[r]))
        torch.cuda.synchronize()
        want = oq.attention_decode(q, full)
        err = ((outs[0] - want).norm(dim=-1) / want.norm(dim=-1)).max().item()
        assert err <= 1e-3, (epoch, err)
        for o in outs[1:]:
            assert torch.equal(o, outs[0])


def test_p2p_single_rank_is_attention_decode(cuda):
    import torch
    B, Hq, Hkv, T = 1, 7, 1, 3000
    full, caches, per = _ranks_setup(cuda, 3, B, Hkv, T, 1)
    xb = torch.zeros(oq.p2p_exchange_bytes(caches[0], Hq, 1), dtype=torch.uint8, device=cuda)
    q = torch.randn((B, Hq, 128), device=cuda)
    got = oq.attention_decode_p2p(q, caches[0], 0, per, 0, 1, [xb], 1)
    want = oq.attention_decode(q, full)
    assert ((got - want).norm(dim=-1) / want.norm(dim=-1)).max().item() <= 1e-5


def test_p2p_rejects_bad_arguments(cuda):
    import torch
    B, Hq, Hkv, T = 1, 7, 1, 64
    full, caches, per = _ranks_setup(cuda, 3, B, Hkv, T, 1)
    xb = torch.zeros(oq.p2p_exchange_bytes(caches[0], Hq, 1), dtype=torch.uint8, device=cuda)
    q = torch.randn((B, Hq, 128), device=cuda)
    with pytest.raises(ValueError):  # epoch 0: the flags' initial value
        oq.attention_decode_p2p(q, caches[0], 0, per, 0, 1, [xb], 0)
    with pytest.raises(ValueError):  # rank out of range
        oq.attention_decode_p2p(q, caches[0], 0, per, 1, 1, [xb], 1)
