"""GPU parity of the fused decode-attention path (K5 qprep + K3 + K4).

Oracle: attention_decode(enc_k, q, keys, Matrix{enc_v.decode(values)},
n_splits) in fp64 (attention.hpp:50-73), one call per (batch, q head) with q
head h reading kv head h // (Hq / Hkv).  Tolerance (north_star): relative
L2 error ||out - ref|| / ||ref|| <= 1e-3 per (b, head) — the kernel feeds
fp16 operands to the tensor cores with fp32 accumulation.
"""
import numpy as np
import pytest

import paper_2605_21226_b200 as oq

pytestmark = pytest.mark.gpu
TOL = 1e-3


def build(orc, cuda, B, Hq, Hkv, T, b=3, qjl=False, seed=0, cap=None):
    import torch
    bd, bn = oq.default_bit_split(b)
    ck = oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=11, qjl=qjl, qjl_seed=12)
    cv = oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=13)
    ek, ev = oq.Encoder(ck), oq.Encoder(cv)
    root = orc.L.orc_stream_child(1234, seed)
    k = orc.gaussian_f32(orc.L.orc_stream_child(root, 0), B * Hkv * T * 128).reshape(-1, 128)
    v = orc.gaussian_f32(orc.L.orc_stream_child(root, 1), B * Hkv * T * 128).reshape(-1, 128)
    q = orc.gaussian_f32(orc.L.orc_stream_child(root, 2), B * Hq * 128).reshape(B, Hq, 128)
    kr = ek.compress(torch.from_numpy(k).to(cuda))
    vr = ev.compress(torch.from_numpy(v).to(cuda))
    cache = oq.KVCache(ek, ev, B, Hkv, cap or T)
    cache.pack(kr, vr, T)
    ok = orc.encoder(rotation_seed=11, b_dir=bd, b_nrm=bn, qjl=qjl, qjl_seed=12)
    ov = orc.encoder(rotation_seed=13, b_dir=bd, b_nrm=bn)
    krn, vrn = kr.cpu().numpy(), vr.cpu().numpy()
    assert np.array_equal(krn, ok.encode_f32(k)), "K codes not bit-exact"
    return dict(cache=cache, q=q, krec=krn.reshape(B, Hkv, T, -1),
                vdec=ov.decode(vrn).reshape(B, Hkv, T, 128), ok=ok)


def oracle_out(d, B, Hq, Hkv, lens=None, n_splits=1):
    G = Hq // Hkv
    out = np.zeros((B, Hq, 128))
    for b in range(B):
        L = d["krec"].shape[2] if lens is None else lens[b]
        for h in range(Hq):
            if L == 0:
                continue
            kv = h // G
            out[b, h] = d["ok"].attention(d["q"][b, h].astype(np.float64),
                                          d["krec"][b, kv, :L], d["vdec"][b, kv, :L], n_splits)
    return out


def rel_err(got, ref):
    num = np.linalg.norm(got - ref, axis=-1)
    den = np.linalg.norm(ref, axis=-1)
    return num / np.maximum(den, 1e-30)


@pytest.mark.parametrize("b,qjl", [(3, False), (2, False), (2, True), (3, True), (4, False),
                                   (4, True)])
def test_attention_matches_oracle(orc, cuda, b, qjl):
    import torch
    B, Hq, Hkv, T = 2, 14, 2, 700
    d = build(orc, cuda, B, Hq, Hkv, T, b=b, qjl=qjl)
    got = oq.attention_decode(torch.from_numpy(d["q"]).to(cuda), d["cache"]).cpu().numpy()
    ref = oracle_out(d, B, Hq, Hkv)
    e = rel_err(got, ref)
    assert e.max() <= TOL, (e.max(), e.mean())


@pytest.mark.parametrize("b", [3, 2])
@pytest.mark.parametrize("G", [1, 7, 8, 16])
def test_gqa_group_sizes(orc, cuda, G, b):
    import torch
    B, Hkv, T = 1, 2, 257
    Hq = G * Hkv
    d = build(orc, cuda, B, Hq, Hkv, T, b=b, seed=G)
    got = oq.attention_decode(torch.from_numpy(d["q"]).to(cuda), d["cache"]).cpu().numpy()
    assert rel_err(got, oracle_out(d, B, Hq, Hkv)).max() <= TOL


@pytest.mark.parametrize("b,qjl", [(3, False), (2, False), (2, True)])
def test_split_count_does_not_change_output(orc, cuda, b, qjl):
    # codec_test.cpp:301-319 at the batched level
    import torch
    B, Hq, Hkv, T = 2, 7, 1, 1000
    d = build(orc, cuda, B, Hq, Hkv, T, b=b, qjl=qjl, seed=5)
    q = torch.from_numpy(d["q"]).to(cuda)
    outs = [oq.attention_decode(q, d["cache"], n_splits=s).cpu().numpy() for s in (1, 3, 8, 32)]
    # Different split counts change the running max each fp16 P operand is
    # scaled by, so results agree to fp16 rounding (~2e-4), not bitwise.
    for o in outs[1:]:
        assert rel_err(o, outs[0]).max() <= TOL
    assert rel_err(outs[0], oracle_out(d, B, Hq, Hkv)).max() <= TOL


@pytest.mark.parametrize("b,qjl", [(3, False), (2, False), (2, True)])
def test_single_key_returns_its_value_row(orc, cuda, b, qjl):
    # codec_test.cpp:338-351: softmax over one key is exactly that value row
    import torch
    d = build(orc, cuda, 1, 7, 1, 1, b=b, qjl=qjl, seed=6)
    got = oq.attention_decode(torch.from_numpy(d["q"]).to(cuda), d["cache"]).cpu().numpy()
    for h in range(7):
        assert rel_err(got[0, h], d["vdec"][0, 0, 0]) <= 1e-3


@pytest.mark.parametrize("b,qjl", [(3, False), (2, False), (2, True), (4, True)])
def test_ragged_lengths(orc, cuda, b, qjl):
    import torch
    B, Hq, Hkv, T = 3, 14, 2, 333
    d = build(orc, cuda, B, Hq, Hkv, T, b=b, qjl=qjl, seed=7)
    lens = [333, 31, 0]
    sl = torch.tensor(lens, dtype=torch.int32, device=cuda)
    got = oq.attention_decode(torch.from_numpy(d["q"]).to(cuda), d["cache"],
                              seq_lens=sl).cpu().numpy()
    ref = oracle_out(d, B, Hq, Hkv, lens=lens)
    assert rel_err(got[:2], ref[:2]).max() <= TOL
    assert np.all(got[2] == 0.0)


@pytest.mark.parametrize("b,qjl", [(3, False), (2, False), (2, True)])
def test_sharded_partials_merge_like_n_splits(orc, cuda, b, qjl):
    """Sequence sharding: per-range partials merged in order == one pass.

    This is the single-GPU image of the multi-GPU mode (each range is what
    one rank owns; the merge is what every rank runs after the all-gather).
    """
    import torch
    B, Hq, Hkv, T = 2, 14, 2, 1000
    d = build(orc, cuda, B, Hq, Hkv, T, b=b, qjl=qjl, seed=8)
    q = torch.from_numpy(d["q"]).to(cuda)
    P = 4
    chunk = -(-T // P)
    parts = [oq.attention_partials(q, d["cache"], r * chunk, min(T, (r + 1) * chunk))
             for r in range(P)]
    gathered = torch.stack(parts)  # [P, rows, 132] == all_gather layout
    rows = B * Hq
    out = oq.attention_combine(d["cache"].enc_v, gathered, rows, P, 132, rows * 132)
    got = out.reshape(B, Hq, 128).cpu().numpy()
    full = oq.attention_decode(q, d["cache"]).cpu().numpy()
    assert rel_err(got, full).max() <= TOL  # fp16 P rounding differs per range
    assert rel_err(got, oracle_out(d, B, Hq, Hkv, n_splits=P)).max() <= TOL


def test_rejects_bad_shapes(orc, cuda):
    # attention.hpp:54-56: empty cache / shape mismatch -> invalid_argument
    import torch
    d = build(orc, cuda, 1, 14, 2, 40, seed=9)
    with pytest.raises(ValueError):
        oq.attention_decode(torch.from_numpy(d["q"]).to(cuda), d["cache"], T=0)
    with pytest.raises(ValueError):  # 7 query heads over 2 KV heads
        oq.attention_decode(torch.from_numpy(d["q"][:, :7]).to(cuda), d["cache"])
    with pytest.raises(ValueError):  # more tokens than the cache holds
        oq.attention_decode(torch.from_numpy(d["q"]).to(cuda), d["cache"], T=41)


@pytest.mark.parametrize("b,qjl", [(3, False), (2, False), (2, True), (4, False)])
def test_long_context_weighted_stream_k(orc, cuda, b, qjl):
    """Contexts long enough for the weighted stream-K split (>= 512 tiles per
    stream: every stream start counts as extra tile units) against the
    reference, with ragged lengths and a partial token range."""
    import torch
    B, Hq, Hkv, T = 2, 14, 2, 20000
    d = build(orc, cuda, B, Hq, Hkv, T, b=b, qjl=qjl, seed=9)
    q = torch.from_numpy(d["q"]).to(cuda)
    got = oq.attention_decode(q, d["cache"]).cpu().numpy()
    assert rel_err(got, oracle_out(d, B, Hq, Hkv)).max() <= TOL
    lens = [19999, 16400]
    sl = torch.tensor(lens, dtype=torch.int32, device=cuda)
    got = oq.attention_decode(q, d["cache"], seq_lens=sl).cpu().numpy()
    assert rel_err(got, oracle_out(d, B, Hq, Hkv, lens=lens)).max() <= TOL
    # two ranges of >= 512 tiles each, merged in order == one pass
    parts = torch.stack([oq.attention_partials(q, d["cache"], 0, 3000),
                         oq.attention_partials(q, d["cache"], 3000, T)])
    rows = B * Hq
    out = oq.attention_combine(d["cache"].enc_v, parts, rows, 2, 132, rows * 132)
    full = oq.attention_decode(q, d["cache"]).cpu().numpy()
    assert rel_err(out.reshape(B, Hq, 128).cpu().numpy(), full).max() <= TOL


@pytest.mark.parametrize("b", [3, 2])
def test_attention_pipeline_host_buffers(orc, cuda, b):
    """AttentionPipeline (host q in, host out back, copies on their own
    streams): every step's output equals attention_decode on the device."""
    import torch
    B, Hq, Hkv, T = 2, 14, 2, 3000
    d = build(orc, cuda, B, Hq, Hkv, T, b=b, seed=11)
    pipe = oq.AttentionPipeline(d["cache"], Hq)
    g = torch.Generator().manual_seed(3)
    qs = [torch.randn((B, Hq, 128), generator=g).pin_memory() for _ in range(5)]
    outs = [torch.empty((B, Hq, 128)).pin_memory() for _ in range(5)]
    for qh, oh in zip(qs, outs):
        pipe.run(qh, oh)
    pipe.synchronize()
    for qh, oh in zip(qs, outs):
        want = oq.attention_decode(qh.to(cuda), d["cache"]).cpu()
        assert torch.equal(oh, want)
