"""GPU: decode-step append path.

oq_cache_append compresses one new key/value per (batch, kv head) stream and
writes it into its token slot of the attention tiles.  Appending a sequence
token by token must produce the very same tile bytes as compressing the whole
sequence and packing it (oq_cache_pack; those records are checked against the
oracle's encoder here too), for K (with and without the QJL
sidecar) and V, with uniform and per-stream (ragged) positions; attention
over the appended cache then equals attention over the packed one.
"""
import numpy as np
import pytest

import paper_2605_21226_b200 as oq

pytestmark = pytest.mark.gpu


def _encoders(bits, qjl):
    bd, bn = oq.default_bit_split(bits)
    ek = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=21, qjl=qjl, qjl_seed=22))
    ev = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=23))
    return ek, ev


@pytest.mark.parametrize("bits,qjl", [(3, False), (2, True), (2, False), (4, False), (4, True)])
def test_append_equals_pack(cuda, orc, bits, qjl):
    import torch
    B, Hkv, T, cap = 2, 2, 70, 96
    n = B * Hkv
    g = torch.Generator(device=cuda).manual_seed(7)
    k = torch.randn((n, T, 128), device=cuda, generator=g)
    v = torch.randn((n, T, 128), device=cuda, generator=g)
    ek, ev = _encoders(bits, qjl)
    packed = oq.KVCache(ek, ev, B, Hkv, cap)
    kr = ek.compress(k.reshape(-1, 128)).reshape(n, T, -1)
    vr = ev.compress(v.reshape(-1, 128)).reshape(n, T, -1)
    packed.pack(kr, vr, T)
    # the packed records are the oracle's (so the appended tiles are pinned to
    # the CPU encoder, not only to the GPU compress path)
    bd, bn = oq.default_bit_split(bits)
    ok = orc.encoder(b_dir=bd, b_nrm=bn, rotation_seed=21, qjl=qjl, qjl_seed=22)
    ov = orc.encoder(b_dir=bd, b_nrm=bn, rotation_seed=23)
    assert np.array_equal(ok.encode_f32(k.reshape(-1, 128).cpu().numpy()),
                          kr.reshape(n * T, -1).cpu().numpy())
    assert np.array_equal(ov.encode_f32(v.reshape(-1, 128).cpu().numpy()),
                          vr.reshape(n * T, -1).cpu().numpy())
    app = oq.KVCache(ek, ev, B, Hkv, cap)
    for t in range(T):
        app.append(k[:, t].reshape(B, Hkv, 128), v[:, t].reshape(B, Hkv, 128))
    assert app.tokens == T
    assert torch.equal(app.k, packed.k), "K tiles differ"
    assert torch.equal(app.v, packed.v), "V tiles differ"
    q = torch.randn((B, 7 * Hkv, 128), device=cuda, generator=g)
    a = oq.attention_decode(q, app)
    b = oq.attention_decode(q, packed)
    assert torch.equal(a, b)


def test_append_ragged_positions(cuda):
    import torch
    B, Hkv, cap = 3, 1, 96
    ek, ev = _encoders(3, False)
    lens = [5, 33, 40]
    g = torch.Generator(device=cuda).manual_seed(9)
    k = torch.randn((B, max(lens), 128), device=cuda, generator=g)
    v = torch.randn((B, max(lens), 128), device=cuda, generator=g)
    app = oq.KVCache(ek, ev, B, Hkv, cap)
    # each step appends token t of every sequence still growing; finished ones
    # are parked at position cap - 1 (a slot attention never reads here)
    for t in range(max(lens)):
        pos = torch.tensor([t if t < L else cap - 1 for L in lens], dtype=torch.int64, device=cuda)
        app.append(k[:, t].reshape(B, 1, 128), v[:, t].reshape(B, 1, 128), pos=pos)
    ref = oq.KVCache(ek, ev, B, Hkv, cap)
    for b, L in enumerate(lens):
        one = oq.KVCache(ek, ev, 1, 1, cap)
        one.pack(ek.compress(k[b, :L]), ev.compress(v[b, :L]), L)
        kt, vt = ek.tile_bytes(0), ev.tile_bytes(1)
        ntile = (L + 31) // 32
        per_k, per_v = (cap + 31) // 32 * kt, (cap + 31) // 32 * vt
        assert torch.equal(app.k[b * per_k:b * per_k + ntile * kt], one.k[:ntile * kt]), b
        assert torch.equal(app.v[b * per_v:b * per_v + ntile * vt], one.v[:ntile * vt]), b


@pytest.mark.parametrize("qjl", [False, True])
def test_append_records_and_bf16(cuda, qjl):
    """The fused K+V append (one launch without QJL) hands back the same OCTO
    records as oq_compress on bf16 inputs, and writes the same tiles as pack."""
    import torch
    B, Hkv, cap = 4, 8, 64
    n = B * Hkv
    ek, ev = _encoders(3, qjl)
    g = torch.Generator(device=cuda).manual_seed(11)
    k = torch.randn((B, Hkv, 128), device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn((B, Hkv, 128), device=cuda, generator=g).to(torch.bfloat16)
    rk = torch.zeros((n, ek.record_bytes), dtype=torch.uint8, device=cuda)
    rv = torch.zeros((n, ev.record_bytes), dtype=torch.uint8, device=cuda)
    app = oq.KVCache(ek, ev, B, Hkv, cap)
    app.append(k, v, pos=37, records=(rk, rv))
    wk, wv = ek.compress(k.reshape(n, 128)), ev.compress(v.reshape(n, 128))
    assert torch.equal(rk, wk) and torch.equal(rv, wv)
    ref = oq.KVCache(ek, ev, B, Hkv, cap)
    z = lambda r: torch.zeros((n, 38, r.shape[1]), dtype=torch.uint8, device=cuda)
    zk, zv = z(wk), z(wv)
    zk[:, 37], zv[:, 37] = wk, wv
    # tokens 0..36 of `ref` are all-zero records; append leaves app's untouched
    # (zero-initialised tiles), so only token 37's fields can differ
    ref.pack(zk, zv, 38)
    kt, vt = ek.tile_bytes(0), ev.tile_bytes(1)
    per_k, per_v = (cap + 31) // 32 * kt, (cap + 31) // 32 * vt
    for s in range(n):
        a = app.k[s * per_k + kt:s * per_k + 2 * kt]
        b = ref.k[s * per_k + kt:s * per_k + 2 * kt]
        assert torch.equal(a, b), s
        assert torch.equal(app.v[s * per_v + vt:s * per_v + 2 * vt],
                           ref.v[s * per_v + vt:s * per_v + 2 * vt]), s


def test_append_then_attention_back_to_back(cuda):
    """Decode-step pattern with no host synchronisation between the append
    and the attention launch that reads it (the attention kernel is launched
    with programmatic dependent launch): every step's output equals the same
    step recomputed after a device synchronisation."""
    import torch
    B, Hkv, cap = 2, 2, 4096
    ek, ev = _encoders(3, False)
    cache = oq.KVCache(ek, ev, B, Hkv, cap)
    g = torch.Generator(device=cuda).manual_seed(3)
    T0 = 3000
    cache.pack(ek.compress(torch.randn((B * Hkv * T0, 128), device=cuda, generator=g)).reshape(
        B * Hkv, T0, -1), ev.compress(torch.randn((B * Hkv * T0, 128), device=cuda,
                                                  generator=g)).reshape(B * Hkv, T0, -1), T0)
    q = torch.randn((B, 7 * Hkv, 128), device=cuda, generator=g)
    ks = torch.randn((40, B, Hkv, 128), device=cuda, generator=g)
    vs = torch.randn((40, B, Hkv, 128), device=cuda, generator=g)
    outs = []
    for t in range(40):  # back to back: append, attention, append, attention, ...
        cache.append(ks[t], vs[t])
        outs.append(oq.attention_decode(q, cache).clone())
    torch.cuda.synchronize()
    # every step's output equals attention over the final cache read up to
    # that step's length (same T, so the same work split), computed after a
    # synchronisation: later appends leave earlier tokens' codes unchanged
    for t in range(40):
        torch.cuda.synchronize()
        want = oq.attention_decode(q, cache, T=T0 + t + 1)
        torch.cuda.synchronize()
        assert torch.equal(want, outs[t]), t
