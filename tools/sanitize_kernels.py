"""Small invocation of every hot kernel (for compute-sanitizer runs)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2605_21226_b200 as oq

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
for bits in (2, 3, 4):
    for rnd in ("local3x3", "scalar"):
        bd, bn = oq.default_bit_split(bits)
        enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rounding=rnd))
        x = torch.randn((3000, 128), device=dev, generator=g)   # partial tail blocks too
        r = enc.compress(x)
        enc.decode(r)
        enc.compress(x[:77].to(torch.bfloat16))  # one-warp-per-key small-batch encoder
B, Hkv, T = 2, 2, 300
bd, bn = oq.default_bit_split(3)
ek = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=5))
ev = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=6))
k = torch.randn((B * Hkv * T, 128), device=dev, generator=g)
v = torch.randn((B * Hkv * T, 128), device=dev, generator=g)
cache = oq.KVCache(ek, ev, B, Hkv, T + 40)
cache.pack(ek.compress(k), ev.compress(v), T)
cache.append(torch.randn((B, Hkv, 128), device=dev), torch.randn((B, Hkv, 128), device=dev))
# fused K+V append with per-stream positions and record outputs, bf16 inputs
rk = torch.empty((B * Hkv, ek.record_bytes), dtype=torch.uint8, device=dev)
rv = torch.empty((B * Hkv, ev.record_bytes), dtype=torch.uint8, device=dev)
cache.append(torch.randn((B, Hkv, 128), device=dev).to(torch.bfloat16),
             torch.randn((B, Hkv, 128), device=dev).to(torch.bfloat16),
             pos=torch.arange(B * Hkv, device=dev) + T, records=(rk, rv))
# QJL keys: one-warp-per-key small batches, the certified pass + whole-key
# rekey of its flagged keys (20000 keys), the fused append with QJL keys
eq3 = oq.Encoder(oq.CodecConfig(b_dir=4, b_nrm=2, qjl=True, rotation_seed=9))
eq3.compress(torch.randn((100, 128), device=dev, generator=g))
eq3.compress(torch.randn((20000, 128), device=dev, generator=g))
eq = oq.Encoder(oq.CodecConfig(b_dir=3, b_nrm=1, qjl=True, rotation_seed=7))
ev2 = oq.Encoder(oq.CodecConfig(b_dir=3, b_nrm=1, rotation_seed=8))
c2 = oq.KVCache(eq, ev2, B, Hkv, 64)
c2.append(torch.randn((B, Hkv, 128), device=dev), torch.randn((B, Hkv, 128), device=dev), pos=3)
q = torch.randn((B, 7 * Hkv, 128), device=dev, generator=g)
oq.attention_decode(q, cache)
oq.attention_partials(q, cache, 0, cache.tokens)
# 2-bit tiles: the 12-warp TMA-ring K3 (its default), with and without QJL keys,
# and the 8-warp register variant
for qjl in (False, True):
    e2k = oq.Encoder(oq.CodecConfig(b_dir=3, b_nrm=1, qjl=qjl, rotation_seed=21))
    e2v = oq.Encoder(oq.CodecConfig(b_dir=3, b_nrm=1, rotation_seed=22))
    c3 = oq.KVCache(e2k, e2v, B, Hkv, 2000)
    c3.pack(e2k.compress(torch.randn((B * Hkv * 2000, 128), device=dev, generator=g)),
            e2v.compress(torch.randn((B * Hkv * 2000, 128), device=dev, generator=g)), 2000)
    oq.attention_decode(q, c3)
    oq.attention_decode(q, c3, n_splits=3)
    oq.attention_partials(q, c3, 100, 1500)
# 13-bit tiles (b = 4: two-replica table, 8-warp TMA ring), with and without QJL
for qjl in (False, True):
    e4k = oq.Encoder(oq.CodecConfig(b_dir=5, b_nrm=3, qjl=qjl, rotation_seed=31))
    e4v = oq.Encoder(oq.CodecConfig(b_dir=5, b_nrm=3, rotation_seed=32))
    c4 = oq.KVCache(e4k, e4v, B, Hkv, 700)
    c4.pack(e4k.compress(torch.randn((B * Hkv * 700, 128), device=dev, generator=g)),
            e4v.compress(torch.randn((B * Hkv * 700, 128), device=dev, generator=g)), 700)
    oq.attention_decode(q, c4)
    oq.attention_decode(q, c4, seq_lens=torch.tensor([650, 90], dtype=torch.int32, device=dev))
# ragged lengths on the 10-bit tiles, and the fused peer-memory exchange with
# one rank (stores, system fence, flag, acquire-spin, merge; two epochs)
oq.attention_decode(q, cache, seq_lens=torch.tensor([T, 17], dtype=torch.int32, device=dev))
xb = torch.zeros(oq.p2p_exchange_bytes(cache, q.shape[1], 1), dtype=torch.uint8, device=dev)
for ep in (1, 2):
    oq.attention_decode_p2p(q, cache, 0, cache.tokens, 0, 1, [xb], ep)
# the exact fp64 per-key API (exact_api.cu)
for cfg in (oq.CodecConfig(b_dir=4, b_nrm=2), oq.CodecConfig(b_dir=5, b_nrm=3, qjl=True),
            oq.CodecConfig(dim=64, b_dir=3, b_nrm=1)):
    e = oq.Encoder(cfg)
    r = e.compress(torch.randn((257, cfg.dim), device=dev, generator=g))
    e.decode_exact(r)
    e.reconstruct_rotated(r)
    rot, sk = e.prepare(torch.randn((3, cfg.dim), device=dev, generator=g))
    e.score_prepared(rot, sk, r)
    e.attention_exact(torch.randn((2, cfg.dim), device=dev, generator=g), r,
                      torch.randn((257, 16), device=dev, generator=g), n_splits=4)
torch.cuda.synchronize()
print("sanitize run ok")
