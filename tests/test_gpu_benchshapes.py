"""GPU parity at the exact BASELINE.json configurations the bench measures.

The other attention tests run at small shapes; these run the *same* code paths
the headline numbers go through (the stream-K split with its per-stream start
cost of 48 tile units at >= 2048 tiles per stream, the byte-coded W = 7 tiles
with the lagged running max, the QJL sign MMAs at B = 32), at full size:

* C1 (configs[0]) as written: d=128, (b_dir, b_nrm) = (4, 2), seed 0, 4096
  keys and values from Stream(0).child(0/1), queries from child(2) (the
  seed_scope convention, bench.hpp:358-365); codes bit-exact, decode within
  1e-5, MSE equal to the oracle's, q.k scores within the fp32 tolerance;
* C3 (configs[2]): B=8, 28 q / 4 kv heads, T=131072, 3-bit K=V;
* C4 (configs[3]): B=32, T=32768, K 2-bit + QJL, V 2-bit;
* C5 (configs[4]) on one GPU: B=1, T=2^20, 2-bit K=V (the P = 1 point of the
  sequence-sharded mode; ranges of it are merged like P ranks would be).

K/V/Q are Gaussian, generated on the device (Philox) and compressed by K1;
sampled streams' inputs are copied to the host and checked bit-exact against
the oracle's Encoder::encode, and every query head of the sampled streams is
compared with the oracle's attention_decode (attention.hpp:50-73) over the
reference decode of the V records, at the north_star's relative L2 tolerance
1e-3 per (b, head).
"""
import concurrent.futures as cf
import ctypes as C
import os

import numpy as np
import pytest

import paper_2605_21226_b200 as oq

pytestmark = pytest.mark.gpu
TOL = 1e-3
THREADS = max(2, min(32, os.cpu_count() or 2))


def rel_err(got, ref):
    num = np.linalg.norm(got - ref, axis=-1)
    den = np.linalg.norm(ref, axis=-1)
    return num / np.maximum(den, 1e-30)


def _decode_parallel(enc, recs):
    """Oracle Encoder::decode over many records, fanned out over host threads."""
    n = recs.shape[0]
    out = np.empty((n, 128))
    chunk = -(-n // THREADS)

    def work(i):
        a, b = i * chunk, min(n, (i + 1) * chunk)
        if a < b:
            out[a:b] = enc.decode(recs[a:b])

    with cf.ThreadPoolExecutor(THREADS) as ex:
        list(ex.map(work, range(THREADS)))
    return out


def build_bench_cache(orc, cuda, bits, qjl, B, Hkv, T, sample, seed=0, v_scale=1.0):
    """Device-generated K/V for B*Hkv streams of T tokens, compressed by K1 and
    packed into the attention tiles.  Returns the cache plus, for each sampled
    stream, its fp32 inputs and its GPU records on the host."""
    import torch
    bd, bn = oq.default_bit_split(bits)
    kw_k = dict(b_dir=bd, b_nrm=bn, rotation_seed=1000 + seed, qjl=qjl, qjl_seed=2000 + seed)
    kw_v = dict(b_dir=bd, b_nrm=bn, rotation_seed=3000 + seed)
    ek, ev = oq.Encoder(oq.CodecConfig(**kw_k)), oq.Encoder(oq.CodecConfig(**kw_v))
    cache = oq.KVCache(ek, ev, B, Hkv, T)
    g = torch.Generator(device=cuda).manual_seed(1234 + seed)
    n_streams = B * Hkv
    per = max(1, (1 << 21) // T)
    ktb, vtb = ek.tile_bytes(0), ev.tile_bytes(1)
    ntile = (T + 31) // 32
    host = {}
    for s0 in range(0, n_streams, per):
        ns = min(per, n_streams - s0)
        k = torch.randn((ns * T, 128), device=cuda, generator=g)
        v = torch.randn((ns * T, 128), device=cuda, generator=g) * v_scale
        kr, vr = ek.compress(k), ev.compress(v)
        kt = cache.k[s0 * ntile * ktb:(s0 + ns) * ntile * ktb]
        vt = cache.v[s0 * ntile * vtb:(s0 + ns) * ntile * vtb]
        L = oq.lib()
        oq._check(L.oq_cache_pack(ek.handle, 0, oq._ptr(kr), ns, T, T, oq._ptr(kt), T,
                                  oq._stream()))
        oq._check(L.oq_cache_pack(ev.handle, 1, oq._ptr(vr), ns, T, T, oq._ptr(vt), T,
                                  oq._stream()))
        for i in range(ns):
            s = s0 + i
            if s in sample:
                sl = slice(i * T, (i + 1) * T)
                host[s] = dict(k=k[sl].cpu().numpy(), v=v[sl].cpu().numpy(),
                               kr=kr[sl].cpu().numpy(), vr=vr[sl].cpu().numpy())
        del k, v, kr, vr
    cache.tokens = T
    torch.cuda.synchronize()
    ok, ov = orc.encoder(**kw_k), orc.encoder(**kw_v)
    return cache, host, ok, ov


def check_codes(ok, ov, host, n_check=None):
    """Sampled streams' K and V records are bit-exact with the oracle's."""
    for s, h in host.items():
        n = h["k"].shape[0] if n_check is None else n_check
        ref_k = ok.encode_f32(h["k"][:n], threads=THREADS)
        bad = np.nonzero(np.any(ref_k != h["kr"][:n], axis=1))[0]
        assert bad.size == 0, f"stream {s}: {bad.size} K records differ (first {bad[:5]})"
        ref_v = ov.encode_f32(h["v"][:n], threads=THREADS)
        bad = np.nonzero(np.any(ref_v != h["vr"][:n], axis=1))[0]
        assert bad.size == 0, f"stream {s}: {bad.size} V records differ (first {bad[:5]})"


def oracle_rows(ok, ov, host, q, Hkv, G, lens=None, ranges=None, n_splits=1):
    """attention_decode per (b, q head) of the sampled streams, in parallel.
    Returns {(b, h): out[128]}."""
    vdec = {s: _decode_parallel(ov, h["vr"]) for s, h in host.items()}
    jobs = []
    for s in host:
        b, kvh = divmod(s, Hkv)
        L = host[s]["kr"].shape[0] if lens is None else lens[b]
        for j in range(G):
            jobs.append((s, b, kvh * G + j, L))

    def work(job):
        s, b, h, L = job
        if L == 0:
            return (b, h), np.zeros(128)
        return (b, h), ok.attention(q[b, h].astype(np.float64), host[s]["kr"][:L],
                                    vdec[s][:L], n_splits)

    with cf.ThreadPoolExecutor(THREADS) as ex:
        return dict(ex.map(work, jobs))


def compare(got, ref_rows):
    errs = {k: float(rel_err(got[k[0], k[1]], v)) for k, v in ref_rows.items()}
    worst = max(errs, key=errs.get)
    print(f"max rel err {errs[worst]:.3e} at (b, head) {worst}; mean "
          f"{np.mean(list(errs.values())):.3e} over {len(errs)} rows")
    assert errs[worst] <= TOL, (worst, errs[worst], sorted(errs.values())[-5:])
    return errs


# ---------------------------------------------------------------------------
def _seed_scope_inputs(orc, n, seed=0):
    """Stream(seed).child(0/1/2): keys, values, queries (fp64), as C1 states."""
    def gauss(child, count):
        out = np.empty(count)
        orc.L.orc_fill_gaussian(orc.L.orc_stream_child(seed, child), 0,
                                out.ctypes.data_as(C.POINTER(C.c_double)), count)
        return out
    return (gauss(0, n * 128).reshape(n, 128), gauss(1, n * 128).reshape(n, 128),
            gauss(2, 16 * 128).reshape(16, 128))


@pytest.mark.parametrize("rounding", ["local3x3", "scalar"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_c1_roundtrip_as_written(orc, cuda, rounding, dtype):
    """BASELINE configs[0]: d=128, K=V=3 bits (4/2), seed 0, 4096 Gaussian keys
    and values: compress, decode, MSE and q.k check against the reference."""
    import torch
    keys, vals, qs = _seed_scope_inputs(orc, 4096)
    if dtype == "float32":
        keys, vals = keys.astype(np.float32), vals.astype(np.float32)
    cfg = oq.CodecConfig(b_dir=4, b_nrm=2, rounding=rounding, rotation_seed=0)
    enc = oq.Encoder(cfg)
    ref = orc.encoder(b_dir=4, b_nrm=2, rounding=rounding, rotation_seed=0)
    for x in (keys, vals):
        xt = torch.from_numpy(np.ascontiguousarray(x)).to(cuda)
        recs = enc.compress(xt).cpu().numpy()
        if dtype == "float32":
            rrec = ref.encode_f32(x)
        else:
            rrec = np.stack([ref.encode_f64(r) for r in x])
        assert np.array_equal(recs, rrec), "codes not bit-exact"
        dec = enc.decode(torch.from_numpy(recs).to(cuda)).cpu().numpy().astype(np.float64)
        rdec = ref.decode(rrec)
        e = rel_err(dec, rdec)
        assert e.max() <= 1e-5, e.max()
        xd = x.astype(np.float64)
        mse_gpu = float(np.mean((xd - dec) ** 2))
        mse_ref = float(np.mean((xd - rdec) ** 2))
        assert abs(mse_gpu - mse_ref) <= 1e-6 * mse_ref, (mse_gpu, mse_ref)
        # q.k through Encoder::score (prepare + score), fp32 kernel vs fp64 oracle
        s_gpu = enc.scores(torch.from_numpy(qs).float().to(cuda),
                           torch.from_numpy(recs).to(cuda)).cpu().numpy()
        s_ref = np.array([[ref.score(q.astype(np.float32).astype(np.float64), r) for r in rrec[:512]]
                          for q in qs])
        scale = np.linalg.norm(qs, axis=1)[:, None] * np.linalg.norm(rdec[:512], axis=1)[None, :]
        assert np.max(np.abs(s_gpu[:, :512] - s_ref) / scale) <= 1e-5


# ---------------------------------------------------------------------------
def test_c3_qwen_shape_3bit_128k(orc, cuda):
    """configs[2] exactly as benched: B=8, 28/4 heads, T=131072, 3-bit K=V
    (stream-K, 4096 tiles per stream -> start cost 48 tile units)."""
    import torch
    B, Hq, Hkv, T = 8, 28, 4, 131072
    sample = [0, 13, 31]
    cache, host, ok, ov = build_bench_cache(orc, cuda, 3, False, B, Hkv, T, sample)
    check_codes(ok, ov, host)
    q = torch.randn((B, Hq, 128), generator=torch.Generator().manual_seed(99))
    got = oq.attention_decode(q.to(cuda), cache, n_splits=0).cpu().numpy()
    compare(got, oracle_rows(ok, ov, host, q.numpy(), Hkv, Hq // Hkv))


def test_c4_qjl_2bit_32k_batch32(orc, cuda):
    """configs[3] exactly as benched: B=32, T=32768, K 2-bit + QJL, V 2-bit
    (byte-coded W = 7 tiles, lagged running max, QJL sign MMAs)."""
    import torch
    B, Hq, Hkv, T = 32, 28, 4, 32768
    sample = [0, 61, 127]
    cache, host, ok, ov = build_bench_cache(orc, cuda, 2, True, B, Hkv, T, sample, seed=1)
    check_codes(ok, ov, host)
    q = torch.randn((B, Hq, 128), generator=torch.Generator().manual_seed(98))
    got = oq.attention_decode(q.to(cuda), cache, n_splits=0).cpu().numpy()
    compare(got, oracle_rows(ok, ov, host, q.numpy(), Hkv, Hq // Hkv))


def test_c5_1m_tokens_2bit(orc, cuda):
    """configs[4] at P = 1: B=1, T=2^20, 2-bit K=V.  Also the P = 8 image of
    the sharded mode: eight contiguous ranges' partials merged in rank order
    (what every rank runs after the all-gather) equal the single pass."""
    import torch
    B, Hq, Hkv, T = 1, 28, 4, 1 << 20
    sample = [0, 3]
    cache, host, ok, ov = build_bench_cache(orc, cuda, 2, False, B, Hkv, T, sample, seed=2)
    check_codes(ok, ov, host, n_check=1 << 18)
    q = torch.randn((B, Hq, 128), generator=torch.Generator().manual_seed(97)).to(cuda)
    got = oq.attention_decode(q, cache, n_splits=0).cpu().numpy()
    compare(got, oracle_rows(ok, ov, host, q.cpu().numpy(), Hkv, Hq // Hkv))
    P, chunk = 8, T // 8
    parts = torch.stack([oq.attention_partials(q, cache, r * chunk, (r + 1) * chunk)
                         for r in range(P)])
    rows = B * Hq
    out = oq.attention_combine(cache.enc_v, parts, rows, P, 132, rows * 132)
    assert rel_err(out.reshape(B, Hq, 128).cpu().numpy(), got).max() <= TOL


@pytest.mark.parametrize("bits,qjl", [(2, False), (2, True), (3, False)])
def test_large_value_norms(orc, cuda, bits, qjl):
    """V rows with norms ~1e4 (gamma_v up to ~1.3e4): the fp16 P*gamma_v
    operand of the PV MMA stays in range, with and without the lagged max
    (W = 7) and QJL keys."""
    import torch
    B, Hq, Hkv, T = 2, 14, 2, 5000
    cache, host, ok, ov = build_bench_cache(orc, cuda, bits, qjl, B, Hkv, T, [0, 3],
                                            seed=3, v_scale=1000.0)
    q = torch.randn((B, Hq, 128), generator=torch.Generator().manual_seed(96))
    got = oq.attention_decode(q.to(cuda), cache).cpu().numpy()
    assert np.all(np.isfinite(got))
    compare(got, oracle_rows(ok, ov, host, q.numpy(), Hkv, Hq // Hkv))


def test_b4_tiles_long_context(orc, cuda):
    """b = 4 (W = 13) tiles at a 64K-token context: the joint table fits only
    two dithered replicas in shared memory (attention.cu table_rep), so this
    is where its residual fp16 bias would show."""
    import torch
    B, Hq, Hkv, T = 1, 14, 2, 65536
    cache, host, ok, ov = build_bench_cache(orc, cuda, 4, False, B, Hkv, T, [0, 1], seed=4)
    check_codes(ok, ov, host, n_check=1 << 14)
    q = torch.randn((B, Hq, 128), generator=torch.Generator().manual_seed(95))
    got = oq.attention_decode(q.to(cuda), cache).cpu().numpy()
    compare(got, oracle_rows(ok, ov, host, q.numpy(), Hkv, Hq // Hkv))


@pytest.mark.parametrize("bits", [3, 4])
def test_qjl_keys_long_context(orc, cuda, bits):
    """QJL keys on the 10- and 13-bit tiles (b = 3, 4) at a 64K-token context:
    the sign-sketch MMA chain and the dithered tables over a long softmax
    average, against the reference."""
    import torch
    B, Hq, Hkv, T = 1, 14, 2, 65536
    cache, host, ok, ov = build_bench_cache(orc, cuda, bits, True, B, Hkv, T, [0, 1],
                                            seed=40 + bits)
    check_codes(ok, ov, host, n_check=1 << 13)
    q = torch.randn((B, Hq, 128), generator=torch.Generator().manual_seed(96 + bits))
    got = oq.attention_decode(q.to(cuda), cache).cpu().numpy()
    compare(got, oracle_rows(ok, ov, host, q.numpy(), Hkv, Hq // Hkv))
