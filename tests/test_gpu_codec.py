"""GPU parity: K1 compress is bit-exact, K2 decode within 1e-5 (rel).

The oracle (oracle/octo_oracle.c, pinned to the reference in
test_oracle.py) is the checker; inputs are the reference's own Gaussian
streams.  Every call goes through the C ABI (liboctoquant_b200.so).
"""
import os

import numpy as np
import pytest

import paper_2605_21226_b200 as oq

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

CONFIGS = [
    dict(b_dir=3, b_nrm=1, rounding="local3x3"),
    dict(b_dir=4, b_nrm=2, rounding="local3x3"),
    dict(b_dir=5, b_nrm=3, rounding="local3x3"),
    dict(b_dir=4, b_nrm=2, rounding="scalar"),
    dict(b_dir=3, b_nrm=1, rounding="scalar"),
    dict(b_dir=5, b_nrm=3, rounding="scalar"),
    dict(b_dir=3, b_nrm=1, rounding="local3x3", qjl=True),
    dict(b_dir=4, b_nrm=2, rounding="local2x2", qjl=True),
    dict(b_dir=3, b_nrm=2, rounding="full"),
    dict(b_dir=6, b_nrm=4, rounding="local3x3"),
    dict(b_dir=8, b_nrm=8, rounding="local3x3", qjl=True),
    dict(b_dir=1, b_nrm=1, rounding="local3x3"),
    dict(dim=64, b_dir=5, b_nrm=3, rounding="local3x3"),
    dict(dim=32, b_dir=4, b_nrm=2, rounding="local3x3", qjl=True),
    dict(dim=16, b_dir=2, b_nrm=4, rounding="local3x3", qjl=True),
    dict(dim=8, b_dir=3, b_nrm=3, rounding="scalar"),
    dict(dim=4, b_dir=2, b_nrm=2, rounding="full"),
    dict(dim=256, b_dir=4, b_nrm=2, rounding="local3x3", rotation_seed=7, qjl=True, qjl_seed=9),
]


def _ids(c):
    return "-".join(f"{k}{v}" for k, v in c.items())


def _inputs(orc, seed, n, dim):
    x = orc.gaussian_f32(orc.L.orc_stream_child(seed, 0), n * dim).reshape(n, dim)
    x[3] = 0.0          # zero key (codec_test.cpp:65-73)
    x[4] *= 1e-30       # below the 1e-12 guard on ||k||
    x[5] *= 1e20        # large norm
    x[6] = 0.0
    x[6, 0] = 5.0       # basis vector (codec_test.cpp:80-115)
    return x


@pytest.mark.parametrize("cfg", CONFIGS, ids=_ids)
def test_compress_bit_exact_and_decode(orc, cuda, cfg):
    import torch
    dim = cfg.get("dim", 128)
    n = 3000
    x = _inputs(orc, 1, n, dim)
    eo = orc.encoder(**cfg)
    enc = oq.Encoder(oq.CodecConfig(**cfg))
    assert enc.record_bytes == eo.rb
    want = eo.encode_f32(x)
    got = enc.compress(torch.from_numpy(x).to(cuda)).cpu().numpy()
    bad = np.nonzero((got != want).any(1))[0]
    assert bad.size == 0, f"{bad.size} mismatching records, first {bad[:5]}"
    # K2 decode: rel err <= 1e-5 per vector vs the fp64 reference decode
    dec = enc.decode(torch.from_numpy(want).to(cuda)).cpu().numpy().astype(np.float64)
    ref = eo.decode(want)
    num = np.linalg.norm(dec - ref, axis=1)
    den = np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
    rel = np.where(np.linalg.norm(ref, axis=1) > 0, num / den, num)
    assert rel.max() <= 1e-5, rel.max()


@pytest.mark.parametrize("dtype", ["float64", "bfloat16", "float16"])
def test_compress_other_dtypes(orc, cuda, dtype):
    import torch
    x = _inputs(orc, 2, 1024, 128)
    t = torch.from_numpy(x).to(cuda).to(getattr(torch, dtype))
    xs = t.float().cpu().numpy()  # the exact values the kernel widens
    cfg = dict(b_dir=4, b_nrm=2)
    got = oq.Encoder(oq.CodecConfig(**cfg)).compress(t).cpu().numpy()
    want = orc.encoder(**cfg).encode_f32(xs)
    assert np.array_equal(got, want)


def test_golden_fixtures(cuda):
    import torch
    z = np.load(os.path.join(GOLDEN, "codes.npz"))
    names = ["scalar", "local2x2", "local3x3", "full"]
    for name in z.files:
        if not name.startswith("rec_"):
            continue
        tag = name[4:]
        dim, bd, bn, rnd, qjl = (int(v) for v in z["cfg_" + tag])
        enc = oq.Encoder(oq.CodecConfig(dim=dim, b_dir=bd, b_nrm=bn, rounding=names[rnd],
                                        qjl=bool(qjl)))
        got = enc.compress(torch.from_numpy(z["x_" + tag]).to(cuda)).cpu().numpy()
        assert np.array_equal(got, z[name]), tag


@pytest.mark.parametrize("b", [2, 3, 4])
def test_c2_million_keys_bit_exact(orc, cuda, b):
    """BASELINE config 2: 2^20 keys, d=128, b in {4,3,2}, bit-exact vs CPU."""
    import torch
    n = 1 << 20
    bd, bn = oq.default_bit_split(b)
    g = torch.Generator(device=cuda).manual_seed(100 + b)
    x = torch.randn((n, 128), device=cuda, generator=g, dtype=torch.float32)
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn))
    got = enc.compress(x).cpu().numpy()
    want = orc.encoder(b_dir=bd, b_nrm=bn).encode_f32(x.cpu().numpy(),
                                                     threads=os.cpu_count() or 8)
    bad = int((got != want).any(1).sum())
    assert bad == 0, f"{bad} of {n} records differ"
    # decode round trip at full size: rel err <= 1e-5
    dec = enc.decode(torch.from_numpy(want).to(cuda))
    idx = torch.randint(0, n, (4096,), generator=torch.Generator().manual_seed(1))
    ref = orc.encoder(b_dir=bd, b_nrm=bn).decode(want[idx.numpy()])
    d = dec[idx.to(cuda)].cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(d - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() <= 1e-5


def test_wire_roundtrip_and_padding(orc, cuda):
    import torch
    cfg = oq.CodecConfig(dim=4, b_dir=3, b_nrm=1)  # 4 dir pad bits, 6 nrm pad bits
    enc = oq.Encoder(cfg)
    x = torch.from_numpy(_inputs(orc, 3, 64, 4)).to(cuda)
    recs = enc.compress(x)
    blob = oq.pack_keys(cfg, recs)
    assert len(blob) == 20 + 64 * 7
    cfg2, back = oq.unpack_keys(blob)
    assert torch.equal(back.cpu(), recs.cpu())
    # codec_test.cpp:496-517: dirty padding is rejected
    for byte, bit in [(20 + 5, 4), (20 + 5, 7), (20 + 6, 2), (20 + 6, 7)]:
        bad = bytearray(blob)
        bad[byte] ^= 1 << bit
        with pytest.raises(oq.FormatError):
            oq.unpack_keys(bytes(bad))


def test_pack_keys_matches_reference_blob(ref, cuda, orc):
    import torch
    cfg = oq.CodecConfig(b_dir=4, b_nrm=2, qjl=True)
    x = _inputs(orc, 4, 100, 128)
    blob = oq.pack_keys(cfg, oq.Encoder(cfg).compress(torch.from_numpy(x).to(cuda)))
    want = ref.encoder(b_dir=4, b_nrm=2, qjl=True).encode_f32(x)
    assert blob[20:] == want.tobytes()


@pytest.mark.parametrize("qjl", [False, True])
def test_empty_batches(cuda, qjl):
    """Zero keys in, zero records out (and back): no launch, no error, the way
    the reference's encode/decode loops simply do nothing."""
    import torch
    enc = oq.Encoder(oq.CodecConfig(b_dir=4, b_nrm=2, qjl=qjl))
    r = enc.compress(torch.zeros((0, 128), device=cuda))
    assert r.shape == (0, enc.record_bytes)
    d = enc.decode(r)
    assert d.shape == (0, 128)
    torch.cuda.synchronize()


def test_rejects_dimension_mismatch(cuda):
    import torch
    with pytest.raises(ValueError):
        oq.Encoder(oq.CodecConfig()).compress(torch.zeros((2, 64), device=cuda))


@pytest.mark.parametrize("dtype", ["bfloat16", "float16"])
@pytest.mark.parametrize("b,rounding", [(2, "local3x3"), (3, "local3x3"), (4, "local3x3"),
                                        (3, "scalar")])
def test_fast_path_16bit_keys_bit_exact(orc, cuda, dtype, b, rounding):
    """The certified fast path (K1a + K1b) on bf16 / fp16 keys, as a decoder
    appends them: 2^17 keys, bit-exact vs the CPU reference on the widened
    values."""
    import torch
    n = 1 << 17
    bd, bn = oq.default_bit_split(b)
    g = torch.Generator(device=cuda).manual_seed(300 + b)
    x = (torch.randn((n, 128), device=cuda, generator=g) * 3.0).to(getattr(torch, dtype))
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rounding=rounding))
    fl = torch.zeros(1, dtype=torch.int32, device=cuda)
    got = enc.compress(x, flagged=fl).cpu().numpy()
    want = orc.encoder(b_dir=bd, b_nrm=bn, rounding=rounding).encode_f32(
        x.float().cpu().numpy(), threads=os.cpu_count() or 8)
    bad = int((got != want).any(1).sum())
    assert bad == 0, f"{bad} of {n} records differ ({int(fl.item())} flagged)"


SMALL = [c for c in CONFIGS if c.get("dim", 128) == 128]  # QJL sidecar included


@pytest.mark.parametrize("dtype", ["float32", "float64", "bfloat16"])
@pytest.mark.parametrize("cfg", SMALL, ids=_ids)
def test_small_batch_kernel_bit_exact(orc, cuda, cfg, dtype):
    """Batches of <= 2048 d=128 keys (a decode step's append) take the
    one-warp-per-key kernel: bit-exact in every rounding mode and bit split,
    ragged batch sizes included."""
    import torch
    for n in (1, 7, 777):
        x = _inputs(orc, 5, max(n, 8), 128)[:n]
        t = torch.from_numpy(x).to(cuda).to(getattr(torch, dtype))
        if dtype == "float64":
            t = t * (1.0 + 1e-9)  # off the fp32 grid: the squares round
        xs = t.double().cpu().numpy()
        got = oq.Encoder(oq.CodecConfig(**cfg)).compress(t).cpu().numpy()
        eo = orc.encoder(**cfg)
        want = np.stack([eo.encode_f64(k) for k in xs]) if dtype == "float64" else \
            eo.encode_f32(xs.astype(np.float32))
        bad = np.nonzero((got != want).any(1))[0]
        assert bad.size == 0, f"n={n}: {bad.size} mismatching records, first {bad[:5]}"


@pytest.mark.parametrize("qjl", [False, True])
@pytest.mark.parametrize("b", [2, 3, 4])
@pytest.mark.parametrize("rounding", ["local3x3", "scalar"])
def test_fast_path_special_keys_bit_exact(orc, cuda, b, rounding, qjl):
    """Batches large enough for the certified fp32 pass (> 8192 keys) with the
    keys it cannot certify at all mixed in: zero keys, norms outside
    [2^-60, 2^60] (every triplet goes to the exact fixup), basis vectors
    (exact ties in the 3x3 window), tiny triplets next to large ones, and
    inf / NaN coordinates — all bit-exact against the CPU reference."""
    import torch
    n = 20000
    bd, bn = oq.default_bit_split(b)
    x = orc.gaussian_f32(orc.L.orc_stream_child(77 + b, 0), n * 128).reshape(n, 128)
    rng = np.random.default_rng(b)
    idx = rng.choice(n, 64, replace=False)
    for j, i in enumerate(idx):
        kind = j % 8
        if qjl and kind in (5, 6):
            # an inf/NaN key's QJL residual norm is NaN, and the NaN's sign bit
            # (the f16 gamma_r's top byte) follows the host's NaN propagation
            # (x86: the default NaN is negative); codes stay bit-exact
            kind = 3
        if kind == 0:
            x[i] = 0.0
        elif kind == 1:
            x[i] *= 1e-25
        elif kind == 2:
            x[i] *= 1e25
        elif kind == 3:
            x[i] = 0.0
            x[i, j % 128] = 3.0
        elif kind == 4:
            x[i, : 3 * (j % 40)] *= 1e-6  # tiny leading triplets
        elif kind == 5:
            x[i, j % 128] = np.inf
        elif kind == 6:
            x[i, j % 128] = np.nan
        else:
            x[i, 0::3] = x[i, 1::3]  # many equal |t0| = |t1| folds
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rounding=rounding, qjl=qjl))
    fl = torch.zeros(1, dtype=torch.int32, device=cuda)
    got = enc.compress(torch.from_numpy(x).to(cuda), flagged=fl).cpu().numpy()
    want = orc.encoder(b_dir=bd, b_nrm=bn, rounding=rounding, qjl=qjl).encode_f32(
        x, threads=os.cpu_count() or 8)
    bad = np.nonzero((got != want).any(1))[0]
    assert bad.size == 0, f"{bad.size} records differ, first {bad[:5]} ({int(fl.item())} flagged)"
    assert int(fl.item()) >= 40  # the special keys all went through the fixup


@pytest.mark.parametrize("b", [2, 3, 4])
def test_fast_path_qjl_bit_exact(orc, cuda, b):
    """The certified pass with the QJL sidecar (residual norm and signs
    certified like the codes; flagged keys re-encoded whole by the exact
    kernel): 2^17 keys, bit-exact, and the flag rate stays small."""
    import torch
    n = 1 << 17
    bd, bn = oq.default_bit_split(b)
    g = torch.Generator(device=cuda).manual_seed(500 + b)
    x = torch.randn((n, 128), device=cuda, generator=g)
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, qjl=True, qjl_seed=9))
    fl = torch.zeros(1, dtype=torch.int32, device=cuda)
    got = enc.compress(x, flagged=fl).cpu().numpy()
    want = orc.encoder(b_dir=bd, b_nrm=bn, qjl=True, qjl_seed=9).encode_f32(
        x.cpu().numpy(), threads=os.cpu_count() or 8)
    bad = int((got != want).any(1).sum())
    assert bad == 0, f"{bad} of {n} records differ ({int(fl.item())} flagged)"
    assert int(fl.item()) < 0.2 * n
