"""Pin the CPU oracle (oracle/octo_oracle.c) before trusting it.

1. Known-answer vectors copied from the reference's own GTest suites
   (/root/reference/proj/tests/*.cpp, cited per test).
2. Bit-for-bit agreement with the reference itself (oracle/_ref, compiled
   from /root/reference/proj/include) on codebooks, codes, decode, score and
   attention.
3. The committed golden fixtures in tests/golden/ (generated from _ref by
   tests/golden/make_golden.py).
"""
import math
import os
import struct

import numpy as np
import pytest

from oracle_bind import record_bytes

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---- rng_test.cpp:12-17 ------------------------------------------------------
def test_stream_seed_derivation(orc):
    L = orc.L
    assert L.orc_stream_child(5, 7) == 0xcd56133855ec691e
    assert L.orc_stream_at(42, 0) == 0xbdd732262feb6e95
    assert L.orc_stream_at(42, 1) == 0x28efe333b266f103


# ---- io_test.cpp:60-84 f16 round-nearest-even ---------------------------------
def _f32(x):
    return struct.unpack("<f", struct.pack("<f", x))[0]


@pytest.mark.parametrize("x,h", [(1.0, 0x3c00), (-0.0, 0x8000), (65504.0, 0x7bff),
                                 (65520.0, 0x7c00), (2.0 ** -24, 0x0001), (2.0 ** -25, 0x0000),
                                 (0.1, 0x2e66), (1.0 + 2.0 ** -11, 0x3c00),
                                 (1.0 + 1.5 * 2.0 ** -11, 0x3c01),
                                 (1.0 + 1.5 * 2.0 ** -10, 0x3c02)])
def test_f16_pinned(orc, x, h):
    assert orc.L.orc_f32_to_f16(_f32(x)) == h


def test_f16_exact_roundtrip(orc):
    for h in range(0, 0x10000, 7):
        if ((h >> 10) & 0x1f) == 0x1f:
            continue
        assert orc.L.orc_f32_to_f16(orc.L.orc_f16_to_f32(h)) == h


# ---- lloydmax_test.cpp:103-137 quantize rule -----------------------------------
def test_quantize_ties_go_up(orc):
    import ctypes as C
    b = np.array([0.0])
    p = b.ctypes.data_as(C.POINTER(C.c_double))
    assert orc.L.orc_quantize(p, 1, -0.2) == 0
    assert orc.L.orc_quantize(p, 1, 0.0) == 1  # boundary -> upper cell
    assert orc.L.orc_quantize(p, 1, -5.0) == 0
    assert orc.L.orc_quantize(p, 1, 5.0) == 1


def test_centroids_map_to_themselves(orc):
    import ctypes as C
    for c, b in (orc.xi_book(3), orc.rho_book(128, 3)):
        p = b.ctypes.data_as(C.POINTER(C.c_double))
        for i, v in enumerate(c):
            assert orc.L.orc_quantize(p, len(b), v) == i


def test_quantize_matches_nearest_centroid(orc):
    import ctypes as C
    c, b = orc.xi_book(4)
    p = b.ctypes.data_as(C.POINTER(C.c_double))
    rng = np.random.default_rng(67)
    for x in rng.uniform(-1, 1, 20000):
        assert orc.L.orc_quantize(p, len(b), x) == int(np.argmin(np.abs(x - c)))


# ---- octahedral_test.cpp:18-70 ------------------------------------------------
def _enc(orc, n):
    import ctypes as C
    a = np.asarray(n, np.float64)
    out = np.empty(2)
    orc.L.orc_oct_encode(a.ctypes.data_as(C.POINTER(C.c_double)),
                         out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def _dec(orc, x, y):
    import ctypes as C
    out = np.empty(3)
    orc.L.orc_oct_decode(x, y, out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def test_oct_pinned(orc):
    assert list(_enc(orc, [0, 0, 1])) == [0.0, 0.0]
    assert list(_enc(orc, [1, 0, 0])) == [1.0, 0.0]
    assert list(_enc(orc, [0, 0, -1])) == [1.0, 1.0]
    s = 1 / math.sqrt(3)
    assert np.allclose(_enc(orc, [s, s, s]), [1 / 3, 1 / 3], atol=1e-12)
    assert list(_enc(orc, [0, 0, 0])) == [0.0, 0.0]
    assert list(_dec(orc, 0.0, 0.0)) == [0.0, 0.0, 1.0]
    for xi in (-1.0, 1.0):
        for eta in (-1.0, 1.0):
            assert list(_dec(orc, xi, eta)) == [0.0, 0.0, -1.0]
    assert np.allclose(_dec(orc, 0.5, 0.5), [0.70710678, 0.70710678, 0.0], atol=1e-8)


# ---- codec_test.cpp ------------------------------------------------------------
def test_payload_sizes(orc):
    # codec_test.cpp:412-421 (43 B default), 535-547 rate tests via sizes
    assert record_bytes(128, 3, 1, False) == 43
    assert record_bytes(128, 4, 2, False) == 58
    assert record_bytes(128, 5, 3, False) == 75
    assert record_bytes(128, 3, 1, True) == 61
    enc = orc.encoder()
    assert enc.rb == 43


def test_zero_key_is_inert(orc):
    # codec_test.cpp:65-73
    enc = orc.encoder()
    rec = enc.encode_f64(np.zeros(128))
    g, d, n, _, _ = enc.codes(rec)
    assert g == 0.0
    assert np.all(enc.decode(rec) == 0.0)


def test_basis_vector_matches_exhaustive_search(orc):
    # codec_test.cpp:80-115: d=4, (2,2), full search == per-triplet argmin
    enc = orc.encoder(dim=4, b_dir=2, b_nrm=2, rounding="full")
    rec = enc.encode_f64(np.array([5.0, 0.0, 0.0, 0.0]))
    g, d, n, _, _ = enc.codes(rec)
    assert g == 5.0
    signs = np.empty(4)
    import ctypes as C
    orc.L.orc_rotation_signs(4, 0, signs.ctypes.data_as(C.POINTER(C.c_double)))
    ur = np.array([1.0, 0, 0, 0]) * signs
    x = ur.copy()
    orc.L.orc_fwht(x.ctypes.data_as(C.POINTER(C.c_double)), 4)
    padded = np.concatenate([x, [0.0, 0.0]])
    xc, _ = orc.xi_book(2)
    rc, _ = orc.rho_book(4, 2)
    for t in range(2):
        tv = padded[3 * t:3 * t + 3]
        best, arg = 1e300, None
        for i in range(4):
            for j in range(4):
                nv = _dec(orc, xc[i], xc[j])
                for r in range(4):
                    l = float(np.sum((tv - rc[r] * nv) ** 2))
                    if l < best:
                        best, arg = l, (i, j, r)
        assert (d[2 * t], d[2 * t + 1], n[t]) == arg


def test_code_assignment_idempotent(orc):
    # codec_test.cpp:190-202 (1000 of the 10^4 keys)
    enc = orc.encoder()
    x = orc.gaussian_f32(13, 1000 * 128).reshape(-1, 128)
    a = enc.encode_f32(x)
    dec = enc.decode(a)
    b = np.stack([enc.encode_f64(k) for k in dec])
    for ra, rb in zip(a, b):
        _, da, na, _, _ = enc.codes(ra)
        _, db, nb, _, _ = enc.codes(rb)
        assert np.array_equal(da, db) and np.array_equal(na, nb)


def test_all_zero_indices_norm(orc):
    # codec_test.cpp:204-219
    enc = orc.encoder()
    rec = np.zeros(43, np.uint8)
    rec[:4] = np.frombuffer(np.float32(1.0).tobytes(), np.uint8)
    dec = enc.decode(rec)[0]
    rho0 = orc.rho_book(128, 1)[0][0]
    xc = orc.xi_book(3)[0]
    n0 = _dec(orc, xc[0], xc[0])
    expected = math.sqrt(rho0 * rho0 * (42.0 + n0[0] ** 2 + n0[1] ** 2))
    assert abs(np.linalg.norm(dec) - expected) < 1e-12


def test_score_equals_dot_with_decode(orc):
    # codec_test.cpp:239-262
    enc = orc.encoder()
    x = orc.gaussian_f32(17, 50 * 128).reshape(-1, 128)
    recs = enc.encode_f32(x)
    dec = enc.decode(recs)
    q = orc.gaussian_f32(18, 10 * 128).reshape(-1, 128).astype(np.float64)
    for qi in q:
        for r, dv in zip(recs, dec):
            s = enc.score(qi, r)
            ref = float(np.dot(qi, dv))
            assert abs(s - ref) <= 1e-9 * max(1.0, np.linalg.norm(qi) * np.linalg.norm(dv))


def test_attention_split_invariance_and_direct_softmax(orc):
    # codec_test.cpp:301-336
    enc = orc.encoder()
    x = orc.gaussian_f32(23, 257 * 128).reshape(-1, 128)
    recs = enc.encode_f32(x)
    vals = orc.gaussian_f32(24, 257 * 16).reshape(-1, 16).astype(np.float64)
    q = orc.gaussian_f32(25, 128).astype(np.float64)
    s1 = enc.attention(q, recs, vals, 1)
    s8 = enc.attention(q, recs, vals, 8)
    assert np.allclose(s1, s8, atol=1e-6)
    logits = np.array([enc.score(q, r) for r in recs]) / math.sqrt(128)
    w = np.exp(logits - logits.max())
    ref = (w[:, None] * vals).sum(0) / w.sum()
    assert np.allclose(s1, ref, atol=1e-9)


def test_single_key_returns_value_row(orc):
    # codec_test.cpp:338-351
    enc = orc.encoder()
    x = orc.gaussian_f32(29, 128).reshape(1, 128)
    vals = orc.gaussian_f32(30, 8).reshape(1, 8).astype(np.float64)
    out = enc.attention(orc.gaussian_f32(31, 128).astype(np.float64), enc.encode_f32(x), vals)
    assert np.array_equal(out, vals[0])


def test_attention_rejects_empty(orc):
    enc = orc.encoder()
    with pytest.raises(ValueError):
        enc.attention(np.zeros(128), np.zeros((0, 43), np.uint8), np.zeros((0, 8)))


# ---- oracle vs the reference itself (oracle/_ref) -------------------------------
@pytest.mark.parametrize("bits", [1, 2, 3, 4, 5, 6])
def test_xi_books_bit_identical_to_reference(orc, ref, bits):
    c1, b1 = orc.xi_book(bits)
    c2, b2 = ref.xi_book(bits)
    assert np.array_equal(c1.view(np.uint64), c2.view(np.uint64))
    assert np.array_equal(b1.view(np.uint64), b2.view(np.uint64))


@pytest.mark.parametrize("dim", [4, 16, 64, 128, 256])
@pytest.mark.parametrize("bits", [1, 2, 3, 4])
def test_rho_books_bit_identical_to_reference(orc, ref, dim, bits):
    c1, b1 = orc.rho_book(dim, bits)
    c2, b2 = ref.rho_book(dim, bits)
    assert np.array_equal(c1.view(np.uint64), c2.view(np.uint64))
    assert np.array_equal(b1.view(np.uint64), b2.view(np.uint64))


CONFIGS = [
    dict(b_dir=3, b_nrm=1, rounding="local3x3"),
    dict(b_dir=4, b_nrm=2, rounding="local3x3"),
    dict(b_dir=5, b_nrm=3, rounding="local3x3"),
    dict(b_dir=4, b_nrm=2, rounding="scalar"),
    dict(b_dir=3, b_nrm=1, rounding="scalar", qjl=True),
    dict(b_dir=4, b_nrm=2, rounding="local2x2", qjl=True),
    dict(b_dir=3, b_nrm=2, rounding="full"),
    dict(dim=64, b_dir=5, b_nrm=3, rounding="local3x3"),
    dict(dim=16, b_dir=2, b_nrm=4, rounding="local3x3", qjl=True),
    dict(dim=4, b_dir=2, b_nrm=2, rounding="full"),
    dict(dim=256, b_dir=4, b_nrm=2, rounding="local3x3", rotation_seed=7, qjl=True, qjl_seed=9),
]


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_codes_bit_identical_to_reference(orc, ref, cfg):
    dim = cfg.get("dim", 128)
    eo, er = orc.encoder(**cfg), ref.encoder(**cfg)
    x = orc.gaussian_f32(orc.L.orc_stream_child(0, 0), 2048 * dim).reshape(-1, dim)
    x[5] = 0.0  # zero key
    x[6] *= 1e-30  # tiny key
    a, b = eo.encode_f32(x), er.encode_f32(x)
    assert np.array_equal(a, b)
    da, db = eo.decode(a), er.decode(b)
    assert np.array_equal(da.view(np.uint64), db.view(np.uint64))


def test_attention_matches_reference(orc, ref):
    eo, er = orc.encoder(b_dir=4, b_nrm=2), ref.encoder(b_dir=4, b_nrm=2)
    x = orc.gaussian_f32(3, 300 * 128).reshape(-1, 128)
    recs = eo.encode_f32(x)
    vals = orc.gaussian_f32(4, 300 * 128).reshape(-1, 128).astype(np.float64)
    q = orc.gaussian_f32(5, 3 * 128).reshape(3, 128).astype(np.float64)
    ro = np.stack([eo.attention(qi, recs, vals, 3) for qi in q])
    rr = er.attention(q, recs, vals, 3)
    assert np.array_equal(ro.view(np.uint64), rr.view(np.uint64))


# ---- golden fixtures ---------------------------------------------------------------
def test_golden_fixtures(orc):
    path = os.path.join(GOLDEN, "codes.npz")
    if not os.path.exists(path):
        pytest.skip("run tests/golden/make_golden.py")
    z = np.load(path, allow_pickle=False)
    for name in z.files:
        if not name.startswith("rec_"):
            continue
        tag = name[4:]
        cfg = dict(zip(["dim", "b_dir", "b_nrm", "rounding", "qjl"], z["cfg_" + tag]))
        enc = orc.encoder(dim=int(cfg["dim"]), b_dir=int(cfg["b_dir"]), b_nrm=int(cfg["b_nrm"]),
                          rounding=int(cfg["rounding"]), qjl=bool(cfg["qjl"]))
        assert np.array_equal(enc.encode_f32(z["x_" + tag]), z[name]), tag
