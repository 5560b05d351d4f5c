"""CPU tests of the product's host side (no GPU needed):

* the C-ABI library loads and exports every symbol include/octoquant_b200.h
  declares;
* host codebook construction (books.cpp) is bit-identical to the reference
  registry books (oracle/_ref) and to the oracle;
* config / rate / wire-header logic matches the reference's semantics and
  error types (codec_test.cpp:40-63, 412-547);
* with no GPU the device entry points fail loudly (no CPU fallback).
"""
import os
import re

import numpy as np
import pytest

import paper_2605_21226_b200 as oq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "octoquant_b200.h")).read()
    names = set(re.findall(r"\b(oq_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) > 20
    L = oq.lib()
    for n in sorted(names):
        assert hasattr(L, n), n


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 5, 6, 7, 8])
def test_product_xi_books_bit_identical(orc, bits):
    c, b = oq.xi_book(bits)
    co, bo = orc.xi_book(bits)
    assert np.array_equal(c.view(np.uint64), co.view(np.uint64))
    assert np.array_equal(b.view(np.uint64), bo.view(np.uint64))


# b_nrm in [1, 4] at every dim, up to 6 at d = 128 (density training at 7-8
# bits takes ~20 s per book on this host and is exercised only on demand).
@pytest.mark.parametrize("dim,bits", [(d, b) for d in (4, 8, 16, 32, 64, 128, 256)
                                      for b in (1, 2, 3, 4)] + [(128, 5), (128, 6)])
def test_product_rho_books_bit_identical(orc, dim, bits):
    c, b = oq.rho_book(dim, bits)
    co, bo = orc.rho_book(dim, bits)
    assert np.array_equal(c.view(np.uint64), co.view(np.uint64))
    assert np.array_equal(b.view(np.uint64), bo.view(np.uint64))


@pytest.mark.parametrize("bits", [2, 3, 4, 5])
def test_product_books_match_reference_itself(ref, bits):
    c, b = oq.xi_book(bits)
    cr, br = ref.xi_book(bits)
    assert np.array_equal(c.view(np.uint64), cr.view(np.uint64))
    c, b = oq.rho_book(128, bits - 1)
    cr, br = ref.rho_book(128, bits - 1)
    assert np.array_equal(c.view(np.uint64), cr.view(np.uint64))


def test_config_validation():
    # codec_test.cpp:40-56
    with pytest.raises(ValueError):
        oq.CodecConfig(dim=96).validate()
    with pytest.raises(ValueError):
        oq.CodecConfig(dim=2).validate()
    with pytest.raises(ValueError):
        oq.CodecConfig(b_dir=9).validate()
    with pytest.raises(ValueError):
        oq.CodecConfig(qjl=True, qjl_seed=0).validate()
    oq.CodecConfig(qjl=True, qjl_seed=1).validate()
    with pytest.raises(ValueError):
        oq.parse_rounding("nearest")
    assert oq.parse_rounding("local2x2") == "local2x2"


def test_default_bit_split():
    # codec_test.cpp:58-63
    assert oq.default_bit_split(2) == (3, 1)
    assert oq.default_bit_split(3) == (4, 2)
    assert oq.default_bit_split(4) == (5, 3)
    with pytest.raises(ValueError):
        oq.default_bit_split(1)


def test_effective_bits():
    # codec_test.cpp:535-547
    assert oq.effective_bits_per_coord(oq.CodecConfig()) == 333.0 / 128.0
    assert oq.effective_bits_per_coord(oq.CodecConfig(qjl=True)) - \
        oq.effective_bits_per_coord(oq.CodecConfig()) == 1.125
    assert oq.effective_bits_per_coord(oq.CodecConfig(dim=64, b_dir=5, b_nrm=3)) == 318.0 / 64.0


def test_record_sizes():
    assert oq.record_bytes(oq.CodecConfig()) == 43
    assert oq.record_bytes(oq.CodecConfig.for_bits(3)) == 58
    assert oq.record_bytes(oq.CodecConfig.for_bits(4)) == 75
    assert oq.record_bytes(oq.CodecConfig(qjl=True)) == 61


def test_wire_header_and_rejections(orc):
    # codec_test.cpp:412-421 (20 + 43 bytes), 519-533 (header mismatch)
    cfg = oq.CodecConfig()
    recs = np.zeros((1, 43), np.uint8)
    blob = oq.pack_keys(cfg, recs)
    assert len(blob) == 20 + 43
    assert blob[:4] == b"OCTO" and blob[4] == 1 and blob[5] == 0 and blob[6] == 3
    from oracle_bind import make_config
    import ctypes as C
    hdr = (C.c_uint8 * 20)()
    orc.L.orc_wire_header(C.byref(make_config()), 1, hdr)
    assert bytes(hdr) == blob[:20]
    bad = b"X" + blob[1:]
    with pytest.raises(oq.FormatError):
        oq.unpack_keys(bad)
    with pytest.raises(oq.FormatError):
        oq.unpack_keys(blob[:-1])
    with pytest.raises(oq.FormatError):
        oq.unpack_keys(blob[:4] + b"\x02" + blob[5:])
    with pytest.raises(oq.FormatError):
        oq.unpack_keys(blob[:5] + b"\x02" + blob[6:])


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        oq.Encoder(oq.CodecConfig())


def test_dir_table_matches_oracle(orc):
    import ctypes as C

    # host-only entry point (no device): codec.hpp:100-107
    xi, _ = oq.xi_book(4)
    out = np.empty(16 * 16 * 3)
    dp = C.POINTER(C.c_double)
    oq._check(oq.lib().oq_dir_table(xi.ctypes.data_as(dp), 16, out.ctypes.data_as(dp)))
    for a in range(16):
        for b in range(16):
            o = np.empty(3)
            orc.L.orc_oct_decode(xi[a], xi[b], o.ctypes.data_as(dp))
            assert np.array_equal(out[3 * (16 * a + b):3 * (16 * a + b) + 3], o)
