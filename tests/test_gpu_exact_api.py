"""The per-key reference API in exact fp64 on the GPU (exact_api.cu), compared
BIT FOR BIT with the reference: Encoder::prepare, reconstruct_rotated, decode,
score (+ qjl_estimate) and attention_decode (to a few ulp: device exp).

Oracle: the reference itself (oracle/_ref) for decode / score / attention, the
C restatement (oracle/) for the rotation and the direction table."""
import ctypes as C

import numpy as np
import pytest

import paper_2605_21226_b200 as oq

pytestmark = pytest.mark.gpu

CONFIGS = [dict(b_dir=3, b_nrm=1), dict(b_dir=4, b_nrm=2), dict(b_dir=5, b_nrm=3, qjl=True),
           dict(b_dir=3, b_nrm=1, qjl=True, dim=64), dict(b_dir=8, b_nrm=4, dim=256),
           dict(b_dir=2, b_nrm=2, dim=4)]


def _rotate(orc, x, dim, seed):
    """Rotation(dim, seed).apply (rotation.hpp:46-50) with the oracle's fwht."""
    s = np.empty(dim)
    orc.L.orc_rotation_signs(dim, seed, s.ctypes.data_as(C.POINTER(C.c_double)))
    y = np.ascontiguousarray(x * s)
    orc.L.orc_fwht(y.ctypes.data_as(C.POINTER(C.c_double)), dim)
    return y


@pytest.mark.parametrize("kw", CONFIGS)
def test_exact_api_bit_identical(orc, ref, cuda, kw):
    import torch
    dim = kw.get("dim", 128)
    kw = dict(kw, rotation_seed=7, qjl_seed=9)
    enc = oq.Encoder(oq.CodecConfig(**kw))
    rng = np.random.default_rng(3)
    keys = rng.standard_normal((300, dim)).astype(np.float32)
    qs = rng.standard_normal((5, dim))
    recs = enc.compress(torch.from_numpy(keys).to(cuda))
    rn = recs.cpu().numpy()
    rk = ref.encoder(dim=dim, b_dir=kw["b_dir"], b_nrm=kw["b_nrm"], rotation_seed=7,
                     qjl=kw.get("qjl", False), qjl_seed=9)
    # decode: Encoder::decode, bit for bit
    dec = enc.decode_exact(recs).cpu().numpy()
    assert np.array_equal(dec.view(np.uint64), rk.decode(rn).view(np.uint64))
    # prepare: R q (and R' R q), bit for bit
    rot, sk = enc.prepare(torch.from_numpy(qs).to(cuda))
    rot_n = rot.cpu().numpy()
    for i, q in enumerate(qs):
        r = _rotate(orc, q, dim, 7)
        assert np.array_equal(rot_n[i].view(np.uint64), r.view(np.uint64))
        if kw.get("qjl"):
            assert np.array_equal(sk.cpu().numpy()[i].view(np.uint64),
                                  _rotate(orc, r, dim, 9).view(np.uint64))
    # score(prepare(q), k), bit for bit
    sc = enc.score_prepared(rot, sk, recs).cpu().numpy()
    for i, q in enumerate(qs):
        for j in range(0, 300, 7):
            assert sc[i, j] == rk.score(q, rn[j]), (i, j)
    # reconstruct_rotated: decode == gamma * R^-1 (reconstruct), via score identity
    ur = enc.reconstruct_rotated(recs).cpu().numpy()
    gam = rn[:, :4].copy().view(np.float32)[:, 0].astype(np.float64)
    if not kw.get("qjl"):
        assert np.allclose(sc, (rot_n @ ur.T) * gam[None, :], rtol=1e-12, atol=1e-12)
    # attention_decode (fp64, device exp): few-ulp agreement with the reference
    vals = rng.standard_normal((300, 16))
    got = enc.attention_exact(torch.from_numpy(qs).to(cuda), recs,
                              torch.from_numpy(vals).to(cuda), n_splits=3).cpu().numpy()
    want = rk.attention(qs, rn, vals, 3)
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.abs(want).max())
