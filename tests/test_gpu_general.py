"""GPU parity of the general path (any codec configuration, OCTO records):
Encoder::score and attention_decode with dense values, as the reference's
own API takes them (attention.hpp:50-73).  fp32 arithmetic: tolerances
1e-5 relative (scores vs |q||k_hat|, outputs vs ||ref||).
"""
import math

import numpy as np
import pytest

import paper_2605_21226_b200 as oq

pytestmark = pytest.mark.gpu

CONFIGS = [
    dict(b_dir=3, b_nrm=1),
    dict(b_dir=4, b_nrm=2),
    dict(b_dir=5, b_nrm=3),
    dict(b_dir=3, b_nrm=1, qjl=True),
    dict(b_dir=6, b_nrm=4, rounding="scalar"),
    dict(dim=64, b_dir=5, b_nrm=3),
    dict(dim=16, b_dir=3, b_nrm=2, qjl=True),
    dict(dim=4, b_dir=2, b_nrm=2, rounding="full"),
    dict(dim=256, b_dir=4, b_nrm=2),
]


def _ids(c):
    return "-".join(f"{k}{v}" for k, v in c.items())


def _setup(orc, cuda, cfg, n, nq, vdim, seed):
    import torch
    dim = cfg.get("dim", 128)
    eo = orc.encoder(**cfg)
    enc = oq.Encoder(oq.CodecConfig(**cfg))
    k = orc.gaussian_f32(orc.L.orc_stream_child(seed, 0), n * dim).reshape(n, dim)
    q = orc.gaussian_f32(orc.L.orc_stream_child(seed, 1), nq * dim).reshape(nq, dim)
    v = orc.gaussian_f32(orc.L.orc_stream_child(seed, 2), n * vdim).reshape(n, vdim)
    recs = enc.compress(torch.from_numpy(k).to(cuda))
    assert np.array_equal(recs.cpu().numpy(), eo.encode_f32(k))
    return eo, enc, recs, q, v


@pytest.mark.parametrize("cfg", CONFIGS, ids=_ids)
def test_scores_match_reference(orc, cuda, cfg):
    # codec_test.cpp:239-262: score == q . decode(k) (here vs the fp64 oracle)
    import torch
    eo, enc, recs, q, _ = _setup(orc, cuda, cfg, 300, 5, 1, 41)
    got = enc.scores(torch.from_numpy(q).to(cuda), recs).cpu().numpy()
    rn = recs.cpu().numpy()
    dec = eo.decode(rn)
    for i in range(q.shape[0]):
        ref = np.array([eo.score(q[i].astype(np.float64), r) for r in rn])
        scale = np.linalg.norm(q[i]) * np.maximum(np.linalg.norm(dec, axis=1), 1e-30)
        assert np.max(np.abs(got[i] - ref) / scale) <= 2e-6


@pytest.mark.parametrize("cfg", CONFIGS, ids=_ids)
@pytest.mark.parametrize("n_splits", [1, 7])
def test_dense_attention_matches_reference(orc, cuda, cfg, n_splits):
    import torch
    eo, enc, recs, q, v = _setup(orc, cuda, cfg, 777, 3, 48, 43)
    got = oq.attention_decode_dense(enc, torch.from_numpy(q).to(cuda), recs,
                                    torch.from_numpy(v).to(cuda), n_splits).cpu().numpy()
    rn = recs.cpu().numpy()
    for i in range(q.shape[0]):
        ref = eo.attention(q[i].astype(np.float64), rn, v.astype(np.float64), n_splits)
        assert np.linalg.norm(got[i] - ref) / np.linalg.norm(ref) <= 1e-5


def test_dense_single_key_and_errors(orc, cuda):
    import torch
    eo, enc, recs, q, v = _setup(orc, cuda, dict(b_dir=4, b_nrm=2), 1, 1, 8, 44)
    out = oq.attention_decode_dense(enc, torch.from_numpy(q).to(cuda), recs,
                                    torch.from_numpy(v).to(cuda)).cpu().numpy()
    assert np.allclose(out[0], v[0], rtol=1e-6, atol=1e-7)  # codec_test.cpp:338-351
    with pytest.raises(ValueError):  # empty cache (codec_test.cpp:353-361)
        oq.attention_decode_dense(enc, torch.from_numpy(q).to(cuda), recs[:0],
                                  torch.from_numpy(v[:0]).to(cuda))
    with pytest.raises(ValueError):
        oq.attention_decode_dense(enc, torch.from_numpy(q).to(cuda), recs,
                                  torch.from_numpy(v).to(cuda), n_splits=0)
