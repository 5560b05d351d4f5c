"""Needle retrieval through the GPU attention path.

The reference's only end-to-end quality gate on attention is run_needle
(bench.hpp:446-501), pinned by acceptance_test.cpp:219-228: per seed, 2048
distractors plus one planted key on the sqrt(d) shell (sample_unit_sphere,
marginals.hpp:66-73, from Stream(kBenchMasterSeed).child(seed).child(0)), a
query = needle + 10 % Gaussian noise (child(4)), the codec bound to the
seed's rotation / QJL seeds (child(2) / child(3)), and the softmax mass the
planted key keeps.  Pins: fp32 0.960 +- 0.01, octo b=2 0.92 +- 0.02,
octo_qjl b=3/4 within 0.01 of fp32 (means over 128 seeds).

Here the keys are compressed by K1 on the GPU and the mass is read out of the
GPU attention: V holds one Gaussian row for the needle and zero rows for the
distractors (a zero vector encodes to gamma = 0 and decodes exactly to 0), so
out = p_0 * v_hat_0 and mass = out . v_hat_0 / |v_hat_0|^2.  All three run
the compressed-V tile kernel (K3): b = 2 (W = 7), b = 3 + QJL (W = 10), b = 4
+ QJL (W = 13).  Each
seed's GPU mass is also compared with the mass computed from the oracle's
fp64 Encoder::score on the same codes.
"""
import numpy as np
import pytest

import paper_2605_21226_b200 as oq
from needle_harness import D, N_SEEDS, _gauss, fp32_mass, needle_case, softmax_mass0

pytestmark = pytest.mark.gpu


def gpu_mass(orc, cuda, seed, bits, qjl):
    import torch
    keys, q, rot, qs = needle_case(orc, seed)
    bd, bn = oq.default_bit_split(bits)
    ck = oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=rot, qjl=qjl, qjl_seed=qs)
    ek = oq.Encoder(ck)
    kr = ek.compress(torch.from_numpy(keys).to(cuda))  # fp64 keys, as the harness feeds them
    n = keys.shape[0]
    # attention_decode scales by 1/sqrt(dim): softmax(score / sqrt(d)) == run_needle's logits
    if ek.tile_bytes(0):
        ev = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=(rot + 1) & 0xFFFFFFFFFFFFFFFF))
        v = torch.zeros((n, D), dtype=torch.float64, device=cuda)
        v[0] = torch.from_numpy(_gauss(orc, orc.L.orc_stream_child(rot, 9), D)).to(cuda)
        vr = ev.compress(v)
        vhat0 = ev.decode(vr[:1]).double()[0]
        cache = oq.KVCache(ek, ev, 1, 1, n)
        cache.pack(kr, vr, n)
        out = oq.attention_decode(torch.from_numpy(q).float().reshape(1, 1, D).to(cuda), cache)
        mass = float((out.double()[0, 0] @ vhat0) / (vhat0 @ vhat0))
        path = "tile"
    else:
        vals = torch.zeros((n, 1), dtype=torch.float32, device=cuda)
        vals[0, 0] = 1.0
        out = oq.attention_decode_dense(ek, torch.from_numpy(q).float().reshape(1, D).to(cuda),
                                        kr, vals)
        mass = float(out[0, 0])
        path = "dense"
    # the oracle's fp64 scores on the same (bit-exact) codes
    ok = orc.encoder(b_dir=bd, b_nrm=bn, rotation_seed=rot, qjl=qjl, qjl_seed=qs)
    krn = kr.cpu().numpy()
    assert np.array_equal(krn[:64], np.stack([ok.encode_f64(k) for k in keys[:64]]))
    qf = q.astype(np.float32).astype(np.float64)
    logits = np.array([ok.score(qf, r) for r in krn]) / np.sqrt(float(D))
    return mass, softmax_mass0(logits), path


def fp32_mass(orc, seed):
    keys, q, _, _ = needle_case(orc, seed)
    return softmax_mass0(keys @ q / np.sqrt(float(D)))


@pytest.fixture(scope="module")
def fp32_ref(orc):
    return float(np.mean([fp32_mass(orc, s) for s in range(N_SEEDS)]))


@pytest.mark.parametrize("bits,qjl,target", [(2, False, "octo b=2: 0.92 +- 0.02"),
                                             (3, True, "octo_qjl b=3: fp32 +- 0.01"),
                                             (4, True, "octo_qjl b=4: fp32 +- 0.01")])
def test_needle_mass_gpu(orc, cuda, fp32_ref, bits, qjl, target):
    res = [gpu_mass(orc, cuda, s, bits, qjl) for s in range(N_SEEDS)]
    g = np.array([r[0] for r in res])
    o = np.array([r[1] for r in res])
    # per seed: the GPU attention's mass vs the oracle's fp64 scores on the same codes
    assert np.max(np.abs(g - o)) <= 5e-3, (np.max(np.abs(g - o)), res[0][2])
    mean = float(g.mean())
    if qjl:
        assert abs(mean - fp32_ref) <= 0.01, (mean, fp32_ref, target)
    else:
        assert abs(mean - 0.92) <= 0.02, (mean, target)
