"""Quality parity through the reference's own acceptance gates.

The reference's synthetic Table-1 harness (bench.hpp:282-425) draws, per
seed, keys/queries from Stream(kBenchMasterSeed).child(seed) (seed_scope,
bench.hpp:358-365) and scores a BoundCodec bound to that seed's rotation /
sketch seeds.  Here the codes come from the GPU (K1 via the C ABI, fp64 keys
exactly as the harness feeds them), and:

* test_golden_csv_row: the octo row of the reference's only golden file
  (tests/data/table1_small.csv:2, produced by `bench table1 --keys 64
  --queries 4 --seeds 2 --codecs octo,tq_mse --bits 2`, cli_test.cpp:109-122)
  is reproduced byte for byte when the metric suite runs on the GPU codes with
  the reference's fp64 decode/score (the oracle, as the checker), and to 2e-5
  with the GPU's own fp32 decode (K2) and scores;
* test_acceptance_pins: the frozen Table-1 targets of acceptance_test.cpp:89-140
  (1024 keys, 16 queries, 64 seeds, scalar rounding): octo cos/MSE within
  0.003 and octo / octo_qjl inner-product error within 5 %, all from GPU
  compress + GPU decode + GPU scores.
"""
import ctypes as C
import math

import numpy as np
import pytest

import paper_2605_21226_b200 as oq

pytestmark = pytest.mark.gpu

MASTER = 0x0C70C0DE5EED  # kBenchMasterSeed, bench.hpp:31
# tests/data/table1_small.csv:2 (octo row)
GOLDEN_OCTO = "octo,2,3,1,scalar,2,0.954339,0.000360999,0.0912274,0.000872784,2.61475,0.127175"


def _gaussian(orc, seed, n):
    out = np.empty(n)
    orc.L.orc_fill_gaussian(seed, 0, out.ctypes.data_as(C.POINTER(C.c_double)), n)
    return out


def seed_scope(orc, seed, n_keys, n_queries, dim=128):
    """detail::seed_scope (bench.hpp:358-365)."""
    root = orc.L.orc_stream_child(MASTER, seed)
    keys = _gaussian(orc, orc.L.orc_stream_child(root, 0), n_keys * dim).reshape(n_keys, dim)
    qs = _gaussian(orc, orc.L.orc_stream_child(root, 1), n_queries * dim).reshape(n_queries, dim)
    return keys, qs, orc.L.orc_stream_child(root, 2), orc.L.orc_stream_child(root, 3)


def pairwise_sum(xs):
    """bench.hpp:33-40, same association order."""
    if len(xs) <= 8:
        s = 0.0
        for x in xs:
            s += x
        return s
    h = len(xs) // 2
    return pairwise_sum(xs[:h]) + pairwise_sum(xs[h:])


def mean_se(xs):
    """bench.hpp:47-58."""
    n = len(xs)
    m = pairwise_sum(xs) / n
    if n < 2:
        return m, 0.0
    sq = [(x - m) * (x - m) for x in xs]
    return m, math.sqrt(pairwise_sum(sq) / (n - 1) / n)


def metric_suite(keys, queries, khat, score):
    """metric_suite (bench.hpp:282-327): sequential fp64 sums per key."""
    cos_t, mse_t = [], []
    d = keys.shape[1]
    for i in range(keys.shape[0]):
        k, kh = keys[i].tolist(), khat[i].tolist()
        dot = nk = nh = err = 0.0
        for j in range(d):
            dot += k[j] * kh[j]
            nk += k[j] * k[j]
            nh += kh[j] * kh[j]
            e = k[j] - kh[j]
            err += e * e
        cos_t.append(dot / math.sqrt(nk * nh) if nk > 0.0 and nh > 0.0 else 1.0)
        mse_t.append(err / d)
    ip_t = []
    for qi in range(queries.shape[0]):
        q = queries[qi].tolist()
        for ki in range(keys.shape[0]):
            k = keys[ki].tolist()
            exact = 0.0
            for j in range(d):
                exact += q[j] * k[j]
            ip_t.append(abs(exact - score(qi, ki)))
    n = keys.shape[0]
    return pairwise_sum(cos_t) / n, pairwise_sum(mse_t) / n, pairwise_sum(ip_t) / len(ip_t)


def g6(v):
    return "%.6g" % v  # detail::g6, bench.hpp:718-722


def gpu_codec(bits, rot, qjl_seed, rounding="scalar", qjl=False):
    bd, bn = oq.default_bit_split(bits)
    return oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rounding=rounding, rotation_seed=rot,
                                     qjl=qjl, qjl_seed=qjl_seed))


def test_golden_csv_row(orc, cuda):
    import torch
    ref_rows, gpu_rows = [], []
    for seed in range(2):
        keys, qs, rot, qjs = seed_scope(orc, seed, 64, 4)
        enc = gpu_codec(2, rot, qjs)
        recs = enc.compress(torch.from_numpy(keys).to(cuda))  # fp64 keys, as the harness
        rn = recs.cpu().numpy()
        ok = orc.encoder(b_dir=3, b_nrm=1, rounding="scalar", rotation_seed=rot, qjl_seed=qjs)
        assert np.array_equal(rn, np.stack([ok.encode_f64(k) for k in keys])), "codes differ"
        # the reference's fp64 decode / score on the GPU codes
        ref_rows.append(metric_suite(keys, qs, ok.decode(rn), lambda qi, ki: ok.score(qs[qi], rn[ki])))
        # the GPU's own decode (K2) and scores
        kh = enc.decode(recs).double().cpu().numpy()
        sc = enc.scores(torch.from_numpy(qs).float().to(cuda), recs).double().cpu().numpy()
        gpu_rows.append(metric_suite(keys, qs, kh, lambda qi, ki: float(sc[qi, ki])))
    cols = list(zip(*ref_rows))
    stats = [mean_se(list(c)) for c in cols]
    line = ",".join(["octo", "2", "3", "1", "scalar", "2"] +
                    [g6(v) for m_se in stats for v in m_se])
    assert line == GOLDEN_OCTO
    golden = [float(x) for x in GOLDEN_OCTO.split(",")[6:]]
    gstats = [v for c in zip(*gpu_rows) for v in mean_se(list(c))]
    for got, want, name in zip(gstats[0::2], golden[0::2], ["cosine", "mse", "ip_abs_err"]):
        assert abs(got - want) <= 2e-5 * abs(want) + 1e-6, (name, got, want)


def test_acceptance_pins(orc, cuda):
    import torch
    seeds, n_keys, n_q = 64, 1024, 16
    pins = {2: (0.9547, 0.0897, 2.682, 2.015), 3: (0.9871, 0.0260, 1.444, 1.084),
            4: (0.9965, 0.0071, 0.753, 0.565)}
    acc = {b: [[], [], [], []] for b in pins}
    for seed in range(seeds):
        keys, qs, rot, qjs = seed_scope(orc, seed, n_keys, n_q)
        kt = torch.from_numpy(keys).to(cuda)
        qt = torch.from_numpy(qs).float().to(cuda)
        exact = qs @ keys.T
        nk = np.einsum("ij,ij->i", keys, keys)
        for b in pins:
            for qjl in (False, True):
                enc = gpu_codec(b, rot, qjs, qjl=qjl)
                recs = enc.compress(kt)
                sc = enc.scores(qt, recs).double().cpu().numpy()
                acc[b][3 if qjl else 2].append(np.abs(exact - sc).mean())
                if qjl:
                    continue  # the sidecar changes scoring only (acceptance_test.cpp:117-121)
                kh = enc.decode(recs).double().cpu().numpy()
                nh = np.einsum("ij,ij->i", kh, kh)
                cos = np.einsum("ij,ij->i", keys, kh) / np.sqrt(nk * nh)
                acc[b][0].append(cos.mean())
                acc[b][1].append(((keys - kh) ** 2).mean(axis=1).mean())
    for b, (c, m, ip, ipq) in pins.items():
        got = [float(np.mean(v)) for v in acc[b]]
        assert abs(got[0] - c) <= 0.003, (b, "cosine", got[0], c)
        assert abs(got[1] - m) <= 0.003, (b, "mse", got[1], m)
        assert abs(got[2] - ip) <= 0.05 * ip, (b, "ip octo", got[2], ip)
        assert abs(got[3] - ipq) <= 0.05 * ipq, (b, "ip octo_qjl", got[3], ipq)
