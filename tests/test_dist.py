"""World-size-2 gloo tests of the sequence-sharded mode's host logic on CPU.

Each rank computes the SoftmaxState of its own token range with the CPU
oracle (the stand-in for the GPU kernel), the partials meet in ONE
all-gather (paper_2605_21226_b200.sharded), and the rank-ordered merge must
reproduce attention_decode over the whole cache — on both ranks, identically.
"""
import math
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _merge_np(g):
    """SoftmaxState::merge (attention.hpp:36-44) over parts in order, natural-log m."""
    parts, rows, W = g.shape
    out = np.zeros((rows, W - 4))
    for r in range(rows):
        M, L, acc = -math.inf, 0.0, np.zeros(W - 4)
        for p in range(parts):
            m, l, a = g[p, r, 0], g[p, r, 1], g[p, r, 4:]
            if l == 0.0:
                continue
            mn = max(M, m)
            sa, sb = math.exp(M - mn) if M > -math.inf else 0.0, math.exp(m - mn)
            L = L * sa + l * sb
            acc = acc * sa + a * sb
            M = mn
        out[r] = acc / L
    return out


def _worker(rank, world, port, T, result_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    from oracle_bind import Oracle
    from paper_2605_21226_b200.sharded import shard_bounds, sharded_decode

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    orc = Oracle()
    enc = orc.encoder(b_dir=4, b_nrm=2)
    k = orc.gaussian_f32(orc.L.orc_stream_child(9, 0), T * 128).reshape(T, 128)
    vals = orc.gaussian_f32(orc.L.orc_stream_child(9, 1), T * 16).reshape(T, 16).astype(
        np.float64)
    qs = orc.gaussian_f32(orc.L.orc_stream_child(9, 2), 3 * 128).reshape(3, 128).astype(
        np.float64)
    recs = enc.encode_f32(k)
    t0, t1 = shard_bounds(T, world, rank)
    part = np.zeros((3, 4 + 16))
    for i, q in enumerate(qs):
        m, l, acc = enc.partial(q, recs, t0, t1, vals)
        part[i, 0], part[i, 1], part[i, 4:] = m, l, acc
    out = sharded_decode(torch.from_numpy(part), lambda g: _merge_np(g.numpy()))
    full = np.stack([enc.attention(q, recs, vals, world) for q in qs])
    result_q.put((rank, np.abs(out - full).max(), out))
    dist.destroy_process_group()


@pytest.mark.parametrize("T", [257, 5, 2])
def test_sharded_merge_matches_full_attention(T):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, T, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    for _, err, _ in res:
        assert err <= 1e-12
    assert np.array_equal(res[0][2], res[1][2])  # identical on every rank


def test_shard_bounds_cover_every_token_once():
    from paper_2605_21226_b200.sharded import shard_bounds
    for T in (0, 1, 7, 128, 1 << 20):
        for P in (1, 2, 3, 4, 8):
            seen = []
            for r in range(P):
                t0, t1 = shard_bounds(T, P, r)
                seen.extend(range(t0, t1)) if T < 5000 else seen.append((t0, t1))
            if T < 5000:
                assert seen == list(range(T))
            else:
                assert seen[0][0] == 0 and seen[-1][1] == T
                assert all(a[1] == b[0] for a, b in zip(seen, seen[1:]))
