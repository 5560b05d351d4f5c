"""CPU model of K3's arithmetic (fp16 tensor-core operands, fp32 accumulation)
against the fp64 reference, to see which rounding dominates the attention
error at long contexts and what a change buys before spending GPU time.

  python tools/exp/k3_numerics.py [T] [bits] [dither] [qhilo]

Models, per stream of T tokens and its 7 query heads:
  K_hat, V_hat rows  = joint-table entries rho*n (fp64 exact, or fp16 as the
                       kernel's table, or fp16 dithered over R replicas: the
                       replica a (token, triplet) lookup reads varies with the
                       token, so each code's value averages to ~the exact one)
  q_rot * s          -> fp16 (optionally hi + lo: two fp16 MMA chains)
  scores (fp32), online softmax (fp32), P * gamma_v -> fp16, acc fp32.
Reference: fp64 everything (the oracle's attention_decode).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import Oracle  # noqa: E402


def unpack_codes(recs, b_dir, b_nrm, nt=43):
    """records [n, rb] -> gamma [n] f32, a, b, r [n, nt] (vectorised bit reads)."""
    n = recs.shape[0]
    gamma = recs[:, :4].copy().view(np.float32)[:, 0]
    bits = np.unpackbits(recs[:, 4:], axis=1, bitorder="little")
    db = (2 * nt * b_dir + 7) // 8

    def field(start, w, count):
        idx = start + np.arange(count)[:, None] * w + np.arange(w)[None, :]
        v = bits[:, idx]  # [n, count, w]
        return (v * (1 << np.arange(w))).sum(-1)
    d = field(0, b_dir, 2 * nt)
    r = field(8 * db, b_nrm, nt)
    return gamma, d[:, 0::2], d[:, 1::2], r


def f16(x):
    return x.astype(np.float16).astype(np.float64)


def dither_tables(exact, R, rng):
    """R replica tables of exact (any shape): each entry rounded down or up to
    fp16 so that the mean over the replicas is within ulp / (2R) of exact."""
    lo = exact.astype(np.float16)
    lo = np.where(lo.astype(np.float64) > exact, np.nextafter(lo, np.float16(-np.inf)), lo)
    hi = np.nextafter(lo, np.float16(np.inf))
    lo64, hi64 = lo.astype(np.float64), hi.astype(np.float64)
    span = np.where(hi64 > lo64, hi64 - lo64, 1.0)
    phi = np.clip((exact - lo64) / span, 0, 1)
    k = np.rint(phi * R)
    order = np.array([int(format(i, f"0{R.bit_length() - 1}b")[::-1], 2) for i in range(R)])
    reps = np.stack([np.where(order[i] < k, hi64, lo64) for i in range(R)])
    return reps  # [R, ...]


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    bits = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dither = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    qhilo = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    qscale = float(os.environ.get("QSCALE", "1"))
    b_dir, b_nrm = bits + 1, bits - 1
    orc = Oracle()
    rng = np.random.default_rng(1)
    ek = orc.encoder(b_dir=b_dir, b_nrm=b_nrm, rotation_seed=11)
    ev = orc.encoder(b_dir=b_dir, b_nrm=b_nrm, rotation_seed=13)
    K = rng.standard_normal((T, 128)).astype(np.float32)
    V = rng.standard_normal((T, 128)).astype(np.float32)
    Q = (rng.standard_normal((7, 128)) * qscale).astype(np.float32)
    kr, vr = ek.encode_f32(K), ev.encode_f32(V)
    vdec = ev.decode(vr)
    ref = np.stack([ek.attention(q.astype(np.float64), kr, vdec) for q in Q])

    # joint table (rotated frame, unit scale): rho_c[r] * oct_decode(xi_a, xi_b)
    xi_c, _ = orc.xi_book(b_dir)
    rho_c, _ = orc.rho_book(128, b_nrm)
    import ctypes as C
    Kd = 1 << b_dir
    dirs = np.zeros((Kd, Kd, 3))
    for a in range(Kd):
        for b in range(Kd):
            o = np.zeros(3)
            orc.L.orc_oct_decode(xi_c[a], xi_c[b], o.ctypes.data_as(C.POINTER(C.c_double)))
            dirs[a, b] = o
    tab = rho_c[:, None, None, None] * dirs[None]  # [KR, K, K, 3]

    def rows(recs, table_fn):
        g, a, b, r = unpack_codes(recs, b_dir, b_nrm)
        u = table_fn(r, a, b)  # [n, 43, 3]
        return g.astype(np.float64), u.reshape(len(g), -1)[:, :128]

    def signs(seed):
        s = np.empty(128)
        orc.L.orc_rotation_signs(128, seed, s.ctypes.data_as(C.POINTER(C.c_double)))
        return s

    def rot(x, s):  # R x: signs then normalized WHT
        y = x * s
        h = 1
        y = y.copy()
        while h < 128:
            y = y.reshape(-1, 2 * h)
            a, b = y[:, :h].copy(), y[:, h:].copy()
            y[:, :h], y[:, h:] = a + b, a - b
            h *= 2
        return y.reshape(-1) / np.sqrt(128.0)

    sk, sv = signs(11), signs(13)
    if os.environ.get("W13"):  # direction table dithered, rho applied in fp16 in-kernel
        reps_n = dither_tables(dirs, dither or 16, rng)  # [R, K, K, 3]
        rho16 = f16(rho_c)
        pick_k = rng.integers(0, dither or 16, size=(T, 43))
        pick_v = rng.integers(0, dither or 16, size=(T, 43))

        reps_r = dither_tables(rho_c, dither or 16, rng)  # [R, KR]
        if os.environ.get("W13") == "2":  # rho dithered too (per-lane register tables)
            def tf(pick):
                return lambda r, a, b: f16(reps_r[pick, r][..., None] * reps_n[pick, a, b])
        else:
            def tf(pick):
                return lambda r, a, b: f16(rho16[r][..., None] * reps_n[pick, a, b])
        kfn, vfn = tf(pick_k), tf(pick_v)
    elif dither < 0:  # model check: everything exact
        kfn = vfn = lambda r, a, b: tab[r, a, b]
    elif dither:
        reps = dither_tables(tab, dither, rng)  # [R, KR, K, K, 3]
        pick_k = rng.integers(0, dither, size=(T, 43))
        pick_v = rng.integers(0, dither, size=(T, 43))

        def tf(pick):
            return lambda r, a, b: reps[pick, r, a, b]
        kfn, vfn = tf(pick_k), tf(pick_v)
    else:
        kfn = vfn = lambda r, a, b: f16(tab[r, a, b])
    exact_fn = lambda r, a, b: tab[r, a, b]  # noqa: E731
    if os.environ.get("KRN"):  # K side through a round-to-nearest table, V dithered
        kfn = lambda r, a, b: f16(tab[r, a, b])  # noqa: E731
    gk, Kh = rows(kr, exact_fn if os.environ.get("KEXACT") else kfn)
    gv, Vh = rows(vr, exact_fn if os.environ.get("VEXACT") else vfn)
    out = np.zeros((7, 128))
    log2e = 1.4426950408889634
    for h in range(7):
        qr = rot(Q[h].astype(np.float64), sk) * (log2e / np.sqrt(128.0))  # q_rot / sqrt(d) * log2e
        qhi = qr if (dither < 0 or os.environ.get("QEXACT")) else f16(qr)
        s = (Kh @ qhi) * gk
        if qhilo:
            s = s + (Kh @ f16(qr - qhi)) * gk
        s = s.astype(np.float32).astype(np.float64)
        m = s.max()
        p = np.exp2(s - m)
        l = p.sum()
        pv = p * gv if (dither < 0 or os.environ.get("PEXACT")) else f16(p * gv)
        acc = pv @ Vh  # rotated frame
        o = acc / l
        # inverse V rotation: WHT then signs
        out[h] = rot(o, np.ones(128)) * sv
    e = np.linalg.norm(out - ref, axis=1) / np.linalg.norm(ref, axis=1)
    print(f"T={T} bits={bits} dither={dither} qhilo={qhilo} qscale={qscale}: "
          f"rel err max {e.max():.2e} mean {e.mean():.2e}")


if __name__ == "__main__":
    main()
