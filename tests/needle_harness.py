"""run_needle's inputs (bench.hpp:446-501) restated for the needle tests
(test infrastructure: shared by test_needle_oracle.py and test_gpu_needle.py)."""
import ctypes as C

import numpy as np

MASTER = 0x0C70C0DE5EED  # kBenchMasterSeed, bench.hpp:31
D, N_DISTRACT, NOISE, N_SEEDS = 128, 2048, 0.10, 128


def _gauss(orc, seed, n):
    out = np.empty(n)
    orc.L.orc_fill_gaussian(seed, 0, out.ctypes.data_as(C.POINTER(C.c_double)), n)
    return out


def needle_case(orc, seed):
    """run_needle's per-seed inputs (bench.hpp:455-476), same fp64 order."""
    root = orc.L.orc_stream_child(MASTER, seed)
    n = N_DISTRACT + 1
    scale = np.sqrt(float(D))
    # sample_unit_sphere per row from one cursor: d = 128 is even, so row i
    # consumes Box-Muller pairs [64 i, 64 (i + 1)) of the stream
    g = _gauss(orc, orc.L.orc_stream_child(root, 0), n * D).reshape(n, D)
    s = np.cumsum(g * g, axis=1)[:, -1]  # sequential sums, as the reference
    keys = (g * (1.0 / np.sqrt(s))[:, None]) * scale
    noise = _gauss(orc, orc.L.orc_stream_child(root, 4), D)
    gn = np.sqrt(np.cumsum(noise * noise)[-1])
    needle = keys[0]
    kn = np.sqrt(np.cumsum(needle * needle)[-1])
    q = needle + NOISE * kn * noise / gn
    return keys, q, orc.L.orc_stream_child(root, 2), orc.L.orc_stream_child(root, 3)


def softmax_mass0(logits):
    m = logits.max()
    z = np.exp(logits - m).sum()
    return np.exp(logits[0] - m) / z


def fp32_mass(orc, seed):
    keys, q, _, _ = needle_case(orc, seed)
    return softmax_mass0(keys @ q / np.sqrt(float(D)))
