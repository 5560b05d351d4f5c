"""Generate tests/golden/codes.npz from the REFERENCE itself (oracle/_ref).

Inputs are Gaussian fp32 keys from the reference's Stream(seed).child(i)
(rng.hpp:26-28, 59-63); outputs are the reference's pack_keys records
(codec.hpp:364-396).  Run here (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bind import ROUNDING, Oracle, RefLib  # noqa: E402

CASES = {
    # tag: (dim, b_dir, b_nrm, rounding, qjl, n)
    "c1_b3_local3x3": (128, 4, 2, "local3x3", 0, 64),
    "c1_b3_scalar": (128, 4, 2, "scalar", 0, 64),
    "b2_local3x3": (128, 3, 1, "local3x3", 0, 64),
    "b4_local3x3": (128, 5, 3, "local3x3", 0, 64),
    "b2_qjl": (128, 3, 1, "local3x3", 1, 64),
    "d64_b4": (64, 5, 3, "local3x3", 0, 32),
    "d4_full": (4, 2, 2, "full", 0, 32),
}


def main():
    orc, ref = Oracle(), RefLib()
    out = {}
    for i, (tag, (dim, bd, bn, rnd, qjl, n)) in enumerate(CASES.items()):
        seed = orc.L.orc_stream_child(0, i)
        x = orc.gaussian_f32(seed, n * dim).reshape(n, dim)
        enc = ref.encoder(dim=dim, b_dir=bd, b_nrm=bn, rounding=rnd, qjl=bool(qjl))
        out["x_" + tag] = x
        out["rec_" + tag] = enc.encode_f32(x)
        out["cfg_" + tag] = np.array([dim, bd, bn, ROUNDING[rnd], qjl], np.int64)
    np.savez_compressed(os.path.join(HERE, "codes.npz"), **out)
    print("wrote", os.path.join(HERE, "codes.npz"), sum(v.nbytes for v in out.values()), "bytes")


if __name__ == "__main__":
    main()
