"""CPU pin of the needle harness restatement (needle_harness.py) against the
reference's acceptance targets (acceptance_test.cpp:219-228), with the
oracle as the codec: fp32 mass 0.960 +- 0.01 and octo b=2 0.92 +- 0.02 over
run_needle's 128 seeds.  The GPU version is test_gpu_needle.py."""
import numpy as np

from needle_harness import D, N_SEEDS, fp32_mass, needle_case, softmax_mass0


def test_fp32_needle_mass(orc):
    m = float(np.mean([fp32_mass(orc, s) for s in range(N_SEEDS)]))
    assert abs(m - 0.960) <= 0.01, m


def test_octo_b2_needle_mass_oracle(orc):
    ms = []
    for s in range(N_SEEDS):
        keys, q, rot, qs = needle_case(orc, s)
        ok = orc.encoder(b_dir=3, b_nrm=1, rotation_seed=rot, qjl_seed=qs)
        recs = np.stack([ok.encode_f64(k) for k in keys])
        ms.append(softmax_mass0(np.array([ok.score(q, r) for r in recs]) / np.sqrt(float(D))))
    assert abs(float(np.mean(ms)) - 0.92) <= 0.02, np.mean(ms)
