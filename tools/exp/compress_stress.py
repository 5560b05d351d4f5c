"""Determinism stress for K1 (certified pass + fixup): the same 2^20 keys
compressed many times at b = 2, 3, 4 must give identical records."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_21226_b200 as oq
x = torch.randn((1 << 20, 128), device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
bad = 0
for b in (2, 3, 4):
    bd, bn = oq.default_bit_split(b)
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn))
    ref = enc.compress(x)
    r = torch.empty_like(ref)
    for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
        enc.compress(x, out=r)
        if not torch.equal(r, ref):
            bad += 1
            print(f"b={b} rep {i}: {(r != ref).any(dim=1).sum().item()} records differ")
print("mismatches:", bad)
