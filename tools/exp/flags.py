"""Flagged-key counts of the certified compress pass at b = 2, 3, 4 (2^20 keys)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_21226_b200 as oq
x = torch.randn((1 << 20, 128), device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
out = []
for b in (2, 3, 4):
    bd, bn = oq.default_bit_split(b)
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn))
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    enc.compress(x, flagged=fl)
    out.append(f"b={b} flagged {fl.item()}")
print(" | ".join(out))
