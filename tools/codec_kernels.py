"""Run K1 compress + K2 decode on 2^20 keys (BASELINE configs[1]) a few times:
the target command for ncu captures of the codec kernels."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2605_21226_b200 as oq

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 3
bd, bn = oq.default_bit_split(bits)
enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn))
x = torch.randn((1 << 20, 128), device="cuda")
r = enc.compress(x)
d = enc.decode(r)
for _ in range(3):
    enc.compress(x, out=r)
    enc.decode(r, out=d)
torch.cuda.synchronize()
