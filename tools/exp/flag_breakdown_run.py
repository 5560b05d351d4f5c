import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2605_21226_b200 as oq
L = oq.lib()
x = torch.randn((1 << 20, 128), device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
names = ["", "hemisphere/sign", "xi bucket", "eta bucket", "3x3 argmax", "norm bucket"]
for b in (2, 3, 4):
    bd, bn = oq.default_bit_split(b)
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn))
    L.oq_debug_flagcat_reset()
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    enc.compress(x, flagged=fl)
    torch.cuda.synchronize()
    h = (C.c_ulonglong * 8)()
    L.oq_debug_flagcat(h)
    print(f"b={b} flagged keys {fl.item()}: " + ", ".join(f"{names[k]} {h[k]}" for k in range(1, 6)))
