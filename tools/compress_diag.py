"""K1 diagnostics on the GPU: flagged-key counts of the certified fp32 pass
and per-kernel times (fast pass + exact fallback) at 2^20 keys."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2605_21226_b200 as oq

n = 1 << 20
x = torch.randn((n, 128), device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
for bits in (2, 3, 4):
    for rnd in ("local3x3", "scalar"):
        bd, bn = oq.default_bit_split(bits)
        enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rounding=rnd))
        fl = torch.zeros(1, dtype=torch.int32, device="cuda")
        r = enc.compress(x, flagged=fl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            enc.compress(x, out=r, flagged=fl)
        e1.record()
        torch.cuda.synchronize()
        print(f"b={bits} {rnd:9s} flagged {int(fl.item()):6d} ({100*fl.item()/n:.3f} %)  "
              f"{e0.elapsed_time(e1)/5*1e3:.1f} us per 2^20 keys", flush=True)
