"""Time K1 (oq_compress) on 2^20 fp32 keys per rounding mode and bit width:
the gap between scalar and local3x3 bounds what the 3x3 search costs."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2605_21226_b200 as oq

dev = torch.device("cuda")
x = torch.randn((1 << 20, 128), device=dev)
a = torch.randn((8192, 8192), device=dev)
for _ in range(30):
    a @ a
for bits in (2, 3, 4):
    bd, bn = oq.default_bit_split(bits)
    for rnd in ("scalar", "local3x3"):
        enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rounding=rnd))
        out = torch.empty((x.shape[0], enc.record_bytes), dtype=torch.uint8, device=dev)
        fl = torch.zeros(1, dtype=torch.int32, device=dev)
        for _ in range(3):
            enc.compress(x, out=out, flagged=fl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            enc.compress(x, out=out)
        e1.record()
        torch.cuda.synchronize()
        enc.compress(x, out=out, flagged=fl)
        print(f"b={bits} {rnd:9s} {e0.elapsed_time(e1) / 10 * 1e3:7.1f} us  flagged {int(fl.item()) / x.shape[0] * 100:.2f} %")
