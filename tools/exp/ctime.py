"""Compress/decode timing at 2^20 fp32 keys (library CUDA events), b = 2/3/4,
plus a record checksum (variants must produce identical bytes)."""
import os
import sys
import zlib

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2605_21226_b200 as oq  # noqa: E402

x = torch.randn((1 << 20, 128), device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
out = []
for b in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "234")]:
    bd, bn = oq.default_bit_split(b)
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn))
    r = enc.compress(x)
    for _ in range(3):
        enc.compress(x, out=r)
    torch.cuda.synchronize()
    oq.timing(True)
    for _ in range(10):
        enc.compress(x, out=r)
    ms, n = oq.timing_collect("compress")
    oq.timing(False)
    out.append(f"b={b} {1e3 * ms / n:.1f}us crc={zlib.crc32(r.cpu().numpy().tobytes()):08x}")
print(" | ".join(out))
