"""K3 step and kernel time at the C3 shape (B=8, 28/4 heads, 128K tokens) for
b = 2, 3, 4 K=V tiles (W = 7, 10, 13) on this GPU."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_21226_b200 as oq  # noqa: E402

dev = torch.device("cuda:0")
for bits in (2, 3, 4):
    cache, _ = bench.build_cache(oq, torch, dev, bits, False, 8, 4, 131072, seed=0)
    q = torch.randn((8, 28, 128), device=dev)
    out = torch.empty_like(q)
    step, kern = bench.time_attention(oq, torch, lambda qd: oq.attention_decode(qd, cache, out=out),
                                      q, 50)
    nbytes = 8 * 4 * 131072 * 2 * bench.rec_bytes(bits, False)
    print(f"b={bits}: step {step * 1e3:.1f} us, K3 {kern * 1e3:.1f} us, "
          f"{nbytes / (step * 1e-3) / 1e9:.0f} GB/s ({100 * nbytes / (step * 1e-3) / 1e9 / 6547.2:.1f} % of peak)")
    del cache
    torch.cuda.empty_cache()
