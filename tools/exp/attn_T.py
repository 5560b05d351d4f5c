import sys; sys.path.insert(0, '.')
import torch, paper_2605_21226_b200 as oq
import bench
dev = torch.device('cuda')
for T in (16384, 32768, 65536, 131072, 262144):
    cache, _ = bench.build_cache(oq, torch, dev, 3, False, 8, 4, T, seed=1)
    q = torch.randn((8, 28, 128), device=dev)
    out = torch.empty((8, 28, 128), device=dev)
    for _ in range(3): oq.attention_decode(q, cache, n_splits=0, out=out)
    torch.cuda.synchronize()
    oq.timing(True)
    for _ in range(20): oq.attention_decode(q, cache, n_splits=0, out=out)
    torch.cuda.synchronize()
    ms, k = oq.timing_collect("attention"); oq.timing(False)
    us = ms / k * 1e3
    tiles = 8 * 4 * T / 32
    print(f"T={T}: K3 {us:.1f} us, {us*1e3/tiles*148:.0f} ns per tile per SM, {8*4*T*116/us/1e3:.0f} GB/s")
    del cache; torch.cuda.empty_cache()
