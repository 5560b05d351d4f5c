import sys, os; sys.path.insert(0, '.')
import torch, paper_2605_21226_b200 as oq
import bench
dev = torch.device('cuda')
for T in (32, 4096, 131072):
    cache, _ = bench.build_cache(oq, torch, dev, 3, False, 8, 4, T, seed=1)
    q = torch.randn((8, 28, 128), device=dev)
    out = torch.empty((8, 28, 128), device=dev)
    for _ in range(3): oq.attention_decode(q, cache, n_splits=0, out=out)
    torch.cuda.synchronize()
    oq.timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): oq.attention_decode(q, cache, n_splits=0, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms, k = oq.timing_collect("attention"); oq.timing(False)
    print(f"{os.environ.get('OQ_ATTN_UNFUSED') and 'unfused' or 'fused'} T={T}: K3 {ms/k*1e3:.1f} us, step {e0.elapsed_time(e1)/50*1e3:.1f} us")
    del cache; torch.cuda.empty_cache()
