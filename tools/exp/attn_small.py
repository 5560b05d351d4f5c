import sys, os; sys.path.insert(0, '.')
import torch, paper_2605_21226_b200 as oq
import bench
dev = torch.device('cuda')
T = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cache, _ = bench.build_cache(oq, torch, dev, 3, False, 8, 4, T, seed=1)
q = torch.randn((8, 28, 128), device=dev)
out = torch.empty((8, 28, 128), device=dev)
for _ in range(6): oq.attention_decode(q, cache, n_splits=0, out=out)
torch.cuda.synchronize()
