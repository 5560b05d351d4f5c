"""Host (CPU) time per public-API attention call vs the GPU step time, C3."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_21226_b200 as oq  # noqa: E402

dev = torch.device("cuda:0")
cache, _ = bench.build_cache(oq, torch, dev, 3, False, 8, 4, 131072, seed=0)
q = torch.randn((8, 28, 128), device=dev)
out = torch.empty_like(q)
for _ in range(5):
    oq.attention_decode(q, cache, n_splits=0, out=out)
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N):
    oq.attention_decode(q, cache, n_splits=0, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e6 * (t1 - t0) / N:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / N:.1f} us/call")
# graph of one step
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        oq.attention_decode(q, cache, n_splits=0, out=out)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    oq.attention_decode(q, cache, n_splits=0, out=out)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N):
    oq.attention_decode(q, cache, n_splits=0, out=out)
e1.record()
torch.cuda.synchronize()
print(f"eager GPU step {1e3 * e0.elapsed_time(e1) / N:.1f} us")
e0.record()
for _ in range(N):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph GPU step {1e3 * e0.elapsed_time(e1) / N:.1f} us")
t0 = time.perf_counter()
for _ in range(N):
    g.replay()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"graph host issue {1e6 * (t1 - t0) / N:.1f} us/replay")
