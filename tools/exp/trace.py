import sys, ctypes as C; sys.path.insert(0, '.')
import torch, numpy as np, paper_2605_21226_b200 as oq
import bench
dev = torch.device('cuda')
T = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cache, _ = bench.build_cache(oq, torch, dev, 3, False, 8, 4, T, seed=1)
q = torch.randn((8, 28, 128), device=dev)
out = torch.empty((8, 28, 128), device=dev)
for _ in range(5): oq.attention_decode(q, cache, n_splits=0, out=out)
torch.cuda.synchronize()
L = oq.lib(); L.oq_debug_trace.argtypes = [C.c_void_p]
buf = np.zeros((148, 16), np.uint64)
L.oq_debug_trace(buf.ctypes.data)
t0 = buf[buf[:, 0] > 0, 0].min()
names = ["start", "staged", "qprep0", "tiles0", "stateout0", "merge0", "atomic0", "end0", "qprep1", "tiles1", "stateout1", "merge1", "atomic1", "end1", "qp_wht", "qp_sync"]
rel = np.where(buf > 0, (buf.astype(np.int64) - int(t0)) / 1000.0, np.nan)
for k, nm in enumerate(names):
    col = rel[:, k]
    v = col[~np.isnan(col)]
    if v.size: print(f"{nm:10s} n={v.size:3d} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
ends = np.nanmax(rel[:, [7, 13]], axis=1)
print("CTA end: min %.2f med %.2f max %.2f" % (np.nanmin(ends), np.nanmedian(ends), np.nanmax(ends)))
