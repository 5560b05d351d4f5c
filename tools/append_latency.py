import sys, time; sys.path.insert(0, '.')
import torch, paper_2605_21226_b200 as oq
dev = torch.device('cuda')
bd, bn = oq.default_bit_split(3)
ek = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn)); ev = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=3))
cache = oq.KVCache(ek, ev, 8, 4, 4096)
kn = torch.randn((8, 4, 128), device=dev).to(torch.bfloat16)
x = kn.reshape(32, 128)
recs = torch.empty((32, ek.record_bytes), dtype=torch.uint8, device=dev)
for _ in range(5): ek.compress(x, out=recs); cache.append(kn, kn, pos=5)
torch.cuda.synchronize()
def t(f, n=200):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    c0 = time.perf_counter(); e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize(); c1 = time.perf_counter()
    return e0.elapsed_time(e1) / n * 1e3, (c1 - c0) / n * 1e6
print('compress 32 bf16 keys: gpu us %.1f  cpu us %.1f' % t(lambda: ek.compress(x, out=recs)))
print('append K+V: gpu us %.1f  cpu us %.1f' % t(lambda: cache.append(kn, kn, pos=5)))
big = torch.randn((1 << 20, 128), device=dev)
r2 = torch.empty((1 << 20, ek.record_bytes), dtype=torch.uint8, device=dev)
print('compress 2^20 fp32: gpu us %.1f  cpu us %.1f' % t(lambda: ek.compress(big, out=r2), 10))
# warm the GPU up, then measure again
a = torch.randn((8192, 8192), device=dev)
for _ in range(50): a @ a
torch.cuda.synchronize()
print('compress 2^20 fp32 (after warm-up): gpu us %.1f  cpu us %.1f' % t(lambda: ek.compress(big, out=r2), 10))
fl = torch.zeros(1, dtype=torch.int32, device=dev)
print('compress 2^20 fp32 flagged: gpu us %.1f  cpu us %.1f' % t(lambda: ek.compress(big, out=r2, flagged=fl), 10), int(fl.item()))

def graph_time(f, reps=20):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        f(); f()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph):
        for _ in range(reps): f()
    gph.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): gph.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (10 * reps) * 1e3
print('graph: compress 32 bf16 keys %.1f us' % graph_time(lambda: ek.compress(x, out=recs)))
print('graph: append K+V %.1f us' % graph_time(lambda: cache.append(kn, kn, pos=5)))
