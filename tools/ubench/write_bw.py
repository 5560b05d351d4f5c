"""HBM bandwidth of write-dominated streams on this GPU (K2 decode writes
512 B per 58 B read): torch fill (write only), copy (1:1), and a 1:8 read:write
expansion (each input float4 replicated 8x), best of 10, CUDA events."""
import torch

n = 1 << 28  # 1 GiB of fp32
dev = torch.device("cuda")
out = torch.empty(n, dtype=torch.float32, device=dev)
src = torch.randn(n // 8, dtype=torch.float32, device=dev)
full = torch.randn(n, dtype=torch.float32, device=dev)


def best(fn, nbytes):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return nbytes / (min(ts) * 1e-3) / 1e9


print("fill (write only)      %.0f GB/s" % best(lambda: out.fill_(1.0), 4 * n))
print("copy (1 read : 1 write) %.0f GB/s" % best(lambda: out.copy_(full), 8 * n))
v = out.view(n // 32, 8, 4)
s4 = src.view(n // 32, 1, 4)
print("expand (1 read : 8 write) %.0f GB/s" % best(lambda: v.copy_(s4.expand(-1, 8, -1)), 4 * n + 4 * n // 8))
