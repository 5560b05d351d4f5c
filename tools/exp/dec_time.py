import sys; sys.path.insert(0, '.')
import torch, paper_2605_21226_b200 as oq
dev = torch.device('cuda')
x = torch.randn((1 << 20, 128), device=dev)
a = torch.randn((8192, 8192), device=dev)
for _ in range(30): a @ a
for bits in (2, 3, 4):
    bd, bn = oq.default_bit_split(bits)
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn))
    r = enc.compress(x)
    o = torch.empty((x.shape[0], 128), device=dev)
    for _ in range(3): enc.decode(r, out=o) if 'out' in enc.decode.__code__.co_varnames else enc.decode(r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): enc.decode(r, out=o) if 'out' in enc.decode.__code__.co_varnames else enc.decode(r)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    nb = x.shape[0] * (enc.record_bytes + 512)
    print(f"decode b={bits}: {ms*1e3:.1f} us  {nb/ms/1e6:.0f} GB/s")
