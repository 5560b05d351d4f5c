import sys; sys.path.insert(0, '.')
import torch, paper_2605_21226_b200 as oq
dev = torch.device('cuda')
x = torch.randn((1 << 20, 128), device=dev)
a = torch.randn((8192, 8192), device=dev)
for _ in range(30): a @ a
for bits in (2, 3):
    bd, bn = oq.default_bit_split(bits)
    enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn))
    out = torch.empty((x.shape[0], enc.record_bytes), dtype=torch.uint8, device=dev)
    for _ in range(3): enc.compress(x, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): enc.compress(x, out=out)
    e1.record(); torch.cuda.synchronize()
    print(f"b={bits} local3x3 {e0.elapsed_time(e1)/10*1e3:.1f} us")
