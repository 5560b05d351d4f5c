import sys; sys.path.insert(0, '.')
import torch, paper_2605_21226_b200 as oq
dev = torch.device('cuda')
bd, bn = oq.default_bit_split(3)
ek = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn)); ev = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=3))
cache = oq.KVCache(ek, ev, 8, 4, 4096)
kn = torch.randn((8, 4, 128), device=dev).to(torch.bfloat16)
for _ in range(4): cache.append(kn, kn, pos=5)
torch.cuda.synchronize()
