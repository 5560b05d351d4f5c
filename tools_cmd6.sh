#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/kc.py <<'PY'
import sys; sys.path.insert(0, "/root/repo")
import torch, paper_2605_21226_b200 as oq
bd, bn = oq.default_bit_split(3)
enc = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn))
x = torch.randn((1 << 20, 128), device="cuda")
r = enc.compress(x)
d = enc.decode(r)
for _ in range(3):
    enc.compress(x, out=r); enc.decode(r, out=d)
torch.cuda.synchronize()
PY
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:"compress_kernel|decode_kernel" -s 2 -c 2 -o gpurun_out/prof_codec -f python /tmp/kc.py > gpurun_out/ncu_codec.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_codec.log
