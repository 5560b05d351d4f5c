#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for impl in regs tma; do for nw in 8 12; do OQ_ATTN_IMPL=$impl OQ_ATTN_WARPS=$nw timeout 300 python bench.py --no-cpu-baseline --no-compress --steps 100 > gpurun_out/bench_${impl}_$nw.log 2>&1; done; done
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/pytest_attn.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_attn.log
for impl in regs tma; do for nw in 8 12; do python - <<PY
import json
f='gpurun_out/bench_${impl}_$nw.log'
l=[x for x in open(f) if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print('$impl', $nw, 'value', round(d['value']), 'kernel', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'],3), 'ms/step', round(d['ms_per_step'],4))
else: print('$impl', $nw, open(f).read()[-600:])
PY
done; done
tail -3 gpurun_out/pytest_attn.log
