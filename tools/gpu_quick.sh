#!/bin/bash
# Quick GPU iteration: attention/codec parity + bench (no CPU baseline).
# Usage under gpurun: bash tools/gpu_quick.sh [pytest-k-expr]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-"attention or codec"}
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/q_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/q_bench.log
timeout 600 python bench.py --no-cpu-baseline --no-compress --no-other-configs --steps 100 --config c4 > gpurun_out/q_bench_c4.log 2>&1
tail -3 gpurun_out/q_pytest.log
python - <<'PY'
import json
for f in ["gpurun_out/q_bench.log", "gpurun_out/q_bench_c4.log"]:
    l=[x for x in open(f) if x.startswith('{')]
    if not l: print(f, open(f).read()[-800:]); continue
    d=json.loads(l[-1]); r=d['roofline']
    print(f, 'value', round(d['value']), 'kernel GB/s', round(r['achieved']), 'frac', round(r['frac'],3), 'kernel us', round(r['kernel_ms']*1e3,1), 'step us', round(d['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['value']), 'clk', d['clocks'].get('sm_mhz'))
    c=d.get('compress')
    if c: print('  compress us', round(c['ms']*1e3,1), 'GB/s', round(c['gbs']), ' decode us', round(c['decode']['ms']*1e3,1), 'GB/s', round(c['decode']['gbs']))
PY
