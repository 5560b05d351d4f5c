cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for nw in 8 12 16; do OQ_ATTN_WARPS=$nw timeout 300 python bench.py --no-cpu-baseline --no-compress --steps 100 > gpurun_out/bench_nw$nw.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_attention.py -q > gpurun_out/pytest_attn.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_attn.log
for nw in 8 12 16; do python - <<PY
import json
l=[x for x in open('gpurun_out/bench_nw$nw.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print($nw, 'value', round(d['value']), 'kernel', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'],3), 'ms/step', round(d['ms_per_step'],4))
else: print($nw, open('gpurun_out/bench_nw$nw.log').read()[-500:])
PY
done
tail -2 gpurun_out/pytest_attn.log
