cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/b_c3.log 2>&1
for c in c4 c5; do timeout 600 python bench.py --no-cpu-baseline --no-compress --no-other-configs --steps 50 --config $c > gpurun_out/b_$c.log 2>&1; done
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_partials -s 4 -c 1 -o gpurun_out/prof_attn_c4 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-compress --no-other-configs --config c4 > gpurun_out/ncu_c4.log 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/b_c3.log", "gpurun_out/b_c4.log", "gpurun_out/b_c5.log"]:
    l=[x for x in open(f) if x.startswith('{')]
    if not l: print(f, open(f).read()[-500:]); continue
    d=json.loads(l[-1]); r=d['roofline']
    print(f, 'value', round(d['value']), 'kernel GB/s', round(r['achieved']), 'frac', round(r['frac'],3), 'kernel us', round(r['kernel_ms']*1e3,1), 'step us', round(d['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['value']))
    c=d.get('compress')
    if c:
        for b,v in c['sweep_bits'].items(): print('  b',b, 'compress us', round(v['compress_ms']*1e3,1), 'flagged', v['flagged_keys'], 'decode us', round(v['decode_ms']*1e3,1), 'GB/s', round(v['decode_gbs']))
PY
