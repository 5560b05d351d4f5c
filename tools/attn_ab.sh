cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
OQ_ATTN_IMPL=ws timeout 900 python -m pytest tests -m gpu -q -x -k "attention" 2>&1 | tail -2
for impl in regs ws; do OQ_ATTN_IMPL=$impl timeout 300 python bench.py --no-cpu-baseline --no-compress --steps 100 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$impl c3 kernel us', round(d['roofline']['kernel_ms']*1e3,1), 'GB/s', round(d['roofline']['achieved']))"; done
for impl in regs ws; do OQ_ATTN_IMPL=$impl timeout 300 python bench.py --no-cpu-baseline --no-compress --steps 100 --config c4 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$impl c4 kernel us', round(d['roofline']['kernel_ms']*1e3,1), 'GB/s', round(d['roofline']['achieved']))"; done
