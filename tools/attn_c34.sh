cd $GRAFT_REPO_ROOT
for c in c3 c4 c5; do timeout 300 python bench.py --no-cpu-baseline --no-compress --no-other-configs --steps 100 --config $c 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c kernel us', round(d['roofline']['kernel_ms']*1e3,1), 'step us', round(d['ms_per_step']*1e3,1))"; done
