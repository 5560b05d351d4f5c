cd $GRAFT_REPO_ROOT
for nw in 8 12; do OQ_ATTN_WARPS=$nw timeout 300 python bench.py --no-cpu-baseline --no-compress --no-other-configs --steps 100 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warps $nw kernel us', round(d['roofline']['kernel_ms']*1e3,1))"; done
