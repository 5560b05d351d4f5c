#!/bin/bash
# A/B of K3 variants selected by OQ_ATTN_WARPS (8 = variant A, 106/108 = K/V
# warp pairs): GPU attention tests, then C3 (and C4/C5) kernel times.
cd "$(dirname "$0")/../.."
for nw in ${NWS:-8 106 108}; do
  OQ_ATTN_WARPS=$nw timeout 600 python -m pytest tests -m gpu -q -x -k "attention and not qjl" 2>&1 | tail -1 | sed "s/^/nw=$nw tests: /"
  for cfg in ${CFGS:-c3}; do
    OQ_ATTN_WARPS=$nw timeout 300 python bench.py --no-cpu-baseline --no-compress --no-other-configs --steps 50 --config $cfg 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']
print('nw=$nw $cfg', 'kernel us %.1f' % (r['kernel_ms']*1e3), 'frac %.3f' % r['frac'], 'step us %.1f' % (d['ms_per_step']*1e3))"
  done
done
