#!/bin/bash
# Time a variant build of the library (tools/exp/<name>.so) against the
# in-tree one on the C3 bench (kernel-only numbers).  Usage under gpurun:
#   bash tools/exp/run_variant.sh lib_noload [config]
cd "$(dirname "$0")/../.."
CFG=${2:-c3}
L=paper_2605_21226_b200/liboctoquant_b200.so
run() { timeout 300 python bench.py --no-cpu-baseline --no-compress --no-other-configs --steps 50 --config $CFG 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']
print('$1', 'kernel us %.1f' % (r['kernel_ms']*1e3), 'frac %.3f' % r['frac'], 'step us %.1f' % (d['ms_per_step']*1e3))"; }
run base
cp $L /tmp/base.so; cp tools/exp/$1.so $L
run $1
cp /tmp/base.so $L
