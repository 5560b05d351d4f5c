#!/bin/bash
# A/B of two library builds (tools/exp/A.so, tools/exp/B.so) on the K3
# workloads, interleaved: A B A B per config.
cd "$(dirname "$0")/../.."
LIB=paper_2605_21226_b200/liboctoquant_b200.so
for cfg in ${CFGS:-c3 c5 c4}; do for r in 1 2; do for v in A B; do
  cp tools/exp/$v.so $LIB
  python bench.py --config $cfg --no-compress --no-cpu-baseline --no-other-configs --steps 100 --warmup 5 |
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$cfg $v', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms']*1e3,1))"
done; done; done
