#!/bin/bash
# K3 timing across the three attention workloads (step us, kernel us), twice each.
cd "$(dirname "$0")/../.."
for cfg in ${CFGS:-c3 c5 c4}; do for i in 1 2; do
  python bench.py --config $cfg --no-compress --no-cpu-baseline --no-other-configs --steps 50 --warmup 5 |
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$cfg', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms']*1e3,1))"
done; done
