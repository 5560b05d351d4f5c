#!/bin/bash
# Interleaved timing of library variants tools/exp/<V>.so on the K3 workloads:
#   VARIANTS="A B C" CFGS="c3 c5 c4" REPS=2 tools/exp/abn.sh
# prints "cfg variant step_us kernel_us" lines; restores the in-tree library.
cd "$(dirname "$0")/../.."
LIB=paper_2605_21226_b200/liboctoquant_b200.so
cp $LIB /tmp/oq_lib_backup.so
# a variant is NAME (tools/exp/NAME.so) or NAME:VAR=value[,VAR2=value] (same
# library, env set)
for cfg in ${CFGS:-c3}; do for r in $(seq ${REPS:-2}); do for vv in ${VARIANTS:-A B}; do
  v=${vv%%:*}; ev=""; [ "$vv" != "$v" ] && ev=${vv#*:}; ev=${ev//,/ }
  cp tools/exp/$v.so $LIB
  env $ev python bench.py --config $cfg --no-compress --no-cpu-baseline --no-other-configs --steps ${STEPS:-100} --warmup 5 |
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$cfg $vv', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms']*1e3,1))"
done; done; done
cp /tmp/oq_lib_backup.so $LIB
