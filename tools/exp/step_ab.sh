#!/bin/bash
# Interleaved decode-step (append K+V + attention) timing of library variants:
#   VARIANTS="A B" REPS=3 tools/exp/step_ab.sh
cd "$(dirname "$0")/../.."
LIB=paper_2605_21226_b200/liboctoquant_b200.so
cp $LIB /tmp/oq_lib_backup.so
for r in $(seq ${REPS:-3}); do for v in ${VARIANTS:-A B}; do
  cp tools/exp/$v.so $LIB
  python bench.py --no-cpu-baseline --no-other-configs --steps ${STEPS:-50} --warmup 5 |
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); s=d['decode_step']; print('$v', round(d['ms_per_step']*1e3,1), round(s['append_us'],1), round(s['append_plus_attention_us'],1), round(s['graph_append_plus_attention_us'],1))"
done; done
cp /tmp/oq_lib_backup.so $LIB
