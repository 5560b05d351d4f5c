#!/bin/bash
# Interleaved K2 decode timing of library variants tools/exp/<V>.so:
#   VARIANTS="A B" REPS=3 tools/exp/dab.sh
cd "$(dirname "$0")/../.."
LIB=paper_2605_21226_b200/liboctoquant_b200.so
cp $LIB /tmp/oq_lib_backup.so
for r in $(seq ${REPS:-3}); do for v in ${VARIANTS:-A B}; do
  cp tools/exp/$v.so $LIB
  echo "$v $(python tools/exp/dec_time.py 2>&1 | tr '\n' ' ')"
done; done
cp /tmp/oq_lib_backup.so $LIB
