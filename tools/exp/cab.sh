#!/bin/bash
# Interleaved compress timing of library variants: VARIANTS="A B" BITS=234 REPS=2
cd "$(dirname "$0")/../.."
LIB=paper_2605_21226_b200/liboctoquant_b200.so
cp $LIB /tmp/oq_lib_backup.so
for r in $(seq ${REPS:-2}); do for v in ${VARIANTS:-A B}; do
  cp tools/exp/$v.so $LIB
  echo "$v $(python tools/exp/ctime.py ${BITS:-234})"
done; done
cp /tmp/oq_lib_backup.so $LIB
