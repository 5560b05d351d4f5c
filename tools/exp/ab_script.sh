#!/bin/bash
# A/B a variant library on any script: bash tools/exp/ab_script.sh <variant> <script.py>
cd "$(dirname "$0")/../.."
L=paper_2605_21226_b200/liboctoquant_b200.so
echo "== base"; python $2
cp $L /tmp/base.so; cp tools/exp/$1.so $L
echo "== $1"; python $2
cp /tmp/base.so $L
