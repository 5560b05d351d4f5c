cd "$(dirname "$0")/../.."
L=paper_2605_21226_b200/liboctoquant_b200.so
cp $L /tmp/base.so
echo "== base"; python tools/exp/cm_short.py
for v in "$@"; do cp tools/exp/$v.so $L; echo "== $v"; python tools/exp/cm_short.py; done
cp /tmp/base.so $L
