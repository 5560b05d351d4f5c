cd "$(dirname "$0")/../.."
L=paper_2605_21226_b200/liboctoquant_b200.so
cp $L /tmp/base.so; cp tools/exp/lib_trace.so $L
python tools/exp/trace.py ${1:-131072}
cp /tmp/base.so $L
