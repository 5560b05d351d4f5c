cd "$(dirname "$0")/../.."
for x in 0 32 48 64 96; do echo "SKO=$x"; OQ_ATTN_SKO=$x python tools/exp/attn_fixed.py 2>&1 | grep 131072; done
timeout 300 python -m pytest tests -m gpu -q -x -k "attention or sharded" 2>&1 | tail -1
