cd "$(dirname "$0")/../.."
for x in 16 24 32 40; do
  r=$(for i in 1 2; do OQ_ATTN_SKO=$x python tools/exp/attn_fixed.py 2>&1 | grep 131072 | sed 's/.*K3 \([0-9.]*\) us.*/\1/'; done | tr '\n' ' ')
  echo "SKO=$x C3 K3 us: $r"
done
