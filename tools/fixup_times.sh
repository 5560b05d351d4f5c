#!/bin/bash
# Per-mode K1 times (tools/compress_modes.py) and the exact-fixup kernel's
# share from an ncu launch list (6 groups of 14 launches: b = 2, 3, 4 x
# scalar, local3x3).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"compress_f" --csv \
    --log-file gpurun_out/fx.csv python tools/compress_modes.py > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/fx.csv")))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
seq = [(r[ki].split("(")[0], float(r[vi].replace(",", "")) / 1e3) for r in rows[h + 1:]]
for name in ("fast", "fixup"):
    v = [t for n, t in seq if name in n]
    print(name, " ".join("%.1f" % (sum(v[i:i + 14]) / len(v[i:i + 14])) for i in range(0, len(v), 14)))
PY
python tools/compress_modes.py
