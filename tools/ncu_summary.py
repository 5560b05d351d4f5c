#!/usr/bin/env python
"""Summarise ncu captures into the markdown committed under profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv
    python tools/ncu_summary.py full gpurun_out/prof_attn.ncu-rep [--units N --unit-name tile]

`launches` reads a `--metrics gpu__time_duration.sum --csv` launch list and
prints per-kernel counts, mean durations and the share of the last decode
step; `full` reads a `--set full` report (raw page + SASS source page) and
prints the roofline-relevant counters, the stall profile and the SASS
instruction mix per work unit.
"""
import argparse
import csv
import io
import re
import subprocess
from collections import Counter, OrderedDict

NCU = "/usr/local/cuda/bin/ncu"

RAW_KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def _csv(args):
    out = subprocess.run([NCU] + args, capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    seq = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", "")) / 1e3)
           for r in data]
    agg = OrderedDict()
    for n, t in seq:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += t
    print("| kernel | launches | mean us |\n|---|---|---|")
    for n, (c, t) in agg.items():
        print(f"| `{n}` | {c} | {t / c:.1f} |")
    # last decode step: the last attention launch with its qprep / combine
    # neighbours (the fused path has neither)
    idx = [i for i, (n, _) in enumerate(seq) if "attn_partials" in n]
    if idx:
        i0 = idx[-1]
        lo = i0 - 1 if i0 > 0 and "qprep" in seq[i0 - 1][0] else i0
        hi = i0 + 2 if i0 + 1 < len(seq) and "combine" in seq[i0 + 1][0] else i0 + 1
        step = seq[lo:hi]
        tot = sum(t for _, t in step)
        print("\nLast decode step (cold-cache, serialised under ncu):")
        for n, t in step:
            print(f"- `{n}`: {t:.1f} us ({100 * t / tot:.1f} % of the step)")


def traffic(path):
    """{kernel: dram read + write bytes per launch} of a --set full report."""
    raw = _csv(["-i", path, "--page", "raw", "--csv"])
    h, units = raw[0], raw[1]
    out = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for v in raw[2:]:
        name = v[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        b = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(key)
            b += float(v[i].replace(",", "")) * scale.get(units[i], 1)
        out[name] = b
    return out


def _sass_sections(src):
    """Split the --page source csv (one section per kernel) into row lists."""
    secs, cur = [], None
    for r in src:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1] if len(r) > 1 else "", "rows": []}
            secs.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    return secs


def full(path, units, unit_name):
    raw = _csv(["-i", path, "--page", "raw", "--csv"])
    h = raw[0]
    src = _csv(["-i", path, "--page", "source", "--csv", "--print-source", "sass"])
    secs = _sass_sections(src)
    for k, v in enumerate(raw[2:]):
        print(f"### `{v[h.index('Kernel Name')]}`\n")
        print("| counter | value |\n|---|---|")
        for key in RAW_KEYS:
            if key in h:
                print(f"| {key} ({raw[1][h.index(key)]}) | {v[h.index(key)]} |")
        print("\nStalls per issued instruction (> 0.05):\n")
        for i, n in enumerate(h):
            if "issue_stalled" in n and "per_issue_active" in n:
                try:
                    if float(v[i]) > 0.05:
                        print(f"- {n.split('stalled_')[1].split('_per')[0]}: {float(v[i]):.2f}")
                except ValueError:
                    pass
        if k >= len(secs):
            continue
        rows = secs[k]["rows"]
        hdr, data = rows[0], rows[1:]
        si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        cnt, stl, tot, stot = Counter(), Counter(), 0, 0
        for r in data:
            try:
                n = int(r[ei].replace(",", ""))
            except (ValueError, IndexError):
                continue
            op = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip())
            op = op.split()[0] if op else "?"
            cnt[op] += n
            tot += n
            sv = int(r[ss] or 0)
            stl[op] += sv
            stot += sv
        per = f"per {unit_name}" if units else "total"
        div = units if units else 1
        print(f"\nSASS mix (warp instructions {per}; total {tot / div:.1f}):\n")
        print(f"| op | {per} | stall share |\n|---|---|---|")
        for op, c in cnt.most_common(16):
            print(f"| {op} | {c / div:.1f} | {100 * stl[op] / max(1, stot):.1f} % |")
        print()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full", "traffic"])
    ap.add_argument("path")
    ap.add_argument("--units", type=float, default=0)
    ap.add_argument("--unit-name", default="unit")
    a = ap.parse_args()
    if a.mode == "launches":
        launches(a.path)
    elif a.mode == "traffic":
        import json
        print(json.dumps(traffic(a.path), indent=1))
    else:
        full(a.path, a.units, a.unit_name)


if __name__ == "__main__":
    main()
