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
    # last decode step = last qprep .. combine window
    idx = [i for i, (n, _) in enumerate(seq) if "qprep" in n]
    if idx:
        i0 = idx[-1]
        step = [(n, t) for n, t in seq[i0:i0 + 3]]
        tot = sum(t for _, t in step)
        print("\nLast decode step (cold-cache, serialised under ncu):")
        for n, t in step:
            print(f"- `{n}`: {t:.1f} us ({100 * t / tot:.1f} % of the step)")


def full(path, units, unit_name):
    raw = _csv(["-i", path, "--page", "raw", "--csv"])
    h, v = raw[0], raw[2]
    print(f"Kernel: `{v[h.index('Kernel Name')]}`\n")
    print("| counter | value |\n|---|---|")
    for k in RAW_KEYS:
        if k in h:
            print(f"| {k} ({raw[1][h.index(k)]}) | {v[h.index(k)]} |")
    print("\nStalls per issued instruction (> 0.05):\n")
    for i, n in enumerate(h):
        if "issue_stalled" in n and "per_issue_active" in n:
            try:
                if float(v[i]) > 0.05:
                    print(f"- {n.split('stalled_')[1].split('_per')[0]}: {float(v[i]):.2f}")
            except ValueError:
                pass
    src = _csv(["-i", path, "--page", "source", "--csv", "--print-source", "sass"])
    hdr, data = src[1], src[2:]
    si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    cnt, stl, tot, stot = Counter(), Counter(), 0, 0
    for r in data:
        try:
            n = int(r[ei].replace(",", ""))
        except ValueError:
            continue
        op = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip())
        op = op.split()[0] if op else "?"
        cnt[op] += n
        tot += n
        s = int(r[ss] or 0)
        stl[op] += s
        stot += s
    per = f"per {unit_name}" if units else "total"
    div = units if units else 1
    print(f"\nSASS mix (warp instructions {per}; total {tot / div:.1f}):\n")
    print(f"| op | {per} | stall share |\n|---|---|---|")
    for k, c in cnt.most_common(24):
        print(f"| {k} | {c / div:.1f} | {100 * stl[k] / max(1, stot):.1f} % |")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("path")
    ap.add_argument("--units", type=float, default=0)
    ap.add_argument("--unit-name", default="unit")
    a = ap.parse_args()
    if a.mode == "launches":
        launches(a.path)
    else:
        full(a.path, a.units, a.unit_name)


if __name__ == "__main__":
    main()
