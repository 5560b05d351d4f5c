"""Write profiles/<name>_summary.md (+ profiles/ncu_traffic.json) from a
`STAGES="smoke pytest bench ncu" bash tools/gpu_round.sh` run in gpurun_out/.

    python tools/write_profile.py r01_call3 "free-text headline"
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*a):
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), *a],
                          capture_output=True, text=True, cwd=ROOT).stdout


def main():
    name, note = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
    g = os.path.join(ROOT, "gpurun_out")
    d = json.loads([x for x in open(os.path.join(g, "bench.log")) if x.startswith("{")][-1])
    tr = {}
    for rep in ("prof_attn_c3.ncu-rep", "prof_attn_c4.ncu-rep", "prof_attn_c5.ncu-rep",
                "prof_codec.ncu-rep"):
        if os.path.exists(os.path.join(g, rep)):
            tr.update(json.loads(run("traffic", os.path.join(g, rep))))
    json.dump({"source": f"ncu --set full --clock-control none, profiles/{name}_summary.md",
               "dram_bytes_per_launch": tr},
              open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    r, c = d["roofline"], d["compress"]
    att = [k for k in tr if k.startswith("attn_partials_kernel<10, 0,")][0]
    pyt = [x for x in open(os.path.join(g, "pytest_gpu.log")) if "passed" in x]
    out = [f"# {name} — {note}\n",
           "Command: `STAGES=\"smoke pytest bench ncu\" bash tools/gpu_round.sh`.  smoke ok; "
           f"`pytest -m gpu`: {pyt[-1].strip() if pyt else '?'}.\n",
           "## Bench line (C3: B=8, 28/4 heads, 128K tokens, 3-bit K=V)\n",
           "```json\n" + json.dumps(d) + "\n```\n",
           f"- step {d['ms_per_step'] * 1e3:.1f} µs (one fused launch) -> **{d['value']:.0f} GB/s**; "
           f"K3 {r['kernel_ms'] * 1e3:.1f} µs -> {r['achieved']:.0f} GB/s = "
           f"{100 * r['frac']:.1f} % of the measured {r['peak']} GB/s copy peak",
           f"- K3 DRAM traffic per launch (ncu): {tr[att] / 1e6:.1f} MB vs "
           f"{r['algorithmic_bytes_per_launch'] / 1e6:.1f} MB algorithmic "
           f"({tr[att] / r['algorithmic_bytes_per_launch']:.3f}x)",
           f"- e2e (pinned q in, out back, public API): {d['e2e']['value']:.0f} GB/s",
           f"- CPU reference (oracle/_ref, {d['cpu_baseline']['cores']} host threads): "
           f"{d['cpu_baseline']['value']:.3f} GB/s",
           (f"- decoder step (append K+V of 32 streams + attention): append "
            f"{d['decode_step']['append_us']:.1f} µs, step {d['decode_step']['append_plus_attention_us']:.1f} µs"
            f" eager / {d['decode_step'].get('graph_append_plus_attention_us', float('nan')):.1f} µs "
            f"CUDA graph\n" if d.get("decode_step") else "\n"),
           "".join(f"- {k.upper()} K3 ({v['workload']}): {v['kernel_us']:.1f} µs -> {v['kernel_gbs']:.0f} GB/s = "
                   f"{100 * v['frac']:.1f} % of peak\n" for k, v in (d.get("other_configs") or {}).items()),
           "| bits | K1 compress µs | G keys/s | GB/s (% HBM) | flagged keys | K2 decode µs | GB/s (% HBM) |",
           "|---|---|---|---|---|---|---|"]
    for b, v in c["sweep_bits"].items():
        out.append(f"| {b} | {v['compress_ms'] * 1e3:.1f} | {v['compress_keys_per_s'] / 1e9:.2f} | "
                   f"{v['compress_gbs']:.0f} ({100 * v['compress_frac_of_hbm']:.1f} %) | "
                   f"{v['flagged_keys']} | {v['decode_ms'] * 1e3:.1f} | {v['decode_gbs']:.0f} "
                   f"({100 * v['decode_frac_of_hbm']:.1f} %) |")
    out.append("\n## Launch list (`ncu --metrics gpu__time_duration.sum`)\n")
    out.append(run("launches", os.path.join(g, "launches.csv")))
    # tiles per launch: B * Hkv * T / 32 (one 8-head chunk per stream at G = 7)
    for cfg, tiles, what in (("c3", 8 * 4 * 131072 // 32, "C3: B=8, T=128K, 3-bit"),
                             ("c4", 32 * 4 * 32768 // 32, "C4: B=32, T=32K, QJL 2-bit K"),
                             ("c5", 8 * 4 * (1 << 20) // 32, "C5 at P = 1: B=8, T=1M, 2-bit")):
        rep = os.path.join(g, f"prof_attn_{cfg}.ncu-rep")
        if os.path.exists(rep):
            out.append(f"## K3, `ncu --set full` — {what}\n")
            out.append(run("full", rep, "--units", str(tiles), "--unit-name", "tile"))
    out.append("## K1 (certified-fp32 pass + exact re-rounding of the undecided triplets) and K2, "
               "`ncu --set full` (2^20 keys, b=3)\n")
    out.append(run("full", os.path.join(g, "prof_codec.ncu-rep")))
    open(os.path.join(ROOT, "profiles", f"{name}_summary.md"), "w").write("\n".join(out))
    print("wrote", f"profiles/{name}_summary.md")


if __name__ == "__main__":
    main()
