"""Summarise ncu outputs into profiles/ (tracked):

  python tools/ncu_summary.py --tag r01 --launches gpurun_out/launches_r01.csv \
      [--rep gpurun_out/k1_full_r01.ncu-rep] [--out profiles]

Writes profiles/<tag>_launches.md (per-kernel share of the serialised launch
list) and profiles/<tag>_k1_full.md (key `--set full` metrics per captured
k1 launch: durations, pipe utilisation, stall reasons, dram bytes, occupancy).
"""
import argparse
import csv
import io
import os
import subprocess
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("--tag", required=True)
ap.add_argument("--launches", default="")
ap.add_argument("--rep", default="")
ap.add_argument("--out", default="profiles")
ap.add_argument("--note", default="")
a = ap.parse_args()
os.makedirs(a.out, exist_ok=True)


def read_csv_text(txt):
    i = txt.index('"ID"')
    return list(csv.DictReader(io.StringIO(txt[i:])))


if a.launches:
    rows = read_csv_text(open(a.launches).read())
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            v *= 1e3
        elif r["Metric Unit"] == "ms":
            v *= 1e6
        elif r["Metric Unit"] == "s":
            v *= 1e9
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(a.out, f"{a.tag}_launches.md"), "w") as f:
        f.write(f"# {a.tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
        if a.note:
            f.write(a.note + "\n\n")
        f.write("Serialised, cold-cache per-launch times: compare SHARES, not absolutes.\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---:|---:|---:|\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{k}` | {v[0]} | {v[1] / 1e6:.2f} | {v[1] / tot * 100:.2f}% |\n")
        f.write(f"\nTotal {tot / 1e6:.1f} ms over {sum(v[0] for v in agg.values())} launches.\n")
    print("wrote", os.path.join(a.out, f"{a.tag}_launches.md"))

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe % of active"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % of active"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % of active"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % of active"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe % of active"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("dram__bytes_read.sum", "dram bytes read"),
    ("dram__bytes_write.sum", "dram bytes write"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("smsp__inst_executed_pipe_xu.sum", "XU warp instructions"),
    ("smsp__inst_executed.sum", "warp instructions"),
]

if a.rep:
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, units = r[0], r[1]
    idx = {n: i for i, n in enumerate(h)}
    with open(os.path.join(a.out, f"{a.tag}_k1_full.md"), "w") as f:
        f.write(f"# {a.tag}: ncu --set full of one finest-layer sweep\n\n")
        if a.note:
            f.write(a.note + "\n\n")
        for row in r[2:]:
            name = row[idx["Kernel Name"]]
            f.write(f"## ID {row[idx['ID']]}: `{name[:80]}`\n\n| metric | value | unit |\n|---|---:|---|\n")
            for key, label in KEYS:
                if key in idx and row[idx[key]] not in ("", "n/a"):
                    f.write(f"| {label} (`{key}`) | {row[idx[key]]} | {units[idx[key]]} |\n")
            stalls = []
            for n, i in idx.items():
                if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
                    try:
                        stalls.append((float(row[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
            tot = sum(v for v, _ in stalls)
            if tot > 0:
                f.write("\nPC-sampling stall reasons (share of samples): ")
                f.write(", ".join(f"{n} {v / tot * 100:.1f}%" for v, n in sorted(stalls, reverse=True)[:8]))
                f.write("\n")
            f.write("\n")
    print("wrote", os.path.join(a.out, f"{a.tag}_k1_full.md"))
