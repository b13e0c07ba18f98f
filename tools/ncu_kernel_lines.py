"""Per-kernel instruction accounting from an ncu report with source:
  python tools/ncu_kernel_lines.py REP LAUNCH_INDEX [N]
prints the kernel's warp instructions by SASS opcode, instructions per MUFU.EX2,
and the top source lines (k1_cell_solve.cu) by instructions and by stall samples."""
import collections
import csv
import subprocess
import sys

import os
rep, idx = os.path.abspath(sys.argv[1]), int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True, cwd="/tmp").stdout
fname, func = "?", "?"
cur = None                  # current source line key
ops = collections.Counter()
line_ins = collections.Counter()
line_smp = collections.Counter()
line_ops = collections.defaultdict(collections.Counter)
line_txt = {}
for r in csv.reader(txt.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No" or len(r) < 8:
        continue
    if r[2] == "-":            # source row
        cur = (fname, r[0])
        line_txt[cur] = r[1].strip()[:80]
        continue
    # SASS row: address, sass text
    try:
        smp, ins = int(r[4]), int(r[7])
    except ValueError:
        continue
    op = r[3].strip().split()
    if op and op[0].startswith("@"):
        op = op[1:]
    opc = op[0] if op else "?"
    ops[opc] += ins
    if cur is not None:
        line_ins[cur] += ins
        line_smp[cur] += smp
        line_ops[cur][opc.split(".")[0]] += ins
tot = sum(ops.values()) or 1
ex2 = sum(v for k, v in ops.items() if k.startswith("MUFU.EX2"))
mufu = sum(v for k, v in ops.items() if k.startswith("MUFU"))
print(f"{func}\n warp instructions {tot:.4g}, MUFU {mufu:.4g} (EX2 {ex2:.4g}), instructions per MUFU {tot / max(mufu, 1):.2f}")
print("--- by opcode")
for k, v in ops.most_common(30):
    print(f"  {100 * v / tot:5.1f}%  {k}")
ts = sum(line_smp.values()) or 1
print("--- source lines by instructions")
for key, v in line_ins.most_common(n):
    mix = ",".join(f"{o}:{c * 100 // v}" for o, c in line_ops[key].most_common(4))
    print(f"  {100 * v / tot:5.1f}% ins {100 * line_smp[key] / ts:5.1f}% smp {key[0]}:{key[1]:>5} {line_txt[key][:60]:60s} [{mix}]")
print("--- source lines by stall samples")
for key, v in line_smp.most_common(n // 2):
    print(f"  {100 * line_ins[key] / tot:5.1f}% ins {100 * v / ts:5.1f}% smp {key[0]}:{key[1]:>5} {line_txt[key][:60]}")

# region totals (k1_cell_solve.cu line ranges; inlined helpers count where they are inlined only
# when their own file is k1_cell_solve.cu -- helpers from other headers go to "other")
if len(sys.argv) > 4:
    regions = []
    for spec in sys.argv[4].split(","):
        name, rng = spec.split("=")
        a, b = rng.split("-")
        regions.append((name, int(a), int(b)))
    agg = collections.Counter()
    aggm = collections.Counter()
    for (f, ln), v in line_ins.items():
        tag = "other:" + f
        if f == "k1_cell_solve.cu" and ln.isdigit():
            for name, a, b in regions:
                if a <= int(ln) <= b:
                    tag = name
                    break
        agg[tag] += v
        aggm[tag] += line_ops[(f, ln)]["MUFU"]
    print("--- regions (instructions)")
    for k, v in agg.most_common():
        print(f"  {100 * v / tot:5.1f}%  {k:32s} MUFU {100 * aggm[k] / max(mufu, 1):5.1f}%")
