"""Per-source-line hotspots from `ncu -i REP --page source --csv --print-source cuda,sass`:
  python tools/ncu_lines.py REP [N]  -> top lines by warp-stall samples and by instructions."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
for r in csv.reader(txt.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or len(r) < 8:
        continue
    if r[2] != "-":
        continue            # SASS rows
    try:
        rows.append((fname, int(r[0]), r[1].strip()[:90], int(r[4]), int(r[7])))
    except ValueError:
        pass
ts = sum(x[3] for x in rows) or 1
ti = sum(x[4] for x in rows) or 1
print(f"total stall samples {ts}, warp instructions {ti}")
print("--- by stall samples")
for f, ln, src, st, ins in sorted(rows, key=lambda x: -x[3])[:n]:
    print(f"{st / ts * 100:5.1f}% smp {ins / ti * 100:5.1f}% ins  {f}:{ln}  {src}")
print("--- by instructions")
for f, ln, src, st, ins in sorted(rows, key=lambda x: -x[4])[:n]:
    print(f"{st / ts * 100:5.1f}% smp {ins / ti * 100:5.1f}% ins  {f}:{ln}  {src}")
