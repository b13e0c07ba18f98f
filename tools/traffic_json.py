"""profiles/k1_traffic.json from an ncu --csv metrics log of the K1 tier
launches of one finest-layer sweep (tools/profile_sweep.py --profile-last):

  python tools/traffic_json.py gpurun_out/k1_traffic_TAG.csv TAG
"""
import csv
import io
import json
import sys
from collections import defaultdict

src, tag = sys.argv[1], sys.argv[2]
txt = open(src).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
per = defaultdict(dict)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
for r in rows:
    k = r["Kernel Name"].replace("void ", "").replace("dd::", "").split("(")[0]
    v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
    name = {"dram__bytes_read.sum": "read", "dram__bytes_write.sum": "write", "gpu__time_duration.sum": "ms"}.get(
        r["Metric Name"], r["Metric Name"])
    per[k][name] = per[k].get(name, 0.0) + v
tot = sum(v.get("read", 0) + v.get("write", 0) for v in per.values())
out = {
    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum of the K1 tier launches "
              f"of the last (kappa=0.5) 2048^2 sweep of cfg 5 (tools/profile_sweep.py --profile-last, DD_SERIAL_TIERS=1); "
              f"profiles/k1_traffic_{tag}.csv",
    "bytes_per_launch": tot,
    "unit": f"bytes per finest-layer sweep ({len(per)} K1 tier launches, tier G included)",
    "per_tier": per,
}
json.dump(out, open("profiles/k1_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
