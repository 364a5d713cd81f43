"""Summarise an ncu launch list (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum, --csv) of bench.py: per-kernel launches, mean time,
share of the library's time, DRAM bytes per launch.  Writes the per-kernel
DRAM bytes into profiles/dram_traffic.json under the given workload name.
usage: python tools/launch_summary.py launches.csv workload [out.md]"""
import csv, json, os, sys
from collections import defaultdict
path, wl = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
h = rows[0]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
per = defaultdict(dict)
for r in rows[1:]:
    per[int(r[ix["ID"]])][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    per[int(r[ix["ID"]])]["name"] = r[ix["Kernel Name"]]
agg = defaultdict(lambda: {"launches": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
for d in per.values():
    n = d["name"].replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    n = n.split("(")[0].split("<")[0].replace("sa::", "").strip()
    if not n.startswith("k_"):
        continue
    a = agg[n]
    a["launches"] += 1
    a["ns"] += d.get("gpu__time_duration.sum", 0.0)
    a["rd"] += d.get("dram__bytes_read.sum", 0.0)
    a["wr"] += d.get("dram__bytes_write.sum", 0.0)
tot = sum(a["ns"] for a in agg.values())
out = {}
lines = ["| kernel | launches | mean time (us) | share | DRAM read / launch (MB) | DRAM write / launch (MB) |",
         "|---|---|---|---|---|---|"]
for n, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
    k = a["launches"]
    out[n] = {"launches": k, "avg_ns": a["ns"] / k, "dram_read_bytes": a["rd"] / k,
              "dram_write_bytes": a["wr"] / k}
    lines.append(f"| {n} | {k} | {a['ns'] / k / 1e3:.1f} | {a['ns'] / tot * 100:.1f} % | "
                 f"{a['rd'] / k / 1e6:.1f} | {a['wr'] / k / 1e6:.1f} |")
print("\n".join(lines))
tp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "dram_traffic.json")
allt = json.load(open(tp)) if os.path.exists(tp) else {}
allt[wl] = out
json.dump(allt, open(tp, "w"), indent=1)
if len(sys.argv) > 3:
    open(sys.argv[3], "w").write("\n".join(lines) + "\n")
