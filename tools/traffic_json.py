"""Merge per-kernel DRAM traffic from ncu reports into profiles/dram_traffic.json
(bench.py reads `traffic` of the dominant kernel from it).
usage: python tools/traffic_json.py WORKLOAD report.ncu-rep [WORKLOAD report ...]"""
import csv, json, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "dram_traffic.json")


def bench_name(k):  # ncu kernel name -> the names bench.py / sa_last_kernel_times use
    k = k.split("(")[0].replace("void ", "").strip()
    m = re.match(r"(?:sa::)?k_rpass<(\d)", k)
    if m: return "k_rpass0" if m.group(1) in ("1", "true") else "k_rpass1"
    m = re.match(r"(?:sa::)?k_rup<(\w+)>", k)
    if m: return "k_rup0" if m.group(1) in ("1", "true") else "k_rup1"
    k = re.sub(r"<.*", "", k).replace("sa::", "")
    return {"k_colcount_win": "k_colcount", "k_scatter_staged": "k_scatter"}.get(k, k)


db = json.load(open(OUT)) if os.path.exists(OUT) else {}
args = sys.argv[1:]
for wl, rep in zip(args[::2], args[1::2]):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    acc = {}
    for v in rows[2:]:
        d = dict(zip(h, v))
        u = dict(zip(h, units))
        scale = lambda k: {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}[u[k]]
        name = bench_name(d["Kernel Name"])
        r = acc.setdefault(name, {"launches": 0, "avg_ns": 0.0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0})
        r["launches"] += 1
        r["dram_read_bytes"] += float(d["dram__bytes_read.sum"]) * scale("dram__bytes_read.sum")
        r["dram_write_bytes"] += float(d["dram__bytes_write.sum"]) * scale("dram__bytes_write.sum")
        dur = float(d["gpu__time_duration.sum"]) * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}[u["gpu__time_duration.sum"]]
        r["avg_ns"] += dur
    for r in acc.values():
        n = r["launches"]
        r["avg_ns"] /= n; r["dram_read_bytes"] /= n; r["dram_write_bytes"] /= n
        r["source"] = os.path.basename(os.path.dirname(rep)) + "/" + os.path.basename(rep)
    db[wl] = acc
json.dump(db, open(OUT, "w"), indent=1)
print(json.dumps({k: list(v) for k, v in db.items()}))
