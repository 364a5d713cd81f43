"""Summarise an ncu source page: CUDA source lines ranked by warp-stall samples.
usage: python tools/ncu_hot.py report.ncu-rep [top] [column, default warp-stall samples]"""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, agg, tot = None, [], 0.0
hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; ix = hdr.index(col); continue
    if hdr is None or r[0] == "" or r[0] == "Function Name": continue
    try: v = float(r[ix] or 0)
    except ValueError: continue
    agg.append((v, f"{fname}:{r[0]}", r[1].strip()[:100])); tot += v
for v, loc, s in sorted(agg, reverse=True)[:top]:
    print(f"{v/tot*100:5.1f}%  {loc:>22}  {s}")
