"""Per-source-line warp-stall samples and executed instructions of ONE kernel
in an ncu report.  usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + rx, "-c", "1"], capture_output=True, text=True).stdout
hdr, agg, fname = None, {}, None
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] in ("File Path", "File Name"): fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; ix = hdr.index("Warp Stall Sampling (All Samples)"); ie = hdr.index("Instructions Executed"); continue
    if hdr is None or r[0] in ("", "Function Name"): continue
    try: v, e = float(r[ix] or 0), float(r[ie] or 0)
    except ValueError: continue
    agg[(fname, r[0])] = (v, e, r[1].strip()[:95])
tv = sum(x[0] for x in agg.values()) or 1; te = sum(x[1] for x in agg.values()) or 1
print(f"total warp instructions {te:.4g}")
for k, (v, e, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v / tv * 100:5.1f}% stall  {e / te * 100:5.1f}% inst  {k[0]}:{k[1]}  {s}")
