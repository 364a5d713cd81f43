"""Per-source-line shared-memory wavefronts (total / ideal / excessive) of ONE kernel in an ncu report.
usage: python tools/ncu_smem.py report.ncu-rep kernel_regex [top]"""
import csv, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + rx, "-c", "1"], capture_output=True, text=True).stdout
hdr, agg, fname = None, {}, None
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] in ("File Path", "File Name"): fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; iw = hdr.index("L1 Wavefronts Shared"); ii = hdr.index("L1 Wavefronts Shared Ideal"); ie = hdr.index("Instructions Executed"); continue
    if hdr is None or r[0] in ("", "Function Name"): continue
    try: w, i, e = float(r[iw] or 0), float(r[ii] or 0), float(r[ie] or 0)
    except ValueError: continue
    agg[(fname, r[0])] = (w, i, e, r[1].strip()[:90])
tw = sum(x[0] for x in agg.values()) or 1
print(f"total shared wavefronts {tw:.4g}, ideal {sum(x[1] for x in agg.values()):.4g}")
for k, (w, i, e, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{w / tw * 100:5.1f}% wf  x{(w / i if i else 0):4.1f} of ideal  {e:10.3g} inst  {k[0]}:{k[1]}  {s}")
