"""CUDA source lines ranked by executed warp instructions (ncu source page)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
col = sys.argv[3] if len(sys.argv) > 3 else "Instructions Executed"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, agg, tot, hdr = None, [], 0.0, None
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; ix = hdr.index(col); continue
    if hdr is None or r[0] in ("", "Function Name"): continue
    try: v = float(r[ix] or 0)
    except ValueError: continue
    agg.append((v, f"{fname}:{r[0]}", r[1].strip()[:100])); tot += v
print(f"total {col}: {tot:.4g}")
for v, loc, s in sorted(agg, reverse=True)[:top]:
    print(f"{v/tot*100:5.1f}% {v:10.3g} {loc:>22}  {s}")
