"""Per-kernel counts of the SASS instructions that show how a kernel moves
data (TMA bulk copies, LDGSTS, mbarrier syncs, shuffles/votes, atomics) in
the built library.  usage: python tools/sass_summary.py [lib.so]"""
import os, re, subprocess, sys
from collections import Counter, defaultdict
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1406_1066_b200", "lib", "libsa_b200.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["UBLKCP", "UTMALDG", "LDGSTS", "SYNCS", "VOTE", "MATCH", "REDUX", "SHFL", "ATOMS", "ATOMG", "RED",
        "LDG", "STG", "LDS", "STS", "BAR"]
per = defaultdict(Counter)
fn = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if fn and m:
        op = m.group(1)
        for k in keys:
            if op == k or (k in ("RED", "LDG", "STG") and op == k):
                per[fn][k] += 1
def short(f):
    f = re.sub(r"^_ZN2sa\d+", "", f)
    f = re.sub(r"^_ZN2sa12_GLOBAL__N_1\d+", "", f)
    return f[:60]
seen = set()
print("%-60s " % "kernel (one instantiation per name)" + " ".join("%7s" % k for k in keys))
for f, c in sorted(per.items()):
    base = re.sub(r"I.*", "", short(f))
    if base in seen or not base.startswith("k_"):
        continue
    seen.add(base)
    print("%-60s " % short(f) + " ".join("%7d" % c[k] for k in keys))
