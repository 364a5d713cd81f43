"""Find the first sweep instance where the GPU differs from the oracle and
describe the first differing column.  usage: python tools/sweep_debug.py [n]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import paper_1406_1066_b200 as sa
from instances import random_triplets
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
found = 0
for seed in range(1_000_000, 1_000_000 + n):
    ii, jj, sr = random_triplets(seed)
    if len(ii) == 0:
        continue
    m, n_ = int(ii.max()), int(jj.max())
    out = sa.assemble(ii.astype(np.int32), jj.astype(np.int32), sr)
    ref = O.assemble_counting(ii.astype(np.int32), jj.astype(np.int32), sr, m, n_)
    if np.array_equal(out.jc, ref.jc) and np.array_equal(out.ir, ref.ir) and out.pr.tobytes() == ref.pr.tobytes():
        continue
    c = int(np.argmax(out.jc != ref.jc)) if not np.array_equal(out.jc, ref.jc) else None
    if c is None:
        k = int(np.argmax((out.ir != ref.ir) | (out.pr.view(np.uint64) != ref.pr.view(np.uint64))))
        c = int(np.searchsorted(ref.jc, k, side="right") - 1)
    else:
        c = c - 1
    sel = np.flatnonzero(jj == c + 1)
    rows = ii[sel]
    print("seed", seed, "L", len(ii), "m", m, "n", n_, "col", c, "count", len(sel), "distinct", len(np.unique(rows)),
          "maxdup", np.bincount(rows).max())
    a0, a1 = out.jc[c], out.jc[c + 1]; b0, b1 = ref.jc[c], ref.jc[c + 1]
    print(" gpu u", a1 - a0, "ref u", b1 - b0)
    print(" gpu ir", out.ir[a0:a1][:20]); print(" ref ir", ref.ir[b0:b1][:20])
    d = np.flatnonzero(out.pr[a0:a0 + min(a1 - a0, b1 - b0)].view(np.uint64) != ref.pr[b0:b0 + min(a1 - a0, b1 - b0)].view(np.uint64))
    print(" first pr diffs", d[:10], out.pr[a0:a1][d[:3]], ref.pr[b0:b1][d[:3]])
    found += 1
    if found >= 3:
        break
print("done")
