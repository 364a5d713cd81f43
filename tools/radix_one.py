"""One assembly of BASELINE config K, twice (for ncu).
usage: python tools/radix_one.py K [path] [scale] [OPT=VAL ...]   (path -1 auto, 0 column, 1 radix)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_1066_b200 as sa
from paper_1406_1066_b200 import _capi, workloads as W
pos = [a for a in sys.argv[1:] if "=" not in a]
k = int(pos[0]); path = int(pos[1]) if len(pos) > 1 else 1
scale = float(pos[2]) if len(pos) > 2 else 1.0
a = sa.default_assembler(0)
a.set_option(_capi.SA_OPT_PATH, path)
for kv in [x for x in sys.argv[1:] if "=" in x]:
    o, v = kv.split("=")
    a.set_option(getattr(_capi, "SA_OPT_" + o), int(v))
w = W.config(k, device=torch.device("cuda", 0), scale=scale)
for _ in range(2):
    out = a.assemble_device(w.ii, w.jj, w.s, m=w.m, n=w.n)
torch.cuda.synchronize()
print("nnz", out.nnz)
