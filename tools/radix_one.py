"""One radix-path assembly of BASELINE config K (for ncu): python tools/radix_one.py K [path]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_1066_b200 as sa
from paper_1406_1066_b200 import _capi, workloads as W
k = int(sys.argv[1]); path = int(sys.argv[2]) if len(sys.argv) > 2 else 1
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
a = sa.default_assembler(0)
a.set_option(_capi.SA_OPT_PATH, path)
w = W.config(k, device=torch.device("cuda", 0), scale=scale)
for _ in range(2):
    out = a.assemble_device(w.ii, w.jj, w.s, m=w.m, n=w.n)
torch.cuda.synchronize()
print("nnz", out.nnz)
