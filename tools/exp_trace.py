"""Per-CTA timeline of k_col_scan (library built with -DSA_TRACE):
usage: python tools/exp_trace.py path/to/libsa_trace.so [config]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1406_1066_b200 import _capi, workloads as W
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _capi.SIGNATURES.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
ctx = ctypes.c_void_p(); lib.sa_create(0, ctypes.byref(ctx))
w = W.config(int(sys.argv[2]) if len(sys.argv) > 2 else 2, device="cuda")
L, M, N = w.L, w.m, w.n
jc = torch.empty(N + 1, dtype=torch.int32, device="cuda"); ir = torch.empty(L, dtype=torch.int32, device="cuda"); pr = torch.empty(L, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream(); lib.sa_set_stream(ctx, ctypes.c_void_p(s.cuda_stream))
for it in range(5):
    lib.sa_assemble_async(ctx, w.ii.data_ptr(), w.jj.data_ptr(), w.s.data_ptr(), 1, L, M, N, jc.data_ptr(), ir.data_ptr(), pr.data_ptr(), L)
torch.cuda.synchronize()
G = (N + 2047) // 2048
buf = np.zeros((1 << 16, 4), np.uint64)
print("copy", lib.sa_debug_trace(buf.ctypes.data, 1 << 16))
t = buf[:G] & ((1 << 54) - 1)
sm = buf[:G, 0] >> 54
t0 = t[:, 0].min()
t = (t.astype(np.int64) - int(t0)) / 1000.0
print("G", G, "kernel span us", t[:, 3].max())
for q in [0, 1, 2, 50, 100, 200, 400, 591, 592, 600, 800, G - 1]:
    if q < G: print(q, "sm", sm[q], "start %.2f agg %.2f incl %.2f end %.2f" % tuple(t[q]))
print("wait (incl-agg) mean %.2f max %.2f" % ((t[:, 2] - t[:, 1]).mean(), (t[:, 2] - t[:, 1]).max()))
print("load (agg-start) mean %.2f max %.2f" % ((t[:, 1] - t[:, 0]).mean(), (t[:, 1] - t[:, 0]).max()))
print("write (end-incl) mean %.2f max %.2f" % ((t[:, 3] - t[:, 2]).mean(), (t[:, 3] - t[:, 2]).max()))
