"""Per-sub-bucket phase times of k_rfold (library built with -DSA_RTRACE=1), in SM cycles.
usage: python tools/rfold_trace.py path/to/libsa_trace.so [config]
Stamps: 0 start, 1 keys in + tables cleared, 2 groups hashed, 3 member/column starts,
4 members + column lists placed, 5 groups ranked, 6 look-back done, 7 values staged,
9 groups folded + jc written (8 unused)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1406_1066_b200 import _capi, workloads as W
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _capi.SIGNATURES.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
ctx = ctypes.c_void_p(); lib.sa_create(0, ctypes.byref(ctx))
w = W.config(int(sys.argv[2]) if len(sys.argv) > 2 else 4, device="cuda")
L, M, N = w.L, w.m, w.n
jc = torch.empty(N + 1, dtype=torch.int32, device="cuda"); ir = torch.empty(L, dtype=torch.int32, device="cuda"); pr = torch.empty(L, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream(); lib.sa_set_stream(ctx, ctypes.c_void_p(s.cuda_stream))
for it in range(3):
    lib.sa_assemble_async(ctx, w.ii.data_ptr(), w.jj.data_ptr(), w.s.data_ptr(), 1, L, M, N, jc.data_ptr(), ir.data_ptr(), pr.data_ptr(), L)
torch.cuda.synchronize()
T = 1 << 15
buf = np.zeros((T, 10), np.int64)
lib.sa_debug_rtrace.restype = ctypes.c_int; lib.sa_debug_rtrace.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.sa_debug_rtrace(buf.ctypes.data, T)
t = buf[1000:]  # skip the first wave
names = ["keys+clear", "hash groups", "starts/scan", "members+lists", "rank", "lookback", "values", "fold+jc"]
t = np.delete(t, 8, axis=1)
tot = (t[:, 8] - t[:, 0]).astype(np.float64)
print("sub-buckets", len(t), "total cycles mean %.0f p50 %.0f p90 %.0f" % (tot.mean(), np.median(tot), np.percentile(tot, 90)))
for k in range(1, 9):
    d = (t[:, k] - t[:, k - 1]).astype(np.float64)
    print(f"{names[k-1]:14s} mean {d.mean():7.0f}  p50 {np.median(d):7.0f}  p90 {np.percentile(d, 90):7.0f}  share {100*d.mean()/tot.mean():5.1f} %")
