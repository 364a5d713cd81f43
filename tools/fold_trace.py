"""Per-tile timeline of k_tile_fold (library built with -DSA_TRACE).
usage: python tools/fold_trace.py path/to/libsa_trace.so [config | dsK]
Stamps: 0 start, 1 entries in (TMA), 2 networks done, 3 values in, 4 count
published, 5 values folded, 6 look-back done, 7 outputs written."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1406_1066_b200 import _capi, workloads as W
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _capi.SIGNATURES.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
ctx = ctypes.c_void_p(); lib.sa_create(0, ctypes.byref(ctx))
cfg = sys.argv[2] if len(sys.argv) > 2 else "2"
if cfg.startswith("ds"):
    ii, jj, sv = W.ransparse(*W.ransparse_spec(int(cfg[2:])))
    w = W.Workload(cfg, torch.from_numpy(ii).cuda(), torch.from_numpy(jj).cuda(), torch.from_numpy(sv).cuda(), int(ii.max()), int(jj.max()))
else:
    w = W.config(int(cfg), device="cuda")
L, M, N = w.L, w.m, w.n
jc = torch.empty(N + 1, dtype=torch.int32, device="cuda"); ir = torch.empty(L, dtype=torch.int32, device="cuda"); pr = torch.empty(L, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream(); lib.sa_set_stream(ctx, ctypes.c_void_p(s.cuda_stream))
for it in range(5):
    lib.sa_assemble_async(ctx, w.ii.data_ptr(), w.jj.data_ptr(), w.s.data_ptr(), 1, L, M, N, jc.data_ptr(), ir.data_ptr(), pr.data_ptr(), L)
torch.cuda.synchronize()
T = 1 << 15
buf = np.zeros((T, 8), np.uint64)
lib.sa_debug_ftrace(buf.ctypes.data, T)
nt = int((buf[:, 0] > 0).sum())
t = buf[:nt].astype(np.int64)
t0 = t[:, 0].min()
t = (t - t0) / 1000.0
print("tiles", nt, "kernel span us %.1f" % t[:, 7].max())
names = ["entries", "networks", "values", "publish", "fold", "lookback", "output"]
for k in range(1, 8):
    d = t[:, k] - t[:, k - 1]
    print(f"{names[k-1]:9s} mean {d.mean():6.2f} us  p50 {np.median(d):6.2f}  p90 {np.percentile(d, 90):6.2f}  max {d.max():7.2f}")
tot = t[:, 7] - t[:, 0]
print(f"{'total':9s} mean {tot.mean():6.2f} us  p50 {np.median(tot):6.2f}  p90 {np.percentile(tot, 90):6.2f}")
# ordering diagnostics: how far behind is the predecessor when a tile publishes?
st = t[:, 0]
pub = t[:, 4]
lag = pub[:-1] - pub[1:]          # predecessor publish - own publish (>0: predecessor later)
print("start order violations (tile starts before its predecessor): %.1f%%" % (100.0 * (st[1:] < st[:-1]).mean()))
print("predecessor publishes after me: %.1f%%, mean lag when late %.2f us" % (100.0 * (lag > 0).mean(), lag[lag > 0].mean() if (lag > 0).any() else 0.0))
