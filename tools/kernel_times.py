"""Per-kernel times (CUDA events inside the C ABI) through a given libsa .so.
usage: python tools/kernel_times.py path/to/libsa.so [config | ds1 | ds2 | ds3]
(config = BASELINE cfg 1-5; dsK = the reference's standard dataset K)"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1406_1066_b200 import _capi, workloads as W
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _capi.SIGNATURES.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
ctx = ctypes.c_void_p(); lib.sa_create(0, ctypes.byref(ctx))
cfg = sys.argv[2] if len(sys.argv) > 2 else "2"
for kv in sys.argv[3:]:  # context options OPT=VAL
    o, v = kv.split("=")
    lib.sa_set_option(ctx, getattr(_capi, "SA_OPT_" + o), int(v))
if cfg.startswith("ds"):
    ii, jj, sv = W.ransparse(*W.ransparse_spec(int(cfg[2:])))
    w = W.Workload(cfg, torch.from_numpy(ii).cuda(), torch.from_numpy(jj).cuda(), torch.from_numpy(sv).cuda(), int(ii.max()), int(jj.max()))
else:
    cfg = int(cfg)
    w = W.config(cfg, device="cuda")
L, M, N = w.L, w.m, w.n
jc = torch.empty(N + 1, dtype=torch.int32, device="cuda"); ir = torch.empty(L, dtype=torch.int32, device="cuda"); pr = torch.empty(L, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream(); lib.sa_set_stream(ctx, ctypes.c_void_p(s.cuda_stream))
lib.sa_enable_timing(ctx, 1)
tot = {}
for it in range(12):
    lib.sa_assemble_async(ctx, w.ii.data_ptr(), w.jj.data_ptr(), w.s.data_ptr(), 1, L, M, N, jc.data_ptr(), ir.data_ptr(), pr.data_ptr(), L)
    arr = (ctypes.c_float * 16)(); names = (ctypes.c_char_p * 16)()
    n = lib.sa_last_kernel_times(ctx, 16, arr, names)
    if it >= 2:
        for k in range(n): tot.setdefault(names[k].decode(), []).append(arr[k])
print(sys.argv[1].split('/')[-1], 'cfg%s' % cfg, *sys.argv[3:], {k: round(sum(v)/len(v)*1e3, 1) for k, v in tot.items()})
