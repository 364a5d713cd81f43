"""Time the phases of the host-buffer path (upload / assemble / fetch)."""
import ctypes, time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1406_1066_b200 as sa
from paper_1406_1066_b200 import workloads as W
from paper_1406_1066_b200.assembly import _ptr

w = W.fem2d(1000)
L, M, N = w.L, w.m, w.n
hi = torch.empty(L, dtype=torch.int32, pin_memory=True); hi.copy_(w.ii)
hj = torch.empty(L, dtype=torch.int32, pin_memory=True); hj.copy_(w.jj)
hs = torch.empty(L, dtype=torch.float64, pin_memory=True); hs.copy_(w.s)
a = sa.default_assembler(0); lib, ctx = a.lib, a.ctx
def phases(out_kind):
    t0 = time.perf_counter()
    lib.sa_host_upload(ctx, hi.data_ptr(), hj.data_ptr(), hs.data_ptr(), 1, L)
    t1 = time.perf_counter()
    nnz = ctypes.c_int64(0); bp = ctypes.c_int64(); bw = ctypes.c_int()
    lib.sa_host_assemble(ctx, M, N, ctypes.byref(nnz), ctypes.byref(bp), ctypes.byref(bw))
    t2 = time.perf_counter()
    if out_kind == "pageable":
        jc = np.empty(N + 1, np.int32); ir = np.empty(nnz.value, np.int32); pr = np.empty(nnz.value, np.float64)
    elif out_kind == "pageable_touched":
        jc = np.zeros(N + 1, np.int32); ir = np.zeros(nnz.value, np.int32); pr = np.zeros(nnz.value, np.float64)
    else:
        jc = torch.empty(N + 1, dtype=torch.int32, pin_memory=True).numpy()
        ir = torch.empty(nnz.value, dtype=torch.int32, pin_memory=True).numpy()
        pr = torch.empty(nnz.value, dtype=torch.float64, pin_memory=True).numpy()
    t3 = time.perf_counter()
    lib.sa_host_fetch(ctx, _ptr(jc), _ptr(ir), _ptr(pr))
    t4 = time.perf_counter()
    return [round((b - a) * 1e3, 2) for a, b in ((t0, t1), (t1, t2), (t2, t3), (t3, t4), (t0, t4))], (jc, ir, pr)
for kind in ("pageable", "pageable_touched", "pinned", "pinned", "pageable"):
    for _ in range(2):
        ph, keep = phases(kind)
    print(kind, "upload/assemble/alloc/fetch/total ms:", ph)
