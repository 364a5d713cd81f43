"""Skewed inputs: a few very long columns (the big-column path).
usage: python tools/big_column_probe.py"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1406_1066_b200 as sa
from oracle import oracle as O
rng = np.random.default_rng(0)
a = sa.default_assembler(0)
for L, ncol, nrow in [(2_000_000, 1, 1_000_000), (10_000_000, 1, 1_000_000), (10_000_000, 20, 1_000_000),
                      (10_000_000, 1, 1000)]:
    ii = rng.integers(1, nrow + 1, size=L).astype(np.int32)
    jj = rng.integers(1, ncol + 1, size=L).astype(np.int32)
    s = rng.standard_normal(L)
    dev = torch.device('cuda', 0)
    ti, tj, ts = (torch.from_numpy(x).to(dev) for x in (ii, jj, s))
    out = a.assemble_device(ti, tj, ts, m=nrow, n=ncol)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = a.assemble_device(ti, tj, ts, m=nrow, n=ncol)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    a.lib.sa_enable_timing(a.ctx, 1)
    a.assemble_device(ti, tj, ts, m=nrow, n=ncol)
    arr = (ctypes.c_float * 16)(); names = (ctypes.c_char_p * 16)()
    k = a.lib.sa_last_kernel_times(a.ctx, 16, arr, names)
    a.lib.sa_enable_timing(a.ctx, 0)
    kt = {names[q].decode(): round(arr[q], 2) for q in range(k)}
    ok = out.to_host().same_as(O.assemble_counting(ii, jj, s, nrow, ncol)) 
    print(f"L={L} cols={ncol} rows={nrow}: {dt*1e3:.1f} ms, parity={ok}, kernels ms {kt}")
