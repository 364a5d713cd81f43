"""Dev check of the radix path (SA_OPT_PATH=1) against the C oracle, and
per-kernel times of both paths on BASELINE workloads.
usage: python tools/radix_check.py [--time CFG ...]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1406_1066_b200 as sa
from paper_1406_1066_b200 import _capi
from paper_1406_1066_b200 import workloads as W
from oracle import oracle as O


def same(a, b):
    return (np.array_equal(a.jc, b.jc) and np.array_equal(a.ir, b.ir)
            and np.asarray(a.pr).tobytes() == np.asarray(b.pr).tobytes())


def check(asm, w, name):
    dev = torch.device("cuda", 0)
    out = asm.assemble_device(w.ii.to(dev), w.jj.to(dev), w.s.to(dev), m=w.m, n=w.n).to_host()
    ref = O.assemble_counting(w.ii.cpu().numpy(), w.jj.cpu().numpy(), w.s.cpu().numpy(), w.m, w.n)
    ok = same(out, ref)
    print(f"{name:40s} L={w.L:>10d} nnz={ref.nnz:>10d} {'OK' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        print("  jc eq", np.array_equal(out.jc, ref.jc), "nnz", out.nnz, ref.nnz)
        if out.nnz == ref.nnz:
            d = np.flatnonzero((out.ir != ref.ir) | (out.pr.view(np.uint64) != ref.pr.view(np.uint64)))
            print("  first diffs", d[:10], out.ir[d[:5]], ref.ir[d[:5]], out.pr[d[:5]], ref.pr[d[:5]])
    return ok


def times(asm, w, path, reps=5):
    lib, ctx = asm.lib, asm.ctx
    asm.set_option(_capi.SA_OPT_PATH, path)
    dev = torch.device("cuda", 0)
    L = w.L
    jc = torch.empty(w.n + 1, dtype=torch.int32, device=dev)
    ir = torch.empty(L, dtype=torch.int32, device=dev)
    pr = torch.empty(L, dtype=torch.float64, device=dev)
    asm._bind_stream()

    def step():
        rc = lib.sa_assemble_async(ctx, w.ii.data_ptr(), w.jj.data_ptr(), w.s.data_ptr(), 1, L, w.m, w.n,
                                   jc.data_ptr(), ir.data_ptr(), pr.data_ptr(), L)
        assert rc == 0, asm._msg()
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    lib.sa_enable_timing(ctx, 1)
    step()
    arr = (ctypes.c_float * 16)()
    names = (ctypes.c_char_p * 16)()
    nk = lib.sa_last_kernel_times(ctx, 16, arr, names)
    lib.sa_enable_timing(ctx, 0)
    kt = {names[k].decode(): round(arr[k], 3) for k in range(nk)}
    nnz = ctypes.c_int64(0)
    lib.sa_finish(ctx, ctypes.byref(nnz), None, None)
    print(f"  path={path} {w.name}: {ms:.3f} ms/step ({L / ms / 1e6:.2f} G triplets/s) nnz={nnz.value} {kt}",
          flush=True)


def main():
    asm = sa.default_assembler(0)
    asm.set_option(_capi.SA_OPT_PATH, 1)
    dev = torch.device("cuda", 0)
    ok = True
    ok &= check(asm, W.random_coo(), "cfg1 random_coo")
    ok &= check(asm, W.random_coo(m=7, n=5, L=300_000, seed=3), "tiny dims, long runs")
    ok &= check(asm, W.random_coo(m=2_000_000, n=1, L=50_000, seed=4), "single column (oversize)")
    ok &= check(asm, W.random_coo(m=3, n=200_000, L=2_000_000, seed=5), "3 rows, wide")
    ok &= check(asm, W.heavy_dup(m=20_000, positions=200_000), "heavy_dup small")
    ok &= check(asm, W.fem2d(64), "fem2d 64")
    ok &= check(asm, W.fem3d(20), "fem3d 20")
    ok &= check(asm, W.random_coo(m=1_000_000, n=1, L=2_000_000, seed=6), "one long column (row split)")
    ok &= check(asm, W.random_coo(m=1_000_000, n=20, L=3_000_000, seed=7), "20 long columns (row split)")
    ok &= check(asm, W.random_coo(m=1000, n=1, L=2_000_000, seed=8), "one column, 1000 rows")
    ok &= check(asm, W.random_coo(m=5_000_000, n=3, L=1_500_000, seed=9), "3 columns, sparse rows")
    ok &= check(asm, W.config(4, scale=0.02), "cfg4 x0.02")
    ok &= check(asm, W.config(2, device=dev), "cfg2 full")
    ok &= check(asm, W.config(3, device=dev), "cfg3 full")
    ok &= check(asm, W.config(4, device=dev, scale=0.1), "cfg4 x0.1")
    print("ALL OK" if ok else "FAILURES", flush=True)
    for k in [int(x) for x in sys.argv[sys.argv.index("--time") + 1:]] if "--time" in sys.argv else []:
        w = W.config(k, device=dev)
        for path in (0, 1):
            times(asm, w, path)
        del w
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
