"""Step time and per-kernel times of BASELINE configs under context-option
variants (dev A/B tool).  usage: python tools/variant_time.py CFG[,CFG..] [OPT=VAL ...]
e.g. python tools/variant_time.py 5 SCATTER_STAGED=0 SCATTER_STAGED=1 PATH=1,RPASS_TMA=1"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_1066_b200 as sa
from paper_1406_1066_b200 import _capi, workloads as W

asm = sa.default_assembler(0)
lib, ctx = asm.lib, asm.ctx
dev = torch.device("cuda", 0)
variants = [None] + [[kv.split("=") for kv in v.split(",")] for v in sys.argv[2:]]
for cfg in [int(c) for c in sys.argv[1].split(",")]:
    w = W.config(cfg, device=dev)
    L = w.L
    jc = torch.empty(w.n + 1, dtype=torch.int32, device=dev)
    ir = torch.empty(L, dtype=torch.int32, device=dev)
    pr = torch.empty(L, dtype=torch.float64, device=dev)
    asm._bind_stream()
    for var in variants:
        for o, v in (var or []):
            asm.set_option(getattr(_capi, "SA_OPT_" + o), int(v))
        def step():
            rc = lib.sa_assemble_async(ctx, w.ii.data_ptr(), w.jj.data_ptr(), w.s.data_ptr(), 1, L, w.m, w.n,
                                       jc.data_ptr(), ir.data_ptr(), pr.data_ptr(), L)
            assert rc == 0, asm._msg()
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        reps = 10 if L < 3e8 else 4
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        lib.sa_enable_timing(ctx, 1)
        kt = {}
        for _ in range(3):
            step()
            arr = (ctypes.c_float * 16)(); names = (ctypes.c_char_p * 16)()
            nk = lib.sa_last_kernel_times(ctx, 16, arr, names)
            for k in range(nk):
                kt.setdefault(names[k].decode(), []).append(arr[k])
        lib.sa_enable_timing(ctx, 0)
        nnz = ctypes.c_int64(0)
        rc = lib.sa_finish(ctx, ctypes.byref(nnz), None, None)
        tag = ",".join("=".join(x) for x in var) if var else "auto"
        print(f"cfg{cfg} {tag:22s} {ms:8.3f} ms  nnz={nnz.value} rc={rc} "
              + " ".join(f"{k}={sum(v)/len(v):.3f}" for k, v in kt.items()), flush=True)
        for o, v in (var or []):
            asm.set_option(getattr(_capi, "SA_OPT_" + o), -1)
    del w, jc, ir, pr
    torch.cuda.empty_cache()
