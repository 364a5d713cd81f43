"""Skewed inputs: a heavy hitter (one (row, col) entry holding a large share of the triplets).
usage: python tools/heavy_hitter_probe.py path/to/libsa.so"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1406_1066_b200 import _capi
from oracle import oracle as O
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _capi.SIGNATURES.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
ctx = ctypes.c_void_p(); lib.sa_create(0, ctypes.byref(ctx))
rng = np.random.default_rng(3)
for L, m, n, share in [(4_000_000, 1_000_000, 1_000_000, 0.5), (10_000_000, 1_000_000, 1_000_000, 0.1), (4_000_000, 2000, 2000, 0.25)]:
    ii = rng.integers(1, m + 1, size=L).astype(np.int32)
    jj = rng.integers(1, n + 1, size=L).astype(np.int32)
    hot = rng.random(L) < share
    ii[hot] = 7; jj[hot] = min(n, 123456)
    s = rng.standard_normal(L)
    ti, tj, ts = (torch.from_numpy(x).cuda() for x in (ii, jj, s))
    jc = torch.empty(n + 1, dtype=torch.int32, device="cuda"); ir = torch.empty(L, dtype=torch.int32, device="cuda"); pr = torch.empty(L, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream(); lib.sa_set_stream(ctx, ctypes.c_void_p(st.cuda_stream))
    lib.sa_enable_timing(ctx, 1)
    for it in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rc = lib.sa_assemble_async(ctx, ti.data_ptr(), tj.data_ptr(), ts.data_ptr(), 1, L, m, n, jc.data_ptr(), ir.data_ptr(), pr.data_ptr(), L)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    arr = (ctypes.c_float * 16)(); names = (ctypes.c_char_p * 16)()
    k = lib.sa_last_kernel_times(ctx, 16, arr, names)
    kt = {names[q].decode(): round(arr[q], 2) for q in range(k)}
    ref = O.assemble_counting(ii, jj, s, m, n)
    nnz = int(jc[-1].item())
    ok = (nnz == ref.nnz and np.array_equal(jc.cpu().numpy(), ref.jc) and np.array_equal(ir[:nnz].cpu().numpy(), ref.ir)
          and pr[:nnz].cpu().numpy().tobytes() == np.asarray(ref.pr).tobytes())
    print(f"L={L} m={m} n={n} hot share={share}: rc={rc} {dt*1e3:.1f} ms parity={ok} kernels ms {kt}", flush=True)
