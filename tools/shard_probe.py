"""Time sa_partition (the multi-GPU column-block partition) on one GPU (no
exchange): rank `rank`'s chunk of the weak-scaling mesh bench.py uses at
`world` GPUs (2D FEM, N = 1000 sqrt(world), contiguous cell chunks), column
blocks split evenly.
usage: python tools/shard_probe.py [world] [rank]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_1066_b200 as sa
from paper_1406_1066_b200.assembly import _ptr
import bench
world = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
w = bench.build_workload(2, "cuda", rank, world)
L, n = w.L, w.n
bounds = [n * r // world for r in range(world + 1)]
a = sa.default_assembler(0); a._bind_stream()
outs = [torch.empty(L, dtype=dt, device="cuda") for dt in (torch.int32, torch.int32, torch.float64)]
hb = (ctypes.c_int32 * (world + 1))(*bounds); hc = (ctypes.c_int64 * world)()
bp, bw = ctypes.c_int64(-1), ctypes.c_int(-1)
def run():
    rc = a.lib.sa_partition(a.ctx, _ptr(w.ii), _ptr(w.jj), _ptr(w.s), 1, L, w.m, n, world, rank, hb,
                            *(_ptr(x) for x in outs), hc, ctypes.byref(bp), ctypes.byref(bw))
    assert rc == 0, rc
for _ in range(3): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): run()
e1.record(); torch.cuda.synchronize()
print("world %d rank %d (L=%d): sa_partition %.3f ms (incl. host sync), counts %s"
      % (world, rank, L, e0.elapsed_time(e1) / 10, [hc[r] for r in range(world)]))
