"""Host-side cost of one sharded step (distributed.assemble_sharded) without
the collectives, on one GPU (boundaries: the even split the global
histogram gives for these meshes): rank `rank` of `world` on the weak-scaling mesh
chunk bench.py uses.  Phases: sampled block histogram, boundaries (host),
sa_partition (+ host read of the counts), segment assembly of the own chunk
(+ sa_finish).  The NCCL exchange is replaced by "nothing received".
usage: python tools/shard_step_probe.py [world] [rank] [OPT=VAL ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1406_1066_b200 import distributed as D
from paper_1406_1066_b200.assembly import default_assembler
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = bench.build_workload(2, "cuda", rank, world)
M, N = w.m, w.n
asm = default_assembler(0); asm._bind_stream()
from paper_1406_1066_b200 import _capi
for kv in sys.argv[3:]:
    o, v = kv.split("=")
    asm.set_option(getattr(_capi, "SA_OPT_" + o), int(v))
ii, jj, s = w.ii, w.jj, w.s
OUT = {}
EV = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
def step(t):
    EV[0].record()
    t.append(("start", time.perf_counter()))
    nblocks = 4096; bsize = (N + nblocks - 1) // nblocks
    st = max(1, len(jj) >> 20)
    hist = D._block_hist_cuda(asm, jj, nblocks, bsize, st)
    D.block_boundaries(hist, world, nblocks, N)  # (cost only: one rank's histogram
    # is not the global one -- the meshes' global histogram splits evenly)
    bounds = [N * r // world for r in range(world + 1)]
    t.append(("hist+bounds", time.perf_counter()))
    EV[1].record()
    parts, counts, _err = D._partition_cuda(asm, ii, jj, s, M, N, bounds, world, rank)
    t.append(("partition", time.perf_counter()))
    EV[2].record()
    col_lo, col_hi = bounds[rank], bounds[rank + 1]
    out = D._assemble_segments_cuda(asm, [(ii, jj, s)], col_lo, M, col_hi - col_lo, OUT)
    t.append(("assemble+finish", time.perf_counter()))
    EV[3].record()
for _ in range(3): step([])
torch.cuda.synchronize()
acc = {}
R = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(R):
    t = []
    step(t)
    for (a, ta), (b, tb) in zip(t, t[1:]):
        acc[b] = acc.get(b, 0) + (tb - ta) / R
    torch.cuda.synchronize()
    for k, name in enumerate(("dev:hist+bounds", "dev:partition", "dev:assemble+finish")):
        acc[name] = acc.get(name, 0) + EV[k].elapsed_time(EV[k + 1]) * 1e-3 / R
e1.record(); torch.cuda.synchronize()
print("world %d rank %d: device %.3f ms/step; host phases (ms): %s" % (
    world, rank, e0.elapsed_time(e1) / R, {k: round(v * 1e3, 3) for k, v in acc.items()}))
