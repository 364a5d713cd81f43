"""Host logic of the multi-GPU column-block assembly (paper_1406_1066_b200/
distributed.py) with world_size 2 on CPU (gloo): the concatenation of the
ranks' column blocks must equal the single-process oracle bit for bit.  The
local assembler here is the CPU oracle (test infrastructure); on GPUs it is
the CUDA pipeline (distributed.gpu_local_assembler)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_local(ii, jj, s, m, n_local):
    from oracle import oracle as O

    out = O.assemble_counting(ii.numpy(), jj.numpy(), s.numpy(), m, n_local)
    return torch.from_numpy(out.jc), torch.from_numpy(out.ir), torch.from_numpy(out.pr)


def _case(kind):
    from paper_1406_1066_b200 import workloads as W
    from instances import random_triplets

    if kind == "fem2d":
        w = W.fem2d(24)
        return w.ii.numpy(), w.jj.numpy(), w.s.numpy(), w.m, w.n
    if kind == "fem3d":
        w = W.fem3d(5)
        return w.ii.numpy(), w.jj.numpy(), w.s.numpy(), w.m, w.n
    if kind == "heavy":
        w = W.heavy_dup(m=500, positions=3000, seed=2)
        return w.ii.numpy(), w.jj.numpy(), w.s.numpy(), w.m, w.n
    ii, jj, s = random_triplets(1_000_777, max_len=20_000, max_dim=300)
    ii, jj = ii.astype(np.int32), jj.astype(np.int32)
    return ii, jj, s, int(ii.max(initial=0)), int(jj.max(initial=0))


def _worker(rank, world, port, kind, result_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    from paper_1406_1066_b200.distributed import assemble_sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        ii, jj, s, m, n = _case(kind)
        L = len(ii)
        lo, hi = L * rank // world, L * (rank + 1) // world
        res = assemble_sharded(torch.from_numpy(ii[lo:hi].copy()), torch.from_numpy(jj[lo:hi].copy()),
                               torch.from_numpy(s[lo:hi].copy()), m, n, _oracle_local, nblocks=64)
        result_q.put((rank, res.col_lo, res.col_hi, res.jc.numpy(), res.ir.numpy(), res.pr.numpy(),
                      res.nnz_offset, res.nnz_total, res.sent_remote))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["fem2d", "fem3d", "heavy", "random"])
def test_two_rank_column_blocks_match_single_process(kind):
    from oracle import oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=180) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ii, jj, s, m, n = _case(kind)
    ref = O.assemble_counting(ii, jj, s, m, n)
    # stitch the column blocks back together
    jc = [0]
    ir, pr = [], []
    assert got[0][1] == 0 and got[-1][2] == n
    for rank, lo, hi, bjc, bir, bpr, off, tot, _ in got:
        assert bjc[0] == off and tot == ref.nnz
        jc.extend(bjc[1:].tolist())
        ir.append(bir)
        pr.append(bpr)
    assert np.array_equal(np.array(jc), ref.jc)
    assert np.array_equal(np.concatenate(ir), ref.ir)
    assert np.concatenate(pr).tobytes() == ref.pr.tobytes()
    if kind in ("fem2d", "fem3d"):
        # element order keeps most triplets local
        sent = sum(g[-1] for g in got)
        assert sent < 0.25 * len(ii)


def test_block_boundaries_balance():
    from paper_1406_1066_b200.distributed import block_boundaries

    hist = torch.tensor([10, 0, 30, 10, 50, 0, 0, 100], dtype=torch.int64)
    b = block_boundaries(hist, 4, 8, 80)
    assert b[0] == 0 and b[-1] == 80 and all(x <= y for x, y in zip(b, b[1:]))
    b1 = block_boundaries(torch.zeros(8, dtype=torch.int64), 2, 8, 80)
    assert b1 == [0, 40, 80]


def _bounce_collectives():
    """gloo collectives for CUDA tensors, bounced through host memory (the
    CUDA-path test below runs several ranks on the one GPU; NCCL refuses two
    ranks on one device).  Only the transport changes; the CUDA kernels of
    each rank run on their own and never wait on another rank's."""
    orig = {k: getattr(dist, k) for k in ("all_reduce", "all_to_all_single", "all_gather")}

    def all_reduce(t, *a, **k):
        c = t.cpu()
        r = orig["all_reduce"](c, *a, **k)
        t.copy_(c)
        return r

    def all_to_all_single(out, inp, *a, **k):
        c = out.cpu()
        r = orig["all_to_all_single"](c, inp.cpu(), *a, **k)
        out.copy_(c)
        return r

    def all_gather(lst, t, *a, **k):
        cl = [x.cpu() for x in lst]
        r = orig["all_gather"](cl, t.cpu(), *a, **k)
        for x, c in zip(lst, cl):
            x.copy_(c)
        return r

    dist.all_reduce, dist.all_to_all_single, dist.all_gather = all_reduce, all_to_all_single, all_gather


def _gpu_worker(rank, world, port, kind, result_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    from paper_1406_1066_b200.distributed import assemble_sharded, gpu_local_assembler

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    _bounce_collectives()
    try:
        ii, jj, s, m, n = _case(kind)
        L = len(ii)
        lo, hi = L * rank // world, L * (rank + 1) // world
        dev = torch.device("cuda", 0)
        t = [torch.from_numpy(x[lo:hi].copy()).to(dev) for x in (ii, jj, s)]
        out = {}
        for _ in range(2):  # the second call reuses the scratch and result buffers
            res = assemble_sharded(*t, m, n, gpu_local_assembler(0), nblocks=64, out=out)
        result_q.put((rank, res.col_lo, res.col_hi, res.jc.cpu().numpy(), res.ir.cpu().numpy(),
                      res.pr.cpu().numpy(), res.nnz_offset, res.nnz_total, res.sent_remote))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("kind,world", [("fem2d", 2), ("fem3d", 3), ("heavy", 2), ("heavy", 3),
                                        ("random", 2)])
def test_cuda_sharded_path_matches_single_process(kind, world):
    """assemble_sharded's CUDA branch (sa_block_histogram, sa_partition,
    exchange, sa_assemble_segments_async over the received and own
    segments, jc offsets) with `world` ranks on the one GPU: the stitched
    column blocks equal the single-process oracle bit for bit."""
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ii, jj, s, m, n = _case(kind)
    ref = O.assemble_counting(ii, jj, s, m, n)
    jc = [0]
    ir, pr = [], []
    assert got[0][1] == 0 and got[-1][2] == n
    for rank, lo, hi, bjc, bir, bpr, off, tot, _ in got:
        assert bjc[0] == off and tot == ref.nnz
        jc.extend(bjc[1:].tolist())
        ir.append(bir)
        pr.append(bpr)
    assert np.array_equal(np.array(jc), ref.jc)
    assert np.array_equal(np.concatenate(ir), ref.ir)
    assert np.concatenate(pr).tobytes() == ref.pr.tobytes()
    if kind == "heavy":  # shuffled input: the exchange moved triplets both ways
        assert all(g[-1] > 0 for g in got)


def _err_case(kind):
    """A fem2d input with one invalid index planted in the LAST rank's chunk
    (and, for "both", a bad column earlier in rank 0's chunk as well)."""
    from paper_1406_1066_b200 import workloads as W

    w = W.fem2d(24)
    ii, jj, s = w.ii.numpy().copy(), w.jj.numpy().copy(), w.s.numpy().copy()
    L = len(ii)
    m, n = w.m, w.n
    if kind == "row":
        ii[L - 7] = 0
    elif kind == "both":  # rows are checked before columns, over the whole input
        jj[5] = -3
        ii[L - 7] = 0
    elif kind == "col":
        jj[L - 100] = 0
    elif kind == "dim":
        jj[L - 3] = n + 5
    return ii, jj, s, m, n


def _err_worker(rank, world, port, kind, cuda, result_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    from paper_1406_1066_b200.distributed import assemble_sharded, gpu_local_assembler
    from paper_1406_1066_b200.errors import BadIndex, DimensionTooSmall

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    if cuda:
        _bounce_collectives()
    try:
        ii, jj, s, m, n = _err_case(kind)
        L = len(ii)
        lo, hi = L * rank // world, L * (rank + 1) // world
        t = [torch.from_numpy(x[lo:hi].copy()) for x in (ii, jj, s)]
        if cuda:
            t = [x.to(torch.device("cuda", 0)) for x in t]
            local = gpu_local_assembler(0)
        else:
            local = _oracle_local
        try:
            assemble_sharded(*t, m, n, local, nblocks=64)
            result_q.put((rank, "none", None, None))
        except BadIndex as e:
            result_q.put((rank, "BadIndex", e.position, e.value))
        except DimensionTooSmall:
            result_q.put((rank, "DimensionTooSmall", None, None))
    finally:
        dist.destroy_process_group()


def _run_err(kind, world, cuda):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_err_worker, args=(r, world, port, kind, cuda, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


def _expected_err(kind):
    """What the one-process reference validation raises (types.py:141-165)."""
    ii, jj, s, m, n = _err_case(kind)
    bad_i = np.flatnonzero(ii < 1)
    bad_j = np.flatnonzero(jj < 1)
    if len(bad_i):
        return ("BadIndex", int(bad_i[0]), int(ii[bad_i[0]]))
    if len(bad_j):
        return ("BadIndex", int(bad_j[0]), int(jj[bad_j[0]]))
    return ("DimensionTooSmall", None, None)


@pytest.mark.parametrize("kind", ["row", "both", "col", "dim"])
def test_validation_error_raised_on_every_rank(kind):
    """an invalid index in one rank's chunk must not leave the
    other ranks blocked in the exchange.  Every rank raises the exception the
    one-process call raises, with the GLOBAL position (rows before columns,
    reference types.py:161-162) and the offending value."""
    got = _run_err(kind, 2, cuda=False)
    exp = _expected_err(kind)
    assert [g[1:] for g in got] == [exp, exp]


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["row", "both", "dim"])
def test_cuda_validation_error_raised_on_every_rank(kind):
    """The same through sa_partition (the CUDA branch, ranks on one GPU)."""
    got = _run_err(kind, 2, cuda=True)
    exp = _expected_err(kind)
    assert [g[1:] for g in got] == [exp, exp]
