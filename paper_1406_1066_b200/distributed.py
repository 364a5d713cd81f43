"""Multi-GPU assembly by column block: one process per GPU.

Each rank holds a contiguous chunk of the global triplet stream (chunks in
rank order = input order).  Per call:

1. every rank histograms (a strided sample of) its triplets into
   ``nblocks`` equal column blocks; one ``all_reduce`` gives the global block
   histogram;
2. contiguous column ranges are assigned to ranks so that each receives about
   L / world triplets (block granularity);
3. each rank partitions its chunk by destination rank, *stably* (the CUDA
   kernels of sa_partition, validating the chunk on the way); only the
   triplets bound for other ranks are written and moved by ``all_to_all``
   (element-ordered FEM keeps ~99.9 % at home);
   a rank concatenates what it receives in source-rank order, which is the
   global input order restricted to its columns -- so duplicates are still
   folded in input order and the result is bit-identical to one GPU;
4. the rank assembles its column block with the single-GPU pipeline reading
   three segments in place -- received from lower ranks, its own chunk
   (other ranks' columns skipped), received from higher ranks -- which is
   the global input order restricted to its columns (bit-identical to one
   GPU); an ``all_gather`` of the per-rank nnz gives the offset of its ``jc``.

The collectives are plain data movement (NCCL over NVLink for CUDA tensors,
gloo for CPU tests); the local assembly is the caller-supplied assembler (the
CUDA pipeline in production).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class ShardResult:
    """Rank-local column block [col_lo, col_hi) of the global CSC matrix."""

    col_lo: int
    col_hi: int
    jc: torch.Tensor        # int64 [col_hi - col_lo + 1], global offsets
    ir: torch.Tensor        # int32 [nnz_local], 0-based rows
    pr: torch.Tensor        # float64 [nnz_local]
    nnz_offset: int         # global position of this block's first entry
    nnz_total: int
    m: int
    n: int
    recv_triplets: int      # triplets assembled here after the exchange
    sent_remote: int        # triplets this rank sent to other ranks
    launches: int = 0       # CUDA kernels this rank launched (partition + assembly)


def block_boundaries(block_hist: torch.Tensor, world: int, nblocks: int, n: int):
    """Split nblocks column blocks into `world` contiguous ranges with about
    equal triplet counts.  Returns (world+1) column boundaries (int list)."""
    import numpy as np

    cum = np.cumsum(block_hist.to(torch.int64).cpu().numpy())
    total = int(cum[-1]) if len(cum) else 0
    bsize = (n + nblocks - 1) // nblocks
    targets = np.array([(total * r) // world for r in range(1, world)], dtype=np.int64)
    # first block whose cumulative count reaches each target
    ks = np.searchsorted(cum, targets, side="left") if len(cum) else np.zeros(0, dtype=np.int64)
    bounds = [0]
    for r in range(1, world):
        col = min(n, (int(ks[r - 1]) + 1) * bsize) if total else (n * r) // world
        bounds.append(max(bounds[-1], col))
    bounds.append(n)
    return bounds


def validate_torch(ii, jj, m, n):
    """Host restatement of sa_partition's index checks (CPU tensors): the
    first row index < 1, else the first column index < 1 (rows before
    columns, reference types.py:161-162), else whether any index exceeds the
    explicit dimensions (DimensionTooSmall, types.py:113-117).  Returns
    (which, local position, value) or ("dim", -1, None) or None."""
    for which, x in (("row", ii), ("col", jj)):
        bad = torch.nonzero(x < 1)
        if len(bad):
            k = int(bad[0, 0])
            return which, k, int(x[k])
    if (len(ii) and int(ii.max()) > m) or (len(jj) and int(jj.max()) > n):
        return "dim", -1, None
    return None


def partition_torch(ii, jj, s, bounds, world, self_rank=-1):
    """Host restatement of sa_partition (CPU tensors: the gloo tests; the
    index checks are validate_torch).  Returns ((i, j, s) of the triplets
    bound for ranks other than `self_rank`, grouped by destination rank,
    stably; per-rank counts including the rank's own).  Columns outside
    [1, bounds[-1]] go nowhere."""
    jj64 = jj.to(torch.int64)
    bt = torch.tensor(bounds[1:-1], dtype=torch.int64, device=jj.device)
    valid = (jj64 >= 1) & (jj64 <= bounds[-1])
    dest = torch.searchsorted(bt, jj64 - 1, right=True)
    dest = torch.where(valid, dest, torch.full_like(dest, world))
    counts = torch.bincount(dest, minlength=world + 1)[:world]
    if 0 <= self_rank < world:
        dest = torch.where(dest == self_rank, torch.full_like(dest, world), dest)
    key = dest.to(torch.uint8) if world < 255 else dest
    order = torch.sort(key, stable=True).indices
    keep = order[: int((dest < world).sum())]
    sv = s.expand(len(jj)) if s.numel() == 1 and len(jj) != 1 else s
    out = (ii[keep].contiguous(), jj[keep].contiguous(), sv[keep].contiguous())
    return out, [int(c) for c in counts.tolist()]


# error words exchanged with the counts: [kind, which, global position, value]
_OK, _BAD, _DIM, _DEV = 0, 1, 2, 3
_NONE = 1 << 62


def _error_word(err, chunk_off):
    """The rank's validation outcome as 4 int64: kind, which (0 row, 1 col),
    GLOBAL position (chunk offset + local position), offending value."""
    if err is None:
        return [_OK, 0, _NONE, 0]
    which, pos, val = err
    if which == "dim":
        return [_DIM, 0, _NONE, 0]
    if which == "dev":
        return [_DEV, 0, _NONE, int(pos)]
    return [_BAD, 0 if which == "row" else 1, chunk_off + int(pos), int(val)]


def _raise_agreed(words):
    """Every rank gets every rank's error word and raises the same exception
    the one-process call would: the first bad row over the whole input, else
    the first bad column, else DimensionTooSmall (reference validation order,
    types.py:141-165 then effective_dims 113-117)."""
    from .errors import BadIndex, DeviceError, DimensionTooSmall

    bad = [w for w in words if w[0] == _BAD]
    if bad:
        w = min(bad, key=lambda w: (w[1], w[2]))
        raise BadIndex(int(w[2]), int(w[3]))
    if any(w[0] == _DIM for w in words):
        raise DimensionTooSmall("indices exceed the explicit dimensions")
    dev = [w for w in words if w[0] == _DEV]
    if dev:
        raise DeviceError(int(dev[0][3]), "sa_partition failed on a peer rank")


def _scratch(asm, name, n, dtype, dev):
    """A reusable device buffer of at least n elements kept on the assembler
    (allocating 10^8-byte tensors per call costs ~0.1 ms of host time)."""
    cache = asm.__dict__.setdefault("_shard_scratch", {})
    buf = cache.get(name)
    if buf is None or buf.numel() < n or buf.dtype != dtype or buf.device != dev:
        buf = cache[name] = torch.empty(max(int(n * 1.25), 1), dtype=dtype, device=dev)
    return buf[:n]


def _block_hist_cuda(asm, jj, nblocks, bsize, step):
    """sa_block_histogram: the sampled column-block histogram in one launch."""
    from .assembly import _ptr

    hist = _scratch(asm, "hist", nblocks, torch.int64, jj.device)
    rc = asm.lib.sa_block_histogram(asm.ctx, _ptr(jj), int(jj.shape[0]), step, nblocks, bsize, _ptr(hist))
    if rc:
        asm._raise(rc)
    return hist


def _partition_cuda(asm, ii, jj, s, m, n, bounds, world, self_rank):
    """sa_partition: the CUDA partition, validating the chunk on the way.
    Returns (outputs, counts, err): the outputs are views of buffers reused
    across calls (valid until the next call on this assembler); err is None
    or (which, chunk-local position, value) / ("dim", -1, None) -- not
    raised here, so that every rank can raise the same exception after the
    count exchange (a rank raising alone would leave its peers blocked in
    the collective)."""
    import ctypes

    from . import _capi
    from .assembly import _ptr

    dev = ii.device
    L = len(ii)
    outs = (_scratch(asm, "pi", max(L, 1), torch.int32, dev), _scratch(asm, "pj", max(L, 1), torch.int32, dev),
            _scratch(asm, "ps", max(L, 1), torch.float64, dev))
    hb = (ctypes.c_int32 * (world + 1))(*bounds)
    hc = (ctypes.c_int64 * world)()
    bp, bw = ctypes.c_int64(-1), ctypes.c_int(-1)
    rc = asm.lib.sa_partition(asm.ctx, _ptr(ii), _ptr(jj), _ptr(s),
                              0 if (s.numel() == 1 and L != 1) else 1, L, m, n, world, self_rank, hb,
                              _ptr(outs[0]), _ptr(outs[1]), _ptr(outs[2]), hc, ctypes.byref(bp),
                              ctypes.byref(bw))
    err = None
    if rc == _capi.SA_ERR_BAD_INDEX:
        row = bw.value == _capi.SA_WHICH_ROW
        arr = ii if row else jj
        err = ("row" if row else "col", bp.value, int(arr[bp.value].item()))
    elif rc == _capi.SA_ERR_DIM_TOO_SMALL:
        err = ("dim", -1, None)
    elif rc:
        err = ("dev", rc, None)
    counts = [0] * world if err else [int(hc[r]) for r in range(world)]
    k = sum(c for r, c in enumerate(counts) if r != self_rank)
    return tuple(x[:k] for x in outs), counts, err


def _assemble_segments_cuda(asm, segs, col_lo, m, n_local, out=None):
    """sa_assemble_segments_async over [(ii, jj, s), ...] read in place.
    `out` (a dict) keeps the jc / ir / pr buffers across calls."""
    import ctypes

    from .assembly import DeviceCsc, _ptr

    dev = segs[0][0].device
    k = len(segs)
    pi = (ctypes.c_void_p * k)(*[_ptr(x[0]) for x in segs])
    pj = (ctypes.c_void_p * k)(*[_ptr(x[1]) for x in segs])
    ps = (ctypes.c_void_p * k)(*[_ptr(x[2]) for x in segs])
    lens = [int(x[0].shape[0]) for x in segs]
    st = (ctypes.c_int64 * k)(*[0 if (x[2].numel() == 1 and n_ != 1) else 1 for x, n_ in zip(segs, lens)])
    ln = (ctypes.c_int64 * k)(*lens)
    cap = max(sum(lens), 1)
    if out is not None:
        def buf(name, k, dt):
            b = out.get(name)
            if b is None or b.numel() < k or b.device != dev:
                b = out[name] = torch.empty(max(int(k * 1.25), 1), dtype=dt, device=dev)
            return b[:k]
        jc, ir, pr = buf("jc", n_local + 1, torch.int32), buf("ir", cap, torch.int32), buf("pr", cap, torch.float64)
    else:
        jc = torch.empty(n_local + 1, dtype=torch.int32, device=dev)
        ir = torch.empty(cap, dtype=torch.int32, device=dev)
        pr = torch.empty(cap, dtype=torch.float64, device=dev)
    asm._bind_stream()
    rc = asm.lib.sa_assemble_segments_async(asm.ctx, k, pi, pj, ps, st, ln, col_lo, m, n_local,
                                            _ptr(jc), _ptr(ir), _ptr(pr), cap)
    if rc:
        asm._raise(rc)
    nnz = ctypes.c_int64(0)
    bp, bw = ctypes.c_int64(-1), ctypes.c_int(-1)
    rc = asm.lib.sa_finish(asm.ctx, ctypes.byref(nnz), ctypes.byref(bp), ctypes.byref(bw))
    if rc:
        asm._raise(rc)
    return DeviceCsc(jc, ir[: nnz.value], pr[: nnz.value], m, n_local)


def assemble_sharded(ii: torch.Tensor, jj: torch.Tensor, s: torch.Tensor, m: int, n: int,
                     local_assemble=None, group=None, nblocks: int = 4096,
                     out: dict | None = None) -> ShardResult:
    """Assemble the global matrix whose triplets are split across the ranks
    of `group` (contiguous chunks in rank order).

    CUDA tensors (local_assemble None or gpu_local_assembler): the CUDA
    partition (sa_partition, which validates the chunk) moves only the
    triplets bound for other ranks; the rank's assembly reads its own chunk
    in place, between what it received from lower and from higher ranks
    (sa_assemble_segments_async).  CPU tensors (gloo tests): the torch
    restatement of the partition, the received and own triplets
    concatenated, and `local_assemble(ii, jj, s, m, n_local)` -> (jc, ir, pr).
    `out` (CUDA path, a dict kept by the caller): the result tensors are
    written into buffers reused across calls (valid until the next call)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = ii.device
    cuda = ii.is_cuda and (local_assemble is None or getattr(local_assemble, "cuda_segments", False))
    asm = None
    if cuda:
        from .assembly import default_assembler

        asm = default_assembler(dev.index if dev.index is not None else 0)
        asm._bind_stream()
        ii, jj, s = ii.contiguous(), jj.contiguous(), s.contiguous()
    if world == 1:  # one rank owns every column: no partition, no exchange
        if cuda:
            out = asm.assemble_device(ii, jj, s, m=m, n=n)
            jc, ir, pr = out.jc, out.ir, out.pr
        else:
            jc, ir, pr = local_assemble(ii, jj, s, m, n)
        k = int(ir.shape[0])  # nnz (the assembly already synchronised for it)
        nl = asm.lib.sa_last_launch_count(asm.ctx) if cuda else 0
        return ShardResult(0, n, jc.to(torch.int64), ir, pr, 0, k, m, n, int(ii.shape[0]), 0, nl)
    nblocks = max(1, min(nblocks, n))
    bsize = (n + nblocks - 1) // nblocks
    # the boundaries only balance the ranks' work: a strided sample of the
    # columns (<= 2^20 per rank) is enough and keeps this off the critical path
    step = max(1, len(jj) >> 20)
    if cuda:
        hist = _block_hist_cuda(asm, jj, nblocks, bsize, step)
    else:
        blk = torch.clamp((jj[::step].to(torch.int64) - 1) // bsize, 0, nblocks - 1)
        hist = torch.bincount(blk, minlength=nblocks).to(torch.int64) * step
    # one all_reduce: the block histogram and every rank's chunk length (the
    # chunk offsets turn chunk-local error positions into global ones)
    lens = torch.zeros(world, dtype=torch.int64, device=dev)
    lens[rank] = int(jj.shape[0])
    red = torch.cat([hist.to(torch.int64), lens])
    dist.all_reduce(red, group=group)
    red = red.cpu()  # one host read: the boundaries and the chunk offset
    hist = red[:nblocks]
    chunk_off = int(red[nblocks:nblocks + rank].sum()) if rank else 0
    bounds = block_boundaries(hist, world, nblocks, n)
    launches = 0
    if cuda:
        parts, counts, err = _partition_cuda(asm, ii, jj, s, m, n, bounds, world, rank)
        launches += asm.lib.sa_last_launch_count(asm.ctx)
    else:
        err = validate_torch(ii, jj, m, n)
        parts, counts = partition_torch(ii, jj, s, bounds, world, rank)
        if err:
            counts = [0] * world
    sc = [0 if r == rank else c for r, c in enumerate(counts)]  # the own triplets stay here
    # one all_to_all: per destination its count and this rank's error word
    word = _error_word(err, chunk_off)
    send = torch.tensor([[c] + word for c in sc], dtype=torch.int64, device=dev)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    recv = recv.cpu()
    words = recv[:, 1:].tolist()
    if any(w[0] != _OK for w in words):
        _raise_agreed(words)
    rc_ = recv[:, 0].tolist()
    sent_remote = sum(sc)

    def exchange(x):
        out = torch.empty(sum(rc_), dtype=x.dtype, device=dev)
        dist.all_to_all_single(out, x, output_split_sizes=rc_, input_split_sizes=sc, group=group)
        return out

    r_ii, r_jj, r_s = (exchange(x) for x in parts)
    col_lo, col_hi = bounds[rank], bounds[rank + 1]
    n_local = col_hi - col_lo
    k_lo = sum(rc_[:rank])  # received from lower ranks precede the own chunk
    lower = (r_ii[:k_lo], r_jj[:k_lo], r_s[:k_lo])
    higher = (r_ii[k_lo:], r_jj[k_lo:], r_s[k_lo:])
    if cuda:
        segs = [x for x in (lower, (ii, jj, s), higher) if x[0].shape[0] > 0] or [(ii, jj, s)]
        res = _assemble_segments_cuda(asm, segs, col_lo, m, n_local, out)
        launches += asm.lib.sa_last_launch_count(asm.ctx)
        jc, ir, pr = res.jc, res.ir, res.pr
    else:
        mine = (jj.to(torch.int64) > col_lo) & (jj.to(torch.int64) <= col_hi)
        sv = s.expand(len(jj)) if s.numel() == 1 and len(jj) != 1 else s
        cat_i = torch.cat([lower[0], ii[mine], higher[0]])
        cat_j = torch.cat([lower[1], jj[mine], higher[1]])
        cat_s = torch.cat([lower[2], sv[mine], higher[2]])
        jc, ir, pr = local_assemble(cat_i, (cat_j.to(torch.int64) - col_lo).to(torch.int32), cat_s, m,
                                    n_local)
    # the rank's nnz is known on the host already (the local assembly
    # synchronised for it); one all_gather and one host read for all ranks'
    nnz_local = torch.tensor([int(ir.shape[0])], dtype=torch.int64, device=dev)
    all_nnz = [torch.empty_like(nnz_local) for _ in range(world)]
    dist.all_gather(all_nnz, nnz_local, group=group)
    nn = torch.cat(all_nnz).cpu().tolist()
    off = sum(nn[:rank])
    if out is not None and cuda:
        b = out.get("jc64")
        if b is None or b.numel() < jc.numel() or b.device != dev:
            b = out["jc64"] = torch.empty(max(int(jc.numel() * 1.25), 1), dtype=torch.int64, device=dev)
        jc_global = torch.add(jc, off, out=b[: jc.numel()])
    else:
        jc_global = jc.to(torch.int64) + off
    return ShardResult(col_lo, col_hi, jc_global, ir, pr, off, sum(nn), m, n,
                       int(r_ii.shape[0]) + counts[rank], sent_remote, launches)


def gpu_local_assembler(device: int = 0):
    """The production local assembler marker: assemble_sharded then reads the
    rank's own chunk in place (CUDA segments) instead of calling it."""
    from .assembly import default_assembler

    asm = default_assembler(device)

    def run(ii, jj, s, m, n_local):
        out = asm.assemble_device(ii.contiguous(), jj.contiguous(), s.contiguous(), m=m, n=n_local)
        return out.jc, out.ir, out.pr

    run.cuda_segments = True
    return run
