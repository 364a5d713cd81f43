"""Multi-GPU assembly by column block: one process per GPU.

Each rank holds a contiguous chunk of the global triplet stream (chunks in
rank order = input order).  Per call:

1. every rank histograms its triplets into ``nblocks`` equal column blocks;
   one ``all_reduce`` gives the global block histogram;
2. contiguous column ranges are assigned to ranks so that each receives about
   L / world triplets (block granularity);
3. each rank partitions its chunk by destination rank, *stably*, and one
   ``all_to_all`` moves the triplets (row, column, value) to their owners;
   a rank concatenates what it receives in source-rank order, which is the
   global input order restricted to its columns -- so duplicates are still
   folded in input order and the result is bit-identical to one GPU;
4. the rank assembles its column block with the single-GPU pipeline (columns
   relabelled to the block) and an ``all_gather`` of the per-rank nnz gives
   the offset of its ``jc``.

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


def block_boundaries(block_hist: torch.Tensor, world: int, nblocks: int, n: int):
    """Split nblocks column blocks into `world` contiguous ranges with about
    equal triplet counts.  Returns (world+1) column boundaries (int list)."""
    cum = torch.cumsum(block_hist.to(torch.int64).cpu(), 0)
    total = int(cum[-1]) if len(cum) else 0
    bsize = (n + nblocks - 1) // nblocks
    bounds = [0]
    for r in range(1, world):
        target = (total * r) // world
        # first block index whose cumulative count reaches the target
        k = int(torch.searchsorted(cum, torch.tensor(target, dtype=torch.int64), right=False))
        col = min(n, (k + 1) * bsize) if total else (n * r) // world
        bounds.append(max(bounds[-1], col))
    bounds.append(n)
    return bounds


def assemble_sharded(ii: torch.Tensor, jj: torch.Tensor, s: torch.Tensor, m: int, n: int,
                     local_assemble, group=None, nblocks: int = 4096) -> ShardResult:
    """Assemble the global matrix whose triplets are split across the ranks
    of `group` (contiguous chunks in rank order).  `local_assemble(ii, jj, s,
    m, n_local)` -> (jc int, ir int32, pr float64) tensors on ii's device."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = ii.device
    nblocks = max(1, min(nblocks, n))
    bsize = (n + nblocks - 1) // nblocks
    jj64 = jj.to(torch.int64)
    blk = torch.clamp((jj64 - 1) // bsize, 0, nblocks - 1)
    hist = torch.bincount(blk, minlength=nblocks).to(torch.int64)
    dist.all_reduce(hist, group=group)
    bounds = block_boundaries(hist, world, nblocks, n)
    bt = torch.tensor(bounds[1:-1], dtype=torch.int64, device=dev)
    dest = torch.searchsorted(bt, jj64 - 1, right=True)  # owner rank of each triplet
    # stable partition by destination (input order kept inside each destination)
    order = torch.sort(dest, stable=True).indices
    send_counts = torch.bincount(dest, minlength=world).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    sc = send_counts.cpu().tolist()
    rc = recv_counts.cpu().tolist()
    sent_remote = sum(c for r, c in enumerate(sc) if r != rank)

    def exchange(x):
        out = torch.empty(sum(rc), dtype=x.dtype, device=dev)
        dist.all_to_all_single(out, x[order].contiguous(), output_split_sizes=rc,
                               input_split_sizes=sc, group=group)
        return out

    r_ii = exchange(ii)
    r_jj = exchange(jj)
    r_s = exchange(s)
    col_lo, col_hi = bounds[rank], bounds[rank + 1]
    n_local = col_hi - col_lo
    r_jj_local = (r_jj.to(torch.int64) - col_lo).to(torch.int32)
    jc, ir, pr = local_assemble(r_ii, r_jj_local, r_s, m, n_local)
    nnz_local = torch.tensor([int(jc[-1]) if len(jc) else 0], dtype=torch.int64, device=dev)
    all_nnz = [torch.empty_like(nnz_local) for _ in range(world)]
    dist.all_gather(all_nnz, nnz_local, group=group)
    counts = [int(x.item()) for x in all_nnz]
    off = sum(counts[:rank])
    jc_global = jc.to(torch.int64) + off
    return ShardResult(col_lo, col_hi, jc_global, ir, pr, off, sum(counts), m, n,
                       int(r_ii.shape[0]), sent_remote)


def gpu_local_assembler(device: int = 0):
    """The production local assembler: the CUDA pipeline (device tensors)."""
    from .assembly import default_assembler

    asm = default_assembler(device)

    def run(ii, jj, s, m, n_local):
        out = asm.assemble_device(ii.contiguous(), jj.contiguous(), s.contiguous(), m=m, n=n_local)
        return out.jc, out.ir, out.pr

    return run
