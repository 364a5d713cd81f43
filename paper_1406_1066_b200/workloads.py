"""Seeded synthetic triplet workloads for the five BASELINE configurations.

All generators return 1-based int32 ``(ii, jj)`` and float64 ``s`` as torch
tensors on the requested device.  The FEM generators are deterministic
integer arithmetic plus exact products, so CPU and CUDA produce identical
bits; the random generators are seeded (same seed + same device type ->
same bits).

cfg1  random COO     m=n=1000, L=1e5, s~U(-1,1)
cfg2  2D P1 FEM      unit square, N=1000 cells per side, 2 triangles per
                     cell, 3x3 local Laplacian -> 9 triplets per element
cfg3  3D P1 FEM      100^3 cubes, 6 Kuhn tetrahedra per cube, 4x4 local
                     Laplacian -> 16 triplets per element
cfg4  heavy-dup      m=n=1e7, 1e8 uniform positions, Poisson(5) repeats,
                     one global shuffle, s~N(0,1)
cfg5  sharded 2D FEM cfg2's recipe with N=8000, split in contiguous chunks
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import torch


@dataclass
class Workload:
    name: str
    ii: torch.Tensor
    jj: torch.Tensor
    s: torch.Tensor
    m: int
    n: int
    expected_nnz: int | None = None

    @property
    def L(self) -> int:
        return int(self.ii.shape[0])


# --- 2D: right-isosceles P1 stiffness (right angle at the listed local vertex)
# T1 = (v00, v10, v11): right angle at v10;  T2 = (v00, v11, v01): right angle at v01
_K2D_T1 = [[0.5, -0.5, 0.0], [-0.5, 1.0, -0.5], [0.0, -0.5, 0.5]]
_K2D_T2 = [[0.5, 0.0, -0.5], [0.0, 0.5, -0.5], [-0.5, -0.5, 1.0]]


def fem2d(N: int, device="cpu", cell_range=None) -> Workload:
    """cfg2 / cfg5: triangulated unit square with N x N cells.

    Nodes are numbered row-major, id = y*(N+1) + x + 1.  Cells run in
    row-major order; each emits T1 then T2, each element its local 3x3
    matrix in row-major local order.  ``cell_range=(c0, c1)`` restricts to a
    contiguous cell range (the per-rank chunk of the sharded config).
    L = 18 N^2, nnz = 7 N^2 + 6 N + 1 (hypotenuse zeros are retained).
    """
    dev = torch.device(device)
    c0, c1 = (0, N * N) if cell_range is None else cell_range
    cell = torch.arange(c0, c1, dtype=torch.int64, device=dev)
    cy = cell // N
    cx = cell - cy * N
    v00 = (cy * (N + 1) + cx + 1).to(torch.int32)
    v10 = v00 + 1
    v01 = v00 + (N + 1)
    v11 = v01 + 1
    t1 = torch.stack([v00, v10, v11], dim=1)
    t2 = torch.stack([v00, v11, v01], dim=1)
    elems = torch.stack([t1, t2], dim=1).reshape(-1, 3)  # (2*cells, 3)
    del t1, t2, v00, v10, v01, v11, cell, cy, cx
    ii = elems[:, :, None].expand(-1, 3, 3).reshape(-1).contiguous()
    jj = elems[:, None, :].expand(-1, 3, 3).reshape(-1).contiguous()
    del elems
    k = torch.tensor([_K2D_T1, _K2D_T2], dtype=torch.float64, device=dev).reshape(1, 2 * 9)
    s = k.expand(c1 - c0, -1).reshape(-1).contiguous()
    return Workload(f"fem2d_N{N}", ii, jj, s, (N + 1) ** 2, (N + 1) ** 2, 7 * N * N + 6 * N + 1)


# --- 3D: Kuhn tetrahedra.  For the axis permutation (a, b, c) the tet is
# v0 = corner, v1 = v0+e_a, v2 = v1+e_b, v3 = v2+e_c; its P1 stiffness is
# (h/6) * tridiag(-1, [1,2,2,1], -1) -- not dyadic, so duplicate sums are
# order-sensitive in floating point.
_K3D = [[1, -1, 0, 0], [-1, 2, -1, 0], [0, -1, 2, -1], [0, 0, -1, 1]]
_PERMS = list(itertools.permutations(range(3)))


def fem3d(N: int, device="cpu") -> Workload:
    """cfg3: N^3 cubes, 6 Kuhn tetrahedra each (permutations in lexicographic
    order), node id = (z*(N+1) + y)*(N+1) + x + 1; L = 96 N^3."""
    dev = torch.device(device)
    n1 = N + 1
    cube = torch.arange(N ** 3, dtype=torch.int64, device=dev)
    cz = cube // (N * N)
    rem = cube - cz * N * N
    cy = rem // N
    cx = rem - cy * N
    corner = ((cz * n1 + cy) * n1 + cx + 1).to(torch.int32)
    del cube, cz, rem, cy, cx
    step = [1, n1, n1 * n1]  # e_x, e_y, e_z offsets
    tets = []
    for a, b, c in _PERMS:
        v0 = corner
        v1 = v0 + step[a]
        v2 = v1 + step[b]
        v3 = v2 + step[c]
        tets.append(torch.stack([v0, v1, v2, v3], dim=1))
    elems = torch.stack(tets, dim=1).reshape(-1, 4)  # (6 N^3, 4)
    del tets, corner
    ii = elems[:, :, None].expand(-1, 4, 4).reshape(-1).contiguous()
    jj = elems[:, None, :].expand(-1, 4, 4).reshape(-1).contiguous()
    del elems
    scale = (1.0 / N) / 6.0
    k = torch.tensor(_K3D, dtype=torch.float64, device=dev).reshape(1, 16) * scale
    s = k.expand(6 * N ** 3, -1).reshape(-1).contiguous()
    return Workload(f"fem3d_N{N}", ii, jj, s, n1 ** 3, n1 ** 3, None)


def random_coo(m: int = 1000, n: int = 1000, L: int = 100_000, seed: int = 1, device="cpu") -> Workload:
    """cfg1: i, j ~ U{1..m} x U{1..n}, s ~ U(-1, 1)."""
    dev = torch.device(device)
    g = torch.Generator(device=dev).manual_seed(seed)
    ii = torch.randint(1, m + 1, (L,), generator=g, device=dev, dtype=torch.int32)
    jj = torch.randint(1, n + 1, (L,), generator=g, device=dev, dtype=torch.int32)
    s = torch.rand(L, generator=g, device=dev, dtype=torch.float64) * 2.0 - 1.0
    return Workload(f"random_coo_{m}x{n}_L{L}", ii, jj, s, m, n, None)


def heavy_dup(m: int = 10_000_000, positions: int = 100_000_000, mean_rep: float = 5.0,
              seed: int = 4, device="cpu") -> Workload:
    """cfg4: `positions` uniform (i, j) pairs, each repeated Poisson(mean_rep)
    times (zero repeats vanish), one global shuffle, s ~ N(0, 1)."""
    dev = torch.device(device)
    g = torch.Generator(device=dev).manual_seed(seed)
    pi = torch.randint(1, m + 1, (positions,), generator=g, device=dev, dtype=torch.int32)
    pj = torch.randint(1, m + 1, (positions,), generator=g, device=dev, dtype=torch.int32)
    reps = torch.poisson(torch.full((positions,), mean_rep, dtype=torch.float32, device=dev),
                         generator=g).to(torch.int64)
    ii = torch.repeat_interleave(pi, reps)
    jj = torch.repeat_interleave(pj, reps)
    del pi, pj, reps
    L = int(ii.shape[0])
    perm = torch.randperm(L, generator=g, device=dev)
    ii = ii[perm].contiguous()
    jj = jj[perm].contiguous()
    del perm
    s = torch.randn(L, generator=g, device=dev, dtype=torch.float64)
    return Workload(f"heavy_dup_{m}_P{positions}", ii, jj, s, m, m, None)


def config(k: int, device="cpu", scale: float = 1.0) -> Workload:
    """BASELINE.json configs[k-1] (k = 1..5); ``scale`` < 1 shrinks sizes
    (for parity tests and bounded CPU samples)."""
    if k == 1:
        return random_coo(device=device)
    if k == 2:
        return fem2d(max(1, round(1000 * math.sqrt(scale))), device)
    if k == 3:
        return fem3d(max(1, round(100 * scale ** (1 / 3))), device)
    if k == 4:
        return heavy_dup(m=max(1, round(10_000_000 * scale)),
                         positions=max(1, round(100_000_000 * scale)), device=device)
    if k == 5:
        return fem2d(max(1, round(8000 * math.sqrt(scale))), device)
    raise ValueError(f"unknown config {k}")


CONFIG_NAMES = {
    1: "cfg1 random COO m=n=1000 L=1e5",
    2: "cfg2 2D P1 FEM N=1000 (L=18e6)",
    3: "cfg3 3D P1 FEM 100^3 Kuhn (L=96e6)",
    4: "cfg4 heavy-dup m=n=1e7, 1e8 positions x Poisson(5) (L~5e8)",
    5: "cfg5 sharded 2D P1 FEM N=8000 (L=1.152e9)",
}


# --- the reference's own benchmark datasets ---------------------------------
# bench.py:27-32 (_DATASETS), 48-59 (dataset_config), 62-81 (gen_ransparse):
# every row draws nnz_row uniform columns, the block is tiled nrep times,
# one global permutation shuffles it, all values 1.0.  Same numpy Generator
# calls in the same order, so the same seed gives the same bits.

RANSPARSE_SEED = 20151023
RANSPARSE_DATASETS = {1: (10_000, 50, 5), 2: (50_000, 50, 1), 3: (50_000, 10, 5)}


def ransparse_spec(ds_id: int, scale: float = 1.0) -> tuple[int, int, int]:
    """(siz, nnz_row, nrep) of standard dataset ``ds_id``; ``scale`` shrinks
    the matrix size linearly (bench.py:48-59)."""
    if ds_id not in RANSPARSE_DATASETS:
        raise ValueError(f"dataset id {ds_id} not in {sorted(RANSPARSE_DATASETS)}")
    if not 0.0 < scale <= 1.0:
        raise ValueError(f"scale {scale} outside (0, 1]")
    siz, nnz_row, nrep = RANSPARSE_DATASETS[ds_id]
    return max(1, round(siz * scale)), nnz_row, nrep


def ransparse(siz: int, nnz_row: int, nrep: int = 1, seed: int = RANSPARSE_SEED):
    """Host (numpy) triplets ``(ii, jj, s)`` of the reference generator
    (bench.py:62-81): int32, int32, float64 (all ones); ``siz`` x ``siz``."""
    import numpy as np

    if siz < 1 or nnz_row < 1 or nrep < 1:
        raise ValueError(f"non-positive generator parameters ({siz}, {nnz_row}, {nrep})")
    rng = np.random.default_rng(seed)
    block = siz * nnz_row
    rows = np.tile(np.arange(1, siz + 1, dtype=np.int32), nnz_row)
    cols = rng.integers(1, siz + 1, size=block, dtype=np.int32)
    rows = np.tile(rows, nrep)
    cols = np.tile(cols, nrep)
    perm = rng.permutation(len(rows))
    return (np.ascontiguousarray(rows[perm]), np.ascontiguousarray(cols[perm]),
            np.ones(len(rows), dtype=np.float64))
