"""Harness hook: the B200 path as an implementation of the reference's own
benchmark harness.

The reference times implementations through ``bench.Impl(name, threads,
run)`` with ``run(req, phase_times=None) -> CscMatrix`` (bench.py:101-107,
made by ``make_impl``, bench.py:110-129) and ``run_bench`` cross-checks every
implementation bit-exactly against the first before timing it
(bench.py:132-196).  ``make_impl("b200")`` returns an object of that shape, so
the reference's ``run_bench`` can time the GPU path beside ``serial`` and
``parallel``:

    from sparseasm import bench as rb
    from paper_1406_1066_b200.harness import make_impl
    rb.run_bench(spec, [rb.make_impl("serial"), make_impl("b200")])

``run`` accepts either request type: the reference's ``AssemblyRequest``
(validated ``triplets`` with ``ii``/``jj``/``sr``, optional ``dims``,
``capacity_hint``) or this package's (``raw_i``/``raw_j``/``raw_s``).
``phase_times`` (if given) receives the host-protocol phases of the C ABI:
``upload`` (host -> device copies enqueued), ``assemble`` (device assembly,
synchronous), ``fetch`` (device -> host copies of jc/ir/pr).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .assembly import _PinnedBlock, _capi, _ptr, default_assembler
from .types import CscMatrix


@dataclass
class Impl:
    """A timed implementation: name, thread count, runner (bench.py:101-107)."""

    name: str
    threads: int
    run: Callable  # (req, phase_times) -> CscMatrix


def _request_arrays(req):
    """(ii, jj, s, m, n, scalar) from either request type."""
    t = getattr(req, "triplets", None)
    if t is not None:  # reference AssemblyRequest: validated int32 / float64
        ii, jj, s = t.ii, t.jj, t.sr
        scalar = False
    else:
        ii, jj, s = req.raw_i, req.raw_j, req.raw_s
        scalar = getattr(req, "value_mode", "vector") == "scalar"
    dims = getattr(req, "dims", None)
    m = n = None
    if dims is not None:
        m, n = int(dims.m), int(dims.n)
    return ii, jj, s, m, n, scalar


def _run_b200(req, phase_times=None, *, device: int = 0) -> CscMatrix:
    ii, jj, s, m, n, scalar = _request_arrays(req)
    if phase_times is None or ii.dtype != np.int32 or jj.dtype != np.int32:
        a = default_assembler(device)
        return a.assemble(ii, jj, s, m=m, n=n, nzmax=getattr(req, "capacity_hint", None))
    # phase-timed host protocol (int32 indices; the reference's validated case)
    a = default_assembler(device)
    lib, ctx = a.lib, a.ctx
    ii = np.ascontiguousarray(ii)
    jj = np.ascontiguousarray(jj)
    s = np.ascontiguousarray(s, dtype=np.float64)
    L = len(ii)
    stride = 0 if (scalar or (len(s) == 1 and L != 1)) else 1
    t0 = time.perf_counter()
    rc = lib.sa_host_upload(ctx, _ptr(ii), _ptr(jj), _ptr(s), stride, L)
    if rc:
        a._raise(rc)
    bad_pos, bad_which = ctypes.c_int64(-1), ctypes.c_int(-1)
    if m is None:
        M, N = ctypes.c_int32(0), ctypes.c_int32(0)
        rc = lib.sa_host_dims(ctx, ctypes.byref(M), ctypes.byref(N), ctypes.byref(bad_pos),
                              ctypes.byref(bad_which))
        if rc:
            a._raise(rc, bad_pos.value, bad_which.value, ii, jj)
        m, n = M.value, N.value
    t1 = time.perf_counter()
    nnz = ctypes.c_int64(0)
    rc = lib.sa_host_assemble(ctx, m, n, ctypes.byref(nnz), ctypes.byref(bad_pos),
                              ctypes.byref(bad_which))
    if rc:
        a._raise(rc, bad_pos.value, bad_which.value, ii, jj)
    t2 = time.perf_counter()
    lib_ = _capi.load()
    jc = np.asarray(_PinnedBlock(lib_, n + 1, np.int32))
    ir = np.asarray(_PinnedBlock(lib_, nnz.value, np.int32))
    pr = np.asarray(_PinnedBlock(lib_, nnz.value, np.float64))
    rc = lib.sa_host_fetch(ctx, _ptr(jc), _ptr(ir), _ptr(pr))
    if rc:
        a._raise(rc)
    t3 = time.perf_counter()
    phase_times["upload"] = phase_times.get("upload", 0.0) + (t1 - t0)
    phase_times["assemble"] = phase_times.get("assemble", 0.0) + (t2 - t1)
    phase_times["fetch"] = phase_times.get("fetch", 0.0) + (t3 - t2)
    return CscMatrix(jc, ir, pr, m, n)


def make_impl(kind: str = "b200", threads: int = 1, device: int = 0) -> Impl:
    """``bench.make_impl`` counterpart (bench.py:110-129) for the GPU path.
    ``threads`` is accepted for signature compatibility (the reference's CPU
    worker count) and reported as 1."""
    if kind != "b200":
        raise ValueError(f"unknown implementation kind {kind!r}")
    return Impl(f"b200-cuda{device}", 1,
                lambda req, pt=None: _run_b200(req, pt, device=device))


@dataclass
class BenchResult:
    """One timed (dataset, implementation) row; the reference's fields
    (bench.py:84-98) so ``mmio.write_bench_csv`` writes the same CSV."""

    dataset_id: str
    impl: str
    threads: int
    mean_seconds: float
    min_seconds: float
    reps: int
    L: int
    M: int
    N: int
    nnz: int
    speedup_vs_serial: float | None = None
    phase_means: dict = field(default_factory=dict)


def _timed(impl: Impl, req, reps: int):
    """One untimed warm-up, then ``reps`` timed calls: (mean, min, mean phases)."""
    impl.run(req)
    times, phases = [], {}
    for _ in range(reps):
        pt: dict[str, float] = {}
        t0 = time.perf_counter()
        impl.run(req, pt)
        times.append(time.perf_counter() - t0)
        for k, v in pt.items():
            phases[k] = phases.get(k, 0.0) + v / reps
    return sum(times) / reps, min(times), phases


def run_bench(triplets, impls: list[Impl], reps: int = 40, dataset_id: str = "custom",
              dims=None) -> list[BenchResult]:
    """Cross-check, then time (the protocol of the reference's run_bench,
    bench.py:132-196) over given triplets ``(ii, jj, s)``.  When the
    reference package is importable, use its own ``bench.run_bench`` instead
    (INTEGRATION.md); this is the self-contained version for the CLI.
    Outputs must agree bit for bit with the first implementation's
    (``ResultMismatch`` otherwise); ``speedup_vs_serial`` is relative to the
    first implementation named ``serial*``."""
    from types import SimpleNamespace

    from .errors import ResultMismatch
    from .types import Dimensions

    if reps < 1:
        raise ValueError("reps must be >= 1")
    ii, jj, s = (np.ascontiguousarray(a, dtype=d) for a, d in
                 zip(triplets, (np.int32, np.int32, np.float64)))
    if dims is None:
        dims = Dimensions(int(ii.max(initial=0)), int(jj.max(initial=0)))
    # reference-shaped request: validated triplets + dims (both Impl kinds accept it)
    req = SimpleNamespace(triplets=SimpleNamespace(ii=ii, jj=jj, sr=s), dims=dims,
                          capacity_hint=None)
    outs = [(impl.name, impl.run(req)) for impl in impls]
    for name, out in outs[1:]:
        if not _same(outs[0][1], out):
            raise ResultMismatch(f"{name} output differs from {outs[0][0]} "
                                 f"(nnz {out.nnz} vs {outs[0][1].nnz})")
    nnz = outs[0][1].nnz if outs else 0
    rows = []
    for impl in impls:
        mean, best, phases = _timed(impl, req, reps)
        rows.append(BenchResult(dataset_id, impl.name, impl.threads, mean, best, reps, len(ii),
                                dims.m, dims.n, nnz, phase_means=phases))
    base = next((r.mean_seconds for r in rows if r.impl.startswith("serial")), None)
    for r in rows:
        r.speedup_vs_serial = base / r.mean_seconds if base else None
    return rows


def _same(a, b) -> bool:
    return (int(a.m) == int(b.m) and int(a.n) == int(b.n)
            and np.array_equal(np.asarray(a.jc), np.asarray(b.jc))
            and np.array_equal(np.asarray(a.ir), np.asarray(b.ir))
            and np.asarray(a.pr, dtype=np.float64).tobytes()
            == np.asarray(b.pr, dtype=np.float64).tobytes())
