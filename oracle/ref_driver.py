"""TEST INFRASTRUCTURE ONLY -- the reference's own CPU kernels, driven as the
reference drives them.

``oracle/_ref/_kernels*.so`` is the reference's Cython kernel module
(/root/reference/pkg/src/sparseasm/_kernels.pyx) compiled unmodified from its
source by ``oracle/Makefile``.  This file restates the two drivers around it:

* ``assemble_serial``   -- serial.py:111-168 (Parts 1-4 + scatter)
* ``assemble_parallel`` -- parallel.py:125-156 (counter merges) and
                           parallel.py:267-358 (barrier-phased threads; the
                           kernels release the GIL)

It is the CPU baseline of bench.py (``cpu_baseline.kind == "reference"`` and
``--impl reference``) and a second parity oracle for tests.
"""

from __future__ import annotations

import importlib.machinery
import importlib.util
import os
import threading

import numpy as np

from .oracle import Csc

_HERE = os.path.dirname(os.path.abspath(__file__))
_K = None


def available() -> bool:
    try:
        kernels()
        return True
    except ImportError:
        return False


def kernels():
    """Load oracle/_ref/_kernels<EXT_SUFFIX> (raises ImportError if unbuilt)."""
    global _K
    if _K is None:
        suffix = importlib.machinery.EXTENSION_SUFFIXES[0]
        path = os.path.join(_HERE, "_ref", "_kernels" + suffix)
        if not os.path.exists(path):
            raise ImportError(f"reference kernels not built: {path}")
        spec = importlib.util.spec_from_file_location("_kernels", path)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        if getattr(mod, "BACKEND", None) != "c":
            raise ImportError("unexpected reference kernel module")
        _K = mod
    return _K


def assemble_serial(ii, jj, sr, M, N) -> Csc:
    """serial.py:111-168 over the reference kernels."""
    K = kernels()
    L = len(ii)
    jr = np.zeros(M + 1, dtype=np.int32)
    K.count_rows(ii, jr)
    rank = np.empty(L, dtype=np.int32)
    K.build_rank(ii, jr, rank)
    jc = np.zeros(N + 1, dtype=np.int32)
    hcol = np.zeros(N + 1, dtype=np.int32)
    irank = np.empty(L, dtype=np.int32)
    K.compress(ii, jj, rank, jr, hcol, jc, irank)
    del hcol, rank, jr
    K.accumulate(jj, jc, irank)
    nnz = int(jc[-1])
    ir = np.empty(nnz, dtype=np.int32)
    pr = np.zeros(nnz, dtype=np.float64)
    K.scatter(ii, sr, irank, ir, pr)
    return Csc(jc, ir, pr, M, N)


def _element_range(length, p, k):  # parallel.py:28-30
    return (length * k) // p, (length * (k + 1)) // p


def _row_range(m, p, k):  # parallel.py:33-35
    return 1 + (m * k) // p, (m * (k + 1)) // p


def _merge_row_counters(jrP, p, m):  # parallel.py:125-141
    np.cumsum(jrP[1 : p + 1], axis=0, out=jrP[1 : p + 1])
    if m:
        tot = jrP[p, 1 : m + 1]
        ends = np.cumsum(tot, dtype=np.int64).astype(jrP.dtype)
        starts = ends - tot
        jrP[0, 1 : m + 1] = starts
        if p > 1:
            jrP[1:p, 1 : m + 1] += starts
        jrP[p, 1 : m + 1] = ends
    jrP[p, 0] = 0


def _merge_col_counters(jcP, p, n):  # parallel.py:144-156
    np.cumsum(jcP[1 : p + 1], axis=0, out=jcP[1 : p + 1])
    jc = np.zeros(n + 1, dtype=np.int32)
    if n:
        tot = jcP[p, 1:]
        ends = np.cumsum(tot, dtype=np.int64).astype(jcP.dtype)
        starts = ends - tot
        jcP[0, 1:] = starts
        if p > 1:
            jcP[1:p, 1:] += starts
        jc[1:] = ends
    return jc


def assemble_parallel(ii, jj, sr, M, N, p: int) -> Csc:
    """parallel.py:267-358: barrier-phased worker threads (p >= 2)."""
    K = kernels()
    L = len(ii)
    if p <= 1:
        return assemble_serial(ii, jj, sr, M, N)
    jrP = np.zeros((p + 1, M + 2), dtype=np.int32)
    rank = np.empty(L, dtype=np.int32)
    irankP = np.empty(L, dtype=np.int32)
    jcP = np.zeros((p + 1, N + 1), dtype=np.int32)
    barrier = threading.Barrier(p)
    shared = {}
    failures = []

    def work(k):
        try:
            lo, hi = _element_range(L, p, k)
            rstart, rend = _row_range(M, p, k)
            K.par_hist(ii, jrP[k + 1], lo, hi)
            barrier.wait()
            if k == 0:
                _merge_row_counters(jrP, p, M)
            barrier.wait()
            K.par_rank(ii, jrP[k], rank, lo, hi)
            barrier.wait()
            hcol = np.zeros(N + 1, dtype=np.int32)
            if rend >= rstart:
                K.par_compress(ii, jj, rank, jrP[p], hcol, jcP[k + 1], irankP, rstart, rend)
            del hcol
            barrier.wait()
            if k == 0:
                shared["jc"] = _merge_col_counters(jcP, p, N)
            barrier.wait()
            if rend >= rstart:
                i0, i1 = int(jrP[p][rstart - 1]), int(jrP[p][rend])
                K.par_fixup(jj, rank, irankP, jcP[k], i0, i1)
            barrier.wait()
            if k == 0:
                nnz = int(shared["jc"][-1])
                shared["ir"] = np.empty(nnz, dtype=np.int32)
                shared["pr"] = np.zeros(nnz, dtype=np.float64)
            barrier.wait()
            if rend >= rstart:
                i0, i1 = int(jrP[p][rstart - 1]), int(jrP[p][rend])
                K.par_scatter(ii, sr, rank, irankP, shared["ir"], shared["pr"], i0, i1)
            barrier.wait()
        except threading.BrokenBarrierError:
            pass
        except Exception as exc:  # propagate to the caller (parallel.py:341-353)
            failures.append(exc)
            barrier.abort()

    threads = [threading.Thread(target=work, args=(k,)) for k in range(p)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if failures:
        raise failures[0]
    return Csc(shared["jc"], shared["ir"], shared["pr"], M, N)
