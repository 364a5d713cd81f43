"""TEST INFRASTRUCTURE ONLY -- numpy/C oracles for sparse(i,j,s,m,n).

Restates, in numpy, the reference's independent sort-based oracle
(/root/reference/pkg/src/sparseasm/oracle.py:17-45) and its input validation
(types.py:93-165), and wraps the C restatement of the serial counting sort
(oracle/sa_oracle.c) through ctypes.  Never imported by the product package.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
INDEX_MAX = 2**31 - 1


@dataclass
class Csc:
    """jc (n+1), ir (nnz, 0-based), pr (nnz) plus shape; the reference CscMatrix."""

    jc: np.ndarray
    ir: np.ndarray
    pr: np.ndarray
    m: int
    n: int

    @property
    def nnz(self) -> int:
        return len(self.ir)

    def same_as(self, other) -> bool:
        """Bit-exact comparison (reference types.py:67-75)."""
        return (
            int(self.m) == int(other.m)
            and int(self.n) == int(other.n)
            and np.array_equal(np.asarray(self.jc), np.asarray(other.jc))
            and np.array_equal(np.asarray(self.ir), np.asarray(other.ir))
            and np.asarray(self.pr, dtype=np.float64).tobytes()
            == np.asarray(other.pr, dtype=np.float64).tobytes()
        )


class OracleBadIndex(ValueError):
    def __init__(self, position, value):
        self.position = position
        self.value = value
        super().__init__(f"bad index at position {position}: {value!r}")


class OracleLengthMismatch(ValueError):
    pass


class OracleDimensionTooSmall(ValueError):
    pass


def _convert_index(raw):
    """types.py:121-138: int path checks 1..2^31-1, float path adds integrality."""
    arr = np.asarray(raw)
    if arr.dtype.kind in "iu":
        bad = (arr < 1) | (arr > INDEX_MAX)
        if bad.any():
            k = int(np.argmax(bad))
            raise OracleBadIndex(k, arr[k])
        out = arr.astype(np.int32)
    else:
        arr = arr.astype(np.float64, copy=False)
        with np.errstate(invalid="ignore"):
            ok = (arr >= 1.0) & (arr == np.ceil(arr)) & (arr <= INDEX_MAX)
        if not ok.all():
            k = int(np.argmin(ok))
            raise OracleBadIndex(k, float(arr[k]))
        out = arr.astype(np.int32)
    return out, int(out.max(initial=0))


def prepare(raw_i, raw_j, raw_s, m=None, n=None):
    """types.py:93-118 + 141-165: validate, broadcast, infer/check dims.

    Returns (ii int32, jj int32, sr float64, M, N).
    """
    raw_i = np.atleast_1d(np.asarray(raw_i))
    raw_j = np.atleast_1d(np.asarray(raw_j))
    raw_s = np.atleast_1d(np.asarray(raw_s, dtype=np.float64))
    if len(raw_i) != len(raw_j):
        raise OracleLengthMismatch("index lengths")
    L = len(raw_i)
    if len(raw_s) == 1 and L != 1:
        raw_s = np.full(L, raw_s[0], dtype=np.float64)
    elif len(raw_s) != L:
        raise OracleLengthMismatch("value length")
    ii, mi = _convert_index(raw_i)
    jj, mj = _convert_index(raw_j)
    if (m is None) != (n is None):
        raise OracleLengthMismatch("explicit dimensions require both m and n")
    if m is None:
        M, N = mi, mj
    else:
        if mi > m or mj > n:
            raise OracleDimensionTooSmall(f"({mi},{mj}) vs ({m},{n})")
        M, N = int(m), int(n)
    return ii, jj, np.ascontiguousarray(raw_s, dtype=np.float64), M, N


def assemble_sorted(ii, jj, sr, M, N) -> Csc:
    """Restatement of reference oracle.py:17-45 (stable lexsort + run merge).

    O(L log L); duplicate groups are summed with np.add.at in ascending input
    order, i.e. pr = ((+0.0 + v1) + v2) + ...
    """
    ii = np.asarray(ii, dtype=np.int32)
    jj = np.asarray(jj, dtype=np.int32)
    sr = np.asarray(sr, dtype=np.float64)
    if len(ii) == 0:
        return Csc(np.zeros(N + 1, np.int32), np.empty(0, np.int32), np.empty(0), M, N)
    order = np.lexsort((ii, jj))
    rows, cols, vals = ii[order], jj[order], sr[order]
    first = np.empty(len(rows), dtype=bool)
    first[0] = True
    first[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
    group = np.cumsum(first) - 1
    pr = np.zeros(int(group[-1]) + 1, dtype=np.float64)
    np.add.at(pr, group, vals)
    ir = (rows[first] - 1).astype(np.int32)
    jc = np.zeros(N + 1, dtype=np.int32)
    np.cumsum(np.bincount(cols[first], minlength=N + 1)[1:], out=jc[1:])
    return Csc(jc, ir, pr, M, N)


_lib = None


def _load_c():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libsa_oracle.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.run(["make", "-C", _HERE, "oracle"], check=True,
                           stdout=subprocess.DEVNULL)
        lib = ctypes.CDLL(path)
        lib.sao_assemble.restype = ctypes.c_int64
        lib.sao_assemble.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
            ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        ]
        lib.sao_validate.restype = ctypes.c_int64
        lib.sao_validate.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


def assemble_counting(ii, jj, sr, M, N, scalar: bool = False) -> Csc:
    """C restatement of the serial counting sort (oracle/sa_oracle.c).

    ``scalar=True`` passes a length-1 ``sr`` with stride 0 (repeated adds of
    the same value, identical to the reference's np.full broadcast).
    """
    lib = _load_c()
    ii = np.ascontiguousarray(ii, dtype=np.int32)
    jj = np.ascontiguousarray(jj, dtype=np.int32)
    sr = np.ascontiguousarray(sr, dtype=np.float64)
    L = len(ii)
    jc = np.zeros(N + 1, dtype=np.int32)
    ir = np.empty(max(L, 1), dtype=np.int32)
    pr = np.empty(max(L, 1), dtype=np.float64)
    nnz = lib.sao_assemble(ii.ctypes.data, jj.ctypes.data, sr.ctypes.data,
                           0 if scalar else 1, L, M, N,
                           jc.ctypes.data, ir.ctypes.data, pr.ctypes.data)
    if nnz < 0:
        raise MemoryError("oracle allocation failed")
    return Csc(jc, ir[:nnz].copy(), pr[:nnz].copy(), M, N)


def validate_c(raw, L=None):
    """C restatement of _kernels.pyx:92-110 for int64 (kind 0) / float64 (kind 1)."""
    lib = _load_c()
    arr = np.ascontiguousarray(raw)
    kind = 0 if arr.dtype.kind in "iu" else 1
    arr = arr.astype(np.int64 if kind == 0 else np.float64)
    out = np.empty(max(len(arr), 1), dtype=np.int32)
    mx = ctypes.c_int32(0)
    bad = lib.sao_validate(arr.ctypes.data, kind, len(arr), out.ctypes.data, ctypes.byref(mx))
    return int(bad), out[: len(arr)], int(mx.value)


def prune_zeros(jc, ir, pr, m, n) -> "Csc":
    """Reference types.py:204-213 (prune_explicit_zeros): drop entries stored
    as exactly 0.0 (either sign; NaN != 0.0 is kept), keep the order,
    recompact jc.  Checker for the device post-pass (sa_prune_zeros)."""
    jc = np.asarray(jc, dtype=np.int64)
    pr = np.asarray(pr, dtype=np.float64)
    keep = pr != 0.0
    before = np.zeros(len(pr) + 1, dtype=np.int64)
    np.cumsum(keep, out=before[1:])
    return Csc(before[jc].astype(np.int32), np.asarray(ir, dtype=np.int32)[keep], pr[keep], m, n)
