"""sparseasm/_b200.py -- the binding a ``sparseasm`` maintainer would add to
route the reference's driver level to the B200 library.

It is written against the reference package only (``sparseasm.types`` /
``sparseasm.errors``) and the C ABI in ``include/sparse_assembly.h``; it does
not import this repository's Python package.  ``assemble_b200`` has the
signature of ``serial.assemble_serial`` (serial.py:111-168) so it can stand
in for it anywhere, including the reference's own tests
(tests/test_reference_suite.py runs them with it routed in) and its harness
(``bench.Impl``, bench.py:101-107).

Library lookup: ``$SPARSEASM_B200_LIB`` (a path to libsa_b200.so), else the
dynamic linker's search path (``libsa_b200.so``).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from sparseasm.errors import BadIndex, DimensionTooSmall
from sparseasm.types import CscMatrix

_vp, _i32, _i64, _int = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
_lock = threading.Lock()
_lib = None
_tls = threading.local()
calls = 0  # assemblies routed to the GPU (observability for tests)


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(os.environ.get("SPARSEASM_B200_LIB", "libsa_b200.so"))
            lib.sa_create.argtypes = [_int, ctypes.POINTER(_vp)]
            lib.sa_last_error.restype = ctypes.c_char_p
            lib.sa_last_error.argtypes = [_vp]
            lib.sa_host_upload.argtypes = [_vp, _vp, _vp, _vp, _i64, _i64]
            lib.sa_host_assemble.argtypes = [_vp, _i32, _i32, ctypes.POINTER(_i64),
                                             ctypes.POINTER(_i64), ctypes.POINTER(_int)]
            lib.sa_host_fetch.argtypes = [_vp, _vp, _vp, _vp]
            _lib = lib
    return _lib


def _ctx():
    ctx = getattr(_tls, "ctx", None)  # one context per host thread (header contract)
    if ctx is None:
        ctx = _vp()
        rc = _load().sa_create(int(os.environ.get("SPARSEASM_B200_DEVICE", "0")), ctypes.byref(ctx))
        if rc:
            raise RuntimeError(f"libsa_b200: sa_create failed (status {rc})")
        _tls.ctx = ctx
    return ctx


def assemble_b200(req, *, kernels=None, tracker=None, phase_times=None) -> CscMatrix:
    """Drop-in for ``assemble_serial(req)``: same result bits (jc, ir, pr),
    same exceptions.  ``kernels`` / ``tracker`` / ``phase_times`` are the CPU
    driver's hooks and are accepted and ignored."""
    global calls
    dims = req.effective_dims()  # the reference's semantics (DimensionTooSmall)
    t = req.triplets             # validated: int32 indices, float64 values (len L)
    ii = np.ascontiguousarray(t.ii, dtype=np.int32)
    jj = np.ascontiguousarray(t.jj, dtype=np.int32)
    sr = np.ascontiguousarray(t.sr, dtype=np.float64)
    L = len(ii)
    lib, ctx = _load(), _ctx()
    rc = lib.sa_host_upload(ctx, ii.ctypes.data, jj.ctypes.data, sr.ctypes.data, 1, L)
    nnz, bad, which = _i64(0), _i64(-1), _int(-1)
    if rc == 0:
        rc = lib.sa_host_assemble(ctx, dims.m, dims.n, ctypes.byref(nnz), ctypes.byref(bad),
                                  ctypes.byref(which))
    if rc == 2:  # SA_ERR_BAD_INDEX
        arr = ii if which.value == 0 else jj
        raise BadIndex(bad.value, arr[bad.value])
    if rc == 3:  # SA_ERR_DIM_TOO_SMALL
        raise DimensionTooSmall(lib.sa_last_error(ctx).decode())
    if rc:
        raise RuntimeError(f"libsa_b200 status {rc}: {lib.sa_last_error(ctx).decode()}")
    jc = np.empty(dims.n + 1, np.int32)
    ir = np.empty(nnz.value, np.int32)
    pr = np.empty(nnz.value, np.float64)
    rc = lib.sa_host_fetch(ctx, jc.ctypes.data, ir.ctypes.data, pr.ctypes.data)
    if rc:
        raise RuntimeError(f"libsa_b200 status {rc}: {lib.sa_last_error(ctx).decode()}")
    calls += 1
    return CscMatrix(jc, ir, pr, dims.m, dims.n)
