"""GPU assembly driver: the host side of the drop-in boundary.

Replaces the reference's drivers (serial.py:111-168, parallel.py:361-389)
and kernel plugin (backend.py, _kernels.pyx) for the path
``assemble(i, j, s, m, n, nzmax)`` (__init__.py:36-46).  All compute runs in
libsa_b200.so (sm_100a); this module only normalises arguments, moves
buffers, and maps C-ABI status codes onto the reference's exceptions.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _capi
from .errors import BadIndex, DeviceError, DimensionTooSmall, LengthMismatch
from .types import INDEX_DTYPE, INDEX_MAX, CscMatrix, Dimensions, normalize_raw

_tls = threading.local()


def _ptr(a) -> int:
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())


@dataclass
class DeviceCsc:
    """Device-resident CSC result (torch CUDA tensors)."""

    jc: "object"
    ir: "object"
    pr: "object"
    m: int
    n: int

    @property
    def nnz(self) -> int:
        return int(self.ir.shape[0])

    def to_host(self) -> CscMatrix:
        return CscMatrix(self.jc.cpu().numpy(), self.ir.cpu().numpy(), self.pr.cpu().numpy(),
                         self.m, self.n)


class Assembler:
    """One C-ABI context (device workspace + stream binding) on one GPU."""

    def __init__(self, device: int = 0):
        self.lib = _capi.load()
        self.device = int(device)
        h = ctypes.c_void_p()
        rc = self.lib.sa_create(self.device, ctypes.byref(h))
        if rc != _capi.SA_OK:
            raise DeviceError(rc, f"sa_create(device={device}) failed")
        self.ctx = h

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.sa_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers -----------------------------------------------------------
    def _msg(self) -> str:
        m = self.lib.sa_last_error(self.ctx)
        return m.decode() if m else ""

    def _raise(self, rc, bad_pos=-1, bad_which=-1, raw_i=None, raw_j=None):
        if rc == _capi.SA_ERR_BAD_INDEX:
            arr = raw_i if bad_which == _capi.SA_WHICH_ROW else raw_j
            raise BadIndex(int(bad_pos), _bad_value(arr, int(bad_pos)))
        if rc == _capi.SA_ERR_DIM_TOO_SMALL:
            raise DimensionTooSmall(self._msg())
        raise DeviceError(rc, self._msg())

    def _bind_stream(self):
        import torch

        s = torch.cuda.current_stream(self.device)
        self.lib.sa_set_stream(self.ctx, ctypes.c_void_p(s.cuda_stream))

    def set_option(self, option: int, value: int) -> None:
        """Force a pipeline variant (_capi.SA_OPT_*: -1 automatic, 0, 1).
        Every variant produces the same bits; tests use this to cover each."""
        rc = self.lib.sa_set_option(self.ctx, int(option), int(value))
        if rc:
            raise ValueError(self._msg())

    def launch_count(self) -> int:
        return int(self.lib.sa_last_launch_count(self.ctx))

    # -- host arrays in, host CSC out (the reference-facing call) ----------
    def assemble(self, i, j, s, m=None, n=None, nzmax=None) -> CscMatrix:
        raw_i, raw_j, raw_s, mode = normalize_raw(i, j, s)
        if raw_i.dtype != np.int32 or raw_j.dtype != np.int32:
            return self._assemble_converted(raw_i, raw_j, raw_s, mode, m, n, nzmax)
        ii = np.ascontiguousarray(raw_i)
        jj = np.ascontiguousarray(raw_j)
        L = len(ii)
        stride = 0 if mode == "scalar" else 1
        lib, ctx = self.lib, self.ctx
        rc = lib.sa_host_upload(ctx, _ptr(ii), _ptr(jj), _ptr(raw_s), stride, L)
        if rc:
            self._raise(rc)
        bad_pos, bad_which = ctypes.c_int64(-1), ctypes.c_int(-1)
        if m is None or n is None:
            M, N = ctypes.c_int32(0), ctypes.c_int32(0)
            rc = lib.sa_host_dims(ctx, ctypes.byref(M), ctypes.byref(N), ctypes.byref(bad_pos),
                                  ctypes.byref(bad_which))
            if rc:
                self._raise(rc, bad_pos.value, bad_which.value, raw_i, raw_j)
            if (m is None) != (n is None):
                raise LengthMismatch("explicit dimensions require both m and n")
            dims = Dimensions(M.value, N.value)
        else:
            dims = Dimensions(int(m), int(n))
            _check_int32_dims(dims)
        nnz = ctypes.c_int64(0)
        rc = lib.sa_host_assemble(ctx, dims.m, dims.n, ctypes.byref(nnz), ctypes.byref(bad_pos),
                                  ctypes.byref(bad_which))
        if rc:
            self._raise(rc, bad_pos.value, bad_which.value, raw_i, raw_j)
        # outputs in page-locked memory (torch's caching host allocator), so
        # the device->host copies run at full PCIe/C2C bandwidth
        jc = _pinned_empty(dims.n + 1, np.int32)
        ir = _pinned_empty(nnz.value, np.int32)
        pr = _pinned_empty(nnz.value, np.float64)
        rc = lib.sa_host_fetch(ctx, _ptr(jc), _ptr(ir), _ptr(pr))
        if rc:
            self._raise(rc)
        return CscMatrix(jc, ir, pr, dims.m, dims.n)

    def _assemble_converted(self, raw_i, raw_j, raw_s, mode, m, n, nzmax) -> CscMatrix:
        """Non-int32 index arrays: validate + convert on the device."""
        import torch

        dev = torch.device("cuda", self.device)
        ti = self._convert(raw_i, dev)
        tj = self._convert(raw_j, dev)
        if isinstance(ti, tuple):  # (position, value) of the first bad row index
            raise BadIndex(*ti)
        if isinstance(tj, tuple):
            raise BadIndex(*tj)
        ts = torch.from_numpy(raw_s).to(dev)
        out = self.assemble_device(ti, tj, ts, m=m, n=n, nzmax=nzmax,
                                   scalar=(mode == "scalar"), _raw=(raw_i, raw_j))
        return out.to_host()

    def _convert(self, raw, dev):
        import torch

        kind = raw.dtype.kind
        if kind in "iu":
            if raw.dtype.itemsize <= 2 or raw.dtype == np.int32:
                host = raw.astype(np.int32)
                dtype = _capi.SA_DTYPE_INT32
            elif raw.dtype == np.uint64:
                big = raw > INDEX_MAX
                if big.any():
                    k = int(np.argmax(big))
                    lows = np.flatnonzero(raw[:k] < 1)
                    k = int(lows[0]) if len(lows) else k
                    return (k, raw[k])
                host = raw.astype(np.int64)
                dtype = _capi.SA_DTYPE_INT64
            else:
                host = raw.astype(np.int64)
                dtype = _capi.SA_DTYPE_INT64
        else:
            host = raw.astype(np.float64)
            dtype = _capi.SA_DTYPE_FLOAT64
        src = torch.from_numpy(np.ascontiguousarray(host)).to(dev)
        out = torch.empty(len(host), dtype=torch.int32, device=dev)
        self._bind_stream()
        bad, mx = ctypes.c_int64(-1), ctypes.c_int32(0)
        rc = self.lib.sa_convert_indices(self.ctx, _ptr(src), dtype, len(host), _ptr(out),
                                         ctypes.byref(bad), ctypes.byref(mx))
        if rc:
            self._raise(rc)
        if bad.value >= 0:
            k = bad.value
            return (k, raw[k] if kind in "iu" else float(raw[k]))
        return out

    # -- device tensors in, device CSC out ----------------------------------
    def assemble_device(self, ii, jj, s, m=None, n=None, nzmax=None, scalar=None,
                        _raw=None) -> DeviceCsc:
        """Assemble device-resident int32 triplets (torch CUDA tensors).

        ``s`` may have length 1 (scalar broadcast).  ``nzmax`` is a capacity
        hint only; outputs are always complete.
        """
        import torch

        L = int(ii.shape[0])
        if int(jj.shape[0]) != L:
            raise LengthMismatch(f"index arrays of lengths {L} and {int(jj.shape[0])}")
        if scalar is None:
            scalar = int(s.shape[0]) == 1 and L != 1
        if not scalar and int(s.shape[0]) != L:
            raise LengthMismatch(f"value array of length {int(s.shape[0])} vs index length {L}")
        for name, t in (("ii", ii), ("jj", jj)):
            if t.dtype != torch.int32 or not t.is_cuda:
                raise TypeError(f"assemble_device: {name} must be an int32 CUDA tensor, got "
                                f"{t.dtype} on {t.device} (assemble() converts other index types)")
        if not s.is_cuda:
            raise TypeError(f"assemble_device: s must be a CUDA tensor, got one on {s.device}")
        ii = ii.contiguous()
        jj = jj.contiguous()
        s = s.contiguous().to(torch.float64)
        self._bind_stream()
        bad_pos, bad_which = ctypes.c_int64(-1), ctypes.c_int(-1)
        raw_i, raw_j = _raw if _raw is not None else (None, None)
        if m is None or n is None:
            M, N = ctypes.c_int32(0), ctypes.c_int32(0)
            rc = self.lib.sa_infer_dims(self.ctx, _ptr(ii), _ptr(jj), L, ctypes.byref(M),
                                        ctypes.byref(N), ctypes.byref(bad_pos),
                                        ctypes.byref(bad_which))
            if rc:
                self._raise_dev(rc, bad_pos.value, bad_which.value, raw_i, raw_j, ii, jj)
            if (m is None) != (n is None):
                raise LengthMismatch("explicit dimensions require both m and n")
            dims = Dimensions(M.value, N.value)
        else:
            dims = Dimensions(int(m), int(n))
            _check_int32_dims(dims)
        cap = max(L, 1)
        dev = ii.device
        jc = torch.empty(dims.n + 1, dtype=torch.int32, device=dev)
        ir = torch.empty(cap, dtype=torch.int32, device=dev)
        pr = torch.empty(cap, dtype=torch.float64, device=dev)
        rc = self.lib.sa_assemble_async(self.ctx, _ptr(ii), _ptr(jj), _ptr(s), 0 if scalar else 1,
                                        L, dims.m, dims.n, _ptr(jc), _ptr(ir), _ptr(pr), cap)
        if rc:
            self._raise(rc)
        nnz = ctypes.c_int64(0)
        rc = self.lib.sa_finish(self.ctx, ctypes.byref(nnz), ctypes.byref(bad_pos),
                                ctypes.byref(bad_which))
        if rc:
            self._raise_dev(rc, bad_pos.value, bad_which.value, raw_i, raw_j, ii, jj)
        k = nnz.value
        return DeviceCsc(jc, ir[:k], pr[:k], dims.m, dims.n)

    # -- Matlab-style post-pass (types.py:204-213) on the device ---------------
    def prune_zeros_device(self, m: DeviceCsc) -> DeviceCsc:
        """Drop entries stored as exactly 0.0 (either sign; NaN kept) from a
        device CSC; returns a new DeviceCsc (sa_prune_zeros)."""
        import torch

        nnz = m.nnz
        dev = m.jc.device
        jc = torch.empty(m.n + 1, dtype=torch.int32, device=dev)
        ir = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        pr = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        self._bind_stream()
        out = ctypes.c_int64(0)
        src_ir = m.ir.contiguous()
        src_pr = m.pr.contiguous()
        rc = self.lib.sa_prune_zeros(self.ctx, _ptr(m.jc.contiguous()), _ptr(src_ir), _ptr(src_pr),
                                     m.n, nnz, _ptr(jc), _ptr(ir), _ptr(pr), ctypes.byref(out))
        if rc:
            self._raise(rc)
        k = out.value
        return DeviceCsc(jc, ir[:k], pr[:k], m.m, m.n)

    def prune_zeros(self, m):
        """prune_explicit_zeros for a host CscMatrix (uploaded, pruned on the
        device, fetched) or a DeviceCsc (stays on the device)."""
        if isinstance(m, DeviceCsc):
            return self.prune_zeros_device(m)
        import torch

        dev = torch.device("cuda", self.device)
        d = DeviceCsc(torch.from_numpy(np.ascontiguousarray(m.jc, dtype=np.int32)).to(dev),
                      torch.from_numpy(np.ascontiguousarray(m.ir, dtype=np.int32)).to(dev),
                      torch.from_numpy(np.ascontiguousarray(m.pr, dtype=np.float64)).to(dev),
                      int(m.m), int(m.n))
        return self.prune_zeros_device(d).to_host()

    def _raise_dev(self, rc, pos, which, raw_i, raw_j, ii, jj):
        if rc == _capi.SA_ERR_BAD_INDEX:
            arr = raw_i if which == _capi.SA_WHICH_ROW else raw_j
            if arr is None:
                t = ii if which == _capi.SA_WHICH_ROW else jj
                raise BadIndex(int(pos), int(t[int(pos)].item()))
            raise BadIndex(int(pos), _bad_value(arr, int(pos)))
        self._raise(rc)


class _PinnedBlock:
    """Owner of one page-locked block from the library's host-buffer cache;
    numpy arrays (and every view of them) keep it alive through .base."""

    def __init__(self, lib, n, dtype):
        self._lib = lib
        nbytes = max(int(n), 1) * np.dtype(dtype).itemsize
        self._ptr = lib.sa_host_buffer(nbytes)
        if not self._ptr:
            raise MemoryError(f"page-locked host allocation of {nbytes} bytes failed or over the cap")
        self.__array_interface__ = {"data": (self._ptr, False), "shape": (int(n),),
                                    "typestr": np.dtype(dtype).str, "version": 3}

    def __del__(self):
        if getattr(self, "_ptr", None):
            self._lib.sa_host_buffer_release(self._ptr)
            self._ptr = None


def _pinned_empty(n, dtype):
    """numpy array in page-locked memory (returned to the cache when the
    array and all its views are gone), so the device->host copy runs at full
    PCIe bandwidth.  The library bounds what it keeps page-locked (8 GB of
    free blocks, 16 GB of live results, sa_capi.cu PinnedCache); beyond that,
    or if pinning fails, an ordinary (pageable) array."""
    try:
        return np.asarray(_PinnedBlock(_capi.load(), n, dtype))
    except MemoryError:
        return np.empty(max(int(n), 0), dtype=dtype)


def _bad_value(arr, k):
    if arr is None:
        return None
    v = arr[k]
    return v if arr.dtype.kind in "iu" else float(v)


def _check_int32_dims(d: Dimensions):
    if d.m > INDEX_MAX or d.n > INDEX_MAX:
        raise DimensionTooSmall(f"dimensions ({d.m}, {d.n}) exceed the int32 index range")


def default_assembler(device: int = 0) -> Assembler:
    """Per-thread, per-device cached Assembler (one context per host thread)."""
    cache = getattr(_tls, "assemblers", None)
    if cache is None:
        cache = _tls.assemblers = {}
    a = cache.get(device)
    if a is None:
        a = cache[device] = Assembler(device)
    return a


def assemble(i, j, s, m=None, n=None, nzmax=None, threads=None, *, device: int = 0) -> CscMatrix:
    """Matlab-style ``sparse(i, j, s, m, n, nzmax)`` on a B200.

    Same signature, conventions and errors as the reference's
    ``sparseasm.assemble`` (__init__.py:36-46): 1-based indices (int or
    integral float), a length-1 ``s`` is broadcast, repeated (i, j) pairs are
    summed in input order (bit-exact), dimensions default to the largest
    index.  ``threads`` (the reference's CPU worker count) is accepted and
    ignored; ``nzmax`` is a hint only.
    """
    return default_assembler(device).assemble(i, j, s, m=m, n=n, nzmax=nzmax)


def prune_explicit_zeros(m, *, device: int = 0):
    """Matlab-style post-pass of the reference (types.py:204-213): drop the
    entries stored as exactly 0.0 (+0.0 and -0.0; NaN is kept) and recompact
    jc.  Runs on the GPU (sa_prune_zeros) for a host CscMatrix or a
    DeviceCsc; returns the same kind."""
    return default_assembler(device).prune_zeros(m)


def validate_and_convert(raw_i, raw_j, raw_s, *, device: int = 0):
    """Reference types.py:141-165 on the device: returns (TripletList,
    Dimensions) with int32 indices, or raises BadIndex / LengthMismatch."""
    from .types import TripletList

    raw_i, raw_j, raw_s, mode = normalize_raw(raw_i, raw_j, raw_s)
    a = default_assembler(device)
    import torch

    dev = torch.device("cuda", device)
    outs = []
    maxima = []
    for raw in (raw_i, raw_j):
        r = a._convert(raw, dev)
        if isinstance(r, tuple):
            raise BadIndex(*r)
        outs.append(r.cpu().numpy())
        maxima.append(int(r.max().item()) if len(r) else 0)
    L = len(raw_i)
    sr = np.full(L, raw_s[0], dtype=np.float64) if mode == "scalar" else raw_s
    return TripletList(outs[0], outs[1], sr), Dimensions(maxima[0], maxima[1])
