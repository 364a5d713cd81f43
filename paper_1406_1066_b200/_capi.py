"""ctypes binding of the C ABI in include/sparse_assembly.h (libsa_b200.so).

There is no CPU fallback: if the CUDA library is missing or cannot be
loaded, every entry point raises ``RuntimeError`` naming the library.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import build as _build

SA_OK = 0
SA_ERR_CUDA = 1
SA_ERR_BAD_INDEX = 2
SA_ERR_DIM_TOO_SMALL = 3
SA_ERR_CAPACITY = 4
SA_ERR_INVALID_ARG = 5
SA_ERR_NOMEM = 6
SA_ERR_INTERNAL = 7

SA_DTYPE_INT32 = 0
SA_DTYPE_INT64 = 1
SA_DTYPE_FLOAT64 = 2

SA_WHICH_ROW = 0
SA_WHICH_COL = 1

SA_OPT_FOLD_STAGED = 0
SA_OPT_SCATTER_STAGED = 1
SA_OPT_PATH = 2
SA_OPT_RPASS_TMA = 3

# every symbol include/sparse_assembly.h declares, with (restype, argtypes)
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_int = ctypes.c_int
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pint = ctypes.POINTER(ctypes.c_int)

SIGNATURES = {
    "sa_version": (_int, []),
    "sa_create": (_int, [_int, ctypes.POINTER(_vp)]),
    "sa_destroy": (None, [_vp]),
    "sa_set_stream": (_int, [_vp, _vp]),
    "sa_set_option": (_int, [_vp, _int, _int]),
    "sa_last_error": (ctypes.c_char_p, [_vp]),
    "sa_convert_indices": (_int, [_vp, _vp, _int, _i64, _vp, _pi64, _pi32]),
    "sa_infer_dims": (_int, [_vp, _vp, _vp, _i64, _pi32, _pi32, _pi64, _pint]),
    "sa_assemble_async": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _i64]),
    "sa_finish": (_int, [_vp, _pi64, _pi64, _pint]),
    "sa_device_nnz": (_vp, [_vp]),
    "sa_host_upload": (_int, [_vp, _vp, _vp, _vp, _i64, _i64]),
    "sa_host_dims": (_int, [_vp, _pi32, _pi32, _pi64, _pint]),
    "sa_host_assemble": (_int, [_vp, _i32, _i32, _pi64, _pi64, _pint]),
    "sa_host_fetch": (_int, [_vp, _vp, _vp, _vp]),
    "sa_prune_zeros": (_int, [_vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _pi64]),
    "sa_block_histogram": (_int, [_vp, _vp, _i64, _i64, _i32, _i64, _vp]),
    "sa_partition": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _i32, _i32, ctypes.POINTER(_i32),
                            _vp, _vp, _vp, _pi64, _pi64, _pint]),
    "sa_assemble_segments_async": (_int, [_vp, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                          ctypes.POINTER(_vp), _pi64, _pi64, _i32, _i32, _i32, _vp,
                                          _vp, _vp, _i64]),
    "sa_last_launch_count": (_int, [_vp]),
    "sa_enable_timing": (_int, [_vp, _int]),
    "sa_host_buffer": (_vp, [ctypes.c_uint64]),
    "sa_host_buffer_release": (None, [_vp]),
    "sa_last_kernel_times": (_int, [_vp, _int, ctypes.POINTER(ctypes.c_float),
                                    ctypes.POINTER(ctypes.c_char_p)]),
}

_lock = threading.Lock()
_lib = None


def library_path() -> str:
    return _build.lib_path()


def load(build_if_missing: bool = True):
    """Load (building first if needed and possible) libsa_b200.so."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not os.path.exists(path):
            if not build_if_missing:
                raise RuntimeError(f"CUDA library {path} is missing; run __graft_entry__.build()")
            try:
                _build.build()
            except Exception as exc:  # no silent fallback
                raise RuntimeError(f"CUDA library {path} is missing and could not be built: {exc}") from exc
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise RuntimeError(f"cannot load CUDA library {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib
