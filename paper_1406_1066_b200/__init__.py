"""B200-native Matlab-compatible sparse assembly: S = sparse(i, j, s, m, n, nzmax).

Raw 1-based (row, column, value) triplets in, compressed-column storage
(``jc``/``ir``/``pr``: int32/int32/float64) out, duplicate (i, j) entries
summed in input order -- bit-identical to the reference package
``sparseasm`` (arxiv 1406.1066, Engblom & Lukarski) for the same inputs.

The compute path is hand-written sm_100a CUDA behind a C ABI
(``include/sparse_assembly.h`` -> ``lib/libsa_b200.so``); this package is its
host side.  There is no CPU fallback: without the CUDA library every entry
point raises.
"""

from .assembly import (
    Assembler,
    DeviceCsc,
    assemble,
    default_assembler,
    prune_explicit_zeros,
    validate_and_convert,
)
from .errors import (
    BadIndex,
    DeviceError,
    DimensionTooSmall,
    LengthMismatch,
    ParseError,
    ResultMismatch,
)
from .types import (
    AssemblyRequest,
    CscMatrix,
    Dimensions,
    TripletList,
    csc_validate,
    normalize_raw,
)

__version__ = "0.1.0"

__all__ = [
    "Assembler",
    "AssemblyRequest",
    "BadIndex",
    "CscMatrix",
    "DeviceCsc",
    "DeviceError",
    "DimensionTooSmall",
    "Dimensions",
    "LengthMismatch",
    "ParseError",
    "ResultMismatch",
    "TripletList",
    "assemble",
    "assemble_request",
    "csc_validate",
    "default_assembler",
    "normalize_raw",
    "prune_explicit_zeros",
    "validate_and_convert",
]


def assemble_request(req: AssemblyRequest, *, device: int = 0) -> CscMatrix:
    """Assemble an :class:`AssemblyRequest` (reference ``assemble_serial(req)``
    / ``assemble_parallel(req, p)`` replacement, serial.py:111, parallel.py:361)."""
    m = req.dims.m if req.dims is not None else None
    n = req.dims.n if req.dims is not None else None
    return assemble(req.raw_i, req.raw_j, req.raw_s, m=m, n=n, nzmax=req.capacity_hint,
                    device=device)
