"""MatrixMarket coordinate I/O and the bench CSV writer
(rank 2).

Same file contract as the reference (mmio.py:43-137): header
``%%MatrixMarket matrix coordinate real|integer general``, a size line
``m n count``, then ``count`` entries ``i j value`` (1-based, duplicates
kept, ``%`` comment lines ignored); values are written with 17 significant
digits so write -> read round trips are bit-faithful.  Host text I/O only --
index validation of what is read goes through the device path
(:func:`paper_1406_1066_b200.validate_and_convert`).
"""

from __future__ import annotations

import numpy as np

from .errors import ParseError
from .types import CscMatrix, Dimensions, TripletList

HEADER = "%%MatrixMarket matrix coordinate real general"


def _check_header(line: str) -> None:
    tok = line.split()
    if len(tok) != 5 or tok[0].lower() != "%%matrixmarket":
        raise ParseError(f"not a MatrixMarket header: {line.strip()!r}", line=1)
    kind = [t.lower() for t in tok[1:]]
    if kind[0] != "matrix" or kind[1] != "coordinate" or kind[3] != "general" \
            or kind[2] not in ("real", "integer"):
        raise ParseError(f"unsupported MatrixMarket type {' '.join(tok[1:])!r} "
                         "(need: matrix coordinate real general)", line=1)


def _scan(path):
    """(size triple, entry lines as (line number, text)), comments skipped."""
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise ParseError("empty file", line=1)
    _check_header(lines[0])
    size = None
    entries = []
    last = 1
    for no, raw in enumerate(lines[1:], start=2):
        last = no
        text = raw.strip()
        if not text or text[0] == "%":
            continue
        if size is None:
            tok = text.split()
            try:
                if len(tok) != 3:
                    raise ValueError
                size = tuple(int(t) for t in tok)
            except ValueError:
                raise ParseError(f"bad size line {text!r}", line=no) from None
            if min(size) < 0:
                raise ParseError(f"negative size {text!r}", line=no)
            continue
        entries.append((no, text))
    if size is None:
        raise ParseError("missing size line", line=last)
    return size, entries, last


def read_triplets_matrixmarket(path, *, device: int = 0):
    """Read a coordinate file -> (TripletList, Dimensions); duplicates kept,
    indices 1-based and validated (BadIndex), within the declared size."""
    (m, n, count), entries, last = _scan(path)
    vals = np.empty((len(entries), 3), dtype=np.float64)
    for k, (no, text) in enumerate(entries):
        tok = text.split()
        if len(tok) != 3:
            raise ParseError(f"expected 'i j value', got {text!r}", line=no)
        try:
            vals[k] = [float(t) for t in tok]
        except ValueError:
            raise ParseError(f"malformed entry {text!r}", line=no) from None
    if len(entries) != count:
        raise ParseError(f"size line promised {count} entries, found {len(entries)}", line=last)
    if count == 0:
        empty_i = np.empty(0, dtype=np.int32)
        return TripletList(empty_i, empty_i.copy(), np.empty(0, dtype=np.float64)), Dimensions(m, n)
    from .assembly import validate_and_convert

    trip, inferred = validate_and_convert(vals[:, 0].copy(), vals[:, 1].copy(), vals[:, 2].copy(),
                                          device=device)
    if inferred.m > m or inferred.n > n:
        raise ParseError(f"entry indices reach ({inferred.m}, {inferred.n}) beyond declared "
                         f"size ({m}, {n})")
    return trip, Dimensions(m, n)


def _num(v: float) -> str:
    return format(v, ".17g")


def write_triplets_matrixmarket(t: TripletList, dims: Dimensions, path) -> None:
    """Triplets in input order (duplicates kept)."""
    rows = [f"{i} {j} {_num(v)}" for i, j, v in zip(np.asarray(t.ii).tolist(),
                                                      np.asarray(t.jj).tolist(),
                                                      np.asarray(t.sr).tolist())]
    with open(path, "w") as fh:
        fh.write("\n".join([HEADER, f"{dims.m} {dims.n} {len(rows)}", *rows]) + "\n")


def write_csc_matrixmarket(mat: CscMatrix, path) -> None:
    """A CSC matrix column-major, rows ascending (its natural order)."""
    jc = np.asarray(mat.jc, dtype=np.int64)
    cols = np.repeat(np.arange(1, mat.n + 1), np.diff(jc))
    rows = [f"{r + 1} {c} {_num(v)}" for r, c, v in zip(np.asarray(mat.ir).tolist(), cols.tolist(),
                                                         np.asarray(mat.pr).tolist())]
    with open(path, "w") as fh:
        fh.write("\n".join([HEADER, f"{mat.m} {mat.n} {len(rows)}", *rows]) + "\n")


# the reference's bench CSV schema (mmio.py:19-31, 140-146)
BENCH_CSV_COLUMNS = ["dataset_id", "impl", "threads", "mean_seconds", "min_seconds", "reps", "L",
                     "M", "N", "nnz", "speedup_vs_serial"]


def write_bench_csv(results, path) -> None:
    """One row per timed (dataset, implementation, threads) combination."""
    import csv

    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=BENCH_CSV_COLUMNS)
        w.writeheader()
        for r in results:
            w.writerow({c: getattr(r, c) for c in BENCH_CSV_COLUMNS})
