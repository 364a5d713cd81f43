"""Command-line front end for the GPU path: assemble, gen, verify, bench.

Mirrors the reference CLI (cli.py:1-241): same subcommands, options and exit
codes (0 success, 1 input/usage error, 2 verification mismatch), with the
assembly running on a B200 (``--device``) instead of CPU worker threads.

    python -m paper_1406_1066_b200 assemble --input t.mtx --output a.mtx [--prune-zeros]
    python -m paper_1406_1066_b200 gen --size 1000 --nnz-row 10 --out t.mtx
    python -m paper_1406_1066_b200 verify --random 200
    python -m paper_1406_1066_b200 bench --dataset 1 --reps 40 --out b.csv [--reference-threads 1,8]

``verify`` and ``bench --reference-threads`` cross-check against the
reference package ``sparseasm`` (its ``assemble_oracle`` / ``assemble_serial``
/ ``assemble_parallel``) and need it importable; the GPU path itself never
uses it.
"""

from __future__ import annotations

import argparse
import sys
import time

import numpy as np

from . import mmio
from .errors import (BadIndex, DeviceError, DimensionTooSmall, LengthMismatch, ParseError,
                     ResultMismatch)
from .types import CscMatrix
from .workloads import RANSPARSE_SEED, ransparse, ransparse_spec


def _thread_list(text: str) -> list[int]:
    try:
        values = [int(x) for x in text.split(",") if x.strip()]
    except ValueError:
        raise argparse.ArgumentTypeError(f"bad thread list {text!r}") from None
    if not values or any(v < 1 for v in values):
        raise argparse.ArgumentTypeError(f"bad thread list {text!r}")
    return values


def _reference():
    """The reference package, or a usage error naming what is missing."""
    try:
        import sparseasm  # noqa: F401
        import sparseasm.bench  # noqa: F401
    except ImportError as exc:
        raise _Usage("this subcommand cross-checks against the reference package "
                     f"'sparseasm', which is not importable ({exc})") from None
    return sparseasm


class _Usage(Exception):
    pass


def _gpu_assemble(ii, jj, s, m, n, nzmax, device):
    from .assembly import assemble

    return assemble(ii, jj, s, m=m, n=n, nzmax=nzmax, device=device)


def cmd_assemble(args) -> int:
    """cli.py:41-62: MatrixMarket triplets -> CSC MatrixMarket."""
    if (args.m is None) != (args.n is None):
        print("error: --m and --n must be given together", file=sys.stderr)
        return 1
    triplets, dims = mmio.read_triplets_matrixmarket(args.input, device=args.device)
    m, n = (args.m, args.n) if args.m is not None else (dims.m, dims.n)
    t0 = time.perf_counter()
    out = _gpu_assemble(triplets.ii, triplets.jj, triplets.sr, m, n, args.nzmax, args.device)
    elapsed = time.perf_counter() - t0
    if args.prune_zeros:
        from .assembly import prune_explicit_zeros

        out = prune_explicit_zeros(out, device=args.device)
    mmio.write_csc_matrixmarket(out, args.output)
    print(f"L={len(triplets)} M={out.m} N={out.n} nnz={out.nnz} elapsed={elapsed:.6f}s",
          file=sys.stderr)
    return 0


def cmd_gen(args) -> int:
    """cli.py:65-73: the reference's random benchmark triplets to a file."""
    if args.size < 1 or args.nnz_row < 1 or args.nrep < 1:
        print("error: --size, --nnz-row and --nrep must be positive", file=sys.stderr)
        return 1
    from .types import Dimensions, TripletList

    ii, jj, s = ransparse(args.size, args.nnz_row, args.nrep, args.seed)
    mmio.write_triplets_matrixmarket(TripletList(ii, jj, s), Dimensions(args.size, args.size),
                                     args.out)
    print(f"wrote {len(ii)} triplets to {args.out}", file=sys.stderr)
    return 0


def _first_difference(out: CscMatrix, ref) -> str:
    if int(out.m) != int(ref.m) or int(out.n) != int(ref.n):
        return f": shape ({out.m}, {out.n}) vs ({ref.m}, {ref.n})"
    if not np.array_equal(np.asarray(out.jc), np.asarray(ref.jc)):
        return f": first differing jc slot {int(np.argmax(np.asarray(out.jc) != np.asarray(ref.jc)))}"
    if not np.array_equal(np.asarray(out.ir), np.asarray(ref.ir)):
        return f": first differing ir slot {int(np.argmax(np.asarray(out.ir) != np.asarray(ref.ir)))}"
    a = np.asarray(out.pr, dtype=np.float64).view(np.uint64)
    b = np.asarray(ref.pr, dtype=np.float64).view(np.uint64)
    return f": first differing pr slot {int(np.argmax(a != b))}"


def _same(a, b) -> bool:
    from .harness import _same as same

    return same(a, b)


def verify_one(checkers, ii, jj, s, m, n, device: int) -> tuple[bool, str]:
    """cli.py:76-100 with the GPU path as the candidate: the GPU result (host
    API and device API) against every checker, bit for bit."""
    from .assembly import default_assembler

    a = default_assembler(device)
    cands = [("b200", a.assemble(ii, jj, s, m=m, n=n))]
    import torch

    dev = torch.device("cuda", device)
    ii32, jj32 = np.asarray(ii), np.asarray(jj)
    if ii32.dtype != np.int32 or jj32.dtype != np.int32:  # device API: int32 indices
        # (the host API above has already validated the raw indices)
        ii32, jj32 = ii32.astype(np.int32), jj32.astype(np.int32)
    d = a.assemble_device(torch.from_numpy(ii32).to(dev), torch.from_numpy(jj32).to(dev),
                          torch.from_numpy(np.asarray(s, dtype=np.float64)).to(dev), m=m, n=n)
    cands.append(("b200-device", d.to_host()))
    for cname, check in checkers:
        ref = check(ii, jj, s, m, n)
        for name, out in cands:
            if not _same(out, ref):
                return False, f"{name} differs from {cname}" + _first_difference(out, ref)
    return True, (f"{len(cands)} GPU results agree with {len(checkers)} reference "
                  f"implementation(s), nnz={cands[0][1].nnz}")


def reference_checkers(threads):
    """(name, fn(ii, jj, s, m, n) -> CSC) for the reference's oracle, serial
    and parallel(p) drivers."""
    sa = _reference()

    def req(ii, jj, s, m, n):
        return sa.AssemblyRequest.from_raw(ii, jj, s, m=m, n=n)

    out = [("oracle", lambda *a: sa.assemble_oracle(req(*a))),
           ("serial", lambda *a: sa.assemble_serial(req(*a)))]
    for p in threads:
        out.append((f"parallel(p={p})", lambda *a, p=p: sa.assemble_parallel(req(*a), p)))
    return out


def cmd_verify(args) -> int:
    """cli.py:103-129: seeded random instances or one input file."""
    checkers = reference_checkers(args.threads or [])
    if args.random:
        rng = np.random.default_rng(args.seed)
        for case in range(args.random):
            length = int(rng.integers(0, 5000))
            m = int(rng.integers(1, 300))
            n = int(rng.integers(1, 300))
            ii = rng.integers(1, m + 1, size=length)
            jj = rng.integers(1, n + 1, size=length)
            s = rng.standard_normal(length)
            ok, message = verify_one(checkers, ii, jj, s, None, None, args.device)
            if not ok:
                print(f"case {case}: {message}", file=sys.stderr)
                return 2
        print(f"{args.random} random instances verified", file=sys.stderr)
        return 0
    if not args.input:
        print("error: need --input or --random N", file=sys.stderr)
        return 1
    triplets, dims = mmio.read_triplets_matrixmarket(args.input, device=args.device)
    ok, message = verify_one(checkers, triplets.ii, triplets.jj, triplets.sr, dims.m, dims.n,
                             args.device)
    print(message, file=sys.stderr)
    return 0 if ok else 2


def cmd_bench(args) -> int:
    """cli.py:132-172: standard dataset, cross-check, time, CSV.  The GPU
    Impl always runs; ``--reference-threads`` adds the reference's serial and
    parallel(p) drivers beside it (and the speedup_vs_serial column)."""
    from .harness import make_impl, run_bench

    siz, nnz_row, nrep = ransparse_spec(args.dataset, args.scale)
    trip = ransparse(siz, nnz_row, nrep, args.seed)
    impls = [make_impl("b200", device=args.device)]
    if args.reference_threads:
        sa = _reference()
        impls.append(sa.bench.make_impl("serial"))
        for p in args.reference_threads:
            impls.append(sa.bench.make_impl("parallel", threads=p))
    results = run_bench(trip, impls, args.reps, dataset_id=str(args.dataset))
    mmio.write_bench_csv(results, args.out)
    for r in results:
        sp = "" if r.speedup_vs_serial is None else f" speedup={r.speedup_vs_serial:.2f}x"
        print(f"{r.impl:>16} p={r.threads} mean={r.mean_seconds:.4f}s "
              f"min={r.min_seconds:.4f}s{sp}", file=sys.stderr)
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="python -m paper_1406_1066_b200",
                                     description="Matlab-compatible sparse assembly on a B200")
    parser.add_argument("--device", type=int, default=0, help="CUDA device ordinal")
    sub = parser.add_subparsers(dest="command", required=True)

    pa = sub.add_parser("assemble", help="assemble a MatrixMarket triplet file")
    pa.add_argument("--input", required=True)
    pa.add_argument("--output", required=True)
    pa.add_argument("--m", type=int)
    pa.add_argument("--n", type=int)
    pa.add_argument("--nzmax", type=int)
    pa.add_argument("--prune-zeros", action="store_true")
    pa.set_defaults(func=cmd_assemble)

    pg = sub.add_parser("gen", help="generate random benchmark triplets")
    pg.add_argument("--size", type=int, required=True)
    pg.add_argument("--nnz-row", type=int, required=True)
    pg.add_argument("--nrep", type=int, default=1)
    pg.add_argument("--seed", type=int, default=RANSPARSE_SEED)
    pg.add_argument("--out", required=True)
    pg.set_defaults(func=cmd_gen)

    pv = sub.add_parser("verify", help="cross-check the GPU path against the reference")
    pv.add_argument("--input")
    pv.add_argument("--threads", type=_thread_list,
                    help="also check the reference's parallel driver at these counts")
    pv.add_argument("--random", type=int, help="verify N seeded random instances")
    pv.add_argument("--seed", type=int, default=RANSPARSE_SEED)
    pv.set_defaults(func=cmd_verify)

    pb = sub.add_parser("bench", help="run the timing harness")
    pb.add_argument("--dataset", type=int, choices=[1, 2, 3], required=True)
    pb.add_argument("--scale", type=float, default=1.0)
    pb.add_argument("--reps", type=int, default=40)
    pb.add_argument("--seed", type=int, default=RANSPARSE_SEED)
    pb.add_argument("--out", required=True)
    pb.add_argument("--reference-threads", type=_thread_list,
                    help="time the reference's serial and parallel(p) drivers beside the GPU")
    pb.set_defaults(func=cmd_bench)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (BadIndex, LengthMismatch, DimensionTooSmall, ParseError, FileNotFoundError,
            ValueError, DeviceError, _Usage) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except ResultMismatch as exc:
        print(f"mismatch: {exc}", file=sys.stderr)
        return 2
