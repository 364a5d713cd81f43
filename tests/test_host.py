"""CPU-only checks of the host side: argument normalisation, types, error
classes, the C-ABI library (loads, exports every declared symbol), and the
workload generators."""

import os
import re

import numpy as np
import pytest

import paper_1406_1066_b200 as sa
from paper_1406_1066_b200 import _capi, workloads as W
from paper_1406_1066_b200.types import normalize_raw

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    text = open(os.path.join(ROOT, "include", "sparse_assembly.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sa_[a-z_]+)\s*\(", text)))


def test_library_builds_loads_and_exports_every_declared_symbol():
    lib = _capi.load()  # builds with nvcc if missing; loads without a GPU
    declared = _header_functions()
    assert len(declared) >= 14
    assert set(declared) == set(_capi.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.sa_version() == 2


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _capi.library_path()],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_normalize_lengths_and_scalar_mode():
    i, j, s, mode = normalize_raw([1, 2, 3], [1, 1, 1], [7.5])
    assert mode == "scalar" and s.dtype == np.float64 and len(s) == 1
    _, _, _, mode = normalize_raw([1], [1], [7.5])
    assert mode == "vector"
    with pytest.raises(sa.LengthMismatch):
        normalize_raw([1, 2], [1], [1.0, 1.0])
    with pytest.raises(sa.LengthMismatch):
        normalize_raw([1, 2], [1, 1], [1.0, 2.0, 3.0])
    i, j, s, mode = normalize_raw(3, 4, 5)  # scalars become length-1 arrays
    assert len(i) == len(j) == len(s) == 1


def test_request_from_raw():
    req = sa.AssemblyRequest.from_raw([1, 2], [1, 1], [3.0])
    assert req.value_mode == "scalar" and req.dims is None
    req = sa.AssemblyRequest.from_raw([1, 2], [1, 1], [3.0, 4.0], m=5, n=2, nzmax=9)
    assert req.value_mode == "vector" and req.dims == sa.Dimensions(5, 2)
    assert req.capacity_hint == 9
    with pytest.raises(sa.LengthMismatch):
        sa.AssemblyRequest.from_raw([1], [1], [1.0], m=3)
    with pytest.raises(ValueError):
        sa.Dimensions(-1, 2)


def test_errors_mirror_reference_fields():
    e = sa.BadIndex(3, 0.5)
    assert isinstance(e, ValueError) and e.position == 3 and e.value == 0.5
    assert issubclass(sa.LengthMismatch, ValueError)
    assert issubclass(sa.DimensionTooSmall, ValueError)


def _mat(jc, ir, pr, m, n):
    return sa.CscMatrix(np.asarray(jc, np.int32), np.asarray(ir, np.int32),
                        np.asarray(pr, np.float64), m, n)


def test_csc_validate():
    assert sa.csc_validate(_mat([0, 3, 5, 7, 10], [0, 1, 3, 1, 2, 2, 3, 0, 2, 3],
                                [10, 3, 3, 9, 7, 8, 8, -2, 7, 5], 4, 4)) == []
    assert sa.csc_validate(_mat([0, 0, 0], [], [], 3, 2)) == []
    assert any("non-decreasing jc" in v for v in sa.csc_validate(_mat([0, 2, 1], [0, 1], [1, 1], 2, 2)))
    assert any("jc[0]" in v for v in sa.csc_validate(_mat([1, 2], [0, 1], [1, 1], 2, 1)))
    assert any("jc[n]" in v for v in sa.csc_validate(_mat([0, 1], [0, 1], [1, 1], 2, 1)))
    assert any("strictly increasing" in v for v in sa.csc_validate(_mat([0, 2], [1, 1], [1, 1], 2, 1)))
    assert any("strictly increasing" in v for v in sa.csc_validate(_mat([0, 2], [1, 0], [1, 1], 2, 1)))
    assert sa.csc_validate(_mat([0, 1, 2], [1, 1], [1, 1], 2, 2)) == []
    assert any("outside" in v for v in sa.csc_validate(_mat([0, 1], [5], [1], 3, 1)))
    assert any("jc length" in v for v in sa.csc_validate(_mat([0, 1], [0], [1], 2, 2)))


def test_prune_oracle_restates_reference_cases():
    """oracle.prune_zeros pins the reference's prune semantics (types.py:204-213)."""
    from oracle import oracle as O

    p = O.prune_zeros([0, 2], [0, 1], [1.0, 2.0], 2, 1)
    assert p.jc.tolist() == [0, 2] and p.ir.tolist() == [0, 1] and p.pr.tolist() == [1.0, 2.0]
    p = O.prune_zeros([0, 2, 3], [0, 1, 1], [0.0, 5.0, -0.0], 2, 2)
    assert p.jc.tolist() == [0, 1, 1] and p.ir.tolist() == [1] and p.pr.tolist() == [5.0]
    p = O.prune_zeros([0, 1, 2], [0, 0], [np.nan, 0.0], 1, 2)
    assert p.nnz == 1 and np.isnan(p.pr[0]) and p.jc.tolist() == [0, 1, 1]
    p = O.prune_zeros([0, 0, 0], [], [], 3, 2)
    assert p.jc.tolist() == [0, 0, 0] and p.nnz == 0


def test_same_as_is_bitwise():
    a = _mat([0, 1], [0], [np.nan], 1, 1)
    b = _mat([0, 1], [0], [np.nan], 1, 1)
    assert a.same_as(b)
    c = _mat([0, 1], [0], [-0.0], 1, 1)
    d = _mat([0, 1], [0], [0.0], 1, 1)
    assert not c.same_as(d)


def test_workload_shapes():
    w = W.fem2d(5)
    assert w.L == 18 * 25 and w.m == w.n == 36 and w.expected_nnz == 7 * 25 + 31
    assert int(w.ii.min()) == 1 and int(w.ii.max()) == 36
    w = W.fem3d(2)
    assert w.L == 96 * 8 and w.m == 27
    # a chunk of cells is the matching slice of the whole
    full = W.fem2d(6)
    part = W.fem2d(6, cell_range=(10, 20))
    assert np.array_equal(part.ii.numpy(), full.ii.numpy()[10 * 18:20 * 18])
    assert np.array_equal(part.s.numpy(), full.s.numpy()[10 * 18:20 * 18])
    w = W.random_coo(L=1000, seed=3)
    assert w.L == 1000 and int(w.ii.max()) <= 1000 and float(w.s.abs().max()) <= 1.0
    w = W.heavy_dup(m=1000, positions=2000, seed=1)
    assert 5000 < w.L < 15000


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1406_1066_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = re.sub(r"#.*|//.*", "", open(os.path.join(dirpath, f)).read())
                # this repo's oracle package / its C library / the compiled
                # reference kernels (the reference package's own
                # assemble_oracle, used by `cli verify` as a checker, is not it)
                assert not re.search(r"\b(from|import)\s+oracle\b|libsa_oracle|ref_driver|"
                                     r"oracle/_ref|sys\.path.*oracle", text), f


def test_harness_impl_shape():
    """The harness hook has the reference's Impl shape (bench.py:101-107)."""
    from paper_1406_1066_b200.harness import Impl, make_impl

    impl = make_impl("b200", threads=8)
    assert isinstance(impl, Impl) and impl.threads == 1 and callable(impl.run)
    with pytest.raises(ValueError):
        make_impl("serial")


def test_matrixmarket_parse_errors(tmp_path):
    """Header / size-line / entry errors are raised before any device work
    (reference mmio.py:43-114 contract)."""
    from paper_1406_1066_b200.mmio import read_triplets_matrixmarket

    def bad(text, line):
        p = tmp_path / "x.mtx"
        p.write_text(text)
        with pytest.raises(sa.ParseError) as e:
            read_triplets_matrixmarket(p)
        assert e.value.line == line

    bad("", 1)
    bad("%%MatrixMarket matrix array real general\n1 1\n", 1)
    bad("%%MatrixMarket matrix coordinate complex general\n1 1 0\n", 1)
    bad("%%MatrixMarket matrix coordinate real general\n% c\n2 x 1\n", 3)
    bad("%%MatrixMarket matrix coordinate real general\n2 -2 1\n", 2)
    bad("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", 3)
    bad("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 q\n", 3)
    bad("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", 3)
    bad("%%MatrixMarket matrix coordinate real general\n% only comments\n", 2)


def test_matrixmarket_empty_and_writers(tmp_path):
    from paper_1406_1066_b200.mmio import (read_triplets_matrixmarket, write_csc_matrixmarket,
                                           write_triplets_matrixmarket)

    p = tmp_path / "e.mtx"
    p.write_text("%%MatrixMarket matrix coordinate integer general\n3 4 0\n")
    t, d = read_triplets_matrixmarket(p)
    assert len(t) == 0 and (d.m, d.n) == (3, 4)
    write_triplets_matrixmarket(sa.TripletList(np.array([2, 1], np.int32), np.array([1, 3], np.int32),
                                               np.array([0.1, -2.5])), sa.Dimensions(2, 3), p)
    assert p.read_text().splitlines() == ["%%MatrixMarket matrix coordinate real general", "2 3 2",
                                          "2 1 0.10000000000000001", "1 3 -2.5"]
    write_csc_matrixmarket(_mat([0, 1, 1, 3], [1, 0, 1], [1.0, 2.0, 3.0], 2, 3), p)
    assert p.read_text().splitlines()[1:] == ["2 3 3", "2 1 1", "1 3 2", "2 3 3"]


def _datasets():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "dataset_digests.json")) as f:
        return json.load(f)


def test_ransparse_matches_reference_generator():
    """workloads.ransparse == the reference's gen_ransparse (bench.py:62-81)
    bit for bit, at the standard datasets' scaled and full sizes."""
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from instances import input_digest

    for d in _datasets():
        assert W.ransparse_spec(d["dataset"], d["scale"]) == (d["siz"], d["nnz_row"], d["nrep"])
        ii, jj, s = W.ransparse(d["siz"], d["nnz_row"], d["nrep"], d["seed"])
        assert len(ii) == d["L"]
        assert input_digest(ii, jj, s) == d["input"], d
    with pytest.raises(ValueError):
        W.ransparse_spec(4)
    with pytest.raises(ValueError):
        W.ransparse_spec(1, 0.0)


def test_cli_gen_and_usage_errors(tmp_path, capsys):
    """cli gen writes the reference generator's triplets; usage errors exit
    1 before any device work (reference cli.py exit codes)."""
    from paper_1406_1066_b200 import cli

    out = tmp_path / "t.mtx"
    assert cli.main(["gen", "--size", "40", "--nnz-row", "3", "--nrep", "2", "--seed", "5",
                     "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    ii, jj, s = W.ransparse(40, 3, 2, 5)
    assert lines[1] == f"40 40 {len(ii)}"
    assert lines[2:5] == [f"{ii[k]} {jj[k]} 1" for k in range(3)]
    assert cli.main(["gen", "--size", "0", "--nnz-row", "3", "--out", str(out)]) == 1
    assert cli.main(["assemble", "--input", str(out), "--output", str(tmp_path / "a"),
                     "--m", "3"]) == 1
    assert cli.main(["verify"]) in (1,)  # no reference package / no input
    assert cli.main(["assemble", "--input", str(tmp_path / "missing.mtx"),
                     "--output", str(tmp_path / "a")]) == 1
    with pytest.raises(SystemExit):
        cli.main(["bench", "--dataset", "1", "--out", "x", "--reference-threads", "0"])


def test_run_bench_protocol_and_csv(tmp_path):
    """harness.run_bench restates the reference protocol (bench.py:132-196):
    cross-check first (ResultMismatch on any difference), then warm-up +
    timed reps, speedup_vs_serial from the serial row; the CSV has the
    reference's columns (mmio.py:19-31)."""
    import csv

    from paper_1406_1066_b200.harness import Impl, run_bench
    from paper_1406_1066_b200.mmio import BENCH_CSV_COLUMNS, write_bench_csv

    calls = []

    def fake(name, pr):
        def run(req, pt=None):
            calls.append((name, pt is not None))
            if pt is not None:
                pt["assemble"] = pt.get("assemble", 0.0) + 1.0
            return _mat([0, 1], [0], [pr], 1, 1)
        return Impl(name, 1, run)

    trip = (np.array([1], np.int32), np.array([1], np.int32), np.array([2.0]))
    res = run_bench(trip, [fake("serial", 2.0), fake("b200", 2.0)], reps=3, dataset_id="7")
    assert [r.impl for r in res] == ["serial", "b200"]
    assert all(r.reps == 3 and r.L == 1 and r.nnz == 1 and (r.M, r.N) == (1, 1) for r in res)
    assert res[0].speedup_vs_serial == pytest.approx(1.0)
    assert res[1].phase_means == {"assemble": 1.0}
    # 1 check + 1 warm-up + 3 timed per impl
    assert sum(1 for c in calls if c[0] == "b200") == 5
    with pytest.raises(sa.ResultMismatch):
        run_bench(trip, [fake("serial", 2.0), fake("b200", -2.0)], reps=1)
    p = tmp_path / "b.csv"
    write_bench_csv(res, p)
    rows = list(csv.DictReader(open(p)))
    assert list(rows[0].keys()) == BENCH_CSV_COLUMNS and rows[1]["impl"] == "b200"


def test_bench_reference_arm_contract():
    """bench.py --impl reference (runs on the host CPU, no GPU needed): one
    JSON line with the driver's keys, the same `config` dictionary the GPU
    arm prints, and a cpu_baseline describing the stock reference run."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--config", "1", "--steps", "3", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("random_coo") and d["config"]["L"] == 100_000
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and 3 <= d["steps"] <= 3
