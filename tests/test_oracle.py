"""Pin the CPU oracles (test infrastructure) against the reference's golden
vectors and against the reference-generated fixtures (tests/golden)."""

import numpy as np
import pytest

from golden_io import error_cases, small_cases, sweep, workloads
from instances import input_digest, output_digest, random_triplets
from oracle import oracle as O
from oracle import stock

CASES = small_cases()


def _check(out, exp):
    assert out.m == exp["m"] and out.n == exp["n"]
    assert np.array_equal(out.jc, exp["jc"])
    assert np.array_equal(out.ir, exp["ir"])
    assert out.pr.tobytes() == exp["pr"].tobytes()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_small_cases_sorted_oracle(case):
    name, i, j, s, m, n, exp = case
    ii, jj, sr, M, N = O.prepare(i, j, s, m, n)
    _check(O.assemble_sorted(ii, jj, sr, M, N), exp)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_small_cases_c_oracle(case):
    name, i, j, s, m, n, exp = case
    ii, jj, sr, M, N = O.prepare(i, j, s, m, n)
    _check(O.assemble_counting(ii, jj, sr, M, N), exp)
    if len(s) == 1 and len(ii) != 1:  # stride-0 scalar path == materialised broadcast
        _check(O.assemble_counting(ii, jj, s, M, N, scalar=True), exp)


def test_golden_example_literal():
    """The paper's running example (reference conftest.py:7-13, PAPER Listing 2)."""
    i = [3, 4, 1, 3, 2, 1, 4, 4, 4, 3, 2, 3, 1]
    j = [3, 3, 1, 4, 1, 1, 4, 3, 1, 3, 2, 2, 4]
    s = [4, 4, 5, 7, 3, 5, 5, 4, 3, 4, 9, 7, -2]
    ii, jj, sr, M, N = O.prepare(i, j, s)
    out = O.assemble_counting(ii, jj, sr, M, N)
    assert out.jc.tolist() == [0, 3, 5, 7, 10]
    assert out.ir.tolist() == [0, 1, 3, 1, 2, 2, 3, 0, 2, 3]
    assert out.pr.tolist() == [10, 3, 3, 9, 7, 8, 8, -2, 7, 5]


ERRS = error_cases()


@pytest.mark.parametrize("case", ERRS, ids=[e[0] for e in ERRS])
def test_validation_semantics(case):
    name, i, j, s, m, n, exc, pos = case
    if exc is None:
        O.prepare(i, j, s, m, n)
        return
    expected = {"BadIndex": O.OracleBadIndex, "LengthMismatch": O.OracleLengthMismatch,
                "DimensionTooSmall": O.OracleDimensionTooSmall}[exc]
    with pytest.raises(expected) as e:
        O.prepare(i, j, s, m, n)
    if pos is not None:
        assert e.value.position == pos


def test_validate_c_matches_numpy():
    rng = np.random.default_rng(3)
    for _ in range(50):
        x = rng.integers(-3, 40, size=int(rng.integers(0, 60))).astype(np.float64)
        if len(x) and rng.random() < 0.3:
            x[rng.integers(0, len(x))] = 2.5
        bad, out, mx = O.validate_c(x)
        okmask = (x >= 1) & (x == np.ceil(x)) & (x <= 2**31 - 1)
        if okmask.all():
            assert bad == -1 and np.array_equal(out, x.astype(np.int32))
            assert mx == (int(x.max()) if len(x) else 0)
        else:
            assert bad == int(np.argmin(okmask))


@pytest.mark.parametrize("name", ["acceptance", "serial40"])
def test_sweep_c_oracle_matches_reference(name):
    """All 1000 acceptance-sweep instances: input digests prove the generator
    restatement; output digests prove the C oracle == the reference."""
    kw, rows = sweep(name)
    for r in rows:
        ii, jj, sr = random_triplets(r["seed"], **kw)
        assert input_digest(ii, jj, sr) == r["input"], r["seed"]
        ii32, jj32 = ii.astype(np.int32), jj.astype(np.int32)
        M = int(ii32.max(initial=0))
        N = int(jj32.max(initial=0))
        out = O.assemble_counting(ii32, jj32, sr, M, N)
        assert (out.m, out.n, out.nnz) == (r["m"], r["n"], r["nnz"])
        assert output_digest(out.jc, out.ir, out.pr) == r["output"], r["seed"]


def test_sweep_sorted_oracle_subset():
    kw, rows = sweep("acceptance")
    for r in rows[::10]:
        ii, jj, sr = random_triplets(r["seed"], **kw)
        ii32, jj32 = ii.astype(np.int32), jj.astype(np.int32)
        out = O.assemble_sorted(ii32, jj32, sr, int(ii32.max(initial=0)), int(jj32.max(initial=0)))
        assert output_digest(out.jc, out.ir, out.pr) == r["output"], r["seed"]


def test_workload_digests_c_oracle():
    from paper_1406_1066_b200 import workloads as W

    for r in workloads():
        w = getattr(W, r["kind"])(**r["kwargs"])
        ii, jj, s = w.ii.numpy(), w.jj.numpy(), w.s.numpy()
        assert input_digest(ii, jj, s) == r["input"], r
        out = O.assemble_counting(ii, jj, s, w.m, w.n)
        assert out.nnz == r["nnz"]
        assert output_digest(out.jc, out.ir, out.pr) == r["output"], r


@pytest.mark.skipif(not stock.available(), reason="oracle/_ref (stock reference) not installed")
def test_stock_reference_serial_and_threaded():
    """The unmodified reference package (oracle/_ref: its drivers and its
    compiled kernels) reproduces the committed reference digests, serially
    and with its threaded driver (parallel.py:361-389)."""
    kw, rows = sweep("acceptance")
    for r in rows[::25]:
        ii, jj, sr = random_triplets(r["seed"], **kw)
        ii32, jj32 = ii.astype(np.int32), jj.astype(np.int32)
        req = stock.request(ii32, jj32, sr, None, None)
        a = stock.serial(req)
        assert output_digest(a.jc, a.ir, a.pr) == r["output"]
        for p in (2, 3, 8):
            b = stock.parallel(req, p)
            assert b.same_as(a)
