"""GPU parity: the CUDA path (through the C ABI) against the reference's
outputs (golden fixtures) and the CPU oracle.  Bar: jc/ir bit-exact and pr
bit-exact (ordered-sum contract), NaN payloads included."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_1406_1066_b200 as sa  # noqa: E402
from golden_io import error_cases, small_cases, sweep, workloads  # noqa: E402
from instances import input_digest, output_digest, random_triplets  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import stock  # noqa: E402

CASES = small_cases()
ERRS = error_cases()


def _check(out, exp):
    assert out.m == exp["m"] and out.n == exp["n"]
    assert np.array_equal(out.jc, exp["jc"])
    assert np.array_equal(out.ir, exp["ir"])
    assert np.asarray(out.pr).tobytes() == exp["pr"].tobytes()


def _same(a, b):
    assert (a.m, a.n) == (b.m, b.n)
    assert np.array_equal(np.asarray(a.jc), np.asarray(b.jc))
    assert np.array_equal(np.asarray(a.ir), np.asarray(b.ir))
    assert np.asarray(a.pr).tobytes() == np.asarray(b.pr).tobytes()


def test_cuda_library_is_the_one_loaded():
    from paper_1406_1066_b200 import _capi

    lib = _capi.load(build_if_missing=False)
    assert lib.sa_version() == 2
    maps = open("/proc/self/maps").read()
    assert _capi.library_path() in maps


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_small_cases_host_api(case):
    name, i, j, s, m, n, exp = case
    ii = i.astype(np.int32) if i.dtype.kind == "i" else i
    jj = j.astype(np.int32) if j.dtype.kind == "i" else j
    _check(sa.assemble(ii, jj, s, m=m, n=n), exp)
    # same through int64 / float64 index conversion on the device
    _check(sa.assemble(i.astype(np.float64), j.astype(np.float64), s, m=m, n=n), exp)
    _check(sa.assemble(i.astype(np.int64), j.astype(np.int64), s, m=m, n=n), exp)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_small_cases_device_api(case):
    name, i, j, s, m, n, exp = case
    dev = torch.device("cuda", 0)
    ti = torch.from_numpy(i.astype(np.int32)).to(dev)
    tj = torch.from_numpy(j.astype(np.int32)).to(dev)
    ts = torch.from_numpy(s).to(dev)
    out = sa.default_assembler(0).assemble_device(ti, tj, ts, m=m, n=n)
    _check(out.to_host(), exp)


@pytest.mark.parametrize("case", ERRS, ids=[e[0] for e in ERRS])
def test_error_semantics(case):
    name, i, j, s, m, n, exc, pos = case
    expected = {"BadIndex": sa.BadIndex, "LengthMismatch": sa.LengthMismatch,
                "DimensionTooSmall": sa.DimensionTooSmall}
    if exc is None:
        sa.assemble(i, j, s, m=m, n=n)
        return
    with pytest.raises(expected[exc]) as e:
        sa.assemble(i, j, s, m=m, n=n)
    if pos is not None:
        assert e.value.position == pos
    if exc == "BadIndex" and i.dtype.kind == "i" and j.dtype.kind == "i":
        with pytest.raises(sa.BadIndex) as e2:  # the int32 fast path too
            sa.assemble(i.astype(np.int32), j.astype(np.int32), s, m=m, n=n)
        assert e2.value.position == pos


@pytest.mark.parametrize("name", ["acceptance", "serial40"])
def test_sweep_bit_exact_vs_reference(name):
    """1000 acceptance-sweep instances (reference test_acceptance.py:50-71),
    incl. empty, NaN, zeros, 1x1..7x7 matrices with ~50k-long duplicate runs."""
    kw, rows = sweep(name)
    bad = []
    for r in rows:
        ii, jj, sr = random_triplets(r["seed"], **kw)
        out = sa.assemble(ii.astype(np.int32), jj.astype(np.int32), sr)
        if (out.m, out.n, out.nnz) != (r["m"], r["n"], r["nnz"]) or \
                output_digest(out.jc, out.ir, out.pr) != r["output"]:
            bad.append(r["seed"])
        if r["seed"] % 97 == 0:
            assert sa.csc_validate(out) == []
    assert bad == []


def test_workload_digests_vs_reference():
    from paper_1406_1066_b200 import workloads as W

    for r in workloads():
        w = getattr(W, r["kind"])(**r["kwargs"])
        assert input_digest(w.ii.numpy(), w.jj.numpy(), w.s.numpy()) == r["input"]
        dev = torch.device("cuda", 0)
        out = sa.default_assembler(0).assemble_device(w.ii.to(dev), w.jj.to(dev), w.s.to(dev),
                                                      m=w.m, n=w.n).to_host()
        assert out.nnz == r["nnz"], r
        assert output_digest(out.jc, out.ir, out.pr) == r["output"], r


@pytest.mark.parametrize("k,scale", [(1, 1.0), (2, 1.0), (3, 1.0), (4, 0.1)])
def test_baseline_configs_bit_exact_vs_c_oracle(k, scale):
    """Full-size cfg1-cfg3 and 1/10-scale cfg4 against the C oracle."""
    from paper_1406_1066_b200 import workloads as W

    dev = torch.device("cuda", 0)
    w = W.config(k, device=dev, scale=scale)
    out = sa.default_assembler(0).assemble_device(w.ii, w.jj, w.s, m=w.m, n=w.n)
    ref = O.assemble_counting(w.ii.cpu().numpy(), w.jj.cpu().numpy(), w.s.cpu().numpy(), w.m, w.n)
    if w.expected_nnz is not None:
        assert ref.nnz == w.expected_nnz
    _same(out.to_host(), ref)


def test_cfg5_properties_full_size():
    """cfg5 (L = 1.152e9) is too big for the oracle in seconds: check
    size-independent properties -- exact nnz, CSC invariants, zero column
    sums (dyadic element matrices, exact in any order), and bit-exact spot
    checks of sampled columns against the oracle on their triplets."""
    from paper_1406_1066_b200 import workloads as W

    dev = torch.device("cuda", 0)
    N = 8000
    w = W.fem2d(N, device=dev)
    out = sa.default_assembler(0).assemble_device(w.ii, w.jj, w.s, m=w.m, n=w.n)
    assert out.nnz == 7 * N * N + 6 * N + 1
    jc = out.jc.to(torch.int64)
    steps = jc[1:] - jc[:-1]
    assert int(jc[0]) == 0 and int(jc[-1]) == out.nnz and bool((steps >= 1).all())
    col = torch.repeat_interleave(torch.arange(w.n, device=dev), steps)
    colsum = torch.zeros(w.n, dtype=torch.float64, device=dev).index_add_(0, col, out.pr)
    assert bool((colsum == 0).all())
    ir = out.ir.to(torch.int64)
    same_col = col[1:] == col[:-1]
    assert bool((ir[1:][same_col] > ir[:-1][same_col]).all())
    cols = torch.tensor([1, 2, 8001, 32_000_000, w.n - 1, w.n], device=dev, dtype=torch.int32)
    mask = torch.isin(w.jj, cols)
    sub_i, sub_j, sub_s = w.ii[mask].cpu().numpy(), w.jj[mask].cpu().numpy(), w.s[mask].cpu().numpy()
    ref = O.assemble_counting(sub_i, sub_j, sub_s, w.m, w.n)
    for c in cols.tolist():
        a0, a1 = int(out.jc[c - 1]), int(out.jc[c])
        b0, b1 = int(ref.jc[c - 1]), int(ref.jc[c])
        assert np.array_equal(out.ir[a0:a1].cpu().numpy(), ref.ir[b0:b1])
        assert out.pr[a0:a1].cpu().numpy().tobytes() == ref.pr[b0:b1].tobytes()
    del w, out


def test_permuted_fem3d_values_follow_input_order():
    """3D Kuhn values are not dyadic: a shuffled input changes some sums in
    the last bit; the GPU must follow each input order exactly."""
    from paper_1406_1066_b200 import workloads as W

    w = W.fem3d(10)
    perm = torch.from_numpy(np.random.default_rng(11).permutation(w.L))
    ii, jj, s = w.ii[perm].numpy(), w.jj[perm].numpy(), w.s[perm].numpy()
    out = sa.assemble(ii, jj, s, m=w.m, n=w.n)
    _same(out, O.assemble_counting(ii, jj, s, w.m, w.n))
    base = O.assemble_counting(w.ii.numpy(), w.jj.numpy(), w.s.numpy(), w.m, w.n)
    assert (base.pr != out.pr).any()  # the test discriminates order


def test_scalar_value_is_repeated_adds():
    rng = np.random.default_rng(5)
    ii = rng.integers(1, 6, size=5000).astype(np.int32)
    jj = rng.integers(1, 4, size=5000).astype(np.int32)
    out = sa.assemble(ii, jj, [0.1])
    ref = O.assemble_counting(ii, jj, np.full(5000, 0.1), 5, 3)
    _same(out, ref)


def test_big_and_small_columns_mixed():
    """A column longer than the tile cap next to ordinary columns, duplicates
    inside the big column, and rows near the int32 limit."""
    rng = np.random.default_rng(9)
    L = 40_000
    jj = rng.integers(1, 200, size=L).astype(np.int32)
    jj[rng.random(L) < 0.4] = 77  # ~16k triplets in column 77
    ii = rng.integers(1, 50, size=L).astype(np.int32)
    ii[rng.random(L) < 0.1] = 2**31 - 1
    s = rng.standard_normal(L)
    s[rng.random(L) < 0.01] = np.nan
    out = sa.assemble(ii, jj, s, m=2**31 - 1, n=200)
    _same(out, O.assemble_sorted(ii, jj, s, 2**31 - 1, 200))  # row-count-independent oracle
    assert sa.csc_validate(out) == []


def test_many_empty_columns_and_sparse_tiles():
    rng = np.random.default_rng(2)
    L = 3000
    ii = rng.integers(1, 10, size=L).astype(np.int32)
    jj = rng.integers(1, 5_000_000, size=L).astype(np.int32)
    s = rng.standard_normal(L)
    out = sa.assemble(ii, jj, s, m=10, n=5_000_000)
    _same(out, O.assemble_counting(ii, jj, s, 10, 5_000_000))


def test_repeat_calls_reuse_workspace():
    a = sa.default_assembler(0)
    for seed in range(8):
        ii, jj, sr = random_triplets(500 + seed, max_len=200_000, max_dim=5000)
        ii, jj = ii.astype(np.int32), jj.astype(np.int32)
        out = a.assemble(ii, jj, sr)
        _same(out, O.assemble_counting(ii, jj, sr, int(ii.max(initial=0)), int(jj.max(initial=0))))
        if len(ii) > 1000:
            assert a.launch_count() >= 5  # init, hist, scan, scatter, (bigcol), fold


def test_idempotent_reassembly():
    ii, jj, sr = random_triplets(77, max_len=20_000, max_dim=300, allow_special=False)
    first = sa.assemble(ii.astype(np.int32), jj.astype(np.int32), sr)
    cols = np.repeat(np.arange(1, first.n + 1, dtype=np.int32), np.diff(first.jc))
    again = sa.assemble(first.ir + 1, cols, first.pr, m=first.m, n=first.n)
    _same(first, again)


def test_prune_explicit_zeros_on_gpu_output():
    out = sa.assemble(np.array([1, 1, 2], np.int32), np.array([1, 1, 1], np.int32), [2.0, -2.0, 5.0])
    p = sa.prune_explicit_zeros(out)
    assert p.nnz == 1 and p.jc.tolist() == [0, 1] and p.ir.tolist() == [1] and p.pr.tolist() == [5.0]


def _prune_case(jc, ir, pr, m, n):
    from oracle import oracle as O

    mat = sa.CscMatrix(np.asarray(jc, np.int32), np.asarray(ir, np.int32), np.asarray(pr, np.float64), m, n)
    got = sa.prune_explicit_zeros(mat)
    ref = O.prune_zeros(jc, ir, pr, m, n)
    _same(got, ref)
    return got


def test_prune_explicit_zeros_reference_cases():
    p = _prune_case([0, 2], [0, 1], [1.0, 2.0], 2, 1)
    assert p.pr.tolist() == [1.0, 2.0]
    p = _prune_case([0, 2, 3], [0, 1, 1], [0.0, 5.0, -0.0], 2, 2)
    assert p.jc.tolist() == [0, 1, 1] and p.ir.tolist() == [1] and p.pr.tolist() == [5.0]
    p = _prune_case([0, 1, 2], [0, 0], [np.nan, 0.0], 1, 2)
    assert p.nnz == 1 and np.isnan(p.pr[0]) and p.jc.tolist() == [0, 1, 1]
    p = _prune_case([0, 0, 0, 0], [], [], 4, 3)
    assert p.nnz == 0 and p.jc.tolist() == [0, 0, 0, 0]
    p = _prune_case([0, 3], [0, 1, 2], [0.0, -0.0, 0.0], 3, 1)
    assert p.nnz == 0 and p.jc.tolist() == [0, 0]


def test_prune_explicit_zeros_multi_tile():
    """Many tiles, empty and all-zero columns, zeros at tile boundaries,
    NaN payloads, a device-resident input."""
    import torch

    rng = np.random.default_rng(7)
    n = 20_000
    counts = rng.integers(0, 9, size=n)
    counts[rng.integers(0, n, 300)] = 0
    jc = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=jc[1:])
    nnz = int(jc[-1])
    ir = np.concatenate([np.sort(rng.choice(1000, size=c, replace=False)) for c in counts]).astype(np.int32)
    pr = rng.standard_normal(nnz)
    pr[rng.random(nnz) < 0.3] = 0.0
    pr[rng.random(nnz) < 0.05] = -0.0
    pr[2047:2050] = 0.0
    pr[rng.random(nnz) < 0.01] = np.nan
    _prune_case(jc, ir, pr, 1000, n)
    dev = torch.device("cuda", 0)
    d = sa.DeviceCsc(torch.from_numpy(jc.astype(np.int32)).to(dev), torch.from_numpy(ir).to(dev),
                     torch.from_numpy(pr).to(dev), 1000, n)
    got = sa.prune_explicit_zeros(d)
    assert isinstance(got, sa.DeviceCsc)
    from oracle import oracle as O

    _same(got.to_host(), O.prune_zeros(jc, ir, pr, 1000, n))


def test_harness_impl_with_reference_shaped_request():
    """make_impl("b200") runs both request types (the reference's validated
    AssemblyRequest shape and this package's), with phase times."""
    from types import SimpleNamespace

    from paper_1406_1066_b200.harness import make_impl

    ii, jj, sr = random_triplets(5, max_len=30_000, max_dim=400, allow_special=False)
    ii, jj = ii.astype(np.int32), jj.astype(np.int32)
    ref = O.assemble_counting(ii, jj, sr, int(ii.max()), int(jj.max()))
    impl = make_impl("b200")
    assert impl.threads == 1 and impl.name.startswith("b200")
    req_ref = SimpleNamespace(triplets=SimpleNamespace(ii=ii, jj=jj, sr=sr), dims=None,
                              capacity_hint=None)
    pt = {}
    _same(impl.run(req_ref, pt), ref)
    assert set(pt) == {"upload", "assemble", "fetch"} and all(v >= 0 for v in pt.values())
    req = sa.AssemblyRequest.from_raw(ii, jj, sr, m=ref.m, n=ref.n)
    _same(impl.run(req), ref)


def test_matrixmarket_round_trip_bit_faithful(tmp_path):
    """write -> read keeps every value bit-exact; the read triplets assemble
    to the oracle's matrix; indices beyond the declared size are rejected."""
    from paper_1406_1066_b200.mmio import read_triplets_matrixmarket, write_triplets_matrixmarket

    ii, jj, sr = random_triplets(11, max_len=3_000, max_dim=50, allow_special=False)
    t = sa.TripletList(ii.astype(np.int32), jj.astype(np.int32), sr)
    p = tmp_path / "r.mtx"
    write_triplets_matrixmarket(t, sa.Dimensions(60, 70), p)
    t2, d2 = read_triplets_matrixmarket(p)
    assert (d2.m, d2.n) == (60, 70)
    assert np.array_equal(t2.ii, t.ii) and np.array_equal(t2.jj, t.jj)
    assert t2.sr.tobytes() == t.sr.tobytes()
    _same(sa.assemble(t2.ii, t2.jj, t2.sr, m=60, n=70), O.assemble_counting(t.ii, t.jj, t.sr, 60, 70))
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(sa.ParseError):
        read_triplets_matrixmarket(p)
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n1.5 1 1.0\n")
    with pytest.raises(sa.BadIndex):
        read_triplets_matrixmarket(p)


@pytest.mark.parametrize("world,self_rank,banded", [(1, -1, False), (2, 0, False), (3, 2, False),
                                                     (8, -1, False), (8, 5, False), (4, 1, True),
                                                     (8, 7, True)])
def test_partition_kernel_matches_torch_restatement(world, self_rank, banded):
    """sa_partition (CUDA) == partition_torch: destinations in rank order,
    stable inside each, the own rank's triplets counted but left in place,
    out-of-block columns dropped; and the chunk validation.  `banded`:
    columns nearly sorted (element-ordered meshes), so most threads take
    the one-destination shortcut and whole tiles stay home."""
    import ctypes

    from paper_1406_1066_b200.assembly import _ptr
    from paper_1406_1066_b200.distributed import partition_torch

    rng = np.random.default_rng(world)
    L, n = 70_001, 5_000
    ii = rng.integers(1, 900, size=L).astype(np.int32)
    jj = rng.integers(1, n + 1, size=L).astype(np.int32)
    if banded:
        jj = np.sort(jj)
        jj[::97] = rng.integers(1, n + 1, size=len(jj[::97]))  # a few far columns
    s = rng.standard_normal(L)
    cuts = sorted(rng.choice(np.arange(1, n), size=world - 1, replace=False).tolist())
    bounds = [0] + cuts + [n]
    dev = torch.device("cuda", 0)
    a = sa.default_assembler(0)
    a._bind_stream()

    def run(ii, jj, m, nn):
        ti, tj, ts = (torch.from_numpy(x).to(dev) for x in (ii, jj, s))
        outs = [torch.empty(L, dtype=dt, device=dev) for dt in (torch.int32, torch.int32, torch.float64)]
        hb = (ctypes.c_int32 * (world + 1))(*bounds)
        hc = (ctypes.c_int64 * world)()
        bp, bw = ctypes.c_int64(-1), ctypes.c_int(-1)
        rc = a.lib.sa_partition(a.ctx, _ptr(ti), _ptr(tj), _ptr(ts), 1, L, m, nn, world, self_rank, hb,
                                *(_ptr(x) for x in outs), hc, ctypes.byref(bp), ctypes.byref(bw))
        return rc, outs, [hc[r] for r in range(world)], bp.value, bw.value

    rc, outs, counts, _, _ = run(ii, jj, 900, n)
    assert rc == 0
    ref, rcounts = partition_torch(torch.from_numpy(ii), torch.from_numpy(jj), torch.from_numpy(s),
                                   bounds, world, self_rank)
    k = len(ref[0])
    assert counts == rcounts and sum(rcounts) == L
    assert k == L - (rcounts[self_rank] if self_rank >= 0 else 0)
    assert torch.equal(outs[0][:k].cpu(), ref[0]) and torch.equal(outs[1][:k].cpu(), ref[1])
    assert outs[2][:k].cpu().numpy().tobytes() == ref[2].numpy().tobytes()
    bad = jj.copy()
    bad[[10, 20_000]] = 0
    rc, _, _, bp, bw = run(ii, bad, 900, n)
    assert rc != 0 and bp == 10 and bw == 1  # SA_WHICH_COL
    rc, _, _, _, _ = run(ii, jj, 500, n)  # rows above M
    assert rc != 0


@pytest.mark.parametrize("L,step,nblocks", [(0, 1, 16), (1, 1, 1), (100_003, 7, 4096), (2_000_000, 1, 333)])
def test_block_histogram_matches_bincount(L, step, nblocks):
    """sa_block_histogram == the torch restatement (distributed.py CPU path):
    every step-th column, clamped blocks, counts scaled by step."""
    from paper_1406_1066_b200.assembly import _ptr

    rng = np.random.default_rng(L)
    n = 50_000
    jj = rng.integers(-3, n + 10, size=L).astype(np.int32)  # out-of-range columns clamp
    bsize = (n + nblocks - 1) // nblocks
    a = sa.default_assembler(0)
    a._bind_stream()
    dev = torch.device("cuda", 0)
    tj = torch.from_numpy(jj).to(dev)
    hist = torch.full((nblocks,), -1, dtype=torch.int64, device=dev)
    assert a.lib.sa_block_histogram(a.ctx, _ptr(tj) if L else None, L, step, nblocks, bsize, _ptr(hist)) == 0
    blk = torch.clamp((torch.from_numpy(jj[::step]).to(torch.int64) - 1) // bsize, 0, nblocks - 1)
    ref = torch.bincount(blk, minlength=nblocks).to(torch.int64) * step
    assert torch.equal(hist.cpu(), ref)


@pytest.mark.parametrize("kind", ["fem2d", "heavy"])
def test_segment_assembly_is_the_sharded_local_block(kind):
    """sa_assemble_segments_async on [received from lower ranks, own chunk in
    place (other columns skipped), received from higher ranks] == the
    oracle's column block of the whole input, bit for bit (the 3-rank
    sharded assembly simulated for each rank on one GPU)."""
    from paper_1406_1066_b200 import workloads as W
    from paper_1406_1066_b200.distributed import _assemble_segments_cuda

    w = W.fem2d(30) if kind == "fem2d" else W.heavy_dup(m=400, positions=20_000, seed=4)
    ii, jj, s = w.ii.numpy(), w.jj.numpy(), w.s.numpy()
    L, m, n = len(ii), w.m, w.n
    world = 3
    chunks = [(L * r // world, L * (r + 1) // world) for r in range(world)]
    bounds = [0, n // 3, (2 * n) // 3, n]
    ref = O.assemble_counting(ii, jj, s, m, n)
    dev = torch.device("cuda", 0)
    a = sa.default_assembler(0)
    for rank in range(world):
        lo, hi = bounds[rank], bounds[rank + 1]

        def block(c0, c1):
            sel = (jj[c0:c1] > lo) & (jj[c0:c1] <= hi)
            return tuple(torch.from_numpy(np.ascontiguousarray(x[c0:c1][sel])).to(dev) for x in (ii, jj, s))

        lower = [block(*chunks[r]) for r in range(rank)]
        higher = [block(*chunks[r]) for r in range(rank + 1, world)]
        cat = lambda parts: tuple(torch.cat([p[q] for p in parts]) for q in range(3))  # noqa: E731
        c0, c1 = chunks[rank]
        own = tuple(torch.from_numpy(np.ascontiguousarray(x[c0:c1])).to(dev) for x in (ii, jj, s))
        segs = ([cat(lower)] if lower else []) + [own] + ([cat(higher)] if higher else [])
        got = _assemble_segments_cuda(a, segs, lo, m, hi - lo).to_host()
        k0, k1 = ref.jc[lo], ref.jc[hi]
        assert np.array_equal(got.jc, ref.jc[lo:hi + 1] - k0)
        assert np.array_equal(got.ir, ref.ir[k0:k1])
        assert got.pr.tobytes() == ref.pr[k0:k1].tobytes()


def test_sharded_path_one_rank_nccl():
    """assemble_sharded through the CUDA partition / NCCL exchange / CUDA
    local assembly (world 1 on the one GPU) == the oracle."""
    import socket

    import torch.distributed as dist

    from paper_1406_1066_b200 import workloads as W
    from paper_1406_1066_b200.distributed import assemble_sharded, gpu_local_assembler

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        w = W.fem3d(7)
        dev = torch.device("cuda", 0)
        res = assemble_sharded(w.ii.to(dev), w.jj.to(dev), w.s.to(dev), w.m, w.n, gpu_local_assembler(0))
        ref = O.assemble_counting(w.ii.numpy(), w.jj.numpy(), w.s.numpy(), w.m, w.n)
        assert res.col_lo == 0 and res.col_hi == w.n and res.nnz_total == ref.nnz
        assert np.array_equal(res.jc.cpu().numpy(), ref.jc)
        assert np.array_equal(res.ir.cpu().numpy(), ref.ir)
        assert res.pr.cpu().numpy().tobytes() == ref.pr.tobytes()
        with pytest.raises(sa.BadIndex):
            bad = w.jj.clone()
            bad[5] = 0
            assemble_sharded(w.ii.to(dev), bad.to(dev), w.s.to(dev), w.m, w.n, gpu_local_assembler(0))
    finally:
        dist.destroy_process_group()


def test_long_columns_with_spans_beyond_the_packed_key():
    """Long columns (25..256 triplets) whose row span (rows 1 .. 2^31-1) and
    position span (> 2^25) do not fit the packed 64-bit bitonic key take the
    serial fallback; also long columns of every length class, duplicates
    across the whole input, NaN values."""
    rng = np.random.default_rng(21)
    L = 34_000_000
    ii = rng.integers(1, 1000, size=L).astype(np.int32)
    jj = rng.integers(1, 2_000_001, size=L).astype(np.int32)  # short columns (~17 each)
    s = rng.standard_normal(L)
    # column 5: 100 triplets split between the start and the end of the input:
    # 31 row bits + 26 position bits + 7 slot bits > 63
    idx = np.concatenate([np.arange(0, 50), np.arange(L - 50, L)])
    jj[idx] = 5
    ii[idx] = rng.choice(np.array([1, 2, 2**31 - 1, 2**31 - 2], np.int64), size=100).astype(np.int32)
    # columns 7 / 8 / 9: 40 / 100 / 200 triplets with ordinary spans and duplicates
    for col, cnt in ((7, 40), (8, 100), (9, 200)):
        sel = rng.choice(L // 2, size=cnt, replace=False) + (L // 4)
        sel = sel[jj[sel] > 9]
        jj[sel] = col
        ii[sel] = rng.integers(1, 12, size=len(sel))
    s[rng.random(L) < 1e-6] = np.nan
    dev = torch.device("cuda", 0)
    got = sa.default_assembler(0).assemble_device(*(torch.from_numpy(x).to(dev) for x in (ii, jj, s)),
                                                  m=2**31 - 1, n=2_000_000).to_host()
    ref = O.assemble_sorted(ii, jj, s, 2**31 - 1, 2_000_000)
    _same(got, ref)


def _dataset_digests():
    import json

    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                           "dataset_digests.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("k", range(6))
def test_reference_bench_datasets_bit_exact(k):
    """The reference's own benchmark datasets (bench.py:27-81, values all 1.0,
    heavy duplication): GPU output == the reference's assemble_serial output
    (tests/golden/dataset_digests.json)."""
    from paper_1406_1066_b200 import workloads as W

    d = _dataset_digests()[k]
    ii, jj, s = W.ransparse(d["siz"], d["nnz_row"], d["nrep"], d["seed"])
    out = sa.assemble(ii, jj, s)
    assert (out.m, out.n, out.nnz) == (d["m"], d["n"], d["nnz"])
    assert output_digest(out.jc, out.ir, out.pr) == d["output"]


def _oracle_checkers():
    def check(ii, jj, s, m, n):
        ii = np.asarray(ii)
        jj = np.asarray(jj)
        if m is None:
            m = int(ii.max()) if len(ii) else 0
            n = int(jj.max()) if len(jj) else 0
        return O.assemble_counting(ii.astype(np.int32), jj.astype(np.int32),
                                   np.asarray(s, dtype=np.float64), m, n)
    return [("oracle", check)]


def test_cli_assemble_verify_bench(tmp_path, monkeypatch, capsys):
    """The CLI end to end on the GPU: gen -> assemble (+ --prune-zeros) ->
    the written CSC equals the oracle's; verify --random / --input with the
    test oracle standing in for the reference package (exit 0, and exit 2 on
    a planted mismatch); bench writes the reference's CSV schema."""
    import csv

    from paper_1406_1066_b200 import cli
    from paper_1406_1066_b200 import workloads as W
    from paper_1406_1066_b200.mmio import BENCH_CSV_COLUMNS

    t = tmp_path / "t.mtx"
    a = tmp_path / "a.mtx"
    assert cli.main(["gen", "--size", "300", "--nnz-row", "4", "--nrep", "3", "--out", str(t)]) == 0
    assert cli.main(["assemble", "--input", str(t), "--output", str(a)]) == 0
    ii, jj, s = W.ransparse(300, 4, 3)
    ref = O.assemble_counting(ii, jj, s, 300, 300)
    lines = a.read_text().splitlines()
    assert lines[1] == f"300 300 {len(ref.ir)}"
    rr = np.array([list(map(float, x.split())) for x in lines[2:]])
    assert np.array_equal(rr[:, 0].astype(np.int64) - 1, ref.ir)
    assert np.array_equal(rr[:, 1].astype(np.int64) - 1, np.repeat(np.arange(300), np.diff(ref.jc)))
    assert np.array_equal(rr[:, 2], ref.pr)
    # explicit larger shape and pruning (values are all >= 1: nothing dropped)
    assert cli.main(["assemble", "--input", str(t), "--output", str(a), "--m", "310", "--n", "305",
                     "--prune-zeros"]) == 0
    assert a.read_text().splitlines()[1].startswith("310 305 ")
    assert cli.main(["assemble", "--input", str(t), "--output", str(a), "--m", "10", "--n",
                     "10"]) == 1  # DimensionTooSmall

    dev = torch.device("cuda", 0)
    with pytest.raises(TypeError):  # the device API takes int32 indices only
        sa.default_assembler(0).assemble_device(torch.ones(3, dtype=torch.int64, device=dev),
                                                torch.ones(3, dtype=torch.int32, device=dev),
                                                torch.ones(3, dtype=torch.float64, device=dev))

    monkeypatch.setattr(cli, "reference_checkers", lambda threads: _oracle_checkers())
    assert cli.main(["verify", "--random", "12", "--seed", "3"]) == 0
    assert cli.main(["verify", "--input", str(t)]) == 0

    def wrong(ii, jj, s, m, n):
        c = _oracle_checkers()[0][1](ii, jj, s, m, n)
        pr = np.array(c.pr, copy=True)
        pr[-1] += 1.0
        return sa.CscMatrix(c.jc, c.ir, pr, c.m, c.n)

    monkeypatch.setattr(cli, "reference_checkers", lambda threads: [("planted", wrong)])
    assert cli.main(["verify", "--input", str(t)]) == 2
    assert "first differing pr slot" in capsys.readouterr().err

    b = tmp_path / "b.csv"
    assert cli.main(["bench", "--dataset", "3", "--scale", "0.02", "--reps", "2", "--out",
                     str(b)]) == 0
    rows = list(csv.DictReader(open(b)))
    assert list(rows[0].keys()) == BENCH_CSV_COLUMNS
    assert rows[0]["impl"].startswith("b200") and int(rows[0]["nnz"]) == 9965


@pytest.mark.parametrize("opt,val", [("FOLD_STAGED", 0), ("FOLD_STAGED", 1),
                                     ("SCATTER_STAGED", 0), ("SCATTER_STAGED", 1),
                                     ("PATH", 0), ("PATH", 1), ("RPASS_TMA", 0), ("RPASS_TMA", 1)])
def test_pipeline_variants_bit_exact(opt, val):
    """Every variant a context option can force gives the reference's bits:
    the fold's chained tile offsets vs staged outputs (k_tile_emit), the
    plain vs shared-memory-staged column scatter (k_scatter_staged, chosen
    automatically only for N > 2^24, i.e. cfg5), and the two pipelines
    (column-cursor vs column-block radix path, sa_radix.cu; with the radix
    path the sweep's 1x1..7x7 matrices with ~50k-long runs go through its
    oversize sub-bucket kernel), and the radix passes with register-loaded
    or TMA-staged input (k_rpass / k_rpass_tma; RPASS_TMA applies when the
    radix path runs, so these two variants also force it).  Whole acceptance sweep, the reference's
    datasets, scaled FEM / heavy-duplicate workloads and full-size cfg2 /
    cfg3."""
    from paper_1406_1066_b200 import _capi
    from paper_1406_1066_b200 import workloads as W

    a = sa.default_assembler(0)
    a.set_option(getattr(_capi, "SA_OPT_" + opt), val)
    if opt == "RPASS_TMA":
        a.set_option(_capi.SA_OPT_PATH, 1)
    try:
        kw, rows = sweep("acceptance")
        bad = []
        for r in rows:
            ii, jj, sr = random_triplets(r["seed"], **kw)
            out = sa.assemble(ii.astype(np.int32), jj.astype(np.int32), sr)
            if output_digest(out.jc, out.ir, out.pr) != r["output"]:
                bad.append(r["seed"])
        assert bad == []
        for d in _dataset_digests():
            ii, jj, s = W.ransparse(d["siz"], d["nnz_row"], d["nrep"], d["seed"])
            out = sa.assemble(ii, jj, s)
            assert output_digest(out.jc, out.ir, out.pr) == d["output"], d
        dev = torch.device("cuda", 0)
        for w in (W.fem3d(30, device=dev), W.heavy_dup(m=20_000, positions=200_000, device=dev),
                  W.fem2d(64, device=dev), W.config(2, device=dev), W.config(3, device=dev)):
            out = a.assemble_device(w.ii, w.jj, w.s, m=w.m, n=w.n)
            ref = O.assemble_counting(w.ii.cpu().numpy(), w.jj.cpu().numpy(), w.s.cpu().numpy(),
                                      w.m, w.n)
            _same(out.to_host(), ref)
            del w, out, ref
    finally:
        a.set_option(getattr(_capi, "SA_OPT_" + opt), -1)
        a.set_option(_capi.SA_OPT_PATH, -1)


@pytest.mark.skipif(not stock.available(), reason="oracle/_ref (stock reference) not installed")
@pytest.mark.parametrize("k", [4, 5])
def test_full_size_bit_exact_vs_stock_reference(k):
    """north_star: bit-exact CSC on all five configs.  cfg4 (heavy-duplicate,
    L ~ 5e8) and cfg5 (2D FEM N = 8000, L = 1.152e9) at FULL size against the
    unmodified reference package (oracle/_ref: stock assemble_parallel over
    its compiled kernels, all host threads; bit-identical to its serial
    driver for every p, test_acceptance.py:135-154): jc / ir equal, pr equal
    byte for byte -- through the automatically chosen pipeline and through
    the other one (cfg4: radix path chosen, column-cursor path forced;
    cfg5: the other way round)."""
    from paper_1406_1066_b200 import _capi
    from paper_1406_1066_b200 import workloads as W

    dev = torch.device("cuda", 0)
    a = sa.default_assembler(0)
    w = W.config(k, device=dev)
    m, n, L = w.m, w.n, w.L
    outs = []
    for path in (-1, 1 if k == 5 else 0):
        a.set_option(_capi.SA_OPT_PATH, path)
        try:
            out = a.assemble_device(w.ii, w.jj, w.s, m=m, n=n)
            outs.append((out.jc.cpu().numpy(), out.ir.cpu().numpy(), out.pr.cpu().numpy()))
            del out
        finally:
            a.set_option(_capi.SA_OPT_PATH, -1)
        torch.cuda.empty_cache()
    ii, jj, s = w.ii.cpu().numpy(), w.jj.cpu().numpy(), w.s.cpu().numpy()
    del w
    torch.cuda.empty_cache()
    ref = stock.parallel(stock.request(ii, jj, s, m, n), stock.host_threads())
    del ii, jj, s
    assert (ref.m, ref.n) == (m, n)
    for jc, ir, pr in outs:
        assert np.array_equal(jc, ref.jc)
        assert np.array_equal(ir, ref.ir)
        assert pr.tobytes() == np.asarray(ref.pr).tobytes()
    if k == 5:
        assert len(outs[0][1]) == 448_048_001 and L == 1_152_000_000


@pytest.mark.parametrize("width", [40, 90, 200])
def test_nan_payloads_in_hash_folded_columns(width):
    """Columns of `width` triplets over few distinct rows (the hash-group
    fold) whose row groups mix several NaN payloads, +-inf (inf - inf),
    -0.0 and ordinary values: every group's sum must carry the x86 payload
    rule (the first NaN the ordered sum meets), bit for bit with the C
    oracle.  The plain-add chain re-folds exactly only for NaN sums."""
    rng = np.random.default_rng(width)
    n, rows = 300, 12
    jj = np.repeat(np.arange(1, n + 1, dtype=np.int32), width)
    ii = rng.integers(1, rows + 1, size=len(jj)).astype(np.int32)
    perm = rng.permutation(len(jj))
    ii, jj = ii[perm], jj[perm]
    s = rng.standard_normal(len(jj))
    payloads = np.array([0x7FF8000000000001, 0x7FF8000000000ABC, 0xFFF8000000000123,
                         0x7FF0000000000007], dtype=np.uint64).view(np.float64)  # last: signalling
    pick = rng.random(len(jj))
    s[pick < 0.02] = rng.choice(payloads, size=int((pick < 0.02).sum()))
    s[(pick >= 0.02) & (pick < 0.03)] = np.inf
    s[(pick >= 0.03) & (pick < 0.04)] = -np.inf
    s[(pick >= 0.04) & (pick < 0.05)] = -0.0
    got = sa.assemble(ii, jj, s, m=rows, n=n)
    ref = O.assemble_counting(ii, jj, s, rows, n)
    assert np.array_equal(got.jc, ref.jc) and np.array_equal(got.ir, ref.ir)
    assert got.pr.tobytes() == ref.pr.tobytes()
    assert np.isnan(ref.pr).sum() > 10  # the case does exercise NaN groups


@pytest.mark.parametrize("world,self_rank", [(2, 1), (5, 0)])
def test_partition_unaligned_inputs(world, self_rank):
    """sa_partition on index arrays that are not 16-byte aligned (views one
    element into a buffer): the scalar-load path, same result as the torch
    restatement."""
    import ctypes

    from paper_1406_1066_b200.assembly import _ptr
    from paper_1406_1066_b200.distributed import partition_torch

    rng = np.random.default_rng(world + 10)
    L, n = 50_003, 4_000
    ii = rng.integers(1, 700, size=L + 1).astype(np.int32)
    jj = np.sort(rng.integers(1, n + 1, size=L + 1)).astype(np.int32)
    s = rng.standard_normal(L + 1)
    bounds = [n * r // world for r in range(world + 1)]
    dev = torch.device("cuda", 0)
    ti, tj, ts = (torch.from_numpy(x).to(dev)[1:] for x in (ii, jj, s))  # 4 / 8-byte offsets
    assert ti.data_ptr() % 16 and tj.data_ptr() % 16
    a = sa.default_assembler(0)
    a._bind_stream()
    outs = [torch.empty(L, dtype=dt, device=dev) for dt in (torch.int32, torch.int32, torch.float64)]
    hb = (ctypes.c_int32 * (world + 1))(*bounds)
    hc = (ctypes.c_int64 * world)()
    bp, bw = ctypes.c_int64(-1), ctypes.c_int(-1)
    rc = a.lib.sa_partition(a.ctx, _ptr(ti), _ptr(tj), _ptr(ts), 1, L, 700, n, world, self_rank, hb,
                            *(_ptr(x) for x in outs), hc, ctypes.byref(bp), ctypes.byref(bw))
    assert rc == 0
    ref, rcounts = partition_torch(torch.from_numpy(ii[1:]), torch.from_numpy(jj[1:]), torch.from_numpy(s[1:]),
                                   bounds, world, self_rank)
    k = len(ref[0])
    assert [hc[r] for r in range(world)] == rcounts
    assert torch.equal(outs[0][:k].cpu(), ref[0]) and torch.equal(outs[1][:k].cpu(), ref[1])
    assert outs[2][:k].cpu().numpy().tobytes() == ref[2].numpy().tobytes()


@pytest.mark.parametrize("m,n,L", [(1_000_000, 1, 2_000_000), (1_000_000, 20, 3_000_000), (1000, 1, 2_000_000),
                                   (5_000_000, 3, 1_500_000), (300, 7, 200_000)])
def test_long_columns_row_split_bit_exact(m, n, L):
    """Few, long columns (the reference's long-run instances, conftest.py:43-45,
    at scale): the automatic choice takes the radix path's row-split plan
    (sub-buckets of 2^z rows of one column, spread over all SMs; a column
    longer than a sub-bucket's capacity per key range goes to k_rbig) --
    bit-exact against the C oracle, jc included for the columns whose start
    lies inside a sub-bucket."""
    from paper_1406_1066_b200 import workloads as W

    w = W.random_coo(m=m, n=n, L=L, seed=m + n)
    got = sa.assemble(w.ii.numpy(), w.jj.numpy(), w.s.numpy(), m=m, n=n)
    ref = O.assemble_counting(w.ii.numpy(), w.jj.numpy(), w.s.numpy(), m, n)
    _same(got, ref)
    assert sa.default_assembler(0).launch_count() > 6  # the radix pipeline ran


@pytest.mark.parametrize("m,n,L", [(5, 5, 400_000), (1000, 1, 6_000_000), (1, 1, 300_000)])
def test_single_key_oversize_sub_buckets_bit_exact(m, n, L):
    """So many repeats per (row, col) that the row-split plan reaches z = 0 (a
    sub-bucket is one key) and every sub-bucket exceeds the fold's capacity:
    k_rbig folds each run in input order with one warp (no sort) -- the
    reference's long-run instances (conftest.py:43-45) at scale, with NaN and
    -0.0 among the values; bit-exact against the C oracle."""
    rng = np.random.default_rng(L + m)
    ii = rng.integers(1, m + 1, size=L).astype(np.int32)
    jj = rng.integers(1, n + 1, size=L).astype(np.int32)
    s = rng.standard_normal(L)
    s[rng.random(L) < 1e-4] = -0.0
    if m == 5:
        s[(ii == 2) & (jj == 3) & (rng.random(L) < 1e-3)] = np.nan
    from paper_1406_1066_b200 import _capi

    ref = O.assemble_counting(ii, jj, s, m, n)
    a = sa.default_assembler(0)
    for path in (-1, 1):  # the automatic choice, and the radix path forced
        a.set_option(_capi.SA_OPT_PATH, path)
        try:
            got = a.assemble(ii, jj, s, m=m, n=n)
        finally:
            a.set_option(_capi.SA_OPT_PATH, -1)
        _same(got, ref)
    assert a.launch_count() > 6  # the radix pipeline ran


@pytest.mark.parametrize("nan_at", [None, 100_000, 5])
@pytest.mark.parametrize("m,n", [(200_000, 200_000), (300, 300)])
def test_heavy_hitter_entry_bit_exact(m, n, nan_at):
    """One (row, col) entry holds half of 600 000 triplets among random ones:
    its run of repeats is folded in input order by one warp (warp_fold_run:
    plain adds per block of 32, redone by the x86 NaN rule when the sum turns
    NaN) in k_rbig (radix path) and k_bigcol (column-cursor path); NaNs with
    distinct payloads inside the run pin the rule.  Both pipelines forced,
    bit-exact against the C oracle."""
    from paper_1406_1066_b200 import _capi

    L = 600_000
    rng = np.random.default_rng(m + (nan_at or 0))
    ii = rng.integers(1, m + 1, size=L).astype(np.int32)
    jj = rng.integers(1, n + 1, size=L).astype(np.int32)
    hot = np.flatnonzero(rng.random(L) < 0.5)
    ii[hot] = 7
    jj[hot] = n - 1
    s = rng.standard_normal(L)
    s[hot[::1000]] = -0.0
    if nan_at is not None:
        pay = np.array([0x7FF8000000000123, 0xFFF8000000000456, 0x7FF0000000000789], dtype=np.uint64).view(np.float64)
        s[hot[nan_at]] = pay[0]
        s[hot[nan_at + 40]] = pay[1]
        s[hot[nan_at + 3000]] = pay[2]  # (signalling: quieted by the first add that meets it)
    ref = O.assemble_counting(ii, jj, s, m, n)
    a = sa.default_assembler(0)
    for path in (0, 1):
        a.set_option(_capi.SA_OPT_PATH, path)
        try:
            got = a.assemble(ii, jj, s, m=m, n=n)
        finally:
            a.set_option(_capi.SA_OPT_PATH, -1)
        _same(got, ref)


@pytest.mark.parametrize("tma", [1, 0])
def test_three_pass_radix_plan_bit_exact(tma):
    """2e8 columns: the radix plan needs three partition passes (28 column
    bits above 256-column sub-buckets), so the middle pass both reads and
    writes the {row, col} pair buffers and the second and third upsweeps read
    their columns out of the pairs -- with TMA-staged and register-loaded
    passes, bit-exact against the C oracle."""
    import ctypes

    from paper_1406_1066_b200 import _capi

    m, n, P, reps = 50_000, 200_000_000, 1_000_000, 4
    rng = np.random.default_rng(77)
    pi = rng.integers(1, m + 1, size=P).astype(np.int32)
    pj = rng.integers(1, n + 1, size=P).astype(np.int32)
    pj[:1000] = n  # the last column, repeated
    sel = rng.permutation(np.repeat(np.arange(P), reps))
    ii, jj = pi[sel], pj[sel]
    s = rng.standard_normal(len(ii))
    ref = O.assemble_counting(ii, jj, s, m, n)
    a = sa.default_assembler(0)
    a.set_option(_capi.SA_OPT_PATH, 1)
    a.set_option(_capi.SA_OPT_RPASS_TMA, tma)
    a.lib.sa_enable_timing(a.ctx, 1)
    try:
        got = a.assemble(ii, jj, s, m=m, n=n)
        arr = (ctypes.c_float * 16)()
        names = (ctypes.c_char_p * 16)()
        nk = a.lib.sa_last_kernel_times(a.ctx, 16, arr, names)
        ran = [names[k].decode() for k in range(nk)]
    finally:
        a.lib.sa_enable_timing(a.ctx, 0)
        a.set_option(_capi.SA_OPT_PATH, -1)
        a.set_option(_capi.SA_OPT_RPASS_TMA, -1)
    _same(got, ref)
    assert "k_rpass2" in ran and "k_rpass3" not in ran, ran


def test_host_dims_inferred_during_chunked_upload():
    """Dimension inference fused into the upload (sa_host_upload runs the
    validation / maxima pass over each landed chunk while the next one is
    copied; sa_host_dims only reads it): inferred m, n over a multi-chunk
    input, and a bad index in a later chunk reported at its GLOBAL position
    (reference types.py:121-138, 161-165)."""
    rng = np.random.default_rng(11)
    L = 40_000_000
    ii = rng.integers(1, 70_001, size=L, dtype=np.int32)
    jj = rng.integers(1, 50_001, size=L, dtype=np.int32)
    s = np.ones(L)
    ii[123] = 90_000  # the row maximum, in the first chunk
    jj[L - 5] = 60_000  # the column maximum, in the last chunk
    out = sa.assemble(ii, jj, s)
    assert (out.m, out.n) == (90_000, 60_000)
    assert int(out.jc[-1]) == len(out.ir) and float(out.pr.sum()) == float(L)
    jj[35_000_001] = 0
    ii[39_000_002] = -2
    with pytest.raises(sa.BadIndex) as e:  # rows before columns
        sa.assemble(ii, jj, s)
    assert (e.value.position, e.value.value) == (39_000_002, -2)
    ii[39_000_002] = 5
    with pytest.raises(sa.BadIndex) as e:
        sa.assemble(ii, jj, s)
    assert (e.value.position, e.value.value) == (35_000_001, 0)


def test_concurrent_contexts_on_one_device():
    """Several contexts (one per host thread, sa_create each; the kernels'
    shared-memory attributes are set per (kernel, device) under a lock) run
    assemblies concurrently on device 0 -- column-cursor inputs with big
    columns (k_bigcol's 64 KB dynamic shared memory), shuffled inputs on the
    radix path and long columns on its row-split plan -- each bit-exact."""
    import threading

    from paper_1406_1066_b200 import workloads as W

    cases = [W.heavy_dup(m=30_000, positions=600_000, seed=21), W.fem3d(12),
             W.random_coo(m=200_000, n=3, L=400_000, seed=22), W.random_coo(m=2000, n=50, L=120_000, seed=23)]
    refs = [O.assemble_counting(w.ii.numpy(), w.jj.numpy(), w.s.numpy(), w.m, w.n) for w in cases]
    errors = []

    def run(k):
        try:
            a = sa.Assembler(0)  # a fresh context in this thread
            for _ in range(3):
                for w, ref in zip(cases[k:] + cases[:k], refs[k:] + refs[:k]):
                    got = a.assemble(w.ii.numpy(), w.jj.numpy(), w.s.numpy(), m=w.m, n=w.n)
                    _same(got, ref)
            a.close()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert errors == []


def _fuzz_case(seed):
    """A random shape: dimensions from 1 to 3e6, lengths up to 6e5, with
    duplication, skew (a few heavy columns / rows), scalar values, NaN and
    signed zeros, sometimes column-ordered (FEM-like) runs."""
    rng = np.random.default_rng(seed)
    m = int(rng.choice([1, 3, 17, 1000, 65_537, 3_000_000]))
    n = int(rng.choice([1, 2, 29, 1000, 65_535, 2_000_000]))
    L = int(rng.integers(0, 600_000))
    ii = rng.integers(1, m + 1, size=L)
    jj = rng.integers(1, n + 1, size=L)
    kind = seed % 5
    if kind == 1 and L:  # heavy duplicates
        k = max(1, L // 7)
        pick = rng.integers(0, k, size=L)
        ii, jj = ii[:k][pick], jj[:k][pick]
    elif kind == 2 and L:  # a few heavy columns
        heavy = rng.random(L) < 0.6
        jj[heavy] = rng.integers(1, min(n, 4) + 1, size=int(heavy.sum()))
    elif kind == 3 and L:  # column-ordered runs
        jj = np.sort(jj)
    s = rng.standard_normal(L)
    if L:
        s[rng.random(L) < 0.01] = np.nan
        s[rng.random(L) < 0.01] = -0.0
    if seed % 7 == 0:
        s = np.array([0.1])  # scalar value
    return ii.astype(np.int32), jj.astype(np.int32), s, m, n


@pytest.mark.parametrize("seed", list(range(64)))
def test_fuzz_both_pipelines_bit_exact(seed):
    """Random shapes through both pipelines (column-cursor and radix, each
    forced; the radix path picks its column-block or row-split plan by
    shape) against the C oracle, bit for bit."""
    from paper_1406_1066_b200 import _capi

    ii, jj, s, m, n = _fuzz_case(seed)
    sv = np.full(len(ii), s[0]) if len(s) == 1 and len(ii) != 1 else s
    ref = O.assemble_counting(ii, jj, sv, m, n)
    a = sa.default_assembler(0)
    for path in (0, 1):
        a.set_option(_capi.SA_OPT_PATH, path)
        try:
            got = a.assemble(ii, jj, s, m=m, n=n)
        finally:
            a.set_option(_capi.SA_OPT_PATH, -1)
        _same(got, ref)


@pytest.mark.parametrize("path", [0, 1])
def test_unaligned_device_views_bit_exact(path):
    """Device views that start one element into their buffers (not 16-byte
    aligned): the radix passes fall back from TMA staging to register loads,
    the column pass and scatter to scalar loads -- same bits as the oracle."""
    from paper_1406_1066_b200 import _capi
    from paper_1406_1066_b200 import workloads as W

    dev = torch.device("cuda", 0)
    for w in (W.heavy_dup(m=50_000, positions=400_000, seed=31), W.fem2d(40)):
        ii, jj, s = (x.to(dev) for x in (w.ii, w.jj, w.s))
        ii2 = torch.cat([ii[:1], ii])[1:]
        jj2 = torch.cat([jj[:1], jj])[1:]
        s2 = torch.cat([s[:1], s])[1:]
        assert ii2.data_ptr() % 16 != 0
        a = sa.default_assembler(0)
        a.set_option(_capi.SA_OPT_PATH, path)
        try:
            got = a.assemble_device(ii2, jj2, s2, m=w.m, n=w.n).to_host()
        finally:
            a.set_option(_capi.SA_OPT_PATH, -1)
        _same(got, O.assemble_counting(w.ii.numpy(), w.jj.numpy(), w.s.numpy(), w.m, w.n))
