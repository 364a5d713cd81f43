"""Generate the committed parity fixtures from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``sparseasm`` installed unmodified into
oracle/_ref/ (its drivers plus its Cython kernels compiled from its own
sources: oracle/Makefile target ``ref``) and writes, next to this script:

  sweep_digests.json    the acceptance sweep (reference
                        test_acceptance.py:33-35, 50-51): for seeds
                        1_000_000 + k, k < 1000, the digest of the
                        reference's random_instance inputs and of the
                        reference's assemble_serial output, plus m, n, L, nnz;
                        and the same for the 40 seeds of test_serial.py:138-144
  small_cases.json      explicit inputs and reference outputs (values as
                        IEEE-754 hex so NaN payloads survive): golden example
                        (conftest.py:7-13), README example, test_serial.py
                        small cases, order-sensitive, scalar, NaN/Inf/-0.0
  workload_digests.json reference outputs for scaled BASELINE workloads
                        produced by paper_1406_1066_b200.workloads on CPU

Nothing on the GPU box reads /root/reference; tests only read these files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_TESTS = "/root/reference/pkg/tests"

sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _import_reference():
    from oracle import stock

    sparseasm = stock.module()  # the unmodified reference package (oracle/_ref)

    assert sparseasm.backend.name() == "c", "reference compiled kernels not active"
    sys.path.insert(0, REF_TESTS)
    import conftest as ref_conftest

    return sparseasm, ref_conftest


def hexf(a):
    return [format(int(x), "016x") for x in np.asarray(a, dtype=np.float64).view(np.uint64)]


def main():
    sparseasm, ref_conftest = _import_reference()
    from instances import (SWEEP_COUNT, SWEEP_SEED_BASE, input_digest, output_digest,
                           random_triplets)

    def ref_out(req):
        a = sparseasm.assemble_serial(req)
        b = sparseasm.assemble_serial(req, kernels=sparseasm.backend.get("python"))
        assert a.same_as(b)
        return a

    # --- sweeps -----------------------------------------------------------
    sweeps = {}
    for name, seeds, kw in (
        ("acceptance", [SWEEP_SEED_BASE + k for k in range(SWEEP_COUNT)],
         dict(max_len=50_000, max_dim=2000)),
        ("serial40", list(range(40)), dict(max_len=3000, max_dim=200)),
    ):
        rows = []
        for seed in seeds:
            req = ref_conftest.random_instance(seed, **kw)
            t = req.triplets
            ii, jj, sr = random_triplets(seed, **kw)
            din = input_digest(t.ii, t.jj, t.sr)
            assert din == input_digest(ii, jj, sr), f"generator restatement differs at {seed}"
            out = ref_out(req)
            rows.append(dict(seed=seed, L=len(t), m=out.m, n=out.n, nnz=out.nnz, input=din,
                             output=output_digest(out.jc, out.ir, out.pr)))
        sweeps[name] = dict(kwargs=kw, instances=rows)
    with open(os.path.join(HERE, "sweep_digests.json"), "w") as f:
        json.dump(sweeps, f, indent=0)

    # --- explicit small cases -------------------------------------------
    nan = float("nan")
    cases = [
        ("golden_example", ref_conftest.EXAMPLE_I, ref_conftest.EXAMPLE_J, ref_conftest.EXAMPLE_S, None, None),
        ("readme_example", [3, 1, 3], [1, 2, 1], [5.0, 2.0, 1.0], None, None),
        ("sorted_example", ref_conftest.SORTED_I, ref_conftest.SORTED_J, ref_conftest.SORTED_S, None, None),
        ("empty", [], [], [], None, None),
        ("empty_explicit", [], [], [], 3, 4),
        ("single", [3], [2], [1.5], None, None),
        ("seven_dups", [2] * 7, [3] * 7, list(np.arange(7.0)), None, None),
        ("order_1e16_first", [1, 1, 1], [1, 1, 1], [1e16, 1.0, 1.0], None, None),
        ("order_1e16_last", [1, 1, 1], [1, 1, 1], [1.0, 1.0, 1e16], None, None),
        ("single_column", [3, 1, 2], [1, 1, 1], [1.0, 2.0, 3.0], None, None),
        ("padded_dims", [1], [1], [4.0], 3, 5),
        ("scalar_tenth", [1] * 10, [1] * 10, [0.1], None, None),
        ("scalar_mixed", [1, 2, 1, 2, 1], [1, 1, 1, 2, 1], [0.1], None, None),
        ("neg_zero_alone", [1], [1], [-0.0], None, None),
        ("neg_zero_pair", [1, 1, 2], [1, 1, 1], [-0.0, -0.0, 0.0], None, None),
        ("nan_isolated", [1, 2, 1], [1, 1, 1], [nan, 5.0, 1.0], None, None),
        ("inf_minus_inf", [1, 1], [1, 1], [float("inf"), float("-inf")], None, None),
        ("cancel_to_zero", [1, 1, 2], [1, 1, 1], [2.0, -2.0, 5.0], None, None),
        ("float_indices", [1.0, 3.0], [2.0, 2.0], [5.0, 6.0], None, None),
        ("denormals", [1, 1, 2], [1, 1, 1], [5e-324, 5e-324, 1e-310], None, None),
    ]
    # NaN payload / sign cases (bits matter: reference keeps the first NaN)
    u = np.array([0xFFF8000000000001, 0x7FF8000000000002, 0x3FF0000000000000,
                  0x7FF0000000000000, 0xFFF0000000000000, 0x7FF4000000000000], dtype=np.uint64)
    cases.append(("nan_payloads", [1, 1, 1, 2, 2, 3], [1, 1, 1, 1, 1, 1], list(u.view(np.float64)), None, None))
    out_cases = []
    for name, i, j, s, m, n in cases:
        req = sparseasm.AssemblyRequest.from_raw(i, j, s, m=m, n=n)
        out = ref_out(req)
        out_cases.append(dict(
            name=name,
            i=[float(x) if isinstance(x, float) else int(x) for x in np.asarray(i).tolist()],
            j=[float(x) if isinstance(x, float) else int(x) for x in np.asarray(j).tolist()],
            i_float=bool(np.asarray(i).dtype.kind == "f"),
            s_hex=hexf(np.atleast_1d(np.asarray(s, dtype=np.float64))),
            m=m, n=n,
            out_m=out.m, out_n=out.n, jc=out.jc.tolist(), ir=out.ir.tolist(), pr_hex=hexf(out.pr)))
    # error cases (reference behaviour: exception class and position)
    errs = []
    for name, i, j, s, m, n in (
        ("bad_zero_row", [1, 0, 2], [1, 1, 1], [1.0, 1.0, 1.0], None, None),
        ("bad_first_position", [1, 2, 0, 0], [1, 1, 1, 1], [0.0] * 4, None, None),
        ("bad_col_negative", [1, 1], [1, -1], [1.0, 1.0], None, None),
        ("bad_row_and_col", [1, 1, -5], [0, 1, 1], [1.0, 1.0, 1.0], None, None),
        ("bad_half", [1, 0.5, 2], [1, 1, 1], [1.0, 1.0, 1.0], None, None),
        ("bad_nan", [1, nan, 2], [1, 1, 1], [1.0, 1.0, 1.0], None, None),
        ("bad_inf", [1, float("inf"), 2], [1, 1, 1], [1.0, 1.0, 1.0], None, None),
        ("bad_2p31", [1, 2 ** 31, 2], [1, 1, 1], [1.0, 1.0, 1.0], None, None),
        ("dim_too_small", [1, 5], [1, 2], [1.0, 1.0], 4, 2),
        ("dim_too_small_col", [1, 2], [1, 3], [1.0, 1.0], 4, 2),
        ("length_mismatch_idx", [1, 2], [1], [1.0, 1.0], None, None),
        ("length_mismatch_val", [1, 2], [1, 1], [1.0, 2.0, 3.0], None, None),
        ("m_without_n", [1], [1], [1.0], 3, None),
    ):
        try:
            req = sparseasm.AssemblyRequest.from_raw(i, j, s, m=m, n=n)
            sparseasm.assemble_serial(req)
            res = dict(exc=None)
        except Exception as exc:  # noqa: BLE001 - recording the reference's behaviour
            res = dict(exc=type(exc).__name__, position=getattr(exc, "position", None))
        errs.append(dict(name=name, i=[float(x) for x in i], i_float=any(isinstance(x, float) for x in i),
                         j=[float(x) for x in j], s=[float(x) for x in s], m=m, n=n, **res))
    with open(os.path.join(HERE, "small_cases.json"), "w") as f:
        json.dump(dict(cases=out_cases, errors=errs), f, indent=0)

    # --- scaled BASELINE workloads ---------------------------------------
    from paper_1406_1066_b200 import workloads as W

    wl = []
    specs = [
        ("fem2d", dict(N=1)), ("fem2d", dict(N=2)), ("fem2d", dict(N=7)), ("fem2d", dict(N=64)),
        ("fem2d", dict(N=300)),
        ("fem3d", dict(N=1)), ("fem3d", dict(N=3)), ("fem3d", dict(N=12)), ("fem3d", dict(N=30)),
        ("random_coo", dict()),
        ("random_coo", dict(m=50, n=40, L=20_000, seed=7)),
        ("heavy_dup", dict(m=20_000, positions=200_000, seed=4)),
        ("heavy_dup", dict(m=300, positions=5_000, mean_rep=40.0, seed=5)),
    ]
    for kind, kw in specs:
        w = getattr(W, kind)(**kw)
        ii, jj, s = w.ii.numpy(), w.jj.numpy(), w.s.numpy()
        req = sparseasm.AssemblyRequest.from_raw(ii, jj, s, m=w.m, n=w.n)
        out = ref_out(req)
        wl.append(dict(kind=kind, kwargs=kw, L=w.L, m=w.m, n=w.n, nnz=out.nnz,
                       input=input_digest(ii, jj, s), output=output_digest(out.jc, out.ir, out.pr)))
    with open(os.path.join(HERE, "workload_digests.json"), "w") as f:
        json.dump(wl, f, indent=0)
    print("wrote", len(sweeps["acceptance"]["instances"]), "sweep digests,", len(out_cases),
          "cases,", len(errs), "error cases,", len(wl), "workloads")


if __name__ == "__main__":
    main()
