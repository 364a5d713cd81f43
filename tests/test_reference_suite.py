"""The reference's own tests, run on the B200 through the drop-in binding.

The reference's test files (copied unmodified next to the stock package by
oracle/Makefile, oracle/_ref/ref_tests/) run in a child pytest with the
plugin tests/refsuite/sa_b200_route.py, which installs integration/_b200.py
as ``sparseasm._b200`` and routes ``assemble_serial`` to it.  Selected:
test_serial.py (small cases, 40 random instances vs the oracle, idempotent
re-assembly, properties; test_serial.py:87-198) and acceptance criteria 1-5
(test_acceptance.py:90-203: the golden example, the 1000-instance sweep
bit-identical to the oracle, determinism against the CPU parallel driver for
p in 1, 2, 3, 4, 8, structural invariants), plus the reference harness
(bench.run_bench, bench.py:132-196) cross-checking the GPU Impl against its
serial CPU driver."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")

needs_ref = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                               reason="oracle/_ref/ref_tests not installed (make -C oracle ref)")


def _env():
    from paper_1406_1066_b200 import _capi

    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests", "refsuite"), ROOT])
    env["SPARSEASM_B200_LIB"] = _capi.library_path()
    return env


@needs_ref
def test_reference_serial_and_acceptance_on_gpu():
    sel = "not criterion_6 and not criterion_7 and not criterion_8 and not criterion_9 " \
          "and not criterion_10"
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "sa_b200_route",
                        "-p", "no:cacheprovider", "test_serial.py", "test_acceptance.py", "-k", sel],
                       cwd=REF_TESTS, env=_env(), capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "failed" not in out.splitlines()[-1]
    n = int(out.split("sa_b200_route: ")[1].split()[0])
    assert n >= 1000, out[-2000:]  # the 1000-instance sweep alone
    for c in (1, 2, 3, 4, 5):
        assert f"acceptance criterion  {c}: PASS" in out


@needs_ref
def test_reference_run_bench_with_b200_impl():
    code = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np
from sparseasm import bench as rb
import sa_b200_route  # installs sparseasm._b200
from sparseasm._b200 import assemble_b200
impl = rb.Impl("b200", 1, lambda req, pt=None: assemble_b200(req))
res = rb.run_bench(rb.dataset_config(1, scale=0.2), [rb.make_impl("serial"), impl], reps=2,
                   dataset_id="1")
assert [r.impl for r in res] == ["serial", "b200"], res
assert res[0].nnz == res[1].nnz > 0
print("run_bench ok", res[1].nnz, res[1].mean_seconds, res[0].mean_seconds)
"""
    r = subprocess.run([sys.executable, "-c", code, os.path.join(ROOT, "tests", "refsuite")],
                       env=_env(), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "run_bench ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
