"""Fixtures for the reference's standard benchmark datasets.

Run in the build container (where /root/reference exists):

    python tests/golden/make_dataset_golden.py

For each (dataset id, scale, seed) below it records the digest of the
reference generator's triplets (sparseasm.bench.gen_ransparse,
bench.py:62-81) and of the reference's assemble_serial output on them
(compiled Cython kernels from oracle/_ref), into dataset_digests.json.
Tests check paper_1406_1066_b200.workloads.ransparse against the input
digests (CPU) and the GPU path against the output digests.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import _import_reference  # noqa: E402

CASES = [(1, 0.05, 20151023), (1, 1.0, 20151023), (2, 0.01, 20151023), (2, 0.1, 7),
         (3, 0.02, 20151023), (3, 0.1, 11)]


def main():
    sparseasm, _ = _import_reference()
    import sparseasm.bench  # noqa: F401
    from instances import input_digest, output_digest

    out = []
    for ds, scale, seed in CASES:
        spec = sparseasm.bench.dataset_config(ds, scale, seed)
        t = sparseasm.bench.gen_ransparse(spec)
        req = sparseasm.AssemblyRequest(t)
        a = sparseasm.assemble_serial(req)
        out.append(dict(dataset=ds, scale=scale, seed=seed, siz=spec.siz, nnz_row=spec.nnz_row,
                        nrep=spec.nrep, L=len(t), nnz=a.nnz, m=a.m, n=a.n,
                        input=input_digest(t.ii, t.jj, t.sr),
                        output=output_digest(a.jc, a.ir, a.pr)))
        print(out[-1])
    with open(os.path.join(HERE, "dataset_digests.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
