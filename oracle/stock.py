"""TEST INFRASTRUCTURE ONLY -- the UNMODIFIED reference package.

``oracle/_ref/`` holds the reference's own package ``sparseasm`` (its Python
drivers and its Cython kernels compiled from its own sources by its own
setup.py; recipe: ``oracle/Makefile`` target ``ref``).  This module only
locates and imports it; every call below goes through the reference's public
API and stock code path:

* ``AssemblyRequest.from_raw``  (types.py:93-100) -- built once, outside
  any timing, as the reference's ``run_bench`` does (bench.py:146-160)
* ``assemble_serial``           (serial.py:111-168)
* ``assemble_parallel(req, p)`` (parallel.py:361-389)

Users: bench.py (``cpu_baseline`` and ``--impl reference``) and the tests
(the full-size parity oracle).  The product package never imports it.
"""

from __future__ import annotations

import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
_mod = None


def module():
    """Import ``sparseasm`` from oracle/_ref (ImportError if not installed)."""
    global _mod
    if _mod is None:
        if not os.path.exists(os.path.join(REF_DIR, "sparseasm", "__init__.py")):
            raise ImportError(f"reference package not installed under {REF_DIR} "
                              "(run: make -C oracle ref, in the build container)")
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import sparseasm  # noqa: E402

        if not os.path.abspath(sparseasm.__file__).startswith(REF_DIR):
            raise ImportError(f"a different sparseasm shadows oracle/_ref: {sparseasm.__file__}")
        from sparseasm import backend

        if backend.name() != "c":
            raise ImportError("reference compiled kernels are not active (backend "
                              f"{backend.name()!r})")
        _mod = sparseasm
    return _mod


def available() -> bool:
    try:
        module()
        return True
    except ImportError:
        return False


def request(ii, jj, s, m, n):
    """The reference's validated request (types.py:93-100)."""
    sa = module()
    return sa.AssemblyRequest.from_raw(ii, jj, s, m, n)


def serial(req):
    """Stock ``assemble_serial`` (serial.py:111-168) -> reference CscMatrix."""
    return module().assemble_serial(req)


def parallel(req, p: int):
    """Stock ``assemble_parallel(req, p)`` (parallel.py:361-389)."""
    return module().assemble_parallel(req, p)


def host_threads() -> int:
    return len(os.sched_getaffinity(0))
