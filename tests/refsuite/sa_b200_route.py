"""pytest plugin (-p sa_b200_route): run the reference's OWN test files with
its serial driver routed to the B200 library through the drop-in binding
integration/_b200.py, installed as ``sparseasm._b200`` exactly as
INTEGRATION.md §2 tells a maintainer to.

Every ``assemble_serial`` the reference's tests reach -- directly, through
``sparseasm.assemble(..., threads=1)`` or through ``bench.make_impl("serial")``
-- then runs on the GPU; ``assemble_parallel`` and ``assemble_oracle`` stay
the reference's CPU code, so the tests compare GPU output against them.
At the end the plugin prints how many assemblies went to the GPU.
"""

import importlib.util
import os
import sys

import sparseasm
import sparseasm.bench
import sparseasm.serial

_HERE = os.path.dirname(os.path.abspath(__file__))
_SHIM = os.path.join(_HERE, "..", "..", "integration", "_b200.py")

spec = importlib.util.spec_from_file_location("sparseasm._b200", _SHIM)
_b200 = importlib.util.module_from_spec(spec)
sys.modules["sparseasm._b200"] = _b200
spec.loader.exec_module(_b200)


def pytest_configure(config):
    # before the test modules import their names from sparseasm
    sparseasm.assemble_serial = _b200.assemble_b200
    sparseasm.serial.assemble_serial = _b200.assemble_b200
    sparseasm.bench.assemble_serial = _b200.assemble_b200


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"sa_b200_route: {_b200.calls} assemblies ran on the GPU")
