"""Readers for the committed golden fixtures (tests/golden/*.json)."""

from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def from_hex(xs):
    return np.array([int(x, 16) for x in xs], dtype=np.uint64).view(np.float64)


def small_cases():
    """[(name, i, j, s, m, n, expected dict(jc, ir, pr, m, n))]"""
    d = _load("small_cases.json")
    out = []
    for c in d["cases"]:
        i = np.array(c["i"], dtype=np.float64 if c["i_float"] else np.int64)
        j = np.array(c["j"], dtype=np.float64 if c["i_float"] else np.int64)
        s = from_hex(c["s_hex"])
        exp = dict(jc=np.array(c["jc"], np.int32), ir=np.array(c["ir"], np.int32),
                   pr=from_hex(c["pr_hex"]), m=c["out_m"], n=c["out_n"])
        out.append((c["name"], i, j, s, c["m"], c["n"], exp))
    return out


def error_cases():
    d = _load("small_cases.json")
    out = []
    for e in d["errors"]:
        i = np.array(e["i"], dtype=np.float64) if e["i_float"] else np.array(e["i"], dtype=np.float64).astype(np.int64)
        j = np.array(e["j"], dtype=np.float64).astype(np.int64)
        out.append((e["name"], i, j, np.array(e["s"]), e["m"], e["n"], e["exc"], e["position"]))
    return out


def sweep(name="acceptance"):
    d = _load("sweep_digests.json")[name]
    return d["kwargs"], d["instances"]


def workloads():
    return _load("workload_digests.json")
