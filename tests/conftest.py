"""Shared test helpers.

* ``gpu`` marker: tests that need a B200 (run with ``-m gpu`` on the GPU box).
* golden fixtures (tests/golden/*, produced by the real reference with
  tests/golden/make_golden.py) loaded into this package's IR.
* chi-square helpers restating the reference's (`tests/conftest.py:154-212`).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

# a JIT compile failure must fail the test instead of silently running the
# interpreter body (the library reads this when it first JIT-compiles)
os.environ.setdefault("SVB_JIT_STRICT", "1")
from scipy import stats

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2512_04216_b200.circuit import Circuit, Instruction  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")

# the frozen reference suite runs in its own pytest process (its conftest.py
# would shadow this one): tests/test_gpu_reference_suite.py
collect_ignore = ["reference_suite"]


def reference_src():
    """Directory holding the reference package `polysim`: the offline install
    baseline/_ref (travels to the GPU box) or the read-only source tree."""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "polysim")):
            return p
    return None


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def load_circuit(spec) -> Circuit:
    c = Circuit(spec["n_qubits"], spec["n_clbits"], name=spec["name"])
    for kind, qs, ps, cl in spec["instructions"]:
        c.append(Instruction(kind, tuple(qs), tuple(ps), cl))
    return c


_cache: dict = {}


def golden(name: str):
    if name not in _cache:
        path = os.path.join(GOLDEN, name)
        if name.endswith(".json"):
            with open(path) as fh:
                _cache[name] = json.load(fh)
        else:
            _cache[name] = dict(np.load(path))
    return _cache[name]


def golden_circuits() -> dict:
    return {k: load_circuit(v) for k, v in golden("circuits.json").items()}


def chisquare_pvalue(counts, expected, shots) -> float:
    """One-sample chi-square with pooling to expected >= 5 (conftest.py:154-184)."""
    support = sorted(set(expected) | set(counts))
    obs = np.array([counts.get(k, 0) for k in support], dtype=float)
    pr = np.array([expected.get(k, 0.0) for k in support], dtype=float)
    keep = pr > 0
    if not keep.all() and obs[~keep].sum() > 0:
        return 0.0
    obs, pr = obs[keep], pr[keep]
    order = np.argsort(pr)
    obs, pr = obs[order], pr[order] * shots
    po, pe, ao, ae = [], [], 0.0, 0.0
    for o, e in zip(obs, pr):
        ao += o
        ae += e
        if ae >= 5:
            po.append(ao)
            pe.append(ae)
            ao = ae = 0.0
    if ae > 0 and pe:
        po[-1] += ao
        pe[-1] += ae
    elif ae > 0:
        po, pe = [ao], [ae]
    if len(pe) < 2:
        return 1.0
    return float(stats.chisquare(po, pe)[1])


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def rng():
    return np.random.default_rng(20260816)
