"""The reference's own tests for the dense state-vector path —
`tests/test_statevector.py`, `test_sampling.py`, `test_pblock.py` (frozen
unmodified by tests/reference_suite/freeze.py) — run against the B200 backend
installed into the reference through `polysim_shim.install(pblock=True,
sampling=True)` (the reference suite must pass against the
new module).  Runs in its own pytest process because the reference's
conftest.py would shadow ours."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, reference_src

pytestmark = pytest.mark.gpu

SUITE = os.path.join(ROOT, "tests", "reference_suite")
FROZEN = os.path.join(SUITE, "_frozen")


def test_reference_suite_passes_through_shim(tmp_path):
    if not os.path.isfile(os.path.join(FROZEN, "test_statevector.py")):
        sys.path.insert(0, SUITE)
        from freeze import freeze

        if not freeze():
            pytest.skip("frozen reference tests absent (run tests/reference_suite/freeze.py where the reference is)")
    if reference_src() is None:
        pytest.skip("reference package (baseline/_ref) absent")
    report = tmp_path / "report.json"
    env = dict(os.environ, SVB_REFSUITE_REPORT=str(report),
               PYTHONPATH=os.pathsep.join([SUITE, ROOT, os.environ.get("PYTHONPATH", "")]))
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "shim_plugin", "-p", "no:cacheprovider",
         "--rootdir", FROZEN, FROZEN],
        cwd=FROZEN, env=env, capture_output=True, text=True, timeout=1500)
    tail = proc.stdout[-4000:] + proc.stderr[-2000:]
    out_dir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out_dir):
        with open(os.path.join(out_dir, "reference_suite.log"), "w") as fh:
            fh.write(proc.stdout + proc.stderr)
    rep = json.loads(report.read_text())
    assert rep["statevector_is_device"] and rep["pblock_is_device"] and rep["alias_table_is_device"], rep
    assert rep["lib"], rep
    assert proc.returncode == 0, tail
    assert rep["collected"] >= 50, rep
