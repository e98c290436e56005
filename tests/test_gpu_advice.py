"""Regression tests for round-1 review findings: clbit width of
the replay path, the shim's qubit cap reaching every bound default, the
precision key of the final_state cache, and non-finite JIT immediates."""
import math
import sys

import numpy as np
import pytest

from conftest import reference_src
from paper_2512_04216_b200 import _lib, suite
from paper_2512_04216_b200 import statevector as sv
from paper_2512_04216_b200.circuit import Circuit, Instruction
from paper_2512_04216_b200.result import BackendError

pytestmark = pytest.mark.gpu


def test_replay_rejects_more_than_64_clbits():
    """One shot's clbits are packed into a uint64: 65 measured clbits in a
    mid-circuit program must raise, not drop bits (the reference builds
    strings, statevector.py:157-179)."""
    n = 5
    c = Circuit(n, 70)
    c.gate("h", 0)
    c.measure(0, 0)
    c.gate("h", 0)
    for k in range(1, 66):
        c.measure(k % n, k)
    with pytest.raises(BackendError):
        sv.run(c, 10, 0)
    # 64 is fine
    c2 = Circuit(n, 64)
    c2.gate("h", 0)
    c2.measure(0, 0)
    c2.gate("h", 0)
    for k in range(1, 64):
        c2.measure(k % n, k)
    res = sv.run(c2, 50, 0)
    assert sum(res.counts.values()) == 50 and all(len(k) == 64 for k in res.counts)


def test_final_state_cache_is_keyed_by_precision():
    c = suite.random_circuit(12, 80, np.random.default_rng(2), measured=False)
    lo = sv.final_state(c, precision="c64")
    hi = sv.final_state(c)  # default c128: must not return the cached c64 state
    from oracle import sv_oracle as orc

    ref = orc.unitary_state(c)
    assert np.linalg.norm(hi - ref) / np.linalg.norm(ref) < 1e-10
    assert np.linalg.norm(lo - ref) / np.linalg.norm(ref) > 1e-12  # it really was the c64 state
    assert sv._state_cache[c].device.precision == "c128"


def test_jit_immediates_propagate_nan():
    """n >= 28 compiles coefficients as immediates: a NaN gate parameter must
    give NaN amplitudes exactly where the interpreter gives them."""
    n = 28
    c = Circuit(n)
    for q in range(6):
        c.gate("h", q)
    c.gate("u", 3, params=(float("nan"), 0.1, 0.2))
    c.gate("rz", 20, params=(0.3,))
    outs = []
    for jit in (24, -1):
        s = sv.DeviceState(n, "c64")
        s.set_option(_lib.OPT_JIT_MIN_N, jit)
        s.apply_instructions(c.instructions)
        outs.append(s.read(0, 1 << 16))
        s.close()
    a, b = outs
    assert np.isnan(a).any()
    np.testing.assert_array_equal(np.isnan(a), np.isnan(b))


def test_shim_cap_reaches_dispatch_and_predictor():
    """install(qubit_cap=30): polysim.dispatch.run_circuit(c, "sv", ...) runs
    a 27-qubit circuit on the device (its default was bound to 26 at import)."""
    src = reference_src()
    if src is None:
        pytest.skip("reference package absent")
    sys.path.insert(0, src)
    try:
        import polysim.dispatch as ref_dispatch
        from polysim.circuit import Circuit as RefCircuit

        from paper_2512_04216_b200 import polysim_shim

        c = RefCircuit(27, 27)
        c.gate("h", 0)
        for q in range(1, 27):
            c.gate("cx", q - 1, q)
        for q in range(27):
            c.measure(q, q)
        polysim_shim.install(qubit_cap=30)
        try:
            res = ref_dispatch.run_circuit(c, "sv", 200, 3)
        finally:
            polysim_shim.uninstall()
        assert set(res.counts) <= {"0" * 27, "1" * 27} and sum(res.counts.values()) == 200
        from polysim.result import QubitCapError

        with pytest.raises(QubitCapError):
            ref_dispatch.run_circuit(c, "sv", 10, 3)
    finally:
        sys.path.remove(src)


def test_compare_matches_host_distance():
    """svb_compare (device distance/overlap) against numpy on a small pair."""
    rng = np.random.default_rng(5)
    a = sv.DeviceState(12, "c128")
    a.apply_instructions(suite.random_circuit(12, 60, rng, measured=False).instructions)
    b = sv.DeviceState(12, "c64")
    b.apply_instructions(suite.random_circuit(12, 60, rng, measured=False).instructions)
    x, y = a.to_numpy(), b.to_numpy()
    r = a.compare(b)
    assert math.isclose(r["dist2"], float(np.sum(np.abs(x - y) ** 2)), rel_tol=1e-9)
    assert math.isclose(r["fidelity"], abs(np.vdot(x, y)) ** 2 / (np.vdot(x, x).real * np.vdot(y, y).real),
                        rel_tol=1e-9, abs_tol=1e-14)
