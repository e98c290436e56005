"""Kernel-level numpy API on device-resident memory: zero_state() arrays live
in CUDA managed memory and the reference's per-call kernels
(`apply_1q` / `apply_2q` / `apply_instruction` / `marginal_probs` /
`_measure_qubit`, statevector.py:33-154) run on them in place, so callers
like calibration.py:215-228 time kernels, not PCIe copies."""
import json
import os
import sys
import time

import numpy as np
import pytest

from conftest import ROOT, reference_src
from oracle import sv_oracle as orc
from paper_2512_04216_b200 import calibration as cal
from paper_2512_04216_b200 import statevector as sv
from paper_2512_04216_b200 import suite
from paper_2512_04216_b200.gates import single_qubit_matrix, two_qubit_matrix

pytestmark = pytest.mark.gpu


def test_zero_state_is_device_resident_and_correct():
    n = 12
    amps = sv.zero_state(n)
    assert amps.ctypes.data in sv._views and amps[0] == 1 and np.count_nonzero(amps) == 1
    ref = orc.zero_state(n)
    c = suite.random_circuit(n, 150, np.random.default_rng(4), measured=False)
    for inst in c.instructions:
        sv.apply_instruction(amps, n, inst)
        orc.apply_instruction(ref, n, inst)
    assert np.linalg.norm(amps - ref) / np.linalg.norm(ref) < 1e-10
    np.testing.assert_allclose(sv.marginal_probs(amps, n, (1, 5, 7)), orc.marginal_probs(ref, n, (1, 5, 7)),
                               atol=1e-13)
    r1, r2 = np.random.default_rng(9), np.random.default_rng(9)
    assert sv._measure_qubit(amps, n, 3, r1) == orc.measure_qubit(ref, n, 3, r2)
    np.testing.assert_allclose(amps, ref, atol=1e-12)
    assert r1.random() == r2.random()
    # host writes are seen by the next device call (unified memory)
    amps[:] = 0
    amps[5] = 1
    sv.apply_1q(amps, n, 0, single_qubit_matrix("x"))
    assert amps[4] == 1 and np.count_nonzero(amps) == 1


def test_resident_calls_avoid_host_copies():
    n = 20
    rx = single_qubit_matrix("rx", (0.3,))
    cx = two_qubit_matrix("cx")
    res = sv.zero_state(n)
    plain = np.zeros(1 << n, dtype=np.complex128)
    plain[0] = 1

    def per_call(a, reps=40):
        sv.apply_1q(a, n, 0, rx)
        t0 = time.perf_counter()
        for i in range(reps):
            sv.apply_1q(a, n, i % n, rx)
            sv.apply_2q(a, n, i % n, (i + 1) % n, cx)
        return (time.perf_counter() - t0) / (2 * reps)

    t_res, t_copy = per_call(res), per_call(plain)
    np.testing.assert_allclose(res, plain, atol=1e-12)
    rec = {"n": n, "resident_s_per_call": t_res, "copy_s_per_call": t_copy, "speedup": t_copy / t_res}
    # the reference's own calibration point through the shim, next to the fused device figure
    src = reference_src()
    if src is not None:
        sys.path.insert(0, src)
        try:
            import polysim.calibration as ref_cal

            from paper_2512_04216_b200 import polysim_shim

            polysim_shim.install()
            try:
                t1, t2 = ref_cal._sv_point(n, 3, 0.02)
            finally:
                polysim_shim.uninstall()
            d1, d2 = cal.sv_point(n, cal.GpuSvConfig(repetitions=3, min_sample_seconds=0.02))
            rec.update({"shimmed_ref_sv_point_s_per_amp": [t1, t2], "device_sv_point_s_per_amp": [d1, d2],
                        "ratio_1q": t1 / d1, "ratio_2q": t2 / d2})
        finally:
            sys.path.remove(src)
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "resident_calls.json"), "w") as fh:
            json.dump(rec, fh)
    assert t_res * 5 < t_copy, rec
