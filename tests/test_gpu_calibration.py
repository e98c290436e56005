"""Device sv cost curves for the reference's predictor."""
import json

import pytest

from paper_2512_04216_b200 import calibration as cal


@pytest.mark.gpu
def test_sv_section_on_device():
    cfg = cal.GpuSvConfig(sv_grid=(2, 8, 14, 20), repetitions=2, min_sample_seconds=1e-4, gates_per_program=64)
    sec = cal.sv_section(cfg)
    json.dumps(sec)
    assert sec["sv"]["grid_n"] == [2, 8, 14, 20]
    for k in ("1q", "2q"):
        vals = sec["sv"]["curves"][k]
        assert len(vals) == 4 and all(v > 0 for v in vals)
        # per-amplitude cost falls as launch overhead amortises over 2^n amplitudes
        assert vals[-1] < vals[0]
    assert sec["shots"]["sv"]["c1"] > 0 and sec["shots"]["sv"]["c2"] > 0
    assert sec["device"]["qubit_cap"] >= 30  # a B200 holds >= 33 qubits at c128
