"""Install the B200 backend into an existing `polysim` installation.

    import paper_2512_04216_b200.polysim_shim as shim
    shim.install()          # polysim's "sv" backend now runs on the GPU

Replaces the public state-vector functions of `polysim.statevector`
(`statevector.py:33-292`) with this package's, so every caller that reaches
the dense path — `dispatch.run_circuit(c, "sv", ...)` (`dispatch.py:21`), the
batch runner, calibration's kernel timings, pblock's block kernels, metrics —
runs on the device without code changes.  `DEFAULT_QUBIT_CAP` keeps the
reference value, so the predictor's hard-coded cap check behaves the same.
`uninstall()` restores the originals.
"""
from __future__ import annotations

from . import statevector as _sv

_NAMES = (
    "run", "final_state", "expectation", "zero_state", "apply_1q", "apply_2q", "apply_instruction",
    "marginal_probs", "_measure_qubit", "_reset_qubit",
)
_saved: dict = {}
_saved_pb: dict = {}


def install(qubit_cap=None, pblock: bool = False) -> None:
    """Route polysim's "sv" backend to the device.  `qubit_cap` (an int, or
    "device" for calibration.device_qubit_cap()) also raises the module
    constant DEFAULT_QUBIT_CAP that predictor.estimate checks
    (predictor.py:63-67); by default it keeps the reference's 26.  With
    `pblock=True`, polysim.pblock's single-device `run` and `PBlockState`
    also run on the device (paper_2512_04216_b200.pblock)."""
    import polysim.statevector as ref  # noqa: F401  (raises ImportError without polysim)

    if _saved:
        return
    for name in _NAMES:
        _saved[name] = getattr(ref, name)
        setattr(ref, name, getattr(_sv, name))
    _saved["_state_cache"] = ref._state_cache
    ref._state_cache = _sv._state_cache
    if pblock:
        import polysim.pblock as ref_pb

        from . import pblock as dev_pb

        _saved_pb["run"] = ref_pb.run
        _saved_pb["PBlockState"] = ref_pb.PBlockState
        ref_pb.run = dev_pb.run
        ref_pb.PBlockState = dev_pb.PBlockState
    if qubit_cap is not None:
        if qubit_cap == "device":
            from .calibration import device_qubit_cap

            qubit_cap = device_qubit_cap()
        _saved["DEFAULT_QUBIT_CAP"] = ref.DEFAULT_QUBIT_CAP
        ref.DEFAULT_QUBIT_CAP = int(qubit_cap)


def uninstall() -> None:
    import polysim.statevector as ref

    for name, fn in _saved.items():
        setattr(ref, name, fn)
    _saved.clear()
    if _saved_pb:
        import polysim.pblock as ref_pb

        for name, fn in _saved_pb.items():
            setattr(ref_pb, name, fn)
        _saved_pb.clear()


def installed() -> bool:
    return bool(_saved)
