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

Options: ``qubit_cap`` lifts the sv cap everywhere the reference reads it —
the module constant (`predictor.py:63-67`) *and* the defaults that were bound
to it at import time (`dispatch.py:18`, `predictor.py:119`, and the installed
run / final_state / expectation); ``pblock=True`` moves polysim.pblock's block
states to the device; ``sampling=True`` replaces `polysim.sampling.AliasTable`
(and the name `polysim.result` imported, `result.py:9`) with the device table.
"""
from __future__ import annotations

import inspect

from . import statevector as _sv

_NAMES = (
    "run", "final_state", "expectation", "zero_state", "apply_1q", "apply_2q", "apply_instruction",
    "marginal_probs", "_measure_qubit", "_reset_qubit",
)
_saved: dict = {}
_saved_pb: dict = {}
_saved_samp: dict = {}
_saved_defaults: list = []  # (function, __defaults__, __kwdefaults__)


def _set_default(fn, name: str, value) -> None:
    """Rebind the default of parameter `name` of `fn` (restored by uninstall)."""
    params = list(inspect.signature(fn).parameters.values())
    _saved_defaults.append((fn, fn.__defaults__, fn.__kwdefaults__))
    p = next(p for p in params if p.name == name)
    if p.kind == inspect.Parameter.KEYWORD_ONLY:
        kw = dict(fn.__kwdefaults__ or {})
        kw[name] = value
        fn.__kwdefaults__ = kw
        return
    positional = [q for q in params if q.kind in (inspect.Parameter.POSITIONAL_ONLY,
                                                     inspect.Parameter.POSITIONAL_OR_KEYWORD)]
    with_default = [q for q in positional if q.default is not inspect.Parameter.empty]
    defaults = list(fn.__defaults__)
    defaults[with_default.index(p)] = value
    fn.__defaults__ = tuple(defaults)


def _lift_cap(cap: int) -> None:
    import polysim.dispatch as ref_dispatch
    import polysim.predictor as ref_pred
    import polysim.statevector as ref

    from . import dispatch as dev_dispatch

    _saved["DEFAULT_QUBIT_CAP"] = ref.DEFAULT_QUBIT_CAP
    ref.DEFAULT_QUBIT_CAP = cap
    _saved["_dev_cap"] = _sv.DEFAULT_QUBIT_CAP
    _sv.DEFAULT_QUBIT_CAP = cap
    for fn in (ref_dispatch.run_circuit, ref_pred.select_backend, dev_dispatch.run_circuit,
               _sv.run, _sv.run_codes, _sv.final_state, _sv.expectation, _sv.expectations):
        _set_default(fn, "qubit_cap", cap)


def install(qubit_cap=None, pblock: bool = False, sampling: bool = False) -> None:
    """Route polysim's "sv" backend to the device.  `qubit_cap` (an int, or
    "device" for calibration.device_qubit_cap()) lifts the sv qubit cap; by
    default it keeps the reference's 26.  With `pblock=True`, polysim.pblock's
    single-device `run` and `PBlockState` also run on the device
    (paper_2512_04216_b200.pblock); with `sampling=True` the alias tables do."""
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
    if sampling:
        import polysim.result as ref_res
        import polysim.sampling as ref_samp

        from . import sampling as dev_samp

        _saved_samp["sampling"] = ref_samp.AliasTable
        _saved_samp["result"] = ref_res.AliasTable
        ref_samp.AliasTable = dev_samp.AliasTable
        ref_res.AliasTable = dev_samp.AliasTable
    if qubit_cap is not None:
        if qubit_cap == "device":
            from .calibration import device_qubit_cap

            qubit_cap = device_qubit_cap()
        _lift_cap(int(qubit_cap))


def uninstall() -> None:
    import polysim.statevector as ref

    while _saved_defaults:
        fn, d, kw = _saved_defaults.pop()
        fn.__defaults__, fn.__kwdefaults__ = d, kw
    if "_dev_cap" in _saved:
        _sv.DEFAULT_QUBIT_CAP = _saved.pop("_dev_cap")
    for name, fn in _saved.items():
        setattr(ref, name, fn)
    _saved.clear()
    if _saved_pb:
        import polysim.pblock as ref_pb

        for name, fn in _saved_pb.items():
            setattr(ref_pb, name, fn)
        _saved_pb.clear()
    if _saved_samp:
        import polysim.result as ref_res
        import polysim.sampling as ref_samp

        ref_samp.AliasTable = _saved_samp["sampling"]
        ref_res.AliasTable = _saved_samp["result"]
        _saved_samp.clear()


def installed() -> bool:
    return bool(_saved)
