"""GPU cost curves for the reference's predictor.

The reference prices the "sv" backend as

    gates x sv_coef(class, n) x 2^n  +  c1 + c2 x shots        (predictor.py:62-74)

with per-gate coefficients from timing one numpy `apply_1q` / `apply_2q` call
per gate (`calibration.py:215-228`) and a shot line fitted on a small terminal
circuit (`calibration.py:290-347`).  On the device a gate is never run alone:
`svb_apply` fuses a whole gate list into HBM passes, so the per-gate price is
measured on a *program* of the same gates (rx cycling over the qubits, cx over
neighbouring pairs, as `_sv_point` does) and divided by its gate count and
2^n.  The shot line is fitted through `statevector.run` exactly like the
reference fits its own.

`calibrate(base)` returns the reference's `CalibrationModel` with the sv curves
(over a grid that extends to the device's capacity) and the sv shot line
replaced by device measurements; the mps / stab entries and alpha come from
`base` (e.g. `polysim.calibration.CalibrationModel.load(...)`), since those
backends stay on the host.  `sv_section()` returns just the sv numbers as a
plain dict (usable without the reference installed).  `device_qubit_cap()` is
the largest n whose state (plus the permutation spare buffer) fits in free
device memory — the number a GPU-aware predictor would use instead of the
module constant `DEFAULT_QUBIT_CAP` (kept at 26 for drop-in behaviour, see
polysim_shim.install(qubit_cap=...)).
"""
from __future__ import annotations

import itertools
import statistics
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import statevector as sv
from .circuit import Circuit
from .gates import single_qubit_matrix, two_qubit_matrix

MODEL_VERSION = 1  # calibration.py:28


@dataclass(frozen=True)
class GpuSvConfig:
    sv_grid: tuple[int, ...] = (2, 4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24, 26, 28, 30)
    shot_counts: tuple[int, ...] = (1, 10, 100, 1000)  # calibration.py:42
    repetitions: int = 5                                # calibration.py:43
    min_sample_seconds: float = 5e-4                     # calibration.py:44
    gates_per_program: int = 256
    precision: str = "c128"
    device: int = 0


def median_seconds(fn, reps: int, min_seconds: float) -> float:
    """Median per-call time, looping each sample past the timer floor
    (the reference's `_median_seconds`, calibration.py:48-62)."""
    samples = []
    for _ in range(reps):
        k = 1
        while True:
            t0 = time.perf_counter()
            for _ in range(k):
                fn()
            dt = time.perf_counter() - t0
            if dt >= min_seconds or k >= 1 << 22:
                samples.append(dt / k)
                break
            k *= 2
    return statistics.median(samples)


def _positive(v: float) -> float:
    return max(float(v), 1e-15)  # calibration.py:65-70: coefficients must be > 0


def _program_1q(n: int, g: int) -> np.ndarray:
    rx = single_qubit_matrix("rx", (0.3,))
    qubits = itertools.cycle(range(n))
    return np.concatenate([sv._single_gate((next(qubits),), rx) for _ in range(g)])


def _program_2q(n: int, g: int) -> np.ndarray:
    cx = two_qubit_matrix("cx")
    pairs = itertools.cycle([(q, (q + 1) % n) for q in range(n)])
    return np.concatenate([sv._single_gate(next(pairs), cx) for _ in range(g)])


def sv_point(n: int, cfg: GpuSvConfig = GpuSvConfig()) -> tuple[float, float]:
    """(seconds per 1q gate per amplitude, seconds per 2q gate per amplitude)
    for a fused program of `gates_per_program` gates applied to a resident
    n-qubit state (the device analogue of `_sv_point`, calibration.py:215-228)."""
    if n < 2:
        raise ValueError("sv_point needs n >= 2")
    g = cfg.gates_per_program
    s = sv.DeviceState(n, cfg.precision, cfg.device)
    try:
        p1, p2 = _program_1q(n, g), _program_2q(n, g)

        def run(p):
            s.apply_gates(p)
            _lib.check(_lib.lib().svb_sync(s.handle))

        run(p1), run(p2)  # JIT compile / warm-up outside the samples
        t1 = median_seconds(lambda: run(p1), cfg.repetitions, cfg.min_sample_seconds)
        t2 = median_seconds(lambda: run(p2), cfg.repetitions, cfg.min_sample_seconds)
    finally:
        s.close()
    dim = float(1 << n)
    return _positive(t1 / (g * dim)), _positive(t2 / (g * dim))


def terminal_workload() -> Circuit:
    """The reference's shot-fit circuit (calibration.py:290-303)."""
    c = Circuit(6, 6)
    c.gate("h", 0)
    for q in range(5):
        c.gate("cx", q, q + 1)
    c.gate("h", 3)
    c.gate("s", 4)
    c.measure_all()
    return c


def fit_shot_model(shot_counts, seconds) -> tuple[float, float]:
    """Least-squares (c1, c2) for seconds ~ c1 + c2 * shots (calibration.py:320-328)."""
    x = np.asarray(shot_counts, dtype=float)
    y = np.asarray(seconds, dtype=float)
    if x.shape != y.shape or x.size < 2:
        raise ValueError("need matching shot counts and timings, at least two points")
    (c1, c2), *_ = np.linalg.lstsq(np.column_stack([np.ones(x.size), x]), y, rcond=None)
    return float(c1), float(c2)


def fit_shot_coeffs(cfg: GpuSvConfig = GpuSvConfig()) -> tuple[float, float]:
    """Shot line of `statevector.run` on the device (calibration.py:331-347)."""
    c = terminal_workload()
    medians = [median_seconds(lambda s=shots: sv.run(c, s, seed=11), cfg.repetitions, cfg.min_sample_seconds)
               for shots in cfg.shot_counts]
    c1, c2 = fit_shot_model(cfg.shot_counts, medians)
    return _positive(c1), _positive(c2)


def qubit_cap_for_bytes(free_bytes: int, precision: str = "c128", spare: bool = True) -> int:
    """Largest n whose state (and, with `spare`, the permutation buffer) fits."""
    s = 16 if precision == "c128" else 8
    need = 2 if spare else 1
    n = 0
    while need * s * (1 << (n + 1)) <= free_bytes:
        n += 1
    return n


def device_qubit_cap(precision: str = "c128", device: int = 0) -> int:
    """Device capacity in qubits: the largest state that fits in free device
    memory with 12.5% headroom (`svb_max_qubits`).  Programs that end in a
    qubit relabeling also need the spare buffer (see qubit_cap_for_bytes)."""
    out = _lib.c_int()
    _lib.check(_lib.lib().svb_max_qubits(device, sv._prec_code(precision), _lib.ctypes.byref(out)))
    return int(out.value)


def sv_section(cfg: GpuSvConfig = GpuSvConfig()) -> dict:
    """Device sv curves + shot line, in the reference's to_dict() layout."""
    cap = device_qubit_cap(cfg.precision, cfg.device)
    grid = tuple(n for n in cfg.sv_grid if 2 <= n <= cap)
    c1q, c2q = [], []
    for n in grid:
        a, b = sv_point(n, cfg)
        c1q.append(a)
        c2q.append(b)
    # per-amplitude costs fall with n until launch overhead is amortised; the
    # reference interpolates them with PCHIP (interpolate.py:27-41), no shape needed
    c1, c2 = fit_shot_coeffs(cfg)
    return {
        "sv": {"grid_n": list(grid), "curves": {"1q": c1q, "2q": c2q}},
        "shots": {"sv": {"c1": c1, "c2": c2}},
        "device": {"qubit_cap": cap, "precision": cfg.precision},
    }


def merge_sv_section(base, section: dict):
    """A CalibrationModel equal to `base` (model or to_dict() dict) with the sv
    curves and the sv shot line taken from `section` (see sv_section)."""
    raw = base.to_dict() if hasattr(base, "to_dict") else dict(base)
    raw = {**raw, "sv": section["sv"], "shots": {**raw["shots"], **section["shots"]}}
    try:
        from polysim.calibration import CalibrationModel  # type: ignore
    except ImportError:
        return raw
    return CalibrationModel.from_dict(raw)


def calibrate(base, cfg: GpuSvConfig = GpuSvConfig()):
    """The reference model `base` with its sv entries measured on the device."""
    return merge_sv_section(base, sv_section(cfg))


__all__ = ["GpuSvConfig", "sv_point", "fit_shot_coeffs", "fit_shot_model", "terminal_workload",
           "qubit_cap_for_bytes", "device_qubit_cap", "sv_section", "merge_sv_section", "calibrate"]
