"""Run results, error types and measurement bookkeeping.

Mirrors `polysim/result.py`: the error hierarchy (`result.py:12-21`), the
`RunResult` record (`result.py:24-32`) and the clbit/bitstring conventions
(`result.py:35-47,64-82`): bitstrings print the lowest measured clbit
rightmost, width = number of distinct measured clbits, and when several
measures write one clbit the last one wins.

When the reference package is importable its classes are reused, so code
that catches ``polysim.result.QubitCapError`` keeps working after the swap.
"""
from __future__ import annotations

from dataclasses import dataclass, field

try:  # drop-in: share the reference's types when it is installed
    from polysim.result import (  # type: ignore
        BackendError,
        NoMeasurementsError,
        QubitCapError,
        RunResult,
    )
except ImportError:  # standalone (e.g. on the GPU box)

    class BackendError(RuntimeError):
        """A backend could not execute the circuit it was given."""

    class NoMeasurementsError(BackendError):
        """The circuit measures nothing."""

    class QubitCapError(BackendError):
        """The circuit needs more qubits than the backend will hold."""

    @dataclass
    class RunResult:
        counts: dict
        shots: int
        backend: str
        seed: int
        wall_time: float
        predicted_time: float | None = None
        metadata: dict = field(default_factory=dict)


def measurement_map(c) -> list[tuple[int, int]]:
    """(qubit, clbit) for every measure, in program order."""
    return [(i.qubits[0], i.clbit) for i in c.instructions if i.kind == "measure"]


def clbit_order(measures) -> list[int]:
    return sorted({cl for _, cl in measures})


def pack_bitstring(values: dict, clbits: list[int]) -> str:
    return "".join("1" if values[c] else "0" for c in clbits[::-1])


def output_bit_sources(measures, measured_qubits) -> list[int]:
    """For output bit p (clbit rank p), the bit index of its qubit within the
    sampled marginal index (rank of the qubit among the sorted measured qubits).
    Last measure into a clbit wins (`result.py:64-74`)."""
    src: dict[int, int] = {}
    for q, cl in measures:
        src[cl] = q
    if len(src) > 63:
        raise BackendError("more than 63 measured clbits")
    rank = {q: j for j, q in enumerate(measured_qubits)}
    return [rank[src[cl]] for cl in sorted(src)]


def format_counts(codes, freqs, width: int) -> dict[str, int]:
    """Sorted (code, count) pairs -> {bitstring: count} (`result.py:80-82`)."""
    fmt = f"0{width}b"
    return {format(int(v), fmt): int(k) for v, k in zip(codes, freqs)}
