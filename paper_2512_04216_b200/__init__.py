"""B200-native state-vector backend for the Maestro / polysim simulator.

Drop-in for `polysim.statevector`; all arithmetic runs
in the in-tree sm_100a library libsvb.so.
"""
from . import circuit, gates, result, suite  # noqa: F401
from .circuit import Circuit, Instruction  # noqa: F401
from .result import BackendError, NoMeasurementsError, QubitCapError, RunResult  # noqa: F401

__all__ = ["Circuit", "Instruction", "RunResult", "BackendError", "NoMeasurementsError", "QubitCapError"]
