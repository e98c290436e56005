"""The one circuit feature the state-vector path consumes.

`statevector.run` / `final_state` branch on
`extract_features(c).terminal_measurement_only` (`statevector.py:205-208,266-268`);
the rule is `features.py:41-64`: any reset, or any unitary touching an
already-measured qubit, makes the circuit non-terminal. Unitaries on
*unmeasured* qubits after a measure keep it terminal (`test_features.py:52-54`).
"""
from __future__ import annotations


def terminal_measurement_only(c) -> bool:
    measured: set[int] = set()
    for inst in c.instructions:
        k = inst.kind
        if k == "barrier":
            continue
        if k == "reset":
            return False
        if k == "measure":
            measured.add(inst.qubits[0])
        elif measured and any(q in measured for q in inst.qubits):
            return False
    return True
