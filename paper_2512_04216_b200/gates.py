"""Gate matrices, numerically identical to the reference (`polysim/gates.py`).

Global phases matter for amplitude parity, so every definition reproduces the
reference's exact formula and evaluation order:

* fixed one-qubit gates ............ `gates.py:15-24`
* rx / ry (cos, -i sin) ............ `gates.py:43-50`
* rz = diag(e^{-i t/2}, e^{+i t/2}) . `gates.py:51-55`
* u(t, p, l) ....................... `gates.py:56-65`
* cx / cz / swap ................... `gates.py:28-36`

Two-qubit matrices use the reference's little-endian local basis: row/column
index = bit(first listed qubit) + 2 * bit(second listed qubit) (`gates.py:3-5`).
"""
from __future__ import annotations

import math

import numpy as np

_R = 1.0 / math.sqrt(2.0)


def _m(rows) -> np.ndarray:
    return np.array(rows, dtype=np.complex128)


_CONST_1Q = {
    "h": _m([[_R, _R], [_R, -_R]]),
    "x": _m([[0, 1], [1, 0]]),
    "y": _m([[0, -1j], [1j, 0]]),
    "z": _m([[1, 0], [0, -1]]),
    "s": _m([[1, 0], [0, 1j]]),
    "sdg": _m([[1, 0], [0, -1j]]),
    "t": _m([[1, 0], [0, np.exp(1j * math.pi / 4)]]),
    "tdg": _m([[1, 0], [0, np.exp(-1j * math.pi / 4)]]),
}

_perm4 = lambda p: _m([[1 if p[r] == c else 0 for c in range(4)] for r in range(4)])  # noqa: E731

_CONST_2Q = {
    # |c,t> with index c + 2t: cx maps 1 -> 3 and 3 -> 1.
    "cx": _perm4([0, 3, 2, 1]),
    "cz": np.diag([1.0, 1.0, 1.0, -1.0]).astype(np.complex128),
    "swap": _perm4([0, 2, 1, 3]),
}


def _rotation(kind: str, params) -> np.ndarray:
    if kind == "rz":
        (t,) = params
        return _m([[np.exp(-0.5j * t), 0], [0, np.exp(0.5j * t)]])
    if kind == "u":
        t, p, l = params
        c, s = math.cos(t / 2), math.sin(t / 2)
        return _m([[c, -np.exp(1j * l) * s], [np.exp(1j * p) * s, np.exp(1j * (p + l)) * c]])
    (t,) = params
    c, s = math.cos(t / 2), math.sin(t / 2)
    if kind == "rx":
        return _m([[c, -1j * s], [-1j * s, c]])
    if kind == "ry":
        return _m([[c, -s], [s, c]])
    raise KeyError(f"not a one-qubit gate kind: {kind}")


def single_qubit_matrix(kind: str, params=()) -> np.ndarray:
    m = _CONST_1Q.get(kind)
    return m if m is not None else _rotation(kind, tuple(params))


def two_qubit_matrix(kind: str) -> np.ndarray:
    if kind not in _CONST_2Q:
        raise KeyError(f"not a two-qubit gate kind: {kind}")
    return _CONST_2Q[kind]


def matrix_of(inst) -> np.ndarray:
    """Matrix of a unitary instruction in the reference's qubit-order convention."""
    if len(inst.qubits) == 1:
        return single_qubit_matrix(inst.kind, inst.params)
    return two_qubit_matrix(inst.kind)
