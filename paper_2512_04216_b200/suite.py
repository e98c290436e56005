"""Workload generators that emit reference IR.

* ``ghz_circuit`` ........ `polysim/suite.py:11-18` (config 1)
* ``qft`` ................ `tests/conftest.py:23-44` (config 2; cp = cx·u·cx·u·u)
* ``qaoa_line_circuit`` .. `polysim/suite.py:43-62` (config 4)
* ``ry_ansatz_circuit`` .. `polysim/suite.py:65-80` (config 4)
* ``random_circuit`` ..... `tests/conftest.py:47-76` (parity tests)
* ``sycamore_circuit`` ... no reference equivalent (configs 3 and 5):
  a rows×cols grid, per cycle one random gate from {√X, √Y, √W} per qubit
  (as rx(π/2), ry(π/2), u(π/2, -π/4, π/4)) followed by cz on one of four
  coupler patterns (ABCD).

All generators consume numpy ``default_rng`` streams exactly as the reference
does, so a given seed yields the same circuit as the reference generator
(checked in tests against fixtures).
"""
from __future__ import annotations

import math

import numpy as np

from .circuit import Circuit


def ghz_circuit(n: int, measured: bool = True) -> Circuit:
    c = Circuit(n, n if measured else 0, name=f"ghz_{n}")
    c.gate("h", 0)
    for q in range(1, n):
        c.gate("cx", q - 1, q)
    return c.measure_all() if measured else c


def controlled_phase(c: Circuit, theta: float, control: int, target: int) -> None:
    """diag(1,1,1,e^{i theta}) from cx and u(0,0,λ) (`conftest.py:27-33`)."""
    c.gate("cx", control, target)
    c.gate("u", target, params=(0.0, 0.0, -theta / 2))
    c.gate("cx", control, target)
    c.gate("u", target, params=(0.0, 0.0, theta / 2))
    c.gate("u", control, params=(0.0, 0.0, theta / 2))


def qft(n: int, c: Circuit | None = None) -> Circuit:
    c = Circuit(n) if c is None else c
    for t in range(n - 1, -1, -1):
        c.gate("h", t)
        for ctl in range(t - 1, -1, -1):
            controlled_phase(c, math.pi / 2 ** (t - ctl), ctl, t)
    for i in range(n // 2):
        c.gate("swap", i, n - 1 - i)
    return c


def qft_bench_circuit(n: int) -> Circuit:
    """Config 2: ry(0.1·(q+1)) preparation, then qft(n)."""
    c = Circuit(n, name=f"qft_ry_{n}")
    for q in range(n):
        c.gate("ry", q, params=(0.1 * (q + 1),))
    return qft(n, c)


def qaoa_line_circuit(n: int, layers: int, seed: int, measured: bool = True) -> Circuit:
    rng = np.random.default_rng(seed)
    c = Circuit(n, n if measured else 0, name=f"qaoa_line_{n}x{layers}")
    for q in range(n):
        c.gate("h", q)
    for _ in range(layers):
        gamma = float(rng.uniform(0.1, math.pi - 0.1))
        beta = float(rng.uniform(0.1, math.pi - 0.1))
        for q in range(n - 1):
            c.gate("cx", q, q + 1).gate("rz", q + 1, params=(2.0 * gamma,)).gate("cx", q, q + 1)
        for q in range(n):
            c.gate("rx", q, params=(2.0 * beta,))
    return c.measure_all() if measured else c


def ry_ansatz_circuit(n: int, layers: int, seed: int, measured: bool = True) -> Circuit:
    rng = np.random.default_rng(seed)
    c = Circuit(n, n if measured else 0, name=f"ry_ansatz_{n}x{layers}")
    for _ in range(layers + 1):
        for q in range(n):
            c.gate("ry", q, params=(float(rng.uniform(0, 2 * math.pi)),))
        if _ < layers:
            for q in range(n - 1):
                c.gate("cx", q, q + 1)
    return c.measure_all() if measured else c


def batch_workload(count: int, base: int = 0) -> list[Circuit]:
    """Config 4: circuit i is qaoa (even i) or ry-ansatz (odd i) on
    n_i = 12 + (i mod 13) qubits."""
    out = []
    for i in range(base, base + count):
        n = 12 + i % 13
        if i % 2 == 0:
            out.append(qaoa_line_circuit(n, 1 + (i // 2) % 2, seed=i))
        else:
            out.append(ry_ansatz_circuit(n, 2, seed=i))
    return out


_ONE_Q = ("h", "x", "y", "z", "s", "sdg")
_ONE_Q_ALL = _ONE_Q + ("t", "tdg", "rx", "ry", "rz", "u")


def random_circuit(n, n_gates, rng, clifford_only=False, measured=True, two_qubit_fraction=0.35):
    c = Circuit(n, n if measured else 0)
    one_q = list(_ONE_Q if clifford_only else _ONE_Q_ALL)
    two_q = ["cx", "cz", "swap"]
    for _ in range(n_gates):
        if n >= 2 and rng.random() < two_qubit_fraction:
            a, b = rng.choice(n, size=2, replace=False)
            c.gate(str(rng.choice(two_q)), int(a), int(b))
            continue
        kind = str(rng.choice(one_q))
        q = int(rng.integers(n))
        if kind in ("rx", "ry", "rz"):
            c.gate(kind, q, params=(float(rng.uniform(0, 2 * math.pi)),))
        elif kind == "u":
            c.gate(kind, q, params=tuple(rng.uniform(0, 2 * math.pi, size=3)))
        else:
            c.gate(kind, q)
    if measured:
        for q in range(n):
            c.measure(q, q)
    return c


_SQRT_GATES = (("rx", (math.pi / 2,)), ("ry", (math.pi / 2,)), ("u", (math.pi / 2, -math.pi / 4, math.pi / 4)))


def sycamore_circuit(rows: int, cols: int, depth: int, seed: int, measured: bool = True) -> Circuit:
    """Sycamore-style random circuit on a rows×cols grid (qubit = r*cols + c).

    Cycle k: each qubit gets a random √X/√Y/√W that differs from its previous
    one, then cz on coupler pattern "ABCD"[k % 4] (A/B: horizontal pairs with
    even/odd column parity, C/D: vertical pairs with even/odd row parity)."""
    rng = np.random.default_rng(seed)
    n = rows * cols
    c = Circuit(n, n if measured else 0, name=f"sycamore_{rows}x{cols}_d{depth}_s{seed}")
    last = [-1] * n
    for k in range(depth):
        for q in range(n):
            g = int(rng.integers(3))
            if g == last[q]:
                g = (g + 1 + int(rng.integers(2))) % 3
            last[q] = g
            kind, params = _SQRT_GATES[g]
            c.gate(kind, q, params=params)
        pat = k % 4
        for r in range(rows):
            for col in range(cols):
                q = r * cols + col
                if pat < 2 and col + 1 < cols and col % 2 == pat:
                    c.gate("cz", q, q + 1)
                elif pat >= 2 and r + 1 < rows and r % 2 == pat - 2:
                    c.gate("cz", q, q + cols)
    return c.measure_all() if measured else c
