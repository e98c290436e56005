"""CPU oracle for the state-vector hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference `polysim` state-vector algorithm
(`/root/reference/pkg/src/polysim/statevector.py`, `result.py`, `sampling.py`,
`gates.py`).  Each function cites the reference lines it restates.  The
arithmetic (operation order, numpy primitives, RNG consumption) is kept
identical so that, on the same inputs, this module reproduces the reference
bit for bit; `tests/test_oracle_golden.py` pins that against fixtures the real
reference produced (`tests/golden/make_golden.py`).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may
import this module, and only as the checker / the timed CPU baseline.  The
product path (`paper_2512_04216_b200`) never imports it.

Third-party arithmetic: numpy (>= 2.0 for `bitwise_count`); RNG = numpy
`default_rng(seed)` = PCG64 seeded through SeedSequence.
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

DEFAULT_QUBIT_CAP = 26  # statevector.py:30

_S2 = 1.0 / math.sqrt(2.0)
_FIXED = {  # gates.py:15-24, 28-36
    "h": [[_S2, _S2], [_S2, -_S2]],
    "x": [[0, 1], [1, 0]],
    "y": [[0, -1j], [1j, 0]],
    "z": [[1, 0], [0, -1]],
    "s": [[1, 0], [0, 1j]],
    "sdg": [[1, 0], [0, -1j]],
    "t": [[1, 0], [0, np.exp(1j * math.pi / 4)]],
    "tdg": [[1, 0], [0, np.exp(-1j * math.pi / 4)]],
    "cx": [[1, 0, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0], [0, 1, 0, 0]],
    "cz": [[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 1, 0], [0, 0, 0, -1]],
    "swap": [[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]],
}
_FIXED = {k: np.array(v, dtype=complex) for k, v in _FIXED.items()}


class OracleError(RuntimeError):
    pass


class OracleCapError(OracleError):
    pass


class OracleNoMeasurements(OracleError):
    pass


def gate_matrix(kind: str, params=()) -> np.ndarray:
    """gates.py:39-74."""
    if kind in _FIXED:
        return _FIXED[kind]
    if kind == "rz":  # gates.py:51-55
        (t,) = params
        return np.array([[np.exp(-0.5j * t), 0], [0, np.exp(0.5j * t)]], dtype=complex)
    if kind == "u":  # gates.py:56-65
        t, p, l = params
        c, s = math.cos(t / 2), math.sin(t / 2)
        return np.array([[c, -np.exp(1j * l) * s],
                         [np.exp(1j * p) * s, np.exp(1j * (p + l)) * c]], dtype=complex)
    (t,) = params  # rx / ry, gates.py:43-50
    c, s = math.cos(t / 2), math.sin(t / 2)
    if kind == "rx":
        return np.array([[c, -1j * s], [-1j * s, c]], dtype=complex)
    return np.array([[c, -s], [s, c]], dtype=complex)


# --- gate kernels ------------------------------------------------------------

def zero_state(n: int) -> np.ndarray:
    """statevector.py:125-128."""
    psi = np.zeros(1 << n, dtype=complex)
    psi[0] = 1.0
    return psi


def apply_1q(psi, n, q, m) -> None:
    """statevector.py:33-53: diagonal, anti-diagonal, dense paths."""
    v = psi.reshape(-1, 2, 1 << q)
    a0, a1 = v[:, 0, :], v[:, 1, :]
    if m[0, 1] == 0 and m[1, 0] == 0:
        if m[0, 0] != 1:
            a0 *= m[0, 0]
        if m[1, 1] != 1:
            a1 *= m[1, 1]
        return
    if m[0, 0] == 0 and m[1, 1] == 0:
        keep = a0.copy()
        a0[...] = a1
        a1[...] = keep
        if m[0, 1] != 1:
            a0 *= m[0, 1]
        if m[1, 0] != 1:
            a1 *= m[1, 0]
        return
    keep = a0.copy()
    a0[...] = m[0, 0] * keep + m[0, 1] * a1
    a1[...] = m[1, 0] * keep + m[1, 1] * a1


def _quarter(psi, qa, qb):
    """statevector.py:56-68: view of the amplitudes with local index i
    (= bit(qa) + 2 bit(qb))."""
    lo, hi = min(qa, qb), max(qa, qb)
    v = psi.reshape(-1, 2, 1 << (hi - lo - 1), 2, 1 << lo)

    def part(i):
        ba, bb = i & 1, (i >> 1) & 1
        return v[:, bb, :, ba, :] if qa < qb else v[:, ba, :, bb, :]

    return part


def apply_2q(psi, n, qa, qb, m) -> None:
    """statevector.py:71-113: diagonal / generalized permutation / dense."""
    part = _quarter(psi, qa, qb)
    nz = [np.flatnonzero(m[r]) for r in range(4)]
    if all(len(z) == 1 for z in nz):
        src = [int(z[0]) for z in nz]
        if src == [0, 1, 2, 3]:
            for r in range(4):
                if m[r, r] != 1:
                    part(r)[...] *= m[r, r]
            return
        seen = [False] * 4
        for s0 in range(4):  # cycle following, statevector.py:81-104
            if seen[s0]:
                continue
            cyc = [s0]
            j = src[s0]
            while j != s0:
                cyc.append(j)
                j = src[j]
            if len(cyc) == 1:
                if m[s0, s0] != 1:
                    part(s0)[...] *= m[s0, s0]
                seen[s0] = True
                continue
            tmp = part(cyc[-1]).copy()
            for k in range(len(cyc) - 1, 0, -1):
                d, s = cyc[k], cyc[k - 1]
                part(d)[...] = m[d, s] * part(s) if m[d, s] != 1 else part(s)
                seen[d] = True
            f = cyc[0]
            part(f)[...] = m[f, cyc[-1]] * tmp if m[f, cyc[-1]] != 1 else tmp
            seen[f] = True
        return
    tmps = [part(r).copy() for r in range(4)]  # statevector.py:105-113
    for r in range(4):
        acc = None
        for c in range(4):
            if m[r, c] == 0:
                continue
            term = tmps[c] if m[r, c] == 1 else m[r, c] * tmps[c]
            acc = term if acc is None else acc + term
        part(r)[...] = 0 if acc is None else acc


def apply_instruction(psi, n, inst) -> None:
    """statevector.py:116-122."""
    if inst.kind == "barrier":
        return
    if len(inst.qubits) == 1:
        apply_1q(psi, n, inst.qubits[0], gate_matrix(inst.kind, inst.params))
    else:
        apply_2q(psi, n, inst.qubits[0], inst.qubits[1], gate_matrix(inst.kind))


def marginal_probs(psi, n, qubits) -> np.ndarray:
    """statevector.py:131-139."""
    p = np.abs(psi.reshape([2] * n)) ** 2
    keep = set(qubits)
    drop = tuple(n - 1 - q for q in range(n) if q not in keep)
    if drop:
        p = p.sum(axis=drop)
    return p.reshape(-1)


# --- alias sampler (sampling.py:30-83) ---------------------------------------

def alias_table(probs):
    """AliasTable.from_probs, sampling.py:30-70 -> (prob_row, alias_row)."""
    probs = np.asarray(probs, dtype=float)
    if probs.ndim != 1 or probs.size == 0:
        raise ValueError("need a non-empty 1-D probability vector")
    if np.any(probs < 0):
        raise ValueError("negative probability")
    total = probs.sum()
    if not np.isclose(total, 1.0, rtol=0, atol=1e-9):
        raise ValueError(f"probabilities sum to {total}, not 1")
    m = probs.size
    scaled = probs * (m / total)
    prob_row = np.ones(m, dtype=float)
    alias_row = np.arange(m, dtype=np.int64)
    big = scaled > 1.0
    larges = np.flatnonzero(big)
    smalls = np.flatnonzero(~big)
    rem = scaled[larges].copy()
    while smalls.size and larges.size:
        deficit = 1.0 - scaled[smalls]
        owner = np.searchsorted(np.cumsum(rem - 1.0), np.cumsum(deficit), side="left")
        np.clip(owner, 0, larges.size - 1, out=owner)
        prob_row[smalls] = scaled[smalls]
        alias_row[smalls] = larges[owner]
        rem = rem - np.bincount(owner, weights=deficit, minlength=larges.size)
        done = rem <= 1.0
        if not done.any():
            break
        smalls = larges[done]
        scaled[smalls] = rem[done]
        larges = larges[~done]
        rem = rem[~done]
    return prob_row, alias_row


def alias_sample(prob_row, alias_row, rng, shots):
    """AliasTable.sample_indices, sampling.py:78-83."""
    v = rng.random(shots) * prob_row.size
    idx = v.astype(np.int64)
    return np.where((v - idx) < prob_row[idx], idx, alias_row[idx])


def sample_terminal(qubits, probs, measures, shots, rng) -> dict:
    """sample_measurement_groups for the sv single-group case, result.py:50-82."""
    pr, al = alias_table(probs)
    idx = alias_sample(pr, al, rng, shots)
    src = {}
    for q, cl in measures:
        src[cl] = q
    clbits = sorted(src)
    if len(clbits) > 63:
        raise OracleError("more than 63 measured clbits")
    pos = {q: j for j, q in enumerate(qubits)}
    codes = np.zeros(shots, dtype=np.int64)
    for p, cl in enumerate(clbits):
        codes |= ((idx >> pos[src[cl]]) & 1).astype(np.int64) << p
    vals, freq = np.unique(codes, return_counts=True)
    w = len(clbits)
    return {format(int(v), f"0{w}b"): int(k) for v, k in zip(vals, freq)}


# --- mid-circuit replay (statevector.py:142-179) -----------------------------

def measure_qubit(psi, n, q, rng) -> int:
    v = psi.reshape(-1, 2, 1 << q)
    p1 = float(np.sum(np.abs(v[:, 1, :]) ** 2))
    out = 1 if rng.random() < p1 else 0
    p = p1 if out else 1.0 - p1
    v[:, 1 - out, :] = 0.0
    psi *= 1.0 / np.sqrt(p)
    return out


def reset_qubit(psi, n, q, rng) -> None:
    if measure_qubit(psi, n, q, rng) == 1:
        apply_1q(psi, n, q, _FIXED["x"])


def replay(prefix, n, suffix, shots, rng) -> dict:
    meas = [(i.qubits[0], i.clbit) for i in suffix if i.kind == "measure"]
    clbits = sorted({cl for _, cl in meas})
    out: dict = {}
    for _ in range(shots):
        psi = prefix.copy()
        vals = {}
        for inst in suffix:
            if inst.kind == "measure":
                vals[inst.clbit] = measure_qubit(psi, n, inst.qubits[0], rng)
            elif inst.kind == "reset":
                reset_qubit(psi, n, inst.qubits[0], rng)
            else:
                apply_instruction(psi, n, inst)
        key = "".join(str(vals[c]) for c in reversed(clbits))
        out[key] = out.get(key, 0) + 1
    return out


# --- backend entry points ----------------------------------------------------

def is_terminal(c) -> bool:
    """features.py:41-64."""
    measured = set()
    for inst in c.instructions:
        if inst.kind == "barrier":
            continue
        if inst.kind == "reset":
            return False
        if inst.kind == "measure":
            measured.add(inst.qubits[0])
        elif any(q in measured for q in inst.qubits):
            return False
    return True


def unitary_state(c) -> np.ndarray:
    n = c.n_qubits
    psi = zero_state(n)
    for inst in c.instructions:
        if inst.kind not in ("measure", "reset", "barrier"):
            apply_instruction(psi, n, inst)
    return psi


def run(c, shots, seed, workers=1, qubit_cap=DEFAULT_QUBIT_CAP) -> dict:
    """statevector.py:182-253 (returns the counts dict)."""
    if c.n_qubits > qubit_cap:
        raise OracleCapError(f"{c.n_qubits} qubits exceeds the configured cap {qubit_cap}")
    if shots < 1:
        raise ValueError("shots must be positive")
    measures = [(i.qubits[0], i.clbit) for i in c.instructions if i.kind == "measure"]
    if not measures:
        raise OracleNoMeasurements("circuit has no measurements")
    n = c.n_qubits
    if is_terminal(c):
        psi = unitary_state(c)
        qubits = tuple(sorted({q for q, _ in measures}))
        probs = marginal_probs(psi, n, qubits)
        return sample_terminal(qubits, probs, measures, shots, np.random.default_rng(seed))
    split = next(i for i, x in enumerate(c.instructions) if x.kind in ("measure", "reset"))
    prefix = zero_state(n)
    for inst in c.instructions[:split]:
        if inst.kind not in ("barrier",):
            apply_instruction(prefix, n, inst)
    suffix = [x for x in c.instructions[split:] if x.kind != "barrier"]
    workers = max(1, min(workers, shots))
    sizes = [shots // workers + (1 if w < shots % workers else 0) for w in range(workers)]
    if workers == 1:
        return replay(prefix, n, suffix, shots, np.random.default_rng(seed))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        parts = [pool.submit(replay, prefix, n, suffix, sizes[w], np.random.default_rng(seed + w))
                 for w in range(workers)]
        merged: dict = {}
        for f in parts:
            for k, v in f.result().items():
                merged[k] = merged.get(k, 0) + v
    return merged


def expectation_from_state(psi, z_qubits) -> float:
    """statevector.py:288-292."""
    probs = np.abs(psi) ** 2
    mask = np.uint64(sum(1 << q for q in set(z_qubits)))
    idx = np.arange(probs.size, dtype=np.uint64)
    parity = (np.bitwise_count(idx & mask) & np.uint64(1)).astype(float)
    return float(np.sum(probs * (1.0 - 2.0 * parity)))
