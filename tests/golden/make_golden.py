"""Generate golden fixtures by running the REAL reference (`polysim`) here.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `polysim` from /root/reference/pkg/src and the reference's own
test helpers (`random_circuit`, `qft`, `ghz` from
/root/reference/pkg/tests/conftest.py) and records, for a fixed list of
seeded circuits and inputs:

* circuits.json      — the circuits themselves (kind, qubits, params, clbit)
* amps.npz           — `statevector.final_state(c)` (complex128)
* counts.json        — `statevector.run(c, shots, seed).counts`
* expect.json        — `statevector.expectation(c, z_qubits)`
* kernels.npz        — `apply_1q` / `apply_2q` on random states (all paths)
* alias.npz          — `AliasTable.from_probs` tables and `sample_indices`
* marginals.npz      — `marginal_probs` over qubit subsets

The fixtures are committed; nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path[:0] = [f"{REF}/src", f"{REF}/tests"]
sys.dont_write_bytecode = True

from polysim import statevector as sv  # noqa: E402
from polysim import suite  # noqa: E402
from polysim.circuit import Circuit, Instruction  # noqa: E402
from polysim.gates import single_qubit_matrix, two_qubit_matrix  # noqa: E402
from polysim.sampling import AliasTable  # noqa: E402
import conftest as ref_conftest  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def dump_circuit(c) -> dict:
    return {
        "name": c.name,
        "n_qubits": c.n_qubits,
        "n_clbits": c.n_clbits,
        "instructions": [[i.kind, list(i.qubits), list(i.params), i.clbit] for i in c.instructions],
    }


def main() -> None:
    circuits: dict[str, dict] = {}
    amps: dict[str, np.ndarray] = {}
    counts: dict[str, dict] = {}
    expect: dict[str, list] = {}

    def add_unitary(key, c):
        circuits[key] = dump_circuit(c)
        amps[key] = sv.final_state(c, qubit_cap=max(26, c.n_qubits))

    # 1. random circuits from the reference's own generator (conftest.py:47-76)
    rng = np.random.default_rng(20260816)
    for k in range(40):
        n = int(rng.integers(1, 11))
        c = ref_conftest.random_circuit(n, int(rng.integers(1, 60)), rng, measured=False)
        add_unitary(f"rand_{k}", c)
    # 2. QFT on x-prepared basis states and ry-prepared states (conftest.py:36-44)
    for n in (3, 4, 6, 9, 12):
        basis = (5 * n + 3) % (1 << n)
        c = Circuit(n)
        for q in range(n):
            if (basis >> q) & 1:
                c.gate("x", q)
        for inst in ref_conftest.qft(n).instructions:
            c.append(inst)
        add_unitary(f"qft_x_{n}", c)
        c = Circuit(n)
        for q in range(n):
            c.gate("ry", q, params=(0.1 * (q + 1),))
        for inst in ref_conftest.qft(n).instructions:
            c.append(inst)
        add_unitary(f"qft_ry_{n}", c)
        expect[f"qft_ry_{n}"] = [[[q], sv.expectation(c, (q,))] for q in range(n)] + [
            [[0, 1, 2], sv.expectation(c, (0, 1, 2))]
        ]
    # 3. structured families (suite.py)
    for n in (5, 8, 12):
        add_unitary(f"ghz_{n}", suite.ghz_circuit(n, measured=False))
        add_unitary(f"w_{n}", suite.w_state_circuit(n, measured=False))
        add_unitary(f"qaoa_{n}", suite.qaoa_line_circuit(n, 2, seed=n, measured=False))
        add_unitary(f"ry_{n}", suite.ry_ansatz_circuit(n, 2, seed=n, measured=False))
    # expectation KATs on random circuits
    for k in range(0, 40, 4):
        key = f"rand_{k}"
        spec = circuits[key]
        c = load(spec)
        n = c.n_qubits
        erng = np.random.default_rng(1000 + k)
        rows = []
        for _ in range(4):
            zq = sorted(set(int(x) for x in erng.integers(0, n, size=int(erng.integers(1, n + 1)))))
            rows.append([zq, sv.expectation(c, tuple(zq))])
        expect[key] = rows

    # 4. sampled counts (terminal path, alias sampler, shared PCG64 stream)
    def add_counts(key, c, shots, seeds, workers=1):
        circuits[key] = dump_circuit(c)
        counts[key] = {
            str(s): sv.run(c, shots=shots, seed=s, workers=workers, qubit_cap=max(26, c.n_qubits)).counts
            for s in seeds
        }

    add_counts("ghz20", suite.ghz_circuit(20), 1024, (0, 7, 42))
    add_counts("ghz3", ref_conftest.ghz(3), 2000, (11,))
    crng = np.random.default_rng(5)
    for k in range(12):
        n = int(crng.integers(2, 11))
        c = ref_conftest.random_circuit(n, int(crng.integers(5, 60)), crng)
        add_counts(f"crand_{k}", c, int(crng.integers(1, 20000)), (int(crng.integers(2**31)), 3))
    c = ref_conftest.random_circuit(10, 60, np.random.default_rng(1))
    add_counts("rand10_60", c, 100_000, (5,))
    for n in (6, 12):
        add_counts(f"qaoa_m{n}", suite.qaoa_line_circuit(n, 1, seed=3), 1000, (0, 1))
        add_counts(f"ry_m{n}", suite.ry_ansatz_circuit(n, 2, seed=4), 1000, (0,))
    # subset / crossed / repeated clbit mappings (result.py:64-82)
    c = Circuit(4, 3)
    c.gate("h", 0).gate("cx", 0, 2).gate("ry", 3, params=(0.4,)).gate("h", 1)
    c.measure(0, 2).measure(3, 0).measure(2, 1).measure(1, 1)
    add_counts("mapping_a", c, 5000, (9, 10))
    c = Circuit(5, 6)
    c.gate("h", 4).gate("cx", 4, 1).gate("rx", 2, params=(1.3,))
    c.measure(4, 5).measure(1, 0).measure(2, 3)
    c.gate("ry", 3, params=(0.2,))  # unitary on an unmeasured qubit: still terminal
    add_counts("mapping_b", c, 3000, (2,))
    # mid-circuit replay path (statevector.py:157-250), sequential and fan-out
    c = Circuit(5, 5)
    c.gate("h", 0).gate("cx", 0, 1).gate("ry", 2, params=(0.7,))
    c.measure(0, 0)
    c.append(Instruction("reset", (1,)))
    c.gate("h", 1).gate("cx", 2, 3).gate("u", 4, params=(1.1, 0.3, -0.4))
    c.measure(1, 1).measure(2, 2).measure(3, 3).measure(4, 4)
    add_counts("mid5", c, 4096, (5,))
    c2 = Circuit(2, 3)
    c2.gate("h", 0).gate("cx", 0, 1).measure(0, 0)
    c2.gate("h", 0)
    c2.measure(0, 1).measure(1, 2)
    add_counts("mid2", c2, 1000, (9,))
    add_counts("mid2_w3", c2, 1000, (9,), workers=3)
    c3 = Circuit(1, 1)
    c3.gate("ry", 0, params=(1.0,)).measure(0, 0).gate("x", 0).measure(0, 0)
    add_counts("collapse1", c3, 500, (3,))

    # 5. kernel-level paths (statevector.py:33-113) on random normalised states
    krng = np.random.default_rng(77)
    kern = {}
    mats1 = {
        "h": single_qubit_matrix("h"), "x": single_qubit_matrix("x"), "y": single_qubit_matrix("y"),
        "t": single_qubit_matrix("t"), "rz": single_qubit_matrix("rz", (0.37,)),
        "u": single_qubit_matrix("u", (0.3, 1.2, -0.7)), "rx": single_qubit_matrix("rx", (2.1,)),
        "u00l": single_qubit_matrix("u", (0.0, 0.0, 0.9)),
    }
    mats2 = {"cx": two_qubit_matrix("cx"), "cz": two_qubit_matrix("cz"), "swap": two_qubit_matrix("swap")}
    # a dense 4x4 (never produced by the IR, but apply_2q accepts it) and a
    # generalized permutation with phases
    a = krng.normal(size=(4, 4)) + 1j * krng.normal(size=(4, 4))
    mats2["dense"], _ = np.linalg.qr(a)
    perm = np.zeros((4, 4), dtype=complex)
    for r, c_ in enumerate((2, 0, 3, 1)):
        perm[r, c_] = np.exp(1j * (0.3 + r))
    mats2["phaseperm"] = perm
    case = 0
    for n in (1, 3, 7):
        for name, m in mats1.items():
            for q in range(n):
                psi = krng.normal(size=1 << n) + 1j * krng.normal(size=1 << n)
                psi /= np.linalg.norm(psi)
                out = psi.copy()
                sv.apply_1q(out, n, q, m)
                kern[f"k{case}_in"], kern[f"k{case}_out"] = psi, out
                kern[f"k{case}_meta"] = np.array([1, n, q, -1])
                kern[f"k{case}_mat"] = m
                case += 1
    for n in (2, 4, 6):
        for name, m in mats2.items():
            for qa in range(n):
                for qb in range(n):
                    if qa == qb:
                        continue
                    psi = krng.normal(size=1 << n) + 1j * krng.normal(size=1 << n)
                    psi /= np.linalg.norm(psi)
                    out = psi.copy()
                    sv.apply_2q(out, n, qa, qb, m)
                    kern[f"k{case}_in"], kern[f"k{case}_out"] = psi, out
                    kern[f"k{case}_meta"] = np.array([2, n, qa, qb])
                    kern[f"k{case}_mat"] = m
                    case += 1
    kern["n_cases"] = np.array(case)

    # 6. alias tables (sampling.py:30-83) incl. zeros, spikes, uniform, 2^k sizes
    arng = np.random.default_rng(31)
    alias = {}
    dists = []
    for m in (1, 2, 3, 4, 7, 64, 1000, 4096, 1 << 16):
        p = arng.random(m) ** 3
        dists.append(p / p.sum())
    p = np.zeros(1000)
    p[3] = 0.999
    rest = arng.random(50)
    p[100:150] = 0.001 * rest / rest.sum()
    dists.append(p)
    dists.append(np.full(4, 0.25))
    dists.append(np.array([0.25, 0.75]))
    p = np.zeros(1 << 12)
    p[0] = p[-1] = 0.5
    dists.append(p)
    for k, p in enumerate(dists):
        t = AliasTable.from_probs(p)
        alias[f"a{k}_p"], alias[f"a{k}_prob"], alias[f"a{k}_alias"] = p, t.prob, t.alias
        alias[f"a{k}_draw"] = t.sample_indices(np.random.default_rng(100 + k), 5000)
    alias["n_cases"] = np.array(len(dists))

    # 7. marginals over subsets (statevector.py:131-139)
    mrng = np.random.default_rng(55)
    marg = {}
    for k in range(10):
        n = int(mrng.integers(1, 9))
        psi = mrng.normal(size=1 << n) + 1j * mrng.normal(size=1 << n)
        psi /= np.linalg.norm(psi)
        qs = tuple(sorted(set(int(x) for x in mrng.integers(0, n, size=int(mrng.integers(1, n + 1))))))
        marg[f"m{k}_psi"], marg[f"m{k}_q"] = psi, np.array(qs)
        marg[f"m{k}_out"] = sv.marginal_probs(psi, n, qs)
    marg["n_cases"] = np.array(10)

    with open(os.path.join(OUT, "circuits.json"), "w") as fh:
        json.dump(circuits, fh, separators=(",", ":"))
    with open(os.path.join(OUT, "counts.json"), "w") as fh:
        json.dump(counts, fh, separators=(",", ":"), sort_keys=True)
    with open(os.path.join(OUT, "expect.json"), "w") as fh:
        json.dump(expect, fh, indent=0)
    np.savez_compressed(os.path.join(OUT, "amps.npz"), **amps)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **kern)
    np.savez_compressed(os.path.join(OUT, "alias.npz"), **alias)
    np.savez_compressed(os.path.join(OUT, "marginals.npz"), **marg)
    print("wrote", len(circuits), "circuits,", len(counts), "count sets,", case, "kernel cases")


def load(spec):
    c = Circuit(spec["n_qubits"], spec["n_clbits"], name=spec["name"])
    for kind, qs, ps, cl in spec["instructions"]:
        c.append(Instruction(kind, tuple(qs), tuple(ps), cl))
    return c


if __name__ == "__main__":
    main()
