"""Golden fixtures for the partitioned-block backend, from the REAL reference.

    python tests/golden/make_golden_pblock.py      (build container only)

Records `polysim.pblock.run(c, shots, seed).counts` (terminal circuits with
several independent blocks, and mid-circuit circuits that replay per shot) and
`PBlockState(...).contract()` after the unitary part, for seeded circuits
written to pblock.json.  Nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path[:0] = [f"{REF}/src", f"{REF}/tests"]
sys.dont_write_bytecode = True

from polysim import pblock  # noqa: E402
from polysim.circuit import Circuit, Instruction  # noqa: E402
import conftest as ref_conftest  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def dump(c) -> dict:
    return {"name": c.name, "n_qubits": c.n_qubits, "n_clbits": c.n_clbits,
            "instructions": [[i.kind, list(i.qubits), list(i.params), i.clbit] for i in c.instructions]}


def sparse_blocks(n, seed):
    """Few 2q gates: several independent blocks at the end."""
    rng = np.random.default_rng(seed)
    c = Circuit(n, n, name=f"blocks_{n}_{seed}")
    for q in range(n):
        c.gate("ry", q, params=(float(rng.uniform(0, 3)),))
    for _ in range(n // 2):
        a, b = (int(x) for x in rng.choice(n, 2, replace=False))
        c.gate("cx", a, b)
        c.gate("rz", b, params=(float(rng.uniform(0, 3)),))
    for q in range(n):
        c.gate("h", q) if rng.random() < 0.5 else c.gate("t", q)
    c.measure_all()
    return c


def mid_circuit(n, seed):
    rng = np.random.default_rng(seed)
    c = Circuit(n, n, name=f"mid_{n}_{seed}")
    for q in range(n):
        c.gate("ry", q, params=(float(rng.uniform(0, 3)),))
    c.gate("cx", 0, 1).gate("cx", 2, 3)
    c.measure(1, 1)
    c.append(Instruction("reset", (2,)))
    c.gate("h", 2).gate("cx", 2, 0).gate("cx", 3, n - 1)
    for q in range(n):
        c.measure(q, q)
    return c


def main():
    cases = []
    for n, seed in ((6, 1), (9, 2), (12, 3)):
        cases.append(("terminal", sparse_blocks(n, seed), 4000, seed + 10))
    rng = np.random.default_rng(5)
    rc = ref_conftest.random_circuit(8, 40, rng)
    rc.name = "rand_8"
    cases.append(("terminal", rc, 3000, 4))
    for n, seed in ((5, 7), (7, 8)):
        cases.append(("replay", mid_circuit(n, seed), 300, seed))
    out = []
    for kind, c, shots, seed in cases:
        res = pblock.run(c, shots, seed)
        st = pblock.PBlockState(c.n_qubits)
        for inst in c.instructions:
            if inst.is_unitary:
                st.apply(inst)
                if kind == "replay":
                    break
        amps = st.contract() if kind == "terminal" else None
        out.append({"kind": kind, "circuit": dump(c), "shots": shots, "seed": seed, "counts": res.counts,
                    "max_block_dim": res.metadata["max_block_dim"],
                    "amps": None if amps is None else [[float(z.real), float(z.imag)] for z in amps]})
    with open(os.path.join(OUT, "pblock.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()
