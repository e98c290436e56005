"""Pin the CPU oracle (oracle/sv_oracle.py) to the real reference's outputs.

Every golden fixture was produced by running `polysim` itself
(tests/golden/make_golden.py); the oracle must reproduce them exactly
(bitwise for counts, alias tables and kernel outputs).
"""
import numpy as np
import pytest

from conftest import golden, golden_circuits
from oracle import sv_oracle as orc


def test_oracle_amplitudes_match_reference():
    circuits = golden_circuits()
    amps = golden("amps.npz")
    assert len(amps) > 60
    for key, ref in amps.items():
        got = orc.unitary_state(circuits[key])
        np.testing.assert_array_equal(got, ref, err_msg=key)


def test_oracle_counts_match_reference():
    circuits = golden_circuits()
    counts = golden("counts.json")
    for key, by_seed in counts.items():
        c = circuits[key]
        for seed, ref in by_seed.items():
            workers = 3 if key.endswith("_w3") else 1
            shots = sum(ref.values())
            got = orc.run(c, shots, int(seed), workers=workers, qubit_cap=max(26, c.n_qubits))
            assert got == ref, (key, seed)


def test_oracle_expectations_match_reference():
    circuits = golden_circuits()
    for key, rows in golden("expect.json").items():
        psi = orc.unitary_state(circuits[key])
        for zq, val in rows:
            assert orc.expectation_from_state(psi, zq) == pytest.approx(val, abs=1e-14), (key, zq)


def test_oracle_kernels_match_reference():
    k = golden("kernels.npz")
    for i in range(int(k["n_cases"])):
        kind, n, qa, qb = (int(x) for x in k[f"k{i}_meta"])
        psi = k[f"k{i}_in"].copy()
        if kind == 1:
            orc.apply_1q(psi, n, qa, k[f"k{i}_mat"])
        else:
            orc.apply_2q(psi, n, qa, qb, k[f"k{i}_mat"])
        np.testing.assert_array_equal(psi, k[f"k{i}_out"], err_msg=str(i))


def test_oracle_alias_tables_match_reference():
    a = golden("alias.npz")
    for i in range(int(a["n_cases"])):
        pr, al = orc.alias_table(a[f"a{i}_p"])
        np.testing.assert_array_equal(pr, a[f"a{i}_prob"])
        np.testing.assert_array_equal(al, a[f"a{i}_alias"])
        draw = orc.alias_sample(pr, al, np.random.default_rng(100 + i), 5000)
        np.testing.assert_array_equal(draw, a[f"a{i}_draw"])


def test_oracle_marginals_match_reference():
    m = golden("marginals.npz")
    for i in range(int(m["n_cases"])):
        psi = m[f"m{i}_psi"]
        n = psi.size.bit_length() - 1
        got = orc.marginal_probs(psi, n, tuple(int(q) for q in m[f"m{i}_q"]))
        np.testing.assert_array_equal(got, m[f"m{i}_out"])


def test_oracle_error_behaviour():
    c = golden_circuits()["ghz20"]
    with pytest.raises(orc.OracleCapError):
        orc.run(c, 10, 0, qubit_cap=19)
    with pytest.raises(ValueError):
        orc.run(c, 0, 0, qubit_cap=26)
