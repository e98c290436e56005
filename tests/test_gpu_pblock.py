"""Partitioned-block backend with device blocks against
fixtures made by the real reference (tests/golden/make_golden_pblock.py)."""
import numpy as np
import pytest

from conftest import golden, load_circuit
from oracle import sv_oracle as orc
from paper_2512_04216_b200 import pblock as pb
from paper_2512_04216_b200 import statevector as sv
from paper_2512_04216_b200 import suite

pytestmark = pytest.mark.gpu


def _cases(kind):
    return [c for c in golden("pblock.json") if c["kind"] == kind]


def test_pblock_terminal_counts_and_blocks_match_reference():
    for case in _cases("terminal"):
        c = load_circuit(case["circuit"])
        res = pb.run(c, case["shots"], case["seed"])
        assert res.metadata["max_block_dim"] == case["max_block_dim"], c.name
        assert res.counts == case["counts"], c.name
        st = pb.PBlockState(c.n_qubits)
        for inst in c.instructions:
            if inst.is_unitary:
                st.apply(inst)
        got = st.contract()
        st.close()
        want = np.array([complex(a, b) for a, b in case["amps"]])
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-10, c.name


def test_pblock_replay_counts_match_reference():
    for case in _cases("replay"):
        c = load_circuit(case["circuit"])
        res = pb.run(c, case["shots"], case["seed"])
        assert res.counts == case["counts"], c.name


def test_pblock_single_block_equals_statevector_counts():
    """pblock counts == sv counts bitwise when everything is one block
    (the reference's test_pblock.py:110-121)."""
    c = suite.ghz_circuit(12)
    for seed in (0, 7):
        got = pb.run(c, 2048, seed).counts
        assert got == sv.run(c, 2048, seed).counts
        assert got == orc.run(c, 2048, seed)  # and both equal the reference algorithm


def test_block_operations_vs_oracle():
    rng = np.random.default_rng(4)
    c = suite.random_circuit(9, 60, rng, measured=False)
    st = pb.PBlockState(9)
    for inst in c.instructions:
        st.apply(inst)
    got = st.contract()
    st.close()
    ref = orc.unitary_state(c)
    assert np.linalg.norm(got - ref) < 1e-10
