"""Dense k-qubit blocks (svb_apply_matrix): the tcgen05 tensor-core engine
(complex64, 3xTF32) and the CUDA-core engine against the oracle.

Parity anchor: a fused block is built from reference gates (the oracle's
restatement of `apply_1q` / `apply_2q`, statevector.py:33-113, applied to the
2^k basis states of the block), then applied in one device pass; the result
must equal applying the same gates one by one with the oracle.  Tolerances:
complex64 1e-5 normwise (north_star), complex128 1e-10."""
import numpy as np
import pytest

from oracle import sv_oracle as orc
from paper_2512_04216_b200 import _lib, suite
from paper_2512_04216_b200 import statevector as sv
from paper_2512_04216_b200.circuit import Instruction

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-10, "c64": 1e-5}


def relerr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def dense_apply(psi, n, qubits, m):
    """psi <- U on `qubits` (local index bit i <-> qubits[i]) by tensordot."""
    t = psi.reshape([2] * n)
    k = len(qubits)
    axes = [n - 1 - q for q in qubits]
    mt = m.reshape([2] * (2 * k))
    out = np.tensordot(mt, t, axes=(list(range(k, 2 * k)), axes[::-1]))
    return np.moveaxis(out, list(range(k)), axes[::-1]).reshape(-1)


def random_unitary(k, rng):
    z = rng.normal(size=(1 << k, 1 << k)) + 1j * rng.normal(size=(1 << k, 1 << k))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def fused_block(gates, k):
    """Matrix of a gate list on local qubits 0..k-1 (oracle gate by gate on basis states)."""
    D = 1 << k
    U = np.zeros((D, D), dtype=np.complex128)
    for j in range(D):
        e = np.zeros(D, dtype=np.complex128)
        e[j] = 1
        for g in gates:
            orc.apply_instruction(e, k, g)
        U[:, j] = e
    return U


def random_state(n, seed, precision="c128"):
    c = suite.random_circuit(n, 6 * n, np.random.default_rng(seed), measured=False)
    s = sv.DeviceState(n, precision)
    s.apply_instructions(c.instructions)
    return s, orc.unitary_state(c)


@pytest.mark.parametrize("k", [3, 4, 5, 6])
def test_tensor_engine_random_unitaries(k):
    rng = np.random.default_rng(100 + k)
    for trial in range(4):
        n = int(rng.integers(k + 7, 19))
        qubits = [int(x) for x in rng.choice(n, size=k, replace=False)]
        if trial == 0:
            qubits = list(range(k))  # the block on the lowest qubits
        U = random_unitary(k, rng)
        s, ref = random_state(n, trial, "c64")
        assert s.apply_matrix(qubits, U, engine="tensor") == "tensor"
        want = dense_apply(ref, n, qubits, U)
        assert relerr(s.to_numpy(), want) < TOL["c64"], (k, n, qubits)
        s.close()


@pytest.mark.parametrize("precision", ["c64", "c128"])
@pytest.mark.parametrize("k", [1, 2, 4, 5])
def test_fma_engine_random_unitaries(precision, k):
    rng = np.random.default_rng(200 + k)
    for trial in range(3):
        n = int(rng.integers(k + 7, 18))
        qubits = [int(x) for x in rng.choice(n, size=k, replace=False)]
        U = random_unitary(k, rng)
        s, ref = random_state(n, trial, precision)
        assert s.apply_matrix(qubits, U, engine="fma") == "fma"
        assert relerr(s.to_numpy(), dense_apply(ref, n, qubits, U)) < TOL[precision]
        s.close()


def test_fused_reference_gates_through_tensor_cores():
    """Blocks fused from reference gates (rx/ry/u/h/cx/cz/swap on 5 qubits),
    24 blocks in a row on 18 qubits: device tensor path == gate-by-gate oracle."""
    rng = np.random.default_rng(7)
    n, k = 18, 5
    s, ref = random_state(n, 3, "c64")
    for b in range(24):
        qubits = [int(x) for x in rng.choice(n, size=k, replace=False)]
        local = suite.random_circuit(k, 25, rng, measured=False).instructions
        U = fused_block(local, k)
        s.apply_matrix(qubits, U, engine="tensor")
        for g in local:
            orc.apply_instruction(ref, n, Instruction(g.kind, tuple(qubits[q] for q in g.qubits), g.params))
    assert relerr(s.to_numpy(), ref) < TOL["c64"]
    s.close()


def test_engine_selection_and_errors():
    rng = np.random.default_rng(1)
    s = sv.DeviceState(14, "c64")
    assert s.apply_matrix([0, 3, 5, 7, 9], random_unitary(5, rng)) == "tensor"  # auto: k >= 5
    assert s.apply_matrix([1, 2, 6, 8], random_unitary(4, rng)) == "fma"
    s.set_option(_lib.OPT_TC_MIN_K, 3)
    assert s.apply_matrix([1, 2, 6], random_unitary(3, rng)) == "tensor"
    s.close()
    d = sv.DeviceState(14, "c128")
    assert d.apply_matrix([0, 3, 5, 7, 9], random_unitary(5, rng)) == "fma"
    with pytest.raises(ValueError):
        d.apply_matrix([0, 3, 5], random_unitary(3, rng), engine="tensor")
    s6 = sv.DeviceState(14, "c64")
    assert s6.apply_matrix([0, 2, 4, 6, 8, 13], random_unitary(6, rng)) == "tensor"
    s6.close()
    with pytest.raises(ValueError):
        d.apply_matrix([0, 0, 5], random_unitary(3, rng))
    d.close()


@pytest.mark.parametrize("k", [5, 6])
def test_tensor_engine_large_state_mirror(k):
    """n = 30 complex64: 16 random k-qubit blocks then their inverses in
    reverse order return the input state (device-side comparison)."""
    rng = np.random.default_rng(11 + k)
    n = 30
    a = sv.DeviceState(n, "c64")
    a.apply_instructions(suite.random_circuit(n, 120, np.random.default_rng(2), measured=False).instructions)
    b = sv.DeviceState(n, "c64")
    b.copy_from(a)
    blocks = [([int(x) for x in rng.choice(n, size=k, replace=False)], random_unitary(k, rng)) for _ in range(16)]
    for q, U in blocks:
        a.apply_matrix(q, U, engine="tensor")
    for q, U in reversed(blocks):
        a.apply_matrix(q, U.conj().T, engine="tensor")
    assert a.compare(b)["rel"] < 1e-5
    a.close()
    b.close()


@pytest.mark.parametrize("k", [3, 4, 5])
def test_tma_staged_tensor_engine(k):
    """The TMA-staged variant (tensor-map tile loads / stores over the
    state's 2^q strides, SVB_TC_TMA=1) against the oracle, in a subprocess so
    the environment switch is read fresh."""
    import os
    import subprocess
    import sys

    code = f"""
import numpy as np, sys
sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))})
sys.path.insert(0, {repr(os.path.dirname(os.path.abspath(__file__)))})
from test_gpu_dense import random_unitary, random_state, dense_apply, relerr
rng = np.random.default_rng({k})
for trial in range(3):
    n = int(rng.integers({k} + 7, 19))
    q = [int(x) for x in rng.choice(n, size={k}, replace=False)]
    if trial == 0:
        q = list(range({k}))
    U = random_unitary({k}, rng)
    s, ref = random_state(n, trial, "c64")
    s.apply_matrix(q, U, engine="tensor")
    err = relerr(s.to_numpy(), dense_apply(ref, n, q, U))
    assert err < 1e-5, (n, q, err)
print("ok")
"""
    env = dict(os.environ, SVB_TC_TMA="1")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]
