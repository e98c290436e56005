"""Batch mode (config 4): persistent shared-memory kernel for small circuits,
the svb_batch_run executor for the rest; per-circuit parity with the oracle
and with sv.run (same program, same CDF draws)."""
import numpy as np
import pytest

from conftest import chisquare_pvalue
from oracle import sv_oracle as orc
from paper_2512_04216_b200 import suite
from paper_2512_04216_b200 import statevector as sv
from paper_2512_04216_b200.batch import run_batch
from paper_2512_04216_b200.circuit import Circuit, Instruction
from paper_2512_04216_b200.result import NoMeasurementsError, RunResult

pytestmark = pytest.mark.gpu


def _expected(c):
    measures = [(i.qubits[0], i.clbit) for i in c.instructions if i.kind == "measure"]
    qubits = tuple(sorted({q for q, _ in measures}))
    psi = orc.unitary_state(c)
    probs = orc.marginal_probs(psi, c.n_qubits, qubits)
    src = {}
    for q, cl in measures:
        src[cl] = q
    clbits = sorted(src)
    pos = {q: j for j, q in enumerate(qubits)}
    out = {}
    for idx, p in enumerate(probs):
        if p <= 1e-14:
            continue
        key = "".join(str((idx >> pos[src[cl]]) & 1) for cl in reversed(clbits))
        out[key] = out.get(key, 0.0) + float(p)
    return out


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_small_batch_matches_oracle(precision):
    rng = np.random.default_rng(40)
    circs = []
    for i in range(30):
        n = int(rng.integers(2, 13 if precision == "c128" else 14))
        c = suite.random_circuit(n, int(rng.integers(5, 60)), rng)
        circs.append(c)
    c = Circuit(4, 3)  # subset + crossed clbits
    c.gate("h", 0).gate("cx", 0, 2).gate("ry", 3, params=(0.4,)).measure(0, 2).measure(3, 0).measure(2, 1)
    circs.append(c)
    shots = 40000
    res = run_batch(circs, shots=shots, seed=3, precision=precision)
    for c, r in zip(circs, res):
        assert isinstance(r, RunResult) and r.metadata["engine"] == "libsvb-batch"
        assert sum(r.counts.values()) == shots
        assert chisquare_pvalue(r.counts, _expected(c), shots) > 1e-3


def test_mixed_batch_routes_and_records_errors():
    rng = np.random.default_rng(41)
    circs = [suite.qaoa_line_circuit(n, 1, seed=n) for n in (8, 12, 14, 16)]
    circs.append(suite.ry_ansatz_circuit(15, 2, seed=2))
    mid = Circuit(3, 2)
    mid.gate("h", 0).measure(0, 0).gate("x", 0).gate("h", 1).measure(1, 1)
    circs.append(mid)
    circs.append(Circuit(2).gate("h", 0))  # no measurements
    res = run_batch(circs, shots=2000, seed=9)
    assert isinstance(res[-1], NoMeasurementsError)
    for c, r in zip(circs[:-1], res[:-1]):
        assert isinstance(r, RunResult)
        assert sum(r.counts.values()) == 2000
    # circuits beyond shared memory take the executor: identical to sv.run
    # (n < 24: the same interpreter kernels in both)
    for k in (2, 3, 4, 5):
        assert res[k].counts == sv.run(circs[k], 2000, 9, sampler="cdf").counts
    # ... and every routed circuit against the oracle's exact distribution
    for c, r in zip(circs[:-2], res[:-2]):
        assert chisquare_pvalue(r.counts, _expected(c), 2000) > 1e-3, c.name
    # mid-circuit circuit: the oracle's own replay, bit for bit
    assert res[-2].counts == orc.run(mid, 2000, 9)


def test_batch_workload_families_chi_square():
    circs = suite.batch_workload(26)  # n = 12..24 QAOA / ry-ansatz (config 4 generator)
    res = run_batch(circs[:13], shots=20000, seed=0)
    for c, r in zip(circs[:13], res):
        if c.n_qubits <= 16:
            assert chisquare_pvalue(r.counts, _expected(c), 20000) > 1e-3, c.name


def test_batch_codes_equal_per_circuit_runs_all_widths():
    """Config 4's generator, one circuit per width 12..24 (both families) plus
    c64: run_batch_codes == sv.run_codes(sampler="cdf") code for code (the
    executor runs the same fused program and the same CDF draws)."""
    from paper_2512_04216_b200.batch import run_batch_codes

    circs = suite.batch_workload(26)
    for precision in ("c128", "c64"):
        res = run_batch_codes(circs, shots=1000, seed=5, precision=precision, chunk=7, jit="sync")
        for c, r in zip(circs, res):
            want = sv.run_codes(c, 1000, 5, precision=precision, sampler="cdf")
            assert np.array_equal(r.codes, want.codes) and np.array_equal(r.counts, want.counts), (c.name, precision)
    # interpreter kernels (no compile) are reproducible run to run
    a = run_batch_codes(circs, shots=1000, seed=5, jit="none")
    b = run_batch_codes(circs, shots=1000, seed=5, jit="none")
    for x, y in zip(a, b):
        assert np.array_equal(x.codes, y.codes) and np.array_equal(x.counts, y.counts)


def test_batch_executor_records_bad_circuits():
    from paper_2512_04216_b200.batch import run_batch_codes

    good = suite.qaoa_line_circuit(14, 1, seed=1)
    big = suite.qaoa_line_circuit(20, 1, seed=2)
    res = run_batch_codes([good, big, good], shots=100, seed=0, qubit_cap=18)
    from paper_2512_04216_b200.result import QubitCapError

    assert isinstance(res[1], QubitCapError)
    assert int(res[0].counts.sum()) == 100 and np.array_equal(res[0].codes, res[2].codes)


def test_concurrent_batch_calls_share_the_device():
    """Two threads running batches at once: one call gets the worker arena,
    the other its own pool buffers (svb_batch_run's try-lock); both give the
    sequential results (interpreter kernels: reproducible)."""
    import threading

    from paper_2512_04216_b200.batch import run_batch_codes

    sets = [suite.batch_workload(60, base=500 + 100 * k) for k in range(2)]
    want = [run_batch_codes(s, shots=500, seed=3, jit="none") for s in sets]
    got = [None, None]

    def work(k):
        got[k] = run_batch_codes(sets[k], shots=500, seed=3, jit="none", chunk=16)

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for a, b in zip(want, got):
        for x, y in zip(a, b):
            assert np.array_equal(x.codes, y.codes) and np.array_equal(x.counts, y.counts)
