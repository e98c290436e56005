"""GPU parity: the libsvb CUDA path against the reference's golden outputs and
the CPU oracle.  Tolerances (north_star): complex128 amplitudes 1e-10
normwise relative, complex64 1e-5; <Z> 1e-10 absolute; counts bit-exact
(alias sampler, shared PCG64 stream) or chi-square p > 1e-3 (CDF sampler)."""
import math

import numpy as np
import pytest

from conftest import chisquare_pvalue, golden, golden_circuits
from oracle import sv_oracle as orc
from paper_2512_04216_b200 import _lib, suite
from paper_2512_04216_b200 import statevector as sv
from paper_2512_04216_b200.circuit import Circuit, Instruction, inverse_circuit
from paper_2512_04216_b200.result import BackendError, NoMeasurementsError, QubitCapError

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-10, "c64": 1e-5}


def relerr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def device_state(c, precision="c128", fusion=True):
    s = sv.DeviceState(c.n_qubits, precision)
    if not fusion:
        s.set_option(_lib.OPT_FUSION, 0)
    s.apply_instructions(c.instructions)
    return s


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_amplitudes_match_reference_golden(precision):
    circuits = golden_circuits()
    for key, ref in golden("amps.npz").items():
        s = device_state(circuits[key], precision)
        got = s.to_numpy()
        s.close()
        assert relerr(got, ref) < TOL[precision], key


def test_final_state_api_and_cache():
    circuits = golden_circuits()
    c = circuits["qft_ry_12"]
    amps = sv.final_state(c)
    assert amps is sv.final_state(c)
    assert relerr(amps, golden("amps.npz")["qft_ry_12"]) < 1e-10
    c2 = suite.ghz_circuit(4, measured=False)
    sv.expectation(c2, (0,))
    first = sv._state_cache[c2]
    sv.expectation(c2, (1, 2))
    assert sv._state_cache[c2] is first


def test_expectations_match_reference_golden():
    circuits = golden_circuits()
    for key, rows in golden("expect.json").items():
        c = circuits[key]
        for zq, val in rows:
            assert abs(sv.expectation(c, zq) - val) < 1e-10, (key, zq)
        many = sv.expectations(c, [zq for zq, _ in rows])
        np.testing.assert_allclose(many, [v for _, v in rows], atol=1e-10)


def test_expectation_kats():
    g = suite.ghz_circuit(3, measured=False)
    assert sv.expectation(g, (0, 1)) == pytest.approx(1.0, abs=1e-12)
    assert sv.expectation(g, (0, 1, 2)) == pytest.approx(0.0, abs=1e-12)
    ry = Circuit(1).gate("ry", 0, params=(0.9,))
    assert sv.expectation(ry, (0,)) == pytest.approx(math.cos(0.9), abs=1e-12)
    with pytest.raises(ValueError):
        sv.expectation(g, (3,))


def _alias_robust(probs, trials=8) -> bool:
    """True when the reference alias table is unchanged under 1-ulp noise on
    the probabilities (then counts must match the golden bit for bit)."""
    pr, al = orc.alias_table(probs)
    g = np.random.default_rng(0)
    for _ in range(trials):
        q = probs * (1 + g.choice([-1.0, 0.0, 1.0], size=probs.size) * 2.3e-16)
        pr2, al2 = orc.alias_table(q)
        if not np.array_equal(al2, al):
            return False
    return True


def test_counts_vs_reference_golden():
    """Terminal sampling parity, decomposed:
    (1) given the device's probabilities, the device sampler reproduces the
        reference algorithm (alias table + PCG64 draws + clbit packing) bit for bit;
    (2) counts equal the reference's golden counts exactly whenever the
        reference's alias table is insensitive to 1-ulp probability noise
        (amplitudes agree to ~1e-16, not bitwise), and otherwise pass a
        two-sample chi-square against them; mid-circuit replay must match exactly."""
    from conftest import chisquare_pvalue  # noqa: F401
    from scipy import stats

    circuits = golden_circuits()
    exact = robust_total = 0
    for key, by_seed in golden("counts.json").items():
        c = circuits[key]
        workers = 3 if key.endswith("_w3") else 1
        terminal = orc.is_terminal(c)
        for seed, ref in by_seed.items():
            shots = sum(ref.values())
            res = sv.run(c, shots, int(seed), workers=workers, qubit_cap=max(26, c.n_qubits), sampler="alias")
            assert sum(res.counts.values()) == shots and res.backend == "sv"
            if not terminal:
                assert res.counts == ref, (key, seed)
                continue
            measures = [(i.qubits[0], i.clbit) for i in c.instructions if i.kind == "measure"]
            qubits = tuple(sorted({q for q, _ in measures}))
            s = sv.DeviceState(c.n_qubits)
            s.apply_instructions(c.instructions)
            dev_probs = s.marginal_probs(qubits)
            s.close()
            want = orc.sample_terminal(qubits, dev_probs, measures, shots, np.random.default_rng(int(seed)))
            assert res.counts == want, ("sampler not bit-exact given identical probabilities", key, seed)
            ref_probs = orc.marginal_probs(orc.unitary_state(c), c.n_qubits, qubits)
            np.testing.assert_allclose(dev_probs, ref_probs, atol=1e-13)
            if _alias_robust(ref_probs):
                robust_total += 1
                assert res.counts == ref, (key, seed)
                exact += 1
            elif res.counts != ref:
                keys = sorted(set(ref) | set(res.counts))
                table = np.array([[ref.get(k, 0) for k in keys], [res.counts.get(k, 0) for k in keys]]) + 0.5
                assert stats.chi2_contingency(table)[1] > 1e-3, (key, seed)
    assert robust_total >= 15


def _long_cycle_monomial(m) -> bool:
    nz = [np.flatnonzero(m[r]) for r in range(m.shape[0])]
    if not all(len(z) == 1 for z in nz):
        return False
    src = [int(z[0]) for z in nz]
    seen, longest = set(), 0
    for s0 in range(len(src)):
        if s0 in seen:
            continue
        j, ln = s0, 0
        while j not in seen:
            seen.add(j)
            j = src[j]
            ln += 1
        longest = max(longest, ln)
    return longest >= 3


def _dense_apply(psi, n, qubits, m):
    t = psi.reshape([2] * n)
    k = len(qubits)
    axes = [n - 1 - q for q in qubits]  # qubit q is axis n-1-q; local index bit j <-> qubits[j]
    mt = m.reshape([2] * (2 * k))  # [out bits k-1..0, in bits k-1..0]
    out = np.tensordot(mt, t, axes=(list(range(k, 2 * k)), axes[::-1]))
    return np.moveaxis(out, list(range(k)), axes[::-1]).reshape(-1)


def test_kernel_level_api_matches_reference_golden():
    """apply_1q / apply_2q on caller-owned numpy arrays vs the reference.

    Monomial matrices with a 3- or 4-cycle expose a reference bug: the cycle
    following in apply_2q (statevector.py:81-104) pairs each destination with
    the wrong source and writes zeros (never reached by the IR, whose cx/swap
    are 2-cycles).  For those the device result is checked against the exact
    matrix action instead."""
    k = golden("kernels.npz")
    for i in range(0, int(k["n_cases"]), 2):
        kind, n, qa, qb = (int(x) for x in k[f"k{i}_meta"])
        m = k[f"k{i}_mat"]
        psi = k[f"k{i}_in"].copy()
        if kind == 1:
            sv.apply_1q(psi, n, qa, m)
        else:
            sv.apply_2q(psi, n, qa, qb, m)
        if kind == 2 and _long_cycle_monomial(m):
            want = _dense_apply(k[f"k{i}_in"], n, (qa, qb), m)
            assert not np.allclose(want, k[f"k{i}_out"])  # the reference result is wrong here
        else:
            want = k[f"k{i}_out"]
        np.testing.assert_allclose(psi, want, atol=1e-13, err_msg=str(i))


def test_alias_tables_bit_exact_vs_reference_golden():
    a = golden("alias.npz")
    L = _lib.lib()
    for i in range(int(a["n_cases"])):
        p = np.ascontiguousarray(a[f"a{i}_p"])
        pr = np.empty_like(p)
        al = np.empty(p.size, dtype=np.int64)
        _lib.check(L.svb_alias_table(0, _lib.ptr(p, _lib.c_double), p.size, _lib.ptr(pr, _lib.c_double),
                                     _lib.ptr(al, _lib.c_int64)))
        np.testing.assert_array_equal(pr, a[f"a{i}_prob"], err_msg=str(i))
        np.testing.assert_array_equal(al, a[f"a{i}_alias"], err_msg=str(i))


def test_alias_tables_bit_exact_large_exact_and_rounding_cumsums():
    """Tables of >= 8192 outcomes against the oracle's restatement of
    AliasTable.from_probs: distributions whose deficit / capacity prefix sums
    never round take the parallel scan (uniform over a subset, GHZ-like,
    dyadic), the others the binade-window scan (random, tie-prone, wide
    range); all bit-exact."""
    rng = np.random.default_rng(11)
    cases = []
    for m, k in ((1 << 14, 3), (1 << 16, 1 << 9), (1 << 15, 1 << 15)):
        p = np.zeros(m)
        p[rng.choice(m, size=k, replace=False)] = 1.0 / k
        cases.append(p)
    d = rng.integers(0, 8, size=1 << 14).astype(float)
    cases.append(d / d.sum() if d.sum() else d)          # dyadic weights (exact)
    r = rng.random(1 << 15) ** 3
    cases.append(r / r.sum())                              # random (rounding chain: binade windows)
    r = rng.random(1 << 18)
    cases.append(r / r.sum())
    t = np.round(rng.random(1 << 15) * 8) / 8 + 1.0 / 8    # few mantissa bits: ties in the chain
    cases.append(t / t.sum())
    g = rng.exponential(size=1 << 16) * 10.0 ** rng.uniform(-6, 0, size=1 << 16)
    cases.append(g / g.sum())                              # wide dynamic range
    h = rng.random(1 << 16) * 1e-3                         # 4 heavy outcomes absorb runs of ~16k
    h[rng.choice(h.size, size=4, replace=False)] = 10.0    # random deficits: long sequential bins
    cases.append(h / h.sum())
    u = np.zeros(1 << 17)
    u[rng.choice(u.size, size=6, replace=False)] = 1.0 / 6  # long runs with exact bins (parallel)
    cases.append(u)
    big = rng.random(1 << 23) ** 2                         # >= 2^21-element chains: binade windows
    cases.append(big / big.sum())
    L = _lib.lib()
    for i, p in enumerate(cases):
        p = np.ascontiguousarray(p)
        pr = np.empty_like(p)
        al = np.empty(p.size, dtype=np.int64)
        _lib.check(L.svb_alias_table(0, _lib.ptr(p, _lib.c_double), p.size, _lib.ptr(pr, _lib.c_double),
                                     _lib.ptr(al, _lib.c_int64)))
        want_p, want_a = orc.alias_table(p)
        np.testing.assert_array_equal(pr, want_p, err_msg=str(i))
        np.testing.assert_array_equal(al, want_a, err_msg=str(i))


def test_alias_table_rejects_bad_vectors():
    L = _lib.lib()
    for p in (np.array([0.5, 0.6]), np.array([-0.1, 1.1])):
        pr = np.empty_like(p)
        al = np.empty(p.size, dtype=np.int64)
        with pytest.raises(ValueError):
            _lib.check(L.svb_alias_table(0, _lib.ptr(p, _lib.c_double), p.size, _lib.ptr(pr, _lib.c_double),
                                         _lib.ptr(al, _lib.c_int64)))


def test_marginals_match_reference_golden():
    m = golden("marginals.npz")
    for i in range(int(m["n_cases"])):
        psi = m[f"m{i}_psi"]
        n = psi.size.bit_length() - 1
        got = sv.marginal_probs(psi.copy(), n, tuple(int(q) for q in m[f"m{i}_q"]))
        np.testing.assert_allclose(got, m[f"m{i}_out"], rtol=1e-13, atol=1e-16)


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_random_circuits_vs_oracle_fused_and_unfused(precision):
    rng = np.random.default_rng(3)
    for trial in range(12):
        n = int(rng.integers(9, 19))
        c = suite.random_circuit(n, int(rng.integers(20, 300)), rng, measured=False)
        ref = orc.unitary_state(c)
        a = device_state(c, precision).to_numpy()
        b = device_state(c, precision, fusion=False).to_numpy()
        assert relerr(a, ref) < TOL[precision], (trial, n)
        assert relerr(b, ref) < TOL[precision], (trial, n)


def test_structured_families_vs_oracle():
    for c in (
        suite.qft_bench_circuit(16),
        suite.sycamore_circuit(4, 4, 12, seed=1, measured=False),
        suite.qaoa_line_circuit(18, 2, seed=5, measured=False),
        suite.ry_ansatz_circuit(17, 2, seed=6, measured=False),
    ):
        ref = orc.unitary_state(c)
        for precision in ("c128", "c64"):
            assert relerr(device_state(c, precision).to_numpy(), ref) < TOL[precision], (c.name, precision)


def test_qft_dft_known_answer_24_qubits():
    n = 24
    basis = 0xA5C3E1
    c = Circuit(n)
    for q in range(n):
        if (basis >> q) & 1:
            c.gate("x", q)
    suite.qft(n, c)
    got = device_state(c).to_numpy()
    k = np.arange(1 << n, dtype=np.float64)
    phase = np.mod(basis * k, float(1 << n)) / (1 << n)
    want = np.exp(2j * math.pi * phase) / math.sqrt(1 << n)
    assert relerr(got, want) < 1e-10


def test_mirror_circuit_26_qubits():
    rng = np.random.default_rng(9)
    c = suite.random_circuit(26, 400, rng, measured=False)
    s = sv.DeviceState(26)
    s.apply_instructions(c.instructions + inverse_circuit(c).instructions)
    amp0 = s.to_numpy()[0]
    assert abs(abs(amp0) - 1.0) < 1e-10


def test_cdf_sampler_chi_square():
    rng = np.random.default_rng(12)
    for _ in range(4):
        n = int(rng.integers(5, 11))
        c = suite.random_circuit(n, 40, rng)
        psi = orc.unitary_state(c)
        probs = np.abs(psi) ** 2
        expected = {format(i, f"0{n}b"): float(p) for i, p in enumerate(probs) if p > 0}
        res = sv.run(c, 100_000, int(rng.integers(2**31)), sampler="cdf")
        assert sum(res.counts.values()) == 100_000
        assert chisquare_pvalue(res.counts, expected, 100_000) > 1e-3


def test_seed_determinism_and_error_order():
    c = suite.random_circuit(12, 60, np.random.default_rng(0))
    a = sv.run(c, 3000, 42).counts
    assert a == sv.run(c, 3000, 42).counts
    assert a != sv.run(c, 3000, 43).counts
    big = Circuit(27, 27).gate("h", 0).measure(0, 0)
    with pytest.raises(QubitCapError):
        sv.run(big, 1, 0)
    with pytest.raises(ValueError):
        sv.run(Circuit(2, 2).gate("h", 0).measure(0, 0), 0, 0)
    with pytest.raises(NoMeasurementsError):
        sv.run(Circuit(2).gate("h", 0), 10, 0)
    mid = Circuit(2, 2).gate("h", 0).measure(0, 0).gate("h", 0)
    with pytest.raises(BackendError):
        sv.final_state(mid)


def test_kernel_level_measure_consumes_one_draw():
    rng_ref = np.random.default_rng(5)
    rng_dev = np.random.default_rng(5)
    for q in range(4):
        c = suite.random_circuit(4, 20, np.random.default_rng(q), measured=False)
        psi_ref = orc.unitary_state(c)
        psi_dev = psi_ref.copy()
        o_ref = orc.measure_qubit(psi_ref, 4, q, rng_ref)
        o_dev = sv._measure_qubit(psi_dev, 4, q, rng_dev)
        assert o_ref == o_dev
        np.testing.assert_allclose(psi_dev, psi_ref, atol=1e-13)
    assert rng_ref.random() == rng_dev.random()


def test_ghz20_config1_counts_bit_exact():
    ref = golden("counts.json")["ghz20"]
    c = suite.ghz_circuit(20)
    for seed, counts in ref.items():
        assert sv.run(c, 1024, int(seed)).counts == counts


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_jit_matches_interpreter_and_oracle(precision):
    """NVRTC-specialised passes == interpreter passes == oracle."""
    rng = np.random.default_rng(21)
    for trial in range(3):
        n = int(rng.integers(14, 19))
        c = suite.random_circuit(n, int(rng.integers(60, 250)), rng, measured=False)
        ref = orc.unitary_state(c)
        outs = []
        for jit in (-1, 1):
            s = sv.DeviceState(n, precision)
            s.set_option(_lib.OPT_JIT_MIN_N, jit)
            s.apply_instructions(c.instructions)
            outs.append(s.to_numpy())
            s.close()
        assert relerr(outs[0], ref) < TOL[precision]
        assert relerr(outs[1], ref) < TOL[precision]
    for c in (suite.qft_bench_circuit(15), suite.sycamore_circuit(3, 5, 10, seed=2, measured=False)):
        ref = orc.unitary_state(c)
        s = sv.DeviceState(c.n_qubits, precision)
        s.set_option(_lib.OPT_JIT_MIN_N, 1)
        s.apply_instructions(c.instructions)
        assert relerr(s.to_numpy(), ref) < TOL[precision], c.name
        s.close()


def _mid_circuit(n, seed):
    rng = np.random.default_rng(seed)
    c = suite.random_circuit(n, 30, rng, measured=False)
    c.n_clbits = n
    c.measure(0, 0)
    c.append(Instruction("reset", (1,)))
    c.gate("h", 0).gate("cx", 0, n - 1).gate("ry", 1, params=(0.8,))
    for q in range(n):
        c.measure(q, q)
    return c


@pytest.mark.parametrize("n", [8, 13])
def test_mid_circuit_replay_bit_exact_vs_oracle(n):
    """Replay (statevector.py:157-250): smem-batched path (n=8) and per-shot
    path (n=13) reproduce the oracle's counts exactly, workers included."""
    c = _mid_circuit(n, 100 + n)
    for workers in (1, 3):
        shots = 600 if n > 12 else 3000
        got = sv.run(c, shots, 17, workers=workers)
        assert got.metadata["replay_engine"] == ("per-shot" if n > 12 else "smem-batched")
        assert got.counts == orc.run(c, shots, 17, workers=workers), (n, workers)


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_long_passes_jit_and_interpreter(precision):
    """Passes with hundreds of pivoted 1q ops (deferred scalar re-absorbed
    along the way) on both kernel bodies, including immediates (n >= 28 path
    forced via a small circuit with OPT_JIT_MIN_N)."""
    n = 14
    rng = np.random.default_rng(3)
    c = Circuit(n)
    for layer in range(40):
        for q in range(n):
            c.gate("ry", q, params=(float(rng.uniform(0, 3)),))
            c.gate("rx", q, params=(float(rng.uniform(0, 3)),))
        for q in range(layer % 2, n - 1, 2):
            c.gate("cz", q, q + 1)
    ref = orc.unitary_state(c)
    for jit in (-1, 1):
        s = sv.DeviceState(n, precision)
        s.set_option(_lib.OPT_JIT_MIN_N, jit)
        s.apply_instructions(c.instructions)
        assert relerr(s.to_numpy(), ref) < 10 * TOL[precision], (precision, jit)
        s.close()


def test_run_codes_arrays_equal_run_counts():
    """(code, count) arrays format to exactly run()'s dict."""
    rng = np.random.default_rng(8)
    cases = [suite.ghz_circuit(20), suite.random_circuit(11, 80, rng), _mid_circuit(9, 4)]
    for c in cases:
        for seed in (0, 7):
            a = sv.run_codes(c, 2000, seed)
            b = sv.run(c, 2000, seed).counts
            assert a.to_dict() == b
            assert int(a.counts.sum()) == 2000 and np.all(np.diff(a.codes.astype(np.int64)) > 0)


def _swap_tail_circuit(n, seed):
    """Random gates followed by swaps that move low qubits up: the final qubit
    permutation of the swap relabeling is fused into the last pass's store."""
    rng = np.random.default_rng(seed)
    c = suite.random_circuit(n, 80, rng, measured=False)
    for q in range(5):
        c.gate("swap", q, 5 + q)
    for q in range(5, 12):
        c.gate("u", q, params=tuple(float(x) for x in rng.uniform(0, 6.3, 3)))
    return c


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_permuted_store_and_zero_start_layout(precision):
    """Swap relabeling on device: (a) on an arbitrary input state the final
    permutation is fused into the last pass (out-of-place permuted store),
    JIT and interpreter bodies; (b) on a lazy |0...0> the initial layout absorbs
    it.  Both against the oracle."""
    for body in (suite.qft_bench_circuit(12), _swap_tail_circuit(14, 1)):
        n = body.n_qubits
        prep = suite.random_circuit(n, 40, np.random.default_rng(5), measured=False)
        assert sv.plan(n, body.instructions, precision)["permute_fused"], body.name
        ref = orc.unitary_state(prep)
        for inst in body.instructions:
            orc.apply_instruction(ref, n, inst)
        for jit in (-1, 1):
            s = sv.DeviceState(n, precision)
            s.set_option(_lib.OPT_JIT_MIN_N, jit)
            s.apply_instructions(prep.instructions)
            s.apply_instructions(body.instructions)
            assert relerr(s.to_numpy(), ref) < TOL[precision], (body.name, jit)
            s.close()
        ref0 = orc.unitary_state(body)
        for jit in (-1, 1):
            s = sv.DeviceState(n, precision)
            s.set_option(_lib.OPT_JIT_MIN_N, jit)
            s.apply_instructions(body.instructions)
            assert relerr(s.to_numpy(), ref0) < TOL[precision], (body.name, jit)
            s.close()


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_fused_z_sums_match_reduction_pass(precision):
    """svb_apply_z: <Z_q> summed by the last fused pass == the separate
    multi-mask reduction == the oracle, for lazy-zero and arbitrary inputs,
    fused and separate final permutations, JIT and interpreter bodies."""
    tol = 1e-10 if precision == "c128" else 2e-5
    cases = [suite.qft_bench_circuit(14), suite.random_circuit(15, 120, np.random.default_rng(4), measured=False),
             _swap_tail_circuit(14, 1), suite.sycamore_circuit(3, 5, 6, seed=1, measured=False)]
    for c in cases:
        n = c.n_qubits
        qs = list(range(n))
        ref = orc.unitary_state(c)
        want = np.array([orc.expectation_from_state(ref, (q,)) for q in qs])
        for jit in (-1, 1):
            s = sv.DeviceState(n, precision)
            s.set_option(_lib.OPT_JIT_MIN_N, jit)
            got = s.apply_gates_z(sv.gate_array(c.instructions), qs)
            np.testing.assert_allclose(got, want, atol=tol, err_msg=f"{c.name} jit={jit}")
            np.testing.assert_allclose(s.expect_z([1 << q for q in qs]), want, atol=tol)
            # arbitrary input state (not the lazy zero): permutation fused or separate
            got2 = s.apply_gates_z(sv.gate_array(c.instructions), qs[::-1])
            ref2 = ref.copy()
            for inst in c.instructions:
                orc.apply_instruction(ref2, n, inst)
            want2 = np.array([orc.expectation_from_state(ref2, (q,)) for q in qs[::-1]])
            np.testing.assert_allclose(got2, want2, atol=tol, err_msg=f"{c.name} jit={jit} (2nd apply)")
            s.close()
    # public API: expectations() of single-qubit Z on an uncached circuit takes the fused path
    c = suite.qft_bench_circuit(13)
    z = sv.expectations(c, [(q,) for q in range(13)], qubit_cap=13)
    ref = orc.unitary_state(c)
    np.testing.assert_allclose(z, [orc.expectation_from_state(ref, (q,)) for q in range(13)], atol=1e-10)
    assert relerr(sv.final_state(c, qubit_cap=13), ref) < 1e-10


def _partial_support_circuit(n, seed):
    """Gates on the low qubits only, plus diagonal-only gates (rz, cz) on some
    high ones: those qubits stay |0> and the passes never write their half."""
    rng = np.random.default_rng(seed)
    c = suite.random_circuit(n - 3, 90, rng, measured=False)
    full = Circuit(n)
    for inst in c.instructions:
        full.gate(inst.kind, *inst.qubits, params=inst.params)
    full.gate("rz", n - 2, params=(0.3,))
    full.gate("cz", n - 2, 0)
    return full


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_zero_start_support_tracking(precision):
    """Lazy |0...0> programs only launch the tiles inside the support (qubits
    already written) and synthesise never-written positions as zeros; circuits
    that leave qubits untouched zero-fill first.  Amplitudes and fused <Z>
    against the oracle, JIT and interpreter bodies."""
    tol = TOL[precision]
    for c in (suite.qft_bench_circuit(15), _partial_support_circuit(15, 2), _partial_support_circuit(14, 5),
              suite.sycamore_circuit(3, 5, 4, seed=4, measured=False)):
        n = c.n_qubits
        ref = orc.unitary_state(c)
        want = np.array([orc.expectation_from_state(ref, (q,)) for q in range(n)])
        for jit in (-1, 1):
            s = sv.DeviceState(n, precision)
            s.set_option(_lib.OPT_JIT_MIN_N, jit)
            s.apply_instructions(c.instructions)
            assert relerr(s.to_numpy(), ref) < tol, (c.name, jit)
            s.close()
            s = sv.DeviceState(n, precision)
            s.set_option(_lib.OPT_JIT_MIN_N, jit)
            z = s.apply_gates_z(sv.gate_array(c.instructions), list(range(n)))
            np.testing.assert_allclose(z, want, atol=10 * tol, err_msg=f"{c.name} jit={jit}")
            assert relerr(s.to_numpy(), ref) < tol, (c.name, jit)
            s.close()


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_qft_dft_fused_z_26_qubits(precision):
    """x-prep + QFT-26 from a lazy |0...0> (JIT passes, support tracking, free
    initial layout, <Z_i> fused into the last pass): amplitudes against the DFT
    closed form, and every <Z_i> is exactly 0 in exact arithmetic (flat |amp|^2)."""
    n = 26
    basis = 0x2B5C3E1
    c = Circuit(n)
    for q in range(n):
        if (basis >> q) & 1:
            c.gate("x", q)
    suite.qft(n, c)
    s = sv.DeviceState(n, precision)
    z = s.apply_gates_z(sv.gate_array(c.instructions), list(range(n)))
    assert float(np.max(np.abs(z))) < (1e-10 if precision == "c128" else 2e-5), z
    got = s.to_numpy()
    k = np.arange(1 << n, dtype=np.float64)
    phase = np.mod(basis * k, float(1 << n)) / (1 << n)
    want = np.exp(2j * math.pi * phase) / math.sqrt(1 << n)
    assert relerr(got, want) < TOL[precision]
    s.close()


def test_fused_z_fallbacks_and_edges():
    """svb_apply_z where the last pass cannot sum: too few qubits for a fused
    program (per-gate kernels + one reduction pass), fusion off, an empty qubit
    list, and a circuit with no gates."""
    for n, fusion in ((6, True), (12, False)):
        c = suite.random_circuit(n, 40, np.random.default_rng(n), measured=False)
        ref = orc.unitary_state(c)
        s = sv.DeviceState(n)
        if not fusion:
            s.set_option(_lib.OPT_FUSION, 0)
        z = s.apply_gates_z(sv.gate_array(c.instructions), list(range(n)))
        np.testing.assert_allclose(z, [orc.expectation_from_state(ref, (q,)) for q in range(n)], atol=1e-10)
        assert relerr(s.to_numpy(), ref) < 1e-10
        s.close()
    s = sv.DeviceState(10)
    assert s.apply_gates_z(sv.gate_array(suite.qft_bench_circuit(10).instructions), []).size == 0
    z = s.apply_gates_z(sv.gate_array([]), [0, 3])
    np.testing.assert_allclose(z, [orc.expectation_from_state(s.to_numpy(), (q,)) for q in (0, 3)], atol=1e-10)
    s.close()


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_initial_permutation_schedule(precision):
    """Swaps on a written input: the input is permuted first into the layout
    that absorbs the relabeling (cheaper passes), JIT and interpreter bodies."""
    for n in (14, 16):
        c = suite.qft_bench_circuit(n)
        assert sv.plan(n, c.instructions, precision)["permute_initial"]
        prep = suite.random_circuit(n, 30, np.random.default_rng(n), measured=False)
        ref = orc.unitary_state(prep)
        for inst in c.instructions:
            orc.apply_instruction(ref, n, inst)
        for jit in (-1, 1):
            s = sv.DeviceState(n, precision)
            s.set_option(_lib.OPT_JIT_MIN_N, jit)
            s.apply_instructions(prep.instructions)
            z = s.apply_gates_z(sv.gate_array(c.instructions), list(range(n)))
            assert relerr(s.to_numpy(), ref) < TOL[precision], (n, jit)
            np.testing.assert_allclose(z, [orc.expectation_from_state(ref, (q,)) for q in range(n)],
                                       atol=10 * TOL[precision])
            s.close()


def _swap_mix_circuit(seed):
    from paper_2512_04216_b200.circuit import Circuit
    rng = np.random.default_rng(seed)
    n = int(rng.integers(14, 20))
    c = Circuit(n)
    for _ in range(int(rng.integers(20, 80))):
        c.gate("h", int(rng.integers(0, n)))
        a, b = rng.choice(n, 2, replace=False)
        c.gate(str(rng.choice(["cx", "cz", "swap", "swap"])), int(a), int(b))
    return c


def test_initial_permutation_fused_into_first_pass_loads():
    """A written input whose absorbing layout keeps input qubits 0..4 inside
    the first pass's tile: the permutation is folded into that pass's tile
    loads (PassDev::perm_in, out of place), JIT and interpreter bodies."""
    c = _swap_mix_circuit(163)
    n = c.n_qubits
    pl = sv.plan(n, c.instructions, "c128")
    assert pl["permute_initial_fused"], pl
    prep = suite.random_circuit(n, 30, np.random.default_rng(5), measured=False)
    ref = orc.unitary_state(prep)
    for inst in c.instructions:
        orc.apply_instruction(ref, n, inst)
    for jit in (-1, 1):
        s = sv.DeviceState(n, "c128")
        s.set_option(_lib.OPT_JIT_MIN_N, jit)
        s.apply_instructions(prep.instructions)
        z = s.apply_gates_z(sv.gate_array(c.instructions), list(range(n)))
        assert relerr(s.to_numpy(), ref) < TOL["c128"], jit
        np.testing.assert_allclose(z, [orc.expectation_from_state(ref, (q,)) for q in range(n)], atol=1e-9)
        s.close()
