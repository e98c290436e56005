"""CPU-only checks of the host side: IR mirror, generators, the C ABI surface,
and the fused-program scheduler run through its CPU emulator (same op
interpreter as the sm_100a kernel) against the oracle."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden, golden_circuits
from oracle import sv_oracle as orc
from paper_2512_04216_b200 import _lib, suite
from paper_2512_04216_b200 import statevector as sv
from paper_2512_04216_b200.circuit import Circuit, CircuitError, Instruction, inverse_circuit
from paper_2512_04216_b200.features import terminal_measurement_only
from paper_2512_04216_b200.gates import single_qubit_matrix, two_qubit_matrix
from paper_2512_04216_b200.result import output_bit_sources


# ------------------------------------------------------------------ IR / gates

def emulate(n: int, instructions, amps, precision: str = "c128", relabel=True):
    """CPU emulation of the fused program (test hook: the same scheduler and op
    interpreter as the device kernel, svb_emulate_apply).  Returns new amplitudes."""
    from paper_2512_04216_b200 import _lib

    arr = sv.gate_array(instructions)
    out = np.ascontiguousarray(amps, dtype=np.complex128).copy()
    _lib.check(_lib.lib().svb_emulate_apply(n, 1 if precision == "c128" else 0, _lib.ptr(arr), int(arr.size),
                                            _lib.ptr(out), int(relabel)))
    return out

def test_ir_validation_mirrors_reference():
    with pytest.raises(CircuitError):
        Instruction("cx", (1, 1))
    with pytest.raises(CircuitError):
        Instruction("rx", (0,))
    with pytest.raises(CircuitError):
        Instruction("measure", (0,))
    with pytest.raises(CircuitError):
        Instruction("foo", (0,))
    with pytest.raises(CircuitError):
        Circuit(2).gate("h", 2)
    with pytest.raises(CircuitError):
        Circuit(0)


def test_gate_matrices_match_oracle_definitions():
    for kind in ("h", "x", "y", "z", "s", "sdg", "t", "tdg"):
        np.testing.assert_array_equal(single_qubit_matrix(kind), orc.gate_matrix(kind))
    for kind, p in (("rx", (0.3,)), ("ry", (1.1,)), ("rz", (2.7,)), ("u", (0.3, 1.2, -0.7))):
        np.testing.assert_array_equal(single_qubit_matrix(kind, p), orc.gate_matrix(kind, p))
    for kind in ("cx", "cz", "swap"):
        np.testing.assert_array_equal(two_qubit_matrix(kind), orc.gate_matrix(kind))


def test_generators_reproduce_reference_circuits():
    ref = golden_circuits()

    def same(a, b):
        return a.n_qubits == b.n_qubits and [
            (i.kind, tuple(i.qubits), tuple(i.params), i.clbit) for i in a.instructions
        ] == [(i.kind, tuple(i.qubits), tuple(i.params), i.clbit) for i in b.instructions]

    for n in (5, 8, 12):
        assert same(suite.ghz_circuit(n, measured=False), ref[f"ghz_{n}"])
        assert same(suite.qaoa_line_circuit(n, 2, seed=n, measured=False), ref[f"qaoa_{n}"])
        assert same(suite.ry_ansatz_circuit(n, 2, seed=n, measured=False), ref[f"ry_{n}"])
    for n in (3, 4, 6, 9, 12):
        c = Circuit(n)
        for q in range(n):
            c.gate("ry", q, params=(0.1 * (q + 1),))
        assert same(suite.qft(n, c), ref[f"qft_ry_{n}"])
    # reference random_circuit stream (conftest.py:47-76)
    rng = np.random.default_rng(20260816)
    for k in range(40):
        n = int(rng.integers(1, 11))
        c = suite.random_circuit(n, int(rng.integers(1, 60)), rng, measured=False)
        assert same(c, ref[f"rand_{k}"]), k


def test_terminal_rule():
    c = Circuit(2, 2)
    c.gate("h", 0).measure(0, 0).gate("x", 1)
    assert terminal_measurement_only(c)
    c.gate("x", 0)
    assert not terminal_measurement_only(c)
    r = Circuit(1, 1)
    r.append(Instruction("reset", (0,)))
    assert not terminal_measurement_only(r)


def test_bit_sources_last_write_wins():
    measures = [(0, 1), (1, 0), (2, 1)]
    assert output_bit_sources(measures, [0, 1, 2]) == [1, 2]


# ------------------------------------------------------------------ C ABI
def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "svb.h")).read()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(svb_\w+)\(", header, flags=re.M))
    assert declared, "no declarations parsed"
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_lib.EXPORTED)


def test_library_reports_errors_without_gpu():
    L = _lib.lib()
    h = ctypes.c_void_p()
    rc = L.svb_create(0, 1, 0, ctypes.byref(h))
    assert rc == _lib.SVB_E_ARG
    assert b"n_qubits" in L.svb_last_error()


# ---------------------------------------------------------- scheduler (CPU)
def _emu_check(c, prec, tol, relabel=1):
    """relabel: 0 = swaps as ops, 1 = swap relabeling + final permutation
    (separate pass or fused into the last pass's store), 2 = relabeling with
    the lazy-zero layout choice (initial layout makes the final map identity)."""
    n = c.n_qubits
    ref = orc.unitary_state(c)
    psi0 = np.zeros(1 << n, dtype=complex)
    psi0[0] = 1
    got = emulate(n, c.instructions, psi0, prec, relabel=relabel)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err < tol, (n, len(c.instructions), err)


@pytest.mark.parametrize("prec,tol,nmin", [("c128", 1e-12, 9), ("c64", 1e-5, 10)])
def test_fused_program_random_circuits(prec, tol, nmin):
    rng = np.random.default_rng(7)
    for trial in range(25):
        n = int(rng.integers(nmin, nmin + 4))
        c = suite.random_circuit(n, int(rng.integers(1, 150)), rng, measured=False)
        _emu_check(c, prec, tol, relabel=trial % 3)


def test_fused_program_structured_circuits():
    for c in (
        suite.qft_bench_circuit(13),
        suite.sycamore_circuit(3, 4, 8, seed=3, measured=False),
        suite.qaoa_line_circuit(12, 2, seed=1, measured=False),
        suite.ry_ansatz_circuit(11, 3, seed=2, measured=False),
        suite.ghz_circuit(14, measured=False),
    ):
        for relabel in (1, 2):
            _emu_check(c, "c128", 1e-12, relabel)
            _emu_check(c, "c64", 1e-5, relabel)


def _random_state(n, seed):
    rng = np.random.default_rng(seed)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return psi / np.linalg.norm(psi)


@pytest.mark.parametrize("n", [12, 13])
def test_permuted_store_fused_into_last_pass(n):
    """QFT-n on an arbitrary input state: its final bit reversal lands in the
    last pass's tile set, so the permutation is done by that pass's store."""
    c = suite.qft_bench_circuit(n)
    p = sv.plan(n, c.instructions, "c128")
    if n == 12:
        assert p["permute_fused"], p
    psi0 = _random_state(n, n)
    ref = psi0.copy()
    for inst in c.instructions:
        orc.apply_instruction(ref, n, inst)
    for prec, tol in (("c128", 1e-12), ("c64", 1e-5)):
        got = emulate(n, c.instructions, psi0, prec, relabel=1)
        assert np.linalg.norm(got - ref) < tol, prec


def test_random_swap_circuits_on_arbitrary_state():
    rng = np.random.default_rng(21)
    fused = 0
    for trial in range(12):
        n = int(rng.integers(10, 13))
        c = Circuit(n)
        for _ in range(int(rng.integers(5, 60))):
            r = rng.random()
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            if r < 0.35:
                c.gate("swap", a, b)
            elif r < 0.6:
                c.gate("cx", a, b)
            else:
                c.gate("u", a, params=tuple(float(x) for x in rng.uniform(0, 6.3, 3)))
        psi0 = _random_state(n, trial)
        ref = psi0.copy()
        for inst in c.instructions:
            orc.apply_instruction(ref, n, inst)
        fused += sv.plan(n, c.instructions, "c128")["permute_fused"]
        got = emulate(n, c.instructions, psi0, "c128", relabel=1)
        assert np.linalg.norm(got - ref) < 1e-12, trial
    assert fused > 0  # the permuted-store path was exercised


@pytest.mark.parametrize("prec,tol", [("c128", 1e-12), ("c64", 1e-5)])
def test_initial_permutation_schedule_on_arbitrary_state(prec, tol):
    """Written input + swaps: schedules that permute the input first (into the
    layout absorbing the relabeling) must equal the gate-by-gate result, for
    swap permutations that are not involutions too."""
    initial = 0
    for seed in range(14):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(12, 16))
        c = suite.random_circuit(n, 120, rng, measured=False)
        psi0 = _random_state(n, seed)
        ref = psi0.copy()
        for inst in c.instructions:
            orc.apply_instruction(ref, n, inst)
        initial += sv.plan(n, c.instructions, prec)["permute_initial"]
        got = emulate(n, c.instructions, psi0, prec, relabel=1)
        assert np.linalg.norm(got - ref) < tol, seed
    q = suite.qft_bench_circuit(13)
    assert sv.plan(13, q.instructions, prec)["permute_initial"] or prec == "c64"
    assert initial > 0


def test_fused_program_dft_known_answer():
    n = 12
    basis = 0b101100111010
    c = Circuit(n)
    for q in range(n):
        if (basis >> q) & 1:
            c.gate("x", q)
    suite.qft(n, c)
    psi0 = np.zeros(1 << n, dtype=complex)
    psi0[0] = 1
    got = emulate(n, c.instructions, psi0, "c128")
    k = np.arange(1 << n)
    want = np.exp(2j * math.pi * basis * k / (1 << n)) / math.sqrt(1 << n)
    np.testing.assert_allclose(got, want, atol=1e-12)


def test_mirror_circuit_returns_to_zero():
    rng = np.random.default_rng(11)
    c = suite.random_circuit(11, 120, rng, measured=False)
    body = c.instructions + inverse_circuit(c).instructions
    psi0 = np.zeros(1 << 11, dtype=complex)
    psi0[0] = 1
    got = emulate(11, body, psi0, "c128")
    assert abs(got[0]) > 1 - 1e-10


def test_plan_pass_counts():
    p = sv.plan(30, suite.qft_bench_circuit(30).instructions, "c128")
    assert p["passes"] == 4 and p["permute"]  # ceil((30 - 5) / 7): every pass advances 7 qubits
    p = sv.plan(30, suite.qft_bench_circuit(30).instructions, "c128", zero_start=True)
    assert p["passes"] == 4 and not p["permute"]  # lazy |0...0>: the layout absorbs the bit reversal
    p = sv.plan(24, [Instruction("h", (q,)) for q in range(24)], "c128")
    assert p["passes"] == math.ceil((24 - 5) / 7)


def test_polysim_shim_installs_and_restores():
    """Drop-in swap of polysim.statevector; needs the reference.
    The qubit cap is lifted everywhere it was bound at import (dispatch.py:18,
    predictor.py:119, the installed functions) and restored by uninstall."""
    import inspect
    import sys as _sys

    from conftest import reference_src

    ref_src = reference_src()
    if ref_src is None:
        pytest.skip("reference package not available")
    _sys.path.insert(0, ref_src)
    try:
        import polysim.dispatch as ref_dispatch
        import polysim.pblock as ref_pb
        import polysim.predictor as ref_pred
        import polysim.result as ref_res
        import polysim.sampling as ref_samp
        import polysim.statevector as ref_sv
        from paper_2512_04216_b200 import pblock as dev_pb
        from paper_2512_04216_b200 import polysim_shim
        from paper_2512_04216_b200 import sampling as dev_samp

        def cap_default(fn):
            return inspect.signature(fn).parameters["qubit_cap"].default

        orig, orig_pb, orig_at = ref_sv.run, ref_pb.run, ref_samp.AliasTable
        polysim_shim.install()
        assert ref_sv.run is sv.run and ref_sv.final_state is sv.final_state
        assert ref_sv.DEFAULT_QUBIT_CAP == 26 and ref_pb.run is orig_pb and ref_samp.AliasTable is orig_at
        polysim_shim.uninstall()
        assert ref_sv.run is orig
        polysim_shim.install(qubit_cap=30, pblock=True, sampling=True)
        assert ref_sv.DEFAULT_QUBIT_CAP == 30 and sv.DEFAULT_QUBIT_CAP == 30
        for fn in (ref_dispatch.run_circuit, ref_pred.select_backend, sv.run, sv.final_state, sv.expectation):
            assert cap_default(fn) == 30, fn
        assert ref_pb.run is dev_pb.run and ref_pb.PBlockState is dev_pb.PBlockState
        assert ref_samp.AliasTable is dev_samp.AliasTable and ref_res.AliasTable is dev_samp.AliasTable
        polysim_shim.uninstall()
        assert ref_sv.DEFAULT_QUBIT_CAP == 26 and ref_pb.run is orig_pb and ref_sv.run is orig
        assert sv.DEFAULT_QUBIT_CAP == 26 and ref_samp.AliasTable is orig_at and ref_res.AliasTable is orig_at
        for fn in (ref_dispatch.run_circuit, ref_pred.select_backend, sv.run, sv.final_state, sv.expectation):
            assert cap_default(fn) == 26, fn
    finally:
        _sys.path.remove(ref_src)


@pytest.mark.parametrize("n", [12, 13])
def test_long_pass_stays_in_range_c64(n):
    """Hundreds of pivoted 1q ops in one pass: the deferred scalar K must be
    re-absorbed before complex64 amplitudes drift toward overflow.  At n = 12
    the whole circuit is one tile, so a pass overflows kMaxRounds and its tail
    is deferred to the next pass."""
    c = Circuit(n)
    rng = np.random.default_rng(3)
    for layer in range(40):
        for q in range(n):
            c.gate("ry", q, params=(float(rng.uniform(0, 3)),))
            c.gate("rx", q, params=(float(rng.uniform(0, 3)),))
        for q in range(layer % 2, n - 1, 2):
            c.gate("cz", q, q + 1)
    assert sv.plan(n, c.instructions, "c64")["passes"] >= 1
    _emu_check(c, "c64", 1e-4)
    _emu_check(c, "c128", 1e-11)


def test_calibration_host_logic():
    """GPU sv cost curves slot into the reference's CalibrationModel/predictor
    (SURVEY §8f rank 2); the timing itself is a gpu test."""
    from paper_2512_04216_b200 import calibration as cal

    assert cal.qubit_cap_for_bytes(180 * 2**30, "c128", spare=False) == 33
    assert cal.qubit_cap_for_bytes(180 * 2**30, "c64", spare=False) == 34
    assert cal.qubit_cap_for_bytes(180 * 2**30, "c128") == 32
    c1, c2 = cal.fit_shot_model([1, 10, 100], [1.0 + 2e-3, 1.0 + 2e-2, 1.0 + 2e-1])
    assert abs(c1 - 1.0) < 1e-12 and abs(c2 - 2e-3) < 1e-12
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        pytest.skip("reference not present (GPU box)")
    import sys as _sys

    _sys.path.insert(0, ref_src)
    try:
        from polysim.calibration import CalibrationModel
        from polysim.predictor import estimate
        from polysim.suite import ghz_circuit

        base = {
            "version": 1, "created": "test",
            "sv": {"grid_n": [2, 4], "curves": {"1q": [1e-8, 1e-8], "2q": [2e-8, 2e-8]}},
            "mps": {"grid_n": [4, 8], "grid_chi": [2, 4],
                    "surfaces": {k: [[1e-6, 1e-6], [1e-6, 1e-6]] for k in ("1q", "2q", "measure")}},
            "stab": {"grid_n": [4, 8], "curves": {"gate": [1e-6, 1e-6], "measure": [1e-6, 1e-6]}},
            "shots": {k: {"c1": 1e-3, "c2": 1e-6} for k in ("sv", "mps", "stab")},
            "alpha": [1.0],
        }
        section = {"sv": {"grid_n": [2, 10, 20], "curves": {"1q": [1e-9, 5e-12, 1e-12], "2q": [2e-9, 6e-12, 2e-12]}},
                   "shots": {"sv": {"c1": 2e-4, "c2": 3e-8}}}
        model = cal.merge_sv_section(CalibrationModel.from_dict(base), section)
        assert isinstance(model, CalibrationModel)
        assert model.sv_grid == (2, 10, 20) and model.shot_coeffs["sv"] == (2e-4, 3e-8)
        assert model.shot_coeffs["mps"] == (1e-3, 1e-6)
        c = ghz_circuit(20)
        t = estimate(c, "sv", model, shots=1000)
        want = (1 * 1e-12 + 19 * 2e-12) * 2**20 + 2e-4 + 3e-8 * 1000
        assert abs(t - want) < 1e-12 * want
    finally:
        _sys.path.remove(ref_src)


@pytest.mark.parametrize("which", ["qft30_c128", "qft20_c128", "qft12_permstore", "syc_c64", "random_c64",
                                   "qft30_zero_start_z", "syc_c64_zero_start"])
def test_jit_sources_compile(which):
    """NVRTC compiles every generated pass kernel (a failure would otherwise
    fall back to the interpreter body at run time)."""
    import ctypes as _ct

    if which == "qft30_c128":
        n, prec, c = 30, 1, suite.qft_bench_circuit(30)
    elif which == "qft20_c128":
        n, prec, c = 20, 1, suite.qft_bench_circuit(20)
    elif which == "qft12_permstore":  # last pass stores to the bit-reversed addresses
        n, prec, c = 12, 1, suite.qft_bench_circuit(12)
    elif which == "qft30_zero_start_z":  # support tracking (dmask loads) + fused <Z> on the last pass
        n, prec, c = 30, 0x301, suite.qft_bench_circuit(30)
    elif which == "syc_c64_zero_start":
        n, prec, c = 28, 0x100, suite.sycamore_circuit(4, 7, 12, seed=0, measured=False)
    elif which == "syc_c64":
        n, prec, c = 28, 0, suite.sycamore_circuit(4, 7, 12, seed=0, measured=False)
    else:
        n, prec = 22, 0
        c = suite.random_circuit(22, 300, np.random.default_rng(2), measured=False)
    g = sv.gate_array(c.instructions)
    cb = _ct.c_int64()
    buf = _ct.create_string_buffer(1 << 14)
    rc = _lib.lib().svb_jit_check(n, prec, g.ctypes.data_as(_ct.c_void_p), int(g.size), _ct.byref(cb), buf, 1 << 14)
    if rc != 0 and b"nvrtc" in buf.value.lower() and b"not available" in buf.value.lower():
        pytest.skip("NVRTC not available")
    assert rc == 0, buf.value.decode(errors="replace")[:2000]
    assert cb.value > 0


def test_bulk_row_store_epilogue_emitted_only_where_rows_are_contiguous(tmp_path, monkeypatch):
    """The one-round direct complex128 pass whose thread bits are qubits 0..7
    (the QFT-30 bench's last pass) gets the bulk-row-store epilogue
    (SVB_BULK_ROWS: rows through shared memory, cp.async.bulk); passes whose
    register rows are not contiguous runs (a written-input QFT-20, complex64
    Sycamore) keep register stores only."""
    import ctypes as _ct

    monkeypatch.setenv("SVB_JIT_NOCOMPILE", "1")

    def dump(n, prec, c, name):
        path = tmp_path / name
        monkeypatch.setenv("SVB_JIT_DUMP", str(path))
        g = sv.gate_array(c.instructions)
        cb = _ct.c_int64()
        buf = _ct.create_string_buffer(1 << 12)
        rc = _lib.lib().svb_jit_check(n, prec, g.ctypes.data_as(_ct.c_void_p), int(g.size), _ct.byref(cb), buf, 1 << 12)
        assert rc == 0, buf.value
        return path.read_text()

    src = dump(30, 0x301, suite.qft_bench_circuit(30), "qft30.cu")
    bodies = src.split('#include "device_core.cuh"')[1:]
    assert len(bodies) == 5  # four passes + the bulk variant jit_check also compiles
    assert ["#if SVB_BULK_ROWS" in b for b in bodies[:4]] == [False, False, False, True]
    assert "svb::bulk_store_row(" in bodies[3] and src.count("#define SVB_BULK_ROWS 1") == 1
    assert "#if SVB_BULK_ROWS" not in dump(20, 1, suite.qft_bench_circuit(20), "qft20.cu")
    syc = suite.sycamore_circuit(4, 7, 12, seed=0, measured=False)
    assert "#if SVB_BULK_ROWS" not in dump(28, 0x100, syc, "syc.cu")


def test_structure_only_jit_sources_do_not_depend_on_angles(tmp_path, monkeypatch):
    """Below 28 qubits the NVRTC passes load their coefficients, so circuits
    that differ only in angles generate the same kernel sources (a VQE / QAOA
    loop compiles once): the deferred diagonals are flushed by structure, not
    by value.  The pivot of a 1q op stays in the source; it changes only for
    angles within ~2^-8 of a singular pivot (|cos(theta/2)| tiny), which the
    angles here avoid."""
    import ctypes as _ct
    import math

    from paper_2512_04216_b200.circuit import Circuit

    def ry_ansatz(n, seed):
        rng = np.random.default_rng(seed)
        c = Circuit(n)
        for layer in range(3):
            for q in range(n):  # |theta - pi| > 0.1: the diagonal stays the pivot
                th = rng.uniform(0.1, math.pi - 0.1) + (math.pi if rng.random() < 0.5 else 0.0)
                c.gate("ry", q, params=(th,))
            if layer < 2:
                for q in range(n - 1):
                    c.gate("cx", q, q + 1)
        return c

    def qaoa(n, seed):
        rng = np.random.default_rng(seed)
        c = Circuit(n)
        for q in range(n):
            c.gate("h", q)
        for _ in range(2):
            g, b = rng.uniform(0.1, 1.4, size=2)  # rx(2b) with 2b away from pi
            for q in range(n - 1):
                c.gate("cx", q, q + 1).gate("rz", q + 1, params=(2 * g,)).gate("cx", q, q + 1)
            for q in range(n):
                c.gate("rx", q, params=(2 * b,))
        return c

    monkeypatch.setenv("SVB_JIT_NOCOMPILE", "1")
    for fam in (ry_ansatz, qaoa):
        srcs = set()
        for seed in range(12):
            c = fam(24, seed)
            path = tmp_path / f"{fam.__name__}{seed}.cu"
            monkeypatch.setenv("SVB_JIT_DUMP", str(path))
            g = sv.gate_array(c.instructions)
            cb = _ct.c_int64()
            buf = _ct.create_string_buffer(1 << 12)
            rc = _lib.lib().svb_jit_check(24, 1 | 0x100, g.ctypes.data_as(_ct.c_void_p), int(g.size), _ct.byref(cb),
                                          buf, 1 << 12)
            assert rc == 0, buf.value
            srcs.add(path.read_text())
        assert len(srcs) == 1, (fam.__name__, len(srcs))


def test_state_pool_keeps_the_latest_release():
    """The idle-state pool (32 GiB) keeps the state released last and closes
    older idle states to make room; a state larger than the cap is closed."""

    class Fake:
        def __init__(self, n, precision):
            self.n, self.precision, self.device, self.closed = n, precision, 0, False

        def close(self):
            self.closed = True

    pool = sv._StatePool()
    a, b, c = Fake(30, "c128"), Fake(32, "c64"), Fake(30, "c128")
    pool.release(a)
    assert pool.bytes == 16 << 30 and not a.closed
    pool.release(b)  # 32 GiB: a is closed to make room
    assert a.closed and not b.closed and pool.bytes == 32 << 30
    pool.release(c)
    assert b.closed and not c.closed and pool.bytes == 16 << 30
    big = Fake(33, "c128")
    pool.release(big)
    assert big.closed and pool.bytes == 16 << 30
    assert pool.acquire(30, "c128", 0) is c and pool.bytes == 0
