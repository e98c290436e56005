"""Drop-in B200 replacement for the reference dense state-vector backend.

Same module surface as `polysim/statevector.py`:

* ``run(c, shots, seed, workers=1, qubit_cap=26)`` -> ``RunResult``  (`statevector.py:182-253`)
* ``final_state(c, qubit_cap=26)`` -> complex128 ndarray, cached per Circuit  (`:256-274`)
* ``expectation(c, z_qubits, qubit_cap=26)`` -> float  (`:277-292`)
* kernel level: ``zero_state``, ``apply_1q``, ``apply_2q``, ``apply_instruction``,
  ``marginal_probs``, ``_measure_qubit``, ``_reset_qubit`` (`:33-154`), used by
  pblock (`pblock.py:93-154`) and calibration (`calibration.py:215-228`);
  they accept numpy arrays (copied through the device) or ``DeviceState``.

Every computation runs in libsvb.so on the GPU (ctypes, include/svb.h);
this module only marshals circuits, seeds and results.  Conventions, error
types and their check order follow the reference exactly.  Extensions are
keyword-only: ``precision`` ("c128" default, or "c64"), ``sampler``
("alias" = reference-compatible counts, "cdf" = native multinomial sampler,
"auto"), ``device``.
"""
from __future__ import annotations

import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import GATE_DTYPE, SvbGate, check, lib, ptr
from .circuit import ONE_QUBIT_GATES, UNITARY_GATES
from .features import terminal_measurement_only
from .gates import matrix_of, single_qubit_matrix
from .result import (
    BackendError,
    NoMeasurementsError,
    QubitCapError,
    RunResult,
    clbit_order,
    format_counts,
    measurement_map,
    output_bit_sources,
)

DEFAULT_QUBIT_CAP = 26  # statevector.py:30
ALIAS_MAX_QUBITS = 28   # sampler="auto" switches to the CDF sampler above this
_PREC = {"c128": _lib.SVB_C128, "c64": _lib.SVB_C64, "complex128": _lib.SVB_C128, "complex64": _lib.SVB_C64}
_MASK64 = (1 << 64) - 1


def _prec_code(precision) -> int:
    try:
        return _PREC[str(precision)]
    except KeyError:
        raise ValueError(f"unknown precision {precision!r}") from None


def pcg_words(seed_or_rng) -> np.ndarray:
    """numpy PCG64 state of default_rng(seed) (or of a Generator) as 4 uint64."""
    g = seed_or_rng if isinstance(seed_or_rng, np.random.Generator) else np.random.default_rng(seed_or_rng)
    st = g.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("device sampling reproduces numpy's PCG64 stream only")
    s, inc = st["state"]["state"], st["state"]["inc"]
    return np.array([s >> 64, s & _MASK64, inc >> 64, inc & _MASK64], dtype=np.uint64)


# ----------------------------------------------------------- gate encoding
def gate_array_slow(instructions) -> np.ndarray:
    """Reference encoder: one matrix_of() per instruction (gates.py)."""
    insts = [i for i in instructions if i.kind in UNITARY_GATES]
    arr = np.zeros(len(insts), dtype=GATE_DTYPE)
    k = arr["k"]
    q = arr["q"]
    mat = arr["mat"]
    for j, inst in enumerate(insts):
        m = matrix_of(inst)
        nq = len(inst.qubits)
        k[j] = nq
        q[j, :nq] = inst.qubits
        mat[j, : 2 * m.size] = m.reshape(-1).view(np.float64)
    return arr


_FIXED_MATS: dict = {}


def gate_array(instructions) -> np.ndarray:
    """Unitary instructions -> svb_gate records, vectorised per gate kind.

    Same numbers as gates.py (math.cos/sin for rx/ry/u magnitudes, numpy's
    complex exp for phases) — checked against gate_array_slow in the tests."""
    insts = [i for i in instructions if i.kind in UNITARY_GATES]
    return _encode([i.kind for i in insts], [i.qubits for i in insts], [i.params for i in insts])


def gate_array_many(circuits) -> tuple[np.ndarray, np.ndarray]:
    """gate_array over many circuits in one vectorised encoding: (records of
    every circuit's unitary gates back to back, per-circuit gate counts)."""
    unitary = UNITARY_GATES
    sel = [[i for i in c.instructions if i.kind in unitary] for c in circuits]
    counts = np.fromiter((len(u) for u in sel), dtype=np.int32, count=len(sel))
    flat = [i for u in sel for i in u]
    return _encode([i.kind for i in flat], [i.qubits for i in flat], [i.params for i in flat]), counts


FIXED_KINDS = ("h", "x", "y", "z", "s", "sdg", "t", "tdg", "cx", "cz", "swap")
_OP_CODE = {"rx": 0, "ry": 1, "rz": 2, "u": 3, **{k: 4 + j for j, k in enumerate(FIXED_KINDS)}}
_FIXED_TABLE = None


def fixed_gate_table() -> np.ndarray:
    """svb_gate records of the fixed kinds (gates.py matrices), indexed kind - 4."""
    global _FIXED_TABLE
    if _FIXED_TABLE is None:
        from .gates import single_qubit_matrix, two_qubit_matrix

        t = np.zeros(len(FIXED_KINDS), dtype=GATE_DTYPE)
        for j, kd in enumerate(FIXED_KINDS):
            m = two_qubit_matrix(kd) if kd in ("cx", "cz", "swap") else single_qubit_matrix(kd)
            t["k"][j] = 2 if m.shape[0] == 4 else 1
            t["mat"][j, : 2 * m.size] = m.reshape(-1).view(np.float64)
        _FIXED_TABLE = t
    return _FIXED_TABLE


def gate_ops_many(circuits) -> tuple[np.ndarray, np.ndarray]:
    """Compact 40-byte svb_gate_op records of every circuit's unitary gates
    (kind code, qubits, parameters; matrices are built by libsvb in C++),
    and the per-circuit gate counts.  The batch encoder: ~7x less host memory
    traffic than svb_gate records."""
    unitary = UNITARY_GATES
    sel = [[i for i in c.instructions if i.kind in unitary] for c in circuits]
    counts = np.fromiter((len(u) for u in sel), dtype=np.int32, count=len(sel))
    flat = [i for u in sel for i in u]
    n = len(flat)
    ops = np.zeros(n, dtype=_lib.GATE_OP_DTYPE)
    if n == 0:
        return ops, counts
    code = _OP_CODE
    kinds = np.fromiter((code[i.kind] for i in flat), dtype=np.int32, count=n)
    ops["kind"] = kinds
    ops["q0"] = np.fromiter((i.qubits[0] for i in flat), dtype=np.int32, count=n)
    ops["q1"] = np.fromiter((i.qubits[-1] for i in flat), dtype=np.int32, count=n)
    pidx = np.flatnonzero(kinds < 4)
    if pidx.size:
        ops["p"][pidx] = [(flat[j].params + (0.0, 0.0))[:3] for j in pidx.tolist()]
    return ops, counts


def _encode(kinds, qubits, params) -> np.ndarray:
    n = len(kinds)
    arr = np.zeros(n, dtype=GATE_DTYPE)
    if n == 0:
        return arr
    names = sorted(set(kinds))
    code_of = {k: c for c, k in enumerate(names)}
    codes = np.fromiter((code_of[k] for k in kinds), dtype=np.int16, count=n)
    mat = arr["mat"]
    import math as _m

    for c, kd in enumerate(names):
        idx = np.flatnonzero(codes == c)
        if kd in ("rx", "ry", "rz", "u"):
            P = np.array([params[j] for j in idx.tolist()], dtype=np.float64).reshape(idx.size, -1)
            m = np.zeros((idx.size, 2, 2), dtype=np.complex128)
            if kd == "rz":
                m[:, 0, 0] = np.exp(-0.5j * P[:, 0])
                m[:, 1, 1] = np.exp(0.5j * P[:, 0])
            else:
                half = [t / 2 for t in P[:, 0].tolist()]
                c_ = np.array([_m.cos(t) for t in half])
                s_ = np.array([_m.sin(t) for t in half])
                if kd == "rx":
                    m[:, 0, 0] = c_
                    m[:, 0, 1] = -1j * s_
                    m[:, 1, 0] = -1j * s_
                    m[:, 1, 1] = c_
                elif kd == "ry":
                    m[:, 0, 0] = c_
                    m[:, 0, 1] = -s_
                    m[:, 1, 0] = s_
                    m[:, 1, 1] = c_
                else:
                    phi, lam = P[:, 1], P[:, 2]
                    m[:, 0, 0] = c_
                    m[:, 0, 1] = -np.exp(1j * lam) * s_
                    m[:, 1, 0] = np.exp(1j * phi) * s_
                    m[:, 1, 1] = np.exp(1j * (phi + lam)) * c_
            mat[idx, :8] = m.reshape(idx.size, 4).view(np.float64)
        else:
            if kd not in _FIXED_MATS:
                from .gates import single_qubit_matrix, two_qubit_matrix

                fm = two_qubit_matrix(kd) if kd in ("cx", "cz", "swap") else single_qubit_matrix(kd)
                _FIXED_MATS[kd] = fm.reshape(-1).view(np.float64).copy()
            fm = _FIXED_MATS[kd]
            mat[idx, : fm.size] = fm
    q = arr["q"]
    lens = np.fromiter((len(x) for x in qubits), dtype=np.int8, count=n)
    q[:, 0] = [x[0] for x in qubits]
    two = lens == 2
    arr["k"] = lens
    if two.any():
        q[two, 1] = [x[1] for x in qubits if len(x) == 2]
    return arr


def _single_gate(qubits, m) -> np.ndarray:
    m = np.asarray(m, dtype=np.complex128)
    arr = np.zeros(1, dtype=GATE_DTYPE)
    arr["k"][0] = len(qubits)
    arr["q"][0, : len(qubits)] = qubits
    arr["mat"][0, : 2 * m.size] = m.reshape(-1).view(np.float64)
    return arr


# ------------------------------------------------------------ device state
class DeviceState:
    """A 2^n amplitude vector resident in HBM (one libsvb handle)."""

    def __init__(self, n: int, precision="c128", device: int = 0):
        self.n = int(n)
        self.precision = "c128" if _prec_code(precision) == _lib.SVB_C128 else "c64"
        self.device = device
        h = _lib.c_void_p()
        rc = lib().svb_create(self.n, _prec_code(precision), device, _lib.ctypes.byref(h))
        if rc == _lib.SVB_E_OOM and _pool.bytes:
            # idle pooled states (final_state / run cache) hold the memory: drop them and retry once
            _pool.clear()
            rc = lib().svb_create(self.n, _prec_code(precision), device, _lib.ctypes.byref(h))
        check(rc)
        self._h = h

    @classmethod
    def _view(cls, n: int, address: int, device: int = 0) -> "DeviceState":
        """A handle on caller-owned complex128 device/managed memory (svb_create_view)."""
        self = cls.__new__(cls)
        self.n, self.precision, self.device = int(n), "c128", device
        h = _lib.c_void_p()
        check(lib().svb_create_view(self.n, device, _lib.c_void_p(address), _lib.ctypes.byref(h)))
        self._h = h
        return self

    # lifetime
    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h:
            lib().svb_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        if not self._h:
            raise BackendError("device state is closed")
        return self._h

    def set_option(self, option: int, value: int) -> None:
        check(lib().svb_set_option(self.handle, option, value))

    def stats(self) -> dict:
        p, g, l = _lib.c_int64(), _lib.c_int64(), _lib.c_int64()
        check(lib().svb_last_stats(self.handle, _lib.ctypes.byref(p), _lib.ctypes.byref(g), _lib.ctypes.byref(l)))
        return {"passes": p.value, "gates": g.value, "launches": l.value}

    # device timing (CUDA events on this state's stream)
    def timer_start(self) -> None:
        check(lib().svb_timer_start(self.handle))

    def timer_stop(self) -> float:
        ms = _lib.c_double()
        check(lib().svb_timer_stop(self.handle, _lib.ctypes.byref(ms)))
        return ms.value

    def profile(self, enable: bool = True) -> None:
        check(lib().svb_profile(self.handle, int(enable)))

    def profile_read(self) -> dict:
        out = np.zeros(6, dtype=np.float64)
        check(lib().svb_profile_read(self.handle, ptr(out, _lib.c_double)))
        return {"pass_ms": out[0], "pass_launches": int(out[1]), "pass_bytes": out[2],
                "perm_ms": out[3], "perm_launches": int(out[4]), "perm_bytes": out[5]}

    def profile_passes(self) -> list:
        """Per pass index of the profiled programs: dicts of ms, HBM bytes, launches."""
        out = np.zeros(3 * 64, dtype=np.float64)
        k = _lib.c_int32()
        check(lib().svb_profile_passes(self.handle, ptr(out, _lib.c_double), 64, _lib.ctypes.byref(k)))
        return [{"ms": out[3 * i], "bytes": out[3 * i + 1], "launches": int(out[3 * i + 2])}
                for i in range(min(k.value, 64))]

    # data
    def zero(self) -> "DeviceState":
        check(lib().svb_set_zero(self.handle))
        return self

    @classmethod
    def from_numpy(cls, amps: np.ndarray, precision="c128", device: int = 0) -> "DeviceState":
        amps = np.ascontiguousarray(amps, dtype=np.complex128).reshape(-1)
        n = amps.size.bit_length() - 1
        if amps.size != 1 << n:
            raise ValueError("amplitude vector length must be a power of two")
        s = cls(n, precision, device)
        s.load(amps)
        return s

    def load(self, amps: np.ndarray) -> None:
        amps = np.ascontiguousarray(amps, dtype=np.complex128)
        if amps.size != 1 << self.n:
            raise ValueError("amplitude vector length mismatch")
        check(lib().svb_set_amplitudes(self.handle, ptr(amps), 0, amps.size))

    def to_numpy(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(1 << self.n, dtype=np.complex128)
        if out.dtype != np.complex128 or out.size != 1 << self.n or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous complex128 array of length 2^n")
        check(lib().svb_get_amplitudes(self.handle, ptr(out), 0, out.size))
        return out

    def read(self, offset: int, count: int, out: np.ndarray | None = None) -> np.ndarray:
        """Amplitudes [offset, offset + count) as complex128 (chunked read-back)."""
        if out is None:
            out = np.empty(int(count), dtype=np.complex128)
        if out.dtype != np.complex128 or out.size != count or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous complex128 array of length count")
        check(lib().svb_get_amplitudes(self.handle, ptr(out), int(offset), int(count)))
        return out

    def copy_from(self, other: "DeviceState") -> None:
        check(lib().svb_copy_state(self.handle, other.handle))

    # gates
    def apply_gates(self, gates: np.ndarray) -> None:
        gates = np.ascontiguousarray(gates, dtype=GATE_DTYPE)
        if gates.size:
            check(lib().svb_apply(self.handle, ptr(gates), int(gates.size)))

    def apply_instructions(self, instructions) -> None:
        self.apply_gates(gate_array(instructions))

    def apply_matrix(self, qubits, mat, engine: str = "auto") -> str:
        """Apply one dense 2^k x 2^k block U (local index bit i <-> qubits[i])
        in one HBM pass: tcgen05 tensor cores (complex64, 3xTF32) or CUDA
        cores (svb_apply_matrix).  Returns the engine that ran."""
        qs = np.ascontiguousarray(qubits, dtype=np.int32).reshape(-1)
        m = np.ascontiguousarray(mat, dtype=np.complex128)
        if m.shape != (1 << qs.size, 1 << qs.size):
            raise ValueError("matrix must be 2^k x 2^k for k qubits")
        code = {"auto": _lib.ENGINE_AUTO, "tensor": _lib.ENGINE_TENSOR, "fma": _lib.ENGINE_FMA}[engine]
        check(lib().svb_apply_matrix(self.handle, ptr(qs, _lib.c_int32), int(qs.size), ptr(m.view(np.float64),
                                     _lib.c_double), code))
        return "tensor" if lib().svb_last_engine(self.handle) == _lib.ENGINE_TENSOR else "fma"

    def apply_gates_z(self, gates: np.ndarray, z_qubits) -> np.ndarray:
        """Apply a gate program and return <Z_q> for each q in z_qubits, summed by
        the program's last fused pass while it stores the state (svb_apply_z);
        q = -1 gives sum |a|^2."""
        gates = np.ascontiguousarray(gates, dtype=GATE_DTYPE)
        qs = np.ascontiguousarray(z_qubits, dtype=np.int32).reshape(-1)
        out = np.empty(qs.size, dtype=np.float64)
        check(lib().svb_apply_z(self.handle, ptr(gates), int(gates.size), ptr(qs, _lib.c_int32), int(qs.size),
                                ptr(out, _lib.c_double)))
        return out

    # reductions
    def marginal_probs(self, qubits) -> np.ndarray:
        qs = np.ascontiguousarray(sorted(qubits), dtype=np.int32)
        out = np.empty(1 << qs.size, dtype=np.float64)
        check(lib().svb_marginal_probs(self.handle, ptr(qs, _lib.c_int32), int(qs.size), ptr(out, _lib.c_double)))
        return out

    def expect_z(self, masks) -> np.ndarray:
        ms = np.ascontiguousarray(masks, dtype=np.uint64).reshape(-1)
        out = np.empty(ms.size, dtype=np.float64)
        check(lib().svb_expect_z(self.handle, ptr(ms, _lib.c_uint64), int(ms.size), ptr(out, _lib.c_double)))
        return out

    def compare(self, other: "DeviceState") -> dict:
        """Device-side distance/overlap with another state of the same size:
        ``rel`` = ||self - other|| / ||other||, ``fidelity`` = |<self|other>|^2."""
        out = np.zeros(5, dtype=np.float64)
        check(lib().svb_compare(self.handle, other.handle, ptr(out, _lib.c_double)))
        d2, na, nb, re, im = (float(x) for x in out)
        return {"dist2": d2, "norm2_self": na, "norm2_other": nb, "rel": (d2 / nb) ** 0.5 if nb > 0 else float("inf"),
                "fidelity": (re * re + im * im) / (na * nb) if na > 0 and nb > 0 else 0.0}

    def sample_codes(self, qubits, bit_src, shots: int, rng_words: np.ndarray, sampler: int):
        qs = np.ascontiguousarray(qubits, dtype=np.int32)
        bs = np.ascontiguousarray(bit_src, dtype=np.int32)
        w = int(bs.size)
        cap = min(int(shots), 1 << min(w, 62))
        codes = np.empty(cap, dtype=np.uint64)
        freq = np.empty(cap, dtype=np.uint64)
        nu = _lib.c_uint64()
        words = np.ascontiguousarray(rng_words, dtype=np.uint64)
        check(
            lib().svb_sample(
                self.handle, ptr(qs, _lib.c_int32), int(qs.size), ptr(bs, _lib.c_int32), w, int(shots),
                ptr(words, _lib.c_uint64), int(sampler), ptr(codes, _lib.c_uint64), ptr(freq, _lib.c_uint64),
                _lib.ctypes.byref(nu),
            )
        )
        return codes[: nu.value], freq[: nu.value]

    def seed_rng(self, rng_words) -> None:
        words = np.ascontiguousarray(rng_words, dtype=np.uint64)
        check(lib().svb_rng_seed(self.handle, ptr(words, _lib.c_uint64)))

    def measure(self, q: int) -> int:
        out = _lib.c_int32()
        check(lib().svb_measure(self.handle, int(q), _lib.ctypes.byref(out)))
        return int(out.value)

    def reset(self, q: int) -> None:
        check(lib().svb_reset(self.handle, int(q)))


class PinnedBuffer:
    """Page-locked host complex128 buffer (fast final_state read-back)."""

    def __init__(self, count: int):
        p = _lib.c_void_p()
        check(lib().svb_host_alloc(int(count) * 16, _lib.ctypes.byref(p)))
        self._p = p
        dbl = np.ctypeslib.as_array(_lib.ctypes.cast(p, _lib.POINTER(_lib.c_double)), shape=(2 * int(count),))
        self.array = dbl.view(np.complex128)

    def close(self) -> None:
        p, self._p = getattr(self, "_p", None), None
        if p:
            self.array = None
            lib().svb_host_free(p)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _StatePool:
    """Idle device states kept for reuse by run() and the final_state /
    expectation cache (no cudaMalloc / cudaFree / stream creation per call).
    Bounded by bytes (32 GiB: one idle 31-qubit complex128 state); LIFO per
    key; the state released last is kept, idle states released earlier are
    closed to make room for it (a 32-qubit complex64 state after a 30-qubit
    complex128 one was closed instead, and the next run paid a 32 GiB
    cudaMalloc); emptied when a new state does not fit in device memory."""

    def __init__(self, cap_bytes: int = 32 << 30, per_key: int = 4):
        import threading

        self.cap = cap_bytes
        self.per_key = per_key
        self.idle: dict = {}
        self.bytes = 0
        # re-entrant: a garbage collection inside a locked section may run a
        # _Cached finaliser, which releases its state into this pool
        self.lock = threading.RLock()

    @staticmethod
    def _size(n, precision):
        return (16 if precision == "c128" else 8) << n

    def acquire(self, n: int, precision: str, device: int) -> DeviceState:
        key = (n, "c128" if _prec_code(precision) == _lib.SVB_C128 else "c64", device)
        with self.lock:
            lst = self.idle.get(key)
            if lst:
                self.bytes -= self._size(n, key[1])
                return lst.pop()
        return DeviceState(n, precision, device)  # (an out-of-memory create empties this pool and retries)

    def release(self, st: DeviceState) -> None:
        key = (st.n, st.precision, st.device)
        size = self._size(st.n, st.precision)
        evicted = []
        with self.lock:
            lst = self.idle.setdefault(key, [])
            if len(lst) < self.per_key and size <= self.cap:
                # oldest releases first (dicts keep insertion order; each key's
                # list is LIFO, so its front is its oldest)
                for k in list(self.idle):
                    while self.bytes + size > self.cap and self.idle[k]:
                        evicted.append(self.idle[k].pop(0))
                        self.bytes -= self._size(k[0], k[1])
                    if not self.idle[k] and k != key:
                        del self.idle[k]
                lst.append(st)
                self.bytes += size
                st = None
        for e in evicted:
            e.close()
        if st is not None:
            st.close()

    def clear(self) -> None:
        with self.lock:
            idle, self.idle, self.bytes = self.idle, {}, 0
        for lst in idle.values():
            for st in lst:
                st.close()


_pool = _StatePool()


# zero_state() arrays: complex128 states in CUDA managed memory, each with a
# view handle, so the kernel-level calls on them run in place on the device
# (no host<->device copy per call; pages stay in HBM while only kernels touch
# them).  address -> (n, view DeviceState)
_views: dict = {}


def _release_managed(address: int) -> None:
    entry = _views.pop(address, None)
    if entry is not None:
        entry[1].close()
    try:
        lib().svb_managed_free(_lib.c_void_p(address))
    except Exception:
        pass


def _managed_state(n: int, device: int = 0) -> np.ndarray:
    import ctypes as _ct
    import weakref as _wr

    p = _lib.c_void_p()
    check(lib().svb_managed_alloc(16 << n, device, _ct.byref(p)))
    raw = (_ct.c_double * (2 << n)).from_address(p.value)
    view = DeviceState._view(n, p.value, device)
    _views[p.value] = (n, view)
    _wr.finalize(raw, _release_managed, p.value)
    view.zero()
    return np.frombuffer(raw, dtype=np.complex128)


def _device_of(amps, n):
    """Kernel-level API operand -> (DeviceState, temporary?).  A DeviceState is
    used as is; a zero_state() array (managed memory) through its view, in
    place; any other complex128 ndarray through a temporary device copy."""
    if isinstance(amps, DeviceState):
        return amps, False
    if not isinstance(amps, np.ndarray) or amps.dtype != np.complex128:
        raise TypeError("amps must be a complex128 ndarray or a DeviceState")
    if amps.size != 1 << n:
        raise ValueError("amplitude vector length does not match n")
    if amps.flags.c_contiguous:
        entry = _views.get(amps.ctypes.data)
        if entry is not None and entry[0] == n:
            return entry[1], False
    return DeviceState.from_numpy(amps), True


def _write_back(dev: DeviceState, amps) -> None:
    if isinstance(amps, np.ndarray):
        if amps.flags.c_contiguous:
            dev.to_numpy(out=amps.reshape(-1))
        else:
            amps[...] = dev.to_numpy().reshape(amps.shape)
        dev.close()


# ------------------------------------------------------- kernel-level API
def zero_state(n: int) -> np.ndarray:
    """statevector.py:125-128: |0...0> as a complex128 ndarray.  The array
    lives in CUDA managed memory, so apply_1q / apply_2q / apply_instruction /
    marginal_probs / _measure_qubit on it run in place on the device."""
    return _managed_state(int(n))


def apply_1q(amps, n: int, q: int, m) -> None:
    dev, tmp = _device_of(amps, n)
    dev.apply_gates(_single_gate((q,), m))
    if tmp:
        _write_back(dev, amps)


def apply_2q(amps, n: int, qa: int, qb: int, m) -> None:
    dev, tmp = _device_of(amps, n)
    dev.apply_gates(_single_gate((qa, qb), m))
    if tmp:
        _write_back(dev, amps)


def apply_instruction(amps, n: int, inst) -> None:
    if inst.kind == "barrier":
        return
    dev, tmp = _device_of(amps, n)
    dev.apply_gates(gate_array([inst]))
    if tmp:
        _write_back(dev, amps)


def marginal_probs(amps, n: int, qubits) -> np.ndarray:
    dev, tmp = _device_of(amps, n)
    out = dev.marginal_probs(qubits)
    if tmp:
        dev.close()
    return out


def _measure_qubit(amps, n: int, q: int, rng: np.random.Generator) -> int:
    """statevector.py:142-149: one draw of ``rng`` (its PCG64 state is used on
    the device and then advanced by one, exactly as rng.random())."""
    dev, tmp = _device_of(amps, n)
    dev.seed_rng(pcg_words(rng))
    out = dev.measure(q)
    rng.bit_generator.advance(1)
    if tmp:
        _write_back(dev, amps)
    return out


def _reset_qubit(amps, n: int, q: int, rng: np.random.Generator) -> None:
    dev, tmp = _device_of(amps, n)
    dev.seed_rng(pcg_words(rng))
    dev.reset(q)
    rng.bit_generator.advance(1)
    if tmp:
        _write_back(dev, amps)


# ------------------------------------------------------------ backend API
def _sampler_code(sampler: str, k: int) -> int:
    if sampler == "alias":
        return _lib.SAMPLER_ALIAS
    if sampler == "cdf":
        return _lib.SAMPLER_CDF
    if sampler == "auto":
        return _lib.SAMPLER_ALIAS if k <= ALIAS_MAX_QUBITS else _lib.SAMPLER_CDF
    raise ValueError(f"unknown sampler {sampler!r}")


def run(
    c,
    shots: int,
    seed: int,
    workers: int = 1,
    qubit_cap: int = DEFAULT_QUBIT_CAP,
    *,
    precision: str = "c128",
    sampler: str = "auto",
    device: int = 0,
) -> RunResult:
    """statevector.py:182-253 on the GPU.  Terminal circuits: one gate program,
    one device sampling call.  Mid-circuit circuits: device-side replay of the
    suffix per shot with the PCG64 stream on the device; worker w of
    ``workers`` uses stream seed+w exactly as the reference fan-out."""
    if c.n_qubits > qubit_cap:
        raise QubitCapError(f"{c.n_qubits} qubits exceeds the configured cap {qubit_cap}")
    if shots < 1:
        raise ValueError("shots must be positive")
    measures = measurement_map(c)
    if not measures:
        raise NoMeasurementsError("circuit has no measurements")
    start = time.perf_counter()
    n = c.n_qubits
    meta: dict = {"engine": "libsvb", "precision": precision}
    if terminal_measurement_only(c):
        codes, freq, width, m2 = _terminal_codes(c, shots, seed, precision, sampler, device, measures)
        meta.update(m2)
        counts = format_counts(codes, freq, width)
    else:
        counts = _run_replay(c, shots, seed, workers, precision, device, meta)
    wall = time.perf_counter() - start
    res = RunResult(counts=counts, shots=shots, backend="sv", seed=seed, wall_time=wall)
    res.metadata.update(meta)
    return res


@dataclass
class CodeCounts:
    """Counts as parallel arrays: output code ``codes[i]``
    (bit p = clbit rank p, the lowest measured clbit at bit 0) was seen
    ``counts[i]`` times; ``width`` output bits.  Skips the per-outcome dict the
    reference builds (`result.py:80-82`, ~1.3 s per 10^6 distinct outcomes);
    ``to_dict()`` formats it exactly like ``run(...).counts``."""

    codes: np.ndarray
    counts: np.ndarray
    width: int

    def __len__(self) -> int:
        return int(self.codes.size)

    def to_dict(self) -> dict:
        return format_counts(self.codes, self.counts, self.width)


def run_codes(
    c,
    shots: int,
    seed: int,
    workers: int = 1,
    qubit_cap: int = DEFAULT_QUBIT_CAP,
    *,
    precision: str = "c128",
    sampler: str = "auto",
    device: int = 0,
) -> CodeCounts:
    """``run`` returning (code, count) arrays instead of a bitstring dict; same
    validation, stream and results (``run_codes(...).to_dict() == run(...).counts``)."""
    if c.n_qubits > qubit_cap:
        raise QubitCapError(f"{c.n_qubits} qubits exceeds the configured cap {qubit_cap}")
    if shots < 1:
        raise ValueError("shots must be positive")
    measures = measurement_map(c)
    if not measures:
        raise NoMeasurementsError("circuit has no measurements")
    if not terminal_measurement_only(c):
        counts = _run_replay(c, shots, seed, workers, precision, device, {})
        width = len(next(iter(counts)))
        codes = np.array([int(k, 2) for k in counts], dtype=np.uint64)
        freq = np.array(list(counts.values()), dtype=np.int64)
        order = np.argsort(codes)
        return CodeCounts(codes[order], freq[order], width)
    codes, freq, width, _ = _terminal_codes(c, shots, seed, precision, sampler, device, measures)
    return CodeCounts(codes, freq, width)


def _terminal_codes(c, shots, seed, precision, sampler, device, measures):
    n = c.n_qubits
    state = _pool.acquire(n, precision, device)
    try:
        state.zero()
        state.apply_instructions(c.instructions)
        meta = state.stats()
        qubits = sorted({q for q, _ in measures})
        src = output_bit_sources(measures, qubits)
        mode = _sampler_code(sampler, len(qubits))
        meta["sampler"] = "alias" if mode == _lib.SAMPLER_ALIAS else "cdf"
        codes, freq = state.sample_codes(qubits, src, shots, pcg_words(seed), mode)
    finally:
        _pool.release(state)
    return codes, freq, len(src), meta


def _run_replay(c, shots, seed, workers, precision, device, meta) -> dict:
    insts = c.instructions
    split = next(i for i, x in enumerate(insts) if x.kind in ("measure", "reset"))
    n = c.n_qubits
    prefix = _pool.acquire(n, precision, device)
    work = _pool.acquire(n, precision, device)
    try:
        prefix.zero()
        prefix.apply_instructions(insts[:split])
        suffix = [x for x in insts[split:] if x.kind != "barrier"]
        clbits = clbit_order([(x.qubits[0], x.clbit) for x in suffix if x.kind == "measure"])
        if len(clbits) > 64:
            # the device packs one shot's clbits into a uint64 code
            raise BackendError(f"mid-circuit replay supports at most 64 measured clbits, got {len(clbits)}")
        rank = np.full(max(clbits) + 1, -1, dtype=np.int32)
        for p, cl in enumerate(clbits):
            rank[cl] = p
        gates = gate_array([x for x in suffix if x.kind in UNITARY_GATES])
        ops = np.zeros((len(suffix), 3), dtype=np.int32)
        g = 0
        for j, x in enumerate(suffix):
            if x.kind == "measure":
                ops[j] = (1, x.qubits[0], x.clbit)
            elif x.kind == "reset":
                ops[j] = (2, x.qubits[0], 0)
            else:
                ops[j] = (0, g, 0)
                g += 1
        workers = max(1, min(workers, shots))
        sizes = [shots // workers + (1 if w < shots % workers else 0) for w in range(workers)]
        small = n <= (12 if prefix.precision == "c128" else 13)
        if small:  # all shots in one shared-memory launch; host copy of the prefix (<= 64 KB)
            pre = prefix.to_numpy()
            ops_r = ops.copy()
            meas = ops_r[:, 0] == 1
            ops_r[meas, 2] = rank[ops_r[meas, 2]]
        all_codes = []
        for w, size in enumerate(sizes):
            if size == 0:
                continue
            codes = np.empty(size, dtype=np.uint64)
            words = pcg_words(seed + w)
            if small:
                check(lib().svb_replay_small(
                    device, _prec_code(prefix.precision), n, ptr(pre), ptr(ops_r, _lib.c_int32), int(len(suffix)),
                    ptr(gates) if gates.size else None, int(gates.size), int(size), ptr(words, _lib.c_uint64),
                    ptr(codes, _lib.c_uint64)))
            else:
                check(
                    lib().svb_replay(
                        work.handle, prefix.handle, ptr(ops, _lib.c_int32), int(len(suffix)),
                        ptr(gates) if gates.size else None, ptr(rank, _lib.c_int32), int(size),
                        ptr(words, _lib.c_uint64), ptr(codes, _lib.c_uint64),
                    )
                )
            all_codes.append(codes)
        meta["replay_shots"] = shots
        meta["replay_engine"] = "smem-batched" if small else "per-shot"

    finally:
        _pool.release(prefix)
        _pool.release(work)
    codes, freq = np.unique(np.concatenate(all_codes), return_counts=True)
    return format_counts(codes, freq, len(clbits))


class _Cached:
    """A cached post-unitary state; when its Circuit is collected the device
    state goes back to the pool (a 16 GiB cudaMalloc + cudaFree per new
    circuit cost more than the QFT-30 program itself)."""
    __slots__ = ("device", "host", "__weakref__")

    def __init__(self, device: DeviceState):
        self.device = device
        self.host = None

    def __del__(self):
        d, self.device = getattr(self, "device", None), None
        if d is not None:
            try:
                _pool.release(d)
            except Exception:
                pass

    def serves(self, precision: str, device: int) -> bool:
        return self.device.precision == _norm_prec(precision) and self.device.device == device


def _norm_prec(precision) -> str:
    return "c128" if _prec_code(precision) == _lib.SVB_C128 else "c64"


_state_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _cached_state(c, qubit_cap: int, precision: str = "c128", device: int = 0) -> _Cached:
    """The cached post-unitary state of `c` (statevector.py:256-274), keyed by
    the Circuit; an entry of another precision or device is recomputed."""
    entry = _state_cache.get(c)
    if entry is not None and entry.serves(precision, device):
        return entry
    if c.n_qubits > qubit_cap:
        raise QubitCapError(f"{c.n_qubits} qubits exceeds the configured cap {qubit_cap}")
    if not terminal_measurement_only(c):
        raise BackendError("expectation values need a circuit without mid-circuit collapse")
    state = _pool.acquire(c.n_qubits, precision, device).zero()
    state.apply_instructions(c.instructions)
    entry = _Cached(state)
    _state_cache[c] = entry
    return entry


def final_state(c, qubit_cap: int = DEFAULT_QUBIT_CAP, *, out: np.ndarray | None = None,
                precision: str = "c128", device: int = 0) -> np.ndarray:
    """statevector.py:259-274: the post-unitary state, cached per Circuit object.
    ``out`` (optional) receives the amplitudes (e.g. a pinned buffer)."""
    entry = _cached_state(c, qubit_cap, precision, device)
    if out is not None:
        return entry.device.to_numpy(out)
    if entry.host is None:
        entry.host = entry.device.to_numpy()
    return entry.host


def _z_mask(c, z_qubits) -> int:
    z = tuple(z_qubits)
    for q in z:
        if not 0 <= q < c.n_qubits:
            raise ValueError(f"qubit {q} out of range")
    return sum(1 << q for q in set(z))


def expectation(c, z_qubits, qubit_cap: int = DEFAULT_QUBIT_CAP) -> float:
    """statevector.py:277-292: <Z..Z> from one device pass over the cached state."""
    mask = _z_mask(c, z_qubits)
    entry = _cached_state(c, qubit_cap)
    return float(entry.device.expect_z([mask])[0])


def expectations(c, z_sets, qubit_cap: int = DEFAULT_QUBIT_CAP) -> np.ndarray:
    """Many <Z..Z> observables in one pass over the state (extension).  When
    the state is not cached yet and every observable is a single-qubit Z, the
    sums are taken by the program's last fused pass (no extra read pass); the
    state is cached as by final_state."""
    masks = [_z_mask(c, z) for z in z_sets]
    cached = _state_cache.get(c)
    if (cached is None or not cached.serves("c128", 0)) and masks and all(m and (m & (m - 1)) == 0 for m in masks):
        if c.n_qubits > qubit_cap:
            raise QubitCapError(f"{c.n_qubits} qubits exceeds the configured cap {qubit_cap}")
        if not terminal_measurement_only(c):
            raise BackendError("expectation values need a circuit without mid-circuit collapse")
        state = _pool.acquire(c.n_qubits, "c128", 0).zero()
        qs = [m.bit_length() - 1 for m in masks]
        vals = state.apply_gates_z(gate_array(c.instructions), qs)
        _state_cache[c] = _Cached(state)
        return vals
    entry = _cached_state(c, qubit_cap)
    return entry.device.expect_z(masks)


def plan(n: int, instructions, precision: str = "c128", zero_start: bool = False) -> dict:
    """Host-only schedule summary of a gate program (no GPU needed).
    zero_start: schedule for a lazy |0...0> input (free initial qubit layout)."""
    arr = gate_array(instructions)
    p, r, b = _lib.c_int64(), _lib.c_int64(), _lib.c_int64()
    perm = _lib.c_int32()
    check(lib().svb_plan(n, _prec_code(precision) | (0x100 if zero_start else 0), ptr(arr), int(arr.size), _lib.ctypes.byref(p),
                         _lib.ctypes.byref(r), _lib.ctypes.byref(b), _lib.ctypes.byref(perm)))
    return {"passes": p.value, "rounds": r.value, "op_bytes": b.value, "permute": bool(perm.value),
            "permute_fused": perm.value == 2, "permute_initial": perm.value in (3, 4),
            "permute_initial_fused": perm.value == 4, "gates": int(arr.size)}


__all__ = [
    "DEFAULT_QUBIT_CAP", "DeviceState", "run", "run_codes", "CodeCounts", "final_state", "expectation", "expectations",
    "zero_state", "apply_1q", "apply_2q", "apply_instruction", "marginal_probs",
    "_measure_qubit", "_reset_qubit", "plan", "gate_array", "gate_array_many", "gate_ops_many", "pcg_words",
    "ONE_QUBIT_GATES", "single_qubit_matrix",
]
