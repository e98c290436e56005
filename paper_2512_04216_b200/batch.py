"""Batched execution of many circuits (config 4; reference `batch.run_batch`,
batch.py:104-222, which runs `run_circuit(c, "sv", shots, seed)` per circuit
sequentially with the same seed for every circuit).

* Terminal circuits whose state fits in shared memory (n <= 12 complex128,
  n <= 13 complex64) run together in ONE persistent kernel launch
  (`svb_batch_small`): one CTA per SM walks the batch, state in shared memory,
  CDF sampling from the circuit's own PCG64 stream.
* Larger terminal circuits go to `svb_batch_run` in chunks: one C call per
  chunk, host worker threads with their own streams schedule and launch each
  circuit's fused program and CDF draw with no per-circuit synchronisation;
  gates travel as compact 40-byte records expanded in C++.
* Mid-circuit circuits (and sampler="alias") run one by one through
  `statevector.run` (device replay / the reference-exact alias sampler).

Results come back in input order: a RunResult per circuit, or the exception
the circuit raised (the reference records per-circuit errors, batch.py:192-194).
"""
from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from . import statevector as sv
from .features import terminal_measurement_only
from .result import NoMeasurementsError, QubitCapError, RunResult, format_counts, measurement_map, output_bit_sources

SMALL_MAX = {"c128": 12, "c64": 13}


def _bit_sources(c):
    """(width, state-index bit of each output bit) of a terminal circuit."""
    measures = measurement_map(c)
    qubits = sorted({q for q, _ in measures})
    src = output_bit_sources(measures, qubits)
    return len(src), [qubits[j] for j in src]


def _codes_small(circuits, shots, words, precision, device) -> np.ndarray:
    """One svb_batch_small launch: (ncirc, shots) codes."""
    nc = len(circuits)
    gates, ngates = sv.gate_array_many(circuits)
    gate_off = np.zeros(nc, dtype=np.int32)
    if nc > 1:
        gate_off[1:] = np.cumsum(ngates)[:-1]
    nq = np.array([c.n_qubits for c in circuits], dtype=np.int32)
    pcg = np.tile(words, nc).astype(np.uint64)
    w = np.zeros(nc, dtype=np.int32)
    bit_src = np.zeros((nc, 64), dtype=np.int8)
    for i, c in enumerate(circuits):
        w[i], bits = _bit_sources(c)
        bit_src[i, : w[i]] = bits
    codes = np.empty((nc, shots), dtype=np.uint64)
    prec = _lib.SVB_C128 if precision == "c128" else _lib.SVB_C64
    _lib.check(_lib.lib().svb_batch_small(
        device, prec, nc, _lib.ptr(nq, _lib.c_int32), _lib.ptr(gate_off, _lib.c_int32), _lib.ptr(ngates, _lib.c_int32),
        _lib.ptr(gates) if gates.size else None, int(gates.size), _lib.ptr(pcg, _lib.c_uint64),
        _lib.ptr(w, _lib.c_int32), _lib.ptr(bit_src, _lib.ctypes.c_int8), int(shots), _lib.ptr(codes, _lib.c_uint64)))
    return codes, w


class _Prepared:
    """Host encoding of one chunk of large circuits for svb_batch_run."""

    def __init__(self, circuits, words):
        nc = len(circuits)
        self.ops, self.ngates = sv.gate_ops_many(circuits)
        self.gate_off = np.zeros(nc, dtype=np.int32)
        if nc > 1:
            self.gate_off[1:] = np.cumsum(self.ngates)[:-1]
        self.nq = np.array([c.n_qubits for c in circuits], dtype=np.int32)
        self.pcg = np.tile(words, nc).astype(np.uint64)
        self.w = np.zeros(nc, dtype=np.int32)
        self.bit_src = np.zeros((nc, 64), dtype=np.int8)
        for i, c in enumerate(circuits):
            self.w[i], bits = _bit_sources(c)
            self.bit_src[i, : self.w[i]] = bits

    def run(self, shots, precision, device, nthreads, jit_mode):
        nc = self.nq.size
        codes = np.empty((nc, shots), dtype=np.uint64)
        status = np.zeros(nc, dtype=np.int32)
        fx = sv.fixed_gate_table()
        prec = _lib.SVB_C128 if precision == "c128" else _lib.SVB_C64
        _lib.check(_lib.lib().svb_batch_run(
            device, prec, nc, _lib.ptr(self.nq, _lib.c_int32), _lib.ptr(self.gate_off, _lib.c_int32),
            _lib.ptr(self.ngates, _lib.c_int32), _lib.ptr(self.ops) if self.ops.size else None, _lib.ptr(fx),
            int(fx.size), int(self.ops.size), _lib.ptr(self.pcg, _lib.c_uint64), _lib.ptr(self.w, _lib.c_int32),
            _lib.ptr(self.bit_src, _lib.ctypes.c_int8), int(shots), int(nthreads), int(jit_mode),
            _lib.ptr(codes, _lib.c_uint64),
            _lib.ptr(status, _lib.c_int32)))
        return codes, status


def _histograms(codes: np.ndarray, widths) -> list:
    """Row-wise (code, count) arrays of a (ncirc, shots) code matrix, like np.unique."""
    codes = np.sort(codes, axis=1)
    nc, shots = codes.shape
    new = np.ones(codes.shape, dtype=bool)
    new[:, 1:] = codes[:, 1:] != codes[:, :-1]
    out = []
    for i in range(nc):
        starts = np.flatnonzero(new[i])
        freq = np.diff(np.append(starts, shots)).astype(np.int64)
        out.append(sv.CodeCounts(codes[i, starts], freq, int(widths[i])))
    return out


def _status_error(code: int):
    msg = _lib.lib().svb_last_error().decode(errors="replace")
    if code == _lib.SVB_E_ARG:
        return ValueError(msg)
    if code == _lib.SVB_E_CAP:
        return QubitCapError(msg)
    from .result import BackendError

    return BackendError(f"libsvb error {code}: {msg}")


_JIT_MODES = {"none": 0, "sync": 1, "async": 2}
last_timing: dict = {}  # wall-clock breakdown of the last run_batch_codes call (seconds)


def _timed(fn, *args):
    t0 = time.perf_counter()
    r = fn(*args)
    return r, time.perf_counter() - t0


def run_batch_codes(circuits, shots: int = 1000, seed: int = 0, *, precision: str = "c128", device: int = 0,
                    nthreads: int = 8, qubit_cap: int = sv.DEFAULT_QUBIT_CAP, chunk: int = 2048,
                    jit: str = "none") -> list:
    """The device batch path: every terminal circuit runs with (shots, seed) and
    the CDF sampler; returns a CodeCounts (or the circuit's exception) per
    circuit in input order.  Small states: one shared-memory persistent
    kernel; the rest: two svb_batch_run calls (the `chunk` largest circuits,
    then the others, encoded while the first call runs: the C call releases
    the GIL).
    jit: "none" (default: interpreter kernels up to 24 qubits — no compile,
    reproducible, the fastest measured on streams of new circuits), "sync"
    (NVRTC-specialised passes from 24 qubits exactly as sv.run, so results
    equal sv.run's; a cold process pays one compile per circuit structure,
    cached on disk), "async" (compiled in the background while the
    interpreter serves; the engine of a circuit then depends on timing)."""
    from concurrent.futures import ThreadPoolExecutor as _TPE

    tm = last_timing
    tm.clear()
    t_start = time.perf_counter()
    results: list = [None] * len(circuits)
    small, large = [], []
    words = sv.pcg_words(seed)
    for i, c in enumerate(circuits):
        if c.n_qubits > qubit_cap:
            results[i] = QubitCapError(f"{c.n_qubits} qubits exceeds the configured cap {qubit_cap}")
        elif shots < 1:
            results[i] = ValueError("shots must be positive")
        elif not measurement_map(c):
            results[i] = NoMeasurementsError("circuit has no measurements")
        elif not terminal_measurement_only(c):
            results[i] = "replay"
        elif c.n_qubits <= SMALL_MAX[precision]:
            small.append(i)
        else:
            large.append(i)
    # largest circuits first across chunks (the GPU tail is then short)
    large.sort(key=lambda i: -circuits[i].n_qubits)
    tm["classify_s"] = time.perf_counter() - t_start
    # two C calls, one after the other (never concurrent: two calls would
    # double the workers contending for the device): the first `chunk`
    # largest circuits, then the rest, encoded while the first call runs;
    # the shared-memory batch of small circuits runs beside them
    bounds = [0] + ([chunk] if len(large) > chunk else []) + [len(large)]
    with _TPE(max_workers=1) as small_pool, _TPE(max_workers=1) as pool:
        fut_small = small_pool.submit(_timed, _codes_small, [circuits[i] for i in small], shots, words, precision,
                                      device) if small else None
        pending = []
        t0 = time.perf_counter()
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            if hi <= lo:
                continue
            idx = large[lo:hi]
            prep = _Prepared([circuits[i] for i in idx], words)
            pending.append((idx, prep.w, pool.submit(_timed, prep.run, shots, precision, device, nthreads,
                                                     _JIT_MODES[jit])))
        tm["encode_s"] = time.perf_counter() - t0
        tm["chunk_call_s"], tm["chunk_wait_s"], tm["hist_s"] = [], 0.0, 0.0
        for idx, w, fut in pending:
            t0 = time.perf_counter()
            (codes, status), dt = fut.result()
            t1 = time.perf_counter()
            tm["chunk_wait_s"] += t1 - t0
            tm["chunk_call_s"].append(dt)
            for i, cc, st in zip(idx, _histograms(codes, w), status.tolist()):
                results[i] = cc if st == 0 else _status_error(st)
            tm["hist_s"] += time.perf_counter() - t1
        if fut_small is not None:
            t0 = time.perf_counter()
            (codes, w), tm["small_call_s"] = fut_small.result()
            tm["small_wait_s"] = time.perf_counter() - t0
            for i, cc in zip(small, _histograms(codes, w)):
                results[i] = cc
    for i, r in enumerate(results):
        if isinstance(r, str):  # mid-circuit measurement: the replay engine, one circuit at a time
            try:
                res = sv.run_codes(circuits[i], shots, seed, qubit_cap=qubit_cap, precision=precision, device=device)
                results[i] = res
            except Exception as exc:
                results[i] = exc
    tm["total_s"] = time.perf_counter() - t_start
    return results


def run_batch(circuits, shots: int = 1000, seed: int = 0, *, precision: str = "c128", sampler: str = "cdf",
              device: int = 0, workers: int = 8, qubit_cap: int = sv.DEFAULT_QUBIT_CAP, jit: str = "none"):
    """Run every circuit with (shots, seed); returns a list of RunResult or
    exception objects, in input order (the reference records per-circuit
    errors, batch.py:192-194).  Default sampler: the device CDF sampler through
    run_batch_codes (counts dicts formatted at the end); sampler="alias" keeps
    the reference's exact alias sampler, one circuit at a time."""
    if sampler != "alias":
        t0 = time.perf_counter()
        raw = run_batch_codes(circuits, shots, seed, precision=precision, device=device, nthreads=workers,
                              qubit_cap=qubit_cap, jit=jit)
        dt = (time.perf_counter() - t0) / max(len(circuits), 1)
        out = []
        for r in raw:
            if isinstance(r, Exception):
                out.append(r)
                continue
            res = RunResult(counts=r.to_dict(), shots=shots, backend="sv", seed=seed, wall_time=dt)
            res.metadata.update({"engine": "libsvb-batch", "precision": precision, "sampler": "cdf"})
            out.append(res)
        return out

    def one(c):
        try:
            return sv.run(c, shots, seed, qubit_cap=qubit_cap, precision=precision, sampler=sampler, device=device)
        except Exception as exc:  # recorded per circuit, like the reference
            return exc

    if workers <= 1:
        return [one(c) for c in circuits]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(one, circuits))
