"""Batched execution of many circuits (config 4; reference `batch.run_batch`,
batch.py:104-222, which runs `run_circuit(c, "sv", shots, seed)` per circuit
sequentially with the same seed for every circuit).

* Terminal circuits whose state fits in shared memory (n <= 12 complex128,
  n <= 13 complex64) run together in ONE persistent kernel launch
  (`svb_batch_small`): one CTA per SM walks the batch, state in shared memory,
  CDF sampling from the circuit's own PCG64 stream.
* Everything else runs through the fused-pass engine (`statevector.run`) on
  pooled device states, `workers` circuits in flight (the C calls release the
  GIL, so host preparation of one circuit overlaps device work of others).

Results come back in input order: a RunResult per circuit, or the exception
the circuit raised (the reference records per-circuit errors, batch.py:192-194).
"""
from __future__ import annotations

import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from . import statevector as sv
from .features import terminal_measurement_only
from .result import NoMeasurementsError, QubitCapError, RunResult, format_counts, measurement_map, output_bit_sources

SMALL_MAX = {"c128": 12, "c64": 13}
_lock = threading.Lock()


def _small_batch(circuits, shots, seed, precision, device):
    """One svb_batch_small launch for terminal circuits that fit in smem."""
    nc = len(circuits)
    encs = [sv.gate_array(c.instructions) for c in circuits]
    ngates = np.array([e.size for e in encs], dtype=np.int32)
    gate_off = np.zeros(nc, dtype=np.int32)
    if nc > 1:
        gate_off[1:] = np.cumsum(ngates)[:-1]
    gates = np.concatenate(encs) if encs else np.zeros(0, dtype=_lib.GATE_DTYPE)
    nq = np.array([c.n_qubits for c in circuits], dtype=np.int32)
    words = sv.pcg_words(seed)
    pcg = np.tile(words, nc).astype(np.uint64)
    w = np.zeros(nc, dtype=np.int32)
    bit_src = np.zeros((nc, 64), dtype=np.int8)
    widths = []
    for i, c in enumerate(circuits):
        measures = measurement_map(c)
        qubits = sorted({q for q, _ in measures})
        src = output_bit_sources(measures, qubits)
        w[i] = len(src)
        bit_src[i, : len(src)] = [qubits[j] for j in src]  # bits of the full index
        widths.append(len(src))
    codes = np.empty((nc, shots), dtype=np.uint64)
    prec = _lib.SVB_C128 if precision == "c128" else _lib.SVB_C64
    _lib.check(_lib.lib().svb_batch_small(
        device, prec, nc, _lib.ptr(nq, _lib.c_int32), _lib.ptr(gate_off, _lib.c_int32), _lib.ptr(ngates, _lib.c_int32),
        _lib.ptr(gates) if gates.size else None, int(gates.size), _lib.ptr(pcg, _lib.c_uint64),
        _lib.ptr(w, _lib.c_int32), _lib.ptr(bit_src, _lib.ctypes.c_int8), int(shots), _lib.ptr(codes, _lib.c_uint64)))
    codes.sort(axis=1)
    out = []
    for i in range(nc):
        row = codes[i]
        starts = np.flatnonzero(np.concatenate(([True], row[1:] != row[:-1])))
        freq = np.diff(np.concatenate((starts, [row.size])))
        out.append(format_counts(row[starts], freq, widths[i]))
    return out


def run_batch(circuits, shots: int = 1000, seed: int = 0, *, precision: str = "c128", sampler: str = "cdf",
              device: int = 0, workers: int = 8, qubit_cap: int = sv.DEFAULT_QUBIT_CAP):
    """Run every circuit with (shots, seed); returns a list of RunResult or
    exception objects, in input order.  Default sampler: the device CDF
    sampler (throughput); sampler="alias" keeps the reference's exact alias
    sampler for every circuit (no shared-memory batching)."""
    results: list = [None] * len(circuits)
    small, large = [], []
    for i, c in enumerate(circuits):
        if c.n_qubits > qubit_cap:
            results[i] = QubitCapError(f"{c.n_qubits} qubits exceeds the configured cap {qubit_cap}")
        elif shots < 1:
            results[i] = ValueError("shots must be positive")
        elif not measurement_map(c):
            results[i] = NoMeasurementsError("circuit has no measurements")
        elif (sampler != "alias" and terminal_measurement_only(c)
              and c.n_qubits <= SMALL_MAX[precision] and c.n_qubits >= 1):
            small.append(i)
        else:
            large.append(i)
    if small:
        t0 = time.perf_counter()
        counts = _small_batch([circuits[i] for i in small], shots, seed, precision, device)
        dt = (time.perf_counter() - t0) / len(small)
        for i, cnt in zip(small, counts):
            r = RunResult(counts=cnt, shots=shots, backend="sv", seed=seed, wall_time=dt)
            r.metadata.update({"engine": "libsvb-batch-smem", "precision": precision, "sampler": "cdf"})
            results[i] = r

    def one(i):
        try:
            return sv.run(circuits[i], shots, seed, qubit_cap=qubit_cap, precision=precision,
                          sampler=sampler, device=device)
        except Exception as exc:  # recorded per circuit, like the reference
            return exc

    if large:
        if workers <= 1:
            for i in large:
                results[i] = one(i)
        else:
            with ThreadPoolExecutor(max_workers=workers) as pool:
                for i, r in zip(large, pool.map(one, large)):
                    results[i] = r
    return results
