"""Partitioned-block simulation with device-resident blocks.

Mirrors the reference's `polysim/pblock.py` (terminal and replay paths of
`run`, `PBlockState`, `reorder_qubits`): every qubit starts as its own 1-qubit
state; a 2-qubit gate merges the two owning blocks (tensor product, qubit list
re-sorted, amplitudes permuted), and measuring a qubit projects its block and
factors the qubit back out.  Here every block is a `DeviceState` in HBM:

* merge        -> `svb_outer` (np.multiply.outer(b, a), pblock.py:76-83) and
                  `svb_permute_qubits` (reorder_qubits, pblock.py:34-43);
* gates        -> queued per block and applied as one fused `svb_apply`
                  program when the block is next read or merged;
* measure      -> the device `_measure_qubit` (one draw of the shot's rng,
                  statevector.py:142-149) and `svb_select_half` for the kept
                  half (pblock.py:111-121);
* marginals    -> `svb_marginal_probs`; terminal draws -> `svb_alias_draw`
                  per group with the shared PCG64 stream (result.py:50-82).

Results equal the reference's pblock on the same seeds (up to floating-point
rounding of the block amplitudes; counts are tested against fixtures made by
the real reference, tests/golden/make_golden_pblock.py).  The distributed
(vQPU telegate) variant is out of scope here: it is a protocol over these same
block operations.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import statevector as sv
from .circuit import Instruction
from .features import terminal_measurement_only
from .result import (
    BackendError,
    NoMeasurementsError,
    RunResult,
    clbit_order,
    format_counts,
    measurement_map,
    pack_bitstring,
)


# idle block states for reuse (blocks are created and dropped at every merge /
# measurement; pooling avoids a cudaMalloc + stream per block)
_blocks = sv._StatePool(cap_bytes=1 << 30, per_key=64)


def reorder_qubits(state: np.ndarray, current: list[int], target: list[int]) -> np.ndarray:
    """Host version of pblock.py:34-43 (used by `contract`, validation only)."""
    m = len(current)
    pos_of = {q: p for p, q in enumerate(current)}
    perm = [m - 1 - pos_of[target[m - 1 - axis]] for axis in range(m)]
    return state.reshape([2] * m).transpose(perm).reshape(-1)


@dataclass
class Block:
    qubits: list[int]  # ascending global indices; position 0 is the local LSB
    dev: sv.DeviceState  # the block's amplitudes in HBM
    pending: list = field(default_factory=list)  # queued local gate records

    @property
    def dim(self) -> int:
        return 1 << len(self.qubits)

    def flush(self) -> None:
        if self.pending:
            self.dev.apply_gates(np.concatenate(self.pending))
            self.pending.clear()

    @property
    def state(self) -> np.ndarray:
        """Host copy of the amplitudes (the reference's `Block.state` array,
        pblock.py:46-51), after the queued gates are applied."""
        self.flush()
        return self.dev.to_numpy()

    @state.setter
    def state(self, amps) -> None:
        amps = np.ascontiguousarray(amps, dtype=np.complex128).reshape(-1)
        self.pending.clear()
        if amps.size != 1 << self.dev.n:
            n = amps.size.bit_length() - 1
            prec, device = self.dev.precision, self.dev.device
            _blocks.release(self.dev)
            self.dev = _blocks.acquire(n, prec, device)
        self.dev.load(amps)


class PBlockState:
    """pblock.py:54-157 with device blocks."""

    def __init__(self, n: int, precision: str = "c128", device: int = 0):
        self.n = n
        self.precision = precision
        self.device = device
        self.block_of: dict[int, Block] = {}
        for q in range(n):
            self.block_of[q] = Block([q], self._basis(0))

    def _basis(self, bit: int) -> sv.DeviceState:
        s = _blocks.acquire(1, self.precision, self.device)
        s.load(np.array([1.0 - bit, bit], dtype=np.complex128))
        return s

    def blocks(self) -> list[Block]:
        seen: list[Block] = []
        for q in range(self.n):
            b = self.block_of[q]
            if all(b is not s for s in seen):
                seen.append(b)
        return seen

    def max_dim(self) -> int:
        return max(b.dim for b in self.blocks())

    def _merge(self, a: Block, b: Block) -> Block:
        a.flush()
        b.flush()
        combined = a.qubits + b.qubits
        target = sorted(combined)
        st = _blocks.acquire(len(combined), self.precision, self.device)
        _lib.check(_lib.lib().svb_outer(st.handle, a.dev.handle, b.dev.handle))
        dest = np.array([target.index(q) for q in combined], dtype=np.int32)
        _lib.check(_lib.lib().svb_permute_qubits(st.handle, _lib.ptr(dest, _lib.c_int32)))
        _blocks.release(a.dev)
        _blocks.release(b.dev)
        merged = Block(target, st)
        for q in target:
            self.block_of[q] = merged
        return merged

    def apply(self, inst: Instruction) -> None:
        if inst.kind == "barrier":
            return
        if len(inst.qubits) == 1:
            block = self.block_of[inst.qubits[0]]
            local = (block.qubits.index(inst.qubits[0]),)
        else:
            qa, qb = inst.qubits
            block = self.block_of[qa]
            other = self.block_of[qb]
            if block is not other:
                block = self._merge(block, other)
            local = (block.qubits.index(qa), block.qubits.index(qb))
        block.pending.append(sv.gate_array([Instruction(inst.kind, local, inst.params)]))

    def measure_and_factor(self, qubit: int, rng: np.random.Generator) -> int:
        block = self.block_of[qubit]
        block.flush()
        n_local = len(block.qubits)
        pos = block.qubits.index(qubit)
        bit = sv._measure_qubit(block.dev, n_local, pos, rng)
        if n_local > 1:
            kept = _blocks.acquire(n_local - 1, self.precision, self.device)
            _lib.check(_lib.lib().svb_select_half(kept.handle, block.dev.handle, pos, bit))
            rest = Block([q for q in block.qubits if q != qubit], kept)
            for q in rest.qubits:
                self.block_of[q] = rest
        _blocks.release(block.dev)
        self.block_of[qubit] = Block([qubit], self._basis(bit))
        return bit

    def reset(self, qubit: int, rng: np.random.Generator) -> None:
        self.measure_and_factor(qubit, rng)
        _blocks.release(self.block_of[qubit].dev)
        self.block_of[qubit] = Block([qubit], self._basis(0))

    def set_basis(self, qubit: int, bit: int) -> None:
        block = self.block_of[qubit]
        if len(block.qubits) != 1:
            raise BackendError("can only set basis state on a factored qubit")
        block.pending.clear()
        _blocks.release(block.dev)
        block.dev = self._basis(bit)

    def contract(self) -> np.ndarray:
        """Global little-endian amplitudes (host; validation at small n)."""
        order: list[int] = []
        vec = np.ones(1, dtype=complex)
        for block in self.blocks():
            block.flush()
            vec = np.multiply.outer(block.dev.to_numpy(), vec).reshape(-1)
            order = order + block.qubits
        return reorder_qubits(vec, order, sorted(order))

    def close(self) -> None:
        for b in self.blocks():
            _blocks.release(b.dev)


def _measured_groups(state: PBlockState, measured: set[int]):
    """pblock.py:160-171: per block, the marginal over its measured qubits."""
    groups = []
    for block in state.blocks():
        qs = tuple(q for q in block.qubits if q in measured)
        if not qs:
            continue
        block.flush()
        probs = block.dev.marginal_probs([block.qubits.index(q) for q in qs])
        groups.append((qs, probs))
    groups.sort(key=lambda g: g[0][0])
    return groups


def sample_measurement_groups(groups, measures, shots: int, rng: np.random.Generator) -> dict:
    """result.py:50-82 with the alias build and draws on the device: group g
    consumes the next `shots` uniforms of the shared stream."""
    if not measures:
        raise NoMeasurementsError("circuit has no measurements")
    qubit_bits: dict[int, np.ndarray] = {}
    for qubits, probs in groups:
        p = np.ascontiguousarray(probs, dtype=np.float64)
        idx = np.empty(shots, dtype=np.uint64)
        words = np.ascontiguousarray(sv.pcg_words(rng), dtype=np.uint64)
        _lib.check(_lib.lib().svb_alias_draw(0, _lib.ptr(p, _lib.c_double), int(p.size), int(shots),
                                             _lib.ptr(words, _lib.c_uint64), _lib.ptr(idx, _lib.c_uint64)))
        rng.bit_generator.advance(shots)
        for j, q in enumerate(qubits):
            qubit_bits[q] = ((idx >> np.uint64(j)) & np.uint64(1)).astype(np.int64)
    latest: dict[int, int] = {}
    for qubit, clbit in measures:
        latest[clbit] = qubit
    clbits = sorted(latest)
    if len(clbits) > 63:
        raise BackendError("more than 63 measured clbits")
    codes = np.zeros(shots, dtype=np.int64)
    for pos, cl in enumerate(clbits):
        codes |= qubit_bits[latest[cl]] << pos
    values, freq = np.unique(codes, return_counts=True)
    return format_counts(values, freq, len(clbits))


def run(c, shots: int, seed: int, workers: int = 1, *, precision: str = "c128", device: int = 0) -> RunResult:
    """pblock.py:174-207 (`workers` is accepted; shots replay sequentially)."""
    if shots < 1:
        raise ValueError("shots must be positive")
    measures = measurement_map(c)
    if not measures:
        raise NoMeasurementsError("circuit has no measurements")
    start = time.perf_counter()
    trace: list[int] = []
    if terminal_measurement_only(c):
        state = PBlockState(c.n_qubits, precision, device)
        try:
            for inst in c.instructions:
                if inst.is_unitary:
                    state.apply(inst)
                    trace.append(state.max_dim())
            groups = _measured_groups(state, {q for q, _ in measures})
        finally:
            state.close()
        counts = sample_measurement_groups(groups, measures, shots, np.random.default_rng(seed))
    else:
        counts = {}
        clbits = clbit_order(measures)
        for s in range(shots):  # pblock.py:210-246: shot s uses default_rng([seed, s])
            rng = np.random.default_rng([seed, s])
            state = PBlockState(c.n_qubits, precision, device)
            values: dict[int, int] = {}
            try:
                for inst in c.instructions:
                    if inst.kind == "measure":
                        values[inst.clbit] = state.measure_and_factor(inst.qubits[0], rng)
                    elif inst.kind == "reset":
                        state.reset(inst.qubits[0], rng)
                    elif inst.is_unitary:
                        state.apply(inst)
                    if s == 0:
                        trace.append(state.max_dim())
            finally:
                state.close()
            key = pack_bitstring(values, clbits)
            counts[key] = counts.get(key, 0) + 1
    wall = time.perf_counter() - start
    return RunResult(counts=counts, shots=shots, backend="pblock", seed=seed, wall_time=wall,
                     metadata={"max_block_dim": max(trace) if trace else 2, "block_dim_trace": trace,
                               "engine": "libsvb"})


__all__ = ["PBlockState", "Block", "reorder_qubits", "sample_measurement_groups", "run"]
