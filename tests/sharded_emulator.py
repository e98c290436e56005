"""CPU emulation of a shard for the multi-process gloo tests (TEST BACKEND:
not part of the product package, which has no CPU path).  Gates go through
libsvb's host emulator of the fused program (the same scheduler and op
interpreter as the device kernel); block pack/unpack, reductions and the
slice sampler are numpy restatements of the device kernels.  Passed to
ShardedState as `backend=EmulatedShard`."""
from __future__ import annotations

import numpy as np


class EmulatedShard:
    def __init__(self, nl: int, precision: str, device: int = 0):
        import torch

        from paper_2512_04216_b200 import _lib

        self._lib = _lib
        self.torch = torch
        self.nl = nl
        self.precision = precision
        self.itemsize = 16
        self.amps = np.zeros(1 << nl, dtype=np.complex128)
        self.writes = 0  # full-shard writes (lazy-zero accounting in the tests)

    def apply(self, gates: np.ndarray) -> None:
        if gates.size:
            L = self._lib
            L.check(L.lib().svb_emulate_apply(self.nl, 1 if self.precision == "c128" else 0, L.ptr(gates),
                                              int(gates.size), L.ptr(self.amps), 1))

    def set_zero_state(self) -> None:
        self.amps[:] = 0
        self.amps[0] = 1.0

    def clear(self) -> None:
        self.amps[:] = 0
        self.writes += 1

    def close(self) -> None:
        pass

    def buffer(self, amps: int):
        return self.torch.empty((amps * self.itemsize,), dtype=self.torch.uint8)

    def _block_idx(self, lbits, block, off, count):
        j = np.arange(off, off + count, dtype=np.int64)
        for L in lbits:  # ascending: insert a zero bit at each L
            j = ((j >> L) << (L + 1)) | (j & ((1 << L) - 1))
        for i, L in enumerate(lbits):
            j |= ((block >> i) & 1) << L
        return j

    def block_out(self, lbits, block, off, count, buf) -> None:
        v = self.amps[self._block_idx(lbits, block, off, count)]
        buf[: count * 16].copy_(self.torch.from_numpy(v.view(np.uint8).copy()))

    def block_in(self, lbits, block, off, count, buf) -> None:
        v = buf[: count * 16].numpy().view(np.complex128)
        self.amps[self._block_idx(lbits, block, off, count)] = v

    def expect(self, masks) -> np.ndarray:
        p = np.abs(self.amps) ** 2
        idx = np.arange(p.size, dtype=np.uint64)
        out = []
        for m in masks:
            par = (np.bitwise_count(idx & np.uint64(m)) & np.uint64(1)).astype(float)
            out.append(float(np.sum(p * (1.0 - 2.0 * par))))
        return np.array(out)

    def apply_z(self, gates: np.ndarray, qubits) -> np.ndarray:
        """apply + sum p (-1)^bit per local qubit (-1: sum p), as the device's fused last pass."""
        self.apply(gates)
        return self.expect([(1 << q) if q >= 0 else 0 for q in qubits])

    def to_numpy(self) -> np.ndarray:
        return self.amps.copy()

    def local_total(self) -> float:
        return float(np.sum(np.abs(self.amps) ** 2))

    def sample_slice(self, shots, words, lo, hi, total, bit_src, code_or):
        bg = np.random.PCG64()
        bg.state = {"bit_generator": "PCG64", "state": {"state": (int(words[0]) << 64) | int(words[1]),
                    "inc": (int(words[2]) << 64) | int(words[3])}, "has_uint32": 0, "uinteger": 0}
        u = np.random.Generator(bg).random(shots)
        tau = u * total
        hi_eff = np.inf if hi is None else hi
        mine = (tau >= lo) & (tau < hi_eff)
        p = np.abs(self.amps) ** 2
        cum = np.cumsum(p)
        idx = np.searchsorted(cum, tau[mine] - lo, side="right")
        idx = np.minimum(idx, p.size - 1)
        codes = np.full(idx.size, np.uint64(code_or), dtype=np.uint64)
        for pbit, src in enumerate(bit_src):
            if src >= 0:
                codes |= ((idx.astype(np.uint64) >> np.uint64(src)) & np.uint64(1)) << np.uint64(pbit)
        vals, freq = np.unique(codes, return_counts=True)
        return vals, freq.astype(np.uint64)
