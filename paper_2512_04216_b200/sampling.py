"""Device alias tables with the reference's `polysim.sampling` surface.

``AliasTable.from_probs`` (`sampling.py:30-70`) builds the Walker/Vose table
on the B200 with the reference's round structure (svb_alias_table: the same
cumsum / searchsorted / bincount rounds, so tables are bit-identical), and
``sample_indices`` (`sampling.py:78-83`) draws on the device from the numpy
PCG64 stream of the caller's Generator (svb_alias_sample), advancing that
Generator by exactly one double per draw as ``rng.random(n)`` would.

``sample_one`` and ``reconstructed_probs`` are the reference's scalar helpers
(one comparison / one bincount on the already-built host copy of the table);
they are not draws of a batch and keep the reference's duck-typed ``rng``
contract (`tests/test_sampling.py:55-72`).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import SamplingError, check, lib, ptr


class _DeviceRows:
    """Owner of a device-resident table (svb_alias_upload / svb_alias_release)."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            if self.handle:
                lib().svb_alias_release(self.handle)
        except Exception:
            pass


@dataclass
class AliasTable:
    size: int
    prob: np.ndarray
    alias: np.ndarray
    outcomes: list | None = None
    device: int = 0

    @classmethod
    def from_probs(cls, probs, outcomes: list | None = None, device: int = 0) -> "AliasTable":
        probs = np.ascontiguousarray(probs, dtype=np.float64)
        if probs.ndim != 1 or probs.size == 0:
            raise SamplingError("need a non-empty 1-D probability vector")
        m = int(probs.size)
        prob_row = np.empty(m, dtype=np.float64)
        alias_row = np.empty(m, dtype=np.int64)
        check(lib().svb_alias_table(device, ptr(probs, _lib.c_double), m, ptr(prob_row, _lib.c_double),
                                    ptr(alias_row, _lib.c_int64)))
        return cls(size=m, prob=prob_row, alias=alias_row, outcomes=outcomes, device=device)

    @classmethod
    def from_distribution(cls, dist: dict, device: int = 0) -> "AliasTable":
        outcomes = sorted(dist)
        probs = np.array([dist[k] for k in outcomes], dtype=float)
        return cls.from_probs(probs, outcomes=outcomes, device=device)

    def sample_indices(self, rng: np.random.Generator, n: int) -> np.ndarray:
        """n draws on the device from rng's PCG64 stream (one double each)."""
        from .statevector import pcg_words

        n = int(n)
        if n == 0:
            return np.empty(0, dtype=np.int64)
        words = pcg_words(rng)
        out = np.empty(n, dtype=np.uint64)
        check(lib().svb_alias_sample_table(self._device_table(), n, ptr(words, _lib.c_uint64),
                                           ptr(out, _lib.c_uint64)))
        rng.bit_generator.advance(n)
        return out.view(np.int64)

    def __getstate__(self):  # the device rows stay with the process that uploaded them
        state = dict(self.__dict__)
        state.pop("_dev", None)
        return state

    def _device_table(self):
        """The rows on the device, uploaded once per (prob, alias) pair: per-draw
        cost independent of the table size (sampling.py:72-77; a per-call upload
        made big tables' draws ~3x dearer).  Re-uploaded when the attributes are
        reassigned; in-place edits of the arrays are not tracked."""
        key = (id(self.prob), id(self.alias), self.size, self.device)
        cached = self.__dict__.get("_dev")
        if cached is not None and cached[0] == key:
            return cached[1].handle
        pr = np.ascontiguousarray(self.prob, dtype=np.float64)
        al = np.ascontiguousarray(self.alias, dtype=np.int64)
        h = _lib.c_void_p()
        check(lib().svb_alias_upload(self.device, ptr(pr, _lib.c_double), ptr(al, _lib.c_int64), self.size,
                                     _lib.ctypes.byref(h)))
        table = _DeviceRows(h)
        self.__dict__["_dev"] = (key, table)
        return table.handle

    def sample_one(self, rng) -> int:
        v = rng.random() * self.size
        idx = int(v)
        return idx if (v - idx) < self.prob[idx] else int(self.alias[idx])

    def reconstructed_probs(self) -> np.ndarray:
        """Probability mass each outcome receives from the table (sampling.py:88-95)."""
        out = self.prob.copy()
        np.add.at(out, self.alias, 1.0 - self.prob)
        return out / self.size


def counts_to_distribution(counts: dict) -> dict:
    """sampling.py:98-104 (pure dict arithmetic)."""
    total = sum(counts.values())
    if total <= 0:
        raise SamplingError("empty counts")
    return {k: v / total for k, v in counts.items()}
