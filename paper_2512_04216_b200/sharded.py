"""Global-qubit sharding of the state vector over ranks.

One process per GPU.  With P = 2^g ranks the 2^n amplitudes are split by the
top g *physical* qubits: rank r holds physical indices [r·2^nl, (r+1)·2^nl),
nl = n - g.  A logical→physical layout (``pos``) lets qubits move between
local and global positions.

* Gates whose non-preserved qubits are all local run locally through the
  fused pass engine.  Each rank first restricts the gate to its own values of
  any global qubit the gate preserves (a diagonal factor or a control on a
  global qubit becomes a local gate or a per-rank phase) — no communication.
* A gate that acts non-diagonally on a global qubit triggers a global↔local
  qubit swap: ranks r and r ^ 2^k exchange the half of their shard whose local
  bit L differs from their rank bit k (pack → send/recv → unpack), and the
  layout records the move.  The local victim is the qubit whose next
  non-diagonal use lies farthest ahead (Belady), so swap rounds are few.
* Reductions: <Z_mask> = local expectation × (-1)^(global bits) then
  all-reduce; sampling uses one shared PCG64 stream: every rank draws all
  uniforms, keeps the shots whose target lands in its slice of the global CDF
  (slices from an all-gather of per-rank totals), so the result does not
  depend on P.

Plumbing is torch.distributed (NCCL for device shards, gloo for the CPU
emulation backend used by the multi-process tests); the arithmetic is
libsvb on the device.
"""
from __future__ import annotations

import math

import numpy as np

from . import _lib
from .circuit import UNITARY_GATES
from .gates import matrix_of
from .result import format_counts, measurement_map, output_bit_sources
from .statevector import DeviceState, gate_array, pcg_words

def _preserved(m: np.ndarray, k: int, j: int) -> bool:
    """True when the 2^k x 2^k matrix never changes local bit j."""
    nz = np.argwhere(m != 0)
    return bool(np.all(((nz[:, 0] >> j) & 1) == ((nz[:, 1] >> j) & 1)))


def _restrict(m: np.ndarray, k: int, j: int, b: int) -> np.ndarray:
    """Block of m with local bit j fixed to b (j preserved) -> 2^(k-1) matrix."""
    idx = [i for i in range(1 << k) if ((i >> j) & 1) == b]
    return m[np.ix_(idx, idx)]


def _gate_rec(qubits, m) -> np.ndarray:
    rec = np.zeros(1, dtype=_lib.GATE_DTYPE)
    rec["k"][0] = len(qubits)
    rec["q"][0, : len(qubits)] = qubits
    rec["mat"][0, : 2 * m.size] = np.ascontiguousarray(m, dtype=np.complex128).reshape(-1).view(np.float64)
    return rec


class _DeviceShard:
    """Local shard in HBM (libsvb).  Exchange buffers are torch CUDA tensors
    (NCCL, NVLink) or, with staging="host", pinned host tensors (gloo; lets
    several processes share one GPU in tests without cross-process waits)."""

    def __init__(self, nl: int, precision: str, device: int, staging: str = "device"):
        import torch

        self.torch = torch
        self.state = DeviceState(nl, precision, device)
        self.nl = nl
        self.device = torch.device("cuda", device)
        self.itemsize = 16 if self.state.precision == "c128" else 8
        self.staging = staging

    def apply(self, gates: np.ndarray) -> None:
        self.state.apply_gates(gates)

    def _dev_half(self):
        return self.torch.empty((self.itemsize << (self.nl - 1),), dtype=self.torch.uint8, device=self.device)

    def half_out(self, L: int, bit: int):
        buf = self._dev_half()
        _lib.check(_lib.lib().svb_half_copy(self.state.handle, L, bit, buf.data_ptr(), 1))
        return buf if self.staging == "device" else buf.cpu()

    def half_in(self, L: int, bit: int, buf) -> None:
        if self.staging != "device":
            buf = buf.to(self.device)
        self.torch.cuda.synchronize(self.device)
        _lib.check(_lib.lib().svb_half_copy(self.state.handle, L, bit, buf.data_ptr(), 0))

    def empty_half(self):
        if self.staging == "device":
            return self._dev_half()
        return self.torch.empty((self.itemsize << (self.nl - 1),), dtype=self.torch.uint8, pin_memory=True)

    def expect(self, masks) -> np.ndarray:
        return self.state.expect_z(masks)

    def to_numpy(self) -> np.ndarray:
        return self.state.to_numpy()

    def sample_slice(self, shots, words, lo, hi, total, bit_src, code_or):
        return _sample_slice(self.state, shots, words, lo, hi, total, bit_src, code_or)

    def local_total(self) -> float:
        return float(self.state.expect_z([0])[0])

    def close(self):
        self.state.close()


class _EmulatedShard:
    """CPU emulation of a shard (TEST BACKEND for the multi-process gloo tests):
    gates through libsvb's CPU emulator of the fused program, data moves with
    numpy.  Never used on a GPU run."""

    def __init__(self, nl: int, precision: str, device: int = 0):
        import torch

        self.torch = torch
        self.nl = nl
        self.precision = precision
        self.amps = np.zeros(1 << nl, dtype=np.complex128)

    def apply(self, gates: np.ndarray) -> None:
        if gates.size:
            _lib.check(_lib.lib().svb_emulate_apply(self.nl, 1 if self.precision == "c128" else 0,
                                                    _lib.ptr(gates), int(gates.size), _lib.ptr(self.amps), 1))

    def _half_idx(self, L, bit):
        idx = np.arange(1 << (self.nl - 1), dtype=np.int64)
        lo = idx & ((1 << L) - 1)
        return ((idx >> L) << (L + 1)) | lo | (bit << L)

    def half_out(self, L, bit):
        return self.torch.from_numpy(self.amps[self._half_idx(L, bit)].copy())

    def half_in(self, L, bit, buf) -> None:
        self.amps[self._half_idx(L, bit)] = buf.numpy()

    def empty_half(self):
        return self.torch.from_numpy(np.empty(1 << (self.nl - 1), dtype=np.complex128))

    def expect(self, masks) -> np.ndarray:
        p = np.abs(self.amps) ** 2
        idx = np.arange(p.size, dtype=np.uint64)
        out = []
        for m in masks:
            par = (np.bitwise_count(idx & np.uint64(m)) & np.uint64(1)).astype(float)
            out.append(float(np.sum(p * (1.0 - 2.0 * par))))
        return np.array(out)

    def to_numpy(self) -> np.ndarray:
        return self.amps.copy()

    def local_total(self) -> float:
        return float(np.sum(np.abs(self.amps) ** 2))

    def sample_slice(self, shots, words, lo, hi, total, bit_src, code_or):
        # restatement of the device CDF slice sampler (test backend only)
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

    def close(self):
        pass


def _sample_slice(state: DeviceState, shots, words, lo, hi, total, bit_src, code_or):
    bs = np.ascontiguousarray(bit_src, dtype=np.int32)
    cap = min(int(shots), 1 << min(bs.size, 62))
    codes = np.empty(cap, dtype=np.uint64)
    freq = np.empty(cap, dtype=np.uint64)
    nu = _lib.c_uint64()
    w = np.ascontiguousarray(words, dtype=np.uint64)
    _lib.check(_lib.lib().svb_sample_slice(
        state.handle, int(shots), _lib.ptr(w, _lib.c_uint64), float(lo),
        float("inf") if hi is None else float(hi), float(total), _lib.ptr(bs, _lib.c_int32), int(bs.size),
        int(code_or), _lib.ptr(codes, _lib.c_uint64), _lib.ptr(freq, _lib.c_uint64), _lib.ctypes.byref(nu)))
    return codes[: nu.value], freq[: nu.value]


class ShardedState:
    """An n-qubit state sharded over the ranks of a torch.distributed group."""

    def __init__(self, n: int, precision: str = "c64", device: int = 0, backend: str = "device", group=None,
                 staging: str = "device"):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        g = self.P.bit_length() - 1
        if 1 << g != self.P:
            raise ValueError("sharded mode needs a power-of-two number of ranks")
        if n - g < 6:
            raise ValueError("too many ranks for this qubit count")
        self.n, self.g, self.nl = n, g, n - g
        self.precision = precision
        self.pos = list(range(n))  # logical -> physical
        if backend == "device":
            self.shard = _DeviceShard(self.nl, precision, device, staging)
        else:
            self.shard = _EmulatedShard(self.nl, precision, device)
        if backend != "device":
            self.shard.amps[:] = 0
            if self.rank == 0:
                self.shard.amps[0] = 1.0
        elif self.rank != 0:
            # zero_state put 1 at local index 0 on every rank: only rank 0 holds |0..0>
            _lib.check(_lib.lib().svb_clear(self.shard.state.handle))
        self.swaps = 0
        self.bytes_sent = 0
        self._plans: dict = {}  # apply() plans by (gates, layout)

    def reset(self) -> None:
        """Back to |0...0> with the identity layout (reuses the shard memory)."""
        self.pos = list(range(self.n))
        self.swaps = 0
        self.bytes_sent = 0
        if isinstance(self.shard, _DeviceShard):
            if self.rank == 0:
                self.shard.state.zero()
            else:
                _lib.check(_lib.lib().svb_clear(self.shard.state.handle))
        else:
            self.shard.amps[:] = 0
            if self.rank == 0:
                self.shard.amps[0] = 1.0

    # ---------------------------------------------------------------- layout
    def _inv(self):
        inv = [0] * self.n
        for lq, ph in enumerate(self.pos):
            inv[ph] = lq
        return inv

    def _rank_bit(self, phys: int) -> int:
        return (self.rank >> (phys - self.nl)) & 1

    def swap_qubits(self, G: int, L: int) -> None:
        """Exchange global physical position G with local position L."""
        k = G - self.nl
        partner = self.rank ^ (1 << k)
        b = self._rank_bit(G)
        send = self.shard.half_out(L, 1 - b)
        recv = self.shard.empty_half()
        ops = [self.dist.P2POp(self.dist.isend, send, partner, self.group),
               self.dist.P2POp(self.dist.irecv, recv, partner, self.group)]
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()
        self.shard.half_in(L, 1 - b, recv)
        inv = self._inv()
        a, c = inv[G], inv[L]
        self.pos[a], self.pos[c] = L, G
        self.swaps += 1
        self.bytes_sent += int(send.numel() * send.element_size())

    # ----------------------------------------------------------------- gates
    def apply(self, instructions) -> None:
        """Apply a gate list: local gates in fused batches, a global<->local swap
        whenever a gate acts non-diagonally on a global qubit.  The plan (swap
        choices and this rank's restricted gate records) depends only on the
        gates, the current layout and the rank, so it is computed once and
        replayed on later calls (the per-gate Python work is most of a step)."""
        insts = [i for i in instructions if i.kind in UNITARY_GATES]
        key = (tuple((i.kind, tuple(i.qubits), tuple(i.params)) for i in insts), tuple(self.pos))
        plan = self._plans.get(key)
        if plan is None:
            plan = self._plan(insts)
            if len(self._plans) >= 8:
                self._plans.pop(next(iter(self._plans)))
            self._plans[key] = plan
        for act in plan:
            if act[0] == "gates":
                self.shard.apply(act[1])
            else:
                self.swap_qubits(act[1], act[2])

    def _plan(self, insts) -> list:
        """Actions [("gates", records) | ("swap", G, L)] from the current layout
        (the layout itself is left unchanged; replaying the swaps updates it)."""
        mats = [matrix_of(i) for i in insts]
        pos = list(self.pos)

        def inv_of():
            inv = [0] * self.n
            for lq, ph in enumerate(pos):
                inv[ph] = lq
            return inv

        # per qubit: indices of future non-diagonal uses (for victim choice)
        uses: list[list[int]] = [[] for _ in range(self.n)]
        for t, (inst, m) in enumerate(zip(insts, mats)):
            k = len(inst.qubits)
            for j, q in enumerate(inst.qubits):
                if not _preserved(m, k, j):
                    uses[q].append(t)
        nxt = [0] * self.n
        actions: list = []
        batch: list[np.ndarray] = []

        def flush():
            if batch:
                actions.append(("gates", np.concatenate(batch)))
                batch.clear()

        for t, (inst, m) in enumerate(zip(insts, mats)):
            k = len(inst.qubits)
            for q in range(self.n):
                while nxt[q] < len(uses[q]) and uses[q][nxt[q]] < t:
                    nxt[q] += 1
            for j, q in enumerate(inst.qubits):
                if pos[q] >= self.nl and not _preserved(m, k, j):
                    flush()
                    busy = {pos[x] for x in inst.qubits}
                    inv = inv_of()
                    best, best_next = None, -1
                    for L in range(self.nl):
                        if L in busy:
                            continue
                        lq = inv[L]
                        nu = uses[lq][nxt[lq]] if nxt[lq] < len(uses[lq]) else 1 << 60
                        if nu > best_next:
                            best, best_next = L, nu
                    G = pos[q]
                    actions.append(("swap", G, best))
                    a, c = inv[G], inv[best]
                    pos[a], pos[c] = best, G
            # restrict to this rank's values of preserved global qubits
            qs = [pos[q] for q in inst.qubits]
            mm = m
            for j in reversed(range(k)):
                if qs[j] >= self.nl:
                    mm = _restrict(mm, len(qs), j, self._rank_bit(qs[j]))
                    qs = qs[:j] + qs[j + 1:]
            if not qs:  # pure per-rank phase: fold into a local diagonal
                ph = complex(mm.reshape(-1)[0])
                if ph != 1:
                    batch.append(_gate_rec((0,), np.array([[ph, 0], [0, ph]])))
                continue
            batch.append(_gate_rec(qs, mm))
        flush()
        return actions

    # ------------------------------------------------------------ reductions
    def _allreduce(self, x: np.ndarray) -> np.ndarray:
        import torch

        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        if not self.dist.is_initialized():
            return t.numpy()
        if isinstance(self.shard, _DeviceShard) and self.dist.get_backend(self.group) == "nccl":
            t = t.to(self.shard.device)
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def expectations(self, z_sets) -> np.ndarray:
        """<Z...Z> for each qubit set: one local pass for all masks + all-reduce."""
        local_masks, signs = [], []
        for z in z_sets:
            lm, s = 0, 1.0
            for q in set(z):
                ph = self.pos[q]
                if ph < self.nl:
                    lm |= 1 << ph
                elif self._rank_bit(ph):
                    s = -s
            local_masks.append(lm)
            signs.append(s)
        vals = self.shard.expect(local_masks) * np.array(signs)
        return self._allreduce(vals)

    def sample(self, measures, shots: int, seed: int) -> dict:
        """Terminal sampling (distributed CDF over the shared PCG64 stream of
        default_rng(seed)); measures = [(qubit, clbit)] as in result.py."""
        import torch

        self.restore_layout()  # CDF order = logical order: counts independent of P
        qubits = sorted({q for q, _ in measures})
        src = output_bit_sources(measures, qubits)
        bit_src, code_or = [], 0
        for p, j in enumerate(src):
            ph = self.pos[qubits[j]]
            if ph < self.nl:
                bit_src.append(ph)
            else:
                bit_src.append(-1)
                code_or |= self._rank_bit(ph) << p
        totals = torch.zeros(self.P, dtype=torch.float64)
        totals[self.rank] = self.shard.local_total()
        if self.P > 1:
            self.dist.all_reduce(totals, group=self.group)
        tot = totals.numpy()
        prefix = np.concatenate([[0.0], np.cumsum(tot)])
        lo = float(prefix[self.rank])
        hi = None if self.rank == self.P - 1 else float(prefix[self.rank + 1])
        vals, freq = self.shard.sample_slice(shots, pcg_words(seed), lo, hi, float(prefix[-1]), bit_src, code_or)
        # gather (code, count) pairs on every rank
        pairs = np.stack([vals.astype(np.uint64), freq.astype(np.uint64)], axis=1) if vals.size else \
            np.zeros((0, 2), dtype=np.uint64)
        if self.P > 1:
            gathered = [None] * self.P
            self.dist.all_gather_object(gathered, pairs, group=self.group)
        else:
            gathered = [pairs]
        allp = np.concatenate([x for x in gathered if x.size], axis=0) if any(x.size for x in gathered) else \
            np.zeros((0, 2), dtype=np.uint64)
        codes, inv = np.unique(allp[:, 0], return_inverse=True)
        counts = np.zeros(codes.size, dtype=np.int64)
        np.add.at(counts, inv, allp[:, 1].astype(np.int64))
        return format_counts(codes, counts, len(src))

    def restore_layout(self) -> None:
        """Move every logical qubit back to its own physical position (swap
        rounds for global positions, one local permutation pass for the rest)."""
        for G in range(self.nl, self.n):  # bring logical G to physical G
            if self.pos[G] == G:
                continue
            p = self.pos[G]
            if p >= self.nl:  # parked on another global position: route through a local one
                busy = {self.pos[x] for x in range(self.nl, self.n)}
                L = next(l for l in range(self.nl) if l not in busy)
                self.swap_qubits(p, L)
                p = self.pos[G]
            self.swap_qubits(G, p)
        inv = self._inv()
        if any(inv[ph] != ph for ph in range(self.nl)):
            gates = []
            cur = list(inv[: self.nl])
            for ph in range(self.nl):  # selection sort with local swap gates
                if cur[ph] != ph:
                    j = cur.index(ph)
                    gates.append(_gate_rec((ph, j), matrix_of(_SwapInst())))
                    cur[ph], cur[j] = cur[j], cur[ph]
            self.shard.apply(np.concatenate(gates))
            self.pos = list(range(self.n))

    def gather(self) -> np.ndarray | None:
        """Full amplitude vector in logical order on rank 0."""
        self.restore_layout()
        local = self.shard.to_numpy()
        import torch

        t = torch.from_numpy(local.view(np.float64).copy())
        if self.P == 1:
            return local
        if self.rank == 0:
            parts = [torch.empty_like(t) for _ in range(self.P)]
            self.dist.gather(t, gather_list=parts, dst=0, group=self.group)
            return np.concatenate([p.numpy().view(np.complex128) for p in parts])
        self.dist.gather(t, dst=0, group=self.group)
        return None

    def close(self):
        self.shard.close()


class _SwapInst:
    kind = "swap"
    qubits = (0, 1)
    params = ()
