"""Global-qubit sharding of the state vector over ranks.

One process per GPU.  With P = 2^g ranks the 2^n amplitudes are split by the
top g *physical* qubits: rank r holds physical indices [r·2^nl, (r+1)·2^nl),
nl = n - g.  A logical→physical layout (``pos``) lets qubits move between
local and global positions.  The reference has no multi-device path
(`PAPER.md:462` lists MPI as future work; `partition.py:73-172` is the
nearest analogue, a cut-minimising placement for another objective).

* Gates whose non-preserved qubits are all local run locally through the
  fused pass engine.  Each rank first restricts the gate to its own values of
  any global qubit the gate preserves (a diagonal factor or a control on a
  global qubit becomes a local gate or a per-rank phase) — no communication.
* A gate that acts non-diagonally on a global qubit triggers a *grouped
  remap*: g' global qubits trade places with g' local ones in ONE all-to-all
  among the 2^g' ranks that differ in those global bits.  Each rank splits its
  shard into 2^g' blocks by the values of the g' local bits, keeps the block
  matching its own rank bits and sends block v to the partner whose bits are
  v: (1 - 2^-g')·s·2^nl bytes per rank per remap, against g'/2·s·2^nl for g'
  one-qubit pairwise swaps.  The remap brings in every global qubit whose next
  non-diagonal use comes before the next use of the local qubit it would
  evict (Belady pairing).  The exchange is chunked (≤ ``chunk_bytes`` per
  partner per stage, two stages): the pack of chunk j+1 on the libsvb stream
  overlaps the transfer of chunk j, so the staging memory is bounded (4 x
  (2^g' - 1) x 512 MiB) and a 36-qubit complex64 state fits on 4 x B200
  (128 GiB shards + 6 GiB of buffers).
* Lazy zero on every rank: a rank whose shard is still the zero vector (all
  ranks but 0 after a reset) neither writes nor computes it until data
  arrives; and while a global and a local logical qubit are both still |0>
  (no non-diagonal gate yet) they swap positions by relabeling alone.
* Reductions: <Z_mask> = local expectation × (-1)^(global bits) then
  all-reduce; sampling uses one shared PCG64 stream: every rank draws all
  uniforms and keeps the shots whose target lands in its slice of the global
  CDF (slices from an all-reduce of per-rank totals), so results do not
  depend on P.  Each rank histograms its shots on the device; the (code,
  count) arrays are all-gathered as tensors.

Plumbing is torch.distributed (NCCL over NVLink for device shards; gloo with
host-staged buffers for the multi-process tests).  The arithmetic is libsvb.
``backend`` may also be a shard factory (tests/sharded_emulator.py provides
a CPU emulation for the gloo tests; the product path has no CPU backend).
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .circuit import UNITARY_GATES
from .gates import matrix_of
from .result import format_counts, output_bit_sources
from .statevector import DeviceState, pcg_words


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


def remap_bytes(n: int, g: int, gp: int, itemsize: int) -> int:
    """Bytes one rank sends in a grouped remap of gp qubits (shard of 2^(n-g))."""
    return (itemsize << (n - g)) - (itemsize << (n - g - gp))


class _DeviceShard:
    """Local shard in HBM (libsvb).  Exchange buffers are torch CUDA tensors
    (NCCL, NVLink) or, with staging="host", pinned host tensors (gloo)."""

    def __init__(self, nl: int, precision: str, device: int, staging: str = "device"):
        import torch

        self.torch = torch
        self.state = DeviceState(nl, precision, device)
        self.nl = nl
        self.device = torch.device("cuda", device)
        self.itemsize = 16 if self.state.precision == "c128" else 8
        self.staging = staging

    # lifetime / content
    def apply(self, gates: np.ndarray) -> None:
        self.state.apply_gates(gates)

    def set_zero_state(self) -> None:  # |0...0> (lazy: the next pass synthesises it)
        self.state.zero()

    def clear(self) -> None:
        _lib.check(_lib.lib().svb_clear(self.state.handle))

    def close(self):
        self.state.close()

    # exchange
    def buffer(self, amps: int):
        if self.staging == "device":
            return self.torch.empty((amps * self.itemsize,), dtype=self.torch.uint8, device=self.device)
        return self.torch.empty((amps * self.itemsize,), dtype=self.torch.uint8, pin_memory=True)

    def _dev(self, buf):
        return buf if self.staging == "device" else buf.to(self.device)

    def block_out(self, lbits, block, off, count, buf) -> None:
        lb = np.ascontiguousarray(lbits, dtype=np.int32)
        if self.staging == "device":
            _lib.check(_lib.lib().svb_block_copy(self.state.handle, _lib.ptr(lb, _lib.c_int32), int(lb.size),
                                                 int(block), int(off), int(count), buf.data_ptr(), 1, 1))
        else:
            tmp = self.torch.empty((count * self.itemsize,), dtype=self.torch.uint8, device=self.device)
            _lib.check(_lib.lib().svb_block_copy(self.state.handle, _lib.ptr(lb, _lib.c_int32), int(lb.size),
                                                 int(block), int(off), int(count), tmp.data_ptr(), 1, 1))
            buf[: count * self.itemsize].copy_(tmp)

    def block_in(self, lbits, block, off, count, buf) -> None:
        lb = np.ascontiguousarray(lbits, dtype=np.int32)
        src = self._dev(buf[: count * self.itemsize])
        self.torch.cuda.current_stream(self.device).synchronize()  # NCCL / H2D done before libsvb reads
        _lib.check(_lib.lib().svb_block_copy(self.state.handle, _lib.ptr(lb, _lib.c_int32), int(lb.size),
                                             int(block), int(off), int(count), src.data_ptr(), 0, 1))

    # reductions
    def expect(self, masks) -> np.ndarray:
        return self.state.expect_z(masks)

    def apply_z(self, gates: np.ndarray, qubits) -> np.ndarray:
        """Apply, with sum p (-1)^bit for each local qubit (-1: sum p) taken by
        the program's last pass as it stores the shard."""
        return self.state.apply_gates_z(gates, qubits)

    def to_numpy(self) -> np.ndarray:
        return self.state.to_numpy()

    def sample_slice(self, shots, words, lo, hi, total, bit_src, code_or):
        return _sample_slice(self.state, shots, words, lo, hi, total, bit_src, code_or)

    def local_total(self) -> float:
        return float(self.state.expect_z([0])[0])


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

    def __init__(self, n: int, precision: str = "c64", device: int = 0, backend="device", group=None,
                 staging: str = "device", chunk_bytes: int = 1 << 29):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        g = self.P.bit_length() - 1
        if 1 << g != self.P:
            raise ValueError("sharded mode needs a power-of-two number of ranks")
        if n - g < 8:
            raise ValueError("too many ranks for this qubit count")
        self.n, self.g, self.nl = n, g, n - g
        self.precision = precision
        if backend == "device":
            self.shard = _DeviceShard(self.nl, precision, device, staging)
        else:
            self.shard = backend(self.nl, precision, device)
        self.itemsize = self.shard.itemsize
        self.chunk_amps = max(1, int(chunk_bytes) // self.itemsize)
        self._bufs: dict = {}
        self._plans: dict = {}  # apply() plans by (gates, layout, touched)
        self.reset()

    def reset(self) -> None:
        """Back to |0...0> with the identity layout.  Only rank 0 holds
        amplitude 1 (lazily); every other shard is the zero vector, kept
        unwritten until an exchange sends it data."""
        self.pos = list(range(self.n))  # logical -> physical
        self.touched = [False] * self.n  # a non-diagonal gate reached the qubit (it may be != |0>)
        self.swaps = 0  # qubits moved by exchanges
        self.remaps = 0  # all-to-all exchanges
        self.relabels = 0  # free moves of untouched qubits
        self.bytes_sent = 0
        if self.rank == 0:
            self.shard.set_zero_state()
            self.zero_shard = False
        else:
            self.zero_shard = True

    # ---------------------------------------------------------------- layout
    def _inv(self, pos=None):
        pos = self.pos if pos is None else pos
        inv = [0] * self.n
        for lq, ph in enumerate(pos):
            inv[ph] = lq
        return inv

    def _rank_bit(self, phys: int) -> int:
        return (self.rank >> (phys - self.nl)) & 1

    def _buffers(self, parts: int, amps: int):
        key = (parts, amps)
        if key not in self._bufs:
            self._bufs = {key: [[self.shard.buffer(amps) for _ in range(parts)] for _ in range(4)]}  # 2 send, 2 recv
        return self._bufs[key]

    def remap(self, pairs) -> None:
        """Grouped exchange: global physical G_i <-> local physical L_i for all
        pairs at once (one all-to-all among the 2^g' partners, chunked)."""
        pairs = sorted(pairs, key=lambda p: p[1])
        gp = len(pairs)
        L = [p[1] for p in pairs]
        kbits = [p[0] - self.nl for p in pairs]
        mine = sum(self._rank_bit(p[0]) << i for i, p in enumerate(pairs))
        partners = []
        for v in range(1 << gp):
            if v == mine:
                continue
            r = self.rank
            for i, k in enumerate(kbits):
                r = (r & ~(1 << k)) | (((v >> i) & 1) << k)
            partners.append((v, r))
        blen = 1 << (self.nl - gp)
        chunk = min(blen, self.chunk_amps)
        bufs = self._buffers(len(partners), chunk)
        send, recv = bufs[0:2], bufs[2:4]
        if self.zero_shard:
            for st in range(2):
                for b in send[st]:
                    b.zero_()
        offs = list(range(0, blen, chunk))
        prev = None
        for j, off in enumerate(offs):
            st = j & 1
            cnt = min(chunk, blen - off)
            if not self.zero_shard:
                for (v, _), b in zip(partners, send[st]):
                    self.shard.block_out(L, v, off, cnt, b)
            ops = []
            for (v, r), sb, rb in zip(partners, send[st], recv[st]):
                ops.append(self.dist.P2POp(self.dist.isend, sb[: cnt * self.itemsize], r, self.group))
                ops.append(self.dist.P2POp(self.dist.irecv, rb[: cnt * self.itemsize], r, self.group))
            reqs = self.dist.batch_isend_irecv(ops)
            if prev is not None:
                self._finish_chunk(prev, partners, recv, L)
            prev = (reqs, off, cnt, st)
        self._finish_chunk(prev, partners, recv, L)
        if self.zero_shard:
            self.zero_shard = False
        inv = self._inv()
        for G, Lp in pairs:
            a, c = inv[G], inv[Lp]
            self.pos[a], self.pos[c] = Lp, G
        self.swaps += gp
        self.remaps += 1
        self.bytes_sent += len(partners) * blen * self.itemsize

    def _finish_chunk(self, prev, partners, recv, L) -> None:
        reqs, off, cnt, st = prev
        for r in reqs:
            r.wait()
        if self.zero_shard:  # first data for this shard: materialise the zeros it holds
            self.shard.clear()
            self.zero_shard = False
        for (v, _), b in zip(partners, recv[st]):
            self.shard.block_in(L, v, off, cnt, b)

    def swap_qubits(self, G: int, L: int) -> None:
        """One global<->local move (a one-qubit grouped remap)."""
        self.remap([(G, L)])

    # ----------------------------------------------------------------- gates
    def apply(self, instructions, z_qubits=None):
        """Apply a gate list: local gates in fused batches, free relabels of
        untouched qubits, grouped remaps when a gate acts non-diagonally on a
        global qubit.  Plans depend only on the gates, the layout, the set of
        touched qubits and the rank: computed once and replayed.

        z_qubits (optional): also return <Z_q> of those logical qubits after
        the gates.  When the plan ends with a batch of local gates, the local
        sums come from that batch's last fused pass (no separate read pass):
        a local qubit contributes sum p (-1)^bit, a global one +-sum p by this
        rank's bit; one all-reduce adds the shards.  Otherwise one reduction
        pass (expectations)."""
        insts = [i for i in instructions if i.kind in UNITARY_GATES]
        key = (tuple((i.kind, tuple(i.qubits), tuple(i.params)) for i in insts), tuple(self.pos),
               tuple(self.touched))
        entry = self._plans.get(key)
        if entry is None:
            entry = (self._plan(insts), plan_touched(self.touched, insts))
            if len(self._plans) >= 8:
                self._plans.pop(next(iter(self._plans)))
            self._plans[key] = entry
        plan, touched_after = entry
        fuse_z = (z_qubits is not None and bool(plan) and plan[-1][0] == "gates"
                  and hasattr(self.shard, "apply_z"))
        zloc = None
        for ai, act in enumerate(plan):
            if act[0] == "gates":
                if self.zero_shard:  # gates map the zero vector to itself
                    continue
                if fuse_z and ai == len(plan) - 1:
                    # the layout no longer changes: local qubits by physical bit, -1 = the norm
                    phys = [self.pos[q] for q in z_qubits]
                    req = sorted({p for p in phys if p < self.nl}) + [-1]
                    got = dict(zip(req, self.shard.apply_z(act[1], req)))
                    zloc = np.array([got[p] if p < self.nl else (-got[-1] if self._rank_bit(p) else got[-1])
                                     for p in phys])
                else:
                    self.shard.apply(act[1])
            elif act[0] == "relabel":
                inv = self._inv()
                for G, Lp in act[1]:
                    a, c = inv[G], inv[Lp]
                    self.pos[a], self.pos[c] = Lp, G
                    inv[G], inv[Lp] = c, a
                self.relabels += len(act[1])
            else:
                self.remap(act[1])
        self.touched = list(touched_after)
        if z_qubits is None:
            return None
        if not fuse_z:
            return self.expectations([(q,) for q in z_qubits])
        if zloc is None:  # a shard of zeros
            zloc = np.zeros(len(z_qubits))
        return self._allreduce(zloc)

    def _plan(self, insts) -> list:
        """Actions [("gates", records) | ("relabel", pairs) | ("remap", pairs)]
        from the current layout (left unchanged; replaying updates it)."""
        mats = [matrix_of(i) for i in insts]
        pos = list(self.pos)
        touched = list(self.touched)
        # per qubit: indices of its non-diagonal uses (victim choice, Belady)
        uses: list[list[int]] = [[] for _ in range(self.n)]
        nondiag = []
        for t, (inst, m) in enumerate(zip(insts, mats)):
            k = len(inst.qubits)
            nd = [q for j, q in enumerate(inst.qubits) if not _preserved(m, k, j)]
            nondiag.append(nd)
            for q in nd:
                uses[q].append(t)
        nxt = [0] * self.n
        never = 1 << 60
        actions: list = []
        batch: list[np.ndarray] = []

        def flush():
            if batch:
                actions.append(("gates", np.concatenate(batch)))
                batch.clear()

        def next_use(q):
            return uses[q][nxt[q]] if nxt[q] < len(uses[q]) else never

        for t, (inst, m) in enumerate(zip(insts, mats)):
            k = len(inst.qubits)
            for q in range(self.n):
                while nxt[q] < len(uses[q]) and uses[q][nxt[q]] < t:
                    nxt[q] += 1
            need = [q for q in nondiag[t] if pos[q] >= self.nl]
            if need:
                flush()
                inv = [0] * self.n
                for lq, ph in enumerate(pos):
                    inv[ph] = lq
                busy = {pos[x] for x in inst.qubits}
                # free relabels: an untouched global qubit and an untouched local one are both |0>
                relab = []
                free_local = [Lp for Lp in range(self.nl) if Lp not in busy and not touched[inv[Lp]]]
                rest = []
                for q in need:
                    if not touched[q] and free_local:
                        Lp = free_local.pop()
                        relab.append((pos[q], Lp))
                        busy.add(Lp)
                        a, c = q, inv[Lp]
                        pos[a], pos[c] = Lp, pos[q]
                        inv[pos[a]], inv[pos[c]] = a, c
                    else:
                        rest.append(q)
                if relab:
                    actions.append(("relabel", relab))
                if rest:
                    # Belady pairing: needed qubits first, then any global qubit used
                    # before the local qubit it would evict
                    cands = sorted((Lp for Lp in range(self.nl) if Lp not in busy),
                                   key=lambda Lp: -next_use(inv[Lp]))
                    glob = [pos[q] for q in rest]
                    others = sorted((G for G in range(self.nl, self.n) if G not in glob),
                                    key=lambda G: next_use(inv[G]))
                    pairs = []
                    for G in glob:
                        pairs.append((G, cands.pop(0)))
                    for G in others:
                        if not cands or next_use(inv[G]) >= never or next_use(inv[G]) >= next_use(inv[cands[0]]):
                            break
                        pairs.append((G, cands.pop(0)))
                    actions.append(("remap", pairs))
                    for G, Lp in pairs:
                        a, c = inv[G], inv[Lp]
                        pos[a], pos[c] = Lp, G
                        inv[G], inv[Lp] = c, a
            for q in nondiag[t]:
                touched[q] = True
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
        vals = np.zeros(len(local_masks)) if self.zero_shard else self.shard.expect(local_masks) * np.array(signs)
        return self._allreduce(vals)

    def _gather_pairs(self, vals: np.ndarray, freq: np.ndarray):
        """All-gather of every rank's (code, count) arrays as tensors."""
        import torch

        if self.P == 1:
            return vals.astype(np.uint64), freq.astype(np.int64)
        dev = self.shard.device if (isinstance(self.shard, _DeviceShard)
                                    and self.dist.get_backend(self.group) == "nccl") else torch.device("cpu")
        size = torch.tensor([vals.size], dtype=torch.int64, device=dev)
        sizes = [torch.zeros_like(size) for _ in range(self.P)]
        self.dist.all_gather(sizes, size, group=self.group)
        mx = max(int(s.item()) for s in sizes)
        pad = np.zeros((2, mx), dtype=np.int64)
        pad[0, : vals.size] = vals.astype(np.uint64).view(np.int64)
        pad[1, : vals.size] = freq.astype(np.int64)
        t = torch.from_numpy(pad).to(dev)
        parts = [torch.empty_like(t) for _ in range(self.P)]
        self.dist.all_gather(parts, t, group=self.group)
        codes = np.concatenate([p[0, : int(s.item())].cpu().numpy() for p, s in zip(parts, sizes)]).view(np.uint64)
        counts = np.concatenate([p[1, : int(s.item())].cpu().numpy() for p, s in zip(parts, sizes)])
        return codes, counts

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
        totals[self.rank] = 0.0 if self.zero_shard else self.shard.local_total()
        if self.P > 1:
            totals = torch.from_numpy(self._allreduce(totals.numpy()))
        tot = totals.numpy()
        prefix = np.concatenate([[0.0], np.cumsum(tot)])
        lo = float(prefix[self.rank])
        hi = None if self.rank == self.P - 1 else float(prefix[self.rank + 1])
        if self.zero_shard or tot[self.rank] == 0.0:
            vals, freq = np.zeros(0, dtype=np.uint64), np.zeros(0, dtype=np.uint64)
        else:
            vals, freq = self.shard.sample_slice(shots, pcg_words(seed), lo, hi, float(prefix[-1]), bit_src, code_or)
        allc, allf = self._gather_pairs(np.asarray(vals), np.asarray(freq))
        codes, inv = np.unique(allc, return_inverse=True)
        counts = np.zeros(codes.size, dtype=np.int64)
        np.add.at(counts, inv, allf.astype(np.int64))
        return format_counts(codes, counts, len(src))

    def restore_layout(self) -> None:
        """Move every logical qubit back to its own physical position: one
        grouped remap for the global positions, one local permutation pass."""
        pairs = []
        pos = list(self.pos)
        for G in range(self.nl, self.n):  # logical G must end at physical G
            if pos[G] == G:
                continue
            p = pos[G]
            if p >= self.nl:  # parked on another global position: route through a local one
                busy = set(pos[x] for x in range(self.nl, self.n)) | {q for pr in pairs for q in pr}
                Lp = next(l for l in range(self.nl) if l not in busy)
                self.remap([(p, Lp)])
                pos = list(self.pos)
                p = pos[G]
            pairs.append((G, p))
        if pairs:
            self.remap(pairs)
        inv = self._inv()
        if any(inv[ph] != ph for ph in range(self.nl)):
            gates = []
            cur = list(inv[: self.nl])
            for ph in range(self.nl):  # selection sort with local swap gates
                if cur[ph] != ph:
                    j = cur.index(ph)
                    gates.append(_gate_rec((ph, j), matrix_of(_SwapInst())))
                    cur[ph], cur[j] = cur[j], cur[ph]
            if not self.zero_shard:
                self.shard.apply(np.concatenate(gates))
            self.pos = list(range(self.n))

    def gather(self) -> np.ndarray | None:
        """Full amplitude vector in logical order on rank 0."""
        self.restore_layout()
        local = np.zeros(1 << self.nl, dtype=np.complex128) if self.zero_shard else self.shard.to_numpy()
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


def plan_touched(touched, insts):
    """Touched flags after a gate list (a non-diagonal action on the qubit)."""
    out = list(touched)
    for inst in insts:
        m = matrix_of(inst)
        k = len(inst.qubits)
        for j, q in enumerate(inst.qubits):
            if not _preserved(m, k, j):
                out[q] = True
    return out


class _SwapInst:
    kind = "swap"
    qubits = (0, 1)
    params = ()
