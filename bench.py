#!/usr/bin/env python
"""Benchmark of the B200 state-vector hot path.

Workload (BASELINE.json configs[1]): QFT on 30 qubits, complex128, one B200 —
ry(0.1·(q+1)) preparation + conftest `qft(30)` = 2250 IR gates — producing the
full amplitude vector and <Z_i> for i = 0..29.  One step = zero the state
(lazy |0...0>), run the whole gate program (fused HBM passes; the swap
relabeling is absorbed by the initial qubit layout of the lazy zero state),
with <Z_i> summed by the last pass as it stores the amplitudes.  Metric: IR gates per second (the first metric
BASELINE.json names); the per-pass HBM GB/s is reported as `roofline`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

* `value`: device-resident throughput, timed with CUDA events recorded on the
  library's stream (all kernels of the state run there).
* `e2e`: the same metric through the public API (`expectations` then
  `final_state(c, out=pinned)`), wall-clock per step including host gate encoding, the
  gate-program upload and the 16 GiB amplitude read-back into pinned memory.
* `cpu_baseline` / `--impl reference`: the numpy restatement of the reference
  algorithm (oracle/, "port") timed on this host on a bounded, evenly spaced
  sample of the same gate list.
* N > 1 (torchrun, NCCL): weak scaling — QFT on 30 + log2(N) qubits, complex128,
  sharded by global qubits (paper_2512_04216_b200/sharded.py): 16 GiB of state
  per GPU at every N, global<->local qubit swaps over NVLink.  ``--sharded``
  forces that path at N = 1.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_QUBITS = 30
PRECISION = "c128"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def measured_traffic():
    """dram read+write bytes per launch of the dominant kernel (the bench step's
    last fused pass) from the committed ncu --set full capture
    (profiles/r01_ncu_qft30_pass_full.json, record "qft30_top"), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_qft30_pass_full.json")) as fh:
            recs = json.load(fh)
        top = [r for r in recs if "top" in r.get("report", "")] or recs[:1]
        return float((top[0]["dram_read_bytes"] + top[0]["dram_write_bytes"]) * 1e9)  # ncu reports GB
    except Exception:
        return None


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: NVML in a thread every ~2 ms (the timed region can be tens of ms),
    else nvidia-smi -lms 200."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    NVML_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.sm: list[float] = []
        self.reasons: set = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            idx = self.device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[self.device])
                except ValueError:
                    pass
            self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._nvml = pynvml
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self._sample_nvml()
            self._t = threading.Thread(target=self._loop_nvml, daemon=True)
            self._t.start()
            return self
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _sample_nvml(self):
        nv = self._nvml
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        for name, b in self.NVML_BITS.items():
            if bits & b:
                self.reasons.add(name)

    def _loop_nvml(self):
        while not self._stop.wait(0.002):
            try:
                self._sample_nvml()
            except Exception:
                return

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self._nvml is not None:
            self._stop.set()
            self._t.join(timeout=2)
            try:
                self._sample_nvml()
            except Exception:
                pass
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        if self._nvml is not None:
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


# ---------------------------------------------------------------- CPU side
def cpu_sample_plan(n_full: int, steps: int, per_step: int):
    """Evenly spaced gates of the QFT-n gate list, and the n it runs at."""
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    # numpy's dense 1q path needs ~3x the 16 GiB state at n=30
    n_cpu = n_full if avail > 4 * (16 << n_full) else 26
    from paper_2512_04216_b200 import suite

    gates = [i for i in suite.qft_bench_circuit(n_cpu).instructions]
    total = steps * per_step
    idx = np.linspace(0, len(gates) - 1, total).astype(int)
    return n_cpu, [gates[i] for i in idx]


def time_cpu_port(n_cpu: int, gates, n_full: int) -> tuple[float, float]:
    """Seconds per gate of the numpy port, scaled to n_full (cost is linear in 2^n)."""
    from oracle import sv_oracle as orc

    psi = orc.zero_state(n_cpu)
    t0 = time.perf_counter()
    for g in gates:
        orc.apply_instruction(psi, n_cpu, g)
    dt = time.perf_counter() - t0
    scale = float(1 << (n_full - n_cpu))
    return dt / len(gates) * scale, dt


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    n_cpu, sample = cpu_sample_plan(N_QUBITS, args.steps + args.warmup, 3)
    per_step = 3
    times = []
    for s in range(args.warmup + args.steps):
        spg, _ = time_cpu_port(n_cpu, sample[s * per_step:(s + 1) * per_step], N_QUBITS)
        if s >= args.warmup:
            times.append(spg)
    sec_per_gate = float(np.mean(times))
    total_gates = 2250
    value = 1.0 / sec_per_gate
    desc = (f"{per_step} evenly spaced gates of the 2250-gate QFT-30 list per step at n={n_cpu}"
            + ("" if n_cpu == N_QUBITS else f", time x{1 << (N_QUBITS - n_cpu)} (cost linear in 2^n)"))
    line = {
        "impl": "reference",
        "metric": "gates/sec (QFT-30 complex128, full amplitudes + <Z_i>)",
        "value": value,
        "unit": "gates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_gates * sec_per_gate * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c128",
        "data": "synthetic (deterministic QFT circuit)",
        "config": {"workload": "qft30_c128_amplitudes_plus_z", "n_qubits": N_QUBITS, "gates": total_gates},
        "cpu_baseline": {"value": value, "unit": "gates/s", "cores": 1, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU side
def run_ours(args, rank: int, world: int, dist):
    from paper_2512_04216_b200 import statevector as sv
    from paper_2512_04216_b200 import suite

    device = int(os.environ.get("LOCAL_RANK", 0))
    c = suite.qft_bench_circuit(N_QUBITS)
    gates = sv.gate_array(c.instructions)
    n_gates = int(gates.size)
    masks = [1 << q for q in range(N_QUBITS)]
    state = sv.DeviceState(N_QUBITS, PRECISION, device)
    plan = sv.plan(N_QUBITS, c.instructions, PRECISION, zero_start=True)  # each step starts from a lazy |0...0>

    zq = list(range(N_QUBITS))

    def step():
        # lazy |0...0>, the fused program, and <Z_i> summed by its last pass
        state.zero()
        return state.apply_gates_z(gates, zq)

    for _ in range(max(args.warmup, 3)):
        z = step()
    # the fused <Z_i> (last pass) agrees with the separate multi-mask reduction pass
    np.testing.assert_allclose(z, state.expect_z(masks), atol=1e-10)
    stats = state.stats()

    def barrier():
        if dist is not None:
            dist.barrier()

    barrier()
    state.profile(True)
    with ClockSampler(device) as clk:
        state.timer_start()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            z = step()  # synchronous: each apply ends with a stream sync
        wall_ms = (time.perf_counter() - w0) * 1e3
        total_ms = state.timer_stop()
    prof = state.profile_read()
    barrier()
    if dist is not None:
        import torch

        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * n_gates / (ms_per_step / 1e3)

    # roofline of the dominant kernel: the fused pass (by program position) with
    # the largest share of the step, CUDA events on the launch stream; bytes =
    # HBM bytes that pass moves (live tiles written, written positions read)
    per_pass = state.profile_passes()
    state.profile(False)
    top = max(range(len(per_pass)), key=lambda i: per_pass[i]["ms"])
    pass_avg_ms = per_pass[top]["ms"] / max(per_pass[top]["launches"], 1)
    pass_bytes = per_pass[top]["bytes"] / max(per_pass[top]["launches"], 1)
    achieved = pass_bytes / (pass_avg_ms / 1e3) / 1e9
    peak, peak_kind = hbm_peak()
    pass_table = [{"ms": p["ms"] / max(p["launches"], 1), "gbytes": p["bytes"] / max(p["launches"], 1) / 1e9}
                  for p in per_pass]

    # dense input: the same program on an already-written (non-lazy) state, so
    # every pass streams the whole 16 GiB (and the bit reversal is a real
    # permutation): the full-state pass throughput, reported beside the step
    for _ in range(2):  # warm-up: this program (no zero start) has its own JIT kernels
        zd = state.apply_gates_z(gates, zq)
    state.profile(True)
    state.timer_start()
    for _ in range(args.steps):
        zd = state.apply_gates_z(gates, zq)
    dense_ms = state.timer_stop() / args.steps
    dense_passes = state.profile_passes()
    state.profile(False)
    dtop = max(range(len(dense_passes)), key=lambda i: dense_passes[i]["ms"])
    d_ms = dense_passes[dtop]["ms"] / max(dense_passes[dtop]["launches"], 1)
    d_bytes = dense_passes[dtop]["bytes"] / max(dense_passes[dtop]["launches"], 1)
    dense = {"value": world * n_gates / (dense_ms / 1e3), "unit": "gates/s", "ms_per_step": dense_ms,
             "passes": [{"ms": p["ms"] / max(p["launches"], 1), "gbytes": p["bytes"] / max(p["launches"], 1) / 1e9}
                        for p in dense_passes],
             "roofline_top_pass": {"achieved": d_bytes / (d_ms / 1e3) / 1e9, "frac": d_bytes / (d_ms / 1e3) / 1e9 / peak,
                                   "avg_launch_ms": d_ms, "bytes_per_launch": d_bytes},
             "note": "input = the previous output (no lazy-zero support skipping, no free initial layout)"}

    # e2e through the public API (host gate encoding + upload + 16 GiB read-back)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    pinned = sv.PinnedBuffer(1 << N_QUBITS)
    e2e_times = []
    for i in range(e2e_steps + 1):
        ci = suite.qft_bench_circuit(N_QUBITS)
        t0 = time.perf_counter()
        zi = sv.expectations(ci, [(q,) for q in range(N_QUBITS)], qubit_cap=N_QUBITS)  # applies + caches
        sv.final_state(ci, qubit_cap=N_QUBITS, out=pinned.array)
        dt = time.perf_counter() - t0
        del ci
        if i > 0:  # first call pays one-time allocations
            e2e_times.append(dt)
    e2e_s = float(np.mean(e2e_times))
    np.testing.assert_allclose(zi, z, atol=1e-10)
    pinned.close()
    state.close()

    line = {
        "metric": "gates/sec (QFT-30 complex128, full amplitudes + <Z_i>)",
        "value": value,
        "unit": "gates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c128",
        "data": "synthetic (deterministic QFT circuit; state 16 GiB >> 126 MB L2, no flush needed)",
        "config": {"workload": "qft30_c128_amplitudes_plus_z", "n_qubits": N_QUBITS, "gates": n_gates,
                   "parallelism": "replicas" if world > 1 else "single", "l2": "inputs larger than L2",
                   "hbm_passes_per_step": stats["passes"], "plan": plan,
                   "start": ("lazy |0...0> each step: the passes launch only tiles inside the written support and "
                             "synthesise never-written positions as exact zeros (DESIGN.md §3); `dense` below is the "
                             "same circuit on an already-written input"),
                   "wall_ms_per_step": wall_ms / args.steps},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": measured_traffic(),
                     "kernel": f"svb_jit (fused pass {top} of {len(per_pass)}, c128)",
                     "peak_kind": peak_kind, "bytes_per_launch": pass_bytes, "avg_launch_ms": pass_avg_ms,
                     "passes": pass_table},
        "dense": dense,
        "e2e": {"value": world * n_gates / e2e_s, "unit": "gates/s",
                "h2d_bytes_per_step": int(gates.nbytes),
                "d2h_bytes_per_step": int((16 << N_QUBITS) + 8 * N_QUBITS), "ms_per_step": e2e_s * 1e3},
        "gpu_launches": int(args.steps * (stats["launches"] + 1)),  # fused passes + the <Z> row sum
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_cpu_baseline:
        n_cpu, sample = cpu_sample_plan(N_QUBITS, 1, args.cpu_gates)
        spg, dt = time_cpu_port(n_cpu, sample, N_QUBITS)
        line["cpu_baseline"] = {
            "value": 1.0 / spg, "unit": "gates/s", "cores": 1, "kind": "port",
            "sample": f"{len(sample)} evenly spaced gates of the QFT-30 list at n={n_cpu}"
                      + ("" if n_cpu == N_QUBITS else f", x{1 << (N_QUBITS - n_cpu)} scaled")
                      + f", {dt:.1f} s wall"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_sharded(args, rank: int, world: int, dist):
    """Weak scaling: QFT-(30 + log2 N) c128 sharded over N GPUs."""
    import torch

    from paper_2512_04216_b200 import suite
    from paper_2512_04216_b200.sharded import ShardedState

    device = int(os.environ.get("LOCAL_RANK", 0))
    g = world.bit_length() - 1
    n = N_QUBITS + g
    c = suite.qft_bench_circuit(n)
    n_gates = len(c.instructions)

    def barrier():
        if dist is not None:
            dist.barrier()

    st = ShardedState(n, PRECISION, device=device, backend="device")

    def step():
        st.reset()
        st.apply(c.instructions)
        z = st.expectations([(q,) for q in range(n)])
        return z, st.swaps, st.bytes_sent

    for _ in range(max(args.warmup, 1)):
        step()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clk:
        w0 = time.perf_counter()
        e0.record()
        for _ in range(args.steps):
            z, swaps, sent = step()  # host gate encoding, device passes, swaps, <Z_i> read back to the host
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        wall_ms = (time.perf_counter() - w0) * 1e3 / args.steps
    total_ms = e0.elapsed_time(e1)
    barrier()
    if dist is not None:
        t = torch.tensor([total_ms, wall_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, wall_ms = float(t[0].item()), float(t[1].item())
    ms = total_ms / args.steps
    line = {
        "metric": "gates/sec (QFT-30 complex128, full amplitudes + <Z_i>)",
        "value": n_gates / (ms / 1e3),
        "unit": "gates/s", "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 1),
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (deterministic QFT circuit, 16 GiB state per GPU >> L2)",
        "config": {"workload": f"qft{n}_c128_sharded_weak", "n_qubits": n, "gates": n_gates,
                   "parallelism": f"sharded{world}", "swaps_per_step": swaps, "bytes_sent_per_rank": sent,
                   "l2": "inputs larger than L2"},
        "e2e": {"value": n_gates / (wall_ms / 1e3), "unit": "gates/s", "h2d_bytes_per_step": int(n_gates * 272),
                "d2h_bytes_per_step": 8 * n, "ms_per_step": wall_ms,
                "note": "wall clock per step, max over ranks: gate encoding + upload, passes, swaps, <Z_i> to the host"},
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-gates", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="sharded path even at N = 1")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
        dist = tdist
    if world > 1 or args.sharded:
        run_sharded(args, rank, world, dist)
    else:
        run_ours(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
