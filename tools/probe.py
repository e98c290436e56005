#!/usr/bin/env python
"""Pass-level performance probes (CUDA events on the library stream).

  python tools/probe.py [--n 30] [--prec c128] [--only NAME]

Each experiment builds one gate program, warms up, then times it and the
fused-pass kernels inside it; prints one JSON line per experiment with the
pass count, the mean pass duration and algorithmic GB/s (2·s·2^n per pass).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2512_04216_b200 import statevector as sv  # noqa: E402
from paper_2512_04216_b200 import suite  # noqa: E402
from paper_2512_04216_b200.circuit import Circuit  # noqa: E402


def experiments(n: int):
    ex = {}
    c = Circuit(n)
    c.gate("h", n - 1)
    ex["h1_top"] = c
    c = Circuit(n)
    for q in range(n - 7, n):
        c.gate("h", q)
    ex["h7_top"] = c
    c = Circuit(n)
    for q in range(n):
        c.gate("h", q)
    ex["h_all"] = c
    c = Circuit(n)
    rng = np.random.default_rng(0)
    for _ in range(60):
        c.gate("rz", int(rng.integers(n)), params=(float(rng.uniform(0, 6)),))
    ex["rz60"] = c
    c = Circuit(n)
    for q in range(0, 5):
        c.gate("h", q)
    ex["h_low5"] = c
    ex["qft"] = suite.qft_bench_circuit(n)
    c = Circuit(n)
    for q in range(n):
        c.gate("x", q)
    suite.qft(n, c)
    ex["qft_noprep"] = c
    rows = 4
    cols = max(1, n // rows)
    if rows * cols == n:
        ex["sycamore_d20"] = suite.sycamore_circuit(rows, cols, 20, seed=0, measured=False)
    return ex


def run(name, c, n, prec, reps):
    gates = sv.gate_array(c.instructions)
    s = sv.DeviceState(n, prec)
    for _ in range(2):
        s.apply_gates(gates)
    s.profile(True)
    s.timer_start()
    for _ in range(reps):
        s.apply_gates(gates)
    total = s.timer_stop() / reps
    prof = s.profile_read()
    st = s.stats()
    s.close()
    npass = max(prof["pass_launches"], 1)
    pass_ms = prof["pass_ms"] / npass
    bytes_pp = prof["pass_bytes"] / npass
    out = {
        "exp": name, "n": n, "prec": prec, "gates": int(gates.size), "passes": st["passes"],
        "ms_total": round(total, 3), "pass_ms_mean": round(pass_ms, 3),
        "pass_GBps": round(bytes_pp / (pass_ms / 1e3) / 1e9, 1) if prof["pass_launches"] else None,
        "perm_ms": round(prof["perm_ms"] / max(prof["perm_launches"], 1), 3),
        "gates_per_s": round(gates.size / (total / 1e3), 1),
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--prec", default="c128")
    ap.add_argument("--only", default=None)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for name, c in experiments(a.n).items():
        if a.only and name not in a.only.split(","):
            continue
        run(name, c, a.n, a.prec, a.reps)


if __name__ == "__main__":
    main()
