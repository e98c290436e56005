"""QFT-30 end-to-end through the public API, split: expectations (encode + apply + <Z>), final_state (16 GiB D2H), release."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
n = 30
pinned = sv.PinnedBuffer(1 << n)
for i in range(5):
    ci = suite.qft_bench_circuit(n)
    t0 = time.perf_counter(); g = sv.gate_array(ci.instructions); t1 = time.perf_counter()
    z = sv.expectations(ci, [(q,) for q in range(n)], qubit_cap=n); t2 = time.perf_counter()
    sv.final_state(ci, qubit_cap=n, out=pinned.array); t3 = time.perf_counter()
    del ci; t4 = time.perf_counter()
    print(f"encode {1e3*(t1-t0):.1f} ms  expectations {1e3*(t2-t1):.1f} ms  final_state {1e3*(t3-t2):.1f} ms  release {1e3*(t4-t3):.1f} ms  total(e2e) {1e3*(t4-t1):.1f}", flush=True)
