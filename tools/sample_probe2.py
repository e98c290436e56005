"""Sampling breakdown probe: CDF sampler timings on a 32-qubit c64 state (repeated)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2512_04216_b200 import statevector as sv, suite
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
g = sv.gate_array(suite.sycamore_circuit(4, n // 4, 20, 0, measured=False).instructions)
s = sv.DeviceState(n, "c64")
s.apply_gates(g)
qubits = list(range(n))
for shots in (10**6, 10**6, 10**6, 10**5, 10**7):
    t0 = time.perf_counter(); s.timer_start()
    codes, freq = s.sample_codes(qubits, qubits, shots, sv.pcg_words(1), 1)
    ms = s.timer_stop(); t1 = time.perf_counter()
    print(json.dumps({"n": n, "shots": shots, "device_ms": ms, "wall_ms": (t1 - t0) * 1e3, "distinct": int(codes.size)}),
          flush=True)
