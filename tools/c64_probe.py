"""Apply times of complex64 programs (interpreter n < 24, NVRTC n >= 24): A/B of launch shapes."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
out = {}
for n in (20, 22, 23):
    c = suite.random_circuit(n, 400, np.random.default_rng(3), measured=False)
    g = sv.gate_array(c.instructions)
    s = sv.DeviceState(n, "c64")
    s.zero(); s.apply_gates(g); s.apply_gates(g)
    best = 1e9
    for _ in range(5):
        s.timer_start(); s.apply_gates(g); best = min(best, s.timer_stop())
    out[f"random{n}_400g_ms"] = round(best, 3)
for n in (26, 28):
    c = suite.sycamore_circuit(4, n // 4, 20, 0, measured=False)
    g = sv.gate_array(c.instructions)
    s = sv.DeviceState(n, "c64")
    s.zero(); s.apply_gates(g)
    best = 1e9
    for _ in range(3):
        s.zero(); s.timer_start(); s.apply_gates(g); best = min(best, s.timer_stop())
    out[f"syc{n}_ms"] = round(best, 3)
print(json.dumps(out))
