"""Per-pass device times of Sycamore-32 c64 applies (SVB_TRACE=1 prints each launch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
c = suite.sycamore_circuit(4, n // 4, 20, 0, measured=False)
g = sv.gate_array(c.instructions)
s = sv.DeviceState(n, "c64")
s.apply_gates(g)
for _ in range(2):
    s.zero(); s.profile(True); s.timer_start(); s.apply_gates(g); t = s.timer_stop(); p = s.profile_read()
    print("apply_ms", t, "pass_ms", p["pass_ms"], flush=True)
