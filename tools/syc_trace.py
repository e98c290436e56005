"""Host/device breakdown of repeated Sycamore-32 c64 applies (run with SVB_TRACE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
g = sv.gate_array(suite.sycamore_circuit(4, 8, 20, 0, measured=False).instructions)
s = sv.DeviceState(32, "c64")
for r in range(4):
    s.zero()
    t0 = time.perf_counter(); s.apply_gates(g); t1 = time.perf_counter()
    print(f"zero-start apply {r}: {(t1 - t0) * 1e3:.1f} ms wall", file=sys.stderr, flush=True)
s.profile(True)
for r in range(3):
    s.zero()
    s.timer_start(); t0 = time.perf_counter(); s.apply_gates(g); t1 = time.perf_counter(); ms = s.timer_stop()
    print(f"profiled zero-start apply {r}: {(t1 - t0) * 1e3:.1f} ms wall, {ms:.1f} ms device", file=sys.stderr, flush=True)
