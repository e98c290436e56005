"""Zero-start vs dense apply wall times (diagnostic; wall clock around the synchronous apply)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
for n, prec, rows, cols in ((32, "c64", 4, 8), (30, "c128", 5, 6), (30, "c64", 5, 6)):
    g = sv.gate_array(suite.sycamore_circuit(rows, cols, 20, 0, measured=False).instructions)
    s = sv.DeviceState(n, prec)
    s.zero(); s.apply_gates(g); s.apply_gates(g)  # compile both programs
    for r in range(3):
        s.zero()
        t0 = time.perf_counter(); s.apply_gates(g); tz = time.perf_counter() - t0
        t0 = time.perf_counter(); s.apply_gates(g); td = time.perf_counter() - t0
        print(json.dumps({"n": n, "prec": prec, "rep": r, "zero_start_ms": tz * 1e3, "dense_ms": td * 1e3}), flush=True)
    s.close()
