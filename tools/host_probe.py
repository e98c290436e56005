"""Host time per apply_gates_z of the QFT-30 bench step (SVB_TRACE=1 prints host/sync split)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
g = sv.gate_array(suite.qft_bench_circuit(30).instructions)
s = sv.DeviceState(30)
for r in range(6):
    s.zero()
    t0 = time.perf_counter(); s.apply_gates_z(g, list(range(30))); t1 = time.perf_counter()
    print(f"step {r}: {(t1 - t0) * 1e3:.3f} ms wall", file=sys.stderr, flush=True)
