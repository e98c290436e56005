"""Apply the QFT-n bench circuit once (target for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
prec = sys.argv[2] if len(sys.argv) > 2 else "c128"
c = suite.qft_bench_circuit(n)
g = sv.gate_array(c.instructions)
s = sv.DeviceState(n, prec)
s.zero(); s.apply_gates(g); s.sync() if hasattr(s, "sync") else None
print("ok")
