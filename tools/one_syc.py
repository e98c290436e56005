"""Apply the Sycamore-32 c64 circuit once (target for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
c = suite.sycamore_circuit(4, n // 4, 20, 0, measured=False)
s = sv.DeviceState(n, "c64")
s.zero(); s.apply_gates(sv.gate_array(c.instructions))
print("ok")
