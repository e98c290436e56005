"""Apply one config-4 circuit (qaoa_line 24 x 2) from |0..0>: target for ncu (argv[1] = interp|jit)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
mode = sys.argv[1] if len(sys.argv) > 1 else "interp"
c = suite.qaoa_line_circuit(24, 2, 0, False)
g = sv.gate_array(c.instructions)
s = sv.DeviceState(24, "c128")
s.set_option(2, -1 if mode == "interp" else 0)
for _ in range(2):
    s.zero(); s.apply_gates(g)
print("ok")
