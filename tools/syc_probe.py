import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite, _lib
n = int(sys.argv[1]); depth = int(sys.argv[2])
c = suite.sycamore_circuit(4, n // 4, depth, 0, measured=False)
g = sv.gate_array(c.instructions)
s = sv.DeviceState(n, "c64"); s.set_option(_lib.OPT_JIT_MIN_N, 1)
s.apply_gates(g); s.apply_gates(g)
print(sv.plan(n, c.instructions, "c64"))
