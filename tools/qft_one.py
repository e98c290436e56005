import sys, os
sys.path.insert(0, os.getcwd())
from paper_2512_04216_b200 import statevector as sv, suite
c = suite.qft_bench_circuit(30); g = sv.gate_array(c.instructions); s = sv.DeviceState(30, "c128")
s.zero(); z = s.apply_gates_z(g, list(range(30)))
print(z[:3])
