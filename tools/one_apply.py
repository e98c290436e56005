"""Apply the QFT-n bench circuit once from a lazy |0...0> (target for ncu captures).
usage: one_apply.py [n] [prec] [z]   (z: fused <Z_i> on the last pass, as in bench.py)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
prec = sys.argv[2] if len(sys.argv) > 2 else "c128"
z = len(sys.argv) > 3 and sys.argv[3].startswith("z")
twice = len(sys.argv) > 3 and sys.argv[3] == "z2"  # then once more on the written state (dense-input program)
c = suite.qft_bench_circuit(n)
g = sv.gate_array(c.instructions)
s = sv.DeviceState(n, prec)
s.zero()
if z:
    s.apply_gates_z(g, list(range(n)))
    if twice:
        s.apply_gates_z(g, list(range(n)))
else:
    s.apply_gates(g)
print("ok")
