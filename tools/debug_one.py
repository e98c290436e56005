import sys, os
sys.path.insert(0, '.')
from paper_2512_04216_b200 import suite, statevector as sv
c = suite.qaoa_line_circuit(18, 2, seed=6)
print(sv.plan(18, c.instructions))
s = sv.DeviceState(18)
try:
    s.apply_instructions(c.instructions); print("apply ok")
except Exception as e:
    print("apply failed", e)
try:
    print(len(sv.run(c, 1000, 0, sampler="cdf").counts))
except Exception as e:
    print("run failed", e)
