"""One dense 5-qubit block on a 30-qubit complex64 state through each engine
(target for ncu captures of k_dense_tc / k_dense_fma)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2512_04216_b200 import statevector as sv
from paper_2512_04216_b200.circuit import Instruction
n, k = 30, int(sys.argv[1]) if len(sys.argv) > 1 else 5
rng = np.random.default_rng(0)
U, _ = np.linalg.qr(rng.normal(size=(1 << k, 1 << k)) + 1j * rng.normal(size=(1 << k, 1 << k)))
s = sv.DeviceState(n, "c64")
s.apply_instructions([Instruction("h", (i,)) for i in range(n)])
q = [3, 11, 17, 22, 29, 7][:k]
for eng in ("tensor", "fma"):
    s.apply_matrix(q, U, engine=eng)
print("ok")
