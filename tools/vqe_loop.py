"""A variational loop at 24-26 qubits through statevector.run_codes: the same
ansatz with new angles each iteration.  Structure-only NVRTC kernels are
compiled on the first iteration only (wall time per iteration printed)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
out = {}
for n in (24, 26):
    ts = []
    for it in range(8):
        c = suite.ry_ansatz_circuit(n, 2, seed=1000 + it)
        t0 = time.perf_counter(); sv.run_codes(c, 1000, it, qubit_cap=n); ts.append(round(time.perf_counter() - t0, 3))
    out[f"ry_ansatz_{n}x2_s"] = ts
print(json.dumps(out))
