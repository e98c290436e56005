"""Cold-process cost of the config-4 batch pieces: which part of the first call is slow.
usage: batch_cold.py small|large|both"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
t0 = time.perf_counter()
from paper_2512_04216_b200 import suite, batch, statevector as sv, _lib
out = {"import_s": round(time.perf_counter() - t0, 3)}
what = sys.argv[1] if len(sys.argv) > 1 else "both"
circs = suite.batch_workload(10000)
small = [c for c in circs if c.n_qubits <= 12]
large = [c for c in circs if c.n_qubits > 12]
t0 = time.perf_counter(); _lib.lib(); out["lib_s"] = round(time.perf_counter() - t0, 3)
for rep in range(2):
    if what in ("small", "both"):
        t0 = time.perf_counter(); batch.run_batch_codes(small, 1000, 0); out[f"small{rep}_s"] = round(time.perf_counter() - t0, 3)
    if what in ("large", "both"):
        t0 = time.perf_counter(); batch.run_batch_codes(large, 1000, 0); out[f"large{rep}_s"] = round(time.perf_counter() - t0, 3)
        out[f"large{rep}_timing"] = {k: (round(v, 3) if isinstance(v, float) else [round(x, 3) for x in v]) for k, v in batch.last_timing.items()}
print(json.dumps(out))
