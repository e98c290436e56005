"""Config-4 batch breakdown: cold vs warm run_batch_codes, host encoding,
per-width device time, dict formatting."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2512_04216_b200 import suite, batch, statevector as sv

circs = suite.batch_workload(10000)
t0 = time.perf_counter(); batch.run_batch_codes(circs, 1000, 0); cold = time.perf_counter() - t0
t0 = time.perf_counter(); r = batch.run_batch_codes(circs, 1000, 0); warm = time.perf_counter() - t0
large = [c for c in circs if c.n_qubits > 12]
t0 = time.perf_counter(); sv.gate_ops_many(large); enc = time.perf_counter() - t0
out = {"cold_s": cold, "warm_s": warm, "encode_large_s": enc, "per_width": {}}
for n in range(12, 25):
    sub = [c for c in circs if c.n_qubits == n]
    t0 = time.perf_counter(); batch.run_batch_codes(sub, 1000, 0); out["per_width"][n] = time.perf_counter() - t0
for nt in (2, 4, 16):
    t0 = time.perf_counter(); batch.run_batch_codes(circs, 1000, 0, nthreads=nt); out[f"warm_nthreads{nt}_s"] = time.perf_counter() - t0
t0 = time.perf_counter(); d = [x.to_dict() for x in r]; out["dicts_s"] = time.perf_counter() - t0
print(json.dumps(out))
