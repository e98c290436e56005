"""Config-4 batch breakdown: first call (cold NVRTC), a repeat of the same
circuits, a fresh set of 10,000 circuits with the same structures (the
steady state for new circuits), the interpreter-only mode, per-width times,
host encoding and dict formatting."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import suite, batch, statevector as sv

def timed(fn):
    t0 = time.perf_counter(); r = fn(); return time.perf_counter() - t0, r

circs = suite.batch_workload(10000)
fresh = suite.batch_workload(10000, base=10000)
out = {}
out["first_call_s"], _ = timed(lambda: batch.run_batch_codes(circs, 1000, 0))
out["repeat_same_circuits_s"], _ = timed(lambda: batch.run_batch_codes(circs, 1000, 0))
out["fresh_circuits_s"], r = timed(lambda: batch.run_batch_codes(fresh, 1000, 0))
out["fresh_circuits_jit_none_s"], _ = timed(lambda: batch.run_batch_codes(fresh, 1000, 1, jit="none"))
out["encode_large_s"], _ = timed(lambda: sv.gate_ops_many([c for c in fresh if c.n_qubits > 12]))
out["per_width_fresh_s"] = {}
for n in range(12, 25):
    sub = [c for c in fresh if c.n_qubits == n]
    out["per_width_fresh_s"][n], _ = timed(lambda: batch.run_batch_codes(sub, 1000, 2))
out["dicts_s"], _ = timed(lambda: [x.to_dict() for x in r])
print(json.dumps(out))
