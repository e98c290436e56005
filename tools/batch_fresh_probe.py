"""Why new circuits of a compiled structure cost more: 24- and 23-qubit
subsets of a fresh config-4 set, per jit mode, with SVB_TRACE timings."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import suite, batch

def timed(fn):
    t0 = time.perf_counter(); fn(); return time.perf_counter() - t0

warm = suite.batch_workload(200)
batch.run_batch_codes(warm, 1000, 0)  # compiles the 24-qubit structures
out = {}
for base in (20000, 30000, 40000):
    fresh = suite.batch_workload(2600, base=base)
    for n in (24, 23):
        sub = [c for c in fresh if c.n_qubits == n]
        for jit in (("sync", "none") if base == 20000 else ("none", "sync")):
            key = f"base{base}_n{n}_{jit}"
            out[key] = {"circuits": len(sub), "s": timed(lambda: batch.run_batch_codes(sub, 1000, 0, jit=jit))}
            for nt in (1,):
                out[key + "_1thread"] = {"s": timed(lambda: batch.run_batch_codes(sub, 1000, 0, jit=jit, nthreads=1))}
print(json.dumps(out, indent=0))
