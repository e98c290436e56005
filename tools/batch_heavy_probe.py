"""Concurrency of L2-overflowing (24-qubit) circuits in svb_batch_run."""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:  # child: one setting
    from paper_2512_04216_b200 import suite, batch
    batch.run_batch_codes(suite.batch_workload(200), 1000, 0)  # compile
    out = {}
    for base in (20000, 30000):
        fresh = suite.batch_workload(10000, base=base)
        sub = [c for c in fresh if c.n_qubits == 24]
        for jit in ("sync", "none"):
            t0 = time.perf_counter(); batch.run_batch_codes(sub, 1000, 0, jit=jit); out[f"n24_{base}_{jit}"] = time.perf_counter() - t0
        t0 = time.perf_counter(); batch.run_batch_codes(fresh, 1000, 0); out[f"all_{base}_sync"] = time.perf_counter() - t0
    print(json.dumps(out))
    sys.exit(0)
res = {}
for h in ("1", "2", "4", "8"):
    env = dict(os.environ, SVB_BATCH_HEAVY=h)
    p = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True, timeout=900)
    res[h] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-500:]
print(json.dumps(res, indent=0))
