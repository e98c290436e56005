"""Config 4: 10,000 QAOA / VQE circuits of 12-24 qubits, 1000 shots each.

Times paper_2512_04216_b200.batch.run_batch end to end (host encoding,
device work, counts dicts) and prints circuits/s; `--cpu` also times the
oracle port (reference algorithm, 1 core) on one circuit per width and
extrapolates the sequential reference batch (batch.run_batch) to the full set.
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2512_04216_b200 import suite
from paper_2512_04216_b200.batch import run_batch, run_batch_codes, SMALL_MAX

ap = argparse.ArgumentParser()
ap.add_argument("--count", type=int, default=10000)
ap.add_argument("--shots", type=int, default=1000)
ap.add_argument("--precision", default="c128")
ap.add_argument("--workers", type=int, default=8)
ap.add_argument("--cpu", action="store_true")
a = ap.parse_args()
t0 = time.perf_counter()
circs = suite.batch_workload(a.count)
gen = time.perf_counter() - t0
ngates = sum(len([i for i in c.instructions if i.kind != "measure"]) for c in circs)
run_batch(circs[:64], shots=a.shots, seed=0, precision=a.precision, workers=a.workers)  # warm-up (pool, kernels)
t0 = time.perf_counter()
rc = run_batch_codes(circs, shots=a.shots, seed=0, precision=a.precision, nthreads=a.workers)
dt_codes = time.perf_counter() - t0
t0 = time.perf_counter()
res = run_batch(circs, shots=a.shots, seed=0, precision=a.precision, workers=a.workers)
dt = time.perf_counter() - t0
errs = sum(1 for r in res if isinstance(r, Exception))
small = sum(1 for c in circs if c.n_qubits <= SMALL_MAX[a.precision])
out = {"config": "batch_qaoa_vqe_12_24", "circuits": a.count, "shots": a.shots, "precision": a.precision,
       "wall_s": dt, "circuits_per_s": a.count / dt, "codes_wall_s": dt_codes, "codes_circuits_per_s": a.count / dt_codes, "gates_per_s": ngates / dt, "errors": errs,
       "smem_batched": small, "engine_path": a.count - small, "generation_s": gen}
if a.cpu:
    from oracle import sv_oracle as orc
    per_n = {}
    for n in range(12, 21):
        c = next(c for c in circs if c.n_qubits == n)
        t = time.perf_counter(); orc.run(c, a.shots, 0, qubit_cap=26); per_n[n] = time.perf_counter() - t
    for n in range(21, 25):
        per_n[n] = per_n[20] * 2 ** (n - 20)
    est = sum(per_n[c.n_qubits] for c in circs)
    out["cpu_reference_estimate_s"] = est
    out["cpu_sample"] = "oracle port, 1 core: one circuit per n = 12..20 timed, n = 21..24 extrapolated x2 per qubit"
print(json.dumps(out))
