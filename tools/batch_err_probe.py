import sys, os
sys.path.insert(0, '.')
from paper_2512_04216_b200 import suite
from paper_2512_04216_b200.batch import run_batch
circs = suite.batch_workload(400)
res = run_batch(circs, shots=1000, seed=0, sampler="cdf")
for c, r in zip(circs, res):
    if isinstance(r, Exception): print(c.name, c.n_qubits, type(r).__name__, str(r)[:300])
print("done")
