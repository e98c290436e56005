"""Dense k-qubit block passes at n qubits (default 30): tensor-core engine vs
CUDA-core engine, device time per pass (CUDA events on the state's stream),
achieved HBM GB/s against the 2*s*2^n algorithmic bytes, and the FMA-pipe
floor of the CUDA-core engine (4*2^k FMA per amplitude).  JSON lines."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2512_04216_b200 import statevector as sv

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
rng = np.random.default_rng(0)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6534.5
FMA_RATE = 148 * 128 * 1.965e9  # FP32 FMA lanes / s (FP64: half)

def unitary(k):
    z = rng.normal(size=(1 << k, 1 << k)) + 1j * rng.normal(size=(1 << k, 1 << k))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))

for prec in ("c64", "c128"):
    s = sv.DeviceState(n, prec)
    s.apply_instructions([])
    from paper_2512_04216_b200.circuit import Instruction
    s.apply_instructions([Instruction("h", (q,)) for q in range(n)])
    nbytes = 2 * (8 if prec == "c64" else 16) * (1 << n)
    for k in range(1, 7):
        for engine in ("tensor", "fma"):
            if engine == "tensor" and (prec != "c64" or not 3 <= k <= 6):
                continue
            if prec == "c128" and k > 5:
                continue
            for placement in ("low", "mixed"):
                q = {"low": list(range(k)), "high": list(range(n - k, n)),
                     "mixed": [int(x) for x in rng.choice(n, size=k, replace=False)]}[placement]
                U = unitary(k)
                s.apply_matrix(q, U, engine=engine)  # warm-up
                s.timer_start()
                for _ in range(reps):
                    s.apply_matrix(q, U, engine=engine)
                ms = s.timer_stop() / reps
                gbs = nbytes / (ms / 1e3) / 1e9
                fma_floor = (1 << n) * 4 * (1 << k) / (FMA_RATE / (2 if prec == "c128" else 1)) * 1e3
                print(json.dumps({"n": n, "precision": prec, "k": k, "engine": engine, "qubits": placement,
                                  "ms": round(ms, 4), "gbs": round(gbs, 1), "frac_hbm": round(gbs / peak, 3),
                                  "hbm_floor_ms": round(nbytes / peak / 1e6, 3), "fma_floor_ms": round(fma_floor, 3)}),
                      flush=True)
    s.close()
