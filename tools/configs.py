"""End-to-end timings of the BASELINE.json configs through the public API."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2512_04216_b200 import statevector as sv, suite

def timeit(fn, reps):
    fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); t.append(time.perf_counter() - t0)
    return min(t), float(np.median(t))

which = sys.argv[1:] or ["ghz20", "syc32", "qft30"]
if "ghz20" in which:
    c = suite.ghz_circuit(20)
    for sampler in ("alias", "cdf"):
        best, med = timeit(lambda: sv.run(c, 1024, 7, sampler=sampler), 5)
        print(json.dumps({"config": "ghz20_1024_shots", "sampler": sampler, "best_ms": best * 1e3, "median_ms": med * 1e3,
                          "gates_per_s": 20 / best}))
if "syc32" in which:
    n = 32
    c = suite.sycamore_circuit(4, 8, 20, 0)
    g = sv.gate_array(c.instructions)
    s = sv.DeviceState(n, "c64")
    t0 = time.perf_counter(); s.apply_gates(g); first = time.perf_counter() - t0  # lazy zero: compiles
    s.apply_gates(g)  # written state: the dense-input program compiles too
    s.profile(True); s.timer_start(); s.apply_gates(g); ms_dense = s.timer_stop(); s.profile(False)
    s.profile(True); s.zero(); s.timer_start(); s.apply_gates(g); ms_apply = s.timer_stop(); p = s.profile_read()
    qubits = list(range(n)); src = list(range(n))
    for shots in (10**6,):
        s.sample_codes(qubits, src, shots, sv.pcg_words(2), 1)  # first call grows the stream-ordered pool
        s.timer_start(); codes, freq = s.sample_codes(qubits, src, shots, sv.pcg_words(1), 1); ms_s = s.timer_stop()
        print(json.dumps({"config": "sycamore32_d20_c64", "gates": int(g.size), "first_apply_s": first, "apply_ms": ms_apply, "apply_dense_input_ms": ms_dense,
                          "passes": p["pass_launches"], "pass_ms_mean": p["pass_ms"] / max(p["pass_launches"], 1),
                          "gates_per_s": g.size / (ms_apply / 1e3), "shots": shots, "sample_ms": ms_s,
                          "shots_per_s": shots / (ms_s / 1e3), "distinct": int(codes.size)}))
    t0 = time.perf_counter(); res = sv.run(c, 10**6, 1, qubit_cap=32, precision="c64", sampler="cdf"); e2e = time.perf_counter() - t0
    print(json.dumps({"config": "sycamore32_d20_c64_e2e_run", "s": e2e, "distinct": len(res.counts)}))
