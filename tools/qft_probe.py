"""Per-pass timings of QFT-30 c128 (zero-start and dense input, with and without the
fused <Z>), and Sycamore-32 c64; run with SVB_TRACE=1 for launch shapes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite

def run(name, s, fn, reps=3):
    fn()
    s.profile(True)
    s.timer_start()
    for _ in range(reps):
        fn()
    ms = s.timer_stop() / reps
    pp = s.profile_passes()
    s.profile(False)
    print(json.dumps({"exp": name, "ms": round(ms, 3),
                      "passes_ms": [round(p["ms"] / max(p["launches"], 1), 3) for p in pp]}), flush=True)

which = sys.argv[1:] or ["qft", "syc"]
if "qft" in which:
    n = 30
    g = sv.gate_array(suite.qft_bench_circuit(n).instructions)
    zq = list(range(n))
    s = sv.DeviceState(n, "c128")
    run("qft30_zero_z", s, lambda: (s.zero(), s.apply_gates_z(g, zq)))
    run("qft30_zero_noz", s, lambda: (s.zero(), s.apply_gates(g)))
    run("qft30_dense_z", s, lambda: s.apply_gates_z(g, zq))
    run("qft30_dense_noz", s, lambda: s.apply_gates(g))
    s.close()
if "syc" in which:
    n = 32
    g = sv.gate_array(suite.sycamore_circuit(4, 8, 20, 0, measured=False).instructions)
    s = sv.DeviceState(n, "c64")
    run("syc32_zero", s, lambda: (s.zero(), s.apply_gates(g)), reps=2)
    run("syc32_dense", s, lambda: s.apply_gates(g), reps=2)
    s.close()
