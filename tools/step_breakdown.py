"""Per-phase device time of the QFT-30 bench step (CUDA events on the library stream)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
c = suite.qft_bench_circuit(n); g = sv.gate_array(c.instructions); masks = [1 << q for q in range(n)]
s = sv.DeviceState(n, "c128")
for _ in range(3):
    s.zero(); s.apply_gates(g); s.expect_z(masks)
out = {}
for name, fn in (("zero", lambda: s.zero()), ("apply", lambda: s.apply_gates(g)), ("expect30", lambda: s.expect_z(masks)),
                 ("expect1", lambda: s.expect_z(masks[:1])), ("zero_apply", lambda: (s.zero(), s.apply_gates(g)))):
    s.timer_start(); t0 = time.perf_counter()
    for _ in range(5): fn()
    out[name + "_ms"] = round(s.timer_stop() / 5, 3); out[name + "_wall_ms"] = round((time.perf_counter() - t0) / 5 * 1e3, 3)
s.zero(); s.profile(True); s.apply_gates(g); p = s.profile_read()
out["passes_ms"] = round(p["pass_ms"], 3); out["perm_ms"] = round(p["perm_ms"], 3)
print(json.dumps(out))
