"""Per-pass device times of config-4 circuits at 20-24 qubits: interpreter vs NVRTC
passes, plus the CDF draw of 1000 shots (one circuit at a time, after warm-up)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
out = {}
for n in (20, 22, 24):
    for c in (suite.qaoa_line_circuit(n, 1, 0, False), suite.qaoa_line_circuit(n, 2, 0, False), suite.ry_ansatz_circuit(n, 2, 1, False)):
        g = sv.gate_array(c.instructions)
        rec = {}
        for mode, jm in (("interp", -1), ("jit", 0)):
            s = sv.DeviceState(n, "c128")
            s.set_option(2, jm)
            for _ in range(3):
                s.zero(); s.apply_gates(g)
            s.zero(); s.profile(True); s.timer_start(); s.apply_gates(g); t = s.timer_stop(); p = s.profile_passes(); s.profile(False)
            rec[mode] = {"apply_ms": round(t, 4), "pass_ms": [round(x["ms"], 4) for x in p]}
            words = np.array([1, 2, 3, 4], dtype=np.uint64)
            qs = list(range(n))
            s.sample_codes(qs, qs, 1000, words, 1)
            s.timer_start(); s.sample_codes(qs, qs, 1000, words, 1); rec[mode]["sample_ms"] = round(s.timer_stop(), 4)
            s.close()
        out[c.name] = rec
        print(c.name, json.dumps(rec), flush=True)
