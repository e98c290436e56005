import sys, time, json
sys.path.insert(0,'.')
from paper_2512_04216_b200 import statevector as sv, suite, _lib
import numpy as np
def run(name, c, n, prec, jit):
    g = sv.gate_array(c.instructions)
    s = sv.DeviceState(n, prec); s.set_option(_lib.OPT_JIT_MIN_N, 1 if jit else -1)
    t=time.time(); s.apply_gates(g); first=time.time()-t
    s.apply_gates(g)
    s.profile(True); s.timer_start()
    for _ in range(3): s.apply_gates(g)
    tot = s.timer_stop()/3; p = s.profile_read(); s.close()
    print(json.dumps({"exp": name, "jit": jit, "first_call_s": round(first,2), "ms": round(tot,2), "pass_ms": round(p["pass_ms"]/max(p["pass_launches"],1),3), "passes": p["pass_launches"]//3}), flush=True)
for jit in (False, True):
    run("qft30", suite.qft_bench_circuit(30), 30, "c128", jit)
    c = __import__('paper_2512_04216_b200.circuit', fromlist=['Circuit']).Circuit(30)
    for q in range(23, 30): c.gate("h", q)
    run("h7_top", c, 30, "c128", jit)
    run("syc32_d4", suite.sycamore_circuit(4, 8, 4, 0, measured=False), 32, "c64", jit)
