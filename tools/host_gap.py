"""Host-side share of the QFT-30 bench step: SVB_TRACE apply host/sync split, and
step time vs the sum of the pass times, profiler on and off (run under gpurun)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
n = 30
c = suite.qft_bench_circuit(n); g = sv.gate_array(c.instructions); zq = list(range(n))
s = sv.DeviceState(n, "c128")
for _ in range(4):
    s.zero(); s.apply_gates_z(g, zq)
t = []
for _ in range(10):
    t0 = time.perf_counter(); s.zero(); t1 = time.perf_counter(); s.apply_gates_z(g, zq); t2 = time.perf_counter()
    t.append((t1 - t0, t2 - t1))
print("zero_ms", [round(a * 1e3, 3) for a, _ in t]); print("apply_z_wall_ms", [round(b * 1e3, 3) for _, b in t])
for prof in (False, True, False):
    s.profile(prof)
    s.timer_start()
    for _ in range(20):
        s.zero(); s.apply_gates_z(g, zq)
    ms = s.timer_stop() / 20
    extra = ""
    if prof:
        pp = s.profile_passes(); extra = f" passes_sum_ms {sum(p['ms'] / max(p['launches'], 1) for p in pp):.3f}"
    print(f"device_step_ms profile={prof} {ms:.3f}{extra}", flush=True)
    s.profile(False)
