"""Sycamore-32 c64 applies with nvidia-smi clock/power sampling (is the pass power-capped?)."""
import os, subprocess, sys, threading, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
samples = []
stop = False
def sampler():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append(out)
        time.sleep(0.05)
c = suite.sycamore_circuit(4, 8, 20, 0, measured=False)
g = sv.gate_array(c.instructions)
s = sv.DeviceState(32, "c64")
s.apply_gates(g); s.sync() if hasattr(s, "sync") else None
th = threading.Thread(target=sampler); th.start()
for _ in range(3):
    s.zero(); s.timer_start(); s.apply_gates(g); print("apply_ms", s.timer_stop())
stop = True; th.join()
print(json.dumps(samples[:40]))
