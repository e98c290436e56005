import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import statevector as sv, suite
n = int(sys.argv[1]); shots = int(sys.argv[2]); mode = int(sys.argv[3])
c = suite.sycamore_circuit(4, n // 4, 4, 0) if n > 20 else suite.ghz_circuit(n)
s = sv.DeviceState(n, "c64" if n > 20 else "c128"); s.apply_instructions(c.instructions)
for _ in range(2):
    t0 = time.perf_counter(); s.sample_codes(list(range(n)), list(range(n)), shots, sv.pcg_words(1), mode); print("sample s", time.perf_counter() - t0)
