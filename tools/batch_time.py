"""Config-4 wall time on fresh circuits (default jit mode), N repetitions, one process.
usage: batch_time.py [reps] [gc|nogc|freeze]"""
import gc, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04216_b200 import suite, batch
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mode = sys.argv[2] if len(sys.argv) > 2 else "gc"
out = {"mode": mode}
sets = [suite.batch_workload(10000, base=10000 * r) for r in range(reps + 1)]
if mode == "freeze":
    gc.collect(); gc.freeze()
for r in range(reps + 1):
    if mode == "nogc":
        gc.disable()
    g0 = gc.get_stats()[2]["collections"]
    t0 = time.perf_counter(); batch.run_batch_codes(sets[r], 1000, 0); dt = time.perf_counter() - t0
    out["first_call_s" if r == 0 else f"fresh{r}_s"] = round(dt, 3)
    out[f"timing_{r}"] = {k: (round(v, 3) if isinstance(v, float) else [round(x, 3) for x in v]) for k, v in batch.last_timing.items()}
    gc.enable()
print(json.dumps(out))
