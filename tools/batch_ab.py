"""A/B of executor settings on fresh config-4 circuits (child processes)."""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    from paper_2512_04216_b200 import suite, batch
    batch.run_batch_codes(suite.batch_workload(200), 1000, 0)  # compile structures
    out = {}
    for base in (20000, 30000):
        fresh = suite.batch_workload(10000, base=base)
        t0 = time.perf_counter(); batch.run_batch_codes(fresh, 1000, 0); out[f"fresh{base}"] = round(time.perf_counter() - t0, 3)
    fresh = suite.batch_workload(10000, base=40000)
    t0 = time.perf_counter(); batch.run_batch_codes(fresh, 1000, 0, jit="none"); out["fresh_none"] = round(time.perf_counter() - t0, 3)
    print(json.dumps(out)); sys.exit(0)
res = {}
for name, env in (("pinned_heavy2", {}), ("pageable_heavy2", {"SVB_PINNED_UPLOAD": "0"}),
                  ("pinned_heavy8", {"SVB_BATCH_HEAVY": "8"}), ("pageable_heavy8", {"SVB_PINNED_UPLOAD": "0", "SVB_BATCH_HEAVY": "8"})):
    p = subprocess.run([sys.executable, __file__, "c"], env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    res[name] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-300:]
    print(name, res[name], flush=True)
