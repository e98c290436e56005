"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel: launches, total, share.
usage: python tools/launch_summary.py launches.csv "<command description>" > profiles/X.csv"""
import csv, collections, sys
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")) if r]
h = rows[0]
ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0].strip()
    v = float(r[iv].replace(",", ""))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[iu], 1.0)
    tot[name] += v * scale; cnt[name] += 1
T = sum(tot.values())
print(f"# ncu launch list of `{sys.argv[2] if len(sys.argv) > 2 else ''}` (--clock-control none;")
print("# cold-cache serialised times: compare shares, not absolutes)")
print("kernel,launches,total_us,share")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k},{cnt[k]},{v:.1f},{v / T:.3f}")
