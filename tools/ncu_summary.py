"""Condense ncu --set full reports of the fused pass into the JSON bench.py reads
(profiles/r01_ncu_qft30_pass_full.json): duration, DRAM bytes, pipe/issue/occupancy
and the top stall reasons.  usage: python tools/ncu_summary.py OUT.json X.ncu-rep [...]"""
import csv, io, json, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]

recs = []
for rep in sys.argv[2:]:
    h, rows = raw(rep)
    for i, r in enumerate(rows):
        g = lambda k: float(r[h.index(k)].replace(",", "")) if k in h and r[h.index(k)] not in ("", "n/a") else None
        stalls = sorted(((g(k), k.split("issue_stalled_")[1].split("_per_issue")[0]) for k in h
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                         and g(k)), reverse=True)[:8]
        recs.append({
            "kernel": "svb_jit (QFT-30 c128 fused pass)", "report": rep.split("/")[-1], "launch": i,
            "duration_ms": g("gpu__time_duration.sum"),
            "dram_read_bytes": g("dram__bytes_read.sum"), "dram_write_bytes": g("dram__bytes_write.sum"),
            "dram_throughput_pct": g("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "inst_executed": g("smsp__inst_executed.sum"), "registers": g("launch__registers_per_thread"),
            "smem_wavefronts_pct": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            "top_stalls": [[round(v, 2), k] for v, k in stalls],
            "units": "dram bytes in GB (ncu), duration in ms",
        })
json.dump(recs, open(sys.argv[1], "w"), indent=1)
print(json.dumps(recs[0], indent=1)[:1500])
