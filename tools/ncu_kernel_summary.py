"""Condense ncu --set full reports into JSON: duration, DRAM bytes, issue /
warp occupancy, FMA / FP64 / tensor pipes, tcgen05 instruction counts, top
stall reasons.  usage: python tools/ncu_kernel_summary.py OUT.json LABEL=X.ncu-rep [...]"""
import csv, io, json, subprocess, sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_GB": "dram__bytes_read.sum",
    "dram_write_GB": "dram__bytes_write.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct_elapsed": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "tc_smem_wavefronts_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lsu_smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "utcmma_executed": "smsp__sass_inst_executed_op_utcmma.sum",
    "tmem_ld_executed": "smsp__sass_inst_executed_op_tmem_ldt.sum",
}

recs = []
for arg in sys.argv[2:]:
    label, rep = arg.split("=", 1)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        def g(k):
            try:
                v = r[h.index(k)]
                return float(v.replace(",", "")) if v not in ("", "n/a") else None
            except ValueError:
                return None
        rec = {"label": label, "report": rep.split("/")[-1], "kernel": r[h.index("Kernel Name")] if "Kernel Name" in h else None}
        for name, key in KEYS.items():
            rec[name] = g(key)
        stalls = sorted(((g(k), k.split("issue_stalled_")[1].split("_per_issue")[0]) for k in h
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                         and g(k)), reverse=True)[:6]
        rec["top_stalls"] = [[round(v, 2), k] for v, k in stalls]
        recs.append(rec)
json.dump(recs, open(sys.argv[1], "w"), indent=1)
for r in recs:
    print(json.dumps({k: r[k] for k in ("label", "duration_ms", "dram_read_GB", "dram_write_GB", "tensor_pipe_pct_elapsed",
                                         "issue_active_pct", "top_stalls")}))
