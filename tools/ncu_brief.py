"""One-screen summary of an ncu --set full report (duration, pipes, issue, stalls, DRAM)."""
import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "local_load_bytes", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        print(rep.split("/")[-1], r[h.index("Kernel Name")] if "Kernel Name" in h else "")
        for k in KEYS:
            if k in h: print(f"  {k} = {r[h.index(k)]}")
        st = sorted(((float(r[i].replace(',', '')), k) for i, k in enumerate(h) if k.startswith("smsp__average_warps_issue_stalled_")
                     and k.endswith("_per_issue_active.ratio") and r[i] not in ("", "n/a")), reverse=True)[:8]
        print("  stalls", [(round(v, 2), k.split("stalled_")[1].split("_per")[0]) for v, k in st])
