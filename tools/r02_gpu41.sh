mkdir -p gpurun_out
timeout 600 python tools/host_gap.py 2>&1 | tail -5
SVB_TRACE=1 timeout 600 python tools/host_gap.py 2>&1 | grep "n=30" | tail -3
