mkdir -p gpurun_out
nproc; grep -m1 "model name" /proc/cpuinfo; uptime
rm -f gpurun_out/g32_trace.csv
SVB_BATCH_TRACE=gpurun_out/g32_trace.csv timeout 900 python tools/batch_time.py 5 gc > gpurun_out/g32_bt.txt 2>&1; tail -1 gpurun_out/g32_bt.txt
