mkdir -p gpurun_out
for w in small large both; do SVB_BATCH_PROFILE=1 timeout 600 python tools/batch_cold.py $w 2>&1 | grep -v "^\[svb\] jit" | tail -6; done > gpurun_out/g35_cold.txt; cat gpurun_out/g35_cold.txt
