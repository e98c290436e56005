mkdir -p gpurun_out
for m in gc nogc freeze gc; do timeout 900 python tools/batch_time.py 4 $m 2>&1 | tail -1; done > gpurun_out/g31_bt.txt; cat gpurun_out/g31_bt.txt
