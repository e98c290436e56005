mkdir -p gpurun_out
rm -f gpurun_out/g33_trace.csv
SVB_BATCH_TRACE=gpurun_out/g33_trace.csv timeout 900 python tools/batch_time.py 5 gc > gpurun_out/g33_bt.txt 2>&1; tail -1 gpurun_out/g33_bt.txt
timeout 900 python tools/batch_time.py 5 gc > gpurun_out/g33_bt2.txt 2>&1; tail -1 gpurun_out/g33_bt2.txt
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/g33_tests.log 2>&1; tail -2 gpurun_out/g33_tests.log
