mkdir -p gpurun_out
timeout 900 python tools/batch_pass_probe.py > gpurun_out/g30_passes.txt 2>&1; cut -c1-200 gpurun_out/g30_passes.txt | grep -o '^[a-z_0-9]*\|"sample_ms": [0-9.]*' | paste - - - | head -9
timeout 900 python tools/batch_time.py 3 > gpurun_out/g30_bt.txt 2>&1; tail -1 gpurun_out/g30_bt.txt
timeout 900 python -m pytest tests/test_gpu_sampling_large.py tests/test_gpu_batch.py tests/test_gpu_parity.py -q -x -k "cdf or sampl or batch or ghz or counts or chi" > gpurun_out/g30_tests.log 2>&1; tail -2 gpurun_out/g30_tests.log
