mkdir -p gpurun_out
timeout 600 python tools/syc_passes.py 32 > gpurun_out/g22_syc.txt 2>&1; tail -3 gpurun_out/g22_syc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_batch.py -q -x -k "c64 or float or batch or dense" > gpurun_out/g22_tests.log 2>&1; tail -3 gpurun_out/g22_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "syc" > gpurun_out/g22_full.log 2>&1; tail -3 gpurun_out/g22_full.log
